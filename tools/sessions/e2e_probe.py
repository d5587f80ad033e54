"""Time the parts of bench.py's e2e loop separately (upload / contract / host read)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
sys.argv = ["bench.py"]
import bench
from paper_2310_03978_b200.tn import Contraction

args = bench.parse()
w = bench.load_workload(args)
stream = torch.cuda.Stream()
ctx = Contraction(device=0, stream=stream)
ctx.setup(w.net, w.samples, w.path, w.sliced)
_, _, _, data_, _ = w.net.flat()
host = np.ascontiguousarray(data_)
with torch.cuda.stream(stream):
    for s in range(3):
        ctx.contract(s, s + 1)
    stream.synchronize()
    for mode in ("plain", "upload", "upload+read"):
        for s in range(3):
            t0 = time.perf_counter()
            if "upload" in mode:
                ctx.upload_tensors(host)
            t1 = time.perf_counter()
            ctx.contract(s, s + 1)
            t2 = time.perf_counter()
            stream.synchronize()
            t3 = time.perf_counter()
            if "read" in mode:
                ctx.sum_slices_host()
            t4 = time.perf_counter()
            print(mode, s, "upload %.1f launch %.1f sync %.1f read %.1f total %.1f ms" % (
                (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t4 - t0) * 1e3),
                "replays", ctx.info()["graph_replays"], flush=True)
