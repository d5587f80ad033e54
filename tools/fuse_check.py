"""C2 slice 5 with the fused plane output on / columns-only / off (GPU), compared."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2310_03978_b200 import Contraction
from tnworkloads import configs
w = configs.c2()
c = Contraction(device=0, stream=torch.cuda.current_stream())
c.setup(w.net, w.samples, w.path, w.sliced)
c.contract(5, 6)
np.save(sys.argv[1], c.sum_slices_host())
print(sum(s["planes_out"] for s in c.plan_json()["steps"]))
''' % ROOT
res = {}
for tag, env in [("on", "1"), ("cols", "2"), ("off", "0")]:
    out = f"/tmp/c2_{tag}.npy"
    r = subprocess.run([sys.executable, "-c", CODE, out], env=dict(os.environ, TN_FUSE_PLANES=env),
                       capture_output=True, text=True)
    print(tag, "fused edges:", r.stdout.strip(), r.stderr[-300:])
    res[tag] = np.load(out)
for a in ("on", "cols"):
    print(a, "vs off: rel_l2 %.3e" % (np.linalg.norm(res[a] - res["off"]) / np.linalg.norm(res["off"])))
