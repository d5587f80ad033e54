#!/usr/bin/env python
"""bench.py — sustained TFLOPS and time-to-solution of the sliced tensor-network
contraction (BASELINE.json metric) on synthetic Sycamore-53 m=18 slices.

A *step* is one pass of the whole hot path (slice select -> every pairwise
contraction of the path -> fused fp64 slice accumulation) over one slice per
GPU.  Slices are independent, so ranks take disjoint
slices with no data-path collective ("scaling": "weak"); the one reduce of the
slice sums happens once per job, after the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.  ``value`` = Σ over all ranks of the Eq. 4
T_cc of the slices processed ÷ the max-over-ranks device time of the K timed
steps.  ``--impl reference`` times the CPU fp64 oracle (the baseline arm of
this tier) on bounded sub-slice samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sustained TFLOPS/GPU and time-to-solution (Sycamore m=18 slices) at 1/2/4/8 B200"
PAPER_M18_TCC = 6.55e20       # paper's whole m=18 job: 2^23 sub-tasks x 7.81e13 flop


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c4", "c5", "c3", "c2"])
    # headline: the paper's sampling boundary (2^16 uniform samples) with
    # per-slice intermediates up to 2^32 elements (32 GiB: sized for 180 GB of HBM3e;
    # DESIGN.md §3 "Why peak 2^32"); --boundary single is the secondary line
    ap.add_argument("--boundary", default="sparse16")
    ap.add_argument("--peak", type=int, default=32)
    ap.add_argument("--order-tag", default="a64", help="order file variant (tools/make_orders.py)")
    ap.add_argument("--precision", default="extended", choices=["extended", "mixed"])
    ap.add_argument("--topk", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph-pass", action="store_true", help="skip the graph-replay timing pass")
    ap.add_argument("--cpu-flops", type=float, default=6e11,
                    help="target T_cc of one oracle sub-slice sample")
    return ap.parse_args(argv)


def load_workload(args):
    from tnworkloads import configs
    if args.workload == "c2":
        return configs.c2()
    if args.workload == "c3":
        return configs.c3()
    if args.workload == "c5":
        return configs.c5("single" if args.boundary == "sparse16" else args.boundary, args.peak,
                          args.order_tag)
    return configs.c4(args.boundary, args.peak, args.order_tag)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "power.draw"]

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


# ----------------------------------------------------------------------------- cpu oracle

def oracle_sample(w, target_flops, time_cap_s=60.0):
    """Time the CPU oracle (as it stands) on one bounded sub-slice of the workload."""
    import numpy as np
    import oracle
    from tnworkloads.paths import slice_greedy, path_cost
    pc = path_cost(w.net, w.samples, w.path, w.sliced)
    extra = []
    fine = list(w.sliced)
    if pc.flops_per_slice > target_flops:
        # refine slice 0 with extra bonds (the workload's own sliced bonds stay first,
        # so sub-slice 0 lies inside slice 0)
        from tnworkloads.treesa import refine_slices
        fine, _ = refine_slices(w.net, w.samples, w.path, w.sliced, target_flops, max_extra=48)
        extra = fine[len(w.sliced):]
    pcs = path_cost(w.net, w.samples, w.path, fine)
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    # every host core for the oracle's BLAS, also under torchrun (which sets
    # OMP_NUM_THREADS=1 per rank); `cores` reports the thread count actually set
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        oracle.contract_slice(w.net, w.path, fine, 0, w.samples)
        dt = time.perf_counter() - t0
    return {"flops": pcs.flops_per_slice, "seconds": dt, "cores": threads,
            "sample": f"oracle (numpy complex128 tensordot) on sub-slice 0 of slice 0 of {w.name}: "
                      f"{len(extra)} extra sliced bonds, T_cc {pcs.flops_per_slice:.3g} flop"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = load_workload(args)
    steps = []
    for s in range(args.warmup + args.steps):
        r = oracle_sample(w, args.cpu_flops)
        if s >= args.warmup:
            steps.append(r)
    secs = sum(r["seconds"] for r in steps)
    flops = sum(r["flops"] for r in steps)
    v = flops / secs / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOPS",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": w.name, "sample": "one oracle sub-slice per step"},
            "cpu_baseline": {"value": v, "unit": "TFLOPS", "cores": steps[0]["cores"],
                             "kind": "oracle", "sample": steps[0]["sample"]},
            "e2e": {"value": v, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- ours

def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2310_03978_b200 import Contraction

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    w = load_workload(args)
    ctx = Contraction(device=local, stream=stream)
    n_slices = ctx.setup(w.net, w.samples, w.path, w.sliced)
    info = ctx.info()
    steps_total = args.warmup + args.steps

    def slice_of(step):
        return (step * world + rank) % n_slices

    def barrier():
        if world > 1:
            dist.barrier()

    with torch.cuda.stream(stream):
        for s in range(args.warmup):
            ctx.contract(slice_of(s), slice_of(s) + 1, args.precision, args.topk)
        stream.synchronize()
        ctx.reset_kernel_stats()
        ctx.set_profiling(True)
        barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(local)
        sampler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.warmup, steps_total):
            ctx.contract(slice_of(s), slice_of(s) + 1, args.precision, args.topk)
        e1.record(stream)
        stream.synchronize()
        clocks = sampler.stop()
        torch.cuda.synchronize()
        barrier()
        ms_local = e0.elapsed_time(e1)
        stats = ctx.kernel_stats()
        step_ms = ctx.step_stats(-1)
        ctx.set_profiling(False)
    # the same slices again without per-launch events: every slice after the first
    # replays the captured CUDA graph of the per-slice launch sequence (product path)
    graph = None
    if not args.no_graph_pass:
        with torch.cuda.stream(stream):
            r0 = ctx.info()["graph_replays"]
            barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            for s in range(args.warmup, steps_total):
                ctx.contract(slice_of(s), slice_of(s) + 1, args.precision, args.topk)
            g1.record(stream)
            stream.synchronize()
            graph = {"ms_per_step": g0.elapsed_time(g1) / args.steps,
                     "graph_replays": ctx.info()["graph_replays"] - r0,
                     "note": "same slices as the timed region, no per-launch events, CUDA-graph "
                             "replay of the per-slice launch sequence; the accumulator double-"
                             "counts these slices, so the reduce below is only a timing check"}
    plan_steps = ctx.plan_json()["steps"]
    top_steps = []
    for s_ in np.argsort(-step_ms)[:16]:
        p_ = plan_steps[int(s_)]
        top_steps.append({"step": int(s_), "ms_per_slice": float(step_ms[s_]) / args.steps,
                          "route": p_["route"] + ("/grouped" if p_.get("grouped") else ""),
                          "J": p_["J"], "m": p_["m"], "n": p_["n"], "k": p_["k"],
                          "tflops": p_["tcc"] * args.steps / max(step_ms[s_], 1e-9) / 1e9})
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # the job's single collective: sum of the per-rank fp64 slice sums (NCCL)
    from paper_2310_03978_b200.distributed import reduce_amplitudes
    t_red = time.perf_counter()
    amps = reduce_amplitudes(ctx, world)
    torch.cuda.synchronize()
    reduce_ms = (time.perf_counter() - t_red) * 1e3

    flops_step = info["flops_per_slice"] * world
    value = flops_step * args.steps / (ms / 1e3) / 1e12
    ms_per_step = ms / args.steps
    peaks, peak_src = measured_peaks()
    g = stats["gemm_tcgen05"]
    launches = sum(v["launches"] for v in stats.values())
    roofline = None
    if g["ms"] > 0:
        achieved = g["flops"] / (g["ms"] / 1e3) / 1e12
        peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
        traffic = None
        tf = os.path.join(ROOT, "profiles", "gemm_traffic.json")
        if os.path.exists(tf):
            try:
                traffic = json.load(open(tf)).get("bytes_per_launch")
            except (OSError, ValueError):
                traffic = None
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "kernel": "cgemm_tcgen05_kernel",
                    "peak_source": f"{peak_src} bf16 dense sustained (= fp16 dense rate)",
                    "passes": 3 if args.precision == "extended" else "mixed",
                    "tensor_pipe_frac": achieved * (3 if args.precision == "extended" else 1) / peak,
                    "share_of_step": g["ms"] / ms_local if ms_local > 0 else None,
                    "launches": g["launches"]}

    e2e = None
    if not args.no_e2e:
        ranks_, labels_, dims_, data_, opens_ = w.net.flat()
        host = np.ascontiguousarray(data_)
        n_e2e = max(1, min(args.steps, 5))
        ctx.reset_accumulator()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        marks = []
        for s in range(n_e2e):
            ctx.upload_tensors(host)                     # h2d of the network tensors
            with torch.cuda.stream(stream):
                ctx.contract(slice_of(s), slice_of(s) + 1, args.precision, args.topk)
            res = ctx.sum_slices_host()                  # d2h of the amplitudes
            marks.append(time.perf_counter())
        dt = marks[-1] - t0
        if world > 1:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e_ms = [round((b_ - a_) * 1e3, 1) for a_, b_ in zip([t0] + marks[:-1], marks)]
        e2e = {"value": info["flops_per_slice"] * n_e2e / dt / 1e12 * world, "unit": "TFLOPS",
               "h2d_bytes_per_step": int(host.size * 8), "d2h_bytes_per_step": int(res.size * 16),
               "steps": n_e2e, "step_ms": e2e_ms}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_sample(w, args.cpu_flops)
        cpu = {"value": r["flops"] / r["seconds"] / 1e12, "unit": "TFLOPS", "cores": r["cores"],
               "kind": "oracle", "sample": r["sample"], "seconds": r["seconds"]}

    if rank == 0:
        t_slice = ms_per_step / 1e3                          # s per slice per GPU
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "fp16x3 (hi/lo split, fp32 chunk-promoted accumulate, fp64 slice sum)"
            if args.precision == "extended" else f"fp16 top-{args.topk} / fp16x3 rest",
            "data": "synthetic",
            "config": {"workload": w.name, "precision": args.precision,
                       "slices_per_step_per_gpu": 1, "n_slices": n_slices,
                       "flops_per_slice": info["flops_per_slice"],
                       "tc_flops_share": info["tc_flops_per_slice"] / info["flops_per_slice"],
                       "peak_intermediate_elements": info["peak_elements"],
                       "n_steps_path": info["n_steps"], "n_tc_steps": info["n_tc_steps"],
                       "l2": "per-slice working set (GBs of intermediates) >> 126 MB L2; no flush",
                       "parallelism": f"slices x{world}"},
            "tflops_per_gpu": value / world,
            "time_to_solution": {
                "measured_path_s": t_slice * n_slices / world,
                "paper_m18_Tcc_normalised_s": PAPER_M18_TCC / (value * 1e12),
                "note": "measured_path = this workload's slices x s/slice / GPUs; normalised = "
                        "paper's 6.55e20 flop m=18 job / this run's aggregate TFLOPS"},
            "roofline": roofline,
            "kernel_stats": stats,
            "top_steps": top_steps,
            "gpu_launches": launches,
            "cuda_graph": graph,
            "clocks": clocks,
            "reduce_ms": reduce_ms,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args, argv):
    """``--gpus N`` (N > 1) outside torchrun: re-launch this script as N ranks (one
    process per GPU) under torch.distributed.run on 127.0.0.1, exactly as the driver
    does; returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args, argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
