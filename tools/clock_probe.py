#!/usr/bin/env python
"""Is a long batch of steps slower per step than short ones, and why?
For each path: CUDA-event time per step over K back-to-back steps for K in
(1, 10, 50, 200), with nvidia-smi SM clock / power / throttle reasons sampled
during each batch (bench.ClockSampler).

    python tools/clock_probe.py [--n 512]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2503_07898_b200 as V  # noqa: E402
from bench import ClockSampler  # noqa: E402


def measure(name, step, ks=(1, 10, 50, 200), reps=3):
    out = {"path": name, "lib": os.environ.get("VOXL_TAG", "")}
    cs = ClockSampler(0)
    time.sleep(0.3)
    step(3)
    torch.cuda.synchronize()
    for k in ks:
        best, worst, clocks = 1e9, 0.0, None
        for _ in range(reps):
            t0 = time.time()
            ts = time.perf_counter()
            step(k)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - ts) * 1e3 / k
            t1 = time.time()
            best, worst = min(best, ms), max(worst, ms)
            clocks = cs.summary(t0, t1)
        out[f"k{k}"] = {"best_ms": round(best, 4), "worst_ms": round(worst, 4), "clocks": clocks}
    cs.stop()
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--only", default="", help="dense: the dense paths only")
    ap.add_argument("--ks", default="1,10,50,200", help="batch lengths (dense and block-sparse)")
    a = ap.parse_args()
    ks = tuple(int(x) for x in a.ks.split(","))
    n = a.n
    dom = (n, n, n)
    torch.cuda.init()
    e = V.DenseEngine(domain=dom, precision="fp32")
    e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
    measure("dense", e.step, ks=ks)
    measure("dense_probe_n", e.step_probe_n, ks=ks)
    e.close()
    if a.only == "dense":
        return
    s = V.SparseEngine(dom, V.obstacle_mask(dom), block_edge=8, strategy="disag_mem", precision="fp32")
    measure("sparse_disag_mem", s.step, ks=ks)
    measure("sparse_disag_mem_probe_n", s.step_probe_n, ks=ks)
    s.close()
    m = V.MultiResEngine(dom, 3, fused=True, precision="fp32")
    measure("multires_fused", m.step, ks=(1, 5, 20, 50))
    measure("multires_fused_probe_n", m.step_probe_n, ks=(1, 5, 20, 50))
    m.close()


if __name__ == "__main__":
    main()
