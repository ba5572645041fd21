#!/usr/bin/env python
"""step(k) vs step_probe_n(k) per-step wall time at 512^3 fp32, short batches
(k = 20, below the pod's power-cap onset), best of 5, alternating -- the
fused-probe overhead of run()'s loop for each engine.

    python tools/probe_overhead.py [--n 512] [--k 20] [--paths dense,sparse,multires]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_07898_b200 as V  # noqa: E402


def best(fn, k, reps=5):
    out = []
    for _ in range(reps):
        t = time.perf_counter()
        fn(k)
        out.append((time.perf_counter() - t) / k * 1e3)
        time.sleep(0.05)
    return min(out)


def compare(name, eng, step, probe_n, k):
    step(2)
    probe_n(2)
    a, b = [], []
    for _ in range(3):
        a.append(best(step, k))
        b.append(best(probe_n, k))
    s, p = min(a), min(b)
    print(json.dumps({"path": name, "step_ms": round(s, 4), "step_probe_n_ms": round(p, 4),
                      "overhead": round(p / s - 1, 4), "lib": os.environ.get("VOXL_TAG", "")}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--paths", default="dense,sparse,multires")
    a = ap.parse_args()
    dom = (a.n,) * 3
    paths = a.paths.split(",")
    if "dense" in paths:
        e = V.DenseEngine(domain=dom, precision="fp32")
        e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
        compare("dense", e, e.step, e.step_probe_n, a.k)
        e.close()
    if "sparse" in paths:
        for strategy in ("disag_mem", "disag_bitmask", "naive"):
            s = V.SparseEngine(dom, V.obstacle_mask(dom), block_edge=8, strategy=strategy, precision="fp32")
            compare("sparse_" + strategy, s, s.step, s.step_probe_n, a.k)
            s.close()
    if "multires" in paths:
        for fused in (True, False):
            m = V.MultiResEngine(dom, 3, fused=fused, precision="fp32")
            compare("multires_" + ("fused" if fused else "staged"), m, m.step, m.step_probe_n, max(4, a.k // 4))
            m.close()


if __name__ == "__main__":
    main()
