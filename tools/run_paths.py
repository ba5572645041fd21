#!/usr/bin/env python
"""Per-step cost of the run() loops (solver.cpp:225-367) on the B200 engines:
step + probe_field every step, wall clock around K iterations, 512^3 fp32.

    python tools/run_paths.py [--n 512] [--steps 20]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_07898_b200 as V  # noqa: E402


def timeit(fn, k):
    fn()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    return (time.perf_counter() - t) / k * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    n, k = a.n, a.steps
    dom = (n, n, n)
    e = V.DenseEngine(domain=dom, precision="fp32")
    e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
    ms_step = timeit(lambda: e.step(1), k)
    ms_run = timeit(lambda: e.step_probe(), k)
    ms_probe = timeit(lambda: e.probe(), k)
    print(json.dumps({"path": "dense", "domain": list(dom), "step_ms": round(ms_step, 4),
                      "run_step_ms": round(ms_run, 4), "probe_ms": round(ms_probe, 4),
                      "run_MLUPS": round(n ** 3 / ms_run / 1e3, 1)}), flush=True)
    e.close()
    s = V.SparseEngine(dom, V.obstacle_mask(dom), block_edge=8, strategy="disag_mem", precision="fp32")
    na = s.num_active
    ms_step = timeit(lambda: s.step(1), k)
    ms_probe = timeit(lambda: s.probe(), k)
    ms_run = timeit(lambda: s.step_probe(), k)
    print(json.dumps({"path": "block_sparse", "domain": list(dom), "active": na, "step_ms": round(ms_step, 4),
                      "probe_ms": round(ms_probe, 4), "run_step_ms": round(ms_run, 4),
                      "run_MLUPS": round(na / ms_run / 1e3, 1)}), flush=True)
    s.close()
    m = V.MultiResEngine(dom, 3, fused=True, precision="fp32")
    lup = m.lup_per_coarse_step()
    ms_step = timeit(lambda: m.step(1), max(2, k // 4))
    ms_probe = timeit(lambda: m.probe(), max(2, k // 4))
    print(json.dumps({"path": "multires", "domain": list(dom), "lup_per_coarse_step": lup,
                      "coarse_step_ms": round(ms_step, 4), "probe_ms": round(ms_probe, 4),
                      "run_step_ms": round(ms_step + ms_probe, 4),
                      "run_MLUPS": round(lup / (ms_step + ms_probe) / 1e3, 1)}), flush=True)
    m.close()


if __name__ == "__main__":
    main()
