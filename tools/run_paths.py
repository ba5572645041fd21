#!/usr/bin/env python
"""Per-step cost of the run() loops (solver.cpp:225-367) on the B200 engines:
step + probe_field every step, 512^3 fp32. Wall clock around K iterations of
  step(1)            the bare step (one host sync per call)
  step_probe_n(K)    run()'s loop: the probe fused into the step kernels,
                     rows read back once per batch (what voxl::b200::run calls)
  step(K)            K bare steps, one sync (the step_probe_n reference point)
  probe()            the stand-alone probe pass

    python tools/run_paths.py [--n 512] [--steps 200]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_07898_b200 as V  # noqa: E402


def timeit(fn, k, per=1):
    fn()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    return (time.perf_counter() - t) / (k * per) * 1e3


def row(path, dom, units, eng, k, step1, stepk, run, probe):
    ms_step1 = timeit(step1, max(2, k // 10))
    ms_stepk = timeit(stepk, 2, k)
    ms_run = timeit(run, 2, k)
    ms_probe = timeit(probe, max(2, k // 10))
    print(json.dumps({"path": path, "domain": list(dom), "units_per_step": units,
                      "step_ms": round(ms_step1, 4), "steps_batch_ms": round(ms_stepk, 4),
                      "run_step_ms": round(ms_run, 4), "probe_ms": round(ms_probe, 4),
                      "run_overhead": round(ms_run / ms_stepk - 1.0, 4),
                      "run_MLUPS": round(units / ms_run / 1e3, 1)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    n, k = a.n, a.steps
    dom = (n, n, n)
    e = V.DenseEngine(domain=dom, precision="fp32")
    e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
    row("dense", dom, n ** 3, e, k, lambda: e.step(1), lambda: e.step(k), lambda: e.step_probe_n(k), e.probe)
    e.close()
    for strategy in ("disag_mem", "disag_bitmask", "naive"):
        s = V.SparseEngine(dom, V.obstacle_mask(dom), block_edge=8, strategy=strategy, precision="fp32")
        row("block_sparse_" + strategy, dom, s.num_active, s, k, lambda: s.step(1), lambda: s.step(k),
            lambda: s.step_probe_n(k), s.probe)
        s.close()
    km = max(4, k // 4)
    for fused in (True, False):
        m = V.MultiResEngine(dom, 3, fused=fused, precision="fp32")
        row("multires_" + ("fused" if fused else "staged"), dom, m.lup_per_coarse_step(), m, km,
            lambda: m.step(1), lambda: m.step(km), lambda: m.step_probe_n(km), m.probe)
        m.close()


if __name__ == "__main__":
    main()
