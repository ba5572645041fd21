#!/usr/bin/env python
"""BASELINE configs[0] end to end: the reference CPU solver's own
reference_dense_run (oracle/_ref, built from /root/reference; single thread,
D3Q19 BGK lid-driven cavity 128^3, tau 0.56, 1000 steps) against the B200
engines on the same input: fp64 must be bitwise equal, fp32 within 1e-5 per
population. Prints one JSON line with both wall times.

    python tools/configs0_parity.py [--steps 1000] [--n 128]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np

import oracle as O
import paper_2503_07898_b200 as V

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=1000)
ap.add_argument("--n", type=int, default=128)
a = ap.parse_args()
n = a.n
cfg = dict(lattice="D3Q19", domain=[n, n, n], tau=0.56, scenario="lid_driven_cavity", velocity=[0.05, 0, 0],
           steps=a.steps)
init = O.ref_initial_state(cfg)
t0 = time.perf_counter()
ref = O.ref_reference_dense_run(cfg)
t_ref = time.perf_counter() - t0
out = {"config": f"configs[0]: D3Q19 BGK cavity {n}^3, tau 0.56, lid (0.05,0,0), {a.steps} steps",
       "reference_seconds": round(t_ref, 2), "reference_MLUPS_1_thread": round(n ** 3 * a.steps / t_ref / 1e6, 3),
       "reference_kind": "reference" if O.ref_available() else "port"}
for prec in ("fp64", "fp32"):
    e = V.DenseEngine(domain=(n, n, n), precision=prec)
    e.set_canonical(init)
    e.step(3)  # warm-up on a copy of the run: restart from the initial state
    e.set_canonical(init)
    t0 = time.perf_counter()
    e.step(a.steps)
    t = time.perf_counter() - t0
    f = e.get_canonical()
    e.close()
    if prec == "fp64":
        out["fp64_bitwise_equal"] = bool(np.array_equal(f, ref))
        out["fp64_max_abs_diff"] = float(np.max(np.abs(f - ref)))
    else:
        out["fp32_max_rel_err"] = float(np.max(np.abs(f - ref) / np.abs(ref)))
    out[f"{prec}_gpu_seconds"] = round(t, 4)
    out[f"{prec}_gpu_MLUPS"] = round(n ** 3 * a.steps / t / 1e6, 1)
m_ref, s_ref = O.port_probe("D3Q19", ref)
out["reference_mass"], out["reference_max_speed"] = m_ref, s_ref
print(json.dumps(out))
