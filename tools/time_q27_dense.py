#!/usr/bin/env python
"""D3Q27 fp32 dense 512^3 cavity: step and step_probe per-step time (variant sweeps)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_07898_b200 as V

e = V.DenseEngine(lattice="D3Q27", domain=(512, 512, 512), precision="fp32")
e.set_equilibrium()
e.timed_steps(10)
t, _ = e.timed_steps(100)
for _ in range(3):
    e.step_probe()
t0 = time.perf_counter()
for _ in range(50):
    e.step_probe()
tp = (time.perf_counter() - t0) / 50 * 1e3
print(json.dumps({"tag": os.environ.get("TAG", ""), "step_ms": round(t / 100, 4), "MLUPS": round(512 ** 3 / (t / 100) / 1e3, 1),
                  "step_probe_ms": round(tp, 4)}))
