#!/usr/bin/env python
"""Per-step wall time of step() vs step_probe() (fused probe + diag row D2H
every step) vs step_probe_n() (rows read back once per batch) at n^3."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2503_07898_b200 as V

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
k = int(sys.argv[2]) if len(sys.argv) > 2 else 50
e = V.DenseEngine(domain=(n, n, n), precision="fp32")
e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
e.step(5)
for _ in range(5):
    e.step_probe()
torch.cuda.synchronize()
t = time.perf_counter(); e.step(k); t1 = time.perf_counter()
for _ in range(k):
    d = e.step_probe()
t2 = time.perf_counter()
rows = e.step_probe_n(k)
t3 = time.perf_counter()
print(json.dumps({"tag": os.environ.get("TAG", ""), "step_ms": round((t1 - t) / k * 1e3, 4),
                  "step_probe_ms": round((t2 - t1) / k * 1e3, 4), "step_probe_n_ms": round((t3 - t2) / k * 1e3, 4),
                  "mass": d.mass, "max_speed": d.max_speed, "mass_n": rows[-1].mass}))
e.close()
