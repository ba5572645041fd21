#!/usr/bin/env python
"""ncu target: 3 plain dense steps then 3 step_probe() calls at n^3, so the
launch list shows the plain vs the fused-probe step kernel side by side."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_07898_b200 as V

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
e = V.DenseEngine(domain=(n, n, n), precision="fp32")
e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
e.step(3)
for _ in range(3):
    e.step_probe()
e.close()
