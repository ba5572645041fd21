"""Small driver for ncu: 512^3 D3Q19 fp32 dense cavity, a few steps."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_07898_b200 as V

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
e = V.DenseEngine(domain=(n, n, n), precision="fp32")
e.set_equilibrium()
e.step(steps)
print("ok", e.probe().mass)
