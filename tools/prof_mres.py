"""ncu driver: 3-level band cavity, fused, a couple of coarse steps."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_07898_b200 as V

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
e = V.MultiResEngine((n, n, n), 3, fused=True, precision="fp32")
e.step(2)
print("ok")
