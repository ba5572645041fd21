import sys, os
sys.path.insert(0, os.getcwd())
import paper_2503_07898_b200 as V
e = V.DenseEngine(domain=(512, 512, 512), precision="fp32", layout="AoS")
e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
e.step(4)
e.close()
