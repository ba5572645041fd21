#!/usr/bin/env python
"""ncu target: one plain and one probed step of the block-sparse (disag_mem)
and multires (fused) engines at n^3, so the launch list shows each step kernel
beside its fused-probe (DIAG) variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_07898_b200 as V

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dom = (n, n, n)
s = V.SparseEngine(dom, V.obstacle_mask(dom), block_edge=8, strategy="disag_mem", precision="fp32")
s.step(1)
s.step_probe_n(1)
s.close()
m = V.MultiResEngine(dom, 3, fused=True, precision="fp32")
m.step(1)
m.step_probe_n(1)
m.close()
