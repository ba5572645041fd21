#!/usr/bin/env python
"""Small runs of every engine kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): dense (3 layouts incl. the fp32 AoS
plane-tile kernel, 3 partitions, both halo modes, D3Q27, fp32/fp64, fused
probe, multi-device schedule with graph replay and the observed trace),
block-sparse (3 strategies, edge 4/8, fused probe, the bulk-copy staging
kernel), multires (fused/staged, obstacle, fused probe), canonical I/O both
ways.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2503_07898_b200 as V
from paper_2503_07898_b200.multires import obstacle_band_level_map

for lat in ("D3Q19", "D3Q27"):
    for prec in ("fp32", "fp64"):
        for layout in ("DisagSoA", "SoA", "AoS"):
            for halo in ("zero_copy", "copy"):
                e = V.DenseEngine(lattice=lat, domain=(20, 12, 18), precision=prec, layout=layout, partitions=3,
                                  halo_mode=halo)
                e.set_equilibrium()
                e.step(3)
                e.step_probe()
                e.step_probe_n(3)
                st = e.get_canonical()
                e.set_canonical(st)
                e.probe()
                e.close()
for lat in ("D3Q19", "D3Q27"):
    for prec in ("fp32", "fp64"):
        for edge in (4, 8):
            for strategy in ("naive", "disag_bitmask", "disag_mem"):
                s = V.SparseEngine((40, 24, 24), block_edge=edge, strategy=strategy, precision=prec, lattice=lat)
                s.step(2)
                s.step_probe()
                s.step_probe_n(2)
                st = s.get_state()
                s.set_state(st)
                s.probe()
                s.close()
dom = (32, 32, 32)
for prec in ("fp32", "fp64"):
    for fused in (True, False):
        m = V.MultiResEngine(dom, 3, fused=fused, precision=prec)
        m.step(2)
        st = m.get_state()
        m.set_state(st)
        m.step(1)
        m.probe()
        m.step_probe_n(2)
        m.close()
        m = V.MultiResEngine(dom, 3, level_map=obstacle_band_level_map(dom, 3), fused=fused, precision=prec,
                             solid_cells=True)
        m.step(2)
        m.close()
for fused in (True, False):  # D2Q9 multires: z = 0 layer of the E^3 blocks
    for edge in (4, 8):
        d2 = (32, 48, 1)
        m = V.MultiResEngine(d2, 3, level_map=V.band_level_map(d2, 3, axis=1), tau=0.6, fused=fused, precision="fp32",
                             block_edge=edge, lattice="D2Q9")
        m.step(2)
        m.set_state(m.get_state())
        m.probe()
        m.close()
# multi-device schedule (all partitions on device 0), graph replay, observed trace
e = V.DenseEngine("D3Q19", (16, 12, 24), 0.6, "lid_driven_cavity", (0.05, 0, 0), partitions=3, devices=[0, 0, 0],
                  graph_steps=2, precision="fp32")
e.set_equilibrium()
e.step(4)
e.step_probe_n(2)
e.trace(True)
e.step(1)
e.trace_json()
e.close()
# block-sparse bulk-copy (TMA) staging kernel
os.environ["VOXL_SPARSE_TMA"] = "1"
for lat in ("D3Q19", "D3Q27"):
    for strategy in ("naive", "disag_bitmask", "disag_mem"):
        s = V.SparseEngine((40, 24, 24), block_edge=8, strategy=strategy, precision="fp32", lattice=lat)
        s.step(2)
        s.step_probe_n(2)
        s.close()
del os.environ["VOXL_SPARSE_TMA"]
print("sanitize run ok")
