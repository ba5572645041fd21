#!/usr/bin/env python
"""fp32 state digests of the dense (SoA / DisagSoA / AoS, D3Q19 / D3Q27, plain
and fused-probe steps), block-sparse and multires engines after a perturbed
start: run once per library build to show that an arithmetic rewrite of the
fp32 kernels leaves every population bit for bit unchanged.

    python tools/fp32_digests.py      (one JSON line per engine)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_07898_b200 as V  # noqa: E402
from paper_2503_07898_b200.initial import initial_state  # noqa: E402

tag = os.environ.get("VOXL_TAG", "")
dom = (64, 48, 40)
for lat in ("D3Q19", "D3Q27"):
    init = initial_state(lat, dom, perturbation=0.05)
    for layout in ("SoA", "DisagSoA", "AoS"):
        for probe in (False, True):
            e = V.DenseEngine(lattice=lat, domain=dom, precision="fp32", partitions=2, layout=layout)
            e.set_canonical(init)
            if probe:
                e.step_probe_n(50)
            else:
                e.step(50)
            print(json.dumps({"lib": tag, "engine": "dense", "lattice": lat, "layout": layout, "probe": probe,
                              "digest": [hex(x) for x in e.digest()]}), flush=True)
            e.close()
n = 64
s = V.SparseEngine((n, n, n), V.obstacle_mask((n, n, n)), block_edge=8, strategy="disag_mem", precision="fp32")
s.step(50)
print(json.dumps({"lib": tag, "engine": "sparse", "digest": [hex(x) for x in s.digest()]}), flush=True)
s.close()
m = V.MultiResEngine((n, n, n), 3, fused=True, precision="fp32")
m.step(10)
print(json.dumps({"lib": tag, "engine": "multires", "digest": [hex(x) for x in m.digest()]}), flush=True)
m.close()
