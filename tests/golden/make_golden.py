"""Regenerate the committed golden fixtures from the REFERENCE library.

Run in the build container (needs oracle/_ref/libvoxl_ref.so, built from
/root/reference/proj/src by oracle/Makefile):

    python tests/golden/make_golden.py

Every array is the reference's own output through its public API
(reference_dense_run, voxl::run, SparseLbmEngine, MultiResLbm); the JSON files
are lattice_to_json / LayoutMap::to_json documents.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

CASES = {
    # name: reference SolverConfig
    "dense_cavity_d3q19_12": dict(lattice="D3Q19", domain=[12, 12, 12], tau=0.56, scenario="lid_driven_cavity",
                                  velocity=[0.05, 0, 0], steps=30),
    "dense_cavity_d2q9_24x16": dict(lattice="D2Q9", domain=[24, 16], tau=0.6, scenario="lid_driven_cavity",
                                    velocity=[0.05, 0, 0], steps=40),
    "dense_cavity_d3q27_8x10x12": dict(lattice="D3Q27", domain=[8, 10, 12], tau=0.6, scenario="lid_driven_cavity",
                                       velocity=[0.05, 0, 0], steps=20),
    "dense_periodic_d3q19_10": dict(lattice="D3Q19", domain=[10, 10, 10], tau=0.8, scenario="periodic_box",
                                    velocity=[0, 0, 0], steps=20, perturbation=0.05, seed=7),
    "sparse_obstacle_d3q19_16": dict(lattice="D3Q19", domain=[16, 16, 16], tau=0.7, scenario="flow_over_obstacle",
                                     velocity=[0.04, 0, 0], steps=10, strategy="naive"),
    "mres3_cavity_d3q19_16": dict(lattice="D3Q19", domain=[16, 16, 16], tau=0.56, scenario="lid_driven_cavity",
                                  velocity=[0.05, 0, 0], steps=2, levels=3, fused=True),
}


def main():
    for name, cfg in CASES.items():
        r = O.RefRun(cfg)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), field=r.field, diagnostics=r.diagnostics,
                            config=json.dumps(cfg))
        print(name, r.field.size)
    lib = O.ref_lib()
    for kind, nm in [(0, "d2q9"), (1, "d3q19"), (2, "d3q27")]:
        with open(os.path.join(HERE, f"lattice_{nm}.json"), "w") as f:
            f.write(O.ref_text(lib.vref_lattice_json, kind))
    with open(os.path.join(HERE, "layout_disag_d2q9.json"), "w") as f:
        f.write(O.ref_text(lib.vref_layout_json, 2, 8, 4, 1, 0, 0, 1))
    for sch, nm in [(0, "aos"), (1, "soa"), (2, "disag")]:
        with open(os.path.join(HERE, f"layout_{nm}_d3q19_4x4x4.json"), "w") as f:
            f.write(O.ref_text(lib.vref_layout_json, sch, 4, 4, 4, 1, 0, 2))


if __name__ == "__main__":
    main()
