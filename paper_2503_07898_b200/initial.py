"""initial_canonical_state (proj/src/solver.cpp:165-187) via the C-ABI."""
from __future__ import annotations

import numpy as np

from ._capi import check, lib

LATTICES = {"D2Q9": 0, "D3Q19": 1, "D3Q27": 2}
SCENARIOS = {"lid_driven_cavity": 0, "flow_over_obstacle": 1, "periodic_box": 2}
Q_OF = {"D2Q9": 9, "D3Q19": 19, "D3Q27": 27}


def initial_state(lattice="D3Q19", domain=(32, 32, 32), scenario="lid_driven_cavity", seed=42,
                  perturbation=0.0) -> np.ndarray:
    nx, ny = domain[0], domain[1]
    nz = domain[2] if len(domain) == 3 else 1
    out = np.empty(nx * ny * nz * Q_OF[lattice], np.float64)
    check(lib.voxl_initial_state(LATTICES[lattice], SCENARIOS[scenario], nx, ny, nz, int(seed), float(perturbation),
                                 out.ctypes.data))
    return out


def initial_canonical_state(config) -> np.ndarray:
    return initial_state(config.lattice, config.domain, config.scenario, config.seed, config.perturbation)
