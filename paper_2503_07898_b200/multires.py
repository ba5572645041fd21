"""Multi-resolution engine (Python side of the C-ABI).

Mirrors mres::MultiResGrid / MultiResLbm (proj/include/voxl/multires.hpp):
level stack with factor-2 refinement, tau_l = 2 tau_{l+1} - 1/2, explosion /
coalescence transitions and fused vs staged execution.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import check, lib

LATTICES = {"D2Q9": 0, "D3Q19": 1, "D3Q27": 2}
Q_OF = {"D2Q9": 9, "D3Q19": 19, "D3Q27": 27}
NO_JUMP = 2 ** 31 - 1


def band_level_map(domain, levels, axis=2) -> np.ndarray:
    """run_multires's level map (solver.cpp:319-335): finest band under the lid."""
    nx, ny = domain[0], domain[1]
    nz = domain[2] if len(domain) == 3 else 1
    out = np.empty(nx * ny * nz, np.int32)
    check(lib.voxl_band_level_map(nx, ny, nz, levels, axis, out.ctypes.data))
    return out


def _desc(domain, levels, tau, lid_u, fused, precision, block_edge, lattice, reference_tables, solid_cells=False):
    d = _capi.MresDesc()
    d.lattice = LATTICES[lattice]
    d.nx, d.ny = domain[0], domain[1]
    d.nz = domain[2] if len(domain) == 3 else 1
    d.levels = levels
    d.tau = tau
    d.lid_u[:] = list(lid_u)
    d.fused = int(fused)
    d.precision = {"fp32": 0, "fp64": 1}[precision] if isinstance(precision, str) else int(precision)
    d.block_edge = block_edge
    d.reference_tables = int(reference_tables)
    d.solid_cells = int(solid_cells)
    return d


SOLID = -1  # level-map value of an obstacle cell (voxl_mres_desc::solid_cells)


def obstacle_band_level_map(domain, levels, radius=None, center=None):
    """The band cavity of run_multires with a solid sphere in the finest band
    (extension: the reference's multires has no obstacle cells). Default
    sphere: centre (nx/2, ny/2, 3 nz/4) - 1/2, radius nz/10; cells with
    |x - c| <= r become SOLID."""
    nx, ny, nz = domain
    m = band_level_map(domain, levels, 2).reshape(nz, ny, nx)
    r = nz / 10.0 if radius is None else float(radius)
    c = (nx / 2 - 0.5, ny / 2 - 0.5, 0.75 * nz - 0.5) if center is None else center
    z = np.arange(nz)[:, None, None]
    y = np.arange(ny)[None, :, None]
    x = np.arange(nx)[None, None, :]
    solid = (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 <= r * r
    m[solid] = SOLID
    return m.reshape(-1)


class MultiResPlan:
    """Host tables at the reference's edge-4 granularity (no device)."""

    def __init__(self, domain=(32, 32, 32), levels=3, level_map=None, tau=0.56, lattice="D3Q19", solid_cells=False):
        if level_map is None:
            level_map = band_level_map(domain, levels, 2 if len(domain) == 3 else 1)
        lm = np.ascontiguousarray(level_map, np.int32)
        d = _desc(domain, levels, tau, (0.05, 0, 0), True, "fp64", 4, lattice, True, solid_cells)
        self._h = C.c_void_p()
        check(lib.voxl_mres_plan_create(C.byref(d), lm.ctypes.data, C.byref(self._h)))
        self.levels = levels

    def level(self, l):
        na, tau, nb, ng, npull = C.c_int64(), C.c_double(), C.c_int(), C.c_int(), C.c_int()
        check(lib.voxl_mres_plan_level(self._h, l, C.byref(na), C.byref(tau), C.byref(nb), C.byref(ng),
                                       C.byref(npull)))
        return dict(num_active=na.value, tau=tau.value, ref_blocks=nb.value, ghosts=ng.value, pulls=npull.value)

    def ref_blocks(self, l):
        nb = self.level(l)["ref_blocks"]
        o = np.empty((nb, 3), np.int32)
        m = np.empty(nb, np.uint64)
        j = np.empty(nb, np.uint8)
        check(lib.voxl_mres_plan_ref_blocks(self._h, l, o.ctypes.data, m.ctypes.data, j.ctypes.data))
        return o, m, j

    def ghosts(self, l):
        n = self.level(l)["ghosts"]
        out = np.empty((n, 6), np.int32)
        check(lib.voxl_mres_plan_ghosts(self._h, l, out.ctypes.data))
        return out

    def pulls(self, l):
        n = self.level(l)["pulls"]
        out = np.empty((n, 7), np.int32)
        check(lib.voxl_mres_plan_pulls(self._h, l, out.ctypes.data))
        return out

    def jump_distance(self, l, v):
        out = C.c_int()
        check(lib.voxl_mres_plan_jump_distance(self._h, l, v[0], v[1], v[2], C.byref(out)))
        return out.value

    def graph_dot(self, fused=True):
        return _capi.text(lib.voxl_mres_plan_text, self._h, 0 if fused else 1)

    def distribution(self):
        return _capi.text(lib.voxl_mres_plan_text, self._h, 2)

    def close(self):
        if self._h:
            check(lib.voxl_mres_plan_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class MultiResEngine:
    def __init__(self, domain=(32, 32, 32), levels=3, level_map=None, tau=0.56, lid_u=(0.05, 0.0, 0.0),
                 fused=True, precision="fp32", block_edge=8, lattice="D3Q19", reference_tables=False,
                 solid_cells=False):
        if level_map is None:
            level_map = band_level_map(domain, levels, 2)
        lm = np.ascontiguousarray(level_map, np.int32)
        d = _desc(domain, levels, tau, lid_u, fused, precision, block_edge, lattice, reference_tables, solid_cells)
        self.q = Q_OF[lattice]
        self.levels = levels
        self._h = C.c_void_p()
        check(lib.voxl_mres_create(C.byref(d), lm.ctypes.data, C.byref(self._h)))

    def step(self, n=1):
        check(lib.voxl_mres_step(self._h, n))

    def timed_steps(self, n):
        out = (C.c_double * 5)()
        check(lib.voxl_mres_timed_steps(self._h, n, out))
        return out[0], dict(collide=out[1], stream=out[2], fused=out[3], transition=out[4])

    def state_len(self):
        n = C.c_int64()
        check(lib.voxl_mres_state_len(self._h, C.byref(n)))
        return n.value

    def digest(self) -> tuple[int, int]:
        """Device digest of the canonical state (csrc/digest.cuh; host restatement
        in digest.py): equal iff the canonical states are bitwise equal."""
        out = (C.c_uint64 * 2)()
        check(lib.voxl_mres_digest(self._h, out))
        return int(out[0]), int(out[1])

    def get_state(self):
        out = np.empty(self.state_len(), np.float64)
        check(lib.voxl_mres_get_state(self._h, out.ctypes.data))
        return out

    def set_state(self, canonical):
        v = np.ascontiguousarray(canonical, np.float64)
        if v.size != self.state_len():
            raise ValueError("set_state: size mismatch")
        check(lib.voxl_mres_set_state(self._h, v.ctypes.data))

    def set_equilibrium(self, rho=1.0, u=(0.0, 0.0, 0.0)):
        check(lib.voxl_mres_set_equilibrium(self._h, rho, (C.c_double * 3)(*u)))

    def probe(self):
        d = _capi.Diag()
        check(lib.voxl_mres_probe(self._h, C.byref(d)))
        return d

    def step_probe_n(self, n: int):
        """n coarse steps with probe_field fused into each level's last
        sub-step (run_multires's per-step rows), one host synchronisation per
        256 steps. Raises VoxlInstability with run()'s text at the first
        failing step (`.rows` = the rows before it)."""
        return _capi.probe_rows(lib.voxl_mres_step_probe_n, self._h, n)

    def total_mass(self):
        m = C.c_double()
        check(lib.voxl_mres_total_mass(self._h, C.byref(m)))
        return m.value

    def graph_dot(self):
        return _capi.text(lib.voxl_mres_text, self._h, 0)

    def distribution(self):
        return _capi.text(lib.voxl_mres_text, self._h, 1)

    def level_info(self, l):
        na, tau, uni, jmp = C.c_int64(), C.c_double(), C.c_int64(), C.c_int64()
        check(lib.voxl_mres_level_info(self._h, l, C.byref(na), C.byref(tau), C.byref(uni), C.byref(jmp)))
        return dict(num_active=na.value, tau=tau.value, uniform_blocks=uni.value, jump_blocks=jmp.value)

    def lup_per_coarse_step(self):
        n = C.c_int64()
        check(lib.voxl_mres_lup_per_coarse_step(self._h, C.byref(n)))
        return n.value

    def close(self):
        if self._h:
            check(lib.voxl_mres_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
