"""Block-sparse wind tunnel engine (Python side of the C-ABI).

Mirrors sparse::SparseLbmEngine (proj/include/voxl/sparse.hpp:175-213): the
three dispatch strategies of Table 2 over a block-sparse grid, flow past an
obstacle with bounce-back on inactive neighbours / domain walls and the
regularized inflow/outflow on the x faces.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import check, lib

STRATEGIES = {"naive": 0, "disag_bitmask": 1, "disag_mem": 2}
LATTICES = {"D3Q19": 1, "D3Q27": 2}
Q_OF = {"D3Q19": 19, "D3Q27": 27}


def obstacle_mask(domain, radius=0.0) -> np.ndarray:
    """run_sparse's active set (solver.cpp:272-283): box minus a sphere."""
    nx, ny, nz = domain
    out = np.empty(nx * ny * nz, np.uint8)
    n = C.c_int64()
    check(lib.voxl_obstacle_mask(nx, ny, nz, float(radius), out.ctypes.data, C.byref(n)))
    return out


def dispatch_plan_json(strategy, n_b, n_nb, q=19, block_size=64, s_w=24, s_i=4, naive_full_domain_storage=False):
    s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
    return _capi.text(lib.voxl_dispatch_plan_json, s, n_b, n_nb, q, block_size, s_w, s_i,
                      int(naive_full_domain_storage))


def _desc(domain, tau, u_bc, block_edge, strategy, precision, lattice):
    d = _capi.SparseDesc()
    d.lattice = LATTICES[lattice]
    d.nx, d.ny, d.nz = domain
    d.tau = tau
    d.u_bc[:] = list(u_bc)
    d.block_edge = block_edge
    d.strategy = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
    d.precision = {"fp32": 0, "fp64": 1}[precision] if isinstance(precision, str) else int(precision)
    return d


class SparsePlan:
    """Host tables of the block-sparse path (no device): BlockSparseGrid::build,
    classify_blocks, arrange, dispatch_plan (sparse.cpp:20-225)."""

    def __init__(self, domain=(32, 32, 32), active=None, block_edge=4, strategy="naive", lattice="D3Q19",
                 radius=0.0, _handle=None, _owner=None):
        self.block_edge = block_edge
        self._owner = _owner
        if _handle is not None:
            self._h = _handle
            self._owned = False
            return
        if active is None:
            active = obstacle_mask(domain, radius)
        act = np.ascontiguousarray(active, np.uint8)
        d = _desc(domain, 0.7, (0.0, 0.0, 0.0), block_edge, strategy, "fp32", lattice)
        self._h = C.c_void_p()
        check(lib.voxl_sparse_plan_create(C.byref(d), act.ctypes.data, C.byref(self._h)))
        self._owned = True

    def info(self):
        na, nb, nbd, nnb = C.c_int64(), C.c_int(), C.c_int64(), C.c_int64()
        check(lib.voxl_sparse_plan_info(self._h, C.byref(na), C.byref(nb), C.byref(nbd), C.byref(nnb)))
        return dict(num_active=na.value, num_blocks=nb.value, n_boundary=nbd.value, n_non_boundary=nnb.value)

    def blocks(self):
        nb = self.info()["num_blocks"]
        words = max(1, self.block_edge ** 3 // 64)
        o = np.empty((nb, 3), np.int32)
        m = np.empty((nb, words), np.uint64)
        c = np.empty(nb, np.uint8)
        check(lib.voxl_sparse_plan_blocks(self._h, o.ctypes.data, m.ctypes.data, c.ctypes.data))
        return o, m, c

    def arrangement(self):
        nb = self.info()["num_blocks"]
        perm = np.empty(nb, np.int32)
        bm = np.zeros(nb, np.uint8)
        mi = np.full(nb * self.block_edge ** 3, -1, np.int32)
        cnt = C.c_int64()
        check(lib.voxl_sparse_plan_arrangement(self._h, perm.ctypes.data, bm.ctypes.data, mi.ctypes.data,
                                               C.byref(cnt)))
        return perm, bm, mi, cnt.value

    def neighbours(self):
        nb = self.info()["num_blocks"]
        out = np.empty((nb, 27), np.int32)
        check(lib.voxl_sparse_plan_neighbours(self._h, out.ctypes.data))
        return out

    def report_json(self) -> str:
        return _capi.text(lib.voxl_sparse_plan_report_json, self._h)

    def close(self):
        if self._h and self._owned:
            check(lib.voxl_sparse_plan_destroy(self._h))
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SparseEngine:
    def __init__(self, domain=(32, 32, 32), active=None, tau=0.7, u_bc=(0.04, 0.0, 0.0), block_edge=8,
                 strategy="disag_mem", precision="fp32", lattice="D3Q19", radius=0.0):
        d = _capi.SparseDesc()
        d.lattice = LATTICES[lattice]
        d.nx, d.ny, d.nz = domain
        d.tau = tau
        d.u_bc[:] = list(u_bc)
        d.block_edge = block_edge
        d.strategy = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
        d.precision = {"fp32": 0, "fp64": 1}[precision] if isinstance(precision, str) else int(precision)
        if active is None:
            active = obstacle_mask(domain, radius)
        self.active = np.ascontiguousarray(active, np.uint8)
        self.q = Q_OF[lattice]
        self.domain = tuple(domain)
        self.block_edge = block_edge
        self._h = C.c_void_p()
        check(lib.voxl_sparse_create(C.byref(d), self.active.ctypes.data, C.byref(self._h)))

    def plan(self) -> SparsePlan:
        p = C.c_void_p()
        check(lib.voxl_sparse_plan_of(self._h, C.byref(p)))
        return SparsePlan(block_edge=self.block_edge, _handle=p, _owner=self)

    def info(self):
        return self.plan().info()

    @property
    def num_active(self):
        return self.info()["num_active"]

    def blocks(self):
        return self.plan().blocks()

    def arrangement(self):
        return self.plan().arrangement()

    def report_json(self) -> str:
        return self.plan().report_json()

    def digest(self) -> tuple[int, int]:
        """Device digest of the canonical state (csrc/digest.cuh; host restatement
        in digest.py): equal iff the canonical states are bitwise equal."""
        out = (C.c_uint64 * 2)()
        check(lib.voxl_sparse_digest(self._h, out))
        return int(out[0]), int(out[1])

    def get_state(self) -> np.ndarray:
        out = np.empty(self.num_active * self.q, np.float64)
        check(lib.voxl_sparse_get_state(self._h, out.ctypes.data))
        return out

    def set_state(self, canonical) -> None:
        v = np.ascontiguousarray(canonical, np.float64)
        if v.size != self.num_active * self.q:
            raise ValueError("set_state: size mismatch")
        check(lib.voxl_sparse_set_state(self._h, v.ctypes.data))

    def set_equilibrium(self, rho=1.0, u=(0.0, 0.0, 0.0)):
        check(lib.voxl_sparse_set_equilibrium(self._h, rho, (C.c_double * 3)(*u)))

    def step(self, n=1):
        check(lib.voxl_sparse_step(self._h, n))

    def step_identity(self, n=1):
        """SparseLbmEngine::step_identity (sparse.cpp:396-404)."""
        check(lib.voxl_sparse_step_identity(self._h, n))

    def timed_steps(self, n):
        t, b, l_ = C.c_double(), C.c_double(), C.c_double()
        check(lib.voxl_sparse_timed_steps(self._h, n, C.byref(t), C.byref(b), C.byref(l_)))
        return t.value, b.value, l_.value

    def probe(self):
        d = _capi.Diag()
        check(lib.voxl_sparse_probe(self._h, C.byref(d)))
        return d

    def step_probe(self):
        """One step with probe_field fused into the step kernels (run_sparse's
        per-step diagnostics row)."""
        d = _capi.Diag()
        check(lib.voxl_sparse_step_probe(self._h, C.byref(d)))
        return d

    def step_probe_n(self, n: int):
        """n steps with probe_field fused into the step kernels (run_sparse's
        per-step rows), one host synchronisation per 256 steps. Raises
        VoxlInstability with run()'s text at the first failing step (`.rows`
        = the rows before it)."""
        return _capi.probe_rows(lib.voxl_sparse_step_probe_n, self._h, n)

    def close(self):
        if self._h:
            check(lib.voxl_sparse_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
