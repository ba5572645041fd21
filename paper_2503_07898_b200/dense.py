"""Dense grid layer and the dense engine (Python side of the C-ABI).

Mirrors the reference's dense API:

* ``layout_json`` / ``layout_addresses`` -- LayoutMap (proj/src/layout.cpp:72-229)
* ``decompose`` / ``classify_voxels``   -- partition.cpp:20-61
* ``DenseEngine``                        -- PartitionedField x2 + step_occ + GatherKernel
  (partition.hpp:95-214, lbm.hpp:123-133), on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import check, lib

LATTICES = {"D2Q9": 0, "D3Q19": 1, "D3Q27": 2}
Q_OF = {"D2Q9": 9, "D3Q19": 19, "D3Q27": 27}
LAYOUTS = {"AoS": 0, "SoA": 1, "DisagSoA": 2}
SCENARIOS = {"lid_driven_cavity": 0, "flow_over_obstacle": 1, "periodic_box": 2}
PRECISIONS = {"fp32": 0, "fp64": 1}
HALO_MODES = {"zero_copy": 0, "copy": 1, "nccl": 2}
# closed step_occ operator set (partition.hpp:173): the LBM GatherKernel and the
# reference tests' identity / five-point Jacobi kernels (partition_test.cpp:189, :234)
OPERATORS = {"lbm": 0, "identity": 1, "jacobi2": 2}


def _kind(lattice):
    return LATTICES[lattice] if isinstance(lattice, str) else int(lattice)


def lattice_json(lattice="D3Q19") -> str:
    """lattice_to_json (proj/src/lattice.cpp:140-158)."""
    return _capi.text(lib.voxl_lattice_json, _kind(lattice))


def layout_json(scheme="DisagSoA", shape=(4, 4, 4), lattice="D3Q19", axis=2, cardinality=0) -> str:
    """LayoutMap::build(...).to_json(); lattice=None selects the generic build."""
    sch = LAYOUTS[scheme] if isinstance(scheme, str) else int(scheme)
    kind = -1 if lattice is None else _kind(lattice)
    return _capi.text(lib.voxl_layout_json, sch, shape[0], shape[1], shape[2], kind, cardinality, axis)


def layout_addresses(scheme="DisagSoA", shape=(4, 4, 4), lattice="D3Q19", axis=2) -> np.ndarray:
    sch = LAYOUTS[scheme] if isinstance(scheme, str) else int(scheme)
    n = C.c_int64()
    check(lib.voxl_layout_addresses(sch, shape[0], shape[1], shape[2], _kind(lattice), axis, None, 0, C.byref(n)))
    out = np.empty(n.value, np.int64)
    check(lib.voxl_layout_addresses(sch, shape[0], shape[1], shape[2], _kind(lattice), axis, out.ctypes.data,
                                    n.value, C.byref(n)))
    return out


def decompose(domain, parts, axis=2, periodic=False):
    slabs = np.empty(2 * parts, np.int32)
    check(lib.voxl_decompose(domain[0], domain[1], domain[2], parts, axis, int(periodic), slabs.ctypes.data))
    return [(int(slabs[2 * p]), int(slabs[2 * p + 1])) for p in range(parts)]


def classify_voxels(domain, parts, p, axis=2, periodic=False) -> np.ndarray:
    slabs = decompose(domain, parts, axis, periodic)
    shape = list(domain)
    shape[axis] = slabs[p][1] - slabs[p][0]
    out = np.empty(int(np.prod(shape)), np.uint8)
    check(lib.voxl_classify_voxels(domain[0], domain[1], domain[2], parts, axis, int(periodic), p,
                                   out.ctypes.data, out.size))
    return out


@dataclass
class TransferRecord:
    step: int
    src: int
    dst: int
    base_src: int
    base_dst: int
    elements: int


def make_desc(lattice="D3Q19", domain=(32, 32, 32), tau=0.56, scenario="lid_driven_cavity",
              velocity=(0.05, 0.0, 0.0), layout="DisagSoA", partitions=1, precision="fp32",
              halo_mode="zero_copy", first_partition=0, local_partitions=-1, op="lbm") -> _capi.DenseDesc:
    d = _capi.DenseDesc()
    d.lattice = _kind(lattice)
    dom = tuple(domain) if len(domain) == 3 else (domain[0], domain[1], 1)
    d.nx, d.ny, d.nz = dom
    d.tau = tau
    d.scenario = SCENARIOS[scenario] if isinstance(scenario, str) else int(scenario)
    d.velocity[:] = list(velocity) + [0.0] * (3 - len(velocity))
    d.layout = LAYOUTS[layout] if isinstance(layout, str) else int(layout)
    d.partitions = partitions
    d.precision = PRECISIONS[precision] if isinstance(precision, str) else int(precision)
    d.halo_mode = HALO_MODES[halo_mode] if isinstance(halo_mode, str) else int(halo_mode)
    d.first_partition = first_partition
    d.local_partitions = local_partitions
    d.op = OPERATORS[op] if isinstance(op, str) else int(op)
    return d


def _records(fn, *args):
    cnt = C.c_int()
    check(fn(*args, None, 0, C.byref(cnt)))
    arr = (_capi.TransferRecordC * max(cnt.value, 1))()
    check(fn(*args, arr, cnt.value, C.byref(cnt)))
    return [TransferRecord(r.step, r.src, r.dst, r.src_base, r.dst_base, r.elements) for r in arr[: cnt.value]]


def plan_ledger(step=0, **desc):
    """Halo-update records of one step (partition.cpp:163-206), device-free."""
    d = make_desc(**desc)
    return _records(lib.voxl_dense_plan_ledger, C.byref(d), step)


class DenseEngine:
    """Dense partitioned LBM engine on the current CUDA device.

    ``set_canonical`` / ``get_canonical`` move fp64 canonical fields (x fastest,
    component innermost -- the reference's dump order); ``step(n)`` runs n
    OCC steps; ``probe()`` is probe_field on the device.
    """

    def __init__(self, lattice="D3Q19", domain=(32, 32, 32), tau=0.56, scenario="lid_driven_cavity",
                 velocity=(0.05, 0.0, 0.0), layout="DisagSoA", partitions=1, precision="fp32",
                 halo_mode="zero_copy", first_partition=0, local_partitions=-1, op="lbm", devices=None,
                 graph_steps=8):
        """``devices``: one CUDA device per partition (the single-process
        multi-device engine, voxl_dense_create_multi); None keeps every
        partition on the current device, launched back to back on one stream."""
        d = make_desc(lattice, domain, tau, scenario, velocity, layout, partitions, precision, halo_mode,
                      first_partition, local_partitions, op)
        dom = (d.nx, d.ny, d.nz)
        self.lattice = lattice if isinstance(lattice, str) else list(LATTICES)[lattice]
        self.op = op if isinstance(op, str) else list(OPERATORS)[op]
        self.q = 2 if self.op == "jacobi2" else Q_OF[self.lattice]
        self.domain = dom
        self.partitions = partitions
        self._h = C.c_void_p()
        if devices is None:
            check(lib.voxl_dense_create(C.byref(d), C.byref(self._h)))
        else:
            devs = (C.c_int * max(partitions, 1))(*[int(x) for x in devices])
            if len(devices) != partitions:
                raise ValueError("devices must name one device per partition")
            check(lib.voxl_dense_create_multi(C.byref(d), devs, graph_steps, C.byref(self._h)))

    @property
    def voxels(self) -> int:
        return int(np.prod(self.domain))

    def set_canonical(self, values: np.ndarray) -> None:
        v = np.ascontiguousarray(values, np.float64)
        if v.size != self.voxels * self.q:
            raise ValueError("fill_canonical: size mismatch")
        check(lib.voxl_dense_set_canonical(self._h, v.ctypes.data))

    def set_equilibrium(self, rho: float = 1.0, u=(0.0, 0.0, 0.0)) -> None:
        uu = (C.c_double * 3)(*u)
        check(lib.voxl_dense_set_equilibrium(self._h, rho, uu))

    def digest(self) -> tuple[int, int]:
        """Device digest of the canonical state (csrc/digest.cuh; host restatement
        in digest.py): equal iff the canonical states are bitwise equal."""
        out = (C.c_uint64 * 2)()
        check(lib.voxl_dense_digest(self._h, out))
        return int(out[0]), int(out[1])

    def get_canonical(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.voxels * self.q, np.float64)
        elif out.dtype != np.float64 or out.size != self.voxels * self.q or not out.flags.c_contiguous:
            raise ValueError("to_canonical: out must be a contiguous float64 array of voxels * q elements")
        check(lib.voxl_dense_get_canonical(self._h, out.ctypes.data))
        return out

    def _plane_elems(self) -> int:
        axis2d = self.lattice == "D2Q9"
        return self.domain[0] * (1 if axis2d else self.domain[1]) * self.q

    def get_canonical_planes(self, k_begin: int, k_end: int) -> np.ndarray:
        """Canonical fp64 values of partition-axis planes [k_begin, k_end)."""
        out = np.empty((k_end - k_begin) * self._plane_elems(), np.float64)
        check(lib.voxl_dense_get_planes(self._h, out.ctypes.data, k_begin, k_end))
        return out

    def set_canonical_planes(self, values: np.ndarray, k_begin: int, k_end: int) -> None:
        v = np.ascontiguousarray(values, np.float64)
        if v.size != (k_end - k_begin) * self._plane_elems():
            raise ValueError("set_canonical_planes: size mismatch")
        check(lib.voxl_dense_set_planes(self._h, v.ctypes.data, k_begin, k_end))

    def step(self, n: int = 1) -> None:
        check(lib.voxl_dense_step(self._h, n))

    def enqueue(self, n: int = 1) -> None:
        check(lib.voxl_dense_enqueue(self._h, n))

    def timed_steps(self, n: int):
        """n steps bracketed by CUDA events on the engine stream -> (total_ms, kernel_ms)."""
        t, k = C.c_double(), C.c_double()
        check(lib.voxl_dense_timed_steps(self._h, n, C.byref(t), C.byref(k)))
        return t.value, k.value

    def synchronize(self) -> None:
        check(lib.voxl_dense_synchronize(self._h))

    def probe(self):
        d = _capi.Diag()
        check(lib.voxl_dense_probe(self._h, C.byref(d)))
        return d

    def step_probe(self):
        """One step with probe_field fused into the step kernel."""
        d = _capi.Diag()
        check(lib.voxl_dense_step_probe(self._h, C.byref(d)))
        return d

    def step_probe_n(self, n: int):
        """n steps, each with probe_field fused, one host synchronisation per
        256 steps: the list of n diagnostics rows. On the first failing step
        raises VoxlInstability with run()'s text; `.rows` holds the rows of
        the steps before it."""
        return _capi.probe_rows(lib.voxl_dense_step_probe_n, self._h, n)

    def trace(self, on: bool = True) -> None:
        """Record the executed schedule of the steps enqueued from now on
        (CUDA-event-timed phases); trace(False) stops and clears it."""
        check(lib.voxl_dense_trace_enable(self._h, 1 if on else 0))

    def trace_json(self) -> str:
        """The recorded phases as JSON (see voxl_dense_trace_json)."""
        return _capi.text(lib.voxl_dense_trace_json, self._h)

    def ledger(self, step: int):
        return _records(lib.voxl_dense_ledger, self._h, step)

    def layout_json(self, partition: int = 0) -> str:
        return _capi.text(lib.voxl_dense_layout_json, self._h, partition)

    def buffer(self, partition: int, which: int = 0):
        p = C.c_void_p()
        n = C.c_size_t()
        check(lib.voxl_dense_buffer(self._h, partition, which, C.byref(p), C.byref(n)))
        return p.value, n.value

    def stream(self) -> int:
        s = C.c_void_p()
        check(lib.voxl_dense_stream(self._h, C.byref(s)))
        return s.value or 0

    def attach_peer(self, partition: int, buf0: int, buf1: int) -> None:
        check(lib.voxl_dense_attach_peer(self._h, partition, C.c_void_p(buf0), C.c_void_p(buf1)))

    def device(self, partition: int) -> int:
        d = C.c_int()
        check(lib.voxl_dense_device(self._h, partition, C.byref(d)))
        return d.value

    def neighbors(self, partition: int):
        """PartitionedField::neighbors (partition.hpp:110): (upper, lower)."""
        u, lo = C.c_int(), C.c_int()
        check(lib.voxl_dense_neighbors(self._h, partition, C.byref(u), C.byref(lo)))
        return u.value, lo.value

    def set_neighbor_links(self, partition: int, upper: int, lower: int) -> None:
        """The reference's fault-injection hook (partition.hpp:111-113)."""
        check(lib.voxl_dense_set_neighbor_links(self._h, partition, upper, lower))

    def close(self) -> None:
        if self._h:
            check(lib.voxl_dense_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
