"""ctypes binding of include/voxl_b200.h (the C-ABI of libvoxl_b200.so).

The product path loads ONLY the in-tree CUDA library. If it is missing the
import fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libvoxl_b200.so")

# status codes (voxl_b200.h)
OK, INVALID_ARGUMENT, OUT_OF_RANGE, RUNTIME, INSTABILITY, CUDA_ERROR, DOMAIN = range(7)


class VoxlError(RuntimeError):
    """Base of the exceptions raised for non-zero C-ABI status codes."""


class VoxlInvalidArgument(VoxlError, ValueError):
    pass


class VoxlOutOfRange(VoxlError, IndexError):
    pass


class VoxlInstability(VoxlError):
    pass


class VoxlCudaError(VoxlError):
    pass


class VoxlDomainError(VoxlError, ArithmeticError):
    pass


_EXC = {INVALID_ARGUMENT: VoxlInvalidArgument, OUT_OF_RANGE: VoxlOutOfRange, RUNTIME: VoxlError,
        INSTABILITY: VoxlInstability, CUDA_ERROR: VoxlCudaError, DOMAIN: VoxlDomainError}


class DenseDesc(C.Structure):
    _fields_ = [("lattice", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("tau", C.c_double),
                ("scenario", C.c_int), ("velocity", C.c_double * 3), ("layout", C.c_int), ("partitions", C.c_int),
                ("precision", C.c_int), ("halo_mode", C.c_int), ("first_partition", C.c_int),
                ("local_partitions", C.c_int), ("op", C.c_int)]


class Diag(C.Structure):
    _fields_ = [("mass", C.c_double), ("max_speed", C.c_double), ("unstable", C.c_int),
                ("bad_population", C.c_int), ("bad_voxel", C.c_int64)]


class TransferRecordC(C.Structure):
    _fields_ = [("step", C.c_int), ("src", C.c_int), ("dst", C.c_int), ("src_base", C.c_int64),
                ("dst_base", C.c_int64), ("elements", C.c_int64)]


class SparseDesc(C.Structure):
    _fields_ = [("lattice", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("tau", C.c_double),
                ("u_bc", C.c_double * 3), ("block_edge", C.c_int), ("strategy", C.c_int), ("precision", C.c_int)]


class MresDesc(C.Structure):
    _fields_ = [("lattice", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("levels", C.c_int),
                ("tau", C.c_double), ("lid_u", C.c_double * 3), ("fused", C.c_int), ("precision", C.c_int),
                ("block_edge", C.c_int), ("reference_tables", C.c_int), ("solid_cells", C.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i64, cp = C.c_void_p, C.c_int64, C.c_char_p
    sigs = {
        "voxl_last_error": ([], cp),
        "voxl_version": ([], C.c_int),
        "voxl_device_count": ([C.POINTER(C.c_int)], C.c_int),
        "voxl_lattice_json": ([C.c_int, cp, i64, C.POINTER(i64)], C.c_int),
        "voxl_layout_json": ([C.c_int] * 7 + [cp, i64, C.POINTER(i64)], C.c_int),
        "voxl_layout_addresses": ([C.c_int] * 6 + [vp, i64, C.POINTER(i64)], C.c_int),
        "voxl_decompose": ([C.c_int] * 6 + [vp], C.c_int),
        "voxl_classify_voxels": ([C.c_int] * 7 + [vp, i64], C.c_int),
        "voxl_dense_create": ([C.POINTER(DenseDesc), C.POINTER(vp)], C.c_int),
        "voxl_dense_create_multi": ([C.POINTER(DenseDesc), vp, C.c_int, C.POINTER(vp)], C.c_int),
        "voxl_dense_device": ([vp, C.c_int, C.POINTER(C.c_int)], C.c_int),
        "voxl_dense_neighbors": ([vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
        "voxl_dense_set_neighbor_links": ([vp, C.c_int, C.c_int, C.c_int], C.c_int),
        "voxl_dense_destroy": ([vp], C.c_int),
        "voxl_dense_set_canonical": ([vp, vp], C.c_int),
        "voxl_dense_get_canonical": ([vp, vp], C.c_int),
        "voxl_dense_digest": ([vp, vp], C.c_int),
        "voxl_dense_set_equilibrium": ([vp, C.c_double, C.POINTER(C.c_double)], C.c_int),
        "voxl_dense_set_planes": ([vp, vp, C.c_int, C.c_int], C.c_int),
        "voxl_dense_get_planes": ([vp, vp, C.c_int, C.c_int], C.c_int),
        "voxl_dense_step": ([vp, C.c_int], C.c_int),
        "voxl_dense_enqueue": ([vp, C.c_int], C.c_int),
        "voxl_dense_synchronize": ([vp], C.c_int),
        "voxl_dense_timed_steps": ([vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
        "voxl_dense_probe": ([vp, C.POINTER(Diag)], C.c_int),
        "voxl_dense_step_probe": ([vp, C.POINTER(Diag)], C.c_int),
        "voxl_dense_step_probe_n": ([vp, C.c_int, C.POINTER(Diag), C.POINTER(C.c_int)], C.c_int),
        "voxl_dense_trace_enable": ([vp, C.c_int], C.c_int),
        "voxl_dense_trace_json": ([vp, cp, i64, C.POINTER(i64)], C.c_int),
        "voxl_dense_ledger": ([vp, C.c_int, vp, C.c_int, C.POINTER(C.c_int)], C.c_int),
        "voxl_dense_plan_ledger": ([C.POINTER(DenseDesc), C.c_int, vp, C.c_int, C.POINTER(C.c_int)], C.c_int),
        "voxl_dense_layout_json": ([vp, C.c_int, cp, i64, C.POINTER(i64)], C.c_int),
        "voxl_dense_steps_done": ([vp, C.POINTER(C.c_int)], C.c_int),
        "voxl_dense_buffer": ([vp, C.c_int, C.c_int, C.POINTER(vp), C.POINTER(C.c_size_t)], C.c_int),
        "voxl_dense_stream": ([vp, C.POINTER(vp)], C.c_int),
        "voxl_dense_shared_stream": ([vp, C.POINTER(vp)], C.c_int),
        "voxl_dense_attach_peer": ([vp, C.c_int, vp, vp], C.c_int),
        "voxl_dense_raw_buffer": ([vp, C.c_int, C.c_int, C.POINTER(vp)], C.c_int),
        "voxl_dense_enable_distributed": ([vp, C.POINTER(vp)], C.c_int),
        "voxl_dense_attach_flags": ([vp, vp, vp], C.c_int),
        "voxl_dense_halo_push": ([vp], C.c_int),
        "voxl_dense_owned_voxels": ([vp, C.POINTER(i64)], C.c_int),
        "voxl_obstacle_mask": ([C.c_int, C.c_int, C.c_int, C.c_double, vp, C.POINTER(i64)], C.c_int),
        "voxl_sparse_create": ([C.POINTER(SparseDesc), vp, C.POINTER(vp)], C.c_int),
        "voxl_sparse_destroy": ([vp], C.c_int),
        "voxl_sparse_plan_create": ([C.POINTER(SparseDesc), vp, C.POINTER(vp)], C.c_int),
        "voxl_sparse_plan_destroy": ([vp], C.c_int),
        "voxl_sparse_plan_of": ([vp, C.POINTER(vp)], C.c_int),
        "voxl_sparse_plan_info": ([vp, C.POINTER(i64), C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(i64)],
                                  C.c_int),
        "voxl_sparse_plan_blocks": ([vp, vp, vp, vp], C.c_int),
        "voxl_sparse_plan_arrangement": ([vp, vp, vp, vp, C.POINTER(i64)], C.c_int),
        "voxl_sparse_plan_report_json": ([vp, cp, i64, C.POINTER(i64)], C.c_int),
        "voxl_sparse_plan_neighbours": ([vp, vp], C.c_int),
        "voxl_sparse_info": ([vp, C.POINTER(i64), C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "voxl_sparse_blocks": ([vp, vp, vp, vp], C.c_int),
        "voxl_sparse_arrangement": ([vp, vp, vp, vp, C.POINTER(i64)], C.c_int),
        "voxl_sparse_report_json": ([vp, cp, i64, C.POINTER(i64)], C.c_int),
        "voxl_sparse_get_state": ([vp, vp], C.c_int),
        "voxl_sparse_digest": ([vp, vp], C.c_int),
        "voxl_sparse_set_state": ([vp, vp], C.c_int),
        "voxl_sparse_set_equilibrium": ([vp, C.c_double, C.POINTER(C.c_double)], C.c_int),
        "voxl_sparse_step": ([vp, C.c_int], C.c_int),
        "voxl_sparse_step_identity": ([vp, C.c_int], C.c_int),
        "voxl_sparse_timed_steps": ([vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)], C.c_int),
        "voxl_sparse_probe": ([vp, C.POINTER(Diag)], C.c_int),
        "voxl_sparse_step_probe": ([vp, C.POINTER(Diag)], C.c_int),
        "voxl_sparse_step_probe_n": ([vp, C.c_int, C.POINTER(Diag), C.POINTER(C.c_int)], C.c_int),
        "voxl_dispatch_plan_json": ([C.c_int, i64, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, cp, i64,
                                     C.POINTER(i64)], C.c_int),
        "voxl_band_level_map": ([C.c_int] * 5 + [vp], C.c_int),
        "voxl_initial_state": ([C.c_int] * 5 + [C.c_uint64, C.c_double, vp], C.c_int),
        "voxl_mres_create": ([C.POINTER(MresDesc), vp, C.POINTER(vp)], C.c_int),
        "voxl_mres_destroy": ([vp], C.c_int),
        "voxl_mres_step": ([vp, C.c_int], C.c_int),
        "voxl_mres_timed_steps": ([vp, C.c_int, vp], C.c_int),
        "voxl_mres_state_len": ([vp, C.POINTER(i64)], C.c_int),
        "voxl_mres_get_state": ([vp, vp], C.c_int),
        "voxl_mres_digest": ([vp, vp], C.c_int),
        "voxl_mres_set_state": ([vp, vp], C.c_int),
        "voxl_mres_set_equilibrium": ([vp, C.c_double, C.POINTER(C.c_double)], C.c_int),
        "voxl_mres_probe": ([vp, C.POINTER(Diag)], C.c_int),
        "voxl_mres_step_probe_n": ([vp, C.c_int, C.POINTER(Diag), C.POINTER(C.c_int)], C.c_int),
        "voxl_mres_total_mass": ([vp, C.POINTER(C.c_double)], C.c_int),
        "voxl_mres_text": ([vp, C.c_int, cp, i64, C.POINTER(i64)], C.c_int),
        "voxl_mres_level_info": ([vp, C.c_int, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(i64),
                                  C.POINTER(i64)], C.c_int),
        "voxl_mres_lup_per_coarse_step": ([vp, C.POINTER(i64)], C.c_int),
        "voxl_mres_plan_create": ([C.POINTER(MresDesc), vp, C.POINTER(vp)], C.c_int),
        "voxl_mres_plan_destroy": ([vp], C.c_int),
        "voxl_mres_plan_level": ([vp, C.c_int, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
        "voxl_mres_plan_ref_blocks": ([vp, C.c_int, vp, vp, vp], C.c_int),
        "voxl_mres_plan_ghosts": ([vp, C.c_int, vp], C.c_int),
        "voxl_mres_plan_pulls": ([vp, C.c_int, vp], C.c_int),
        "voxl_mres_plan_jump_distance": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)], C.c_int),
        "voxl_mres_plan_text": ([vp, C.c_int, cp, i64, C.POINTER(i64)], C.c_int),
        "voxl_ipc_export": ([vp, vp], C.c_int),
        "voxl_ipc_open": ([vp, C.POINTER(vp)], C.c_int),
        "voxl_ipc_close": ([vp], C.c_int),
        "voxl_enable_peer_access": ([C.c_int], C.c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def check(status: int) -> None:
    if status != OK:
        msg = lib.voxl_last_error().decode()
        raise _EXC.get(status, VoxlError)(msg)


def probe_rows(fn, h, n: int):
    """n probed steps through a voxl_*_step_probe_n entry point: the list of
    diagnostics rows. On the first failing step raises VoxlInstability with
    run()'s text; `.rows` holds the rows of the steps before it."""
    rows = (Diag * max(n, 1))()
    done = C.c_int()
    st = fn(h, n, rows, C.byref(done))
    out = [rows[i] for i in range(done.value)]
    if st != OK:
        try:
            check(st)
        except VoxlError as e:
            e.rows = out
            raise
    return out


def text(fn, *args) -> str:
    n = C.c_int64()
    check(fn(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(fn(*args, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()
