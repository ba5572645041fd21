"""ctypes bindings for the CPU checkers under oracle/_ref/ (TEST INFRASTRUCTURE ONLY).

Two libraries, both built by oracle/Makefile:

* ``libvoxl_ref.so``   -- the UNMODIFIED reference library compiled from
  /root/reference/proj/src plus ref_shim.cpp (the reference's own C++ API).
* ``libvoxl_oracle.so`` -- voxl_oracle.c, the plain-C restatement of the path.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / --impl
reference legs may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

LATTICES = {"D2Q9": 0, "D3Q19": 1, "D3Q27": 2}
Q_OF = {"D2Q9": 9, "D3Q19": 19, "D3Q27": 27}
SCENARIOS = {"lid_driven_cavity": 0, "flow_over_obstacle": 1, "periodic_box": 2}
LAYOUTS = {"AoS": 0, "SoA": 1, "DisagSoA": 2}

_dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    """Build the checkers (port always; the reference only where its sources exist)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref", "-j8"], check=True)


def build_dropin() -> None:
    """The drop-in test driver (reference run() vs voxl::b200::run on the
    reference's types); needs the reference sources and the built libvoxl_b200."""
    import subprocess

    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "dropin"], check=True)


def dropin_driver():
    """Path of the prebuilt drop-in driver, or None."""
    p = os.path.join(REF_DIR, "dropin_reference")
    return p if os.path.exists(p) else None


_port = None
_ref = None


def port_lib():
    global _port
    if _port is None:
        lib = C.CDLL(os.path.join(REF_DIR, "libvoxl_oracle.so"))
        lib.vo_rules_for.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_void_p]
        lib.vo_initial_state.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_double, _dp]
        lib.vo_dense_run.argtypes = [C.c_int, C.c_void_p, C.c_double, C.c_int, _dp]
        lib.vo_probe.argtypes = [C.c_int, _dp, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        lib.vo_sparse_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_double, _dp, C.c_int, _dp]
        lib.vo_obstacle_mask.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p]
        lib.vo_obstacle_mask.restype = C.c_int64
        lib.vo_mres_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_double, _dp,
                                    C.c_int, C.c_void_p, C.c_int64]
        lib.vo_mres_run.restype = C.c_int64
        lib.vo_band_level_map.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        lib.vo_jacobi2_run.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libvoxl_ref.so"))


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(os.path.join(REF_DIR, "libvoxl_ref.so"))
        vp, cp, i64 = C.c_void_p, C.c_char_p, C.c_int64
        lib.vref_last_error.restype = cp
        lib.vref_run.argtypes = [cp]
        lib.vref_run.restype = vp
        lib.vref_run_field_len.argtypes = [vp]
        lib.vref_run_field_len.restype = i64
        lib.vref_run_field.argtypes = [vp, _dp]
        lib.vref_run_diag_rows.argtypes = [vp]
        lib.vref_run_diag.argtypes = [vp, _dp]
        lib.vref_run_text.argtypes = [vp, C.c_int, C.c_char_p, i64]
        lib.vref_run_free.argtypes = [vp]
        lib.vref_reference_dense_run.argtypes = [cp, _dp]
        lib.vref_dense_steps_from.argtypes = [cp, _dp, _dp]
        lib.vref_dense_create.argtypes = [cp, _dp]
        lib.vref_dense_create.restype = vp
        lib.vref_dense_step.argtypes = [vp, C.c_int]
        lib.vref_dense_read.argtypes = [vp, _dp]
        lib.vref_dense_free.argtypes = [vp]
        lib.vref_occ_run.argtypes = [C.c_int] * 9 + [_dp, _dp, C.POINTER(i64), C.POINTER(i64)]
        lib.vref_initial_state.argtypes = [cp, _dp]
        lib.vref_probe.argtypes = [C.c_int, _dp, i64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.vref_lattice_json.argtypes = [C.c_int, C.c_char_p, i64]
        lib.vref_layout_json.argtypes = [C.c_int] * 7 + [C.c_char_p, i64]
        lib.vref_layout_addresses.argtypes = [C.c_int] * 6 + [vp]
        lib.vref_decompose.argtypes = [C.c_int] * 6 + [vp]
        lib.vref_classify_voxels.argtypes = [C.c_int] * 7 + [vp]
        lib.vref_layout_params.argtypes = [C.c_int, C.c_int, i64, C.POINTER(i64), C.POINTER(i64)]
        lib.vref_sparse_create.argtypes = [cp, C.c_int]
        lib.vref_sparse_create.restype = vp
        lib.vref_sparse_free.argtypes = [vp]
        lib.vref_sparse_step.argtypes = [vp, C.c_int]
        lib.vref_sparse_num_active.argtypes = [vp]
        lib.vref_sparse_num_active.restype = i64
        lib.vref_sparse_num_blocks.argtypes = [vp]
        lib.vref_sparse_blocks.argtypes = [vp, vp, vp, vp]
        lib.vref_sparse_arrangement.argtypes = [vp, vp, vp, vp]
        lib.vref_sparse_arrangement.restype = i64
        lib.vref_sparse_report_json.argtypes = [vp, C.c_char_p, i64]
        lib.vref_sparse_state.argtypes = [vp, _dp]
        lib.vref_sparse_set_state.argtypes = [vp, _dp]
        lib.vref_mres_create.argtypes = [cp]
        lib.vref_mres_create.restype = vp
        lib.vref_mres_free.argtypes = [vp]
        lib.vref_mres_step.argtypes = [vp, C.c_int]
        lib.vref_mres_levels.argtypes = [vp]
        lib.vref_mres_num_active.argtypes = [vp, C.c_int]
        lib.vref_mres_num_active.restype = i64
        lib.vref_mres_num_blocks.argtypes = [vp, C.c_int]
        lib.vref_mres_tau.argtypes = [vp, C.c_int]
        lib.vref_mres_tau.restype = C.c_double
        lib.vref_mres_blocks.argtypes = [vp, C.c_int, vp, vp, vp]
        lib.vref_mres_num_ghosts.argtypes = [vp, C.c_int]
        lib.vref_mres_ghosts.argtypes = [vp, C.c_int, vp]
        lib.vref_mres_num_pulls.argtypes = [vp, C.c_int]
        lib.vref_mres_pulls.argtypes = [vp, C.c_int, vp]
        lib.vref_mres_state_len.argtypes = [vp]
        lib.vref_mres_state_len.restype = i64
        lib.vref_mres_state.argtypes = [vp, _dp]
        lib.vref_mres_total_mass.argtypes = [vp]
        lib.vref_mres_total_mass.restype = C.c_double
        lib.vref_mres_text.argtypes = [vp, C.c_int, C.c_char_p, i64]
        lib.vref_mres_set_state.argtypes = [vp, _dp]
        lib.vref_probed_steps.argtypes = [C.c_int, vp, C.c_int, _dp, C.c_char_p, i64]
        _ref = lib
    return _ref


def ref_error() -> str:
    return ref_lib().vref_last_error().decode()


def config_json(**kw) -> str:
    """A reference SolverConfig document (solver.cpp:59-99 keys)."""
    return json.dumps(kw)


# ---- port (C restatement) ---------------------------------------------------------

class _Rules(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("periodic", C.c_int * 3), ("wrap", C.c_int * 3),
                ("has_lid", C.c_int), ("lid_axis", C.c_int), ("lid_at_max", C.c_int),
                ("lid_u", C.c_double * 3)]


def _dims(domain):
    nx, ny = domain[0], domain[1]
    nz = domain[2] if len(domain) == 3 else 1
    return nx, ny, nz


def port_initial_state(lattice="D3Q19", domain=(32, 32, 32), scenario="lid_driven_cavity",
                       seed=42, perturbation=0.0) -> np.ndarray:
    nx, ny, nz = _dims(domain)
    out = np.empty(nx * ny * nz * Q_OF[lattice], np.float64)
    port_lib().vo_initial_state(LATTICES[lattice], SCENARIOS[scenario], nx, ny, nz, seed, perturbation, out)
    return out


def port_dense_run(lattice="D3Q19", domain=(32, 32, 32), tau=0.56, scenario="lid_driven_cavity",
                   velocity=(0.05, 0.0, 0.0), steps=10, state=None, seed=42, perturbation=0.0) -> np.ndarray:
    """reference_dense_run restated (solver.cpp:189-206)."""
    nx, ny, nz = _dims(domain)
    lib = port_lib()
    r = _Rules()
    lib.vo_rules_for(LATTICES[lattice], SCENARIOS[scenario], nx, ny, nz,
                     np.asarray(velocity, np.float64), C.byref(r))
    if state is None:
        state = port_initial_state(lattice, domain, scenario, seed, perturbation)
    state = np.array(state, np.float64, copy=True)
    rc = lib.vo_dense_run(LATTICES[lattice], C.byref(r), tau, steps, state)
    if rc:
        raise RuntimeError("oracle dense run failed (non-positive density / non-finite state)")
    return state


def port_probe(lattice, canonical):
    q = Q_OF[lattice]
    m, s = C.c_double(), C.c_double()
    bv, bp = C.c_int64(), C.c_int()
    rc = port_lib().vo_probe(LATTICES[lattice], np.ascontiguousarray(canonical, np.float64),
                             canonical.size // q, C.byref(m), C.byref(s), C.byref(bv), C.byref(bp))
    if rc:
        raise RuntimeError(f"instability: voxel {bv.value}, population {bp.value}")
    return m.value, s.value


def obstacle_mask(domain, radius=0.0) -> np.ndarray:
    nx, ny, nz = _dims(domain)
    m = np.empty(nx * ny * nz, np.uint8)
    port_lib().vo_obstacle_mask(nx, ny, nz, radius, m.ctypes.data)
    return m


def port_sparse_run(lattice="D3Q19", domain=(32, 32, 32), tau=0.7, velocity=(0.04, 0.0, 0.0), steps=10,
                    active=None, state=None) -> np.ndarray:
    """SparseLbmEngine::step restated over a dense mask; returns the dense (x fastest)
    population array (inactive voxels carry their initial values)."""
    nx, ny, nz = _dims(domain)
    q = Q_OF[lattice]
    if active is None:
        active = obstacle_mask(domain)
    if state is None:
        w = port_initial_state(lattice, (1, 1, 1) if len(domain) == 3 else (1, 1), "lid_driven_cavity")
        state = np.tile(w, nx * ny * nz)
    state = np.array(state, np.float64, copy=True)
    rc = port_lib().vo_sparse_run(LATTICES[lattice], nx, ny, nz, np.ascontiguousarray(active, np.uint8).ctypes.data,
                                  tau, np.asarray(velocity, np.float64), steps, state)
    if rc:
        raise RuntimeError("oracle sparse run failed")
    return state


def sparse_canonical(domain, active, dense_state, q) -> np.ndarray:
    """Active voxels sorted by pack_coord (x slowest, z fastest) -- sparse.cpp:416-438."""
    nx, ny, nz = _dims(domain)
    st = dense_state.reshape(nz, ny, nx, q)
    act = active.reshape(nz, ny, nx).astype(bool)
    # transpose to (x, y, z) so C-order iteration is x slowest, z fastest
    st_t = st.transpose(2, 1, 0, 3)
    act_t = act.transpose(2, 1, 0)
    return st_t[act_t].reshape(-1)


def band_level_map(domain, levels, axis=2) -> np.ndarray:
    nx, ny, nz = _dims(domain)
    m = np.empty(nx * ny * nz, np.int32)
    port_lib().vo_band_level_map(nx, ny, nz, levels, axis, m.ctypes.data)
    return m


def port_mres_run(lattice="D3Q19", domain=(32, 32, 32), levels=3, tau=0.56, velocity=(0.05, 0.0, 0.0),
                  steps=2, level_map=None) -> np.ndarray:
    nx, ny, nz = _dims(domain)
    if level_map is None:
        level_map = band_level_map(domain, levels, 2 if len(domain) == 3 else 1)
    lib = port_lib()
    lm = np.ascontiguousarray(level_map, np.int32)
    n = lib.vo_mres_run(LATTICES[lattice], nx, ny, nz, levels, lm.ctypes.data, tau,
                        np.asarray(velocity, np.float64), 0, None, 0)
    out = np.empty(n, np.float64)
    lib.vo_mres_run(LATTICES[lattice], nx, ny, nz, levels, lm.ctypes.data, tau,
                    np.asarray(velocity, np.float64), steps, out.ctypes.data, n)
    return out


def port_jacobi2_run(domain, steps, state) -> np.ndarray:
    """Five-point Jacobi of partition_test.cpp:234-247 on one grid (2 components)."""
    nx, ny, nz = _dims(domain)
    out = np.array(state, np.float64, copy=True)
    port_lib().vo_jacobi2_run(nx, ny, nz, steps, out)
    return out


# ---- reference library ------------------------------------------------------------

OPS = {"identity": 1, "jacobi2": 2}


def ref_occ_run(op, domain, parts, axis, layout, steps, init, lattice="D3Q19"):
    """step_occ (partition.hpp:173) over a PartitionedField pair with the reference
    tests' identity / Jacobi kernels -> (canonical result, step-0 ledger alpha, beta)."""
    nx, ny, nz = _dims(domain)
    out = np.empty_like(np.ascontiguousarray(init, np.float64))
    a, b = C.c_int64(), C.c_int64()
    schemes = {"AoS": 0, "SoA": 1, "DisagSoA": 2}
    if ref_lib().vref_occ_run(OPS[op], LATTICES[lattice], nx, ny, nz, parts, axis, schemes[layout], steps,
                              np.ascontiguousarray(init, np.float64), out, C.byref(a), C.byref(b)):
        raise RuntimeError(ref_error())
    return out, a.value, b.value

def ref_reference_dense_run(cfg: dict) -> np.ndarray:
    lib = ref_lib()
    nx, ny, nz = _dims(cfg["domain"])
    out = np.empty(nx * ny * nz * Q_OF[cfg.get("lattice", "D3Q19")], np.float64)
    if lib.vref_reference_dense_run(json.dumps(cfg).encode(), out):
        raise RuntimeError(ref_error())
    return out


def ref_dense_steps_from(cfg: dict, init: np.ndarray) -> np.ndarray:
    out = np.empty_like(init)
    if ref_lib().vref_dense_steps_from(json.dumps(cfg).encode(), np.ascontiguousarray(init), out):
        raise RuntimeError(ref_error())
    return out


class RefDense:
    """A resident reference dense state (reference_dense_run's loop,
    solver.cpp:189-206, split into create / step / read): the reference's own
    fused_stream_collide sweeps without per-call allocation or copies."""

    def __init__(self, cfg: dict, init: np.ndarray):
        self.n = init.size
        self._h = ref_lib().vref_dense_create(json.dumps(cfg).encode(), np.ascontiguousarray(init, np.float64))
        if not self._h:
            raise RuntimeError(ref_error())

    def step(self, n=1):
        if ref_lib().vref_dense_step(self._h, n):
            raise RuntimeError(ref_error())

    def state(self) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        ref_lib().vref_dense_read(self._h, out)
        return out

    def close(self):
        if self._h:
            ref_lib().vref_dense_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


def ref_probed_steps(kind: int, handle, steps: int):
    """run()'s per-step loop (step + probe_field, solver.cpp:245-255) on a
    resident reference engine (kind 0 RefDense, 1 RefSparse, 2 RefMres):
    (rows [(mass, max_speed)], abort text or "")."""
    diag = np.zeros(2 * max(steps, 1), np.float64)
    msg = C.create_string_buffer(512)
    done = ref_lib().vref_probed_steps(kind, handle, steps, diag, msg, 512)
    return [(diag[2 * i], diag[2 * i + 1]) for i in range(done)], msg.value.decode()


def ref_initial_state(cfg: dict) -> np.ndarray:
    nx, ny, nz = _dims(cfg["domain"])
    out = np.empty(nx * ny * nz * Q_OF[cfg.get("lattice", "D3Q19")], np.float64)
    if ref_lib().vref_initial_state(json.dumps(cfg).encode(), out):
        raise RuntimeError(ref_error())
    return out


class RefRun:
    """voxl::run(config) result (solver.cpp:369)."""

    def __init__(self, cfg: dict):
        lib = ref_lib()
        self._h = lib.vref_run(json.dumps(cfg).encode())
        if not self._h:
            raise RuntimeError(ref_error())
        n = lib.vref_run_field_len(self._h)
        self.field = np.empty(n, np.float64)
        lib.vref_run_field(self._h, self.field)
        rows = lib.vref_run_diag_rows(self._h)
        d = np.empty(max(rows, 1) * 3, np.float64)
        lib.vref_run_diag(self._h, d)
        self.diagnostics = d[: rows * 3].reshape(rows, 3)
        self.ledger_csv = self._text(0)
        self.trace_json = self._text(1)
        self.dispatch_json = self._text(2)
        self.graph_dot = self._text(3)
        self.distribution = self._text(4)
        self.header_json = self._text(5)
        self.diagnostics_csv = self._text(6)
        lib.vref_run_free(self._h)
        self._h = None

    def _text(self, what):
        lib = ref_lib()
        n = lib.vref_run_text(self._h, what, None, 0)
        buf = C.create_string_buffer(n + 1)
        lib.vref_run_text(self._h, what, buf, n + 1)
        return buf.value.decode()


def ref_text(fn, *args) -> str:
    n = fn(*args, None, 0)
    if n < 0:
        raise RuntimeError(ref_error())
    buf = C.create_string_buffer(n + 1)
    fn(*args, buf, n + 1)
    return buf.value.decode()


class RefSparse:
    def __init__(self, cfg: dict, block_edge=4):
        lib = ref_lib()
        self.lib = lib
        self.h = lib.vref_sparse_create(json.dumps(cfg).encode(), block_edge)
        if not self.h:
            raise RuntimeError(ref_error())
        self.q = Q_OF[cfg.get("lattice", "D3Q19")]

    def step(self, n=1):
        if self.lib.vref_sparse_step(self.h, n):
            raise RuntimeError(ref_error())

    @property
    def num_active(self):
        return self.lib.vref_sparse_num_active(self.h)

    def blocks(self):
        nb = self.lib.vref_sparse_num_blocks(self.h)
        o = np.empty((nb, 3), np.int32)
        m = np.empty(nb, np.uint64)
        c = np.empty(nb, np.int32)
        self.lib.vref_sparse_blocks(self.h, o.ctypes.data, m.ctypes.data, c.ctypes.data)
        return o, m, c

    def arrangement(self, block_volume=64):
        nb = self.lib.vref_sparse_num_blocks(self.h)
        perm = np.empty(nb, np.int32)
        bm = np.zeros(nb, np.uint8)
        mi = np.full(nb * block_volume, -1, np.int32)
        cnt = self.lib.vref_sparse_arrangement(self.h, perm.ctypes.data, bm.ctypes.data, mi.ctypes.data)
        return perm, bm, mi, cnt

    def report_json(self):
        return ref_text(self.lib.vref_sparse_report_json, self.h)

    def state(self):
        out = np.empty(self.num_active * self.q, np.float64)
        self.lib.vref_sparse_state(self.h, out)
        return out

    def set_state(self, canonical):
        self.lib.vref_sparse_set_state(self.h, np.ascontiguousarray(canonical, np.float64))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.vref_sparse_free(self.h)
            self.h = None


class RefMres:
    def __init__(self, cfg: dict):
        lib = ref_lib()
        self.lib = lib
        self.h = lib.vref_mres_create(json.dumps(cfg).encode())
        if not self.h:
            raise RuntimeError(ref_error())

    def step(self, n=1):
        if self.lib.vref_mres_step(self.h, n):
            raise RuntimeError(ref_error())

    @property
    def levels(self):
        return self.lib.vref_mres_levels(self.h)

    def tau(self, l):
        return self.lib.vref_mres_tau(self.h, l)

    def num_active(self, l):
        return self.lib.vref_mres_num_active(self.h, l)

    def blocks(self, l):
        nb = self.lib.vref_mres_num_blocks(self.h, l)
        o = np.empty((nb, 3), np.int32)
        m = np.empty(nb, np.uint64)
        c = np.empty(nb, np.int32)
        self.lib.vref_mres_blocks(self.h, l, o.ctypes.data, m.ctypes.data, c.ctypes.data)
        return o, m, c

    def ghosts(self, l):
        n = self.lib.vref_mres_num_ghosts(self.h, l)
        out = np.empty((n, 6), np.int32)
        self.lib.vref_mres_ghosts(self.h, l, out.ctypes.data)
        return out

    def pulls(self, l):
        n = self.lib.vref_mres_num_pulls(self.h, l)
        out = np.empty((n, 7), np.int32)
        self.lib.vref_mres_pulls(self.h, l, out.ctypes.data)
        return out

    def state(self):
        n = self.lib.vref_mres_state_len(self.h)
        out = np.empty(n, np.float64)
        self.lib.vref_mres_state(self.h, out)
        return out

    def set_state(self, canonical):
        self.lib.vref_mres_set_state(self.h, np.ascontiguousarray(canonical, np.float64))

    def total_mass(self):
        return self.lib.vref_mres_total_mass(self.h)

    def graph_dot(self):
        return ref_text(self.lib.vref_mres_text, self.h, 0)

    def distribution(self):
        return ref_text(self.lib.vref_mres_text, self.h, 1)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.vref_mres_free(self.h)
            self.h = None
