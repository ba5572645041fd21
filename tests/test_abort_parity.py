"""run()'s abort text on an unstable run, against the reference library itself.

The reference's run() (solver.cpp:245-255, 285-293, 341-349) steps, probes the
canonical state, and on the first failure throws
"run aborted at step N: " + what(), with what() either probe_field's
"instability at step N, voxel V, population I" (lbm.cpp:124-128) or
macroscopic's "macroscopic: non-positive density" (lattice.cpp:124). A large
population injected into the initial state drives both kinds; the B200 engines
must name the same step, voxel and population, and the rows before the
failure must agree: max |u| to 1e-12 relative, the mass to the reference's own
rounding bound. probe_field sums every population into one fp64 accumulator in
canonical order (lbm.cpp:116-123); recursive summation of n positive terms is
off the exact sum by up to (n - 1) * 2^-53 * sum (Higham, Accuracy and Stability
of Numerical Algorithms, eq. 4.4), and it is biased when many equal terms (the
rest state) are added to a large partial sum -- which the injected populations
make larger. The B200 rows are exact sums of the per-cell moments rounded to
2^-64 (diag_ring.cuh).
"""
import numpy as np
import pytest

import oracle as O
import paper_2503_07898_b200 as V
from paper_2503_07898_b200 import solver as S

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")

# (canonical element, value): instability at step 0 (|f| > 1e3 after the
# collision), non-positive density one step later
INJECT_DENSE = [((3 * 64 + 2 * 8 + 1) * 19 + 0, 1e4), ((3 * 64 + 2 * 8 + 1) * 19 + 5, 1e4),
                ((3 * 64 + 2 * 8 + 1) * 19 + 0, 3000.0), ((5 * 64 + 5 * 8 + 6) * 19 + 3, 2500.0),
                ((2 * 64 + 2 * 8 + 2) * 19 + 7, -5.0)]


def _rows_close(ours, ref, n_terms):
    assert len(ours) == len(ref)
    tol = max(1e-12, n_terms * 2.0 ** -53)
    for (m, u), (rm, ru) in zip(ours, ref):
        assert abs(m - rm) <= tol * abs(rm)
        assert abs(u - ru) <= 1e-12 * max(abs(ru), 1e-300)


def _ours_loop(step_fn, probe_fn, steps):
    """run()'s loop over the B200 engine: the abort text and the rows."""
    rows = []
    for step in range(steps):
        try:
            d = step_fn()
            if probe_fn is not None:
                d = probe_fn()
            S._unstable(d, step)
        except (V.VoxlInstability, RuntimeError) as e:
            return rows, str(e)
        rows.append((d.mass, d.max_speed))
    return rows, ""


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("elem,value", INJECT_DENSE)
@pytest.mark.parametrize("parts,layout", [(1, "DisagSoA"), (3, "DisagSoA"), (2, "SoA"), (2, "AoS")])
def test_dense_abort_text_equals_reference(elem, value, parts, layout):
    cfg = dict(lattice="D3Q19", domain=[8, 8, 8], tau=0.56, scenario="lid_driven_cavity", velocity=[0.05, 0, 0],
               steps=1)
    st = O.ref_initial_state(cfg)
    st[elem] = value
    ref = O.RefDense(cfg, st)
    ref_rows, ref_msg = O.ref_probed_steps(0, ref._h, 20)
    assert ref_msg.startswith("run aborted at step")
    # batched rows (one read-back per batch): the engine's own abort
    e = V.DenseEngine(domain=(8, 8, 8), precision="fp64", partitions=parts, layout=layout)
    e.set_canonical(st)
    with pytest.raises(V.VoxlInstability) as info:
        e.step_probe_n(20)
    assert str(info.value) == ref_msg
    _rows_close([(d.mass, d.max_speed) for d in info.value.rows], ref_rows, st.size)
    e.close()
    # one step at a time (run()'s per-step shape)
    e = V.DenseEngine(domain=(8, 8, 8), precision="fp64", partitions=parts, layout=layout)
    e.set_canonical(st)
    rows, msg = _ours_loop(e.step_probe, None, 20)
    e.close()
    assert msg == ref_msg
    _rows_close(rows, ref_rows, st.size)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("elem,value", [(100 * 19 + 0, 1e4), (300 * 19 + 5, 1e4), (50 * 19, 3000.0)])
@pytest.mark.parametrize("strategy,edge", [("naive", 4), ("disag_mem", 8), ("disag_bitmask", 8)])
def test_sparse_abort_text_equals_reference(elem, value, strategy, edge):
    dom = (16, 16, 16)
    cfg = dict(lattice="D3Q19", domain=list(dom), tau=0.7, scenario="flow_over_obstacle", velocity=[0.04, 0, 0],
               steps=1, strategy=strategy)
    ref = O.RefSparse(cfg)
    st = ref.state()
    st[elem] = value
    ref.set_state(st)
    ref_rows, ref_msg = O.ref_probed_steps(1, ref.h, 10)
    assert ref_msg.startswith("run aborted at step")
    e = V.SparseEngine(dom, V.obstacle_mask(dom), tau=0.7, u_bc=(0.04, 0, 0), block_edge=edge, strategy=strategy,
                       precision="fp64")
    e.set_state(st)
    rows, msg = _ours_loop(e.step_probe, None, 10)
    e.close()
    assert msg == ref_msg
    _rows_close(rows, ref_rows, st.size)
    # batched rows (run_sparse's loop, one read-back per batch)
    e = V.SparseEngine(dom, V.obstacle_mask(dom), tau=0.7, u_bc=(0.04, 0, 0), block_edge=edge, strategy=strategy,
                       precision="fp64")
    e.set_state(st)
    with pytest.raises(V.VoxlInstability) as info:
        e.step_probe_n(10)
    e.close()
    assert str(info.value) == ref_msg
    _rows_close([(d.mass, d.max_speed) for d in info.value.rows], ref_rows, st.size)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("elem,value", [(100 * 19 + 0, 1e4), (300 * 19 + 5, 1e4), (50 * 19, 3000.0),
                                        (2100 * 19 + 2, 1e4)])  # 2100: a coarse (level-1) cell
@pytest.mark.parametrize("fused", [True, False])
def test_multires_abort_text_equals_reference(elem, value, fused):
    dom = (16, 16, 16)
    cfg = dict(lattice="D3Q19", domain=list(dom), tau=0.56, scenario="lid_driven_cavity", velocity=[0.05, 0, 0],
               steps=1, levels=2, fused=fused)
    ref = O.RefMres(cfg)
    st = ref.state()
    st[elem] = value
    ref.set_state(st)
    ref_rows, ref_msg = O.ref_probed_steps(2, ref.h, 10)
    assert ref_msg.startswith("run aborted at step")
    e = V.MultiResEngine(dom, 2, fused=fused, precision="fp64", block_edge=8)
    e.set_state(st)
    rows, msg = _ours_loop(lambda: e.step(1), e.probe, 10)
    e.close()
    assert msg == ref_msg
    _rows_close(rows, ref_rows, st.size)
    # the probe fused into each level's last sub-step, rows once per batch
    for edge in (8, 4):
        e = V.MultiResEngine(dom, 2, fused=fused, precision="fp64", block_edge=edge)
        e.set_state(st)
        with pytest.raises(V.VoxlInstability) as info:
            e.step_probe_n(10)
        e.close()
        assert str(info.value) == ref_msg
        _rows_close([(d.mass, d.max_speed) for d in info.value.rows], ref_rows, st.size)
