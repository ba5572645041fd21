"""The closed step_occ operator set (partition.hpp:169-174): the generic kernels
the reference's partition tests drive through step_occ -- identity
(partition_test.cpp:176-200) and the five-point Jacobi on a 2-component field
(partition_test.cpp:229-274) -- plus the block-sparse identity sweep
(sparse_test.cpp:210-226)."""
import numpy as np
import pytest

import oracle as O
import paper_2503_07898_b200 as V
from paper_2503_07898_b200.dense import plan_ledger

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
LAYOUTS = ["AoS", "SoA", "DisagSoA"]


def _field(n, lo, hi, seed):
    return np.random.default_rng(seed).uniform(lo, hi, n)


# ---- CPU: oracle pinned to the reference, ledgers ------------------------------------

@needs_ref
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("parts", [1, 2, 4])
def test_jacobi2_oracle_matches_reference_step_occ(layout, parts):
    dom = (12, 16, 1)
    init = _field(12 * 16 * 2, -1.0, 1.0, 3210)
    ref, _, _ = O.ref_occ_run("jacobi2", dom, parts, 1, layout, 10, init)
    assert np.array_equal(ref, O.port_jacobi2_run(dom, 10, init))


@needs_ref
def test_jacobi2_oracle_matches_reference_3d_z_slabs():
    dom = (10, 9, 8)
    init = _field(10 * 9 * 8 * 2, -1.0, 1.0, 5)
    ref, _, _ = O.ref_occ_run("jacobi2", dom, 3, 2, "DisagSoA", 6, init)
    assert np.array_equal(ref, O.port_jacobi2_run(dom, 6, init))


@needs_ref
def test_identity_reference_kat_and_our_ledger():
    """partition_test.cpp:176-200: field unchanged, alpha == 2, beta == 2*5*16."""
    init = _field(4 * 4 * 8 * 19, 0.5, 1.5, 11)
    out, alpha, beta = O.ref_occ_run("identity", (4, 4, 8), 2, 2, "DisagSoA", 1, init)
    assert np.array_equal(out, init) and (alpha, beta) == (2, 2 * 5 * 16)
    recs = plan_ledger(0, domain=(4, 4, 8), partitions=2, layout="DisagSoA", op="identity")
    assert (len(recs), sum(r.elements for r in recs)) == (alpha, beta)


@needs_ref
@pytest.mark.parametrize("layout", LAYOUTS)
def test_jacobi2_ledger_matches_reference(layout):
    init = _field(12 * 16 * 2, -1.0, 1.0, 1)
    _, alpha, beta = O.ref_occ_run("jacobi2", (12, 16, 1), 4, 1, layout, 1, init)
    recs = plan_ledger(0, domain=(12, 16), partitions=4, layout=layout, op="jacobi2")
    assert (len(recs), sum(r.elements for r in recs)) == (alpha, beta)


# ---- GPU ------------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("parts", [1, 2, 3])
@pytest.mark.parametrize("halo", ["zero_copy", "copy"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_identity_operator_leaves_field_unchanged(layout, parts, halo, precision):
    dom = (6, 5, 9)
    init = _field(6 * 5 * 9 * 19, 0.5, 1.5, 11)
    e = V.DenseEngine(domain=dom, layout=layout, partitions=parts, halo_mode=halo, precision=precision,
                      op="identity")
    e.set_canonical(init)
    e.step(3)
    want = init if precision == "fp64" else init.astype(np.float32).astype(np.float64)
    assert np.array_equal(e.get_canonical(), want)


@pytest.mark.gpu
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("parts", [1, 2, 4])
@pytest.mark.parametrize("halo", ["zero_copy", "copy"])
def test_jacobi2_partition_invariance_bitwise(layout, parts, halo):
    """partition_test.cpp:229-274 on the device: every (layout, partitions) run is
    bitwise the single-grid oracle."""
    dom = (12, 16)
    init = _field(12 * 16 * 2, -1.0, 1.0, 3210)
    ref = O.port_jacobi2_run(dom, 10, init)
    e = V.DenseEngine(domain=dom, layout=layout, partitions=parts, halo_mode=halo, precision="fp64", op="jacobi2")
    e.set_canonical(init)
    e.step(10)
    assert np.array_equal(e.get_canonical(), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_jacobi2_3d_and_large(precision):
    dom = (300, 130, 6)
    init = _field(300 * 130 * 6 * 2, -1.0, 1.0, 9)
    ref = O.port_jacobi2_run(dom, 25, init)
    e = V.DenseEngine(domain=dom, partitions=3, precision=precision, op="jacobi2")
    e.set_canonical(init)
    e.step(25)
    out = e.get_canonical()
    if precision == "fp64":
        assert np.array_equal(out, ref)
    else:
        assert np.max(np.abs(out - ref)) <= 1e-6


@pytest.mark.gpu
def test_non_lbm_operator_rejects_probe_and_equilibrium():
    e = V.DenseEngine(domain=(8, 8), op="jacobi2")
    with pytest.raises(V.VoxlInvalidArgument):
        e.probe()
    with pytest.raises(V.VoxlInvalidArgument):
        e.set_equilibrium()


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["naive", "disag_bitmask", "disag_mem"])
def test_sparse_identity_sweep(strategy):
    """sparse_test.cpp:210-226: identity sweeps leave the state unchanged; the
    report is the strategy's; the LBM steps afterwards continue as the oracle."""
    dom = (24, 20, 16)
    act = O.obstacle_mask(dom)
    st5 = O.port_sparse_run("D3Q19", dom, 0.7, (0.04, 0, 0), 5, act)
    e = V.SparseEngine(dom, act, block_edge=8, strategy=strategy, precision="fp64")
    e.step(5)
    before = e.get_state()
    e.step_identity(3)
    assert np.array_equal(e.get_state(), before)
    assert np.array_equal(before, O.sparse_canonical(dom, act, st5, 19))
    e.step(4)
    st9 = O.port_sparse_run("D3Q19", dom, 0.7, (0.04, 0, 0), 9, act)
    assert np.array_equal(e.get_state(), O.sparse_canonical(dom, act, st9, 19))
