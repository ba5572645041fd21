"""Block-sparse path: host tables bit-exact vs the reference (CPU) and the CUDA
engine's physics vs the oracle (GPU; fp64 bitwise, fp32 within 1e-5)."""
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2503_07898_b200 as V

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")


def test_obstacle_mask_matches_oracle():
    for dom in [(32, 32, 32), (24, 20, 16), (17, 19, 23)]:
        assert np.array_equal(V.obstacle_mask(dom), O.obstacle_mask(dom))


@needs_ref
@pytest.mark.parametrize("strategy", ["naive", "disag_bitmask", "disag_mem"])
@pytest.mark.parametrize("domain", [(32, 32, 32), (24, 20, 16), (19, 13, 22)])
def test_tables_bit_exact_vs_reference_edge4(strategy, domain):
    cfg = dict(lattice="D3Q19", domain=list(domain), tau=0.7, scenario="flow_over_obstacle",
               velocity=[0.04, 0, 0], steps=0, strategy=strategy)
    ref = O.RefSparse(cfg, 4)
    ours = V.SparsePlan(domain, block_edge=4, strategy=strategy)
    ro, rm, rc = ref.blocks()
    oo, om, oc = ours.blocks()
    assert np.array_equal(ro, oo)
    assert np.array_equal(rm, om[:, 0])
    assert np.array_equal(rc.astype(np.uint8), oc)
    rp, rb, rmi, rcnt = ref.arrangement()
    op, ob, omi, ocnt = ours.arrangement()
    assert np.array_equal(rp, op)
    assert rcnt == ocnt
    if strategy == "disag_bitmask":
        assert np.array_equal(rb, ob)
        assert np.array_equal(rmi, omi)
    assert ref.report_json() == ours.report_json()
    assert ref.num_active == ours.info()["num_active"]


@needs_ref
@pytest.mark.parametrize("edge", [1, 2])
def test_small_edges_match_reference(edge):
    cfg = dict(lattice="D3Q19", domain=[12, 10, 9], tau=0.7, scenario="flow_over_obstacle", velocity=[0.04, 0, 0],
               steps=0, strategy="disag_mem")
    ref = O.RefSparse(cfg, edge)
    ours = V.SparsePlan((12, 10, 9), block_edge=edge, strategy="disag_mem")
    ro, rm, rc = ref.blocks()
    oo, om, oc = ours.blocks()
    assert np.array_equal(ro, oo) and np.array_equal(rm, om[:, 0]) and np.array_equal(rc.astype(np.uint8), oc)


@pytest.mark.parametrize("strategy", ["naive", "disag_bitmask", "disag_mem"])
def test_edge8_tables_properties(strategy):
    dom = (40, 36, 28)
    act = V.obstacle_mask(dom)
    p = V.SparsePlan(dom, act, block_edge=8, strategy=strategy)
    info = p.info()
    assert info["num_active"] == int(act.sum())
    o, m, c = p.blocks()
    # masks cover exactly the active set
    a3 = act.reshape(dom[2], dom[1], dom[0])
    cover = np.zeros_like(a3)
    for (ox, oy, oz), words in zip(o, m):
        bits = np.unpackbits(words.view(np.uint8), bitorder="little").reshape(8, 8, 8)
        sub = cover[oz:oz + 8, oy:oy + 8, ox:ox + 8]
        sub |= bits[: sub.shape[0], : sub.shape[1], : sub.shape[2]]
    assert np.array_equal(cover, a3)
    # classification: boundary iff an active voxel on x == 0 or x == nx-1
    for (ox, oy, oz), cls in zip(o, c):
        face = a3[oz:oz + 8, oy:oy + 8, ox:ox + 8]
        xs = np.arange(ox, ox + face.shape[2])
        expect = bool(face[:, :, (xs == 0) | (xs == dom[0] - 1)].any())
        assert bool(cls) == expect
    if strategy == "disag_mem":
        assert np.all(np.diff(c.astype(int)) <= 0)  # boundary blocks form a prefix
    nbr = p.neighbours()
    assert np.array_equal(nbr[:, 13], np.arange(len(o)))
    rep = json.loads(p.report_json())
    assert rep["strategy"] == strategy


def test_dispatch_plan_table2():
    """Table 2 rows (SPEC sparse examples; sparse.cpp:199-225)."""
    j = json.loads(V.dispatch_plan_json("naive", 10, 20, q=27, block_size=64, s_w=24, s_i=4))
    assert j["kernels"] == [{"name": "combined", "blocks": 30, "cost": 81}]
    assert j["extra_storage_bytes"] == 24 * 20 * 64 and j["indexing"] == "direct"
    j = json.loads(V.dispatch_plan_json("naive", 10, 20, q=27, naive_full_domain_storage=True))
    assert j["extra_storage_bytes"] == 24 * 30 * 64
    j = json.loads(V.dispatch_plan_json("disag_mem", 32, 32, q=19))
    assert [k["blocks"] for k in j["kernels"]] == [32, 32] and j["extra_storage_bytes"] == 0
    assert [k["cost"] for k in j["kernels"]] == [57, 38]
    j = json.loads(V.dispatch_plan_json("disag_bitmask", 32, 32, q=19, block_size=64, s_i=4))
    assert j["extra_storage_bytes"] == 16384 and j["indexing"] == "indirect"
    assert [k["blocks"] for k in j["kernels"]] == [64, 64]


# ---- GPU physics -----------------------------------------------------------------------

def _oracle(dom, steps, tau=0.7):
    act = O.obstacle_mask(dom)
    st = O.port_sparse_run("D3Q19", dom, tau, (0.04, 0, 0), steps, act)
    return O.sparse_canonical(dom, act, st, 19)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["naive", "disag_bitmask", "disag_mem"])
@pytest.mark.parametrize("edge", [4, 8])
@pytest.mark.parametrize("dom", [(32, 32, 32), (24, 20, 16)])
def test_fp64_bitwise_vs_oracle(strategy, edge, dom):
    ref = _oracle(dom, 20)
    e = V.SparseEngine(dom, block_edge=edge, strategy=strategy, precision="fp64")
    e.step(20)
    out = e.get_state()
    assert np.array_equal(out, ref), np.abs(out - ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["naive", "disag_mem"])
def test_d3q27_fp64_bitwise_vs_oracle(strategy):
    dom = (24, 20, 16)
    act = O.obstacle_mask(dom)
    st = O.port_sparse_run("D3Q27", dom, 0.7, (0.04, 0, 0), 10, act)
    ref = O.sparse_canonical(dom, act, st, 27)
    e = V.SparseEngine(dom, block_edge=8, strategy=strategy, precision="fp64", lattice="D3Q27")
    e.step(10)
    assert np.array_equal(e.get_state(), ref)


def _random_mask(rng, dom):
    """Random sparse domain: a few spheres and boxes carved out of the box."""
    nz, ny, nx = dom[2], dom[1], dom[0]
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    act = np.ones((nz, ny, nx), bool)
    for _ in range(int(rng.integers(1, 4))):
        c = rng.uniform(0, 1, 3) * (nx, ny, nz)
        r = rng.uniform(1.5, min(dom) / 3)
        act &= (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2 > r * r
    for _ in range(int(rng.integers(0, 3))):
        lo = rng.integers(0, np.array(dom) - 2)
        hi = lo + rng.integers(1, 6, 3)
        act[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] = False
    return act.astype(np.uint8).reshape(-1)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_random_sparse_domains_all_strategies(seed):
    """sparse_test.cpp:267-302 style property: random domains, every strategy and
    block edge bitwise equal to the oracle (hence to each other)."""
    rng = np.random.default_rng(7000 + seed)
    dom = tuple(int(v) for v in rng.integers(12, 28, 3))
    act = _random_mask(rng, dom)
    st = O.port_sparse_run("D3Q19", dom, 0.7, (0.04, 0, 0), 8, act)
    ref = O.sparse_canonical(dom, act, st, 19)
    for strategy in ("naive", "disag_bitmask", "disag_mem"):
        for edge in (4, 8):
            e = V.SparseEngine(dom, act, block_edge=edge, strategy=strategy, precision="fp64")
            e.step(8)
            assert np.array_equal(e.get_state(), ref), (strategy, edge)
            e.close()


@pytest.mark.gpu
def test_fp64_bitwise_golden():
    z = np.load(os.path.join(GOLDEN, "sparse_obstacle_d3q19_16.npz"))
    cfg = json.loads(str(z["config"]))
    e = V.SparseEngine(tuple(cfg["domain"]), block_edge=8, strategy="disag_mem", precision="fp64")
    e.step(cfg["steps"])
    assert np.array_equal(e.get_state(), z["field"])


@pytest.mark.gpu
def test_set_state_roundtrip_and_continue():
    dom = (24, 20, 16)
    ref10 = _oracle(dom, 10)
    e = V.SparseEngine(dom, block_edge=8, strategy="disag_mem", precision="fp64")
    e.set_state(ref10)
    assert np.array_equal(e.get_state(), ref10)
    e.step(10)
    assert np.array_equal(e.get_state(), _oracle(dom, 20))


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["naive", "disag_mem"])
def test_fp32_tolerance(strategy):
    dom = (64, 48, 48)
    kw = dict(block_edge=8, strategy=strategy)
    e64 = V.SparseEngine(dom, precision="fp64", **kw)
    e32 = V.SparseEngine(dom, precision="fp32", **kw)
    e64.step(300)
    e32.step(300)
    a, b = e64.get_state(), e32.get_state()
    rel = np.abs(a - b) / np.abs(a)
    print("sparse fp32 max rel err after 300 steps:", rel.max())
    assert rel.max() <= 1e-5


@pytest.mark.gpu
def test_probe_matches_oracle():
    dom = (32, 32, 32)
    ref = _oracle(dom, 15)
    m_ref, s_ref = O.port_probe("D3Q19", ref)
    e = V.SparseEngine(dom, block_edge=8, precision="fp64")
    e.step(15)
    d = e.probe()
    assert d.unstable == 0
    assert abs(d.mass - m_ref) <= 1e-12 * m_ref and abs(d.max_speed - s_ref) <= 1e-14


@pytest.mark.gpu
def test_fp32_tolerance_1000_steps():
    """BASELINE tolerance at its stated horizon: fp32 (shifted storage) vs the
    fp64 engine (bitwise = reference) after 1000 steps, regularized x-faces and
    sphere, kernel split."""
    dom = (48, 32, 32)
    kw = dict(block_edge=8, strategy="disag_mem")
    e64 = V.SparseEngine(dom, precision="fp64", **kw)
    e32 = V.SparseEngine(dom, precision="fp32", **kw)
    e64.step(1000)
    e32.step(1000)
    a, b = e64.get_state(), e32.get_state()
    rel = np.abs(a - b) / np.abs(a)
    print("sparse fp32 max rel err after 1000 steps:", rel.max())
    assert rel.max() <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_state_io_multichunk_roundtrip(precision):
    """set_state / get_state of 2.0 M active voxels through the pipelined
    staging (several 64 MiB chunks; fp32 wire format for fp32): stored values
    are exactly R(f - w_i) and read back as double(g) + w_i."""
    dom = (128, 128, 128)
    e = V.SparseEngine(dom, block_edge=8, strategy="disag_mem", precision=precision)
    n = e.num_active
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    rng = np.random.default_rng(3)
    f = (w[None, :] * (1.0 + 0.05 * rng.standard_normal((n, 19)))).reshape(-1)
    e.set_state(f)
    out = e.get_state()
    e.close()
    if precision == "fp64":
        assert np.array_equal(out, f)
    else:
        ww = np.tile(w, n)
        assert np.array_equal(out, (f - ww).astype(np.float32).astype(np.float64) + ww)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["naive", "disag_bitmask", "disag_mem"])
@pytest.mark.parametrize("precision,edge", [("fp64", 8), ("fp32", 8), ("fp64", 4)])
def test_step_probe_equals_step_plus_probe(strategy, precision, edge):
    """The fused probe (per-warp partials of the step kernels) gives the state
    of a plain step and the diagnostics of probe() on it: fp64 to summation
    order, fp32 to the moment rounding (pre- vs post-collision moments)."""
    dom = (40, 32, 24)
    a = V.SparseEngine(dom, block_edge=edge, strategy=strategy, precision=precision)
    b = V.SparseEngine(dom, block_edge=edge, strategy=strategy, precision=precision)
    tol_m, tol_u = (1e-12, 1e-12) if precision == "fp64" else (1e-9, 1e-6)
    for _ in range(6):
        da = a.step_probe()
        b.step(1)
        db = b.probe()
        assert da.unstable == 0 and db.unstable == 0
        assert abs(da.mass - db.mass) <= tol_m * db.mass
        assert abs(da.max_speed - db.max_speed) <= tol_u * db.max_speed + 1e-12
    assert np.array_equal(a.get_state(), b.get_state())
    a.close()
    b.close()


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["naive", "disag_bitmask", "disag_mem"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_step_probe_n_batches(strategy, precision):
    """run_sparse's rows accumulated on the device over a run longer than one
    batch (256 steps) against step + probe() on a twin engine, fields bitwise."""
    dom = (24, 16, 16)
    a = V.SparseEngine(dom, block_edge=8, strategy=strategy, precision=precision)
    b = V.SparseEngine(dom, block_edge=8, strategy=strategy, precision=precision)
    tol_m, tol_u = (1e-12, 1e-12) if precision == "fp64" else (1e-9, 1e-6)
    rows = a.step_probe_n(270)
    assert len(rows) == 270
    for k in range(270):
        b.step(1)
        if k % 53 == 0 or k == 269:
            db = b.probe()
            assert rows[k].unstable == 0 and db.unstable == 0
            assert abs(rows[k].mass - db.mass) <= tol_m * db.mass
            assert abs(rows[k].max_speed - db.max_speed) <= tol_u * db.max_speed + 1e-12
    assert np.array_equal(a.get_state(), b.get_state())
    a.close()
    b.close()


def _sparse_run(dom, strategy, lattice, steps, tma, probe=False):
    import os

    old = os.environ.get("VOXL_SPARSE_TMA")
    os.environ["VOXL_SPARSE_TMA"] = "1" if tma else "0"
    try:
        e = V.SparseEngine(dom, block_edge=8, strategy=strategy, precision="fp32", lattice=lattice)
    finally:
        if old is None:
            del os.environ["VOXL_SPARSE_TMA"]
        else:
            os.environ["VOXL_SPARSE_TMA"] = old
    rows = [(d.mass, d.max_speed) for d in e.step_probe_n(steps)] if probe else None
    if not probe:
        e.step(steps)
    out = e.get_state()
    e.close()
    return out, rows


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["naive", "disag_bitmask", "disag_mem"])
@pytest.mark.parametrize("lattice", ["D3Q19", "D3Q27"])
@pytest.mark.parametrize("probe", [False, True])
def test_tma_block_staging_bitwise(strategy, lattice, probe):
    """The bulk-copy staged kernel (one block per CTA, own populations from
    shared memory) against the register-pull kernel: fields bitwise equal,
    probe rows too (same warps' per-cell terms)."""
    dom = (40, 32, 24)
    a, ra = _sparse_run(dom, strategy, lattice, 25, True, probe)
    b, rb = _sparse_run(dom, strategy, lattice, 25, False, probe)
    assert np.array_equal(a, b)
    if probe:
        assert len(ra) == len(rb) == 25
        for (m1, u1), (m2, u2) in zip(ra, rb):
            assert abs(m1 - m2) <= 1e-12 * m2 and abs(u1 - u2) <= 1e-12 * u2
