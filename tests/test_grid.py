"""Host grid layer of the product (C-ABI, no device needed) vs the reference.

Bit-exact targets (BASELINE north star): layout maps, decomposition, voxel
classification and the halo ledger.
"""
import csv
import io
import json
import os

import numpy as np
import pytest

import oracle as O
import paper_2503_07898_b200 as V

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")


def test_lattice_descriptors_match_golden():
    for nm, kind in (("d2q9", "D2Q9"), ("d3q19", "D3Q19"), ("d3q27", "D3Q27")):
        with open(os.path.join(GOLDEN, f"lattice_{nm}.json")) as f:
            assert V.lattice_json(kind) == f.read()


def test_layout_golden_d2q9():
    with open(os.path.join(GOLDEN, "layout_disag_d2q9.json")) as f:
        assert json.loads(V.layout_json("DisagSoA", (8, 4, 1), "D2Q9", 1)) == json.load(f)


@pytest.mark.parametrize("scheme", ["aos", "soa", "disag"])
def test_layout_golden_d3q19(scheme):
    name = {"aos": "AoS", "soa": "SoA", "disag": "DisagSoA"}[scheme]
    with open(os.path.join(GOLDEN, f"layout_{scheme}_d3q19_4x4x4.json")) as f:
        assert V.layout_json(name, (4, 4, 4), "D3Q19", 2) == f.read()


def test_disag_soa_halo_message_is_one_span():
    """US[p][0:5s) -> LH[p-1], LS[p][0:5s) -> UH[p+1]."""
    doc = json.loads(V.layout_json("DisagSoA", (512, 512, 64), "D3Q19", 2))
    g = {x["tag"]: x for x in doc["groups"]}
    s = 512 * 512
    assert g["UpperHalo"]["offset"] == 0
    assert g["UpperShared"]["component_order"][3] == 0  # down-set {3,8,11,13,16} leads
    assert [g["LowerShared"]["component_order"][c] for c in (4, 9, 12, 14, 17)] == [0, 1, 2, 3, 4]
    recs = V.plan_ledger(0, domain=(512, 512, 512), partitions=8)
    assert len(recs) == 14 and all(r.elements == 5 * s for r in recs)


@needs_ref
@pytest.mark.parametrize("scheme", [0, 1, 2])
@pytest.mark.parametrize("lattice,shape,axis", [(0, (8, 4, 1), 1), (1, (4, 5, 6), 2), (2, (3, 4, 5), 2),
                                                (1, (6, 3, 2), 2), (0, (5, 7, 1), 1)])
def test_layout_addresses_match_reference(scheme, lattice, shape, axis):
    ours = V.layout_addresses(scheme, shape, lattice, axis)
    ref = np.empty_like(ours)
    n = O.ref_lib().vref_layout_addresses(scheme, shape[0], shape[1], shape[2], lattice, axis, ref.ctypes.data)
    assert n == ours.size
    assert np.array_equal(ours, ref)
    # bijection onto [0, total_len)
    assert np.array_equal(np.sort(ours), np.arange(ours.size))
    assert O.ref_text(O.ref_lib().vref_layout_json, scheme, *shape, lattice, 0, axis) == \
        V.layout_json(scheme, shape, lattice, axis)


@needs_ref
@pytest.mark.parametrize("domain,parts,periodic", [((16, 16, 16), 1, False), ((16, 16, 16), 4, False),
                                                   ((10, 10, 10), 3, True), ((8, 8, 21), 8, False)])
def test_decompose_classify_match_reference(domain, parts, periodic):
    ours = V.decompose(domain, parts, 2, periodic)
    slabs = np.empty(2 * parts, np.int32)
    assert O.ref_lib().vref_decompose(*domain, parts, 2, int(periodic), slabs.ctypes.data) == 0
    assert ours == [(int(slabs[2 * p]), int(slabs[2 * p + 1])) for p in range(parts)]
    for p in range(parts):
        cls = V.classify_voxels(domain, parts, p, 2, periodic)
        ref = np.empty_like(cls)
        O.ref_lib().vref_classify_voxels(*domain, parts, 2, int(periodic), p, ref.ctypes.data)
        assert np.array_equal(cls, ref)


def test_decompose_errors_mirror_reference():
    with pytest.raises(V.VoxlInvalidArgument):
        V.decompose((4, 4, 4), 3)
    with pytest.raises(V.VoxlInvalidArgument):
        V.layout_json("DisagSoA", (4, 4, 1), "D3Q19", 2)


def _ref_ledger(cfg):
    r = O.RefRun(cfg)
    rows = list(csv.DictReader(io.StringIO(r.ledger_csv)))
    return [(int(x["step"]), int(x["src"]), int(x["dst"]), int(x["base_src"]), int(x["base_dst"]),
             int(x["elements"])) for x in rows]


@needs_ref
@pytest.mark.parametrize("lattice,domain", [("D3Q19", [16, 16, 16]), ("D2Q9", [16, 24]), ("D3Q27", [8, 8, 16])])
@pytest.mark.parametrize("layout", ["AoS", "SoA", "DisagSoA"])
def test_ledger_matches_reference(lattice, domain, layout):
    cfg = dict(lattice=lattice, domain=domain, tau=0.6, scenario="lid_driven_cavity", velocity=[0.05, 0, 0],
               steps=2, layout=layout, partitions=4)
    ref = _ref_ledger(cfg)
    ours = []
    for step in range(2):
        ours += [(r.step, r.src, r.dst, r.base_src, r.base_dst, r.elements)
                 for r in V.plan_ledger(step, lattice=lattice, domain=domain, layout=layout, partitions=4)]
    assert ours == ref


@needs_ref
def test_ledger_alpha_beta_equals_model():
    """Acceptance C2: per-step (alpha, beta) of interior partitions == layout_params."""
    lib = O.ref_lib()
    import ctypes as C
    for lattice, kind in (("D2Q9", 0), ("D3Q19", 1), ("D3Q27", 2)):
        dom = (32, 32) if lattice == "D2Q9" else (32, 32, 32)
        s = 32 if lattice == "D2Q9" else 32 * 32
        for layout, sch in (("AoS", 0), ("SoA", 1), ("DisagSoA", 2)):
            recs = V.plan_ledger(0, lattice=lattice, domain=dom, layout=layout, partitions=4)
            for p in (1, 2):
                sent = [r for r in recs if r.src == p]
                a, b = C.c_int64(), C.c_int64()
                lib.vref_layout_params(kind, sch, s, C.byref(a), C.byref(b))
                assert len(sent) == a.value and sum(r.elements for r in sent) == b.value
