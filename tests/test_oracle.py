"""Pin the C restatement oracle (oracle/voxl_oracle.c) before trusting it.

CPU only. The oracle is checked bitwise against (a) the committed golden
fixtures produced by the reference library (tests/golden/make_golden.py) and
(b) where the reference sources exist, the reference library itself
(oracle/_ref/libvoxl_ref.so) on fresh seeded cases.
"""
import json
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return z["field"], z["diagnostics"], json.loads(str(z["config"]))


@pytest.mark.parametrize("name", ["dense_cavity_d3q19_12", "dense_cavity_d2q9_24x16", "dense_cavity_d3q27_8x10x12",
                                  "dense_periodic_d3q19_10"])
def test_dense_oracle_matches_golden(name):
    field, diag, cfg = load(name)
    out = O.port_dense_run(cfg["lattice"], tuple(cfg["domain"]), cfg["tau"], cfg["scenario"], tuple(cfg["velocity"]),
                           cfg["steps"], seed=cfg.get("seed", 42), perturbation=cfg.get("perturbation", 0.0))
    assert out.size == field.size
    assert np.array_equal(out, field), np.abs(out - field).max()
    # diagnostics of the final step (probe_field on the canonical state)
    m, s = O.port_probe(cfg["lattice"], out)
    assert abs(m - diag[-1, 1]) <= 1e-12 * abs(diag[-1, 1])
    assert abs(s - diag[-1, 2]) <= 1e-12


def test_sparse_oracle_matches_golden():
    field, _, cfg = load("sparse_obstacle_d3q19_16")
    dom = tuple(cfg["domain"])
    act = O.obstacle_mask(dom)
    st = O.port_sparse_run("D3Q19", dom, cfg["tau"], tuple(cfg["velocity"]), cfg["steps"], act)
    assert np.array_equal(O.sparse_canonical(dom, act, st, 19), field)


def test_mres_oracle_matches_golden():
    field, _, cfg = load("mres3_cavity_d3q19_16")
    out = O.port_mres_run("D3Q19", tuple(cfg["domain"]), cfg["levels"], cfg["tau"], tuple(cfg["velocity"]),
                          cfg["steps"])
    assert np.array_equal(out, field)


def test_golden_descriptors_match_reference_goldens():
    """The reference's own golden files (proj/tests/golden) equal our regenerated copies."""
    ref_dir = "/root/reference/proj/tests/golden"
    if not os.path.isdir(ref_dir):
        pytest.skip("reference tree absent")
    for name in ("lattice_d2q9.json", "layout_disag_d2q9.json"):
        with open(os.path.join(ref_dir, name)) as a, open(os.path.join(GOLDEN, name)) as b:
            assert json.load(a) == json.load(b)


@needs_ref
@pytest.mark.parametrize("lattice,domain,scenario,tau,steps", [
    ("D3Q19", [16, 16, 16], "lid_driven_cavity", 0.56, 40),
    ("D3Q19", [9, 11, 13], "lid_driven_cavity", 0.7, 25),
    ("D2Q9", [32, 20], "lid_driven_cavity", 0.6, 60),
    ("D3Q27", [10, 9, 8], "lid_driven_cavity", 0.58, 20),
    ("D3Q19", [12, 12, 12], "periodic_box", 0.9, 20),
])
def test_dense_oracle_vs_reference_library(lattice, domain, scenario, tau, steps):
    cfg = dict(lattice=lattice, domain=domain, tau=tau, scenario=scenario, velocity=[0.05, 0.0, 0.0], steps=steps,
               perturbation=0.05 if scenario == "periodic_box" else 0.0, seed=2024)
    ref = O.ref_reference_dense_run(cfg)
    out = O.port_dense_run(lattice, tuple(domain), tau, scenario, (0.05, 0.0, 0.0), steps, seed=2024,
                           perturbation=cfg["perturbation"])
    assert np.array_equal(ref, out)


@needs_ref
def test_initial_state_rng_matches_reference():
    cfg = dict(lattice="D3Q19", domain=[6, 7, 8], scenario="periodic_box", velocity=[0, 0, 0], perturbation=0.1,
               seed=99, steps=0)
    assert np.array_equal(O.ref_initial_state(cfg), O.port_initial_state("D3Q19", (6, 7, 8), "periodic_box", 99, 0.1))


@needs_ref
@pytest.mark.parametrize("strategy", ["naive", "disag_bitmask", "disag_mem"])
def test_sparse_oracle_vs_reference_strategies(strategy):
    cfg = dict(lattice="D3Q19", domain=[24, 20, 16], tau=0.7, scenario="flow_over_obstacle", velocity=[0.04, 0, 0],
               steps=12, strategy=strategy)
    r = O.RefRun(cfg)
    dom = (24, 20, 16)
    act = O.obstacle_mask(dom)
    st = O.port_sparse_run("D3Q19", dom, 0.7, (0.04, 0, 0), 12, act)
    assert np.array_equal(O.sparse_canonical(dom, act, st, 19), r.field)


@needs_ref
@pytest.mark.parametrize("levels,fused", [(2, True), (2, False), (3, True), (3, False)])
def test_mres_oracle_vs_reference(levels, fused):
    cfg = dict(lattice="D3Q19", domain=[32, 32, 32], tau=0.56, scenario="lid_driven_cavity", velocity=[0.05, 0, 0],
               steps=3, levels=levels, fused=fused)
    r = O.RefRun(cfg)
    out = O.port_mres_run("D3Q19", (32, 32, 32), levels, 0.56, (0.05, 0, 0), 3)
    assert np.array_equal(out, r.field)


@needs_ref
def test_mres_oracle_2d_vs_reference():
    cfg = dict(lattice="D2Q9", domain=[32, 32], tau=0.6, scenario="lid_driven_cavity", velocity=[0.05, 0, 0],
               steps=4, levels=3, fused=True)
    r = O.RefRun(cfg)
    out = O.port_mres_run("D2Q9", (32, 32), 3, 0.6, (0.05, 0, 0), 4)
    assert np.array_equal(out, r.field)


@needs_ref
def test_resident_reference_dense_equals_reference_dense_run():
    """RefDense (what bench.py's CPU legs time: create once, sweep, read) is
    reference_dense_run's loop: same bits after the same number of steps."""
    cfg = dict(lattice="D3Q19", domain=[12, 10, 14], tau=0.56, scenario="lid_driven_cavity",
               velocity=[0.05, 0, 0], steps=9)
    r = O.RefDense(cfg, O.ref_initial_state(cfg))
    r.step(4)
    r.step(5)
    assert np.array_equal(r.state(), O.ref_reference_dense_run(cfg))
    r.close()
