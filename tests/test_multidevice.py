"""Single-process multi-device dense engine (voxl_dense_create_multi).

The reference holds every partition in one process (PartitionedField,
partition.hpp:92-126) and steps them with step_occ; the B200 engine places
partition p on devices[p] and runs the two-stream OCC schedule per partition,
ordered across partitions by cross-device events, optionally replayed from a
captured CUDA graph. This box has one GPU, so the schedule runs with every
partition on device 0 (its own streams and events per partition, the same
code path as distinct devices); the >= 2-GPU cases run where the devices exist.

Parity: fp64 bitwise against the oracle / the one-stream engine; fp32 bitwise
against the one-stream engine (same kernels, same per-voxel arithmetic).
"""
import numpy as np
import pytest

import oracle as O
import paper_2503_07898_b200 as V

pytestmark = pytest.mark.gpu


def _device_count():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


def _run(steps, init, dom=(24, 20, 32), scenario="lid_driven_cavity", tau=0.56, vel=(0.05, 0, 0), **kw):
    e = V.DenseEngine("D3Q19", dom, tau, scenario, vel, **kw)
    e.set_canonical(init)
    e.step(steps)
    out = e.get_canonical()
    e.close()
    return out


@pytest.mark.parametrize("layout", ["AoS", "SoA", "DisagSoA"])
@pytest.mark.parametrize("parts", [1, 2, 3, 4])
@pytest.mark.parametrize("halo", ["zero_copy", "copy"])
@pytest.mark.parametrize("graph_steps", [0, 8])
def test_multi_schedule_fp64_bitwise_vs_oracle(layout, parts, halo, graph_steps):
    dom = (24, 20, 32)
    init = O.port_initial_state("D3Q19", dom)
    ref = O.port_dense_run("D3Q19", dom, 0.56, "lid_driven_cavity", (0.05, 0, 0), 21)
    out = _run(21, init, dom, precision="fp64", layout=layout, partitions=parts, halo_mode=halo,
               devices=[0] * parts, graph_steps=graph_steps)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("parts", [1, 2, 3])
def test_multi_schedule_periodic_fp64(parts):
    dom = (12, 10, 14)
    init = O.port_initial_state("D3Q19", dom, "periodic_box", 7, 0.05)
    ref = O.port_dense_run("D3Q19", dom, 0.8, "periodic_box", (0, 0, 0), 25, seed=7, perturbation=0.05)
    out = _run(25, init, dom, "periodic_box", 0.8, (0, 0, 0), precision="fp64", partitions=parts,
               devices=[0] * parts)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("parts", [2, 4])
def test_multi_schedule_fp32_equals_one_stream_engine(parts):
    dom = (64, 48, 40)
    init = O.port_initial_state("D3Q19", dom)
    a = _run(30, init, dom, precision="fp32", partitions=parts)
    b = _run(30, init, dom, precision="fp32", partitions=parts, devices=[0] * parts)
    assert np.array_equal(a, b)


def test_multi_schedule_d2q9_and_d3q27():
    for lat, dom in (("D2Q9", (24, 30, 1)), ("D3Q27", (10, 12, 16))):
        init = O.port_initial_state(lat, dom)
        ref = O.port_dense_run(lat, dom, 0.6, "lid_driven_cavity", (0.05, 0, 0), 12)
        e = V.DenseEngine(lat, dom, 0.6, "lid_driven_cavity", (0.05, 0, 0), precision="fp64", partitions=3,
                          devices=[0, 0, 0], graph_steps=4)
        e.set_canonical(init)
        e.step(12)
        assert np.array_equal(e.get_canonical(), ref), lat
        e.close()


@pytest.mark.parametrize("parts", [1, 3])
def test_multi_probe_rows_equal_one_stream_rows(parts):
    """run()'s per-step rows (one ring per device, integer sums combined on the
    host) are bit-identical to the one-stream engine's."""
    dom = (32, 32, 32)
    init = O.port_initial_state("D3Q19", dom)
    rows = []
    for devices in (None, [0] * parts):
        e = V.DenseEngine("D3Q19", dom, precision="fp64", partitions=parts, devices=devices)
        e.set_canonical(init)
        rows.append([(d.mass, d.max_speed) for d in e.step_probe_n(40)])
        e.close()
    assert rows[0] == rows[1]


def test_multi_abort_step_under_graph_replay():
    """A failing voxel inside a replayed graph reports the absolute step (the
    graph's kernels read the step base from the device)."""
    dom = (8, 8, 8)
    st = O.port_initial_state("D3Q19", dom)
    st[(3 * 64 + 2 * 8 + 1) * 19 + 0] = 3000.0  # non-positive density one step after loading
    msgs = []
    for kw in ({}, {"devices": [0, 0], "graph_steps": 2}):
        e = V.DenseEngine("D3Q19", dom, precision="fp64", partitions=2, **kw)
        e.set_canonical(O.port_initial_state("D3Q19", dom))
        e.step(3)  # the replays start at an odd step, parity 1
        e.set_canonical(st)
        with pytest.raises(V.VoxlInstability) as info:
            e.step(40)
        msgs.append(str(info.value))
        e.close()
    assert msgs[0] == msgs[1]
    assert msgs[0].startswith("run aborted at step ")


def test_neighbor_links_symmetry_check():
    """partition_test.cpp:167-174: a broken link is rejected at the next halo update."""
    e = V.DenseEngine("D3Q19", (4, 4, 8), precision="fp64", partitions=2, layout="SoA")
    assert e.neighbors(0) == (-1, 1) and e.neighbors(1) == (0, -1)
    e.set_neighbor_links(0, -1, -1)
    with pytest.raises(V.VoxlError, match="halo_update: asymmetric neighbor links"):
        e.step(1)
    e.close()
    m = V.DenseEngine("D3Q19", (4, 4, 8), precision="fp64", partitions=2, devices=[0, 0])
    m.set_neighbor_links(1, -1, -1)
    with pytest.raises(V.VoxlError, match="asymmetric"):
        m.step(1)
    m.close()


def test_device_placement_and_argument_errors():
    e = V.DenseEngine("D3Q19", (8, 8, 12), partitions=3, devices=[0, 0, 0])
    assert [e.device(p) for p in range(3)] == [0, 0, 0]
    e.close()
    with pytest.raises(V.VoxlInvalidArgument, match="does not exist"):
        V.DenseEngine("D3Q19", (8, 8, 12), partitions=2, devices=[0, 4096])
    with pytest.raises(V.VoxlInvalidArgument, match="graph_steps"):
        V.DenseEngine("D3Q19", (8, 8, 12), partitions=2, devices=[0, 0], graph_steps=3)
    with pytest.raises(V.VoxlInvalidArgument, match="one distinct device per partition"):
        V.DenseEngine("D3Q19", (8, 8, 12), partitions=2, devices=[0, 0], halo_mode="nccl")
    with pytest.raises(V.VoxlInvalidArgument, match="multi-device"):
        V.DenseEngine("D3Q19", (8, 8, 12), partitions=2, halo_mode="nccl")


@pytest.mark.skipif(_device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("halo", ["zero_copy", "copy", "nccl"])
def test_two_devices_bitwise(halo):
    n = _device_count()
    parts = min(n, 4)
    dom = (32, 24, 8 * parts)
    init = O.port_initial_state("D3Q19", dom)
    ref = O.port_dense_run("D3Q19", dom, 0.56, "lid_driven_cavity", (0.05, 0, 0), 20)
    out = _run(20, init, dom, precision="fp64", partitions=parts, halo_mode=halo, devices=list(range(parts)))
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("devices,halo", [(None, "zero_copy"), (None, "copy"), ([0, 0, 0], "zero_copy"),
                                          ([0, 0, 0], "copy")])
def test_observed_trace_lists_the_executed_schedule(devices, halo):
    """The observed TraceLog (voxl_dense_trace_json): one record per launched
    phase, in launch order, with device-measured, ordered times -- the
    single-stream schedule launches one "step" kernel per partition (plus a
    "halo_copy" phase in copy mode), the multi-device OCC schedule "interior"
    and "shared" kernels per partition on their two streams."""
    import json

    dom = (16, 12, 24)
    kw = dict(devices=devices) if devices else {}
    e = V.DenseEngine("D3Q19", dom, 0.6, "lid_driven_cavity", (0.05, 0, 0), partitions=3, halo_mode=halo, **kw)
    e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
    e.trace(True)
    e.step(2)
    rec = json.loads(e.trace_json())
    e.trace(False)
    assert json.loads(e.trace_json()) == []
    e.close()
    if devices is None:
        want = []
        for s in range(2):
            want += [(s, 1, "step", p) for p in range(3)]
            if halo == "copy":
                want.append((s, 2, "halo_copy", -1))
    else:
        want = []
        for s in range(2):
            want += [(s, 1, "interior", p) for p in range(3)]
            for p in range(3):
                want.append((s, 2, "shared", p))
                if halo == "copy":
                    want.append((s, 2, "halo_copy", p))
    assert [(r["step"], r["stage"], r["phase"], r["partition"]) for r in rec] == want
    for r in rec:
        assert 0.0 <= r["begin_ms"] <= r["end_ms"]
        assert r["device"] == 0
    # a partition's step s+1 work starts after its step s work ended (same stream order)
    by = {}
    for r in rec:
        by.setdefault((r["phase"], r["partition"]), []).append(r)
    for rs in by.values():
        for a, b in zip(rs, rs[1:]):
            assert b["begin_ms"] >= a["end_ms"] - 1e-3


@pytest.mark.parametrize("layout", ["AoS", "DisagSoA"])
@pytest.mark.parametrize("halo", ["zero_copy", "copy"])
def test_multi_schedule_fp32_aos_tile_bitwise(layout, halo):
    """fp32 through the multi-device schedule (interior / shared-layer
    launches of the AoS plane-tile kernel on their two streams, graph replay)
    against the one-stream SoA engine: bitwise (same collision arithmetic)."""
    dom = (40, 18, 36)
    init = O.port_initial_state("D3Q19", dom)
    ref = _run(17, init, dom, precision="fp32", layout="SoA", partitions=1)
    out = _run(17, init, dom, precision="fp32", layout=layout, partitions=3, halo_mode=halo, devices=[0, 0, 0],
               graph_steps=4)
    assert np.array_equal(out, ref)
