"""Multi-process (one rank per GPU) dense path.

CPU: world_size-2/4 gloo tests of the host logic -- the per-rank exchange plan
derived from the reference-order ledger, and the span send/recv itself on
DisagSoA/SoA/AoS buffers (the NCCL comparison path's exchange, run over gloo).
GPU: two ranks sharing one device exercise the real zero-copy path (CUDA IPC
buffers, device step flags) and must stay bitwise equal to the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle as O
import paper_2503_07898_b200 as V
from paper_2503_07898_b200.multigpu import exchange_plan


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("layout", ["AoS", "SoA", "DisagSoA"])
def test_exchange_plan_pairs_up(world, layout):
    desc = dict(lattice="D3Q19", domain=(8, 8, 4 * world), layout=layout)
    plans = [exchange_plan(r, world, **desc) for r in range(world)]
    for r, (sends, _) in enumerate(plans):
        for peer, _, n in sends:
            recvs_of_peer = [x for x in plans[peer][1] if x[0] == r]
            assert n in [x[2] for x in recvs_of_peer]
        expect = {"DisagSoA": 1, "SoA": 5, "AoS": 1}[layout]
        for nb in (r - 1, r + 1):
            if 0 <= nb < world:
                assert len([s for s in sends if s[0] == nb]) == expect


def _halo_worker(rank, world, port, layout, result_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_07898_b200.multigpu import exchange_halos

    dom = (6, 5, 4 * world)
    q = 19
    canon = np.arange(dom[0] * dom[1] * dom[2] * q, dtype=np.float64) + 0.5
    slabs = V.decompose(dom, world, 2)
    k0, k1 = slabs[rank]
    shape = (dom[0], dom[1], k1 - k0)
    addr = V.layout_addresses(layout, shape, "D3Q19", 2).reshape(shape[2] + 2, dom[1], dom[0], q)
    buf = np.zeros(addr.size, np.float64)
    g = canon.reshape(dom[2], dom[1], dom[0], q)
    buf[addr[1:-1].ravel()] = g[k0:k1].ravel()
    t = torch.from_numpy(buf)
    sends, recvs = exchange_plan(rank, world, lattice="D3Q19", domain=dom, layout=layout)
    exchange_halos(dist, t, sends, recvs)
    ok = True
    lat = np.array([[0, 0, 0], [-1, 0, 0], [0, -1, 0], [0, 0, -1], [0, 0, 1], [0, 1, 0], [1, 0, 0]])
    up = [4, 9, 12, 14, 17]  # e_z > 0 (halo UH holds these), down = e_z < 0 (halo LH)
    down = [3, 8, 11, 13, 16]
    if rank > 0:  # upper halo = upper neighbour's last slab, up-crossing set (all comps for AoS)
        comps = range(q) if layout == "AoS" else up
        for c in comps:
            ok &= np.array_equal(buf[addr[0, :, :, c].ravel()], g[k0 - 1, :, :, c].ravel())
    if rank < world - 1:
        comps = range(q) if layout == "AoS" else down
        for c in comps:
            ok &= np.array_equal(buf[addr[-1, :, :, c].ravel()], g[k1, :, :, c].ravel())
    _ = lat
    result_q.put((rank, bool(ok)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("layout", ["SoA", "DisagSoA", "AoS"])
def test_gloo_span_exchange_fills_halos(world, layout):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, layout, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()), res


def _gpu_worker(rank, world, port, result_q, halo="zero_copy"):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_07898_b200.multigpu import DistributedDense

    dom = (24, 20, 32)
    eng = DistributedDense(domain=dom, precision="fp64", halo_mode=halo)
    init = O.port_initial_state("D3Q19", dom)
    k0, k1 = eng.slab()
    s = dom[0] * dom[1] * 19
    eng.set_canonical_planes(init[k0 * s:k1 * s], k0, k1)
    eng.refresh_halos()
    eng.step(20)
    for _ in range(10):
        eng.step_probe()  # run()'s per-step probe path, fused into the step
    out = eng.get_canonical_planes(k0, k1)
    d = eng.probe()
    result_q.put((rank, k0, k1, out, d.mass))
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,halo", [(2, "zero_copy"), (3, "zero_copy"), (2, "copy"), (3, "copy")])
def test_multiprocess_halo_modes_bitwise(world, halo):
    """Ranks share cuda:0 here (the box has one GPU per call). zero_copy: the
    IPC buffers, peer stores and device step flags are the same code path as on
    8 GPUs. copy: the OCC schedule with the span exchange on the shared-layer
    stream (NCCL on separate GPUs; gloo through host memory here)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, halo)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    dom = (24, 20, 32)
    ref = O.port_dense_run("D3Q19", dom, 0.56, "lid_driven_cavity", (0.05, 0, 0), 30)
    s = dom[0] * dom[1] * 19
    for rank, k0, k1, out, mass in res:
        assert np.array_equal(out, ref[k0 * s:k1 * s]), f"rank {rank} differs"
    m_ref, _ = O.port_probe("D3Q19", ref)
    assert abs(res[0][4] - m_ref) <= 1e-12 * m_ref


@pytest.mark.gpu
def test_bench_multirank_path_on_one_gpu():
    """bench.py under torchrun with 2 ranks sharing cuda:0 (VOXL_SHARE_DEVICE=1):
    the N>1 code path end to end (IPC buffers, device flags, max-over-ranks)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VOXL_SHARE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--steps", "10", "--warmup",
           "3", "--size", "64", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=root, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == "strong"
    assert abs(line["diag"]["mass"] - 64 ** 3) < 1e-6 * 64 ** 3 and line["diag"]["unstable"] == 0
    e2e = line["e2e"]
    # the copied tensors are the fp32 wire buffers (the host converts fp64 canonical <-> fp32)
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] == 64 ** 3 * 19 * 4 // 10
    assert abs(e2e["final_mass"] - 64 ** 3) < 1e-6 * 64 ** 3


def test_bench_self_launch_command():
    """`python bench.py --gpus N` without a launcher re-executes itself under
    torchrun with one rank per GPU on 127.0.0.1 (CPU check of the command)."""
    import importlib.util

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    cmd = bench.launch_command(["--gpus", "8", "--steps", "20", "--warmup", "5"], 8, 29577)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29577" in cmd
    assert cmd[-7].endswith("bench.py") and cmd[-6:] == ["--gpus", "8", "--steps", "20", "--warmup", "5"]


@pytest.mark.gpu
def test_bench_gpus_2_without_torchrun():
    """`python bench.py --gpus 2` with no torchrun wrapper runs 2 ranks and
    reports n_gpus = 2 (ranks share cuda:0 on the one-GPU box)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VOXL_SHARE_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "6", "--warmup", "3", "--size", "64", "--no-cpu",
           "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=root, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["partitions"] == 2


def _stall_worker(rank, world, port, result_q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["VOXL_HALO_TIMEOUT_S"] = "2"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_07898_b200.multigpu import DistributedDense

    eng = DistributedDense(domain=(16, 16, 16), precision="fp32", halo_mode="zero_copy")
    eng.set_equilibrium(1.0, (0.0, 0.0, 0.0))
    msg = None
    if rank == 0:  # rank 1 never steps: rank 0's second step waits for a signal that never comes
        try:
            eng.step(3)
        except Exception as exc:  # noqa: BLE001
            msg = str(exc)
    result_q.put((rank, msg))
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_zero_copy_stalled_neighbour_errors_instead_of_hanging():
    """A neighbour that stops signalling (crashed rank) surfaces as an error
    after VOXL_HALO_TIMEOUT_S instead of a spin that wedges the GPU."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stall_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[1] is None
    assert res[0] is not None and "halo exchange stalled at step 1" in res[0], res[0]
