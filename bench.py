#!/usr/bin/env python
"""Benchmark of the dense D3Q19 fp32 LBM step (BASELINE.json metric) on B200.

    python bench.py --gpus N --steps K --warmup W [--impl ours|reference]

Workload (BASELINE configs[1]): D3Q19 BGK lid-driven cavity, dense 512^3,
fp32, DisagSoA layout, z-slab partitions with zero-copy halo; at N>1 the
512^3 domain is split into N slabs, one per rank (strong scaling; --weak puts
512^3 on every rank). A "step" is one collide-and-stream pass over the whole
domain. The state is 2 x 10.2 GB of populations: far larger than L2, so no L2
flush is needed between steps.

One JSON line on rank 0: value = whole-job MLUPS with inputs resident in HBM,
timed with CUDA events on the engine stream (max over ranks); e2e = the same
metric through the reference-facing API with host buffers (canonical fp64 state
uploaded, per-step diagnostics read back, final state downloaded); roofline of
the step kernel; cpu_baseline = the reference library compiled from
/root/reference (oracle/_ref) timed on this host; paths = BASELINE configs[3]
(block-sparse, disaggregated boundary kernel vs monolithic) and configs[4]
(3-level multires obstacle flow, fused vs staged) measured in the same run
(N=1 only; --no-paths skips them).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

Q = 19
BYTES_PER_LUP = 2 * Q * 4  # fp32 D3Q19: each population read once and written once


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=512, help="cubic domain edge (512 = BASELINE configs[1])")
    ap.add_argument("--weak", action="store_true", help="size^3 per GPU (configs[2]) instead of split")
    ap.add_argument("--halo", default="zero_copy", choices=["zero_copy", "copy"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-size", type=int, default=0, help="domain edge of the e2e run (default: --size)")
    ap.add_argument("--e2e-steps", type=int, default=1000,
                    help="steps of the e2e run() (default 1000: BASELINE configs[0]'s run length); a second e2e "
                         "run at --steps is reported beside it")
    ap.add_argument("--no-paths", action="store_true", help="skip the block-sparse / multires lines (configs[3-4])")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms while running."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.rows = []
        self.marks = []
        self._proc = None
        self._t = None
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self):
        self.marks.append(time.time())

    def stop(self):
        if self._proc:
            time.sleep(0.25)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()

    def summary(self, t0, t1):
        rows = [r for t, r in self.rows if t0 - 0.15 <= t <= t1 + 0.15] or [r for _, r in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def traffic_from_profiles():
    """dram bytes per launch of the dense step kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "dense_step_ncu.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("voxels_per_launch")
    return None, None


# ---- CPU reference (oracle/_ref: the reference library built from /root/reference) ----

class RefReplicas:
    """The reference's own dense loop (reference_dense_run, solver.cpp:189-206:
    fused_stream_collide sweeps with A/B swap; oracle/_ref, built from
    /root/reference) on `threads` independent edge^3 cavity replicas, one
    resident state per host thread. Allocation and the initial copy happen
    here, outside every timed sweep. Falls back to the plain-C restatement
    (oracle/voxl_oracle.c, kind "port") only if the reference did not build."""

    def __init__(self, threads: int, edge: int):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        from concurrent.futures import ThreadPoolExecutor

        self.O, self.threads, self.edge = O, threads, edge
        cfg = dict(lattice="D3Q19", domain=[edge] * 3, tau=0.56, scenario="lid_driven_cavity",
                   velocity=[0.05, 0, 0], steps=1)
        self.kind = "reference" if O.ref_available() else "port"
        if self.kind == "reference":
            init = O.ref_initial_state(cfg)
            self.states = [O.RefDense(cfg, init) for _ in range(threads)]
        else:
            init = O.port_initial_state("D3Q19", (edge,) * 3)
            self.states = [init.copy() for _ in range(threads)]
        self.ex = ThreadPoolExecutor(threads)

    def _one(self, i):
        if self.kind == "reference":
            self.states[i].step(1)
        else:
            e = self.edge
            self.states[i] = self.O.port_dense_run("D3Q19", (e, e, e), 0.56, "lid_driven_cavity", (0.05, 0, 0), 1,
                                                   state=self.states[i])

    def sweep(self) -> float:
        """One sweep of every replica, concurrently; wall seconds."""
        t0 = time.perf_counter()
        list(self.ex.map(self._one, range(self.threads)))
        return time.perf_counter() - t0

    def mlups(self, seconds: float, sweeps: int = 1) -> float:
        return self.threads * self.edge ** 3 * sweeps / seconds / 1e6

    def close(self):
        self.ex.shutdown()
        if self.kind == "reference":
            for st in self.states:
                st.close()


def cpu_reference_sample(threads: int, budget_s: float, edge: int = 128):
    """(MLUPS, sweeps, seconds, kind) of the reference loop on `threads`
    replicas, sweeps sized to ~budget_s after one untimed warm-up sweep."""
    rep = RefReplicas(threads, edge)
    t_one = rep.sweep()
    sweeps = max(1, min(30, int(budget_s / max(t_one, 1e-3))))
    dt = sum(rep.sweep() for _ in range(sweeps))
    out = rep.mlups(dt, sweeps), sweeps, dt, rep.kind
    rep.close()
    return out


def run_reference_arm(args, rank):
    """bench.py --impl reference: the reference's CPU implementation of the
    path on all host cores (one single-threaded reference_dense_run loop per
    core -- the reference has no parallel solver), K timed steps after W
    warm-up steps, one step = one sweep of every replica."""
    if rank != 0:
        return
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64 << 30
    cores = os.cpu_count() or 1
    edge = 128
    per = 2 * edge ** 3 * Q * 8
    threads = max(1, min(cores, int(0.5 * avail // per)))
    # size each step so that K + W steps finish in ~2-3 minutes
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    rep = RefReplicas(threads, edge)
    one_step = rep.sweep()
    if one_step > per_step_budget:
        rep.close()
        edge = max(16, int(edge * (per_step_budget / one_step) ** (1 / 3)))
        rep = RefReplicas(threads, edge)
    t_steps = []
    for s in range(args.warmup + args.steps):
        dt = rep.sweep()
        if s >= args.warmup:
            t_steps.append(dt)
    kind = rep.kind
    rep.close()
    t_med = statistics.median(t_steps)
    value = threads * edge ** 3 / t_med / 1e6
    line = {
        "metric": "MLUPS (D3Q19 fp32) at 1/2/4/8 B200 and % of HBM roofline vs CPU ref",
        "impl": "reference", "value": round(value, 3), "unit": "MLUPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t_med, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (rest-equilibrium lid-driven cavity)",
        "config": {"workload": f"D3Q19 BGK lid-driven cavity, reference CPU reference_dense_run loop "
                               f"(fused_stream_collide), {threads} independent {edge}^3 replicas (one per host thread)",
                   "lattice": "D3Q19", "tau": 0.56, "lid_u": [0.05, 0, 0]},
        "cpu_baseline": {"value": round(value, 3), "unit": "MLUPS", "cores": threads, "kind": kind,
                         "sample": f"{threads} x {edge}^3 cavity replicas, resident states, one fused_stream_collide "
                                   f"sweep each per step (the reference is single-threaded; replicas fill the host "
                                   f"cores)"},
        "e2e": {"value": round(value, 3), "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm ------------------------------------------------------------------------------

def launch_command(argv, gpus: int, port: int):
    """The torchrun command bench.py re-executes itself under when asked for
    N > 1 GPUs without a launcher: one rank per GPU on this node."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)


def free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    args = parse()
    launched = "WORLD_SIZE" in os.environ
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    if args.gpus > 1 and not launched:
        # `python bench.py --gpus N` alone: put N GPUs to work by re-launching
        # under torchrun (one rank per GPU), which prints the one JSON line
        if os.environ.get("VOXL_SHARE_DEVICE") != "1":
            import torch

            have = torch.cuda.device_count()
            if have < args.gpus:
                print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}), flush=True)
                sys.exit(1)
        sys.exit(subprocess.call(launch_command(sys.argv[1:], args.gpus, free_port())))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    import numpy as np
    import torch

    # VOXL_SHARE_DEVICE=1: every rank on cuda:0 over gloo -- exercises the
    # multi-process IPC / device-flag path on a single-GPU box (timings are
    # then time-sliced and not meaningful).
    share = os.environ.get("VOXL_SHARE_DEVICE") == "1"
    dev = 0 if share else local_rank
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    import paper_2503_07898_b200 as V

    n = args.size
    domain = (n, n, n * world) if args.weak else (n, n, n)
    if world > 1:
        from paper_2503_07898_b200 import multigpu

        eng = multigpu.DistributedDense(domain=domain, precision="fp32", halo_mode=args.halo)
    else:
        eng = V.DenseEngine(domain=domain, precision="fp32", layout="DisagSoA", partitions=1,
                            halo_mode=args.halo)
    eng.set_equilibrium(1.0, (0.0, 0.0, 0.0))
    voxels_total = domain[0] * domain[1] * domain[2]
    voxels_local = eng.owned_voxels() if world > 1 else voxels_total

    sampler = ClockSampler(dev) if rank == 0 else None
    eng.timed_steps(args.warmup)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    total_ms, kernel_ms = eng.timed_steps(args.steps)
    torch.cuda.synchronize()
    t1 = time.time()
    if dist:
        t = torch.tensor([total_ms], device="cpu" if share else "cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    clocks = None
    if sampler:
        sampler.stop()
        clocks = sampler.summary(t0, t1)
    diag = eng.probe()

    value = voxels_total * args.steps / (total_ms / 1e3) / 1e6
    peak, peak_kind = measured_peaks()
    avg_kernel_ms = kernel_ms / args.steps
    achieved = BYTES_PER_LUP * voxels_local / (avg_kernel_ms / 1e3) / 1e9
    dram, vox_prof = traffic_from_profiles()
    traffic = None
    if dram and vox_prof:
        traffic = round(dram / vox_prof * voxels_local)

    e2e = None
    if not args.no_e2e and world == 1 and rank == 0:
        e2e = e2e_run(args, V, np)
    elif not args.no_e2e and world > 1:
        e2e = e2e_run_dist(args, eng, dist, voxels_total, share, np)
    paths = None
    if not args.no_paths and world == 1 and rank == 0:
        eng.close()  # the 20 GB dense state makes room for the other engines
        eng = None
        paths = secondary_paths(args, V, peak)
    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        try:
            mlups, steps, dt, kind = cpu_reference_sample(1, 12.0, 128)
            cpu = {"value": round(mlups, 3), "unit": "MLUPS", "cores": 1, "kind": kind,
                   "sample": f"D3Q19 cavity 128^3 (configs[0] size), {steps} sweeps of the reference_dense_run "
                             f"loop (fused_stream_collide, fp64, single thread, resident state) in {dt:.1f} s"}
        except Exception as exc:  # the checker is optional on the box; report why
            cpu = {"value": None, "unit": "MLUPS", "cores": 1, "kind": "reference", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": "MLUPS (D3Q19 fp32) at 1/2/4/8 B200 and % of HBM roofline vs CPU ref",
            "value": round(value, 1), "unit": "MLUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (rest-equilibrium lid-driven cavity, device-initialised)",
            "config": {"workload": f"D3Q19 BGK lid-driven cavity dense {domain[0]}x{domain[1]}x{domain[2]} fp32, "
                                   f"DisagSoA, {world} z-slab partition(s), {args.halo} halo",
                       "domain": list(domain), "tau": 0.56, "lid_u": [0.05, 0, 0], "layout": "DisagSoA",
                       "partitions": world, "halo": args.halo,
                       "l2": "state 2x10.2 GB >> 126 MB L2; no flush needed"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "peak_kind": peak_kind,
                         "bytes_per_lup": BYTES_PER_LUP, "voxels_per_launch": voxels_local,
                         "avg_kernel_ms": round(avg_kernel_ms, 4),
                         "frac_of_8tbs": round(achieved / 8000.0, 4),
                         "peak_note": "MEASURED_PEAKS hbm_gbs is a torch copy; the float4 copy ceiling of "
                                      "tools/micro/membw.cu is ~6.8 TB/s on this pool, so frac can exceed 1"},
            "clocks": clocks,
            "gpu_launches": args.steps * (1 if world == 1 else 4),
            "diag": {"mass": diag.mass, "max_speed": diag.max_speed, "unstable": diag.unstable},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "paths": paths,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def secondary_paths(args, V, peak):
    """BASELINE configs[3] and configs[4] on the same GPU, same timing rules
    (CUDA events on the engine stream, warm-up first, states >> L2):
    block-sparse 512^3 sphere wind tunnel, regularized x-faces, 8^3 blocks,
    disaggregated boundary kernel (disag_mem) vs monolithic (naive); 3-level
    multires obstacle flow, fused vs staged. MLUPS count active voxels /
    LUP = sum_l N_l 2^(L-1-l) per coarse step; 152 B per update."""
    from paper_2503_07898_b200.multires import obstacle_band_level_map

    n = args.size
    dom = (n, n, n)
    out = {}
    try:
        act = V.obstacle_mask(dom)
        for strategy in ("disag_mem", "naive"):
            e = V.SparseEngine(dom, act, block_edge=8, strategy=strategy, precision="fp32")
            na = e.info()["num_active"]
            e.timed_steps(5)
            ms, _, _ = e.timed_steps(20)
            e.close()
            gbs = BYTES_PER_LUP * na * 20 / (ms / 1e3) / 1e9
            out[f"sparse_{strategy}"] = {"MLUPS": round(na * 20 / (ms / 1e3) / 1e6, 1),
                                         "frac": round(gbs / peak, 4), "ms_per_step": round(ms / 20, 4),
                                         "active_voxels": na}
        lm = obstacle_band_level_map(dom, 3)
        for fused in (True, False):
            e = V.MultiResEngine(dom, levels=3, level_map=lm, fused=fused, precision="fp32", solid_cells=True)
            lup = e.lup_per_coarse_step()
            e.timed_steps(2)
            ms, _ = e.timed_steps(5)
            e.close()
            gbs = BYTES_PER_LUP * lup * 5 / (ms / 1e3) / 1e9
            out["multires_obstacle_" + ("fused" if fused else "staged")] = {
                "MLUPS": round(lup * 5 / (ms / 1e3) / 1e6, 1), "frac": round(gbs / peak, 4),
                "ms_per_coarse_step": round(ms / 5, 4), "lup_per_coarse_step": lup}
        out["config"] = (f"configs[3]: D3Q19 block-sparse {n}^3 sphere r={n / 5:g} wind tunnel, 8^3 blocks, fp32, "
                         f"20 steps; configs[4]: D3Q19 3-level multires {n}^3 band + solid sphere, fp32, 5 coarse "
                         f"steps; frac = achieved (152 B/update) / MEASURED_PEAKS hbm_gbs")
    except Exception as exc:  # reported, never fatal for the headline line
        out["error"] = f"{type(exc).__name__}: {exc}"
    return out


def e2e_run(args, V, np):
    """The same metric through the reference-facing API with host buffers, in
    run()'s shape (solver.cpp:225-266): fill_canonical from a pinned fp64
    canonical host array, K steps each followed by probe_field (fused into the
    step kernel, rows read back once per 256 steps), and to_canonical of the
    final field. K = --e2e-steps (default 1000, the run length of BASELINE
    configs[0]); the same run at --steps is reported as `short_run`."""
    import torch

    n = args.e2e_size or args.size
    dom = (n, n, n)
    vox = n ** 3
    eng = V.DenseEngine(domain=dom, precision="fp32", layout="DisagSoA", partitions=1)
    host_in = torch.empty(vox * Q, dtype=torch.float64, pin_memory=True).numpy()
    host_out = torch.empty(vox * Q, dtype=torch.float64, pin_memory=True).numpy()
    # rest-equilibrium canonical input (initial_canonical_state, solver.cpp:165-187)
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    host_in.reshape(vox, Q)[:] = w

    def one(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.set_canonical(host_in)
        t1 = time.perf_counter()
        rows = eng.step_probe_n(steps)  # run()'s loop: step + fused probe_field
        t2 = time.perf_counter()
        eng.get_canonical(host_out)
        t3 = time.perf_counter()
        # the fp32 engine moves its storage format over PCIe (canon_io.cuh):
        # the host converts fp64 <-> fp32 wire buffers, which are what is copied
        wire_in = vox * Q * 4
        wire_out = vox * Q * 4 + ((steps + 255) // 256) * 256 * 32
        return {"value": round(vox * steps / (t3 - t0) / 1e6, 1), "unit": "MLUPS", "steps": steps,
                "h2d_bytes_per_step": int(wire_in / steps), "d2h_bytes_per_step": int(wire_out / steps),
                "seconds": round(t3 - t0, 3), "set_s": round(t1 - t0, 3), "steps_s": round(t2 - t1, 3),
                "get_s": round(t3 - t2, 3), "final_mass": rows[-1].mass if rows else None}

    main = one(args.e2e_steps)
    short = one(args.steps) if args.steps != args.e2e_steps else None
    eng.close()
    main.update({"canonical_fp64_bytes": vox * Q * 8, "domain": list(dom),
                 "path": "DenseEngine.set_canonical(host fp64 -> fp32 wire) + step_probe_n(steps) (fused probe, rows "
                         "D2H per 256-step batch) + get_canonical(fp32 wire -> host fp64)"})
    if short:
        main["short_run"] = {k: short[k] for k in ("steps", "value", "seconds", "set_s", "steps_s", "get_s")}
    return main


def e2e_run_dist(args, eng, dist, voxels_total, share, np):
    """e2e at N ranks through the same API: every rank uploads its slab of the
    fp64 canonical field from pinned host memory (fill_canonical of its
    partition), refreshes the halos, runs K steps each with its slab's
    probe_field row read back (rows combine as sum / max; no per-step
    collective), and downloads its slab. Wall time max over ranks."""
    import torch

    k0, k1 = eng.slab()
    dom = eng.desc["domain"]
    elems = (k1 - k0) * dom[0] * dom[1] * Q
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 1 << 40
    # two pinned slabs per rank; every rank of the node allocates at once
    if 2 * elems * 8 * eng.world > 0.6 * avail:
        return {"value": None, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "skipped": f"host memory: {2 * elems * 8 * eng.world / 2**30:.0f} GiB of pinned slabs needed, "
                           f"{avail / 2**30:.0f} GiB available"}
    host_in = torch.empty(elems, dtype=torch.float64, pin_memory=True).numpy()
    host_out = torch.empty(elems, dtype=torch.float64, pin_memory=True).numpy()
    w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
    host_in.reshape(-1, Q)[:] = w
    steps = args.steps
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.set_canonical_planes(host_in, k0, k1)
    eng.refresh_halos()
    rows = eng.step_probe_n(steps)  # this rank's run() loop: step + fused probe, rows per 256-step batch
    last = rows[-1]
    eng.get_canonical_planes(k0, k1, out=host_out)
    dt = time.perf_counter() - t0
    t = torch.tensor([dt, last.max_speed], dtype=torch.float64, device="cpu" if share else "cuda")
    m = torch.tensor([last.mass], dtype=torch.float64, device=t.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(m)
    dt = float(t[0].item())
    bytes_in = voxels_total * Q * 4  # fp32 wire buffers (the host converts fp64 canonical <-> fp32)
    bytes_out = voxels_total * Q * 4 + steps * 32 * eng.world
    return {"value": round(voxels_total * steps / dt / 1e6, 1), "unit": "MLUPS",
            "h2d_bytes_per_step": int(bytes_in / steps), "d2h_bytes_per_step": int(bytes_out / steps),
            "domain": list(dom), "seconds": round(dt, 3), "final_mass": float(m.item()),
            "final_max_speed": float(t[1].item()),
            "path": "per rank: DistributedDense.set_canonical_planes(host fp64 slab -> fp32 wire) + refresh_halos + "
                    "step_probe_n(steps) (rank rows D2H per 256-step batch) + get_canonical_planes; wall time max "
                    "over ranks"}


if __name__ == "__main__":
    main()
