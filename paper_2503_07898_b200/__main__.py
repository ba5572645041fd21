"""`python -m paper_2503_07898_b200 <run|verify|ledger|model|report>` -- the
reference CLI's subcommands (proj/tools/main.cpp:30-229) on the B200 engines.

Exit codes as the reference (main.cpp:261-269): 0 ok, 1 failure, 2 config error.
"""
from __future__ import annotations

import argparse
import sys

import numpy as np


def cmd_run(config_path: str, out_dir: str, observed_trace: bool = False) -> int:
    from .solver import config_from_json, run, write_outputs

    with open(config_path, "rb") as f:
        cfg = config_from_json(f.read().decode())
    res = run(cfg, observed_trace)
    write_outputs(res, out_dir)
    step, mass, umax = res.diagnostics[-1] if res.diagnostics else (0, 0.0, 0.0)
    print(f"run complete: {cfg.steps} steps, final mass {mass:.6g}, max |u| {umax:.6g}")
    print(f"outputs written to {out_dir}")
    return 0


def _report(a, b, what) -> int:
    if a.size != b.size:
        print(f"FAIL {what}: size mismatch {a.size} vs {b.size}")
        return 1
    diff = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
    if diff.size:
        i = int(diff[0])
        print(f"FAIL {what}: first divergence at flat index {i} ({a[i]} vs {b[i]})")
        return 1
    print(f"PASS {what}")
    return 0


def cmd_verify() -> int:
    """cmd_verify (main.cpp:75-137) in fp64 parity mode on the device."""
    from .solver import SolverConfig, run

    fails = 0
    base = SolverConfig(lattice="D3Q19", domain=(16, 16, 16), scenario="lid_driven_cavity", tau=0.56,
                        velocity=(0.05, 0.0, 0.0), steps=20, precision="fp64")
    ref = run(base).field
    for layout in ("AoS", "SoA", "DisagSoA"):
        for parts in (1, 2, 4):
            c = SolverConfig(**{**base.__dict__, "layout": layout, "partitions": parts})
            fails += _report(ref, run(c).field, f"partition_invariance {layout} x{parts}")
    sp = SolverConfig(lattice="D3Q19", domain=(16, 16, 16), scenario="flow_over_obstacle", tau=0.7,
                      velocity=(0.04, 0.0, 0.0), steps=10, strategy="naive", precision="fp64")
    naive = run(sp).field
    for s in ("disag_bitmask", "disag_mem"):
        fails += _report(naive, run(SolverConfig(**{**sp.__dict__, "strategy": s})).field,
                         f"sparse_equivalence {s}")
    mr = SolverConfig(lattice="D3Q19", domain=(16, 16, 16), scenario="lid_driven_cavity", tau=0.56,
                      velocity=(0.05, 0.0, 0.0), steps=5, levels=2, fused=False, precision="fp64")
    staged = run(mr).field
    fused = run(SolverConfig(**{**mr.__dict__, "fused": True})).field
    fails += _report(staged, fused, "fusion_soundness 2-level")
    if fails == 0:
        print("all verification suites passed")
    return 0 if fails == 0 else 1


def cmd_ledger(config_path: str) -> int:
    """cmd_ledger (main.cpp:139-176): per-step (alpha, beta) of each partition vs layout_params."""
    from .dense import plan_ledger
    from .solver import ConfigError, config_from_json

    with open(config_path, "rb") as f:
        c = config_from_json(f.read().decode())
    if c.levels > 1 or c.scenario == "flow_over_obstacle":
        raise ConfigError("ledger requires a dense partitioned run")
    steps = min(c.steps, 10)
    s = int(np.prod(c.domain)) // c.domain[c.partition_axis()]
    q = {"D2Q9": 9, "D3Q19": 19, "D3Q27": 27}[c.lattice]
    cross = {"D2Q9": 3, "D3Q19": 5, "D3Q27": 9}[c.lattice]
    model = {"AoS": (2, 2 * q * s), "SoA": (2 * cross, 2 * cross * s), "DisagSoA": (2, 2 * cross * s)}[c.layout]
    periodic = c.scenario == "periodic_box"
    print("step,partition,alpha,beta,model_alpha,model_beta,match")
    ok = True
    for step in range(steps):
        recs = plan_ledger(step, lattice=c.lattice, domain=c.domain, layout=c.layout, partitions=c.partitions,
                           scenario=c.scenario)
        for p in range(c.partitions):
            sent = [r for r in recs if r.src == p]
            a, b = len(sent), sum(r.elements for r in sent)
            if not (periodic or 0 < p < c.partitions - 1):
                print(f"{step},{p},{a},{b},,,(end partition)")
                continue
            m = (a, b) == model
            ok &= m
            print(f"{step},{p},{a},{b},{model[0]},{model[1]},{'yes' if m else 'NO'}")
    if not ok:
        print("ledger does not match the model")
        return 1
    return 0


def cmd_model() -> int:
    """cmd_model (main.cpp:178-184): Tables 1 and 3 (commodel.cpp:50-75)."""
    print("# five-point stencil on a 2-component vector field (beta per boundary row)")
    print("layout,alpha,beta,coalesced")
    for name, (a, b, co) in (("AoS", (2, 2, "no")), ("SoA", (4, 2, "yes")), ("DisagSoA", (2, 2, "yes"))):
        print(f"{name},{a},{b}*dx,{co}")
    print("# LBM halo update, s = boundary cross-section voxels")
    print("lattice,layout,alpha,beta,coalesced")
    for lat, q, c in (("D2Q9", 9, 3), ("D3Q19", 19, 5), ("D3Q27", 27, 9)):
        print(f"{lat},AoS,2,{2 * q}s,no")
        print(f"{lat},SoA,{2 * c},{2 * c}s,yes")
        print(f"{lat},DisagSoA,2,{2 * c}s,yes")
    return 0


def cmd_report(out_dir: str) -> int:
    """cmd_report (main.cpp:186-229): one-screen summary of a `run` output directory."""
    import os

    from .solver import config_from_json

    if not os.path.exists(out_dir):
        print(f"report: directory not found: {out_dir}", file=sys.stderr)
        return 2

    def text(name):
        with open(os.path.join(out_dir, name), "rb") as f:
            return f.read().decode()

    def has(name):
        return os.path.exists(os.path.join(out_dir, name))

    print(f"report for {out_dir}")
    if has("config.json"):
        c = config_from_json(text("config.json"))
        nx, ny, nz = c.domain
        print(f"  scenario: {c.scenario}, lattice {c.lattice}, domain {nx}x{ny}x{nz}, steps {c.steps}")
    if has("diagnostics.csv"):
        rows = [ln for ln in text("diagnostics.csv").split("\n")[1:] if ln]
        print(f"  final diagnostics (step,mass,max_u): {rows[-1] if rows else ''}")
    if has("ledger.csv"):
        rows = [ln for ln in text("ledger.csv").split("\n")[1:] if ln]
        elements = sum(int(ln.rsplit(",", 1)[1]) for ln in rows)
        print(f"  ledger: {len(rows)} transfer records, {elements} elements total")
    if has("dispatch.json"):
        sys.stdout.write("  dispatch: " + text("dispatch.json"))
    if has("distribution.txt"):
        sys.stdout.write("  level distribution (% of finest cells): " + text("distribution.txt"))
    sys.stdout.flush()
    return 0


def main(argv=None) -> int:
    from .solver import ConfigError

    ap = argparse.ArgumentParser(prog="voxl-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("--config", required=True)
    r.add_argument("--out", default="out")
    r.add_argument("--observed-trace", action="store_true",
                   help="also write trace_observed.json: the executed step schedule (dense runs)")
    sub.add_parser("verify")
    lg = sub.add_parser("ledger")
    lg.add_argument("--config", required=True)
    sub.add_parser("model")
    rp = sub.add_parser("report")
    rp.add_argument("--dir", required=True)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "run":
            return cmd_run(a.config, a.out, a.observed_trace)
        if a.cmd == "verify":
            return cmd_verify()
        if a.cmd == "ledger":
            return cmd_ledger(a.config)
        if a.cmd == "report":
            return cmd_report(a.dir)
        return cmd_model()
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except (RuntimeError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
