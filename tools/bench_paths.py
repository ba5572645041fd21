#!/usr/bin/env python
"""Throughput of the secondary hot paths (BASELINE configs[3], configs[4]).

    python tools/bench_paths.py sparse [--n 256] [--steps 50]
    python tools/bench_paths.py multires [--n 512] [--steps 5]
    python tools/bench_paths.py dense [--n 512] [--steps 50]

Prints one JSON line per variant: MLUPS (active voxels for sparse; LUP =
sum_l N_l * 2^(L-1-l) per coarse step for multires) and the fraction of the
HBM roofline at 2 Q 4 B/LUP (fp32: 152 B D3Q19, 216 B D3Q27), per kernel where the engine exposes
per-kernel event times.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def bytes_per_lup(lattice):
    return 2 * (19 if lattice == "D3Q19" else 27) * 4


def peak():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        return float(json.load(f)["hbm_gbs"])


def sparse(args):
    import paper_2503_07898_b200 as V

    n = args.n
    dom = (n, n, n)
    act = V.obstacle_mask(dom)
    for strategy in ("naive", "disag_bitmask", "disag_mem"):
        e = V.SparseEngine(dom, act, block_edge=8, strategy=strategy, precision="fp32", lattice=args.lattice)
        info = e.info()
        e.timed_steps(args.warmup)
        total, b_ms, l_ms = e.timed_steps(args.steps)
        na = info["num_active"]
        mlups = na * args.steps / (total / 1e3) / 1e6
        gbs = bytes_per_lup(args.lattice) * na * args.steps / (total / 1e3) / 1e9
        line = {"path": "block_sparse", "lattice": args.lattice, "strategy": strategy, "domain": list(dom), "block_edge": 8,
                "active_voxels": na, "blocks": info["num_blocks"], "n_boundary": info["n_boundary"],
                "steps": args.steps, "ms_per_step": round(total / args.steps, 4), "MLUPS": round(mlups, 1),
                "achieved_GBs": round(gbs, 1), "frac_of_measured_peak": round(gbs / peak(), 4),
                "frac_of_8TBs": round(gbs / 8000, 4),
                "boundary_kernel_ms": round(b_ms / args.steps, 4), "light_kernel_ms": round(l_ms / args.steps, 4),
                "report": json.loads(e.report_json())}
        line["lib"] = os.environ.get("VOXL_TAG", "")
        print(json.dumps(line), flush=True)
        e.close()


def multires(args):
    import paper_2503_07898_b200 as V

    from paper_2503_07898_b200.multires import obstacle_band_level_map

    n = args.n
    for scenario, fused in [(s, f) for s in ("cavity", "obstacle") for f in (False, True)]:
        if scenario == "obstacle":
            # configs[4]: flow past an obstacle (solid sphere in the finest band;
            # extension, parity vs the oracle's restatement only)
            lm = obstacle_band_level_map((n, n, n), 3)
            e = V.MultiResEngine((n, n, n), levels=3, level_map=lm, fused=fused, precision="fp32", solid_cells=True,
                                 lattice=args.lattice)
        else:
            e = V.MultiResEngine((n, n, n), levels=3, fused=fused, precision="fp32", lattice=args.lattice)
        lup = e.lup_per_coarse_step()
        e.timed_steps(args.warmup)
        total, detail = e.timed_steps(args.steps)
        mlups = lup * args.steps / (total / 1e3) / 1e6
        gbs = bytes_per_lup(args.lattice) * lup * args.steps / (total / 1e3) / 1e9
        line = {"path": "multires", "lattice": args.lattice, "scenario": scenario, "levels": 3, "fused": fused, "domain": [n] * 3, "lup_per_coarse_step": lup,
                "steps": args.steps, "ms_per_coarse_step": round(total / args.steps, 4), "MLUPS": round(mlups, 1),
                "achieved_GBs": round(gbs, 1), "frac_of_measured_peak": round(gbs / peak(), 4),
                "frac_of_8TBs": round(gbs / 8000, 4), "kernels_ms": detail, "distribution": e.distribution()}
        line["lib"] = os.environ.get("VOXL_TAG", "")
        print(json.dumps(line), flush=True)
        e.close()


def dense(args):
    """The dense step across lattice, precision, layout and partition count
    (the paper's layout study: AoS vs SoA vs DisagSoA; D3Q27 and fp64 at the
    same size). Bytes/LUP = 2 * Q * sizeof(real)."""
    import paper_2503_07898_b200 as V

    n = args.n
    cases = [("D3Q19", "fp32", "DisagSoA", 1), ("D3Q19", "fp32", "SoA", 1), ("D3Q19", "fp32", "AoS", 1),
             ("D3Q19", "fp32", "DisagSoA", 8), ("D3Q19", "fp32", "AoS", 8), ("D3Q27", "fp32", "DisagSoA", 1),
             ("D3Q27", "fp32", "AoS", 1), ("D3Q19", "fp64", "DisagSoA", 1)]
    if args.layouts:
        cases = [c for c in cases if c[2] in args.layouts.split(",")]
    for lat, prec, layout, parts in cases:
        q = 19 if lat == "D3Q19" else 27
        bpl = 2 * q * (4 if prec == "fp32" else 8)
        e = V.DenseEngine(lattice=lat, domain=(n, n, n), precision=prec, layout=layout, partitions=parts)
        e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
        e.timed_steps(args.warmup)
        total, kern = e.timed_steps(args.steps)
        vox = n ** 3
        mlups = vox * args.steps / (total / 1e3) / 1e6
        gbs = bpl * vox * args.steps / (total / 1e3) / 1e9
        line = {"path": "dense", "lattice": lat, "precision": prec, "layout": layout, "partitions": parts,
                "domain": [n] * 3, "bytes_per_lup": bpl, "steps": args.steps,
                "ms_per_step": round(total / args.steps, 4), "MLUPS": round(mlups, 1), "achieved_GBs": round(gbs, 1),
                "frac_of_measured_peak": round(gbs / peak(), 4), "frac_of_8TBs": round(gbs / 8000, 4)}
        line["lib"] = os.environ.get("VOXL_TAG", "")
        print(json.dumps(line), flush=True)
        e.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("path", choices=["sparse", "multires", "dense"])
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--lattice", default="D3Q19", choices=["D3Q19", "D3Q27"], help="sparse / multires lattice")
    ap.add_argument("--layouts", default="", help="dense: only these layouts (comma-separated)")
    a = ap.parse_args()
    {"sparse": sparse, "multires": multires, "dense": dense}[a.path](a)
