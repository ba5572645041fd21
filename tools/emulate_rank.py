#!/usr/bin/env python
"""One rank of the N-GPU strong-scaling run, emulated on one GPU.

Builds partition r of decompose(512^3, N) exactly as a torchrun rank would
(DenseEngine with first_partition=r, local_partitions=1, distributed OCC
schedule: interior stream + high-priority shared-layer stream, wait/signal
kernels, peer halo stores), but the two neighbours' buffers and flag words are
allocated locally and the flags are pre-released, so the rank never blocks.
The measured step time is therefore the per-rank cost of the schedule without
the NVLink transfer (10 MiB / step / rank, ~13 us at 770 GB/s, overlapped with
the interior kernel). Efficiency bound = t_1gpu / (N * t_rank).

    python tools/emulate_rank.py --gpus 8 --steps 100
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--weak", action="store_true", help="configs[2]: size^3 per rank (domain size x size x size*N)")
    a = ap.parse_args()
    import torch

    import paper_2503_07898_b200 as V
    from paper_2503_07898_b200._capi import check, lib

    n = a.size
    dom = (n, n, n)
    out = {"size": n, "scaling": "weak" if a.weak else "strong"}
    # single-GPU reference step
    e1 = V.DenseEngine(domain=dom, precision="fp32")
    e1.set_equilibrium()
    e1.timed_steps(a.warmup)
    t1, _ = e1.timed_steps(a.steps)
    out["t_1gpu_ms"] = t1 / a.steps
    e1.close()
    torch.cuda.empty_cache()
    for world in [w for w in (2, 4, 8) if w <= a.gpus]:
        r = world // 2 - 1 if world > 2 else 0  # an interior rank when one exists
        wdom = (n, n, n * world) if a.weak else dom
        eng = V.DenseEngine(domain=wdom, precision="fp32", partitions=world, first_partition=r, local_partitions=1)
        flags = C.c_void_p()
        check(lib.voxl_dense_enable_distributed(eng._h, C.byref(flags)))
        # release every wait: flags[0] = flags[1] = 2^31
        torch.cuda.synchronize()
        from paper_2503_07898_b200.multigpu import _CudaArray

        fl = torch.as_tensor(_CudaArray(flags.value, 4, "<i4"), device="cuda")
        fl[:2].fill_(2 ** 31 - 1)  # word 2 is the stall marker: keep 0
        torch.cuda.synchronize()
        keep = [fl]
        dummy_flags = torch.zeros(8, dtype=torch.int32, device="cuda")
        keep.append(dummy_flags)
        for nb in (r - 1, r + 1):
            if 0 <= nb < world:
                _, nbytes = eng.buffer(r, 0)
                b0 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                b1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
                keep += [b0, b1]
                eng.attach_peer(nb, b0.data_ptr(), b1.data_ptr())
        up = dummy_flags.data_ptr() + 4 if r > 0 else None
        low = dummy_flags.data_ptr() if r < world - 1 else None
        check(lib.voxl_dense_attach_flags(eng._h, C.c_void_p(up), C.c_void_p(low)))
        eng.set_equilibrium()
        eng.timed_steps(a.warmup)
        tr, _ = eng.timed_steps(a.steps)
        tr /= a.steps
        if a.weak:  # per-rank work fixed: efficiency = t_1 / t_N
            out[f"rank{r}_of_{world}"] = {"t_rank_ms": round(tr, 4),
                                          "efficiency_bound": round(out["t_1gpu_ms"] / tr, 4),
                                          "MLUPS_job_bound": round(world * n ** 3 / (tr / 1e3) / 1e6, 1)}
        else:
            out[f"rank{r}_of_{world}"] = {"t_rank_ms": round(tr, 4),
                                          "efficiency_bound": round(out["t_1gpu_ms"] / (world * tr), 4),
                                          "MLUPS_job_bound": round(n ** 3 / (tr / 1e3) / 1e6, 1)}
        eng.close()
        del keep
        torch.cuda.empty_cache()
    out["t_1gpu_ms"] = round(out["t_1gpu_ms"], 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
