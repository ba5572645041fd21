#!/usr/bin/env python
"""Host launch overhead of the multi-device OCC schedule and what CUDA-graph
replay takes off it: P partitions on one process (all on device 0 here, each
with its own interior / shared-layer streams and cross-stream events), steps
enqueued from the host (graph_steps=0) vs replayed from captured graphs of G
steps. Per-step wall time over K steps (one sync), best of 3.

    python tools/graph_replay.py [--sizes 64,128,256,512] [--parts 1,2,4,8] [--k 200]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2503_07898_b200 as V  # noqa: E402


def per_step(e, k):
    e.step(4)
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        e.step(k)
        best = min(best, (time.perf_counter() - t) / k * 1e3)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128,256,512")
    ap.add_argument("--parts", default="1,2,4,8")
    ap.add_argument("--k", type=int, default=200)
    a = ap.parse_args()
    for n in map(int, a.sizes.split(",")):
        k = a.k if n <= 256 else max(20, a.k // 10)
        single = V.DenseEngine(domain=(n, n, n), precision="fp32")
        single.set_equilibrium(1.0, (0.0, 0.0, 0.0))
        t1 = per_step(single, k)
        single.close()
        for p in map(int, a.parts.split(",")):
            row = {"n": n, "partitions": p, "one_stream_ms": round(t1, 4)}
            for g in (0, 8):
                e = V.DenseEngine(domain=(n, n, n), precision="fp32", partitions=p, devices=[0] * p, graph_steps=g)
                e.set_equilibrium(1.0, (0.0, 0.0, 0.0))
                row["host_enqueue_ms" if g == 0 else "graph_replay_ms"] = round(per_step(e, k), 4)
                e.close()
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
