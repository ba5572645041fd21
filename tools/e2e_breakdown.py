#!/usr/bin/env python
"""Where the e2e time goes: set_canonical (H2D fp64 + scatter), K x step_probe,
get_canonical (gather + D2H fp64), and raw pinned H2D / D2H bandwidth."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2503_07898_b200 as V

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
vox = n ** 3
Q = 19
out = {"n": n, "steps": steps}
hin = torch.empty(vox * Q, dtype=torch.float64, pin_memory=True)
hout = torch.empty(vox * Q, dtype=torch.float64, pin_memory=True)
d = torch.empty(vox * Q, dtype=torch.float64, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(hin, non_blocking=True)), ("d2h", lambda: hout.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    out[name + "_GBs_torch_copy"] = round(vox * Q * 8 / dt / 1e9, 2)
del d
torch.cuda.empty_cache()
w = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)
hin.numpy().reshape(vox, Q)[:] = w
e = V.DenseEngine(domain=(n, n, n), precision="fp32")
e.set_canonical(hin.numpy()); e.step_probe(); e.get_canonical(hout.numpy())
t0 = time.perf_counter(); e.set_canonical(hin.numpy()); t1 = time.perf_counter()
for _ in range(steps):
    e.step_probe()
t2 = time.perf_counter(); e.get_canonical(hout.numpy()); t3 = time.perf_counter()
out.update(set_s=round(t1 - t0, 4), steps_s=round(t2 - t1, 4), get_s=round(t3 - t2, 4),
           set_GBs=round(vox * Q * 8 / (t1 - t0) / 1e9, 2), get_GBs=round(vox * Q * 8 / (t3 - t2) / 1e9, 2),
           step_probe_ms=round((t2 - t1) / steps * 1e3, 4))
t = time.perf_counter(); e.step(steps); t4 = time.perf_counter()
out["step_ms_nosync"] = round((t4 - t) / steps * 1e3, 4)
print(json.dumps(out))
