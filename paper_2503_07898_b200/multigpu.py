"""One process per GPU: the dense engine over z-slabs with a zero-copy halo.

Rank r owns partition r of ``decompose(domain, world)`` (partition.cpp:20-41).
At construction the ranks exchange CUDA IPC handles of their two population
buffers and of their step-flag words through ``torch.distributed``
(plumbing only); afterwards every step is device-driven:

    wait(flags >= t) -> shared layers k=0,n-1 (+ peer stores of the 5 crossing
    populations into the neighbours' halo spans) -> signal(t+1) -> interior.

The comparison path (``halo_mode="copy"``) runs the same two-stream OCC
schedule without peer stores and exchanges the same contiguous spans with NCCL
send/recv (``exchange_halos``), the transport the paper's GPU baseline uses.
The exchange is enqueued on the shared-layer stream right after the shared
layers, so it overlaps the interior kernel exactly like the zero-copy stores
do; only the transport differs. Over gloo (ranks sharing one GPU in the tests)
the spans are staged through host memory.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import check, lib
from .dense import DenseEngine, plan_ledger


def exchange_plan(rank: int, world: int, **desc):
    """(sends, recvs) of one halo update for `rank`, from the reference-order
    ledger (partition.cpp:163-206): lists of (peer, element offset, elements)."""
    recs = plan_ledger(0, partitions=world, **desc)
    sends = [(r.dst, r.base_src, r.elements) for r in recs if r.src == rank]
    recvs = [(r.src, r.base_dst, r.elements) for r in recs if r.dst == rank]
    return sends, recvs


def exchange_halos(dist, buf, sends, recvs, group=None):
    """NCCL/gloo send/recv of the halo spans of one flat population buffer
    (a torch tensor on the rank's device, or on CPU for gloo)."""
    ops = []
    for peer, base, n in recvs:
        ops.append(dist.P2POp(dist.irecv, buf[base:base + n], peer, group))
    for peer, base, n in sends:
        ops.append(dist.P2POp(dist.isend, buf[base:base + n], peer, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


class _CudaArray:
    """Minimal __cuda_array_interface__ view of an engine buffer."""

    def __init__(self, ptr, nelem, typestr):
        self.__cuda_array_interface__ = {"shape": (nelem,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class DistributedDense:
    """The rank-local slab of a dense domain decomposed over all ranks."""

    def __init__(self, domain=(512, 512, 512), precision="fp32", halo_mode="zero_copy", layout="DisagSoA",
                 lattice="D3Q19", tau=0.56, scenario="lid_driven_cavity", velocity=(0.05, 0.0, 0.0)):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.halo_mode = halo_mode
        self.desc = dict(lattice=lattice, domain=tuple(domain), tau=tau, scenario=scenario, velocity=velocity,
                         layout=layout, precision=precision)
        self.eng = DenseEngine(partitions=self.world, halo_mode=halo_mode, first_partition=self.rank,
                               local_partitions=1, **self.desc)
        dev = torch.cuda.current_device()
        esize = 8 if precision == "fp64" else 4
        self.typestr = "<f8" if esize == 8 else "<f4"
        # IPC export of both buffers and the flag words
        raw = []
        for w in range(2):
            p = C.c_void_p()
            check(lib.voxl_dense_raw_buffer(self.eng._h, self.rank, w, C.byref(p)))
            raw.append(p.value)
        flags = C.c_void_p()
        check(lib.voxl_dense_enable_distributed(self.eng._h, C.byref(flags)))
        if halo_mode != "zero_copy":
            flags = C.c_void_p()  # copy mode: no step flags, NCCL orders the exchange
        handles = {"rank": self.rank, "device": dev, "bufs": [], "flags": None}
        for ptr in raw:
            h = C.create_string_buffer(64)
            check(lib.voxl_ipc_export(C.c_void_p(ptr), h))
            handles["bufs"].append(h.raw)
        if flags.value:
            h = C.create_string_buffer(64)
            check(lib.voxl_ipc_export(flags, h))
            handles["flags"] = h.raw
        gathered = [None] * self.world
        dist.all_gather_object(gathered, handles)
        periodic = scenario == "periodic_box"
        up = self.rank - 1 if self.rank > 0 else (self.world - 1 if periodic else -1)
        low = self.rank + 1 if self.rank < self.world - 1 else (0 if periodic else -1)
        self.up, self.low = up, low
        self._opened = []
        if halo_mode == "zero_copy":
            slots = {}
            for nb in sorted({x for x in (up, low) if x >= 0}):
                g = gathered[nb]
                if g["device"] != dev:
                    check(lib.voxl_enable_peer_access(g["device"]))
                ptrs = []
                for hb in g["bufs"]:
                    if nb == self.rank:
                        ptrs = raw
                        break
                    p = C.c_void_p()
                    check(lib.voxl_ipc_open(hb, C.byref(p)))
                    self._opened.append(p.value)
                    ptrs.append(p.value)
                check(lib.voxl_dense_attach_peer(self.eng._h, nb, C.c_void_p(ptrs[0]), C.c_void_p(ptrs[1])))
                if nb == self.rank:
                    slots[nb] = flags.value
                else:
                    p = C.c_void_p()
                    check(lib.voxl_ipc_open(g["flags"], C.byref(p)))
                    self._opened.append(p.value)
                    slots[nb] = p.value
            up_slot = slots[up] + 4 if up >= 0 else None
            low_slot = slots[low] + 0 if low >= 0 else None
            check(lib.voxl_dense_attach_flags(self.eng._h, C.c_void_p(up_slot), C.c_void_p(low_slot)))
        else:
            self.sends, self.recvs = exchange_plan(self.rank, self.world, **{k: v for k, v in self.desc.items()
                                                                            if k != "precision"})
            size = self.eng.buffer(self.rank, 0)[1] // esize
            self._views = [torch.as_tensor(_CudaArray(p, size, self.typestr), device="cuda") for p in raw]
            self._raw = raw
            ss = C.c_void_p()
            check(lib.voxl_dense_shared_stream(self.eng._h, C.byref(ss)))
            self._stream = torch.cuda.ExternalStream(ss.value)
        dist.barrier()

    # -- engine facade ----------------------------------------------------------------
    def owned_voxels(self) -> int:
        v = C.c_int64()
        check(lib.voxl_dense_owned_voxels(self.eng._h, C.byref(v)))
        return v.value

    def set_equilibrium(self, rho=1.0, u=(0.0, 0.0, 0.0)):
        self.eng.set_equilibrium(rho, u)
        self.dist.barrier()

    def slab(self):
        """[begin, end) of this rank's partition along the partition axis."""
        from .dense import decompose

        dom = self.desc["domain"]
        axis = 1 if self.desc["lattice"] == "D2Q9" else 2
        return decompose(dom if len(dom) == 3 else (dom[0], dom[1], 1), self.world, axis,
                         self.desc["scenario"] == "periodic_box")[self.rank]

    def set_canonical_planes(self, host, k_begin, k_end):
        k0, k1 = self.slab()
        if not (k0 <= k_begin <= k_end <= k1):
            raise ValueError(f"set_canonical_planes: planes [{k_begin}, {k_end}) outside this rank's slab [{k0}, {k1})")
        h = np.ascontiguousarray(host, np.float64)
        dom = self.desc["domain"]
        cross = dom[0] * (dom[1] if len(dom) == 3 and self.desc["lattice"] != "D2Q9" else 1)
        if h.size != (k_end - k_begin) * cross * self.eng.q:
            raise ValueError("set_canonical_planes: size mismatch")
        check(lib.voxl_dense_set_planes(self.eng._h, h.ctypes.data, k_begin, k_end))

    def get_canonical_planes(self, k_begin, k_end, out=None):
        dom = self.desc["domain"]
        cross = dom[0] * (dom[1] if len(dom) == 3 and self.desc["lattice"] != "D2Q9" else 1)
        n = (k_end - k_begin) * cross * self.eng.q
        if out is None:
            out = np.empty(n, np.float64)
        k0, k1 = self.slab()
        if not (k0 <= k_begin <= k_end <= k1):
            raise ValueError(f"get_canonical_planes: planes [{k_begin}, {k_end}) outside this rank's slab [{k0}, {k1})")
        if not (out.dtype == np.float64 and out.size == n and out.flags.c_contiguous):
            raise ValueError("get_canonical_planes: out must be a contiguous float64 array of the slab's size")
        check(lib.voxl_dense_get_planes(self.eng._h, out.ctypes.data, k_begin, k_end))
        return out

    def refresh_halos(self):
        """After a canonical load: fill every neighbour halo (peer copies or NCCL)."""
        self.dist.barrier()
        if self.halo_mode == "zero_copy":
            check(lib.voxl_dense_halo_push(self.eng._h))
        else:
            self._nccl_exchange()
        self.dist.barrier()

    def _nccl_exchange(self):
        """Halo spans of the current buffer, on the shared-layer stream (after
        this step's shared layers, next to its interior kernel)."""
        import torch

        cur = self.eng.buffer(self.rank, 0)[0]
        view = self._views[self._raw.index(cur)]
        with torch.cuda.stream(self._stream):
            if self.dist.get_backend() == "nccl":
                exchange_halos(self.dist, view, self.sends, self.recvs)
                return
            # gloo moves host tensors only: stage the spans through host memory
            self._stream.synchronize()
            host = {}
            for peer, base, n in self.sends + self.recvs:
                host[(base, n)] = view[base:base + n].cpu()
            ops = [self.dist.P2POp(self.dist.irecv, host[(b, n)], peer) for peer, b, n in self.recvs]
            ops += [self.dist.P2POp(self.dist.isend, host[(b, n)], peer) for peer, b, n in self.sends]
            if ops:
                for w in self.dist.batch_isend_irecv(ops):
                    w.wait()
            for peer, base, n in self.recvs:
                view[base:base + n].copy_(host[(base, n)])

    def step(self, n=1):
        if self.halo_mode == "zero_copy":
            self.eng.step(n)
        else:
            for _ in range(n):
                self.eng.enqueue(1)
                self._nccl_exchange()
            self.eng.synchronize()

    def step_probe(self):
        """One step with this rank's probe_field fused (lbm.cpp:116-138); the
        diagnostics row covers the rank's own slab. Rows combine across ranks
        as mass = sum, max_speed = max (`combine_rows`), so run()'s per-step
        diagnostics need no per-step collective."""
        d = self.eng.step_probe()
        if self.halo_mode != "zero_copy":
            self._nccl_exchange()
        return d

    def step_probe_n(self, n):
        """n steps with this rank's probe_field fused, rows read back once per
        256 steps (zero-copy halo: the engine's own batched loop); the copy
        mode exchanges halos from the host between steps, so it probes step
        by step. Rows cover the rank's slab (`combine_rows` across ranks)."""
        if self.halo_mode == "zero_copy":
            return self.eng.step_probe_n(n)
        return [self.step_probe() for _ in range(n)]

    def timed_steps(self, n):
        if self.halo_mode == "zero_copy":
            return self.eng.timed_steps(n)
        import torch

        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(self._stream)
        self.step(n)
        end.record(self._stream)
        end.synchronize()
        ms = start.elapsed_time(end)
        return ms, ms

    def probe(self):
        """Mass summed over ranks, max speed max over ranks."""
        import torch

        d = self.eng.probe()
        dev = "cuda" if self.dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([d.mass], dtype=torch.float64, device=dev)
        s = torch.tensor([d.max_speed, float(d.unstable)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t)
        self.dist.all_reduce(s, op=self.dist.ReduceOp.MAX)
        d.mass, d.max_speed, d.unstable = float(t.item()), float(s[0].item()), int(s[1].item())
        return d

    def close(self):
        for p in self._opened:
            lib.voxl_ipc_close(C.c_void_p(p))
        self._opened = []
        self.eng.close()
