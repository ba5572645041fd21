// dense.cu -- dense pull + BGK kernels and the partitioned engine (see dense.cuh).
//
// Hot kernel: dense_step_kernel. One thread per voxel; a block is 256 voxels of
// one cross-section row, so each warp reads 32 consecutive values of a
// population plane (x-shifted by at most one element: the overfetched sector
// is the neighbouring warp's and hits L2) and writes 128 B aligned runs. Every
// stored population is read exactly once and written exactly once per step:
// algorithmic traffic is 2*Q*sizeof(real) bytes per lattice update (152 B for
// D3Q19 fp32), the HBM roofline of this operator.
#include "dense.cuh"
#include "digest.cuh"
#include "canon_io.cuh"
#include "lattice.cuh"
#include "diag_ring.cuh"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <type_traits>

#include <dlfcn.h>
#include <nccl.h>

namespace voxl_b200 {

namespace {

#ifndef VOXL_DENSE_BLOCK
#define VOXL_DENSE_BLOCK 256
#endif
#ifndef VOXL_DENSE_MINB
#define VOXL_DENSE_MINB 0
#endif
// D3Q27 fp32 at 512^3 (-DVOXL_DENSE_MINB27 sweep, ms per step / per
// step_probe): plain step unconstrained (54 registers, 4 CTAs/SM) 4.58, with
// 5 CTAs/SM 4.72, 4 CTAs/SM at 48 registers 4.73-4.74; fused-probe step with
// 6 CTAs/SM (40 registers, 100 B spill) 5.17, with 5 CTAs/SM 4.77.
#ifndef VOXL_DENSE_MINB27
#define VOXL_DENSE_MINB27 0
#endif
#ifndef VOXL_DIAG_MINB27
#define VOXL_DIAG_MINB27 5
#endif
// 256-thread CTAs: +4 % DRAM throughput over 128 on B200 (tools/micro/membw.cu).
// Sweep at 512^3 (-DVOXL_DENSE_BLOCK / MINB sweep, GLUPS): 256 threads 42.70-42.82,
// 512 42.54-42.66, 512 with 3 CTAs/SM 42.66, 1024 28.2, 256 with 5 CTAs/SM 41.68.
constexpr int kBlock = VOXL_DENSE_BLOCK;
#ifndef VOXL_DIAG_MINB
#define VOXL_DIAG_MINB 6
#endif
// fused probe: one lane per warp commits the warp's partial into the step's
// accumulator lanes (diag_ring.cuh) with fire-and-forget reductions -- no CTA
// barrier and no partial array in HBM. Earlier layouts at 512^3 (step_probe,
// ms): per-warp 16-byte partials + two reduction kernels 3.33-3.35 (+0.28 GB
// of DRAM writes per launch), per-CTA partials after a barrier 3.41-3.43.

template <int Q, class R>
struct StepArgs {
    const R* in;
    R* out;
    long long plane[kGroupCount][Q];  // element offset per (group, component)
    R* up_out;                        // upper neighbour's next buffer (its LowerHalo), or null
    long long up_plane[Q];
    unsigned up_mask;
    R* low_out;                       // lower neighbour's next buffer (its UpperHalo), or null
    long long low_plane[Q];
    unsigned low_mask;
    R lid[Q];  // moving-wall term per direction (lbm.hpp:66-69), 0 where unused
    R omega, keep;
    int na, nb, n, s;
    int k_first, k_step;
    int kg0, nk;
    int wall_a, wall_b, wall_k;
    int periodic_a, periodic_b;
    int has_lid;
    int step;
    const int* step_base;  // graph replays: absolute step = *step_base + step (read only on a failure)
    int remote_fence;  // remote halo stores cross a process/device: membar.sys after them
    int uniform_groups;  // all groups share one plane table (AoS / SoA)
    long long fast_base;  // byte offset of the interior plane table's component 0
    long long fast_in_off[Q];   // per-direction pull byte offset relative to fast_base + lin
    long long fast_out_off[Q];  // per-direction store byte offset
    int* error_flag;
    unsigned long long* diag_acc;    // fused probe: the step's accumulator lanes (diag_ring.cuh)
    unsigned long long* diag_bad;    // (canonical voxel << 5) | population of the first offender
};

__device__ __forceinline__ int group_of(int k, int n) {
    return k == -1 ? 0 : (k == 0 ? 1 : (k == n - 1 ? 3 : (k == n ? 4 : 2)));
}

// Cache hints on the fast path, measured at 512^3 (-DVOXL_LD_HINT / ST_HINT sweep,
// GLUPS): plain 42.90, st.global.cs stores 42.29, ld.global.lu loads 40.46,
// both 38.7 -- the x-shifted pulls reuse lines through L2, so plain wins.
#ifndef VOXL_ST_HINT  // fast-path stores: 0 plain st.global, 1 st.global.cs (evict-first streaming)
#define VOXL_ST_HINT 0
#endif
#ifndef VOXL_LD_HINT  // fast-path loads: 0 ld.global.nc, 1 ld.global.lu (last use)
#define VOXL_LD_HINT 0
#endif

#ifndef VOXL_OPAQUE_BASE  // bit 0: the fast path's pull base, bit 1: its store base
#define VOXL_OPAQUE_BASE 2
#endif

/// Hide a pointer's provenance from the optimiser (no instruction emitted).
template <class T>
__device__ __forceinline__ void opaque_ptr(T*& p) {
#if VOXL_OPAQUE_BASE
    asm("" : "+l"(p));
#endif
}

template <class R>
__device__ __forceinline__ R ld_ro(const R* p) {
    return __ldg(p);
}

template <class R>
__device__ __forceinline__ R ld_fast(const R* p) {
#if VOXL_LD_HINT == 1
    return __ldlu(p);
#else
    return __ldg(p);
#endif
}

template <class R>
__device__ __forceinline__ void st_fast(R* p, R v) {
#if VOXL_ST_HINT == 1
    __stcs(p, v);
#else
    // st.global spelled out: the fast path's base pointer is opaque to the
    // compiler (opaque_ptr), which would otherwise emit generic ST
    if constexpr (sizeof(R) == 4) asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
    else asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
#endif
}

/// Fused pull-stream + bounce-back/lid + BGK for one voxel per thread
/// (gather_pull lbm.hpp:40-74 then bgk_relax lattice.cpp:131-138).
/// AXIS is the partition axis (2 in 3D, 1 in 2D); `a` is x, `b` the remaining
/// cross-section axis, `k` the local coordinate along AXIS.
template <class L, class R, bool Exact, bool AOS, int AXIS, bool WRAP, bool DIAG>
__global__ void __launch_bounds__(kBlock, sizeof(R) != 4 ? 0
                                          : DIAG ? (L::Q == 27 ? VOXL_DIAG_MINB27 : VOXL_DIAG_MINB) * 256 / kBlock
                                                 : (L::Q == 27 ? VOXL_DENSE_MINB27 : VOXL_DENSE_MINB))
    dense_step_kernel(const __grid_constant__ StepArgs<L::Q, R> A) {
    constexpr int Q = L::Q;
    constexpr int OTHER = AXIS == 2 ? 1 : 2;
    using Ar = Arith<R, Exact>;
    const int a = blockIdx.x * kBlock + threadIdx.x;
    R f[Q];
    const bool live = a < A.na;
    // fused probe_field (DIAG): per-voxel mass and |u|^2 of this step's
    // result, and the instability test on the post-collision populations
    using P = std::conditional_t<Exact || sizeof(R) == 8, double, float>;
    P dg_mass = P(0), dg_v2 = P(0);
    int dg_bad = -1;  // first offending population of this voxel (probe_voxel)
    if (live) [&] {
    const int b = blockIdx.y;
    const int k = A.k_first + int(blockIdx.z) * A.k_step;
    const int kg = A.kg0 + k;
    const int na = A.na, s = A.s;
    const int cross = b * na + a;
    const int lin = (k + 1) * s + cross;
    const int gm = group_of(k - 1, A.n), g0 = group_of(k, A.n), gp = group_of(k + 1, A.n);

    constexpr long long VS = AOS ? Q : 1;

    // Fast path (warp-uniform): no lane of this warp touches a wall and the
    // source planes k-1..k+1 share one plane table (interior group, or any
    // group of a non-disaggregated layout). Every population address is then
    // one per-thread base pointer plus a block-uniform byte offset per
    // direction, so each pull is a single LDG [R.64 + UR] and each push a
    // single STG.
    if constexpr (!WRAP) {
        const int a_w0 = a - (threadIdx.x & 31);
        const int a_w1 = min(a_w0 + 31, na - 1);
        const bool wall = (A.wall_a && (a_w0 == 0 || a_w1 == na - 1)) || (A.wall_b && (b == 0 || b == A.nb - 1)) ||
                          (A.wall_k && (kg == 0 || kg == A.nk - 1)) || a_w1 - a_w0 != 31;
        const bool uniform_planes = A.uniform_groups || (gm == 2 && g0 == 2 && gp == 2);
        if (!wall && uniform_planes) {
            const char* base_in = reinterpret_cast<const char*>(A.in) + A.fast_base + (long long)lin * (VS * sizeof(R));
            // opaque to the optimiser: otherwise nvcc re-associates the sum
            // and spends three integer adds per access (lin*4 + off_i, + base,
            // carry) instead of two (base + off_i with carry); measured on the
            // stores only -- on the pulls it costs the DIAG kernel a spill
#if VOXL_OPAQUE_BASE & 1
            opaque_ptr(base_in);
#endif
            static_for<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                f[i] = ld_fast(reinterpret_cast<const R*>(base_in + A.fast_in_off[i]));
            });
            bool ok = true;
            R rho, u[3], dr = R(0);
            if constexpr (Exact) bgk_relax<L, R, true>(f, A.omega, A.keep, rho, u, ok);
            else bgk_relax_shifted<L, R, kBgkTrim && !DIAG>(f, A.omega, A.keep, rho, u, ok, DIAG ? &dr : nullptr);
            if (!ok) atomicMin(A.error_flag, A.step_base ? *A.step_base + A.step : A.step);
            if constexpr (DIAG) probe_voxel<L, R, Exact, P>(f, rho, dr, u, dg_mass, dg_v2, dg_bad);
            char* base_out = reinterpret_cast<char*>(A.out) + A.fast_base + (long long)lin * (VS * sizeof(R));
#if VOXL_OPAQUE_BASE & 2
            opaque_ptr(base_out);
#endif
            static_for<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                st_fast(reinterpret_cast<R*>(base_out + A.fast_out_off[i]), f[i]);
            });
            return;
        }
    }

    const bool a_lo = A.wall_a && a == 0, a_hi = A.wall_a && a == na - 1;
    const bool b_lo = A.wall_b && b == 0, b_hi = A.wall_b && b == A.nb - 1;
    const bool k_lo = A.wall_k && kg == 0, k_hi = A.wall_k && kg == A.nk - 1;
    static_for<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int ea = L::e(i, 0), eb = L::e(i, OTHER), ek = L::e(i, AXIS);
        bool oob = false;
        if constexpr (ea > 0) oob = oob || a_lo;
        if constexpr (ea < 0) oob = oob || a_hi;
        if constexpr (eb > 0) oob = oob || b_lo;
        if constexpr (eb < 0) oob = oob || b_hi;
        if constexpr (ek > 0) oob = oob || k_lo;
        if constexpr (ek < 0) oob = oob || k_hi;
        int src_lin;
        if constexpr (WRAP) {
            int sa = a - ea, sb = b - eb;
            if (A.periodic_a) sa = sa < 0 ? sa + na : (sa >= na ? sa - na : sa);
            if (A.periodic_b) sb = sb < 0 ? sb + A.nb : (sb >= A.nb ? sb - A.nb : sb);
            src_lin = (k - ek + 1) * s + sb * na + sa;
        } else {
            src_lin = lin - ea - eb * na - ek * s;
        }
        constexpr int sel = ek > 0 ? 0 : (ek < 0 ? 2 : 1);
        const int gs = sel == 0 ? gm : (sel == 2 ? gp : g0);
        const R* p_src = A.in + A.plane[gs][i] + (long long)src_lin * VS;
        constexpr int oi = L::opp(i);
        const R* p_own = A.in + A.plane[g0][oi] + (long long)lin * VS;
        R v = ld_ro(oob ? p_own : p_src);
        if constexpr (ek < 0) {
            if (A.has_lid && k_hi) v = Ar::add(v, A.lid[i]);
        }
        f[i] = v;
    });

    bool ok = true;
    R rho, u[3], dr = R(0);
    if constexpr (Exact) bgk_relax<L, R, true>(f, A.omega, A.keep, rho, u, ok);
    else bgk_relax_shifted<L, R, kBgkTrim && !DIAG>(f, A.omega, A.keep, rho, u, ok, DIAG ? &dr : nullptr);
    if (!ok) atomicMin(A.error_flag, A.step_base ? *A.step_base + A.step : A.step);
    if constexpr (DIAG) probe_voxel<L, R, Exact, P>(f, rho, dr, u, dg_mass, dg_v2, dg_bad);

    static_for<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        A.out[A.plane[g0][i] + (long long)lin * VS] = f[i];
    });
    // Zero-copy halo: the shared layers store their face-crossing populations
    // directly into the neighbour's halo group of its next buffer
    // (halo_update partition.cpp:196-205 without the copy).
    if (k == 0 && A.up_out) {
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            if ((A.up_mask >> i) & 1u) A.up_out[A.up_plane[i] + (long long)cross * VS] = f[i];
        });
    }
    if (k == A.n - 1 && A.low_out) {
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            if ((A.low_mask >> i) & 1u) A.low_out[A.low_plane[i] + (long long)cross * VS] = f[i];
        });
    }
    // Cross-GPU ordering: the peer stores above must be performed before this
    // step's completion flag (written by signal_kernel after this kernel).
    if (A.remote_fence && ((k == 0 && A.up_out) || (k == A.n - 1 && A.low_out))) __threadfence_system();
    }();

    // Fused probe_field (lbm.cpp:116-138): the per-voxel terms were taken in
    // probe_voxel; the warp's mass and max |u|^2 go into the step's
    // accumulator lanes (order-independent integer sums, diag_ring.cuh) and
    // the first offender into the step's bad word.
    if constexpr (DIAG) {
        P pm = dg_mass, pv = dg_v2;
        // the voxel's coordinates are re-derived from the special registers
        // here rather than kept live through the step (register budget)
        if (dg_bad >= 0) {
            const unsigned long long canon =
                (unsigned long long)(A.kg0 + A.k_first + int(blockIdx.z) * A.k_step) * A.s +
                (unsigned long long)(blockIdx.y * A.na + blockIdx.x * kBlock + threadIdx.x);
            atomicMin(A.diag_bad, (canon << 5) | (unsigned long long)dg_bad);
        }
        const unsigned live_lanes = __ballot_sync(0xffffffffu, int(blockIdx.x * kBlock + threadIdx.x) < A.na);
        // accumulator lane: any mapping gives the same (integer) sums; the
        // SM id and the warp's slot in its CTA spread the warps resident at
        // one time over the lanes in two instructions
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        const unsigned long long warp_id = smid * (kBlock / 32) + (threadIdx.x >> 5);
        if constexpr (std::is_same_v<P, float>) {
            diag_warp_commit_f32<true, false>(A.diag_acc, warp_id, pm, pv, live_lanes);
        } else {
            for (int o = 16; o > 0; o >>= 1) {
                pm += __shfl_xor_sync(0xffffffffu, pm, o);
                pv = max(pv, __shfl_xor_sync(0xffffffffu, pv, o));
            }
            if ((threadIdx.x & 31) == 0 && live_lanes) diag_commit(A.diag_acc, warp_id, double(pm), double(pv));
        }
    }
}

// ---- AoS step through shared-memory plane tiles (fp32, 3D) --------------------------
//
// The AoS layout keeps a voxel's Q populations in one 4Q-byte record. The
// one-voxel-per-thread kernel above pulls population i of record (x - e_i):
// a warp's load then touches 32 records 4Q bytes apart (Q sectors for 128
// useful bytes), and the x/y/z neighbourhood of a warp (~34 x 9 records) is
// far more than L1 holds per warp at full occupancy, so every pull goes to L2
// at Q-fold sector amplification (21 % of copy bandwidth measured).
//
// This kernel stages records instead of populations. A CTA owns a 32 x 8
// (x, y) column of the slab and marches it along z through a ring of plane
// tiles (34 x 10 records with the x/y halo) in shared memory. Each tile row
// is one contiguous span of global memory (the records of consecutive x are
// adjacent) and is filled by 16-byte cp.async (TMA-free async copies; the
// smem row is shifted so that it shares the global span's 16-byte phase),
// one plane ahead of the plane being computed. A voxel's pulls are then
// shared-memory reads (record stride Q words, odd for Q = 19 / 27: bank-
// conflict free), the collision is the same bgk_relax_shifted as every
// other fp32 kernel (bitwise equal results), and the outputs go back through
// the ring slot the plane k-1 tile just vacated, so each output row is again
// one contiguous span of 16-byte stores. Traffic: every record is read once
// per plane pass plus the tile halo (34 x 10 / 256 = 1.33x from L2, mostly
// hits) and written once.
#ifndef VOXL_AOS_TY
#define VOXL_AOS_TY 8
#endif
#ifndef VOXL_AOS_CHUNK
#define VOXL_AOS_CHUNK 96
#endif
#ifndef VOXL_AOS_SLOTS19
#define VOXL_AOS_SLOTS19 4
#endif
#ifndef VOXL_AOS_MINB
#define VOXL_AOS_MINB 2
#endif
constexpr int kAosTX = 32, kAosTY = VOXL_AOS_TY, kAosChunk = VOXL_AOS_CHUNK;
constexpr int kAosThreads = kAosTX * kAosTY;

/// Tile geometry in words: row pitch (a multiple of 4, so every row has the
/// same 16-byte phase), plane slot size (one pitch of phase slack), slots.
template <int Q>
struct AosTile {
    static constexpr int RX = kAosTX + 2, RY = kAosTY + 2;
    static constexpr int pitch = (RX * Q + 3) / 4 * 4;
    static constexpr int slot_words = RY * pitch + 4;
    static constexpr int slots = Q <= 19 ? VOXL_AOS_SLOTS19 : 3;  // 2 CTAs per SM either way
    static constexpr int smem_bytes = slots * slot_words * 4;
};

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(float* smem, const float* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

/// A warp copies one contiguous row of `nw` words global -> shared (cp.async):
/// 16-byte chunks where both sides share the 16-byte phase, single words for
/// the unaligned head and tail (never outside the row).
__device__ __forceinline__ void aos_row_load(float* sm, const float* g, int nw, int lane) {
    const int head = int((4 - ((reinterpret_cast<std::uintptr_t>(g) >> 2) & 3)) & 3);
    const bool same_phase = ((reinterpret_cast<std::uintptr_t>(g) ^ reinterpret_cast<std::uintptr_t>(sm)) & 15) == 0;
    if (!same_phase || nw < head + 4) {
        for (int o = lane; o < nw; o += 32) cp_async4(sm + o, g + o);
        return;
    }
    const int chunks = (nw - head) >> 2, body_end = head + 4 * chunks;
    if (lane < head) cp_async4(sm + lane, g + lane);
    if (lane < nw - body_end) cp_async4(sm + body_end + lane, g + body_end + lane);
    for (int c = lane; c < chunks; c += 32) cp_async16(sm + head + 4 * c, g + head + 4 * c);
}

/// A warp stores one contiguous row of `nw` words shared -> global.
__device__ __forceinline__ void aos_row_store(float* g, const float* sm, int nw, int lane) {
    const int head = int((4 - ((reinterpret_cast<std::uintptr_t>(g) >> 2) & 3)) & 3);
    const bool same_phase = ((reinterpret_cast<std::uintptr_t>(g) ^ reinterpret_cast<std::uintptr_t>(sm)) & 15) == 0;
    if (!same_phase || nw < head + 4) {
        for (int o = lane; o < nw; o += 32) g[o] = sm[o];
        return;
    }
    const int chunks = (nw - head) >> 2, body_end = head + 4 * chunks;
    if (lane < head) g[lane] = sm[lane];
    if (lane < nw - body_end) g[body_end + lane] = sm[body_end + lane];
    for (int c = lane; c < chunks; c += 32)
        *reinterpret_cast<float4*>(g + head + 4 * c) = *reinterpret_cast<const float4*>(sm + head + 4 * c);
}

/// Plane kk (local, -1..n) of the CTA's tile into a ring slot: rows b0-1 ..
/// b0+TY, records a0-1 .. a0+TX, clipped to the slab (walls never read
/// outside it; the k = -1 / n planes are the partition halos). One warp per
/// row.
template <int Q>
__device__ __forceinline__ void aos_load_plane(const StepArgs<Q, float>& A, float* tile, int kk, int a0, int b0) {
    using T = AosTile<Q>;
    const int a_lo = max(a0 - 1, 0), a_hi = min(a0 + kAosTX, A.na - 1);
    const int b_lo = max(b0 - 1, 0), b_hi = min(b0 + kAosTY, A.nb - 1);
    const int nw = (a_hi - a_lo + 1) * Q;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    for (int bb = b_lo + warp; bb <= b_hi; bb += kAosThreads / 32) {
        const float* g = A.in + ((long long)(kk + 1) * A.s + (long long)bb * A.na + a_lo) * Q;
        float* sm = tile + (bb - (b0 - 1)) * T::pitch + (a_lo - (a0 - 1)) * Q;
        aos_row_load(sm, g, nw, lane);
    }
}

template <class L, bool DIAG>
__global__ void __launch_bounds__(kAosThreads, VOXL_AOS_MINB)
    dense_aos_tiled_kernel(const __grid_constant__ StepArgs<L::Q, float> A, int k_base, int z_stride, int chunk,
                           int k_end) {
    constexpr int Q = L::Q;
    using T = AosTile<Q>;
    constexpr int NS = T::slots;
    using R = float;
    extern __shared__ __align__(16) float aos_smem[];
    const int tx = threadIdx.x & (kAosTX - 1), ty = threadIdx.x / kAosTX;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    const int a0 = blockIdx.x * kAosTX, b0 = blockIdx.y * kAosTY;
    const int a = a0 + tx, b = b0 + ty;
    const bool live = a < A.na && b < A.nb;
    const int kb = k_base + int(blockIdx.z) * z_stride;
    const int ke = min(kb + chunk, k_end);
    // the tiles start `phase` words into their slots so that tile rows share
    // the 16-byte phase of their global spans (the same for every row and
    // plane when na * Q is a multiple of 4; otherwise rows fall back to words)
    const int a_lo = max(a0 - 1, 0);
    const int phase = int(((long long)a_lo * Q - (long long)(a_lo - (a0 - 1)) * Q) & 3);
    auto tile = [&](int kk) { return aos_smem + ((kk + 1) % NS) * T::slot_words + phase; };  // kk >= -1
    // prologue: planes kb-1, kb, kb+1, and kb+2 ahead when the ring has room
    for (int kk = kb - 1; kk <= kb + 1; ++kk) aos_load_plane<Q>(A, tile(kk), kk, a0, b0);
    cp_async_commit();
    if (NS == 4 && kb + 2 <= ke) aos_load_plane<Q>(A, tile(kb + 2), kb + 2, a0, b0);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const bool a_lo_w = A.wall_a && a == 0, a_hi_w = A.wall_a && a == A.na - 1;
    const bool b_lo_w = A.wall_b && b == 0, b_hi_w = A.wall_b && b == A.nb - 1;
    const int own = (ty + 1) * T::pitch + (tx + 1) * Q;
    for (int k = kb; k < ke; ++k) {
        const int kg = A.kg0 + k;
        using P = float;
        P dg_mass = P(0), dg_v2 = P(0);
        int dg_bad = -1;
        R f[Q];
        if (live) {
            const bool k_lo = A.wall_k && kg == 0, k_hi = A.wall_k && kg == A.nk - 1;
            const float* pm = tile(k - 1);
            const float* p0 = tile(k);
            const float* pp = tile(k + 1);
            static_for<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                constexpr int ex = L::e(i, 0), ey = L::e(i, 1), ez = L::e(i, 2);
                bool oob = false;
                if constexpr (ex > 0) oob = oob || a_lo_w;
                if constexpr (ex < 0) oob = oob || a_hi_w;
                if constexpr (ey > 0) oob = oob || b_lo_w;
                if constexpr (ey < 0) oob = oob || b_hi_w;
                if constexpr (ez > 0) oob = oob || k_lo;
                if constexpr (ez < 0) oob = oob || k_hi;
                const float* plane = ez > 0 ? pm : (ez < 0 ? pp : p0);
                constexpr int shift = -ey * T::pitch - ex * Q + i;
                R v = oob ? p0[own + L::opp(i)] : plane[own + shift];
                if constexpr (ez < 0) {
                    if (A.has_lid && k_hi) v = Arith<R, false>::add(v, A.lid[i]);
                }
                f[i] = v;
            });
            bool ok = true;
            R rho, u[3], dr = R(0);
            bgk_relax_shifted<L, R>(f, A.omega, A.keep, rho, u, ok, DIAG ? &dr : nullptr);
            if (!ok) atomicMin(A.error_flag, A.step_base ? *A.step_base + A.step : A.step);
            if constexpr (DIAG) probe_voxel<L, R, false, P>(f, rho, dr, u, dg_mass, dg_v2, dg_bad);
        }
        if constexpr (DIAG) {
            if (live && dg_bad >= 0) {
                const unsigned long long canon = (unsigned long long)kg * A.s + (unsigned long long)b * A.na + a;
                atomicMin(A.diag_bad, (canon << 5) | (unsigned long long)dg_bad);
            }
            const unsigned lanes = __ballot_sync(0xffffffffu, live);
            const unsigned long long row = ((unsigned long long)kg * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
            diag_warp_commit_f32(A.diag_acc, row * kAosTY + ty, dg_mass, dg_v2, lanes);
        }
        // the output records go through the slot of plane k-1 (read by no
        // one after this barrier), 32 records x Q words per row, 16-byte phase 0
        float* out_s = aos_smem + ((k + NS) % NS) * T::slot_words;
        __syncthreads();
        if (live) {
            static_for<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                out_s[threadIdx.x * Q + i] = f[i];
            });
        }
        __syncthreads();
        {
            // output rows: contiguous spans of (records x Q) words; the shared
            // layers also store them into the neighbour's halo plane
            // (zero-copy halo: AoS sends every population)
            const int nw = min(kAosTX, A.na - a0) * Q;
            const int bb = b0 + warp;
            if (bb < A.nb) {
                const long long cross = ((long long)bb * A.na + a0) * Q;
                const float* src = out_s + warp * kAosTX * Q;
                aos_row_store(A.out + (long long)(k + 1) * A.s * Q + cross, src, nw, lane);
                if (k == 0 && A.up_out) aos_row_store(A.up_out + A.up_plane[0] + cross, src, nw, lane);
                if (k == A.n - 1 && A.low_out) aos_row_store(A.low_out + A.low_plane[0] + cross, src, nw, lane);
                if (A.remote_fence && ((k == 0 && A.up_out) || (k == A.n - 1 && A.low_out))) __threadfence_system();
            }
        }
        __syncthreads();  // the staging slot is free: the next plane goes there
        const int next = k + NS - 1;  // k+3 (4 slots, k+2 already in flight) or k+2 (3 slots)
        if (next <= ke && next <= A.n) aos_load_plane<Q>(A, tile(next), next, a0, b0);
        cp_async_commit();
        if constexpr (NS == 4) cp_async_wait<1>();  // plane k+2 landed (k+3 may be in flight)
        else cp_async_wait<0>();
        __syncthreads();
    }
    cp_async_wait<0>();
}

constexpr int kOpIdentity = int(Operator::Identity);
constexpr int kOpJacobi2 = int(Operator::Jacobi2);

/// The generic step_occ kernels (see Operator): one thread per voxel, same
/// geometry, plane tables and zero-copy halo stores as dense_step_kernel.
///   identity: out(v, c) = in(v, c)                      (partition_test.cpp:189-191)
///   jacobi2:  out(v, c) = 0.5 in(v, c) + 0.5 (n ? sum / n : 0), sum over the
///             in-domain neighbours +x, -x, +y, -y in that order
///                                                      (partition_test.cpp:234-247)
/// The y neighbours are k +- 1 (halo groups at the slab faces) when the
/// partition axis is y, else the b +- 1 rows of the same plane.
template <int OP, int Q, class R, bool Exact, bool AOS, int AXIS>
__global__ void __launch_bounds__(kBlock) dense_operator_kernel(const __grid_constant__ StepArgs<Q, R> A) {
    using Ar = Arith<R, Exact>;
    const int a = blockIdx.x * kBlock + threadIdx.x;
    if (a >= A.na) return;
    const int b = blockIdx.y;
    const int k = A.k_first + int(blockIdx.z) * A.k_step;
    const int kg = A.kg0 + k;
    const int na = A.na, s = A.s;
    const int cross = b * na + a;
    const long long lin = (long long)(k + 1) * s + cross;
    const int gm = group_of(k - 1, A.n), g0 = group_of(k, A.n), gp = group_of(k + 1, A.n);
    constexpr long long VS = AOS ? Q : 1;
    R f[Q];
#pragma unroll
    for (int c = 0; c < Q; ++c) {
        const R v = ld_ro(A.in + A.plane[g0][c] + lin * VS);
        if constexpr (OP == kOpIdentity) {
            f[c] = v;
        } else {
            R sum = R(0);
            int cnt = 0;
            if (a + 1 < na) { sum = Ar::add(sum, ld_ro(A.in + A.plane[g0][c] + (lin + 1) * VS)); ++cnt; }
            if (a - 1 >= 0) { sum = Ar::add(sum, ld_ro(A.in + A.plane[g0][c] + (lin - 1) * VS)); ++cnt; }
            if constexpr (AXIS == 1) {
                if (kg + 1 < A.nk) { sum = Ar::add(sum, ld_ro(A.in + A.plane[gp][c] + (lin + s) * VS)); ++cnt; }
                if (kg - 1 >= 0) { sum = Ar::add(sum, ld_ro(A.in + A.plane[gm][c] + (lin - s) * VS)); ++cnt; }
            } else {
                if (b + 1 < A.nb) { sum = Ar::add(sum, ld_ro(A.in + A.plane[g0][c] + (lin + na) * VS)); ++cnt; }
                if (b - 1 >= 0) { sum = Ar::add(sum, ld_ro(A.in + A.plane[g0][c] + (lin - na) * VS)); ++cnt; }
            }
            const R mean = cnt ? sum / R(cnt) : R(0);
            f[c] = Ar::add(Ar::mul(R(0.5), v), Ar::mul(R(0.5), mean));
        }
    }
#pragma unroll
    for (int c = 0; c < Q; ++c) A.out[A.plane[g0][c] + lin * VS] = f[c];
    if (k == 0 && A.up_out) {
#pragma unroll
        for (int c = 0; c < Q; ++c)
            if ((A.up_mask >> c) & 1u) A.up_out[A.up_plane[c] + (long long)cross * VS] = f[c];
    }
    if (k == A.n - 1 && A.low_out) {
#pragma unroll
        for (int c = 0; c < Q; ++c)
            if ((A.low_mask >> c) & 1u) A.low_out[A.low_plane[c] + (long long)cross * VS] = f[c];
    }
    if (A.remote_fence && ((k == 0 && A.up_out) || (k == A.n - 1 && A.low_out))) __threadfence_system();
}

// ---- cross-GPU step flags ---------------------------------------------------------------

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

/// Blocks the stream until both neighbours have finished the shared layers of
/// step target-1 (RAW: our halos are filled; WAR: they no longer read the
/// halo slots we are about to overwrite).
/// Spin until both neighbours signalled step `target`. A neighbour that never
/// signals (its process died) must not wedge the GPU: after kHaloWaitNs the
/// kernel records the step in flags[2] and returns; check_errors() turns that
/// into an error on the host. Limit: VOXL_HALO_TIMEOUT_S (default 120 s).

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void wait_flags_kernel(unsigned* flags, int need_up, int need_low, unsigned target,
                                  unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    const unsigned long long t0 = global_ns();
    for (int w = 0; w < 2; ++w) {
        if (!(w == 0 ? need_up : need_low)) continue;
        while (ld_acquire_sys(flags + w) < target) {
            __nanosleep(64);
            if (global_ns() - t0 > timeout_ns) {
                atomicCAS(flags + 2, 0u, target + 1);  // keep the first stalled step
                return;
            }
        }
    }
}

__global__ void signal_flags_kernel(unsigned* up_slot, unsigned* low_slot, unsigned value) {
    if (threadIdx.x != 0) return;
    __threadfence_system();
    if (up_slot) st_release_sys(up_slot, value);
    if (low_slot) st_release_sys(low_slot, value);
}

// ---- canonical <-> layout -----------------------------------------------------------

template <int Q>
struct CanonArgs {
    long long plane[kGroupCount][Q];
    double shift[Q];  // w_i for shifted fp32 storage (g = f - w), 0 for fp64
    long long vs;
    int na, s, n;
    int k_lo, k_hi;   // local k range being moved
    int kg_stage0;    // global k of staging plane 0
    int kg0;          // partition's global offset
};

/// S = double: fp64 canonical staging, storage = R(f - shift). S = R (fp32
/// wire format): the host already applied the same fp64 subtraction and
/// rounding (HostPool conversion), so the kernel only permutes.
template <int Q, class R, bool ToDevice, class S = double>
__global__ void canon_kernel(R* buf, S* staging, const __grid_constant__ CanonArgs<Q> A) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long count = (long long)(A.k_hi - A.k_lo) * A.s;
    if (t >= count) return;
    const int k = A.k_lo + int(t / A.s);
    const int cross = int(t % A.s);
    const int g = group_of(k, A.n);
    const long long lin = (long long)(k + 1) * A.s + cross;
    const long long st = ((long long)(A.kg0 + k - A.kg_stage0) * A.s + cross) * Q;
    for (int c = 0; c < Q; ++c) {
        R* p = buf + A.plane[g][c] + lin * A.vs;
        if constexpr (std::is_same_v<S, double>) {
            if constexpr (ToDevice) *p = R(staging[st + c] - A.shift[c]);
            else staging[st + c] = double(*p) + A.shift[c];
        } else {
            if constexpr (ToDevice) *p = staging[st + c];
            else staging[st + c] = *p;
        }
    }
}

/// Uniform state over every voxel of the partition, halos included
/// (make_equilibrium_state lbm.cpp:72-83 / initial_canonical_state's rest case).
template <int Q, class R>
__global__ void fill_kernel(R* buf, const __grid_constant__ CanonArgs<Q> A, const __grid_constant__ StepArgs<Q, R> V) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long count = (long long)(A.n + 2) * A.s;
    if (t >= count) return;
    const int k = int(t / A.s) - 1;
    const int cross = int(t % A.s);
    const int g = group_of(k, A.n);
    const long long lin = (long long)(k + 1) * A.s + cross;
    for (int c = 0; c < Q; ++c) buf[A.plane[g][c] + lin * A.vs] = V.lid[c];
}

template <int Q, class R>
void launch_canon(unsigned blocks, int threads, R* buf, void* staging, bool wire32, bool to_device,
                  const CanonArgs<Q>& A, cudaStream_t st) {
    if (wire32) {
        if constexpr (sizeof(R) == 4) {
            if (to_device) canon_kernel<Q, R, true, R><<<blocks, threads, 0, st>>>(buf, static_cast<R*>(staging), A);
            else canon_kernel<Q, R, false, R><<<blocks, threads, 0, st>>>(buf, static_cast<R*>(staging), A);
        } else {
            throw std::logic_error("fp32 wire format on an fp64 engine");
        }
    } else {
        auto* sd = static_cast<double*>(staging);
        if (to_device) canon_kernel<Q, R, true><<<blocks, threads, 0, st>>>(buf, sd, A);
        else canon_kernel<Q, R, false><<<blocks, threads, 0, st>>>(buf, sd, A);
    }
    VOXL_CUDA(cudaGetLastError());
}

// ---- diagnostics (probe_field, lbm.cpp:116-138) ------------------------------------

constexpr int kProbeBlocks = 592;  // 4 x 148 SMs
constexpr int kProbeThreads = 256;

template <class L, class R>
__global__ void __launch_bounds__(kProbeThreads) probe_kernel(const R* buf, const __grid_constant__ CanonArgs<L::Q> A,
                                                            double* partial, unsigned long long* bad) {
    constexpr int Q = L::Q;
    const long long count = (long long)A.n * A.s;
    double mass = 0.0, vmax = 0.0;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < count;
         t += (long long)gridDim.x * blockDim.x) {
        const int k = int(t / A.s), cross = int(t % A.s);
        const int g = group_of(k, A.n);
        const long long lin = (long long)(k + 1) * A.s + cross;
        // all Q loads issued back to back, then the fp64 moments; |u|^2 with a
        // single division (max |u| = sqrt(max |u|^2): sqrt is monotone and
        // correctly rounded, applied once on the host)
        R raw[Q];
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            raw[i] = buf[A.plane[g][i] + lin * A.vs];
        });
        double r = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
        int bad_pop = -1;
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            const double fi = double(raw[i]) + A.shift[i];
            if (bad_pop < 0 && !(fabs(fi) <= 1e3)) bad_pop = i;
            mass += fi;
            r += fi;
            mx = acc_term<double, false, L::ex(i)>(mx, fi);
            my = acc_term<double, false, L::ey(i)>(my, fi);
            mz = acc_term<double, false, L::ez(i)>(mz, fi);
        });
        if (bad_pop >= 0 || !(r > 0.0)) {
            const unsigned long long canon = (unsigned long long)(A.kg0 + k) * A.s + cross;
            atomicMin(bad, (canon << 5) | (unsigned long long)(bad_pop < 0 ? kBadDensity : bad_pop));
        } else {
            vmax = fmax(vmax, (mx * mx + my * my + mz * mz) / (r * r));
        }
    }
    __shared__ double sm[kProbeThreads], sv[kProbeThreads];
    sm[threadIdx.x] = mass;
    sv[threadIdx.x] = vmax;
    __syncthreads();
    for (int w = kProbeThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            sm[threadIdx.x] += sm[threadIdx.x + w];
            sv[threadIdx.x] = fmax(sv[threadIdx.x], sv[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = sm[0];
        partial[2 * blockIdx.x + 1] = sv[0];
    }
}

/// Fixed-order reduction of n (mass, max) partials by one 256-thread block:
/// thread j sums the contiguous slice j, then a fixed pairwise tree. (A single
/// thread walking the partials serialises one L2 round trip per element:
/// ~0.35 ms for 592 partials.) Deterministic run to run.
__device__ __forceinline__ void block_reduce_partials(const double* partial, int n, double& m_out, double& v_out) {
    __shared__ double sm[256], sv[256];
    const int per = (n + 255) / 256;
    const int lo = threadIdx.x * per, hi = min(n, lo + per);
    double m = 0.0, v = 0.0;
    for (int i = lo; i < hi; ++i) {
        m += partial[2 * i];
        v = fmax(v, partial[2 * i + 1]);
    }
    sm[threadIdx.x] = m;
    sv[threadIdx.x] = v;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            sm[threadIdx.x] += sm[threadIdx.x + w];
            sv[threadIdx.x] = fmax(sv[threadIdx.x], sv[threadIdx.x + w]);
        }
        __syncthreads();
    }
    m_out = sm[0];
    v_out = sv[0];
}

__global__ void __launch_bounds__(256) probe_final_kernel(const double* partial, int n, double* out) {
    double m, v;
    block_reduce_partials(partial, n, m, v);
    if (threadIdx.x == 0) {
        out[0] += m;
        out[1] = fmax(out[1], v);
    }
}


// ---- launch plumbing ------------------------------------------------------------------

template <class L>
constexpr int axis_of() {
    return L::dim == 3 ? 2 : 1;
}

struct PartGeom {
    int na, nb, n, s, kg0, nk;
};

PartGeom geom_of(const Decomposition& d, int p) {
    PartGeom g{};
    const int axis = d.axis;
    const int other = axis == 2 ? 1 : 2;
    g.na = d.domain[0];
    g.nb = d.domain[other];
    g.n = d.thickness(p);
    g.s = g.na * g.nb;
    g.kg0 = d.slabs[p].first;
    g.nk = d.domain[axis];
    return g;
}

/// Per-(group, component) plane tables, the neighbours' halo targets of the
/// zero-copy stores, and the slab geometry of one step launch.
template <int Q, class R>
PartGeom fill_geometry(StepArgs<Q, R>& A, const Decomposition& d, const std::vector<LayoutMap>& maps, int p,
                       const void* in, void* out, void* up_out, void* low_out, int k_first, int k_step,
                       bool remote_fence) {
    const PartGeom g = geom_of(d, p);
    A.remote_fence = remote_fence;
    A.in = static_cast<const R*>(in);
    A.out = static_cast<R*>(out);
    for (int gr = 0; gr < kGroupCount; ++gr)
        for (int c = 0; c < Q; ++c) A.plane[gr][c] = maps[p].plane_offset(gr, c);
    const bool aos = maps[p].scheme() == LayoutScheme::AoS;
    const int up = d.upper_neighbor(p), low = d.lower_neighbor(p);
    A.up_out = static_cast<R*>(up_out);
    A.low_out = static_cast<R*>(low_out);
    A.up_mask = A.low_mask = 0;
    if (up >= 0 && up_out) {
        const LayoutMap& nm = maps[up];
        const std::vector<int>& comps = nm.transfer().down;
        for (int c = 0; c < Q; ++c) {
            const bool send = aos || std::find(comps.begin(), comps.end(), c) != comps.end();
            if (send) A.up_mask |= 1u << c;
            // neighbour's LowerHalo, k = n_up: lin = (n_up + 1) * s + cross
            A.up_plane[c] = nm.plane_offset(int(GroupTag::LowerHalo), c) +
                            (long long)(nm.shape()[d.axis] + 1) * g.s * nm.voxel_stride();
        }
    }
    if (low >= 0 && low_out) {
        const LayoutMap& nm = maps[low];
        const std::vector<int>& comps = nm.transfer().up;
        for (int c = 0; c < Q; ++c) {
            const bool send = aos || std::find(comps.begin(), comps.end(), c) != comps.end();
            if (send) A.low_mask |= 1u << c;
            A.low_plane[c] = nm.plane_offset(int(GroupTag::UpperHalo), c);  // k = -1: lin = cross
        }
    }
    A.na = g.na;
    A.nb = g.nb;
    A.n = g.n;
    A.s = g.s;
    A.k_first = k_first;
    A.k_step = k_step;
    A.kg0 = g.kg0;
    A.nk = g.nk;
    return g;
}

template <class L, class R, bool Exact>
struct DenseOps {
    static constexpr int Q = L::Q;
    static constexpr int AXIS = axis_of<L>();

    /// fp32 stores g = f - w (bgk_relax_shifted); fp64 parity mode stores f.
    static void fill_shift(double (&shift)[Q]) {
        for (int c = 0; c < Q; ++c) shift[c] = Exact ? 0.0 : L::w(c);
    }

    static void fill_planes(const LayoutMap& m, long long (&plane)[kGroupCount][Q]) {
        for (int g = 0; g < kGroupCount; ++g)
            for (int c = 0; c < Q; ++c) plane[g][c] = m.plane_offset(g, c);
    }

    static void launch_step(const DenseConfig& cfg, const Decomposition& d, const std::vector<LayoutMap>& maps,
                            int p, const void* in, void* out, void* up_out, void* low_out, bool wrap,
                            int step, int* error_flag, int k_first, int k_step, int k_count, cudaStream_t st,
                            bool remote_fence = false, DiagTarget* diag = nullptr, const int* step_base = nullptr) {
        if (k_count <= 0) return;
        StepArgs<Q, R> A{};
        A.step_base = step_base;
        const PartGeom g = fill_geometry(A, d, maps, p, in, out, up_out, low_out, k_first, k_step, remote_fence);
        const bool aos = maps[p].scheme() == LayoutScheme::AoS;
        const bool lid = cfg.scenario == Scenario::LidDrivenCavity;
        for (int i = 0; i < Q; ++i) {
            // (((2.0 * w_i) * 1.0) * 3.0) * eu, eu = (ex*u0 + ey*u1) + ez*u2 (lbm.hpp:66-69)
            const double eu = double(L::ex(i)) * cfg.velocity[0] + double(L::ey(i)) * cfg.velocity[1] +
                              double(L::ez(i)) * cfg.velocity[2];
            A.lid[i] = R(2.0 * L::w(i) * 1.0 * 3.0 * eu);
        }
        const double inv_tau = 1.0 / cfg.tau;
        if constexpr (Exact) {
            A.omega = R(inv_tau);
            A.keep = R(1.0 - inv_tau);
        } else {
            A.omega = R(inv_tau);
            A.keep = R(1.0) - R(inv_tau);
        }
        const bool periodic = cfg.scenario == Scenario::PeriodicBox;
        A.wall_a = !periodic;
        A.wall_b = !periodic && L::dim == 3;
        A.wall_k = !periodic;
        A.periodic_a = periodic;
        A.periodic_b = periodic && L::dim == 3;
        A.has_lid = lid;
        A.step = step;
        A.error_flag = error_flag;
        constexpr int OTHER = AXIS == 2 ? 1 : 2;
        const long long vs = maps[p].voxel_stride();
        A.uniform_groups = maps[p].scheme() != LayoutScheme::DisagSoA;
        const int gi = int(GroupTag::Interior);
        A.fast_base = A.plane[gi][0] * (long long)sizeof(R);
        for (int i = 0; i < Q; ++i) {
            const long long shift = -(long long)L::e(i, 0) - (long long)L::e(i, OTHER) * g.na -
                                    (long long)L::e(i, AXIS) * g.s;
            const long long rel = A.plane[gi][i] - A.plane[gi][0];
            A.fast_in_off[i] = (rel + vs * shift) * (long long)sizeof(R);
            A.fast_out_off[i] = rel * (long long)sizeof(R);
        }

        const dim3 grid((g.na + kBlock - 1) / kBlock, g.nb, k_count);
        A.diag_acc = diag ? diag->acc : nullptr;
        A.diag_bad = diag ? diag->bad : nullptr;
        using T = std::true_type;
        using F = std::false_type;
        if constexpr (std::is_same_v<R, float> && L::dim == 3) {
            // AoS fp32 3D without periodic wrap: the plane-tile kernel
            if (aos && !wrap && g.na >= 1) {
                constexpr int smem = AosTile<Q>::smem_bytes;
                auto launch = [&](auto kern) {
                    // opt in to the large dynamic shared memory (per kernel and device; a host-side call)
                    VOXL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                    int kb = k_first, zs = kAosChunk, chunk = kAosChunk, ke = k_first + k_count, zc;
                    if (k_step != 1 && k_count > 1) {  // the shared layers: one plane per CTA
                        zs = k_step;
                        chunk = 1;
                        ke = k_first + (k_count - 1) * k_step + 1;
                        zc = k_count;
                    } else {
                        zc = (k_count + kAosChunk - 1) / kAosChunk;
                    }
                    const dim3 tg((g.na + kAosTX - 1) / kAosTX, (g.nb + kAosTY - 1) / kAosTY, zc);
                    kern<<<tg, kAosThreads, smem, st>>>(A, kb, zs, chunk, ke);
                };
                if (diag) launch(dense_aos_tiled_kernel<L, true>);
                else launch(dense_aos_tiled_kernel<L, false>);
                VOXL_CUDA(cudaGetLastError());
                return;
            }
        }
        auto go = [&](auto aos_c, auto wrap_c, auto diag_c) {
            dense_step_kernel<L, R, Exact, decltype(aos_c)::value, AXIS, decltype(wrap_c)::value,
                              decltype(diag_c)::value><<<grid, kBlock, 0, st>>>(A);
        };
        auto with_diag = [&](auto a_c, auto w_c) { diag ? go(a_c, w_c, T{}) : go(a_c, w_c, F{}); };
        if (aos) wrap ? with_diag(T{}, T{}) : with_diag(T{}, F{});
        else wrap ? with_diag(F{}, T{}) : with_diag(F{}, F{});
        VOXL_CUDA(cudaGetLastError());
    }

    /// CTA count of one launch (diagnostics partial slots).
    static long long launch_ctas(const Decomposition& d, int p, int k_count) {
        const PartGeom g = geom_of(d, p);
        return (long long)((g.na + kBlock - 1) / kBlock) * g.nb * k_count;
    }

    static void host_shift(double* shift) {
        double sh[Q];
        fill_shift(sh);
        for (int c = 0; c < Q; ++c) shift[c] = sh[c];
    }

    static void canon(const Decomposition& d, const LayoutMap& m, int p, void* buf, void* staging, bool wire32,
                      int k_lo, int k_hi, int kg_stage0, bool to_device, cudaStream_t st) {
        CanonArgs<Q> A{};
        fill_planes(m, A.plane);
        fill_shift(A.shift);
        const PartGeom g = geom_of(d, p);
        A.vs = m.voxel_stride();
        A.na = g.na;
        A.s = g.s;
        A.n = g.n;
        A.k_lo = k_lo;
        A.k_hi = k_hi;
        A.kg_stage0 = kg_stage0;
        A.kg0 = g.kg0;
        const long long count = (long long)(k_hi - k_lo) * g.s;
        if (count <= 0) return;
        const int threads = 256;
        const unsigned blocks = unsigned((count + threads - 1) / threads);
        launch_canon<Q, R>(blocks, threads, static_cast<R*>(buf), staging, wire32, to_device, A, st);
    }

    static void fill(const Decomposition& d, const LayoutMap& m, int p, void* buf, const double* feq,
                     cudaStream_t st) {
        CanonArgs<Q> A{};
        fill_planes(m, A.plane);
        fill_shift(A.shift);
        const PartGeom g = geom_of(d, p);
        A.vs = m.voxel_stride();
        A.na = g.na;
        A.s = g.s;
        A.n = g.n;
        StepArgs<Q, R> V{};
        for (int c = 0; c < Q; ++c) V.lid[c] = R(feq[c] - A.shift[c]);
        const long long count = (long long)(g.n + 2) * g.s;
        fill_kernel<Q, R><<<unsigned((count + 255) / 256), 256, 0, st>>>(static_cast<R*>(buf), A, V);
        VOXL_CUDA(cudaGetLastError());
    }

    static void probe(const Decomposition& d, const LayoutMap& m, int p, const void* buf, double* partial,
                      unsigned long long* bad, double* out, cudaStream_t st) {
        CanonArgs<Q> A{};
        fill_planes(m, A.plane);
        fill_shift(A.shift);
        const PartGeom g = geom_of(d, p);
        A.vs = m.voxel_stride();
        A.na = g.na;
        A.s = g.s;
        A.n = g.n;
        A.kg0 = g.kg0;
        probe_kernel<L, R><<<kProbeBlocks, kProbeThreads, 0, st>>>(static_cast<const R*>(buf), A, partial, bad);
        probe_final_kernel<<<1, 256, 0, st>>>(partial, kProbeBlocks, out);
        VOXL_CUDA(cudaGetLastError());
    }
};

/// Launch plumbing of the generic operators (same interface as DenseOps).
/// Values are stored unshifted in both precisions.
template <int OP, int Q, class R, bool Exact>
struct OperatorOps {
    static void launch_step(const DenseConfig&, const Decomposition& d, const std::vector<LayoutMap>& maps, int p,
                            const void* in, void* out, void* up_out, void* low_out, bool, int, int*, int k_first,
                            int k_step, int k_count, cudaStream_t st, bool remote_fence = false,
                            DiagTarget* diag = nullptr, const int* = nullptr) {
        if (diag) throw std::invalid_argument("probe_field requires the lbm operator");
        if (k_count <= 0) return;
        StepArgs<Q, R> A{};
        const PartGeom g = fill_geometry(A, d, maps, p, in, out, up_out, low_out, k_first, k_step, remote_fence);
        const dim3 grid((g.na + kBlock - 1) / kBlock, g.nb, k_count);
        auto go = [&](auto aos_c, auto axis_c) {
            dense_operator_kernel<OP, Q, R, Exact, decltype(aos_c)::value, decltype(axis_c)::value>
                <<<grid, kBlock, 0, st>>>(A);
        };
        using T = std::true_type;
        using F = std::false_type;
        using Y = std::integral_constant<int, 1>;
        using Z = std::integral_constant<int, 2>;
        const bool aos = maps[p].scheme() == LayoutScheme::AoS;
        if (d.axis == 1) aos ? go(T{}, Y{}) : go(F{}, Y{});
        else aos ? go(T{}, Z{}) : go(F{}, Z{});
        VOXL_CUDA(cudaGetLastError());
    }

    static long long launch_ctas(const Decomposition& d, int p, int k_count) {
        const PartGeom g = geom_of(d, p);
        return (long long)((g.na + kBlock - 1) / kBlock) * g.nb * k_count;
    }

    static void host_shift(double* shift) {
        for (int c = 0; c < Q; ++c) shift[c] = 0.0;
    }

    static void canon(const Decomposition& d, const LayoutMap& m, int p, void* buf, void* staging, bool wire32,
                      int k_lo, int k_hi, int kg_stage0, bool to_device, cudaStream_t st) {
        CanonArgs<Q> A{};
        for (int gr = 0; gr < kGroupCount; ++gr)
            for (int c = 0; c < Q; ++c) A.plane[gr][c] = m.plane_offset(gr, c);
        const PartGeom g = geom_of(d, p);
        A.vs = m.voxel_stride();
        A.na = g.na;
        A.s = g.s;
        A.n = g.n;
        A.k_lo = k_lo;
        A.k_hi = k_hi;
        A.kg_stage0 = kg_stage0;
        A.kg0 = g.kg0;
        const long long count = (long long)(k_hi - k_lo) * g.s;
        if (count <= 0) return;
        const unsigned blocks = unsigned((count + 255) / 256);
        launch_canon<Q, R>(blocks, 256, static_cast<R*>(buf), staging, wire32, to_device, A, st);
    }

    static void fill(const Decomposition&, const LayoutMap&, int, void*, const double*, cudaStream_t) {
        throw std::invalid_argument("set_equilibrium requires the lbm operator");
    }

    static void probe(const Decomposition&, const LayoutMap&, int, const void*, double*, unsigned long long*, double*,
                      cudaStream_t) {
        throw std::invalid_argument("probe_field requires the lbm operator");
    }
};

template <class F>
void dispatch(const DenseConfig& cfg, F&& f) {
    const Precision prec = cfg.precision;
    auto by_prec = [&](auto lat) {
        using L = decltype(lat);
        constexpr int Q = L::Q;
        switch (cfg.op) {
            case Operator::Lbm:
                if (prec == Precision::F64) f(DenseOps<L, double, true>{});
                else f(DenseOps<L, float, false>{});
                break;
            case Operator::Identity:
                if (prec == Precision::F64) f(OperatorOps<kOpIdentity, Q, double, true>{});
                else f(OperatorOps<kOpIdentity, Q, float, false>{});
                break;
            default: throw std::invalid_argument("unknown operator");
        }
    };
    if (cfg.op == Operator::Jacobi2) {
        if (prec == Precision::F64) f(OperatorOps<kOpJacobi2, 2, double, true>{});
        else f(OperatorOps<kOpJacobi2, 2, float, false>{});
        return;
    }
    switch (cfg.lattice) {
        case kD2Q9: by_prec(D2Q9{}); break;
        case kD3Q19: by_prec(D3Q19{}); break;
        case kD3Q27: by_prec(D3Q27{}); break;
        default: throw std::invalid_argument("unknown lattice kind");
    }
}

} // namespace

OperatorShape operator_shape(const DenseConfig& cfg) {
    OperatorShape o;
    if (cfg.op == Operator::Jacobi2) {
        o.q = 2;
        o.axis = cfg.domain[2] == 1 ? 1 : 2;
        o.transfer = TransferSets::all(2);
        return o;
    }
    if (cfg.op != Operator::Lbm && cfg.op != Operator::Identity) throw std::invalid_argument("unknown operator");
    if (cfg.lattice < 0 || cfg.lattice > 2) throw std::invalid_argument("unknown lattice kind");
    const LatticeTable t = make_lattice(cfg.lattice);
    o.q = t.q;
    o.axis = t.dim == 2 ? 1 : 2;
    o.transfer = TransferSets::for_lattice(cfg.lattice, o.axis);
    return o;
}

namespace {

} // namespace

// ---- engine ------------------------------------------------------------------------

namespace {

/// Makes `device` current for a scope (multi-device engines launch on the
/// partition's device).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int device) {
        VOXL_CUDA(cudaGetDevice(&prev));
        if (device != prev) VOXL_CUDA(cudaSetDevice(device));
    }
    ~DeviceGuard() {
        int now = -1;
        if (cudaGetDevice(&now) == cudaSuccess && now != prev) cudaSetDevice(prev);
    }
};

__global__ void advance_step_kernel(int* step_base, int n) { *step_base += n; }

} // namespace

/// NCCL transport of the halo spans for the in-process multi-device engine
/// (halo mode Nccl): one communicator per partition device from
/// ncclCommInitAll, every step's sends and receives in one group on the
/// partitions' shared-layer streams. libnccl is opened at run time (dlopen),
/// so the library carries no link-time NCCL dependency and shares whichever
/// libnccl.so.2 the process already loaded.
struct DenseEngine::NcclHalo {
    void* lib = nullptr;
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::vector<ncclComm_t> comms;

    void check(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            throw CudaError(std::string("nccl ") + what + ": " + (error_string ? error_string(r) : "error"));
    }
    explicit NcclHalo(const std::vector<int>& devices) {
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) throw std::runtime_error(std::string("nccl halo mode: cannot load libnccl.so.2: ") + dlerror());
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
            if (!fn) throw std::runtime_error(std::string("nccl halo mode: missing symbol ") + name);
        };
        sym(init_all, "ncclCommInitAll");
        sym(destroy, "ncclCommDestroy");
        sym(group_start, "ncclGroupStart");
        sym(group_end, "ncclGroupEnd");
        sym(send, "ncclSend");
        sym(recv, "ncclRecv");
        sym(error_string, "ncclGetErrorString");
        comms.resize(devices.size());
        check(init_all(comms.data(), int(devices.size()), devices.data()), "ncclCommInitAll");
    }
    ~NcclHalo() {
        for (ncclComm_t c : comms)
            if (c) destroy(c);
    }
};

DenseEngine::DenseEngine(const DenseConfig& cfg) : cfg_(cfg), io_(std::make_unique<CanonPipe>()) {
    static_assert(kBadDensity == 31, "bad-word population field is 5 bits");
    const OperatorShape shape = operator_shape(cfg_);
    q_ = shape.q;
    axis_ = shape.axis;
    if (cfg_.op != Operator::Jacobi2) {
        const LatticeTable t = make_lattice(cfg_.lattice);
        if (t.dim == 2 && cfg_.domain[2] != 1)
            throw std::invalid_argument("invalid configuration: D2Q9 requires nz == 1; ");
        if (t.dim == 3 && cfg_.domain[2] < 2)
            throw std::invalid_argument("invalid configuration: 3D lattices require nz >= 2; ");
    }
    if (cfg_.op == Operator::Lbm && !(cfg_.tau > 0.5))
        throw std::invalid_argument("invalid configuration: tau must be > 0.5; ");
    if (cfg_.domain[0] < 2 || cfg_.domain[1] < 2)
        throw std::invalid_argument("invalid configuration: domain extents must be >= 2; ");
    if (cfg_.scenario == Scenario::FlowOverObstacle)
        throw std::invalid_argument("dense engine: flow_over_obstacle runs on the block-sparse engine");
    esize_ = cfg_.precision == Precision::F64 ? 8 : 4;
    decomp_ = decompose(cfg_.domain, cfg_.partitions, axis_, cfg_.scenario == Scenario::PeriodicBox);
    if (cfg_.local_partitions < 0) {
        cfg_.first_partition = 0;
        cfg_.local_partitions = cfg_.partitions;
    }
    if (cfg_.first_partition < 0 || cfg_.first_partition + cfg_.local_partitions > cfg_.partitions)
        throw std::invalid_argument("dense engine: bad local partition range");
    int primary = 0;
    VOXL_CUDA(cudaGetDevice(&primary));
    if (!cfg_.devices.empty()) {
        if (cfg_.local_partitions != cfg_.partitions)
            throw std::invalid_argument("dense engine: devices[] places every partition of a single-process engine");
        if (int(cfg_.devices.size()) != cfg_.partitions)
            throw std::invalid_argument("dense engine: devices[] must name one device per partition");
        int count = 0;
        VOXL_CUDA(cudaGetDeviceCount(&count));
        for (int d : cfg_.devices)
            if (d < 0 || d >= count)
                throw std::invalid_argument("dense engine: device " + std::to_string(d) + " does not exist (" +
                                            std::to_string(count) + " visible)");
        if (cfg_.graph_steps < 0 || cfg_.graph_steps % 2)
            throw std::invalid_argument("dense engine: graph_steps must be even and >= 0");
        multi_ = true;
    }
    if (cfg_.halo == HaloMode::Nccl && !multi_)
        throw std::invalid_argument("nccl halo mode needs a multi-device engine (devices[])");
    for (int p = 0; p < cfg_.partitions; ++p) {
        std::array<int, 3> owned = cfg_.domain;
        owned[axis_] = decomp_.thickness(p);
        maps_.push_back(LayoutMap::build(cfg_.layout, owned, q_, axis_, shape.transfer));
        links_.emplace_back(decomp_.upper_neighbor(p), decomp_.lower_neighbor(p));
    }
    parts_.resize(cfg_.partitions);
    VOXL_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    for (int p = 0; p < cfg_.partitions; ++p) {
        parts_[p].device = multi_ ? cfg_.devices[p] : primary;
        if (!local(p)) continue;
        const std::size_t bytes = buffer_bytes(p);
        DeviceGuard g(parts_[p].device);
        for (int w = 0; w < 2; ++w) {
            VOXL_CUDA(cudaMalloc(&parts_[p].buf[w], bytes));
            VOXL_CUDA(cudaMemset(parts_[p].buf[w], 0, bytes));
        }
        parts_[p].owned = true;
    }
    VOXL_CUDA(cudaMalloc(&error_flag_, sizeof(int)));
    const int big = INT_MAX;
    VOXL_CUDA(cudaMemcpyAsync(error_flag_, &big, sizeof(int), cudaMemcpyHostToDevice, stream_));
    diag_scratch_len_ = 2 * kProbeBlocks + 4;
    VOXL_CUDA(cudaMalloc(&diag_scratch_, diag_scratch_len_ * sizeof(double)));
    VOXL_CUDA(cudaMallocHost(&diag_row_host_, 4 * sizeof(double)));
    if (multi_) setup_multi();
    VOXL_CUDA(cudaStreamSynchronize(stream_));
}

int DenseEngine::dev_index(int device) const {
    for (std::size_t i = 0; i < dx_.size(); ++i)
        if (dx_[i].device == device) return int(i);
    throw std::logic_error("dense engine: device not registered");
}

void DenseEngine::setup_multi() {
    int primary = 0;
    VOXL_CUDA(cudaGetDevice(&primary));
    std::vector<int> devs{primary};
    for (int d : cfg_.devices)
        if (std::find(devs.begin(), devs.end(), d) == devs.end()) devs.push_back(d);
    // Peer access between every pair of engine devices: the shared-layer
    // kernels store into the neighbours' halos, the canonical I/O and probe
    // kernels on the engine stream read every partition, and a failing voxel
    // sets the engine's error flag (one word on the primary device).
    for (int a : devs)
        for (int b : devs) {
            if (a == b) continue;
            int ok = 0;
            VOXL_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
            if (!ok)
                throw std::runtime_error("dense engine: device " + std::to_string(a) + " cannot access device " +
                                         std::to_string(b) + " (no peer path)");
            DeviceGuard g(a);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else VOXL_CUDA(e);
        }
    dx_.resize(devs.size());
    for (std::size_t i = 0; i < devs.size(); ++i) {
        DevExec& d = dx_[i];
        d.device = devs[i];
        DeviceGuard g(d.device);
        if (i == 0) d.aux = stream_;
        else VOXL_CUDA(cudaStreamCreateWithFlags(&d.aux, cudaStreamNonBlocking));
        VOXL_CUDA(cudaEventCreateWithFlags(&d.ev, cudaEventDisableTiming));
    }
    px_.resize(std::size_t(cfg_.partitions));
    for (int p = 0; p < cfg_.partitions; ++p) {
        PartExec& x = px_[std::size_t(p)];
        DeviceGuard g(parts_[p].device);
        int lo = 0, hi = 0;
        VOXL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        VOXL_CUDA(cudaStreamCreateWithFlags(&x.interior, cudaStreamNonBlocking));
        VOXL_CUDA(cudaStreamCreateWithPriority(&x.shared, cudaStreamNonBlocking, hi));
        for (int i = 0; i < 2; ++i) {
            VOXL_CUDA(cudaEventCreateWithFlags(&x.ev_i[i], cudaEventDisableTiming));
            VOXL_CUDA(cudaEventCreateWithFlags(&x.ev_s[i], cudaEventDisableTiming));
        }
    }
    VOXL_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    VOXL_CUDA(cudaMalloc(&step_base_, sizeof(int)));
    VOXL_CUDA(cudaMemset(step_base_, 0, sizeof(int)));
    if (cfg_.halo == HaloMode::Nccl) {
        std::vector<int> sorted = cfg_.devices;
        std::sort(sorted.begin(), sorted.end());
        if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
            throw std::invalid_argument("nccl halo mode: one distinct device per partition (ncclCommInitAll)");
        nccl_ = std::make_unique<NcclHalo>(cfg_.devices);
    }
}

DenseEngine::~DenseEngine() {
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto& x : px_) {
        cudaStreamSynchronize(x.interior);
        cudaStreamSynchronize(x.shared);
    }
    for (auto& d : dx_)
        if (d.aux) cudaStreamSynchronize(d.aux);
    nccl_.reset();
    for (auto& g : graph_)
        if (g) cudaGraphExecDestroy(g);
    for (auto& x : px_) {
        cudaStreamDestroy(x.interior);
        cudaStreamDestroy(x.shared);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(x.ev_i[i]);
            cudaEventDestroy(x.ev_s[i]);
        }
    }
    for (std::size_t i = 0; i < dx_.size(); ++i) {
        dx_[i].ring.reset();
        cudaEventDestroy(dx_[i].ev);
        if (i > 0) cudaStreamDestroy(dx_[i].aux);
    }
    if (step_base_) cudaFree(step_base_);
    for (auto& p : parts_)
        if (p.owned)
            for (void* b : p.buf) cudaFree(b);
    cudaFree(error_flag_);
    cudaFree(diag_scratch_);
    if (diag_row_host_) cudaFreeHost(diag_row_host_);
    if (flags_ && distributed_) cudaFree(flags_);
    if (shared_stream_) {
        cudaStreamSynchronize(shared_stream_);
        for (int i = 0; i < 2; ++i) {
            cudaEventDestroy(ev_shared_[i]);
            cudaEventDestroy(ev_interior_[i]);
        }
        cudaEventDestroy(ev_join_);
        cudaStreamDestroy(shared_stream_);
    }
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (stream_) cudaStreamDestroy(stream_);
}

std::int64_t DenseEngine::owned_voxels() const {
    std::int64_t v = 0;
    const std::int64_t s = maps_[0].cross_section();
    for (int p = 0; p < cfg_.partitions; ++p)
        if (local(p)) v += std::int64_t(decomp_.thickness(p)) * s;
    return v;
}

std::size_t DenseEngine::buffer_bytes(int p) const { return std::size_t(maps_[p].total_len()) * esize_; }

void* DenseEngine::buffer(int p, int which) const { return parts_[p].buf[which == 0 ? cur_ : cur_ ^ 1]; }

void DenseEngine::attach_peer(int p, void* b0, void* b1) {
    if (p < 0 || p >= cfg_.partitions) throw std::invalid_argument("attach_peer: no such partition");
    if (local(p)) throw std::invalid_argument("attach_peer: partition is owned locally");
    bool neighbour = false;
    for (int q = 0; q < cfg_.partitions; ++q)
        if (local(q) && (links_[q].first == p || links_[q].second == p)) neighbour = true;
    if (!neighbour) throw std::invalid_argument("attach_peer: partition is not a neighbour of an owned partition");
    if (!b0 || !b1) throw std::invalid_argument("attach_peer: null buffer");
    parts_[p].buf[0] = b0;
    parts_[p].buf[1] = b1;
}

void DenseEngine::scatter_gather(double* host, int k_begin, int k_end, bool to_device, unsigned long long* digest) {
    join_streams();
    const std::int64_t s = maps_[0].cross_section();
    // rows = canonical planes; fp32 engines use the fp32 wire format (canon_io.cuh)
    const bool wire32 = esize_ == 4 && host != nullptr;
    double shift[27] = {};
    if (wire32) dispatch(cfg_, [&](auto ops) { decltype(ops)::host_shift(shift); });
    auto layout = [&](long long r0, long long r1, void* slot, bool w32) {
        const int k0 = k_begin + int(r0), k1 = k_begin + int(r1);
        for (int p = 0; p < cfg_.partitions; ++p) {
            if (!local(p)) continue;
            const int lo = std::max(k0, decomp_.slabs[p].first), hi = std::min(k1, decomp_.slabs[p].second);
            if (lo >= hi) continue;
            dispatch(cfg_, [&](auto ops) {
                decltype(ops)::canon(decomp_, maps_[p], p, parts_[p].buf[cur_], slot, w32,
                                     lo - decomp_.slabs[p].first, hi - decomp_.slabs[p].first, k0, to_device,
                                     stream_);
            });
        }
    };
    auto consume = [&](long long r0, long long r1, void* slot) {
        digest_accumulate(static_cast<const double*>(slot), (r1 - r0) * s * q_, (k_begin + r0) * s * q_, digest,
                          stream_);
    };
    io_->run(host, k_end - k_begin, s, q_, to_device, wire32, shift, stream_, layout, consume, digest != nullptr);
}

void DenseEngine::check_plane_range(const char* who, int k_begin, int k_end) const {
    int lo = INT_MAX, hi = INT_MIN;
    for (int p = 0; p < cfg_.partitions; ++p)
        if (local(p)) {
            lo = std::min(lo, decomp_.slabs[p].first);
            hi = std::max(hi, decomp_.slabs[p].second);
        }
    if (!(lo <= k_begin && k_begin <= k_end && k_end <= hi))
        throw std::out_of_range(std::string(who) + ": planes [" + std::to_string(k_begin) + ", " +
                                std::to_string(k_end) + ") outside the owned slabs [" + std::to_string(lo) + ", " +
                                std::to_string(hi) + ")");
}

void DenseEngine::set_canonical_planes(const double* host, int k_begin, int k_end) {
    check_plane_range("set_canonical_planes", k_begin, k_end);
    scatter_gather(const_cast<double*>(host), k_begin, k_end, true);
}

void DenseEngine::get_canonical_planes(double* host, int k_begin, int k_end) {
    check_plane_range("get_canonical_planes", k_begin, k_end);
    scatter_gather(host, k_begin, k_end, false);
}

void DenseEngine::set_canonical(const double* host) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int p = 0; p < cfg_.partitions; ++p)
        if (local(p)) {
            lo = std::min(lo, decomp_.slabs[p].first);
            hi = std::max(hi, decomp_.slabs[p].second);
        }
    const std::int64_t s = maps_[0].cross_section();
    scatter_gather(const_cast<double*>(host) + std::size_t(lo) * s * q_, lo, hi, true);
    // fill_canonical leaves halos stale; the first step_occ's halo_update
    // refreshes them. Do the same refresh here for the single-process engine
    // (multi-process engines refresh through their shared-layer stores).
    if (cfg_.local_partitions == cfg_.partitions) halo_copy(0);
}

void DenseEngine::digest(unsigned long long out[2]) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int p = 0; p < cfg_.partitions; ++p)
        if (local(p)) {
            lo = std::min(lo, decomp_.slabs[p].first);
            hi = std::max(hi, decomp_.slabs[p].second);
        }
    unsigned long long* acc = nullptr;
    VOXL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&acc), 2 * sizeof(unsigned long long), stream_));
    VOXL_CUDA(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), stream_));
    scatter_gather(nullptr, lo, hi, false, acc);
    VOXL_CUDA(cudaMemcpyAsync(out, acc, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaFreeAsync(acc, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
}

void DenseEngine::set_equilibrium(double rho, const double u[3]) {
    // equilibrium (lattice.cpp:104-113) evaluated on the host in the reference's
    // double op order, then broadcast to every voxel of both parities.
    if (cfg_.op != Operator::Lbm) throw std::invalid_argument("set_equilibrium requires the lbm operator");
    const LatticeTable t = make_lattice(cfg_.lattice);
    double feq[27];
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int i = 0; i < t.q; ++i) {
        const double eu = double(t.e[i][0]) * u[0] + double(t.e[i][1]) * u[1] + double(t.e[i][2]) * u[2];
        const double w = double(t.wnum[i]) / double(t.wden[i]);
        feq[i] = w * rho * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * uu);
    }
    for (int p = 0; p < cfg_.partitions; ++p) {
        if (!local(p)) continue;
        for (int w = 0; w < 2; ++w)
            dispatch(cfg_, [&](auto ops) {
                decltype(ops)::fill(decomp_, maps_[p], p, parts_[p].buf[w], feq, stream_);
            });
    }
    VOXL_CUDA(cudaStreamSynchronize(stream_));
}

void DenseEngine::get_canonical(double* host) {
    int lo = INT_MAX, hi = INT_MIN;
    for (int p = 0; p < cfg_.partitions; ++p)
        if (local(p)) {
            lo = std::min(lo, decomp_.slabs[p].first);
            hi = std::max(hi, decomp_.slabs[p].second);
        }
    const std::int64_t s = maps_[0].cross_section();
    scatter_gather(host + std::size_t(lo) * s * q_, lo, hi, false);
}

void DenseEngine::halo_copy(int which) {
    // halo_update (partition.cpp:163-206): one cudaMemcpyAsync per contiguous
    // span, source = shared slab of p, destination = neighbour's halo slab
    // (peer copies when the partitions live on different devices).
    check_links();
    const int par = which == 0 ? cur_ : cur_ ^ 1;
    for (const auto& r : ledger_records(0)) {
        if (!parts_[r.src].buf[par] || !parts_[r.dst].buf[par]) continue;
        char* dst = static_cast<char*>(parts_[r.dst].buf[par]) + r.dst_span.base * esize_;
        const char* src = static_cast<const char*>(parts_[r.src].buf[par]) + r.src_span.base * esize_;
        VOXL_CUDA(cudaMemcpyAsync(dst, src, std::size_t(r.elements) * esize_, cudaMemcpyDefault, stream_));
    }
}

void DenseEngine::set_neighbor_links(int p, int upper, int lower) {
    if (p < 0 || p >= cfg_.partitions) throw std::out_of_range("set_neighbor_links: no such partition");
    links_[std::size_t(p)] = {upper, lower};
}

void DenseEngine::check_links() const {
    // halo_update's symmetry test (partition.cpp:165-171), run before every
    // batch of steps and every halo refresh.
    const int P = cfg_.partitions;
    for (int p = 0; p < P; ++p) {
        const auto [up, low] = links_[std::size_t(p)];
        if (up >= P || low >= P) throw std::runtime_error("halo_update: asymmetric neighbor links");
        if (up >= 0 && links_[std::size_t(up)].second != p)
            throw std::runtime_error("halo_update: asymmetric neighbor links");
        if (low >= 0 && links_[std::size_t(low)].first != p)
            throw std::runtime_error("halo_update: asymmetric neighbor links");
        // the plane tables address the decomposition's neighbours: a symmetric
        // re-wiring to any other partition is a span-structure change
        if ((up >= 0 && up != decomp_.upper_neighbor(p)) || (low >= 0 && low != decomp_.lower_neighbor(p)))
            throw std::runtime_error("halo_update: span structure mismatch");
    }
}

void DenseEngine::enable_distributed() {
    if (multi_) throw std::invalid_argument("enable_distributed: a multi-device engine owns every partition");
    if (!shared_stream_) {
        int lo = 0, hi = 0;
        VOXL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        VOXL_CUDA(cudaStreamCreateWithPriority(&shared_stream_, cudaStreamNonBlocking, hi));
        for (int i = 0; i < 2; ++i) {
            VOXL_CUDA(cudaEventCreateWithFlags(&ev_shared_[i], cudaEventDisableTiming));
            VOXL_CUDA(cudaEventCreateWithFlags(&ev_interior_[i], cudaEventDisableTiming));
        }
        VOXL_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
        VOXL_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    }
    if (const char* e = std::getenv("VOXL_HALO_TIMEOUT_S")) {
        const double sec = std::atof(e);
        if (sec > 0) halo_timeout_ns_ = (unsigned long long)(sec * 1e9);
    }
    if (!flags_) {
        VOXL_CUDA(cudaMalloc(&flags_, 4 * sizeof(std::uint32_t)));
        VOXL_CUDA(cudaMemset(flags_, 0, 4 * sizeof(std::uint32_t)));
    }
    distributed_ = true;
}

void DenseEngine::attach_flags(std::uint32_t* up, std::uint32_t* low) {
    remote_flag_up_ = up;
    remote_flag_low_ = low;
}

void DenseEngine::halo_push() {
    join_streams();
    // Our shared slabs -> neighbours' halos of the current parity (peer copies).
    const auto recs = halo_records(decomp_, maps_, 0);
    for (const auto& r : recs) {
        if (!local(r.src) || !parts_[r.dst].buf[cur_]) continue;
        char* dst = static_cast<char*>(parts_[r.dst].buf[cur_]) + r.dst_span.base * esize_;
        const char* src = static_cast<const char*>(parts_[r.src].buf[cur_]) + r.src_span.base * esize_;
        VOXL_CUDA(cudaMemcpyAsync(dst, src, std::size_t(r.elements) * esize_, cudaMemcpyDefault, stream_));
    }
    VOXL_CUDA(cudaStreamSynchronize(stream_));
}

void DenseEngine::launch_step_distributed(DiagTarget* diag) {
    // One owned partition p; neighbours live in other processes / devices.
    // Per step: wait(neighbour flags >= t) -> shared layers (k = 0, n-1) with
    // peer halo stores -> signal(t + 1) -> interior (k = 1 .. n-2). The interior
    // kernel never touches a halo, so it overlaps the neighbours' exchange.
    //
    // Two streams (OCC, paper Fig. 4c): the interior kernel runs on stream_
    // (I) and overlaps the high-priority shared-layer stream (S) that waits for
    // the neighbours, stores the crossing populations into their halos and
    // signals them. Cross-stream order, per step t:
    //   I: after shared(t-1) [RAW on planes 0/n-1, WAR on planes 1/n-2] -> interior(t)
    //   S: after interior(t-1) [RAW on planes 1/n-2, WAR on planes 0/n-1]
    //      -> wait(flags >= t) -> shared(t) -> signal(t+1)
    // Parity-alternating events keep "the previous step's" record addressable.
    const int p = cfg_.first_partition;
    const bool wrap = cfg_.scenario == Scenario::PeriodicBox;
    const bool zero_copy = cfg_.halo == HaloMode::ZeroCopy;
    const int in = cur_, out = cur_ ^ 1;
    const int up = links_[std::size_t(p)].first, low = links_[std::size_t(p)].second;
    const unsigned t = unsigned(steps_done_);
    const int par = int(t & 1u), prev = par ^ 1;
    if (!occ_ready_) {
        for (int i = 0; i < 2; ++i) {
            VOXL_CUDA(cudaEventRecord(ev_shared_[i], stream_));
            VOXL_CUDA(cudaEventRecord(ev_interior_[i], stream_));
        }
        occ_ready_ = true;
    }
    const int n = decomp_.thickness(p);
    // I: interior(t)
    VOXL_CUDA(cudaStreamWaitEvent(stream_, ev_shared_[prev], 0));
    trace_.phase(steps_done_, 1, "interior", p, cur_device(), "interior", stream_, [&] {
        dispatch(cfg_, [&](auto ops) {
            using Ops = decltype(ops);
            Ops::launch_step(cfg_, decomp_, maps_, p, parts_[p].buf[in], parts_[p].buf[out], nullptr, nullptr, wrap,
                             steps_done_, error_flag_, 1, 1, n - 2, stream_, false, diag);
        });
    });
    VOXL_CUDA(cudaEventRecord(ev_interior_[par], stream_));
    // S: wait -> shared(t) -> signal
    VOXL_CUDA(cudaStreamWaitEvent(shared_stream_, ev_interior_[prev], 0));
    if (zero_copy) {
        wait_flags_kernel<<<1, 32, 0, shared_stream_>>>(flags_, up >= 0, low >= 0, t, halo_timeout_ns_);
        VOXL_CUDA(cudaGetLastError());
    }
    void* up_out = (zero_copy && up >= 0) ? parts_[up].buf[out] : nullptr;
    void* low_out = (zero_copy && low >= 0) ? parts_[low].buf[out] : nullptr;
    trace_.phase(steps_done_, 2, "shared", p, cur_device(), "shared", shared_stream_, [&] {
        dispatch(cfg_, [&](auto ops) {
            using Ops = decltype(ops);
            Ops::launch_step(cfg_, decomp_, maps_, p, parts_[p].buf[in], parts_[p].buf[out], up_out, low_out, wrap,
                             steps_done_, error_flag_, 0, n - 1, 2, shared_stream_, true, diag);
        });
    });
    if (zero_copy) {
        signal_flags_kernel<<<1, 32, 0, shared_stream_>>>(remote_flag_up_, remote_flag_low_, t + 1);
        VOXL_CUDA(cudaGetLastError());
    }
    VOXL_CUDA(cudaEventRecord(ev_shared_[par], shared_stream_));
    cur_ = out;
    ++steps_done_;
    // Diagnostics reductions need the whole step: join S into I. The
    // copy-mode exchange is issued on S by the caller (after shared(t), next
    // to interior(t)); shared(t+1) follows it in S's order, and nothing on I
    // touches the halo planes or the shared layers it sends.
    if (diag) join_streams();
}

void DenseEngine::join_streams() {
    if (!shared_stream_) return;
    VOXL_CUDA(cudaEventRecord(ev_join_, shared_stream_));
    VOXL_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
}

void DenseEngine::launch_step(DiagTarget* diag) {
    if (distributed_) {
        launch_step_distributed(diag);
        return;
    }
    const bool wrap = cfg_.scenario == Scenario::PeriodicBox;
    const bool zero_copy = cfg_.halo == HaloMode::ZeroCopy;
    const int in = cur_, out = cur_ ^ 1;
    for (int p = 0; p < cfg_.partitions; ++p) {
        if (!local(p)) continue;
        const int up = links_[std::size_t(p)].first, low = links_[std::size_t(p)].second;
        void* up_out = (zero_copy && up >= 0) ? parts_[up].buf[out] : nullptr;
        void* low_out = (zero_copy && low >= 0) ? parts_[low].buf[out] : nullptr;
        const int n = decomp_.thickness(p);
        // one kernel per partition: every plane, the shared layers storing
        // their crossing populations into the neighbours' halos (zero copy)
        trace_.phase(steps_done_, 1, "step", p, cur_device(), "engine", stream_, [&] {
            dispatch(cfg_, [&](auto ops) {
                decltype(ops)::launch_step(cfg_, decomp_, maps_, p, parts_[p].buf[in], parts_[p].buf[out], up_out,
                                           low_out, wrap, steps_done_, error_flag_, 0, 1, n, stream_, false, diag);
            });
        });
    }
    cur_ = out;
    if (!zero_copy) trace_.phase(steps_done_, 2, "halo_copy", -1, cur_device(), "engine", stream_, [&] { halo_copy(0); });
    ++steps_done_;
}

void DenseEngine::enqueue_steps(int n) {
    check_links();
    if (multi_) {
        enqueue_multi(n, nullptr, true);
        return;
    }
    for (int i = 0; i < n; ++i) launch_step();
}

// ---- single-process multi-device schedule ----------------------------------------------
//
// Partition p runs on devices[p] with two streams, the multi-process OCC
// schedule (launch_step_distributed) with the step flags replaced by
// cross-device event waits, since every partition lives in this process:
//
//   I_p: after S_p(t-1)                                  -> interior(t)     [planes 1..n-2]
//   S_p: after I_p(t-1), S_up(t-1), S_low(t-1)           -> shared(t)       [planes 0, n-1]
//        (+ zero-copy peer stores into the neighbours' halos of the next
//         buffer, or span copies / NCCL send-recv after it)
//
// S_up(t-1)/S_low(t-1) cover both hazards on the neighbours' halos: RAW (they
// filled ours for step t) and WAR (they finished reading the halo slots of the
// buffer our shared(t) now stores into). The interior never reads a halo, so it
// overlaps the whole exchange. A batch of steps forks from the engine stream
// (ev_fork_) and joins back into it, so the engine stream orders a batch
// against I/O, probes and the next batch; graph replays capture exactly that
// fork -> steps -> join shape.

void DenseEngine::launch_step_multi(int step_off, bool first, const DiagTarget* dev_diag, bool capturing) {
    const bool wrap = cfg_.scenario == Scenario::PeriodicBox;
    const bool zero_copy = cfg_.halo == HaloMode::ZeroCopy;
    const int in = cur_, out = cur_ ^ 1;
    const int par = steps_done_ & 1, prev = par ^ 1;
    const int step_arg = capturing ? step_off : steps_done_;
    const int* sb = capturing ? step_base_ : nullptr;
    const int P = cfg_.partitions;
    auto ready = [&](int p) { return dev_diag ? dx_[std::size_t(dev_index(parts_[p].device))].ev : ev_fork_; };
    auto diag_of = [&](int p) -> DiagTarget* {
        if (!dev_diag) return nullptr;
        return const_cast<DiagTarget*>(&dev_diag[dev_index(parts_[p].device)]);
    };
    for (int p = 0; p < P; ++p) {
        PartExec& x = px_[std::size_t(p)];
        DeviceGuard g(parts_[p].device);
        VOXL_CUDA(cudaStreamWaitEvent(x.interior, first ? ready(p) : x.ev_s[prev], 0));
        const int n = decomp_.thickness(p);
        trace_.phase(steps_done_, 1, "interior", p, parts_[p].device, "interior", x.interior, [&] {
            dispatch(cfg_, [&](auto ops) {
                decltype(ops)::launch_step(cfg_, decomp_, maps_, p, parts_[p].buf[in], parts_[p].buf[out], nullptr,
                                           nullptr, wrap, step_arg, error_flag_, 1, 1, n - 2, x.interior, false,
                                           diag_of(p), sb);
            });
        });
        VOXL_CUDA(cudaEventRecord(x.ev_i[par], x.interior));
    }
    for (int p = 0; p < P; ++p) {
        PartExec& x = px_[std::size_t(p)];
        DeviceGuard g(parts_[p].device);
        const int up = links_[std::size_t(p)].first, low = links_[std::size_t(p)].second;
        if (first) {
            VOXL_CUDA(cudaStreamWaitEvent(x.shared, ready(p), 0));
        } else {
            VOXL_CUDA(cudaStreamWaitEvent(x.shared, x.ev_i[prev], 0));
            if (up >= 0 && up != p) VOXL_CUDA(cudaStreamWaitEvent(x.shared, px_[std::size_t(up)].ev_s[prev], 0));
            if (low >= 0 && low != p && low != up)
                VOXL_CUDA(cudaStreamWaitEvent(x.shared, px_[std::size_t(low)].ev_s[prev], 0));
        }
        const int n = decomp_.thickness(p);
        void* up_out = (zero_copy && up >= 0) ? parts_[up].buf[out] : nullptr;
        void* low_out = (zero_copy && low >= 0) ? parts_[low].buf[out] : nullptr;
        trace_.phase(steps_done_, 2, "shared", p, parts_[p].device, "shared", x.shared, [&] {
            dispatch(cfg_, [&](auto ops) {
                decltype(ops)::launch_step(cfg_, decomp_, maps_, p, parts_[p].buf[in], parts_[p].buf[out], up_out,
                                           low_out, wrap, step_arg, error_flag_, 0, n - 1, 2, x.shared, false,
                                           diag_of(p), sb);
            });
        });
        if (cfg_.halo == HaloMode::Copy)
            trace_.phase(steps_done_, 2, "halo_copy", p, parts_[p].device, "shared", x.shared, [&] {
                for (const auto& r : ledger_records(0)) {
                    if (r.src != p) continue;
                    char* dst = static_cast<char*>(parts_[r.dst].buf[out]) + r.dst_span.base * esize_;
                    const char* src = static_cast<const char*>(parts_[r.src].buf[out]) + r.src_span.base * esize_;
                    VOXL_CUDA(
                        cudaMemcpyAsync(dst, src, std::size_t(r.elements) * esize_, cudaMemcpyDefault, x.shared));
                }
            });
    }
    if (nccl_) {
        // every partition's sends and receives in one group (one thread drives
        // all communicators); records in the reference's order on both sides
        nccl_->check(nccl_->group_start(), "ncclGroupStart");
        for (const auto& r : ledger_records(0)) {
            const std::size_t bytes = std::size_t(r.elements) * esize_;
            const char* src = static_cast<const char*>(parts_[r.src].buf[out]) + r.src_span.base * esize_;
            char* dst = static_cast<char*>(parts_[r.dst].buf[out]) + r.dst_span.base * esize_;
            nccl_->check(nccl_->send(src, bytes, ncclInt8, r.dst, nccl_->comms[std::size_t(r.src)],
                                     px_[std::size_t(r.src)].shared), "ncclSend");
            nccl_->check(nccl_->recv(dst, bytes, ncclInt8, r.src, nccl_->comms[std::size_t(r.dst)],
                                     px_[std::size_t(r.dst)].shared), "ncclRecv");
        }
        nccl_->check(nccl_->group_end(), "ncclGroupEnd");
    }
    for (int p = 0; p < P; ++p) {
        DeviceGuard g(parts_[p].device);
        VOXL_CUDA(cudaEventRecord(px_[std::size_t(p)].ev_s[par], px_[std::size_t(p)].shared));
    }
    cur_ = out;
    ++steps_done_;
}

void DenseEngine::fork_multi() {
    VOXL_CUDA(cudaEventRecord(ev_fork_, stream_));
}

void DenseEngine::join_multi() {
    // the engine stream waits for the last step's two streams of every partition
    const int last = (steps_done_ - 1) & 1;
    for (auto& x : px_) {
        VOXL_CUDA(cudaStreamWaitEvent(stream_, x.ev_i[last], 0));
        VOXL_CUDA(cudaStreamWaitEvent(stream_, x.ev_s[last], 0));
    }
}

void DenseEngine::capture_graph(int parity) {
    // fork -> graph_steps steps -> join -> step counter += graph_steps, captured
    // from the engine stream; cross-device waits become graph edges. The host
    // bookkeeping (parity, step count) advances during capture and is rolled
    // back: replaying the graph advances it.
    const int saved_cur = cur_, saved_steps = steps_done_;
    cur_ = parity;
    steps_done_ = parity;  // event parity follows the step count
    cudaGraph_t graph = nullptr;
    VOXL_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeRelaxed));
    try {
        fork_multi();
        for (int s = 0; s < cfg_.graph_steps; ++s) launch_step_multi(s, s == 0, nullptr, true);
        join_multi();
        advance_step_kernel<<<1, 1, 0, stream_>>>(step_base_, cfg_.graph_steps);
        VOXL_CUDA(cudaGetLastError());
    } catch (...) {
        cudaStreamEndCapture(stream_, &graph);
        if (graph) cudaGraphDestroy(graph);
        cur_ = saved_cur;
        steps_done_ = saved_steps;
        throw;
    }
    VOXL_CUDA(cudaStreamEndCapture(stream_, &graph));
    cur_ = saved_cur;
    steps_done_ = saved_steps;
    const cudaError_t e = cudaGraphInstantiate(&graph_[parity], graph, 0);
    cudaGraphDestroy(graph);
    VOXL_CUDA(e);
}

void DenseEngine::enqueue_multi(int n, const DiagTarget* dev_diag, bool use_graph) {
    if (n <= 0) return;
    int done = 0;
    const int G = cfg_.graph_steps;
    if (use_graph && !dev_diag && !nccl_ && !trace_.enabled() && G > 0 && n >= G) {
        // the graph's kernels report a failing step as *step_base + offset
        const int base = steps_done_;
        VOXL_CUDA(cudaMemcpyAsync(step_base_, &base, sizeof(int), cudaMemcpyHostToDevice, stream_));
        VOXL_CUDA(cudaStreamSynchronize(stream_));  // `base` is a stack value
        while (n - done >= G) {
            if (!graph_[cur_]) {
                try {
                    capture_graph(cur_);
                } catch (const CudaError& e) {
                    // a driver that cannot capture this schedule (e.g. across
                    // devices) keeps the same launches issued from the host
                    graph_note_ = e.what();
                    cfg_.graph_steps = 0;
                    cudaGetLastError();
                    break;
                }
            }
            VOXL_CUDA(cudaGraphLaunch(graph_[cur_], stream_));
            steps_done_ += G;  // G is even: the parity is unchanged
            done += G;
        }
    }
    if (done == n) return;
    fork_multi();
    for (int s = done; s < n; ++s) launch_step_multi(s - done, s == done, nullptr, false);
    join_multi();
}

double DenseEngine::timed_steps(int n, double* kernel_ms) {
    if (multi_) {
        // one event pair on the engine stream around the whole fork -> steps ->
        // join batch (the partitions' streams overlap inside it)
        check_links();
        cudaEvent_t e0, e1;
        VOXL_CUDA(cudaEventCreate(&e0));
        VOXL_CUDA(cudaEventCreate(&e1));
        VOXL_CUDA(cudaEventRecord(e0, stream_));
        enqueue_multi(n, nullptr, true);
        VOXL_CUDA(cudaEventRecord(e1, stream_));
        VOXL_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        VOXL_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (kernel_ms) *kernel_ms = ms;
        check_errors();
        return ms;
    }
    // CUDA events on the launching stream: one pair around each step (the
    // step's kernels), plus the span from the first to the last event.
    std::vector<cudaEvent_t> ev(2 * std::size_t(n));
    for (auto& e : ev) VOXL_CUDA(cudaEventCreate(&e));
    for (int i = 0; i < n; ++i) {
        VOXL_CUDA(cudaEventRecord(ev[2 * i], stream_));
        launch_step();
        if (i == n - 1) join_streams();
        VOXL_CUDA(cudaEventRecord(ev[2 * i + 1], stream_));
    }
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    double ksum = 0.0;
    for (int i = 0; i < n; ++i) {
        float ms = 0.f;
        VOXL_CUDA(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
        ksum += ms;
    }
    float total = 0.f;
    if (n > 0) VOXL_CUDA(cudaEventElapsedTime(&total, ev[0], ev[2 * n - 1]));
    for (auto& e : ev) cudaEventDestroy(e);
    if (kernel_ms) *kernel_ms = ksum;
    check_errors();
    return total;
}

void DenseEngine::check_errors() {
    join_streams();
    int flag = INT_MAX;
    std::uint32_t stalled = 0;
    VOXL_CUDA(cudaMemcpyAsync(&flag, error_flag_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
    if (distributed_ && flags_)
        VOXL_CUDA(cudaMemcpyAsync(&stalled, flags_ + 2, sizeof(std::uint32_t), cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    if (stalled)
        throw std::runtime_error("halo exchange stalled at step " + std::to_string(stalled - 1) +
                                 ": a neighbour partition stopped signalling (zero-copy step flags)");
    if (flag != INT_MAX)
        throw InstabilityError("run aborted at step " + std::to_string(flag) +
                               ": macroscopic: non-positive density");
}

void DenseEngine::step(int n) {
    if (n < 0) throw std::invalid_argument("step: n must be >= 0");
    enqueue_steps(n);
    check_errors();
}

int DenseEngine::step_probe_n(int n, DenseDiag* rows, std::string* abort_msg) {
    // Batches of up to kDiagBatch steps: each step launches the step kernel
    // with probe_field fused (accumulating into the step's ring slot); one
    // reduction kernel, one copy and one host synchronisation per batch.
    if (n < 0) throw std::invalid_argument("step_probe: n must be >= 0");
    check_links();
    if (multi_) return step_probe_n_multi(n, rows, abort_msg);
    if (!ring_) ring_ = std::make_unique<DiagRing>();
    int done = 0;
    while (done < n) {
        const int b = std::min(n - done, kDiagBatch);
        const int step0 = steps_done_;
        ring_->begin(b, stream_);
        // the shared-layer stream (multi-process OCC) writes the ring too
        if (shared_stream_) {
            VOXL_CUDA(cudaEventRecord(ev_fork_, stream_));
            VOXL_CUDA(cudaStreamWaitEvent(shared_stream_, ev_fork_, 0));
        }
        for (int s = 0; s < b; ++s) {
            DiagTarget dt;
            dt.acc = ring_->acc(s);
            dt.bad = ring_->bad(s);
            launch_step(&dt);
        }
        join_streams();
        ring_->reduce(error_flag_, stream_);
        VOXL_CUDA(cudaStreamSynchronize(stream_));
        const DiagRow* r = ring_->rows();
        std::string msg;
        const int fail = first_failure(r, b, step0, ring_->error_flag(), &msg);
        const int good = fail < 0 ? b : fail;
        for (int s = 0; s < good; ++s) {
            DenseDiag& d = rows[done + s];
            d = DenseDiag{};
            d.mass = r[s].mass;
            d.max_speed = std::sqrt(r[s].v2);
        }
        done += good;
        if (fail >= 0) {
            if (abort_msg) *abort_msg = msg;
            last_bad_ = r[fail].bad;
            return done;
        }
    }
    return done;
}

int DenseEngine::step_probe_n_multi(int n, DenseDiag* rows, std::string* abort_msg) {
    // As step_probe_n, with one accumulator ring per device: each device's
    // kernels commit into their own ring (no cross-device atomics), and the
    // exact integer sums of the rings add up on the host before the single
    // rounding to fp64 -- the same row bit for bit as one device would give.
    for (auto& d : dx_)
        if (!d.ring) {
            DeviceGuard g(d.device);
            d.ring = std::make_unique<DiagRing>();
        }
    std::vector<DiagTarget> dt(dx_.size());
    std::vector<DiagRaw> raw;
    int done = 0;
    while (done < n) {
        const int b = std::min(n - done, kDiagBatch);
        const int step0 = steps_done_;
        fork_multi();
        for (auto& d : dx_) {
            DeviceGuard g(d.device);
            if (d.aux != stream_) VOXL_CUDA(cudaStreamWaitEvent(d.aux, ev_fork_, 0));
            d.ring->begin(b, d.aux);
            VOXL_CUDA(cudaEventRecord(d.ev, d.aux));
        }
        for (int s = 0; s < b; ++s) {
            for (std::size_t i = 0; i < dx_.size(); ++i) {
                dt[i].acc = dx_[i].ring->acc(s);
                dt[i].bad = dx_[i].ring->bad(s);
            }
            launch_step_multi(s, s == 0, dt.data(), false);
        }
        const int last = (steps_done_ - 1) & 1;
        for (std::size_t i = 0; i < dx_.size(); ++i) {
            DevExec& d = dx_[i];
            DeviceGuard g(d.device);
            for (int p = 0; p < cfg_.partitions; ++p) {
                if (parts_[p].device != d.device) continue;
                VOXL_CUDA(cudaStreamWaitEvent(d.aux, px_[std::size_t(p)].ev_i[last], 0));
                VOXL_CUDA(cudaStreamWaitEvent(d.aux, px_[std::size_t(p)].ev_s[last], 0));
            }
            d.ring->reduce(i == 0 ? error_flag_ : nullptr, d.aux);
            VOXL_CUDA(cudaEventRecord(d.ev, d.aux));
            if (i > 0) VOXL_CUDA(cudaStreamWaitEvent(stream_, d.ev, 0));
        }
        join_multi();
        for (auto& d : dx_) VOXL_CUDA(cudaStreamSynchronize(d.aux));
        raw.assign(dx_[0].ring->raw(), dx_[0].ring->raw() + b);
        for (std::size_t i = 1; i < dx_.size(); ++i)
            for (int s = 0; s < b; ++s) diag_accumulate(raw[std::size_t(s)], dx_[i].ring->raw()[s]);
        std::vector<DiagRow> r(static_cast<std::size_t>(b));
        for (int s = 0; s < b; ++s) r[std::size_t(s)] = diag_compose(raw[std::size_t(s)]);
        std::string msg;
        const int fail = first_failure(r.data(), b, step0, dx_[0].ring->error_flag(), &msg);
        const int good = fail < 0 ? b : fail;
        for (int s = 0; s < good; ++s) {
            DenseDiag& d = rows[done + s];
            d = DenseDiag{};
            d.mass = r[std::size_t(s)].mass;
            d.max_speed = std::sqrt(r[std::size_t(s)].v2);
        }
        done += good;
        if (fail >= 0) {
            if (abort_msg) *abort_msg = msg;
            last_bad_ = r[std::size_t(fail)].bad;
            return done;
        }
    }
    return done;
}

DenseDiag DenseEngine::step_probe() {
    // One probed step; a probe_field instability comes back in the row (the
    // caller composes run()'s text), a non-positive density throws.
    DenseDiag d;
    std::string msg;
    if (step_probe_n(1, &d, &msg) == 1) return d;
    if (msg.find("macroscopic") != std::string::npos) throw InstabilityError(msg);
    d = DenseDiag{};
    d.unstable = 1;
    d.bad_voxel = std::int64_t(last_bad_ >> 5);
    d.bad_population = int(last_bad_ & 31u);
    d.mass = std::nan("");
    d.max_speed = std::nan("");
    return d;
}

DenseDiag DenseEngine::probe() {
    join_streams();
    double* partial = diag_scratch_;
    double* out = diag_scratch_ + 2 * kProbeBlocks;
    auto* bad = reinterpret_cast<unsigned long long*>(diag_scratch_ + 2 * kProbeBlocks + 2);
    const double zero[2] = {0.0, 0.0};
    const unsigned long long none = ~0ull;
    VOXL_CUDA(cudaMemcpyAsync(out, zero, sizeof zero, cudaMemcpyHostToDevice, stream_));
    VOXL_CUDA(cudaMemcpyAsync(bad, &none, sizeof none, cudaMemcpyHostToDevice, stream_));
    for (int p = 0; p < cfg_.partitions; ++p) {
        if (!local(p)) continue;
        dispatch(cfg_, [&](auto ops) {
            decltype(ops)::probe(decomp_, maps_[p], p, parts_[p].buf[cur_], partial, bad, out, stream_);
        });
    }
    double res[2];
    unsigned long long b = 0;
    VOXL_CUDA(cudaMemcpyAsync(res, out, sizeof res, cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaMemcpyAsync(&b, bad, sizeof b, cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    DenseDiag d;
    d.mass = res[0];
    d.max_speed = std::sqrt(res[1]);  // the kernels reduce |u|^2
    if (b != ~0ull) {
        d.unstable = 1;
        d.bad_voxel = std::int64_t(b >> 5);
        d.bad_population = int(b & 31);
    }
    return d;
}

std::vector<TransferRecord> DenseEngine::ledger_records(int step) const {
    // the decomposition's records, less the links a caller cut (set_neighbor_links)
    std::vector<TransferRecord> out;
    for (const auto& r : halo_records(decomp_, maps_, step))
        if (links_[std::size_t(r.src)].first == r.dst || links_[std::size_t(r.src)].second == r.dst) out.push_back(r);
    return out;
}

} // namespace voxl_b200
