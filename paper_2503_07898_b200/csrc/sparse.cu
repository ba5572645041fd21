// sparse.cu -- block-sparse kernels and engine (see sparse.cuh).
//
// One CTA per block (E^3 threads, one voxel each). The CTA stages its 27
// neighbour-block indices and activity masks in shared memory; each pull then
// resolves "source active?" with a shared-memory bit test and reads the source
// population straight from the neighbour block's SoA plane (a warp covers
// 32 / E rows of one block, so a plane read is one contiguous run plus the
// lanes that cross into the x-neighbour block). Inactive sources bounce back
// off the voxel's own opposite population (sparse.cpp:321-345). Algorithmic
// traffic: 2*Q*sizeof(real) per active voxel, plus 27 ints and 27*E^3/8 mask
// bytes per block of metadata (L2-resident, < 0.2 % at E = 8).
#include "sparse.cuh"
#include "lattice.cuh"
#include "digest.cuh"
#include "canon_io.cuh"
#include "block_probe.cuh"
#include "diag_ring.cuh"
#include "phase_trace.cuh"
#include "tma.cuh"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <cstdlib>

// fused-probe commit of the block kernels (diag_ring.cuh): per-word zero
// tests and the L2 evict_last policy kept unless measured otherwise
#ifndef VOXL_BLOCK_DIAG_UNCOND
#define VOXL_BLOCK_DIAG_UNCOND 0
#endif
#ifndef VOXL_BLOCK_DIAG_POLICY
#define VOXL_BLOCK_DIAG_POLICY 1
#endif

namespace voxl_b200 {

namespace {

// Velocity source of the regularized boundary (Table 2 "indexing" column).
enum VelSource : int { kVelConst = 0, kVelIndirect = 1, kVelInline = 2 };
// Kernel flavours.
enum SparseMode : int { kLight = 0, kHeavy = 1 };

template <int Q, class R>
struct SparseArgs {
    const R* cur;
    R* nxt;
    const std::int32_t* nbr;      // 27 per block
    const std::uint64_t* masks;   // WORDS per block
    const std::uint8_t* full;     // 1 iff the block and its 26 neighbours are all fully active
    const int* origins;           // 3 per block
    int block_begin;
    const std::uint8_t* bitmask;  // DisagBitmask: skip blocks whose bit != want
    int bitmask_want;
    int tma;                      // host: one block per CTA staged by a bulk copy (sparse_tma_kernel)
    int scan_span;                // > 0 (bitmask sweep): each CTA pair walks this many consecutive blocks
    int scan_blocks;              //   of the sweep's scan_blocks
    const int* span_lo;           // bitmask sweep, balanced: CTA pair p walks blocks [span_lo[p], span_lo[p+1])
    int span_pairs;               //   for p < span_pairs
    int vel_source;
    const std::int32_t* meta_index;  // per slot (DisagBitmask)
    const R* compact_meta;           // 3 per boundary voxel (DisagBitmask)
    const R* naive_meta;             // 3 per slot (Naive)
    R u_bc[3];
    int nx;
    R omega, keep;
    double shift[Q];  // w_i for shifted fp32 storage
    int step;
    int* error_flag;
    // fused probe_field (DIAG kernels): the step's accumulator lanes and
    // first-offender word (diag_ring.cuh); canon[slot] = the voxel's index in
    // canonical_state order (read for an unstable voxel only)
    unsigned long long* diag_acc;
    unsigned long long* diag_bad;
    const std::int32_t* canon;
};

/// equilibrium (lattice.cpp:104-113) at given (rho, u), reference op order.
template <class L, class R, bool Exact>
__device__ __forceinline__ void equilibrium_dev(R rho, const R (&u)[3], R (&feq)[L::Q]) {
    using A = Arith<R, Exact>;
    const R uu = A::add(A::add(A::mul(u[0], u[0]), A::mul(u[1], u[1])), A::mul(u[2], u[2]));
    const R c15uu = A::mul(R(1.5), uu);
    static_for<L::Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        R eu = R(0);
        eu = acc_term<R, Exact, L::ex(i)>(eu, u[0]);
        eu = acc_term<R, Exact, L::ey(i)>(eu, u[1]);
        eu = acc_term<R, Exact, L::ez(i)>(eu, u[2]);
        constexpr double wi = L::w(i);
        const R poly = A::sub(A::add(A::add(R(1), A::mul(R(3), eu)), A::mul(A::mul(R(4.5), eu), eu)), c15uu);
        feq[i] = A::mul(A::mul(R(wi), rho), poly);
    });
}

/// regularized_reconstruct (lbm.cpp:10-59) for a face with inward normal
/// +-x (the wind tunnel's only regularized faces), reference op order.
template <class L, class R, bool Exact>
__device__ __forceinline__ bool regularized_dev(int sign, const R (&ubc)[3], R (&f)[L::Q]) {
    using A = Arith<R, Exact>;
    const R u_n = A::mul(ubc[0], R(sign));
    if (!(fabs(A::sub(R(1), u_n)) > R(1e-12))) return false;
    R sum0 = R(0), sum_in = R(0);
    static_for<L::Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int ex = L::ex(i);
        const int en = ex * sign;
        if (en == 0) sum0 = A::add(sum0, f[i]);
        else if (en < 0) sum_in = A::add(sum_in, f[i]);
    });
    R rho;
    if constexpr (Exact) rho = A::add(sum0, A::mul(R(2), sum_in)) / A::sub(R(1), u_n);
    else rho = fma_rn(R(2), sum_in, sum0) / A::sub(R(1), u_n);  // FMA spelled out (Arith<float, false>)
    R feq[L::Q];
    equilibrium_dev<L, R, Exact>(rho, ubc, feq);
    R fneq[L::Q];
    static_for<L::Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int oi = L::opp(i);
        const int en = L::ex(i) * sign;
        fneq[i] = en > 0 ? A::sub(f[oi], feq[oi]) : A::sub(f[i], feq[i]);
    });
    // Pi_ab = sum_i fneq_i e_ia e_ib (sequential over i; zero terms skipped).
    R pi[3][3];
    static_for<3>([&](auto AA) {
        constexpr int a = decltype(AA)::value;
        static_for<3>([&](auto BB) {
            constexpr int b = decltype(BB)::value;
            R acc = R(0);
            static_for<L::Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                acc = acc_term<R, Exact, L::e(i, a) * L::e(i, b)>(acc, fneq[i]);
            });
            pi[a][b] = acc;
        });
    });
    constexpr double cs2 = 1.0 / 3.0;
    constexpr double cdiag1 = 1.0 - cs2, cdiag0 = 0.0 - cs2;
    static_for<L::Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        R qpi = R(0);
        static_for<3>([&](auto AA) {
            constexpr int a = decltype(AA)::value;
            static_for<3>([&](auto BB) {
                constexpr int b = decltype(BB)::value;
                constexpr int eab = L::e(i, a) * L::e(i, b);
                if constexpr (a == b) {
                    constexpr double c = eab ? cdiag1 : cdiag0;
                    qpi = A::add(qpi, A::mul(R(c), pi[a][b]));
                } else {
                    qpi = acc_term<R, Exact, eab>(qpi, pi[a][b]);
                }
            });
        });
        constexpr double wi = L::w(i);
        f[i] = A::add(feq[i], A::mul(A::mul(R(wi), R(4.5)), qpi));
    });
    return true;
}

/// CTAs per block: 8^3 blocks are split over two 256-thread CTAs (6 CTAs / SM
/// instead of 3), so each CTA's metadata prologue hides behind five others.
template <int E>
constexpr int kSplit = E == 8 ? 2 : 1;

// Heavy (regularized) kernel: 4 resident 256-thread CTAs per SM (64
// registers, no spill for D3Q19) instead of the unconstrained 72 registers /
// 3 CTAs. Measured at 512^3 disag_mem (-DVOXL_HEAVY_MINB sweep): D3Q19
// 40.88 -> 41.21 GLUPS, D3Q27 28.01 -> 28.69 (the boundary kernel shares the
// GPU with the light one, so its occupancy sets how much it slows it).
#ifndef VOXL_HEAVY_MINB
#define VOXL_HEAVY_MINB 4
#endif
template <class L, class R, bool Exact, int E, int MODE, bool DIAG, bool TMA = false>
__device__ __forceinline__ void sparse_block(const SparseArgs<L::Q, R>& A, int b, int half, const R* s_own = nullptr,
                                             unsigned long long* bar = nullptr, unsigned parity = 0);

template <class L, class R, bool Exact, int E, int MODE, bool DIAG = false>
__global__ void __launch_bounds__(E* E* E / kSplit<E>, E == 8 && sizeof(R) == 4 ? (MODE == 0 ? block_min_ctas(L::Q) : VOXL_HEAVY_MINB) : 1)
    sparse_step_kernel(const __grid_constant__ SparseArgs<L::Q, R> A) {
    constexpr int S = kSplit<E>;
    if (A.span_lo) {
        // DisagBitmask boundary sweep as one long-lived CTA pair per SM
        // (sparse.cpp:369-380: every block visited, skipped unless its bit
        // matches). Pair p walks the blocks [span_lo[p], span_lo[p+1]), cut
        // so that every span holds the same number of boundary blocks; the
        // CTA tests blockDim.x bitmask bytes at once, compacts the hits into
        // shared memory (ballot + warp prefix) and updates them in order.
        constexpr int T = E * E * E / S;
        constexpr int WARPS = (T + 31) / 32;
        __shared__ int s_hit[T];
        __shared__ int s_cnt[WARPS + 1];
        const int pair = int(blockIdx.x) / S;
        const int lo = A.span_lo[pair], hi = A.span_lo[pair + 1];
        const int lane = int(threadIdx.x) & 31, warp = int(threadIdx.x) >> 5;
        for (int base = lo; base < hi; base += T) {
            const int b = base + int(threadIdx.x);
            const bool hit = b < hi && int(A.bitmask[b]) == A.bitmask_want;
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (lane == 0) s_cnt[warp] = __popc(m);
            __syncthreads();
            int off = 0, total = 0;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) {
                off += w < warp ? s_cnt[w] : 0;
                total += s_cnt[w];
            }
            if (hit) s_hit[off + __popc(m & ((1u << lane) - 1u))] = b;
            __syncthreads();
            for (int i = 0; i < total; ++i) {
                sparse_block<L, R, Exact, E, MODE, DIAG>(A, s_hit[i], int(blockIdx.x) % S);
                __syncthreads();  // shared neighbourhood tables are rewritten by the next block
            }
            __syncthreads();  // s_cnt / s_hit are rewritten by the next chunk
        }
        return;
    }
    if (A.scan_span > 0) {
        // DisagBitmask sweep (sparse.cpp:369-380): every block is visited and
        // skipped unless its bit matches. A CTA per block would spend most of
        // the boundary sweep dispatching CTAs that exit at once (0.44 of
        // 0.66 ms at 512^3), so each CTA walks a span of consecutive blocks
        // and skips with one broadcast byte load per block. (A persistent
        // grid was measured worse: its resident 64-register CTAs starve the
        // concurrent light sweep for the whole step.)
        const int lo = A.block_begin + int(blockIdx.x) / S * A.scan_span;
        const int hi = min(lo + A.scan_span, A.block_begin + A.scan_blocks);
        for (int b = lo; b < hi; ++b) {
            if (A.bitmask && int(A.bitmask[b]) != A.bitmask_want) continue;  // CTA-uniform
            sparse_block<L, R, Exact, E, MODE, DIAG>(A, b, int(blockIdx.x) % S);
            __syncthreads();  // shared neighbourhood tables are rewritten by the next block
        }
        return;
    }
    const int b = A.block_begin + int(blockIdx.x) / S;
    if (A.bitmask && int(A.bitmask[b]) != A.bitmask_want) return;  // CTA-uniform skip
    sparse_block<L, R, Exact, E, MODE, DIAG>(A, b, int(blockIdx.x) % S);
}

/// Bulk-copy block staging (opt-in, VOXL_SPARSE_TMA=1): one block per CTA
/// (E^3 threads); the block's Q population planes -- one contiguous span of
/// Q * E^3 values (BlockField layout) -- land in shared memory by a single
/// cp.async.bulk (tma.cuh) that overlaps the CTA's metadata prologue, and
/// own-block pulls (all but the face-crossing ones: 81 % at E = 8, D3Q19)
/// read shared memory. Same arithmetic as sparse_step_kernel (bitwise equal
/// results). Measured slower than the register-pull kernel at 512^3 (light
/// kernel under ncu 3.20 vs 2.94 ms; a persistent, double-buffered variant
/// 4.10 ms): a CTA idles for its copy's full latency before it computes, and
/// 3 x 512-thread CTAs per SM hide that worse than 6 x 256-thread CTAs with
/// 19 loads each in flight. Kept as the measured alternative.
#ifndef VOXL_TMA_MINB_LIGHT
#define VOXL_TMA_MINB_LIGHT 3
#endif
#ifndef VOXL_TMA_MINB_HEAVY
#define VOXL_TMA_MINB_HEAVY 2
#endif
template <class L, class R, bool Exact, int E, int MODE, bool DIAG>
__global__ void __launch_bounds__(E* E* E, MODE == kHeavy ? VOXL_TMA_MINB_HEAVY : (L::Q == 27 ? 2 : VOXL_TMA_MINB_LIGHT))
    sparse_tma_kernel(const __grid_constant__ SparseArgs<L::Q, R> A) {
    constexpr int Q = L::Q, BV = E * E * E;
    extern __shared__ __align__(128) unsigned char sp_tma_smem[];
    R* s_own = reinterpret_cast<R*>(sp_tma_smem);
    __shared__ __align__(8) unsigned long long s_bar;
    const int b = A.block_begin + int(blockIdx.x);
    if (A.bitmask && int(A.bitmask[b]) != A.bitmask_want) return;  // CTA-uniform skip, before any copy
    if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        mbar_arrive_expect_tx(&s_bar, unsigned(Q * BV * sizeof(R)));
        tma_bulk_g2s(s_own, A.cur + (long long)b * Q * BV, unsigned(Q * BV * sizeof(R)), &s_bar);
    }
    // sparse_block's first __syncthreads publishes the initialised barrier
    sparse_block<L, R, Exact, E, MODE, DIAG, true>(A, b, 0, s_own, &s_bar, 0u);
    // the copy must complete before the CTA (and its shared memory) retires,
    // also when every thread of the block returned early
    if (threadIdx.x == 0) mbar_wait(&s_bar, 0);
}

template <class L, class R, bool Exact, int E, int MODE, bool DIAG, bool TMA>
__device__ __forceinline__ void sparse_block(const SparseArgs<L::Q, R>& A, int b, int half, const R* s_own,
                                             unsigned long long* bar, unsigned parity) {
    constexpr int Q = L::Q;
    constexpr int BV = E * E * E;
    constexpr int W = BV >= 64 ? BV / 64 : 1;
    constexpr int S = kSplit<E>;
    __shared__ const R* s_ptr[27];  // component-0 plane of neighbour block d (own block if absent)
    __shared__ int s_nbr[27];
    __shared__ unsigned long long s_mask[27][W];
    __shared__ int s_full;
    const int tid = threadIdx.x;
    const int t = tid + half * (BV / S);  // local voxel index in the block
    if (tid < 27) {
        const int nb = A.nbr[(long long)b * 27 + tid];
        s_nbr[tid] = nb;
        s_ptr[tid] = A.cur + (long long)(nb < 0 ? b : nb) * Q * BV;
    }
    if (tid == 32) s_full = A.full[b];
    __syncthreads();
    // CTA-uniform: every block of the 27-neighbourhood exists and is fully
    // active, so no pull can hit a solid and the mask tests are skipped.
    const bool full = s_full != 0;
    bool live = true;
    if (!full) {
        for (int j = tid; j < 27 * W; j += BV / S) {
            const int d = j / W, w = j % W;
            const int nb = s_nbr[d];
            s_mask[d][w] = nb >= 0 ? A.masks[(long long)nb * W + w] : 0ull;
        }
        __syncthreads();
        live = (s_mask[13][t >> 6] >> (t & 63)) & 1ull;
        if constexpr (!DIAG) {
            if (!live) return;  // inactive slot
        }
    }
    if constexpr (TMA) mbar_wait(bar, parity);  // the block's own populations have landed in shared memory
    // fused probe_field terms of this cell (DIAG)
    using P = std::conditional_t<Exact || sizeof(R) == 8, double, float>;
    P dg_mass = P(0), dg_v2 = P(0);
    int dg_bad = -1;  // first offending population of this voxel (probe_voxel)
    if (live) [&] {
    constexpr int LOG = E == 8 ? 3 : (E == 4 ? 2 : (E == 2 ? 1 : 0));
    const int lx = t & (E - 1), ly = (t >> LOG) & (E - 1), lz = t >> (2 * LOG);
    const long long self_base = (long long)b * Q * BV;
    const bool xlo = lx == 0, xhi = lx == E - 1, ylo = ly == 0, yhi = ly == E - 1, zlo = lz == 0, zhi = lz == E - 1;
    // SWAR field-wise add mod E: source local = (lx-ex, ly-ey, lz-ez) mod E.
    constexpr int H = (1 << (LOG - 1)) | (1 << (2 * LOG - 1)) | (1 << (3 * LOG - 1));
    constexpr int LM = (BV - 1) & ~H;
    const int tL = t & LM, tH = t & H;

    R g[Q];
    static_for<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int ex = L::ex(i), ey = L::ey(i), ez = L::ez(i);
        constexpr int oi = L::opp(i);
        constexpr int D = ((-ex) & (E - 1)) | (((-ey) & (E - 1)) << LOG) | (((-ez) & (E - 1)) << (2 * LOG));
        const int sl = (tL + (D & LM)) ^ (tH ^ (D & H));
        int d = 13;
        if constexpr (ex > 0) d -= xlo;
        if constexpr (ex < 0) d += xhi;
        if constexpr (ey > 0) d -= 3 * ylo;
        if constexpr (ey < 0) d += 3 * yhi;
        if constexpr (ez > 0) d -= 9 * zlo;
        if constexpr (ez < 0) d += 9 * zhi;
        if constexpr (TMA) {
            // own-block pulls from the shared-memory copy, face pulls from
            // the neighbour blocks in global memory (L2)
            const bool solid = !full && !((s_mask[d][sl >> 6] >> (sl & 63)) & 1ull);
            if (solid) g[i] = s_own[oi * BV + t];
            else if (d == 13) g[i] = s_own[i * BV + sl];
            else g[i] = __ldg(s_ptr[d] + (i * BV + sl));
        } else {
            const R* src = s_ptr[d] + (i * BV + sl);
            if (!full) {
                const bool solid = !((s_mask[d][sl >> 6] >> (sl & 63)) & 1ull);
                if (solid) src = A.cur + self_base + (oi * BV + t);
            }
            g[i] = __ldg(src);
        }
    });

    bool ok = true;
    if constexpr (MODE == kHeavy) {
        const int x = A.origins[3 * b] + lx;
        if (x == 0 || x == A.nx - 1) {
            R u[3];
            if (A.vel_source == kVelConst) {
                u[0] = A.u_bc[0];
                u[1] = A.u_bc[1];
                u[2] = A.u_bc[2];
            } else if (A.vel_source == kVelIndirect) {
                const int id = A.meta_index[(long long)b * BV + t];
                u[0] = A.compact_meta[3 * (long long)id];
                u[1] = A.compact_meta[3 * (long long)id + 1];
                u[2] = A.compact_meta[3 * (long long)id + 2];
            } else {
                const long long s3 = 3 * ((long long)b * BV + t);
                u[0] = A.naive_meta[s3];
                u[1] = A.naive_meta[s3 + 1];
                u[2] = A.naive_meta[s3 + 2];
            }
            if constexpr (!Exact) {  // reconstruct on the unshifted populations
                static_for<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    g[i] += R(A.shift[i]);
                });
            }
            ok = regularized_dev<L, R, Exact>(x == 0 ? 1 : -1, u, g);
            if constexpr (!Exact) {
                static_for<Q>([&](auto I) {
                    constexpr int i = decltype(I)::value;
                    g[i] -= R(A.shift[i]);
                });
            }
        }
    }
    R rho, uu[3], dr = R(0);
    if constexpr (Exact) bgk_relax<L, R, true>(g, A.omega, A.keep, rho, uu, ok);
    else bgk_relax_shifted<L, R>(g, A.omega, A.keep, rho, uu, ok, DIAG ? &dr : nullptr);
    if (!ok) atomicMin(A.error_flag, A.step);
    if constexpr (DIAG) probe_voxel<L, R, Exact, P>(g, rho, dr, uu, dg_mass, dg_v2, dg_bad);
    static_for<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        A.nxt[self_base + (long long)i * BV + t] = g[i];
    });
    }();

    // Fused probe_field (lbm.cpp:116-138): the warp's mass and max |u|^2 go
    // into the step's accumulator lanes (order-independent integer sums,
    // diag_ring.cuh); an unstable voxel names itself by canonical index.
    if constexpr (DIAG) {
        if (live && dg_bad >= 0)
            atomicMin(A.diag_bad, ((unsigned long long)A.canon[(long long)b * BV + t] << 5) |
                                      (unsigned long long)dg_bad);
        P pm = dg_mass, pv = dg_bad >= 0 ? P(0) : dg_v2;
        const unsigned lanes = __ballot_sync(0xffffffffu, live);
        constexpr int kWarps = (BV / S + 31) / 32;
        const unsigned long long warp_id = ((unsigned long long)b * S + half) * kWarps + (tid >> 5);
        if constexpr (std::is_same_v<P, float>) {
            diag_warp_commit_f32<VOXL_BLOCK_DIAG_UNCOND != 0, VOXL_BLOCK_DIAG_POLICY != 0>(A.diag_acc, warp_id, pm, pv, lanes);
        } else {
            for (int o = 16; o > 0; o >>= 1) {
                pm += __shfl_xor_sync(0xffffffffu, pm, o);
                pv = max(pv, __shfl_xor_sync(0xffffffffu, pv, o));
            }
            if ((tid & 31) == 0 && lanes) diag_commit(A.diag_acc, warp_id, double(pm), double(pv));
        }
    }
}

template <int Q, class R>
__global__ void sparse_fill_kernel(R* buf, long long total, int bv, const __grid_constant__ SparseArgs<Q, R> A) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int c = int((e / bv) % Q);
    buf[e] = R(A.shift[c]);  // shift[] carries (feq - storage shift) here
}

template <class L, class R>
__global__ void sparse_probe_kernel(const R* buf, const std::int64_t* slots, long long n, int bv,
                                    const __grid_constant__ SparseArgs<L::Q, R> A, double* partial,
                                    unsigned long long* bad) {
    constexpr int Q = L::Q;
    double mass = 0.0, vmax = 0.0;
    const int lb = __ffs(bv) - 1;  // block volume is a power of two
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        const long long slot = slots[v];
        const R* p = buf + ((slot >> lb) * Q << lb) + (slot & (bv - 1));
        R raw[Q];
        static_for<Q>([&](auto I) {  // all loads in flight before the fp64 arithmetic
            constexpr int i = decltype(I)::value;
            raw[i] = p[(long long)i * bv];
        });
        int bp = -1;
        double r = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            const double fi = double(raw[i]) + A.shift[i];
            if (bp < 0 && !(fabs(fi) <= 1e3)) bp = i;
            mass += fi;
            r += fi;
            mx = acc_term<double, false, L::ex(i)>(mx, fi);
            my = acc_term<double, false, L::ey(i)>(my, fi);
            mz = acc_term<double, false, L::ez(i)>(mz, fi);
        });
        if (bp >= 0 || !(r > 0.0)) {
            atomicMin(bad, ((unsigned long long)v << 5) | (unsigned long long)(bp < 0 ? kBadDensity : bp));
        } else {
            const double ux = mx / r, uy = my / r, uz = mz / r;
            vmax = fmax(vmax, sqrt(ux * ux + uy * uy + uz * uz));
        }
    }
    __shared__ double sm[256], sv[256];
    sm[threadIdx.x] = mass;
    sv[threadIdx.x] = vmax;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
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

constexpr int kSpProbeBlocks = 592;
#ifndef VOXL_BITMASK_SPAN
#define VOXL_BITMASK_SPAN 64
#endif
constexpr int kBitmaskSpan = VOXL_BITMASK_SPAN;  // blocks per CTA pair of the bitmask boundary sweep
#ifndef VOXL_BITMASK_PAIRS
#define VOXL_BITMASK_PAIRS 0
#endif
// bitmask boundary sweep: CTA pairs with balanced spans (0: one per SM in
// D3Q19, fixed kBitmaskSpan spans in D3Q27; -1: always fixed spans)
constexpr int kBitmaskPairs = VOXL_BITMASK_PAIRS;
#ifndef VOXL_HEAVY_LOW_PRIO
#define VOXL_HEAVY_LOW_PRIO 0
#endif
constexpr bool kHeavyLowPrio = VOXL_HEAVY_LOW_PRIO != 0;
#ifndef VOXL_HEAVY_CTAS
#define VOXL_HEAVY_CTAS 0
#endif
constexpr int kHeavyCtas = VOXL_HEAVY_CTAS;  // DisagMem boundary kernel: CTA pairs (0: one per SM, -1: per block)

template <class L, class R, bool Exact>
struct SparseOps {
    static constexpr int Q = L::Q;

    static SparseArgs<Q, R> base_args(const SparseConfig& cfg) {
        SparseArgs<Q, R> A{};
        const double inv_tau = 1.0 / cfg.tau;
        A.omega = R(inv_tau);
        A.keep = Exact ? R(1.0 - inv_tau) : R(1) - R(inv_tau);
        for (int a = 0; a < 3; ++a) A.u_bc[a] = R(cfg.u_bc[a]);
        A.nx = cfg.domain[0];
        for (int c = 0; c < Q; ++c) A.shift[c] = Exact ? 0.0 : L::w(c);
        return A;
    }


    template <int E>
    static void launch_e(SparseArgs<Q, R>& A, int mode, int nblocks, cudaStream_t st) {
        if (nblocks <= 0) return;
        constexpr int S = kSplit<E>;
        dim3 grid(nblocks * S);
        const dim3 block(E * E * E / S);
        if (A.span_lo) {  // balanced bitmask sweep: span_pairs CTA pairs
            grid = dim3(A.span_pairs * S);
        } else if (A.scan_span > 0) {  // bitmask sweep: one CTA pair per span of blocks
            A.scan_blocks = nblocks;
            grid = dim3((nblocks + A.scan_span - 1) / A.scan_span * S);
        } else if constexpr (E == 8 && std::is_same_v<R, float>) {
            if (A.tma) {  // one CTA per block, the block staged by a bulk copy
                constexpr int smem = Q * E * E * E * int(sizeof(R));
                auto go = [&](auto kern) {
                    VOXL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                    kern<<<nblocks, E * E * E, smem, st>>>(A);
                };
                if (A.diag_acc) {
                    if (mode == kHeavy) go(sparse_tma_kernel<L, R, Exact, E, kHeavy, true>);
                    else go(sparse_tma_kernel<L, R, Exact, E, kLight, true>);
                } else {
                    if (mode == kHeavy) go(sparse_tma_kernel<L, R, Exact, E, kHeavy, false>);
                    else go(sparse_tma_kernel<L, R, Exact, E, kLight, false>);
                }
                VOXL_CUDA(cudaGetLastError());
                return;
            }
        }
        if (A.diag_acc) {
            if (mode == kHeavy) sparse_step_kernel<L, R, Exact, E, kHeavy, true><<<grid, block, 0, st>>>(A);
            else sparse_step_kernel<L, R, Exact, E, kLight, true><<<grid, block, 0, st>>>(A);
        } else {
            if (mode == kHeavy) sparse_step_kernel<L, R, Exact, E, kHeavy><<<grid, block, 0, st>>>(A);
            else sparse_step_kernel<L, R, Exact, E, kLight><<<grid, block, 0, st>>>(A);
        }
        VOXL_CUDA(cudaGetLastError());
    }

    static void launch(int edge, SparseArgs<Q, R>& A, int mode, int nblocks, cudaStream_t st) {
        NvtxRange r(mode == kHeavy ? (A.scan_span || A.span_lo ? "voxl sparse boundary sweep" : "voxl sparse boundary")
                                   : (A.bitmask ? "voxl sparse light sweep" : "voxl sparse light"));
        switch (edge) {
            case 4: launch_e<4>(A, mode, nblocks, st); break;
            case 8: launch_e<8>(A, mode, nblocks, st); break;
            default: throw std::invalid_argument("sparse engine: device kernels support block edge 4 or 8");
        }
    }
};

template <class F>
void sparse_dispatch(int lattice, Precision prec, F&& f) {
    auto by_prec = [&](auto lat) {
        using L = decltype(lat);
        if (prec == Precision::F64) f(SparseOps<L, double, true>{});
        else f(SparseOps<L, float, false>{});
    };
    switch (lattice) {
        case kD3Q19: by_prec(D3Q19{}); break;
        case kD3Q27: by_prec(D3Q27{}); break;
        default: throw std::invalid_argument("sparse engine: D3Q19 or D3Q27 only (3D wind tunnel)");
    }
}

} // namespace

SparseEngine::SparseEngine(const SparseConfig& cfg, const std::uint8_t* active)
    : cfg_(cfg), io_(std::make_unique<CanonPipe>()) {
    if (!(cfg_.tau > 0.5)) throw std::invalid_argument("sparse engine: tau must be > 0.5");
    if (cfg_.lattice != kD3Q19 && cfg_.lattice != kD3Q27)
        throw std::invalid_argument("sparse engine: D3Q19 or D3Q27 only (3D wind tunnel)");
    if (cfg_.edge != 4 && cfg_.edge != 8) throw std::invalid_argument("sparse engine: block edge must be 4 or 8");
    q_ = make_lattice(cfg_.lattice).q;
    esize_ = cfg_.precision == Precision::F64 ? 8 : 4;
    T_ = SparseTables::build(cfg_.domain, active, cfg_.edge, cfg_.strategy, q_);

    {
        int dev = 0;
        VOXL_CUDA(cudaGetDevice(&dev));
        VOXL_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, dev));
    }
    // bulk-copy block staging (sparse_tma_kernel, measured slower): VOXL_SPARSE_TMA=1
    if (const char* e = std::getenv("VOXL_SPARSE_TMA")) tma_ = std::atoi(e) != 0;
    VOXL_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    {
        int lo = 0, hi = 0;
        VOXL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        VOXL_CUDA(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, hi));
        VOXL_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        VOXL_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    }
    const std::size_t nb = std::size_t(grid_.num_blocks());
    const std::size_t bytes = nb * q_ * grid_.block_volume() * esize_;
    for (auto& b : buf_) {
        VOXL_CUDA(cudaMalloc(&b, bytes));
        VOXL_CUDA(cudaMemsetAsync(b, 0, bytes, stream_));
    }
    const auto nbr = grid_.neighbour_table();
    VOXL_CUDA(cudaMalloc(&d_nbr_, nbr.size() * sizeof(std::int32_t)));
    VOXL_CUDA(cudaMemcpy(d_nbr_, nbr.data(), nbr.size() * sizeof(std::int32_t), cudaMemcpyHostToDevice));
    VOXL_CUDA(cudaMalloc(&d_masks_, grid_.masks().size() * sizeof(std::uint64_t)));
    VOXL_CUDA(cudaMemcpy(d_masks_, grid_.masks().data(), grid_.masks().size() * sizeof(std::uint64_t),
                         cudaMemcpyHostToDevice));
    {
        std::vector<std::uint8_t> full(nb, 0);
        for (std::size_t b = 0; b < nb; ++b) {
            bool f = true;
            for (int d = 0; d < 27 && f; ++d) {
                const int n = nbr[b * 27 + d];
                if (n < 0) {
                    f = false;
                    break;
                }
                for (int w = 0; w < grid_.mask_words() && f; ++w) {
                    const std::uint64_t want =
                        grid_.block_volume() >= 64 ? ~0ull : ((1ull << grid_.block_volume()) - 1);
                    f = grid_.mask(n, w) == want;
                }
            }
            full[b] = f;
        }
        VOXL_CUDA(cudaMalloc(&d_full_, nb));
        VOXL_CUDA(cudaMemcpy(d_full_, full.data(), nb, cudaMemcpyHostToDevice));
    }
    std::vector<int> org(nb * 3);
    for (std::size_t b = 0; b < nb; ++b)
        for (int a = 0; a < 3; ++a) org[3 * b + a] = grid_.blocks()[b].origin[a];
    VOXL_CUDA(cudaMalloc(&d_origins_, org.size() * sizeof(int)));
    VOXL_CUDA(cudaMemcpy(d_origins_, org.data(), org.size() * sizeof(int), cudaMemcpyHostToDevice));
    // Boundary-velocity metadata per strategy (sparse.cpp:271-295).
    auto upload_real = [&](const std::vector<double>& v, void** dst) {
        VOXL_CUDA(cudaMalloc(dst, std::max<std::size_t>(1, v.size()) * esize_));
        if (esize_ == 8) {
            VOXL_CUDA(cudaMemcpy(*dst, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
        } else {
            std::vector<float> f(v.begin(), v.end());
            VOXL_CUDA(cudaMemcpy(*dst, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
        }
    };
    const int e = grid_.edge(), nx = cfg_.domain[0];
    if (cfg_.strategy == Strategy::Naive) {
        std::vector<double> meta(nb * grid_.block_volume() * 3, 0.0);
        for (std::size_t b = 0; b < nb; ++b)
            for (int local = 0; local < grid_.block_volume(); ++local) {
                if (!grid_.bit(int(b), local)) continue;
                const int x = grid_.blocks()[b].origin[0] + local % e;
                if (x == 0 || x == nx - 1)
                    for (int d = 0; d < 3; ++d) meta[(b * grid_.block_volume() + local) * 3 + d] = cfg_.u_bc[d];
            }
        upload_real(meta, &d_naive_meta_);
    } else if (cfg_.strategy == Strategy::DisagBitmask) {
        std::vector<double> compact(std::size_t(arr_.boundary_voxel_count) * 3);
        for (std::int64_t i = 0; i < arr_.boundary_voxel_count; ++i)
            for (int d = 0; d < 3; ++d) compact[std::size_t(i) * 3 + d] = cfg_.u_bc[d];
        upload_real(compact, &d_compact_meta_);
        VOXL_CUDA(cudaMalloc(&d_meta_index_, arr_.voxel_meta_index.size() * sizeof(std::int32_t)));
        VOXL_CUDA(cudaMemcpy(d_meta_index_, arr_.voxel_meta_index.data(),
                             arr_.voxel_meta_index.size() * sizeof(std::int32_t), cudaMemcpyHostToDevice));
        VOXL_CUDA(cudaMalloc(&d_bitmask_, nb));
        VOXL_CUDA(cudaMemcpy(d_bitmask_, arr_.boundary_bitmask.data(), nb, cudaMemcpyHostToDevice));
        // the boundary sweep's spans: pair p starts at the (p * n_b / pairs)-th
        // boundary block, so every pair updates the same number of them and
        // every block is tested by exactly one pair
        const int pairs = kBitmaskPairs < 0 ? 0 : (kBitmaskPairs > 0 ? kBitmaskPairs : (q_ == 19 ? sm_count_ : 0));
        std::int64_t n_b = 0;
        for (std::size_t b = 0; b < nb; ++b) n_b += arr_.boundary_bitmask[b] ? 1 : 0;
        if (pairs > 0 && n_b > 0) {
            std::vector<int> lo(std::size_t(pairs) + 1, int(nb));
            lo[0] = 0;
            std::int64_t seen = 0;
            int p = 1;
            for (std::size_t b = 0; b < nb && p < pairs; ++b) {
                if (!arr_.boundary_bitmask[b]) continue;
                while (p < pairs && seen == (std::int64_t(p) * n_b + pairs - 1) / pairs) lo[std::size_t(p++)] = int(b);
                ++seen;
            }
            bitmask_pairs_ = pairs;
            VOXL_CUDA(cudaMalloc(&d_bitmask_spans_, lo.size() * sizeof(int)));
            VOXL_CUDA(cudaMemcpy(d_bitmask_spans_, lo.data(), lo.size() * sizeof(int), cudaMemcpyHostToDevice));
        }
    }
    VOXL_CUDA(cudaMalloc(&d_error_, sizeof(int)));
    const int big = INT_MAX;
    VOXL_CUDA(cudaMemcpy(d_error_, &big, sizeof(int), cudaMemcpyHostToDevice));
    VOXL_CUDA(cudaMalloc(&d_diag_, (2 * kSpProbeBlocks + 4) * sizeof(double)));
    const double u0[3] = {0.0, 0.0, 0.0};
    set_equilibrium(1.0, u0);  // the reference's rest start (sparse.cpp:297-303)
}

SparseEngine::~SparseEngine() {
    if (stream_) cudaStreamSynchronize(stream_);
    for (void* b : buf_) cudaFree(b);
    cudaFree(d_nbr_);
    cudaFree(d_masks_);
    cudaFree(d_full_);
    cudaFree(d_origins_);
    cudaFree(d_bitmask_);
    cudaFree(d_bitmask_spans_);
    cudaFree(d_meta_index_);
    cudaFree(d_compact_meta_);
    cudaFree(d_naive_meta_);
    cudaFree(d_slots_);
    cudaFree(d_error_);
    cudaFree(d_diag_);
    cudaFree(d_canon_);
    if (side_) {
        cudaStreamSynchronize(side_);
        cudaEventDestroy(ev_fork_);
        cudaEventDestroy(ev_join_);
        cudaStreamDestroy(side_);
    }
    if (stream_) cudaStreamDestroy(stream_);
}

void SparseEngine::set_equilibrium(double rho, const double u[3]) {
    // Every slot of both buffers (inactive slots included, as the reference
    // initialises whole blocks) at equilibrium(rho, u).
    const LatticeTable t = make_lattice(cfg_.lattice);
    double feq[27];
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int i = 0; i < t.q; ++i) {
        const double eu = double(t.e[i][0]) * u[0] + double(t.e[i][1]) * u[1] + double(t.e[i][2]) * u[2];
        const double w = double(t.wnum[i]) / double(t.wden[i]);
        feq[i] = w * rho * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * uu);
    }
    const long long total = (long long)grid_.num_blocks() * q_ * grid_.block_volume();
    sparse_dispatch(cfg_.lattice, cfg_.precision, [&](auto ops) {
        using Ops = decltype(ops);
        auto A = Ops::base_args(cfg_);
        for (int c = 0; c < q_; ++c) A.shift[c] = feq[c] - A.shift[c];
        using R = std::remove_pointer_t<decltype(A.nxt)>;
        for (void* b : buf_)
            sparse_fill_kernel<Ops::Q, R><<<unsigned((total + 255) / 256), 256, 0, stream_>>>(
                static_cast<R*>(b), total, grid_.block_volume(), A);
        VOXL_CUDA(cudaGetLastError());
    });
    VOXL_CUDA(cudaStreamSynchronize(stream_));
}

void SparseEngine::ensure_slots() {
    if (d_slots_) return;
    const auto slots = canonical_slots(grid_);
    VOXL_CUDA(cudaMalloc(&d_slots_, slots.size() * sizeof(std::int64_t)));
    VOXL_CUDA(cudaMemcpy(d_slots_, slots.data(), slots.size() * sizeof(std::int64_t), cudaMemcpyHostToDevice));
}

void SparseEngine::transfer(double* host, bool to_device, unsigned long long* digest) {
    // canonical_state / set_state (sparse.cpp:416-453) through the shared
    // pipeline (canon_io.cuh): rows = canonical cells, fp32 wire format for
    // fp32 engines
    ensure_slots();
    const long long n = grid_.num_active();
    const bool wire32 = esize_ == 4 && host != nullptr;
    sparse_dispatch(cfg_.lattice, cfg_.precision, [&](auto ops) {
        using Ops = decltype(ops);
        auto A = Ops::base_args(cfg_);
        using R = std::remove_pointer_t<decltype(A.nxt)>;
        R* buf = static_cast<R*>(buf_[cur_]);
        const int bv = grid_.block_volume();
        auto layout = [&](long long r0, long long r1, void* slot, bool w32) {
            launch_slot_io<Ops::Q, R>(buf, slot, w32, d_slots_ + r0, r1 - r0, bv, A.shift, to_device, stream_);
        };
        auto consume = [&](long long r0, long long r1, void* slot) {
            digest_accumulate(static_cast<const double*>(slot), (r1 - r0) * Ops::Q, r0 * Ops::Q, digest, stream_);
        };
        io_->run(host, n, 1, Ops::Q, to_device, wire32, A.shift, stream_, layout, consume, digest != nullptr);
    });
}

void SparseEngine::set_state(const double* canonical) { transfer(const_cast<double*>(canonical), true, nullptr); }

void SparseEngine::get_state(double* canonical) { transfer(canonical, false, nullptr); }

void SparseEngine::digest(unsigned long long out[2]) {
    unsigned long long* acc = nullptr;
    VOXL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&acc), 2 * sizeof(unsigned long long), stream_));
    VOXL_CUDA(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), stream_));
    transfer(nullptr, false, acc);
    VOXL_CUDA(cudaMemcpyAsync(out, acc, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaFreeAsync(acc, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
}

void SparseEngine::launch(int /*which*/, cudaEvent_t* ev_b, cudaEvent_t* ev_l, const DiagTarget* diag) {
    // sweep / step (sparse.cpp:359-394) as real kernels.
    sparse_dispatch(cfg_.lattice, cfg_.precision, [&](auto ops) {
        using Ops = decltype(ops);
        auto A = Ops::base_args(cfg_);
        using R = std::remove_pointer_t<decltype(A.nxt)>;
        if (diag) {  // fused probe_field (step_probe_n)
            A.diag_acc = diag->acc;
            A.diag_bad = diag->bad;
            A.canon = d_canon_;
        }
        A.cur = static_cast<const R*>(buf_[cur_]);
        A.nxt = static_cast<R*>(buf_[cur_ ^ 1]);
        A.tma = tma_ ? 1 : 0;
        A.nbr = d_nbr_;
        A.masks = d_masks_;
        A.full = d_full_;
        A.origins = d_origins_;
        A.step = steps_done_;
        A.error_flag = d_error_;
        A.meta_index = d_meta_index_;
        A.compact_meta = static_cast<const R*>(d_compact_meta_);
        A.naive_meta = static_cast<const R*>(d_naive_meta_);
        const int nb = grid_.num_blocks();
        const int edge = grid_.edge();
        switch (cfg_.strategy) {
            case Strategy::Naive:
                A.vel_source = kVelInline;
                A.block_begin = 0;
                if (ev_b) VOXL_CUDA(cudaEventRecord(ev_b[0], stream_));
                Ops::launch(edge, A, kHeavy, nb, stream_);
                if (ev_b) VOXL_CUDA(cudaEventRecord(ev_b[1], stream_));
                if (ev_l) {
                    VOXL_CUDA(cudaEventRecord(ev_l[0], stream_));
                    VOXL_CUDA(cudaEventRecord(ev_l[1], stream_));
                }
                break;
            case Strategy::DisagBitmask: {
                // both sweeps scan every block and skip the other class's
                // blocks by bitmask (sparse.cpp:369-380); they write disjoint
                // blocks, so the boundary sweep (spans of blocks per CTA,
                // kBitmaskSpan) runs on the high-priority side stream
                // concurrently with the light sweep, as in DisagMem
                A.vel_source = kVelIndirect;
                A.block_begin = 0;
                A.bitmask = d_bitmask_;
                const bool split = classes_.n_boundary > 0 && classes_.n_boundary < nb;
                // VOXL_HEAVY_LOW_PRIO: the light sweep on the high-priority
                // stream, the boundary sweep behind it on the engine stream
                cudaStream_t hs = split ? (kHeavyLowPrio ? stream_ : side_) : stream_;
                cudaStream_t ls = split ? (kHeavyLowPrio ? side_ : stream_) : stream_;
                if (split) {
                    VOXL_CUDA(cudaEventRecord(ev_fork_, stream_));
                    VOXL_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
                }
                A.bitmask_want = 1;
                if (d_bitmask_spans_) {  // one CTA pair per SM over balanced spans
                    A.span_lo = d_bitmask_spans_;
                    A.span_pairs = bitmask_pairs_;
                } else {
                    A.scan_span = kBitmaskSpan;
                }
                if (ev_b) VOXL_CUDA(cudaEventRecord(ev_b[0], hs));
                Ops::launch(edge, A, kHeavy, nb, hs);
                if (ev_b) VOXL_CUDA(cudaEventRecord(ev_b[1], hs));
                A.scan_span = 0;
                A.span_lo = nullptr;
                A.bitmask_want = 0;
                if (ev_l) VOXL_CUDA(cudaEventRecord(ev_l[0], ls));
                Ops::launch(edge, A, kLight, nb, ls);
                if (ev_l) VOXL_CUDA(cudaEventRecord(ev_l[1], ls));
                if (split) {
                    VOXL_CUDA(cudaEventRecord(ev_join_, side_));
                    VOXL_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
                }
                break;
            }
            case Strategy::DisagMem: {
                A.vel_source = kVelConst;
                // boundary blocks [0, n_b) with the heavy kernel on the side
                // stream, blocks [n_b, nb) with the light kernel on the engine
                // stream, concurrently; joined before the next step.
                const int n_b = int(classes_.n_boundary);
                const bool split = n_b > 0 && n_b < nb;
                cudaStream_t hs = split ? (kHeavyLowPrio ? stream_ : side_) : stream_;
                cudaStream_t ls = split ? (kHeavyLowPrio ? side_ : stream_) : stream_;
                if (split) {
                    VOXL_CUDA(cudaEventRecord(ev_fork_, stream_));
                    VOXL_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
                }
                A.block_begin = 0;
                if (ev_b) VOXL_CUDA(cudaEventRecord(ev_b[0], hs));
                // D3Q19: the boundary kernel as one long-lived CTA pair per
                // SM, each walking a contiguous span of the boundary blocks:
                // it holds few SM slots while the light kernel streams
                // (512^3: 3.171 vs 3.197 ms per step with a CTA pair per
                // block). D3Q27 keeps a pair per block: its heavier boundary
                // update, serialised that way, outlasts the light kernel
                // (4.665 vs 4.577 ms).
                const int pairs = kHeavyCtas < 0 ? 0 : (kHeavyCtas > 0 ? kHeavyCtas : (q_ == 19 ? sm_count_ : 0));
                if (pairs > 0 && n_b > 0) A.scan_span = (n_b + pairs - 1) / pairs;
                if (n_b > 0) Ops::launch(edge, A, kHeavy, n_b, hs);
                A.scan_span = 0;
                if (ev_b) VOXL_CUDA(cudaEventRecord(ev_b[1], hs));
                A.block_begin = n_b;
                if (ev_l) VOXL_CUDA(cudaEventRecord(ev_l[0], ls));
                if (nb > n_b) Ops::launch(edge, A, kLight, nb - n_b, ls);
                if (ev_l) VOXL_CUDA(cudaEventRecord(ev_l[1], ls));
                if (split) {
                    VOXL_CUDA(cudaEventRecord(ev_join_, side_));
                    VOXL_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
                }
                break;
            }
        }
    });
    cur_ ^= 1;
    ++steps_done_;
}

void SparseEngine::check_errors() {
    int flag = INT_MAX;
    VOXL_CUDA(cudaMemcpyAsync(&flag, d_error_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    if (flag != INT_MAX)
        throw InstabilityError("run aborted at step " + std::to_string(flag) + ": macroscopic: non-positive density");
}

void SparseEngine::step(int n) {
    for (int i = 0; i < n; ++i) launch(0, nullptr, nullptr);
    check_errors();
}

namespace {
__global__ void sparse_canon_kernel(const std::int64_t* slots, long long n, std::int32_t* canon) {
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x)
        canon[slots[v]] = std::int32_t(v);
}
} // namespace

int SparseEngine::step_probe_n(int n, DenseDiag* rows, std::string* abort_msg) {
    // Batches of up to kDiagBatch steps (run_sparse's per-step loop,
    // solver.cpp:287-291): each step's kernels fold probe_field's terms into
    // the step's accumulator lanes and name an unstable voxel by canonical
    // index; one reduction kernel, one copy and one host synchronisation per
    // batch.
    if (n < 0) throw std::invalid_argument("step_probe: n must be >= 0");
    if (!ring_) ring_ = std::make_unique<DiagRing>();
    if (!d_canon_) {
        ensure_slots();
        const std::size_t ns = std::size_t(grid_.num_blocks()) * std::size_t(grid_.block_volume());
        VOXL_CUDA(cudaMalloc(&d_canon_, ns * sizeof(std::int32_t)));
        VOXL_CUDA(cudaMemsetAsync(d_canon_, 0xFF, ns * sizeof(std::int32_t), stream_));
        sparse_canon_kernel<<<kSpProbeBlocks, 256, 0, stream_>>>(d_slots_, grid_.num_active(), d_canon_);
        VOXL_CUDA(cudaGetLastError());
    }
    int done = 0;
    while (done < n) {
        const int b = std::min(n - done, kDiagBatch);
        const int step0 = steps_done_;
        ring_->begin(b, stream_);  // side-stream sweeps fork from the engine stream after this
        for (int s = 0; s < b; ++s) {
            DiagTarget dt;
            dt.acc = ring_->acc(s);
            dt.bad = ring_->bad(s);
            launch(0, nullptr, nullptr, &dt);
        }
        ring_->reduce(d_error_, stream_);
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

DenseDiag SparseEngine::step_probe() {
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
    return d;
}

void SparseEngine::step_identity(int n) {
    // step_identity (sparse.cpp:396-404): the sweeps copy every active voxel
    // cur -> nxt. Inactive slots are never observable (canonical_state reads
    // active voxels only), so one device copy of the field is the same step.
    const std::size_t bytes = std::size_t(grid_.num_blocks()) * q_ * grid_.block_volume() * esize_;
    for (int i = 0; i < n; ++i) {
        VOXL_CUDA(cudaMemcpyAsync(buf_[cur_ ^ 1], buf_[cur_], bytes, cudaMemcpyDeviceToDevice, stream_));
        cur_ ^= 1;
        ++steps_done_;
    }
    VOXL_CUDA(cudaStreamSynchronize(stream_));
}

double SparseEngine::timed_steps(int n, double* boundary_ms, double* light_ms) {
    std::vector<cudaEvent_t> ev(4 * std::size_t(n) + 2);
    for (auto& e : ev) VOXL_CUDA(cudaEventCreate(&e));
    VOXL_CUDA(cudaEventRecord(ev[4 * n], stream_));
    for (int i = 0; i < n; ++i) launch(0, &ev[4 * i], &ev[4 * i + 2]);
    VOXL_CUDA(cudaEventRecord(ev[4 * n + 1], stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    double sb = 0, sl = 0;
    for (int i = 0; i < n; ++i) {
        float a = 0, b = 0;
        VOXL_CUDA(cudaEventElapsedTime(&a, ev[4 * i], ev[4 * i + 1]));
        VOXL_CUDA(cudaEventElapsedTime(&b, ev[4 * i + 2], ev[4 * i + 3]));
        sb += a;
        sl += b;
    }
    float total = 0;
    VOXL_CUDA(cudaEventElapsedTime(&total, ev[4 * n], ev[4 * n + 1]));
    for (auto& e : ev) cudaEventDestroy(e);
    if (boundary_ms) *boundary_ms = sb;
    if (light_ms) *light_ms = sl;
    check_errors();
    return total;
}

DenseDiag SparseEngine::probe() {
    // probe_field over canonical_state (solver.cpp:290): sums and max |u| in
    // storage order (block_probe.cuh); the canonical-order kernel only runs
    // to name the first unstable cell when there is one.
    double* partial = d_diag_;
    double* out = d_diag_ + 2 * kSpProbeBlocks;
    auto* bad = reinterpret_cast<unsigned long long*>(out + 2);
    auto* bad_any = reinterpret_cast<unsigned int*>(out + 3);
    VOXL_CUDA(cudaMemsetAsync(out, 0, 4 * sizeof(double), stream_));
    double res[2];
    unsigned int any = 0;
    sparse_dispatch(cfg_.lattice, cfg_.precision, [&](auto ops) {
        using Ops = decltype(ops);
        using L = std::conditional_t<Ops::Q == 19, D3Q19, D3Q27>;
        auto A = Ops::base_args(cfg_);
        using R = std::remove_pointer_t<decltype(A.nxt)>;
        launch_block_probe<L, R>(static_cast<const R*>(buf_[cur_]), d_masks_, grid_.mask_words(),
                                 grid_.block_volume(), grid_.num_blocks(), A.shift, partial, out, bad_any, stream_);
    });
    VOXL_CUDA(cudaMemcpyAsync(res, out, sizeof res, cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaMemcpyAsync(&any, bad_any, sizeof any, cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    DenseDiag d;
    d.mass = res[0];
    d.max_speed = std::sqrt(res[1]);
    if (any) {
        ensure_slots();
        const long long n = grid_.num_active();
        const unsigned long long none = ~0ull;
        VOXL_CUDA(cudaMemcpyAsync(bad, &none, sizeof none, cudaMemcpyHostToDevice, stream_));
        sparse_dispatch(cfg_.lattice, cfg_.precision, [&](auto ops) {
            using Ops = decltype(ops);
            using L = std::conditional_t<Ops::Q == 19, D3Q19, D3Q27>;
            auto A = Ops::base_args(cfg_);
            using R = std::remove_pointer_t<decltype(A.nxt)>;
            sparse_probe_kernel<L, R><<<kSpProbeBlocks, 256, 0, stream_>>>(
                static_cast<const R*>(buf_[cur_]), d_slots_, n, grid_.block_volume(), A, partial, bad);
            VOXL_CUDA(cudaGetLastError());
        });
        unsigned long long b = 0;
        VOXL_CUDA(cudaMemcpyAsync(&b, bad, sizeof b, cudaMemcpyDeviceToHost, stream_));
        VOXL_CUDA(cudaStreamSynchronize(stream_));
        d.unstable = 1;
        d.bad_voxel = std::int64_t(b >> 5);
        d.bad_population = int(b & 31);
    }
    return d;
}

} // namespace voxl_b200
