// multires.cu -- multi-resolution kernels and engine (see multires.cuh).
#include "multires.cuh"
#include "lattice.cuh"
#include "digest.cuh"
#include "canon_io.cuh"
#include "block_probe.cuh"
#include "diag_ring.cuh"
#include "phase_trace.cuh"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <type_traits>

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

enum BlockClass : std::uint8_t { kNone = 0, kUniform = 1, kJump = 2 };
enum TimeClass : int { kTCollide = 0, kTStream = 1, kTFused = 2, kTTransition = 3 };

template <int Q, class R>
struct MresArgs {
    const R* cur;
    R* nxt;
    R* post;
    R* post_ahead;  // kStreamAhead: the other post buffer (next step's jump-block collide)
    double* probe_partial;       // kProbe: (sum f, max |u|^2) per CTA
    unsigned int* probe_bad;     // kProbe: any unstable cell
    int step_probe_base;         // kProbe: first probed block (partial slot 0)
    const std::int32_t* nbr;
    const std::uint64_t* amask;
    const std::uint8_t* cls;
    const int* org;
    int block_begin;              // first block of this launch (blocks are class-ordered)
    const std::uint8_t* full;     // 1 iff every cell of the block is active
    const std::uint64_t* smask;   // solid cells per block (obstacle extension), or null
    const std::uint8_t* nsolid;   // 1 iff some active cell of the block has a solid box neighbour
    int n[3];
    R omega, keep;
    R lid[Q];  // 2 w_j rho0 3 (e_j . u_lid) per pulled direction j (multires.cpp:499-503)
    int has_lid;
    int step;
    int* error_flag;
    // fused probe_field of run_multires (DIAG kernels, a level's last
    // sub-step of the coarse step): accumulator lanes and first-offender word
    // of the step (diag_ring.cuh); canon[slot] = the cell's index in the
    // level's canonical order, cell0 = the level's first canonical cell
    unsigned long long* diag_acc;
    unsigned long long* diag_bad;
    const std::int32_t* canon;
    long long cell0;
};

template <int E>
struct BlockGeom {
    static constexpr int BV = E * E * E;
    static constexpr int W = BV >= 64 ? BV / 64 : 1;
    static constexpr int LOG = E == 8 ? 3 : (E == 4 ? 2 : (E == 2 ? 1 : 0));
    static constexpr int H = (1 << (LOG - 1)) | (1 << (2 * LOG - 1)) | (1 << (3 * LOG - 1));
    static constexpr int LM = (BV - 1) & ~H;
};

/// Neighbour-block index d (0..26) and source local index for the cell at
/// local t shifted by (sx, sy, sz) in {-1, 0, 1}^3 (compile time).
template <int E, int SX, int SY, int SZ>
__device__ __forceinline__ void shifted(int t, bool xlo, bool xhi, bool ylo, bool yhi, bool zlo, bool zhi, int& d,
                                        int& sl) {
    using G = BlockGeom<E>;
    constexpr int D = (SX & (E - 1)) | ((SY & (E - 1)) << G::LOG) | ((SZ & (E - 1)) << (2 * G::LOG));
    sl = ((t & G::LM) + (D & G::LM)) ^ ((t & G::H) ^ (D & G::H));
    d = 13;
    if constexpr (SX < 0) d -= xlo;
    if constexpr (SX > 0) d += xhi;
    if constexpr (SY < 0) d -= 3 * ylo;
    if constexpr (SY > 0) d += 3 * yhi;
    if constexpr (SZ < 0) d -= 9 * zlo;
    if constexpr (SZ > 0) d += 9 * zhi;
}

__device__ __forceinline__ bool bit_of(const unsigned long long* words, int local) {
    return (words[local >> 6] >> (local & 63)) & 1ull;
}

/// collide_level (multires.cpp:443-456): post = BGK(cur) on the listed blocks.
template <class L, class R, bool Exact, int E>
__global__ void __launch_bounds__(E* E* E) mres_collide_kernel(const __grid_constant__ MresArgs<L::Q, R> A) {
    constexpr int Q = L::Q, BV = E * E * E, W = BlockGeom<E>::W;
    const int b = A.block_begin + int(blockIdx.x);
    const int t = threadIdx.x;
    if (!((A.amask[(long long)b * W + (t >> 6)] >> (t & 63)) & 1ull)) return;
    const long long base = (long long)b * Q * BV + t;
    R f[Q];
    static_for<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        f[i] = __ldg(A.cur + base + i * BV);
    });
    bool ok = true;
    R rho, u[3];
    if constexpr (Exact) bgk_relax<L, R, true>(f, A.omega, A.keep, rho, u, ok);
    else bgk_relax_shifted<L, R>(f, A.omega, A.keep, rho, u, ok);
    if (!ok) atomicMin(A.error_flag, A.step);
    static_for<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        A.post[base + i * BV] = f[i];
    });
}

/// Pull (+ optional collide) over the listed blocks: g_i(v) = src[v - e_i][i]
/// for in-domain sources (active, ghost or ring slots of the post buffer --
/// every one exists by construction, so no activity test is needed), own
/// src[v][opp i] plus the lid term for wall sources (stream_voxel,
/// multires.cpp:485-531). MODE kStream: stream_level (write g). MODE kFused:
/// the fused uniform-block kernel (uniform blocks keep post-collision
/// storage, so collide-after-pull is the reference's collide-before-pull of
/// the next step), one pass at 2 Q sizeof(real) bytes per update. MODE
/// kStreamAhead: the fused-mode jump-block stream -- writes g (the next cur,
/// which explosion/coalescence and readout need) and also BGK(g) into the
/// other post buffer, i.e. the next step's collide_level of the jump blocks
/// (multires.cpp:443-456), so fused mode launches no separate collide.
constexpr int kStream = 0, kFused = 1, kStreamAhead = 2, kProbe = 3;

/// kProbe: probe_field terms (lbm.cpp:116-138) of the pulled pre-collision
/// state, with block_probe_kernel's per-cell arithmetic (block_probe.cuh).
struct ProbeAcc {
    double mass = 0.0, vmax = 0.0;
    bool bad = false;
};

/// DIAG: the probe_field terms of one pulled cell (probe_first_bad /
/// probe_moments, lattice.cuh) in the precision the collision forms them.
template <class R, bool Exact>
struct DiagCell {
    using P = std::conditional_t<Exact || sizeof(R) == 8, double, float>;
    P m = P(0), v = P(0);
    int bad = -1;
};

template <class L, class R, bool Exact, int E, int MODE, bool INNER, bool SOLID, bool DIAG = false>
__device__ __forceinline__ void mres_pull_body(const MresArgs<L::Q, R>& A, int b, int t, const R* const* s_src,
                                               ProbeAcc* acc = nullptr, DiagCell<R, Exact>* dc = nullptr);

/// CTAs per block: 8^3 blocks are split over two 256-thread CTAs (6 CTAs / SM
/// at 40 registers), so each CTA's metadata prologue hides behind five others.
template <int E>
constexpr int kSplit = E == 8 ? 2 : 1;

/// SOLID: the level has obstacle cells (a separate instantiation, so grids
/// without them keep the register budget of the plain kernel).
template <class L, class R, bool Exact, int E, int MODE, bool SOLID, bool DIAG = false>
__global__ void __launch_bounds__(E* E* E / kSplit<E>, (E == 8 && sizeof(R) == 4) ? block_min_ctas(L::Q) : 1)
    mres_pull_kernel(const __grid_constant__ MresArgs<L::Q, R> A) {
    constexpr int Q = L::Q, BV = E * E * E, W = BlockGeom<E>::W, S = kSplit<E>;
    __shared__ const R* s_src[27];
    __shared__ int s_inner, s_full, s_solid;
    const int b = A.block_begin + int(blockIdx.x) / S;
    const int tid = threadIdx.x;
    const int t = tid + (int(blockIdx.x) % S) * (BV / S);  // local voxel index in the block
    if (tid < 27) {
        const int nb = A.nbr[(long long)b * 27 + tid];
        s_src[tid] = A.post + (long long)(nb < 0 ? b : nb) * Q * BV;
    }
    // metadata loads in different warps so their latencies overlap (E = 4
    // runs 64-thread CTAs: stay below 64 there)
    if (tid == 32) {
        // block strictly inside the level domain: no pull can leave it
        const int* o = A.org + 3 * b;
        s_inner = o[0] > 0 && o[1] > 0 && o[2] > 0 && o[0] + E < A.n[0] && o[1] + E < A.n[1] && o[2] + E < A.n[2];
    }
    if (tid == (BV / S > 64 ? 64 : 33)) s_full = A.full[b];
    if constexpr (SOLID) {
        if (tid == (BV / S > 64 ? 96 : 34)) s_solid = A.nsolid[b];
    }
    __syncthreads();
    const bool active = s_full || ((A.amask[(long long)b * W + (t >> 6)] >> (t & 63)) & 1ull);
    if constexpr (MODE != kProbe && DIAG) {
        // fused probe_field: every thread reaches the warp reduction; the
        // warp's mass and max |u|^2 go into the step's accumulator lanes
        // (order-independent integer sums, diag_ring.cuh), the first
        // offender into the step's bad word by canonical index
        DiagCell<R, Exact> dc;
        if (active) {
            if (SOLID && s_solid) mres_pull_body<L, R, Exact, E, MODE, false, SOLID, true>(A, b, t, s_src, nullptr, &dc);
            else if (s_inner) mres_pull_body<L, R, Exact, E, MODE, true, false, true>(A, b, t, s_src, nullptr, &dc);
            else mres_pull_body<L, R, Exact, E, MODE, false, false, true>(A, b, t, s_src, nullptr, &dc);
            if (dc.bad >= 0) {
                const long long canon = A.cell0 + A.canon[(long long)b * (E * E * E) + t];
                atomicMin(A.diag_bad, ((unsigned long long)canon << 5) | (unsigned long long)dc.bad);
            }
        }
        using P = typename DiagCell<R, Exact>::P;
        P pm = dc.m, pv = dc.v;
        const unsigned live = __ballot_sync(0xffffffffu, active);
        const unsigned long long warp_id = (unsigned long long)blockIdx.x * (E * E * E / S / 32) + (tid >> 5);
        if constexpr (std::is_same_v<P, float>) {
            diag_warp_commit_f32<VOXL_BLOCK_DIAG_UNCOND != 0, VOXL_BLOCK_DIAG_POLICY != 0>(A.diag_acc, warp_id, pm, pv, live);
        } else {
            for (int o = 16; o > 0; o >>= 1) {
                pm += __shfl_xor_sync(0xffffffffu, pm, o);
                pv = max(pv, __shfl_xor_sync(0xffffffffu, pv, o));
            }
            if ((tid & 31) == 0 && live) diag_commit(A.diag_acc, warp_id, double(pm), double(pv));
        }
    } else if constexpr (MODE != kProbe) {
        if (!active) return;
        if constexpr (SOLID) {
            if (s_solid) {
                mres_pull_body<L, R, Exact, E, MODE, false, true>(A, b, t, s_src);
                return;
            }
        }
        if (s_inner) mres_pull_body<L, R, Exact, E, MODE, true, false>(A, b, t, s_src);
        else mres_pull_body<L, R, Exact, E, MODE, false, false>(A, b, t, s_src);
    } else {
        // every thread reaches the CTA reduction; partial slot = CTA index
        // from the first probed block (fixed grid, fixed tree: deterministic)
        ProbeAcc acc;
        if (active) {
            if (SOLID && s_solid) mres_pull_body<L, R, Exact, E, MODE, false, SOLID>(A, b, t, s_src, &acc);
            else if (s_inner) mres_pull_body<L, R, Exact, E, MODE, true, false>(A, b, t, s_src, &acc);
            else mres_pull_body<L, R, Exact, E, MODE, false, false>(A, b, t, s_src, &acc);
        }
        if (acc.bad) atomicOr(A.probe_bad, 1u);
        constexpr int NT = BV / S;
        __shared__ double sm[NT], sv[NT];
        sm[tid] = acc.mass;
        sv[tid] = acc.vmax;
        __syncthreads();
        for (int w = NT / 2; w > 0; w >>= 1) {
            if (tid < w) {
                sm[tid] += sm[tid + w];
                sv[tid] = fmax(sv[tid], sv[tid + w]);
            }
            __syncthreads();
        }
        if (tid == 0) {
            const long long slot = (long long)(b - A.step_probe_base) * S + int(blockIdx.x) % S;
            A.probe_partial[2 * slot] = sm[0];
            A.probe_partial[2 * slot + 1] = sv[0];
        }
    }
}

/// Pull over blocks [begin, begin + count): the part below `n_plain` (blocks
/// that cannot see a solid cell) runs the plain kernel, the rest the
/// solid-aware one when the level has obstacle cells.
template <class L, class R, bool Exact, int E, int MODE, bool DIAG = false>
void launch_pull(MresArgs<L::Q, R> A, int begin, int count, int n_plain, cudaStream_t st) {
    const dim3 block(E * E * E / kSplit<E>);
    const int split = std::min(begin + count, std::max(begin, n_plain));
    const std::uint8_t* ns = A.nsolid;
    if (split > begin) {
        A.block_begin = begin;
        A.nsolid = nullptr;
        mres_pull_kernel<L, R, Exact, E, MODE, false, DIAG><<<(split - begin) * kSplit<E>, block, 0, st>>>(A);
    }
    if (begin + count > split) {
        A.block_begin = split;
        A.nsolid = ns;
        if (ns)
            mres_pull_kernel<L, R, Exact, E, MODE, true, DIAG><<<(begin + count - split) * kSplit<E>, block, 0, st>>>(A);
        else
            mres_pull_kernel<L, R, Exact, E, MODE, false, DIAG><<<(begin + count - split) * kSplit<E>, block, 0, st>>>(A);
    }
}

/// launch_pull with the fused probe when `diag` is set (run_multires's
/// per-step row, taken by a level's last sub-step of the coarse step).
template <class L, class R, bool Exact, int E, int MODE>
void launch_pull_diag(MresArgs<L::Q, R> A, int begin, int count, int n_plain, cudaStream_t st,
                      const DiagTarget* diag, const std::int32_t* canon, long long cell0) {
    if (!diag) return launch_pull<L, R, Exact, E, MODE>(A, begin, count, n_plain, st);
    A.diag_acc = diag->acc;
    A.diag_bad = diag->bad;
    A.canon = canon;
    A.cell0 = cell0;
    launch_pull<L, R, Exact, E, MODE, true>(A, begin, count, n_plain, st);
}

template <class L, class R, bool Exact, int E, int MODE, bool INNER, bool SOLID, bool DIAG>
__device__ __forceinline__ void mres_pull_body(const MresArgs<L::Q, R>& A, int b, int t, const R* const* s_src,
                                               ProbeAcc* acc, DiagCell<R, Exact>* dc) {
    constexpr int Q = L::Q, BV = E * E * E;
    using Ar = Arith<R, Exact>;
    constexpr int LOG = BlockGeom<E>::LOG;
    const int lx = t & (E - 1), ly = (t >> LOG) & (E - 1), lz = t >> (2 * LOG);
    const int x = A.org[3 * b] + lx, y = A.org[3 * b + 1] + ly, z = A.org[3 * b + 2] + lz;
    const bool xlo = lx == 0, xhi = lx == E - 1, ylo = ly == 0, yhi = ly == E - 1, zlo = lz == 0, zhi = lz == E - 1;
    const bool dxlo = x == 0, dxhi = x == A.n[0] - 1, dylo = y == 0, dyhi = y == A.n[1] - 1, dzlo = z == 0,
               dzhi = z == A.n[2] - 1;
    const R* own_src = s_src[13] + t;
    R g[Q];
    static_for<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int ex = L::ex(i), ey = L::ey(i), ez = L::ez(i);
        constexpr int oi = L::opp(i);
        int d, sl;
        shifted<E, -ex, -ey, -ez>(t, xlo, xhi, ylo, yhi, zlo, zhi, d, sl);
        if constexpr (INNER) {
            g[i] = __ldg(s_src[d] + (i * BV + sl));
        } else {
            bool oob = false;
            if constexpr (ex > 0) oob = oob || dxlo;
            if constexpr (ex < 0) oob = oob || dxhi;
            if constexpr (ey > 0) oob = oob || dylo;
            if constexpr (ey < 0) oob = oob || dyhi;
            if constexpr (ez > 0) oob = oob || dzlo;
            if constexpr (ez < 0) oob = oob || dzhi;
            if constexpr (SOLID && (ex != 0 || ey != 0 || ez != 0)) {
                // obstacle cells bounce back like the walls; a source block
                // missing from the extended grid can only be all-solid there
                if (!oob) {
                    const int nb = A.nbr[(long long)b * 27 + d];
                    oob = nb < 0 || ((A.smask[(long long)nb * BlockGeom<E>::W + (sl >> 6)] >> (sl & 63)) & 1ull);
                }
            }
            const R* p = oob ? own_src + oi * BV : s_src[d] + (i * BV + sl);
            R v = __ldg(p);
            // lid on the max face of the partition axis (rules_for,
            // solver.cpp:150-163): z in 3D, y in 2D
            if constexpr ((L::dim == 3 ? ez : ey) < 0) {
                if (A.has_lid && (L::dim == 3 ? dzhi : dyhi)) v = Ar::add(v, A.lid[i]);
            }
            g[i] = v;
        }
    });
    if constexpr (MODE == kProbe) {
        // the uniform cell's pre-collision state, exactly what gather_uniform
        // would store in cur, reduced instead of written
        double r = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
        bool bh = false;
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            const double fi = double(g[i]) + (Exact ? 0.0 : L::w(i));
            bh = bh || !(fabs(fi) <= 1e3);
            r += fi;
            mx = acc_term<double, false, L::ex(i)>(mx, fi);
            my = acc_term<double, false, L::ey(i)>(my, fi);
            mz = acc_term<double, false, L::ez(i)>(mz, fi);
        });
        acc->mass += r;
        if (bh || !(r > 0.0)) {
            acc->bad = true;
        } else {
            const double ux = mx / r, uy = my / r, uz = mz / r;
            acc->vmax = fmax(acc->vmax, ux * ux + uy * uy + uz * uz);
        }
        return;
    }
    // DIAG: g is the level's cur after this sub-step (the reference's state
    // that probe_field reads): the population test runs before the
    // collision overwrites g, the moments come from the collision
    int dbad = -1;
    if constexpr (DIAG) dbad = probe_first_bad<L, R, Exact>(g);
    if constexpr (DIAG && MODE == kStream) {
        R rho, dr, u[3];
        pulled_moments<L, R, Exact>(g, rho, dr, u);
        probe_moments<L, R, Exact>(dbad, rho, dr, u, dc->m, dc->v, dc->bad);
    }
    auto collide = [&] {
        bool ok = true;
        R rho, u[3], dr = R(0);
        if constexpr (Exact) bgk_relax<L, R, true>(g, A.omega, A.keep, rho, u, ok);
        else bgk_relax_shifted<L, R>(g, A.omega, A.keep, rho, u, ok, DIAG ? &dr : nullptr);
        if (!ok) atomicMin(A.error_flag, A.step);
        if constexpr (DIAG && MODE != kStream) probe_moments<L, R, Exact>(dbad, rho, dr, u, dc->m, dc->v, dc->bad);
    };
    if constexpr (MODE == kFused) collide();
    const long long cell = (long long)b * Q * BV + t;
    static_for<Q>([&](auto I) {
        constexpr int i = decltype(I)::value;
        A.nxt[cell + i * BV] = g[i];
    });
    if constexpr (MODE == kStreamAhead) {
        collide();
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            A.post_ahead[cell + i * BV] = g[i];
        });
    }
}

/// explode (multires.cpp:458-467): ghost cells of the fine level <- the
/// post-collision populations of their parent, a plain copy. One launch fills
/// both fine post parities in fused mode (one explosion serves both fine
/// sub-steps, multires.cpp:563-570). One thread per (population, ghost),
/// population-major so a warp's stores of one population are contiguous: the
/// launch is a few MB, so it is latency-bound and wants every load in flight
/// at once (a thread-per-ghost loop over Q serialises 19 load/store round
/// trips). Slot -> element offsets use shifts: the block volume E^3 is a power
/// of two (64-bit division is ~100 instructions).
template <int Q, class R>
__global__ void mres_explode_kernel(R* __restrict__ fine_a, R* __restrict__ fine_b,
                                    const R* __restrict__ coarse_post, const std::int64_t* __restrict__ dst,
                                    const std::int64_t* __restrict__ src, int n, int lb) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n * Q) return;
    const int c = int(t / n), g = int(t - (long long)c * n);
    const long long bv = 1ll << lb, ds = __ldg(dst + g), ss = __ldg(src + g);
    const long long dbase = ((ds >> lb) * Q << lb) + (ds & (bv - 1)) + c * bv;
    const long long sbase = ((ss >> lb) * Q << lb) + (ss & (bv - 1)) + c * bv;
    const R v = __ldg(coarse_post + sbase);
    fine_a[dbase] = v;
    if (fine_b) fine_b[dbase] = v;
}

/// coalesce (multires.cpp:469-483): ring(l) <- mean of the 8 children's
/// current (post-stream) populations, children_of order, sum * (1/8). One
/// thread per (population, ring cell), the children summed in order.
template <int Q, class R, bool Exact>
__global__ void mres_coalesce_kernel(R* __restrict__ coarse_post, const R* __restrict__ fine_cur,
                                     const std::int64_t* __restrict__ dst, const std::int64_t* __restrict__ child,
                                     int n, int lbc, int lbf, int nchild) {
    using A = Arith<R, Exact>;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)n * Q) return;
    const int c = int(t / n), g = int(t - (long long)c * n);
    const long long bvc = 1ll << lbc, bvf = 1ll << lbf, ds = __ldg(dst + g);
    const long long dbase = ((ds >> lbc) * Q << lbc) + (ds & (bvc - 1)) + c * bvc;
    R v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k < nchild) {
            const long long cs = __ldg(child + (long long)g * 8 + k);
            v[k] = __ldg(fine_cur + ((cs >> lbf) * Q << lbf) + (cs & (bvf - 1)) + c * bvf);
        }
    }
    const R scale = R(1.0 / double(nchild));
    R sum = R(0);
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (k < nchild) sum = A::add(sum, v[k]);
    coarse_post[dbase] = A::mul(sum, scale);
}

/// probe_field (lbm.cpp:116-138) and total_mass (multires.cpp:600-609) on
/// the device, over one level's cells in canonical order (slots[v]), read
/// straight from the state buffer (fp64 value = storage + shift, exactly the
/// canonical_state value): per-CTA partial sums of the populations and max |u|
/// (u = m / rho, true division, as macroscopic lattice.cpp:115-129), the
/// first unstable (cell, population) by atomicMin. Fixed grid and fixed
/// reduction order, so the result is run-to-run deterministic.
constexpr int kMresProbeBlocks = 296;

template <class L, class R>
__global__ void __launch_bounds__(256) mres_slot_probe_kernel(const R* cur, const std::int64_t* slots, long long n,
                                                              int lb, const __grid_constant__ ShiftQ<L::Q> sh,
                                                              long long cell0, double* partial,
                                                              unsigned long long* bad) {
    constexpr int Q = L::Q;
    double mass = 0.0, vmax = 0.0;
    const long long bv = 1ll << lb;
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        const long long slot = slots[v];
        const R* f = cur + ((slot >> lb) * Q << lb) + (slot & (bv - 1));
        R raw[Q];
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            raw[i] = f[i * bv];
        });
        double r = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
        int bp = -1;
        static_for<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            const double fi = double(raw[i]) + sh.v[i];
            if (bp < 0 && !(fabs(fi) <= 1e3)) bp = i;
            r += fi;
            mx = acc_term<double, false, L::ex(i)>(mx, fi);
            my = acc_term<double, false, L::ey(i)>(my, fi);
            mz = acc_term<double, false, L::ez(i)>(mz, fi);
        });
        mass += r;
        if (bp >= 0 || !(r > 0.0)) {
            atomicMin(bad, ((unsigned long long)(cell0 + v) << 5) | (unsigned long long)(bp < 0 ? kBadDensity : bp));
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
    if (threadIdx.x == 0) {  // accumulated over the staging chunks of a level, in chunk order
        partial[2 * blockIdx.x] += sm[0];
        partial[2 * blockIdx.x + 1] = fmax(partial[2 * blockIdx.x + 1], sv[0]);
    }
}

/// out = {sum of all cells, max |u|, sum_l 8^l * level sum (total_mass)}.
__global__ void mres_probe_final(const double* partial, int levels, int per, double child, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double all = 0.0, v = 0.0, weighted = 0.0, vol = 1.0;
    for (int l = 0; l < levels; ++l) {
        double lev = 0.0;
        for (int i = 0; i < per; ++i) {
            lev += partial[2 * (l * per + i)];
            v = fmax(v, partial[2 * (l * per + i) + 1]);
        }
        all += lev;
        weighted += lev * vol;
        vol *= child;
    }
    out[0] = all;
    out[1] = v;
    out[2] = weighted;
}

template <class R>
__global__ void mres_fill_kernel(R* buf, long long total, int bv, int q, const double* val) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    buf[e] = R(val[int((e / bv) % q)]);
}

template <class F>
void mres_dispatch(int lattice, Precision prec, int edge, F&& f) {
    auto by_edge = [&](auto lat, auto real, auto exact) {
        using L = decltype(lat);
        using R = decltype(real);
        if (edge == 8) f(L{}, R{}, exact, std::integral_constant<int, 8>{});
        else if (edge == 4) f(L{}, R{}, exact, std::integral_constant<int, 4>{});
        else throw std::invalid_argument("multires engine: block edge must be 4 or 8");
    };
    auto by_prec = [&](auto lat) {
        if (prec == Precision::F64) by_edge(lat, double{}, std::true_type{});
        else by_edge(lat, float{}, std::false_type{});
    };
    switch (lattice) {
        case kD2Q9: by_prec(D2Q9{}); break;  // nz = 1: the z = 0 layer of E^3 blocks
        case kD3Q19: by_prec(D3Q19{}); break;
        case kD3Q27: by_prec(D3Q27{}); break;
        default: throw std::invalid_argument("multires engine: unknown lattice");
    }
}

/// Population count as a compile-time constant for the Q-templated helpers
/// (canonical I/O, transitions): D2Q9, D3Q19, D3Q27.
template <class F>
void q_dispatch(int q, F&& f) {
    switch (q) {
        case 9: f(std::integral_constant<int, 9>{}); break;
        case 19: f(std::integral_constant<int, 19>{}); break;
        case 27: f(std::integral_constant<int, 27>{}); break;
        default: throw std::invalid_argument("multires engine: unsupported population count");
    }
}

inline std::int64_t lin3(const std::array<int, 3>& d, int x, int y, int z) {
    return (std::int64_t(z) * d[1] + y) * d[0] + x;
}

/// 26-neighbourhood dilation of a byte mask (separable max filter).
std::vector<std::uint8_t> box_dilate(const std::vector<std::uint8_t>& m, const std::array<int, 3>& d) {
    std::vector<std::uint8_t> a = m, b(m.size());
    for (int axis = 0; axis < 3; ++axis) {
        const std::int64_t stride = axis == 0 ? 1 : (axis == 1 ? d[0] : std::int64_t(d[0]) * d[1]);
        for (int z = 0; z < d[2]; ++z)
            for (int y = 0; y < d[1]; ++y)
                for (int x = 0; x < d[0]; ++x) {
                    const std::int64_t i = lin3(d, x, y, z);
                    const int c = axis == 0 ? x : (axis == 1 ? y : z);
                    std::uint8_t v = a[i];
                    if (c > 0) v |= a[i - stride];
                    if (c + 1 < d[axis]) v |= a[i + stride];
                    b[i] = v;
                }
        std::swap(a, b);
    }
    return a;
}

} // namespace

struct MultiResEngine::Level {
    std::array<int, 3> n{1, 1, 1};
    BlockGrid ext;
    void* cur = nullptr;
    void* nxt = nullptr;
    // post[parity]: post-collision of jump / staged cells (this step), of
    // uniform cells (fused mode: their persistent state), ghost and ring slots.
    void* post[2] = {nullptr, nullptr};
    int parity = 0;
    std::int32_t* nbr = nullptr;
    std::uint64_t* amask = nullptr;
    std::uint8_t* cls = nullptr;
    std::uint8_t* full = nullptr;
    std::uint64_t* smask = nullptr;  // obstacle extension: solid cells per block
    std::uint8_t* nsolid = nullptr;  // per block: an active cell has a solid box neighbour
    int* org = nullptr;
    int* all_blocks = nullptr;
    int* uni_blocks = nullptr;
    int* jump_blocks = nullptr;
    int n_all = 0, n_uni = 0, n_jump = 0;
    int n_plain = 0;  // blocks [0, n_plain) are uniform and never pull from a solid cell
    std::int64_t* explode_dst = nullptr;  // ghost cells of this level
    std::int64_t* explode_src = nullptr;  // parent slots at level + 1
    int n_ghost = 0;
    std::int64_t* coal_dst = nullptr;    // ring cells of this level
    std::int64_t* coal_child = nullptr;  // 8 child slots at level - 1
    int n_ring = 0;
    std::int64_t* slots = nullptr;
    std::int64_t n_active = 0;
    std::int32_t* canon = nullptr;  // slot -> canonical index in the level (built by the first probed step)
    long long cell0 = 0;            // canonical index of the level's first cell (levels finest first)
    double inv_tau = 1.0;
    std::int64_t slot(int x, int y, int z) const {
        const int e = ext.edge();
        const int b = ext.find_block(x / e, y / e, z / e);
        if (b < 0) return -1;
        const int local = ((z % e) * e + (y % e)) * e + (x % e);
        return std::int64_t(b) * ext.block_volume() + local;
    }
};

MultiResEngine::MultiResEngine(const MresConfig& cfg, const std::int32_t* level_map)
    : cfg_(cfg), io_(std::make_unique<CanonPipe>()) {
    if (cfg_.lattice != kD2Q9 && cfg_.lattice != kD3Q19 && cfg_.lattice != kD3Q27)
        throw std::invalid_argument("multires engine: unknown lattice");
    if (cfg_.edge != 4 && cfg_.edge != 8) throw std::invalid_argument("multires engine: block edge must be 4 or 8");
    const LatticeTable lat = make_lattice(cfg_.lattice);
    q_ = lat.q;
    esize_ = cfg_.precision == Precision::F64 ? 8 : 4;
    grid_ = MresGrid::build(cfg_.domain, cfg_.levels, cfg_.lattice, level_map, cfg_.tau, cfg_.reference_tables,
                            cfg_.allow_solid);
    const int L = grid_.num_levels();
    const int E = cfg_.edge;
    for (int l = 0; l < L; ++l) {
        const MresLevel& G = grid_.level(l);
        if (!(G.tau > 0.5)) throw std::invalid_argument("multires: derived tau must stay > 0.5");
    }
    VOXL_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    {
        int lo = 0, hi = 0;
        VOXL_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        VOXL_CUDA(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, hi));
        VOXL_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        VOXL_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    }
    std::vector<std::vector<std::uint8_t>> ghost(L), ring(L);
    for (int l = 0; l < L; ++l) {
        const MresLevel& G = grid_.level(l);
        const auto& d = G.domain;
        const std::size_t vol = G.active.size();
        const auto near = box_dilate(G.active, d);
        ghost[l].assign(vol, 0);
        ring[l].assign(vol, 0);
        std::vector<std::uint8_t> other(vol, 0);
        for (std::size_t i = 0; i < vol; ++i) {
            other[i] = !G.active[i] && (G.refined[i] || G.under_coarse[i]);
            if (!near[i] || G.active[i] || (!G.solid.empty() && G.solid[i])) continue;
            if (G.under_coarse[i]) ghost[l][i] = 1;
            else if (!G.refined[i])
                throw std::invalid_argument("multires: active region has an uncovered neighbor");
        }
        // refined ring: refined cells an active cell pulls from along a lattice direction
        for (int z = 0; z < d[2]; ++z)
            for (int y = 0; y < d[1]; ++y)
                for (int x = 0; x < d[0]; ++x) {
                    const std::int64_t i = lin3(d, x, y, z);
                    if (!near[i] || G.active[i] || !G.refined[i]) continue;
                    for (int q = 0; q < lat.q && !ring[l][i]; ++q) {
                        const int a = x + lat.e[q][0], b = y + lat.e[q][1], c = z + lat.e[q][2];
                        if (a < 0 || b < 0 || c < 0 || a >= d[0] || b >= d[1] || c >= d[2]) continue;
                        if (G.active[lin3(d, a, b, c)]) ring[l][i] = 1;
                    }
                }
        const auto crossing_near = box_dilate(other, d);
        Level* V = new Level;
        lv_.push_back(V);
        V->n = d;
        V->n_active = G.num_active;
        V->inv_tau = 1.0 / G.tau;
        std::vector<std::uint8_t> ext(vol);
        for (std::size_t i = 0; i < vol; ++i) ext[i] = G.active[i] | ghost[l][i] | ring[l][i];
        V->ext = BlockGrid::build(d, ext.data(), E);
        const int nb = V->ext.num_blocks(), W = V->ext.mask_words(), BV = V->ext.block_volume();
        // Per-block fusion class, then the disaggregated order (the paper's
        // DisagMem idea applied to multires): uniform blocks first, then jump
        // blocks, then ghost/ring-only blocks -- each launch covers one
        // contiguous range, so a CTA indexes its block directly.
        auto classify = [&](const BlockGrid& bg, int b, std::uint64_t* mask_out, bool* full_out) {
            const auto& o = bg.blocks()[b].origin;
            bool any = false, cross = false, full = true;
            for (int local = 0; local < BV; ++local) {
                const int x = o[0] + local % E, y = o[1] + (local / E) % E, z = o[2] + local / (E * E);
                if (x >= d[0] || y >= d[1] || z >= d[2]) {
                    full = false;
                    continue;
                }
                const std::int64_t i = lin3(d, x, y, z);
                if (!G.active[i]) {
                    full = false;
                    continue;
                }
                any = true;
                if (mask_out) mask_out[local >> 6] |= 1ull << (local & 63);
                if (crossing_near[i]) cross = true;
            }
            if (full_out) *full_out = full;
            return any ? (cross ? kJump : kUniform) : kNone;
        };
        // obstacle extension: does an active cell of the block have a solid box
        // neighbour (the only blocks that need the solid-aware pull)?
        const std::vector<std::uint8_t> near_solid =
            G.solid.empty() ? std::vector<std::uint8_t>() : box_dilate(G.solid, d);
        auto touches_solid = [&](const BlockGrid& bg, int b) {
            if (near_solid.empty()) return false;
            const auto& o = bg.blocks()[b].origin;
            for (int local = 0; local < BV; ++local) {
                const int x = o[0] + local % E, y = o[1] + (local / E) % E, z = o[2] + local / (E * E);
                if (x >= d[0] || y >= d[1] || z >= d[2]) continue;
                const std::int64_t i = lin3(d, x, y, z);
                if (G.active[i] && near_solid[i]) return true;
            }
            return false;
        };
        {
            // order: uniform, uniform next to a solid, jump, ghost/ring-only
            std::vector<int> perm(nb), rk(nb);
            for (int b = 0; b < nb; ++b) {
                perm[b] = b;
                const auto c = classify(V->ext, b, nullptr, nullptr);
                rk[b] = c == kUniform ? (touches_solid(V->ext, b) ? 1 : 0) : (c == kJump ? 2 : 3);
            }
            std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return rk[x] < rk[y]; });
            V->n_plain = int(std::count(rk.begin(), rk.end(), 0));
            V->ext.permute(perm);
        }
        const BlockGrid& bg = V->ext;
        std::vector<std::uint64_t> am(std::size_t(nb) * W, 0);
        std::vector<std::uint8_t> cls(nb, kNone), full(nb, 0);
        std::vector<int> org(std::size_t(nb) * 3), all, uni, jmp;
        for (int b = 0; b < nb; ++b) {
            const auto& o = bg.blocks()[b].origin;
            for (int a = 0; a < 3; ++a) org[std::size_t(b) * 3 + a] = o[a];
            bool f = false;
            cls[b] = classify(bg, b, &am[std::size_t(b) * W], &f);
            full[b] = f;
            if (cls[b] != kNone) {
                all.push_back(b);
                (cls[b] == kJump ? jmp : uni).push_back(b);
            }
        }
        VOXL_CUDA(cudaMalloc(&V->full, std::max(1, nb)));
        VOXL_CUDA(cudaMemcpy(V->full, full.data(), nb, cudaMemcpyHostToDevice));
        if (!G.solid.empty()) {
            // obstacle extension: solid bits per ext block, and the per-block
            // flag of the solid-aware pull
            std::vector<std::uint64_t> sm(std::size_t(nb) * W, 0);
            std::vector<std::uint8_t> ns(nb, 0);
            for (int b = 0; b < nb; ++b) {
                const auto& o = bg.blocks()[b].origin;
                ns[b] = touches_solid(bg, b);
                for (int local = 0; local < BV; ++local) {
                    const int x = o[0] + local % E, y = o[1] + (local / E) % E, z = o[2] + local / (E * E);
                    if (x >= d[0] || y >= d[1] || z >= d[2]) continue;
                    if (G.solid[lin3(d, x, y, z)]) sm[std::size_t(b) * W + (local >> 6)] |= 1ull << (local & 63);
                }
            }
            VOXL_CUDA(cudaMalloc(&V->smask, sm.size() * sizeof(std::uint64_t)));
            VOXL_CUDA(cudaMemcpy(V->smask, sm.data(), sm.size() * sizeof(std::uint64_t), cudaMemcpyHostToDevice));
            VOXL_CUDA(cudaMalloc(&V->nsolid, std::max(1, nb)));
            VOXL_CUDA(cudaMemcpy(V->nsolid, ns.data(), nb, cudaMemcpyHostToDevice));
        }
        V->n_all = int(all.size());
        V->n_uni = int(uni.size());
        V->n_jump = int(jmp.size());
        auto up_i32 = [&](const std::vector<int>& v, int** dst) {
            VOXL_CUDA(cudaMalloc(dst, std::max<std::size_t>(1, v.size()) * sizeof(int)));
            if (!v.empty()) VOXL_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
        };
        up_i32(all, &V->all_blocks);
        up_i32(uni, &V->uni_blocks);
        up_i32(jmp, &V->jump_blocks);
        up_i32(org, &V->org);
        const auto nbr = bg.neighbour_table();
        VOXL_CUDA(cudaMalloc(&V->nbr, nbr.size() * sizeof(std::int32_t)));
        VOXL_CUDA(cudaMemcpy(V->nbr, nbr.data(), nbr.size() * sizeof(std::int32_t), cudaMemcpyHostToDevice));
        VOXL_CUDA(cudaMalloc(&V->amask, am.size() * sizeof(std::uint64_t)));
        VOXL_CUDA(cudaMemcpy(V->amask, am.data(), am.size() * sizeof(std::uint64_t), cudaMemcpyHostToDevice));
        VOXL_CUDA(cudaMalloc(&V->cls, nb));
        VOXL_CUDA(cudaMemcpy(V->cls, cls.data(), nb, cudaMemcpyHostToDevice));
        const std::size_t bytes = std::size_t(nb) * q_ * BV * esize_;
        for (void** p : {&V->cur, &V->nxt, &V->post[0], &V->post[1]}) {
            VOXL_CUDA(cudaMalloc(p, bytes));
            VOXL_CUDA(cudaMemsetAsync(*p, 0, bytes, stream_));
        }
        // canonical slots: active cells, x slowest, z fastest
        std::vector<std::int64_t> slots;
        slots.reserve(std::size_t(G.num_active));
        for (int x = 0; x < d[0]; ++x)
            for (int y = 0; y < d[1]; ++y)
                for (int z = 0; z < d[2]; ++z)
                    if (G.active[lin3(d, x, y, z)]) slots.push_back(V->slot(x, y, z));
        VOXL_CUDA(cudaMalloc(&V->slots, std::max<std::size_t>(1, slots.size()) * sizeof(std::int64_t)));
        VOXL_CUDA(cudaMemcpy(V->slots, slots.data(), slots.size() * sizeof(std::int64_t), cudaMemcpyHostToDevice));
    }
    // explosion pairs (ghost at l, parent at l+1) and coalescence records
    // (ring at l, children at l-1), now that every level's slots exist.
    const int dim = grid_.dim();
    side_transitions_ = cfg_.fused;
    for (int l = 0; l < L; ++l) {
        const MresLevel& G = grid_.level(l);
        const auto& d = G.domain;
        std::vector<std::int64_t> gd, gs, cd, cc;
        for (int z = 0; z < d[2]; ++z)
            for (int y = 0; y < d[1]; ++y)
                for (int x = 0; x < d[0]; ++x) {
                    const std::int64_t i = lin3(d, x, y, z);
                    if (ghost[l][i]) {
                        gd.push_back(lv_[l]->slot(x, y, z));
                        gs.push_back(lv_[l + 1]->slot(x >> 1, y >> 1, dim == 3 ? z >> 1 : z));
                    }
                    if (ring[l][i]) {
                        cd.push_back(lv_[l]->slot(x, y, z));
                        const int zhi = dim == 3 ? 1 : 0;
                        int k = 0;
                        for (int dz = 0; dz <= zhi; ++dz)
                            for (int dy = 0; dy <= 1; ++dy)
                                for (int dx = 0; dx <= 1; ++dx, ++k) {
                                    const int cz = dim == 3 ? 2 * z + dz : z;
                                    const std::int64_t s = lv_[l - 1]->slot(2 * x + dx, 2 * y + dy, cz);
                                    if (s < 0 || !grid_.active(l - 1, 2 * x + dx, 2 * y + dy, cz))
                                        throw std::invalid_argument("multires: refined cell with inactive children");
                                    cc.push_back(s);
                                }
                        for (; k < 8; ++k) cc.push_back(cc.back());
                    }
                }
        // Side-stream transitions (fused mode) rely on two facts of the
        // classification (multires.cpp:196-247): a ghost's parent has a
        // refined box neighbour (the parent of the fine cell that pulls from
        // the ghost), so it is a jump cell of level l + 1; and each ring
        // cell's 2^dim children share one even-aligned block with a
        // distance-0 cell, so they lie in a jump block of level l - 1.
        // Checked here; any exception keeps the transitions on the engine
        // stream.
        auto in_jump = [&](const Level* W, std::int64_t slot) {
            const std::int64_t b = slot >> log2_exact(W->ext.block_volume());
            return b >= W->n_uni && b < W->n_all;
        };
        for (const std::int64_t sl : gs)
            if (!in_jump(lv_[l + 1], sl)) side_transitions_ = false;
        for (const std::int64_t sl : cc)
            if (!in_jump(lv_[l - 1], sl)) side_transitions_ = false;
        Level* V = lv_[l];
        V->n_ghost = int(gd.size());
        V->n_ring = int(cd.size());
        auto up64 = [&](const std::vector<std::int64_t>& v, std::int64_t** dst) {
            VOXL_CUDA(cudaMalloc(dst, std::max<std::size_t>(1, v.size()) * sizeof(std::int64_t)));
            if (!v.empty())
                VOXL_CUDA(cudaMemcpy(*dst, v.data(), v.size() * sizeof(std::int64_t), cudaMemcpyHostToDevice));
        };
        up64(gd, &V->explode_dst);
        up64(gs, &V->explode_src);
        up64(cd, &V->coal_dst);
        up64(cc, &V->coal_child);
    }
    VOXL_CUDA(cudaMalloc(&d_error_, sizeof(int)));
    const int big = INT_MAX;
    VOXL_CUDA(cudaMemcpy(d_error_, &big, sizeof(int), cudaMemcpyHostToDevice));
    const double u0[3] = {0.0, 0.0, 0.0};
    set_equilibrium(1.0, u0);  // multires.cpp:574-575
}

MultiResEngine::~MultiResEngine() {
    if (stream_) cudaStreamSynchronize(stream_);
    for (Level* V : lv_) {
        for (void* p : {V->cur, V->nxt, V->post[0], V->post[1]}) cudaFree(p);
        cudaFree(V->nbr);
        cudaFree(V->amask);
        cudaFree(V->cls);
        cudaFree(V->full);
        cudaFree(V->smask);
        cudaFree(V->nsolid);
        cudaFree(V->org);
        cudaFree(V->all_blocks);
        cudaFree(V->uni_blocks);
        cudaFree(V->jump_blocks);
        cudaFree(V->explode_dst);
        cudaFree(V->explode_src);
        cudaFree(V->coal_dst);
        cudaFree(V->coal_child);
        cudaFree(V->slots);
        cudaFree(V->canon);
        delete V;
    }
    cudaFree(d_error_);
    cudaFree(d_diag_);
    cudaFree(probe_scratch_);
    if (side_) {
        cudaStreamSynchronize(side_);
        cudaEventDestroy(ev_fork_);
        cudaEventDestroy(ev_join_);
        cudaStreamDestroy(side_);
    }
    if (stream_) cudaStreamDestroy(stream_);
}

std::int64_t MultiResEngine::state_len() const {
    std::int64_t n = 0;
    for (const Level* V : lv_) n += V->n_active * q_;
    return n;
}

void MultiResEngine::set_equilibrium(double rho, const double u[3]) {
    // set_uniform_equilibrium (multires.cpp:578-587): every slot of cur.
    const LatticeTable t = make_lattice(cfg_.lattice);
    std::vector<double> val(q_);
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int i = 0; i < q_; ++i) {
        const double eu = double(t.e[i][0]) * u[0] + double(t.e[i][1]) * u[1] + double(t.e[i][2]) * u[2];
        const double w = double(t.wnum[i]) / double(t.wden[i]);
        val[i] = w * rho * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * uu) - (esize_ == 8 ? 0.0 : w);
    }
    double* d_val = nullptr;
    VOXL_CUDA(cudaMalloc(&d_val, q_ * sizeof(double)));
    VOXL_CUDA(cudaMemcpy(d_val, val.data(), q_ * sizeof(double), cudaMemcpyHostToDevice));
    for (Level* V : lv_) {
        const long long total = (long long)V->ext.num_blocks() * q_ * V->ext.block_volume();
        for (void* p : {V->cur, V->nxt, V->post[0], V->post[1]}) {
            if (esize_ == 8)
                mres_fill_kernel<double><<<unsigned((total + 255) / 256), 256, 0, stream_>>>(
                    static_cast<double*>(p), total, V->ext.block_volume(), q_, d_val);
            else
                mres_fill_kernel<float><<<unsigned((total + 255) / 256), 256, 0, stream_>>>(
                    static_cast<float*>(p), total, V->ext.block_volume(), q_, d_val);
        }
        VOXL_CUDA(cudaGetLastError());
    }
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(d_val);
    load_uniform_post();
}

void MultiResEngine::set_state(const double* canonical) {
    transfer(const_cast<double*>(canonical), true, nullptr);
    load_uniform_post();
}

void MultiResEngine::get_state(double* canonical) { read_state(canonical, nullptr); }

void MultiResEngine::digest(unsigned long long out[2]) {
    unsigned long long* acc = nullptr;
    VOXL_CUDA(cudaMalloc(reinterpret_cast<void**>(&acc), 2 * sizeof(unsigned long long)));
    VOXL_CUDA(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), stream_));
    read_state(nullptr, acc);
    VOXL_CUDA(cudaMemcpyAsync(out, acc, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    cudaFree(acc);
}

void MultiResEngine::read_state(double* canonical, unsigned long long* digest) {
    // canonical_state (multires.cpp:578-598): levels finest first
    sync_state();
    transfer(canonical, false, digest);
}

void MultiResEngine::transfer(double* host, bool to_device, unsigned long long* digest) {
    // per level, the level's cells through the shared pipeline (canon_io.cuh);
    // device-only gathers feed the digest chunk by chunk
    const LatticeTable t = make_lattice(cfg_.lattice);
    double shift[27] = {};
    for (int i = 0; i < q_; ++i) shift[i] = esize_ == 8 ? 0.0 : double(t.wnum[i]) / double(t.wden[i]);
    const bool wire32 = esize_ == 4 && host != nullptr;
    std::int64_t off = 0;  // canonical element offset of the level
    for (std::size_t l = 0; l < lv_.size(); ++l) {
        Level* V = lv_[l];
        const long long n = V->n_active;
        const int bv = V->ext.block_volume();
        auto layout = [&](long long r0, long long r1, void* slot, bool w32) {
            if (esize_ == 8) {
                q_dispatch(q_, [&](auto QC) {
                    launch_slot_io<decltype(QC)::value, double>(static_cast<double*>(V->cur), slot, w32, V->slots + r0,
                                                                 r1 - r0, bv, shift, to_device, stream_);
                });
            } else {
                q_dispatch(q_, [&](auto QC) {
                    launch_slot_io<decltype(QC)::value, float>(static_cast<float*>(V->cur), slot, w32, V->slots + r0,
                                                                r1 - r0, bv, shift, to_device, stream_);
                });
            }
        };
        auto consume = [&](long long r0, long long r1, void* slot) {
            digest_accumulate(static_cast<const double*>(slot), (r1 - r0) * q_, off + r0 * q_, digest, stream_);
        };
        io_->run(host ? host + off : nullptr, n, 1, q_, to_device, wire32, shift, stream_, layout, consume,
                 digest != nullptr);
        off += n * q_;
    }
    VOXL_CUDA(cudaStreamSynchronize(stream_));
}

void MultiResEngine::mark_begin(int cls, cudaEvent_t* b, cudaStream_t s) {
    // NVTX range per launch class (phase_trace.cuh), closed by mark_end
    static const char* const kNames[] = {"voxl mres collide", "voxl mres stream", "voxl mres fused",
                                         "voxl mres transition"};
    nvtxRangePushA(kNames[cls & 3]);
    if (!events_) return;
    VOXL_CUDA(cudaEventCreate(b));
    VOXL_CUDA(cudaEventRecord(*b, s ? s : stream_));
}

void MultiResEngine::mark_end(int cls, cudaEvent_t b, cudaStream_t s) {
    nvtxRangePop();
    if (!events_) return;
    cudaEvent_t e;
    VOXL_CUDA(cudaEventCreate(&e));
    VOXL_CUDA(cudaEventRecord(e, s ? s : stream_));
    events_->push_back({cls, {b, e}});
}

namespace {

template <class L, class R, bool Exact>
MresArgs<L::Q, R> level_args(const MresConfig& cfg, MultiResEngine::Level* V, int step, int* err) {
    MresArgs<L::Q, R> A{};
    A.cur = static_cast<const R*>(V->cur);
    A.nxt = static_cast<R*>(V->nxt);
    A.post = static_cast<R*>(V->post[V->parity]);
    A.nbr = V->nbr;
    A.amask = V->amask;
    A.cls = V->cls;
    A.org = V->org;
    A.full = V->full;
    A.smask = V->smask;
    A.nsolid = V->nsolid;
    for (int a = 0; a < 3; ++a) A.n[a] = V->n[a];
    const double inv_tau = V->inv_tau;
    A.omega = R(inv_tau);
    A.keep = Exact ? R(1.0 - inv_tau) : R(1) - R(inv_tau);
    for (int i = 0; i < L::Q; ++i) {
        const double eu = double(L::ex(i)) * cfg.lid_u[0] + double(L::ey(i)) * cfg.lid_u[1] +
                          double(L::ez(i)) * cfg.lid_u[2];
        A.lid[i] = R(2.0 * L::w(i) * 1.0 * 3.0 * eu);
    }
    A.has_lid = 1;  // multires runs are lid-driven cavities (solver.cpp:41-42)
    A.step = step;
    A.error_flag = err;
    return A;
}

} // namespace

void MultiResEngine::launch_collide(int l, bool jump_only) {
    Level* V = lv_[l];
    const int nb = jump_only ? V->n_jump : V->n_all;
    if (nb == 0) return;
    cudaEvent_t b{};
    mark_begin(kTCollide, &b);
    mres_dispatch(cfg_.lattice, cfg_.precision, cfg_.edge, [&](auto lat, auto real, auto exact, auto e) {
        using L = decltype(lat);
        using R = decltype(real);
        constexpr bool X = decltype(exact)::value;
        constexpr int E = decltype(e)::value;
        auto A = level_args<L, R, X>(cfg_, V, steps_done_, d_error_);
        A.block_begin = jump_only ? V->n_uni : 0;
        mres_collide_kernel<L, R, X, E><<<nb, E * E * E, 0, stream_>>>(A);
    });
    VOXL_CUDA(cudaGetLastError());
    mark_end(kTCollide, b);
}

void MultiResEngine::launch_stream(int l, bool jump_only, cudaStream_t s, const DiagTarget* diag) {
    Level* V = lv_[l];
    const int nb = jump_only ? V->n_jump : V->n_all;
    if (nb == 0) return;
    cudaStream_t st = s ? s : stream_;
    cudaEvent_t b{};
    mark_begin(kTStream, &b, st);
    mres_dispatch(cfg_.lattice, cfg_.precision, cfg_.edge, [&](auto lat, auto real, auto exact, auto e) {
        using L = decltype(lat);
        using R = decltype(real);
        constexpr bool X = decltype(exact)::value;
        constexpr int E = decltype(e)::value;
        auto A = level_args<L, R, X>(cfg_, V, cfg_.fused ? ahead_step_ : steps_done_, d_error_);
        if (cfg_.fused) {  // post -> nxt, and BGK(nxt) -> the other post buffer
            A.post_ahead = static_cast<R*>(V->post[V->parity ^ 1]);
            launch_pull_diag<L, R, X, E, kStreamAhead>(A, jump_only ? V->n_uni : 0, nb, V->n_plain, st, diag,
                                                       V->canon, V->cell0);
        } else {  // post -> nxt
            launch_pull_diag<L, R, X, E, kStream>(A, jump_only ? V->n_uni : 0, nb, V->n_plain, st, diag, V->canon,
                                                  V->cell0);
        }
    });
    VOXL_CUDA(cudaGetLastError());
    mark_end(kTStream, b, st);
}

void MultiResEngine::gather_uniform(int l) {
    // Pre-collision state of the uniform cells (the reference's cur) after
    // the last step: the pull, without collision, of the previous step's
    // post-collision buffer (post[parity ^ 1] still holds it: uniform, jump
    // and ghost slots of that step) -- bitwise what the fused kernel had in
    // registers before it collided.
    Level* V = lv_[l];
    if (V->n_uni == 0) return;
    mres_dispatch(cfg_.lattice, cfg_.precision, cfg_.edge, [&](auto lat, auto real, auto exact, auto e) {
        using L = decltype(lat);
        using R = decltype(real);
        constexpr bool X = decltype(exact)::value;
        constexpr int E = decltype(e)::value;
        auto A = level_args<L, R, X>(cfg_, V, steps_done_, d_error_);
        A.post = static_cast<R*>(V->post[V->parity ^ 1]);
        A.nxt = static_cast<R*>(V->cur);
        launch_pull<L, R, X, E, kStream>(A, 0, V->n_uni, V->n_plain, stream_);
    });
    VOXL_CUDA(cudaGetLastError());
}

void MultiResEngine::sync_state() {
    if (!cfg_.fused || cur_valid_) return;
    for (int l = 0; l < int(lv_.size()); ++l) gather_uniform(l);
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    cur_valid_ = true;
}

void MultiResEngine::load_uniform_post() {
    // After cur changed on the host side: post = BGK(cur) for every block
    // (what the reference's next collide_level computes). From then on the
    // fused uniform kernel keeps the uniform blocks' post current and the
    // jump-block stream (kStreamAhead) the jump blocks', so fused mode never
    // launches collide_level on its own.
    if (!cfg_.fused) return;
    for (int l = 0; l < int(lv_.size()); ++l) {
        Level* V = lv_[l];
        if (V->n_all == 0) continue;
        mres_dispatch(cfg_.lattice, cfg_.precision, cfg_.edge, [&](auto lat, auto real, auto exact, auto e) {
            using L = decltype(lat);
            using R = decltype(real);
            constexpr bool X = decltype(exact)::value;
            constexpr int E = decltype(e)::value;
            auto A = level_args<L, R, X>(cfg_, V, steps_done_, d_error_);
            A.block_begin = 0;
            mres_collide_kernel<L, R, X, E><<<V->n_all, E * E * E, 0, stream_>>>(A);
        });
        VOXL_CUDA(cudaGetLastError());
    }
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    cur_valid_ = true;
}

void MultiResEngine::launch_fused(int l, const DiagTarget* diag) {
    Level* V = lv_[l];
    if (V->n_uni == 0) return;
    cudaEvent_t b{};
    mark_begin(kTFused, &b);
    mres_dispatch(cfg_.lattice, cfg_.precision, cfg_.edge, [&](auto lat, auto real, auto exact, auto e) {
        using L = decltype(lat);
        using R = decltype(real);
        constexpr bool X = decltype(exact)::value;
        constexpr int E = decltype(e)::value;
        auto A = level_args<L, R, X>(cfg_, V, ahead_step_, d_error_);  // the collision is the next sub-step's
        A.nxt = static_cast<R*>(V->post[V->parity ^ 1]);  // post[p] -> post[p^1]
        launch_pull_diag<L, R, X, E, kFused>(A, 0, V->n_uni, V->n_plain, stream_, diag, V->canon, V->cell0);
    });
    VOXL_CUDA(cudaGetLastError());
    mark_end(kTFused, b);
}

void MultiResEngine::launch_explode(int coarse, cudaStream_t st) {
    Level* F = lv_[coarse - 1];
    Level* Cc = lv_[coarse];
    if (F->n_ghost == 0) return;
    cudaEvent_t b{};
    mark_begin(kTTransition, &b, st);
    const unsigned grid = unsigned(((long long)F->n_ghost * q_ + 255) / 256);
    // One explosion serves both fine sub-steps (multires.cpp:563-570); the
    // fine level flips its post parity between them, so fill both copies.
    void* da = F->post[cfg_.fused ? 0 : F->parity];
    void* db = cfg_.fused ? F->post[1] : nullptr;
    const void* src = Cc->post[Cc->parity];
    const int lb = log2_exact(F->ext.block_volume());
    if (esize_ == 8) {
        q_dispatch(q_, [&](auto QC) {
            mres_explode_kernel<decltype(QC)::value, double><<<grid, 256, 0, st>>>(
                static_cast<double*>(da), static_cast<double*>(db), static_cast<const double*>(src), F->explode_dst,
                F->explode_src, F->n_ghost, lb);
        });
    } else {
        q_dispatch(q_, [&](auto QC) {
            mres_explode_kernel<decltype(QC)::value, float><<<grid, 256, 0, st>>>(
                static_cast<float*>(da), static_cast<float*>(db), static_cast<const float*>(src), F->explode_dst,
                F->explode_src, F->n_ghost, lb);
        });
    }
    VOXL_CUDA(cudaGetLastError());
    mark_end(kTTransition, b, st);
}

void MultiResEngine::launch_coalesce(int coarse, cudaStream_t st) {
    Level* F = lv_[coarse - 1];
    Level* Cc = lv_[coarse];
    if (Cc->n_ring == 0) return;
    cudaEvent_t b{};
    mark_begin(kTTransition, &b, st);
    const unsigned grid = unsigned(((long long)Cc->n_ring * q_ + 255) / 256);
    const int nchild = grid_.dim() == 3 ? 8 : 4;
    const int bvc = log2_exact(Cc->ext.block_volume()), bvf = log2_exact(F->ext.block_volume());
    if (esize_ == 8) {
        q_dispatch(q_, [&](auto QC) {
            mres_coalesce_kernel<decltype(QC)::value, double, true><<<grid, 256, 0, st>>>(
                static_cast<double*>(Cc->post[Cc->parity]), static_cast<const double*>(F->cur), Cc->coal_dst,
                Cc->coal_child, Cc->n_ring, bvc, bvf, nchild);
        });
    } else {
        q_dispatch(q_, [&](auto QC) {
            mres_coalesce_kernel<decltype(QC)::value, float, false><<<grid, 256, 0, st>>>(
                static_cast<float*>(Cc->post[Cc->parity]), static_cast<const float*>(F->cur), Cc->coal_dst,
                Cc->coal_child, Cc->n_ring, bvc, bvf, nchild);
        });
    }
    VOXL_CUDA(cudaGetLastError());
    mark_end(kTTransition, b, st);
}

void MultiResEngine::advance(int l) {
    // advance (multires.cpp:563-567). Fused mode: the jump blocks' collide
    // was done by the previous jump-block stream (or load_uniform_post).
    // Only jump cells read ghost (exploded) and ring (coalesced) slots, and
    // only jump cells are ghost parents and ring children (checked at build,
    // side_transitions_), so in fused mode explosion and coalescence run on
    // the side stream in order with the jump-block streams, and the long
    // fused uniform kernels on the engine stream never wait for them.
    if (!cfg_.fused) launch_collide(l, false);
    if (sub_.size() != lv_.size()) sub_.assign(lv_.size(), 0);
    const int per = 1 << (int(lv_.size()) - 1 - l);  // advance(l) calls per coarse step
    const int sub = sub_[std::size_t(l)];
    sub_[std::size_t(l)] = sub + 1 == per ? 0 : sub + 1;
    const int ahead = steps_done_ + (sub + 1 == per ? 1 : 0);
    if (l > 0) {
        if (side_transitions_) {
            VOXL_CUDA(cudaEventRecord(ev_fork_, stream_));
            VOXL_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
        }
        launch_explode(l, side_transitions_ ? side_ : stream_);
        advance(l - 1);
        advance(l - 1);
        if (side_transitions_) {
            // the fine level's last stream may have run on the engine stream
            // (a level without uniform or without jump blocks)
            VOXL_CUDA(cudaEventRecord(ev_fork_, stream_));
            VOXL_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
        }
        launch_coalesce(l, side_transitions_ ? side_ : stream_);
    }
    Level* V = lv_[l];
    ahead_step_ = ahead;
    // run_multires probes the state after the coarse step: each level's
    // cur after its last sub-step, i.e. what this sub-step's pull computes
    const DiagTarget* dg = sub + 1 == per ? diag_ : nullptr;
    if (cfg_.fused && V->n_uni > 0 && V->n_jump > 0) {
        // jump stream (side stream, high priority) || fused uniform (engine stream)
        VOXL_CUDA(cudaEventRecord(ev_fork_, stream_));
        VOXL_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
        launch_stream(l, true, side_, dg);
        launch_fused(l, dg);
        VOXL_CUDA(cudaEventRecord(ev_join_, side_));
        VOXL_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
    } else {
        if (side_transitions_) {  // this level's stream may read the side stream's transitions
            VOXL_CUDA(cudaEventRecord(ev_join_, side_));
            VOXL_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
        }
        if (cfg_.fused) launch_fused(l, dg);
        launch_stream(l, cfg_.fused, nullptr, dg);
    }
    std::swap(V->cur, V->nxt);
    if (cfg_.fused) V->parity ^= 1;
    cur_valid_ = false;
}

void MultiResEngine::check_errors() {
    int flag = INT_MAX;
    VOXL_CUDA(cudaMemcpyAsync(&flag, d_error_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    // flag == steps_done_: a collide-ahead of a step that has not run yet
    // (fused mode); it throws once that step has run, as the reference would
    if (flag < steps_done_)
        throw InstabilityError("run aborted at step " + std::to_string(flag) + ": macroscopic: non-positive density");
}

void MultiResEngine::coarse_step(int n) {
    for (int i = 0; i < n; ++i) {
        advance(grid_.num_levels() - 1);
        ++steps_done_;
    }
    check_errors();
}

MresTimes MultiResEngine::timed_steps(int n) {
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev;
    events_ = &ev;
    cudaEvent_t t0, t1;
    VOXL_CUDA(cudaEventCreate(&t0));
    VOXL_CUDA(cudaEventCreate(&t1));
    VOXL_CUDA(cudaEventRecord(t0, stream_));
    for (int i = 0; i < n; ++i) {
        advance(grid_.num_levels() - 1);
        ++steps_done_;
    }
    VOXL_CUDA(cudaEventRecord(t1, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    events_ = nullptr;
    MresTimes T;
    float ms = 0;
    VOXL_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    T.total = ms;
    for (auto& e : ev) {
        float m = 0;
        VOXL_CUDA(cudaEventElapsedTime(&m, e.second.first, e.second.second));
        (e.first == kTCollide ? T.collide : e.first == kTStream ? T.stream : e.first == kTFused ? T.fused
                                                                                                 : T.transition) += m;
        cudaEventDestroy(e.second.first);
        cudaEventDestroy(e.second.second);
    }
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    check_errors();
    return T;
}

void MultiResEngine::device_probe(double out[3], DenseDiag* d) {
    // Sums and max |u| per level in storage order over the active slots
    // (block_probe.cuh), combined in a fixed order; the canonical-order kernel
    // only runs to name the first unstable cell when there is one. Only the
    // result row comes back to the host.
    const std::size_t per_level = 2 * std::size_t(kMresProbeBlocks);
    const std::size_t need = per_level * lv_.size() + 5;
    if (diag_len_ < need) {
        cudaFree(d_diag_);
        VOXL_CUDA(cudaMalloc(&d_diag_, need * sizeof(double)));
        diag_len_ = need;
    }
    double* row = d_diag_ + per_level * lv_.size();
    auto* bad = reinterpret_cast<unsigned long long*>(row + 3);
    auto* bad_any = reinterpret_cast<unsigned int*>(row + 4);
    VOXL_CUDA(cudaMemsetAsync(d_diag_, 0, need * sizeof(double), stream_));
    // Fused mode keeps the uniform cells' pre-collision state implicit (their
    // post-collision storage): probe it through the collision-free pull that
    // gather_uniform would store (kProbe), reduced in registers instead of
    // written and re-read; the jump (and ghost-only) blocks' cur is stored.
    const bool pull_probe = cfg_.fused && !cur_valid_;
    constexpr int kHalf = kMresProbeBlocks / 2;
    auto shift_of = [&](auto lat) {
        using L = decltype(lat);
        ShiftQ<L::Q> sh{};
        for (int i = 0; i < L::Q; ++i) sh.v[i] = esize_ == 8 ? 0.0 : L::w(i);
        return sh;
    };
    for (std::size_t l = 0; l < lv_.size(); ++l) {
        Level* V = lv_[l];
        const long long nb = V->ext.num_blocks();
        if (V->n_active == 0 || nb == 0) continue;
        const int lb = log2_exact(V->ext.block_volume());
        const int bv = V->ext.block_volume(), words = V->ext.mask_words();
        const long long first = pull_probe ? V->n_uni : 0;  // blocks probed from storage
        double* slots = d_diag_ + per_level * l;
        mres_dispatch(cfg_.lattice, cfg_.precision, cfg_.edge, [&](auto lat, auto real, auto exact, auto e) {
            using L = decltype(lat);
            using R = decltype(real);
            constexpr bool X = decltype(exact)::value;
            constexpr int E = decltype(e)::value;
            if (pull_probe && V->n_uni > 0) {
                const long long parts = (long long)V->n_uni * kSplit<E>;
                if (probe_scratch_len_ < std::size_t(2 * parts)) {
                    cudaFree(probe_scratch_);
                    VOXL_CUDA(cudaMalloc(&probe_scratch_, 2 * parts * sizeof(double)));
                    probe_scratch_len_ = std::size_t(2 * parts);
                }
                auto A = level_args<L, R, X>(cfg_, V, steps_done_, d_error_);
                A.post = static_cast<R*>(V->post[V->parity ^ 1]);
                A.probe_partial = probe_scratch_;
                A.probe_bad = bad_any;
                A.step_probe_base = 0;
                launch_pull<L, R, X, E, kProbe>(A, 0, V->n_uni, V->n_plain, stream_);
                partials_reduce_kernel<<<kHalf, 256, 0, stream_>>>(probe_scratch_, parts, slots);
                slots += 2 * kHalf;
            }
            const long long n = nb - first;
            if (n > 0) {
                const int ctas = int(std::min<long long>(pull_probe ? kHalf : kMresProbeBlocks, n));
                block_probe_kernel<L, R><<<ctas, 256, 0, stream_>>>(
                    static_cast<const R*>(V->cur) + first * L::Q * bv, V->amask + first * words, words, lb, n,
                    shift_of(lat), slots, bad_any);
            }
        });
        VOXL_CUDA(cudaGetLastError());
    }
    mres_probe_final<<<1, 32, 0, stream_>>>(d_diag_, int(lv_.size()), kMresProbeBlocks,
                                            double(grid_.dim() == 3 ? 8 : 4), row);
    VOXL_CUDA(cudaGetLastError());
    double h[5];
    VOXL_CUDA(cudaMemcpyAsync(h, row, sizeof h, cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    unsigned int any;
    std::memcpy(&any, &h[4], sizeof any);
    out[0] = h[0];
    out[1] = std::sqrt(h[1]);  // the kernels reduce |u|^2
    out[2] = h[2];
    if (!d) return;
    d->mass = out[0];
    d->max_speed = out[1];
    if (!any) return;
    // name the first unstable cell in canonical order (levels finest first)
    sync_state();
    const unsigned long long none = ~0ull;
    VOXL_CUDA(cudaMemcpyAsync(bad, &none, sizeof none, cudaMemcpyHostToDevice, stream_));
    long long cell0 = 0;
    for (std::size_t l = 0; l < lv_.size(); ++l) {
        Level* V = lv_[l];
        const long long n = V->n_active;
        if (n > 0) {
            const int lb = log2_exact(V->ext.block_volume());
            mres_dispatch(cfg_.lattice, cfg_.precision, cfg_.edge, [&](auto lat, auto real, auto, auto) {
                using L = decltype(lat);
                using R = decltype(real);
                mres_slot_probe_kernel<L, R><<<kMresProbeBlocks, 256, 0, stream_>>>(
                    static_cast<const R*>(V->cur), V->slots, n, lb, shift_of(lat), cell0, d_diag_, bad);
            });
            VOXL_CUDA(cudaGetLastError());
        }
        cell0 += n;
    }
    unsigned long long b = 0;
    VOXL_CUDA(cudaMemcpyAsync(&b, bad, sizeof b, cudaMemcpyDeviceToHost, stream_));
    VOXL_CUDA(cudaStreamSynchronize(stream_));
    d->unstable = 1;
    d->bad_voxel = std::int64_t(b >> 5);
    d->bad_population = int(b & 31u);
}

namespace {
__global__ void mres_canon_kernel(const std::int64_t* slots, long long n, std::int32_t* canon) {
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x)
        canon[slots[v]] = std::int32_t(v);
}
} // namespace

void MultiResEngine::build_canon_maps() {
    long long cell0 = 0;
    for (Level* V : lv_) {
        V->cell0 = cell0;
        cell0 += V->n_active;
        if (V->canon || V->n_active == 0) continue;
        const std::size_t n = std::size_t(V->ext.num_blocks()) * std::size_t(V->ext.block_volume());
        VOXL_CUDA(cudaMalloc(&V->canon, n * sizeof(std::int32_t)));
        VOXL_CUDA(cudaMemsetAsync(V->canon, 0xFF, n * sizeof(std::int32_t), stream_));
        mres_canon_kernel<<<kMresProbeBlocks, 256, 0, stream_>>>(V->slots, V->n_active, V->canon);
        VOXL_CUDA(cudaGetLastError());
    }
}

int MultiResEngine::step_probe_n(int n, DenseDiag* rows, std::string* abort_msg) {
    // Batches of up to kDiagBatch coarse steps. Each level's last sub-step
    // kernels (fused uniform + jump stream, or the staged stream) pull the
    // level's cur of the coarse step's end and fold probe_field's terms into
    // the step's accumulator lanes before colliding it; one reduction kernel,
    // one copy and one host synchronisation per batch (the reference probes
    // canonical_state after every coarse_step, solver.cpp:343-345).
    if (n < 0) throw std::invalid_argument("step_probe: n must be >= 0");
    if (!ring_) ring_ = std::make_unique<DiagRing>();
    build_canon_maps();
    int done = 0;
    while (done < n) {
        const int b = std::min(n - done, kDiagBatch);
        const int step0 = steps_done_;
        ring_->begin(b, stream_);  // every side-stream launch forks from the engine stream after this
        DiagTarget dt;
        for (int s = 0; s < b; ++s) {
            dt.acc = ring_->acc(s);
            dt.bad = ring_->bad(s);
            diag_ = &dt;
            advance(grid_.num_levels() - 1);
            ++steps_done_;
        }
        diag_ = nullptr;
        if (side_) {
            VOXL_CUDA(cudaEventRecord(ev_join_, side_));
            VOXL_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
        }
        ring_->reduce(d_error_, stream_);
        VOXL_CUDA(cudaStreamSynchronize(stream_));
        const DiagRow* r = ring_->rows();
        std::string msg;
        // a collide-ahead error of step steps_done_ (not run yet) stays
        // pending: first_failure only reports steps of this batch
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
            return done;
        }
    }
    return done;
}

DenseDiag MultiResEngine::probe() {
    // probe_field over canonical_state (solver.cpp:345): sum over all levels'
    // cells and max |u|, reduced on the device.
    DenseDiag d;
    double o[3];
    device_probe(o, &d);
    return d;
}

double MultiResEngine::total_mass() {
    // total_mass (multires.cpp:600-609): per-level sums weighted by 8^l
    double o[3];
    device_probe(o, nullptr);
    return o[2];
}

std::array<std::int64_t, 2> MultiResEngine::fusion_counts(int l) const { return {lv_[l]->n_uni, lv_[l]->n_jump}; }

std::string MultiResEngine::graph_dot() const {
    if (grid_.has_reference_tables() && cfg_.edge == 4) return grid_.graph_dot(cfg_.fused);
    std::vector<std::array<std::int64_t, 2>> counts;
    for (int l = 0; l < grid_.num_levels(); ++l) counts.push_back(fusion_counts(l));
    return grid_.graph_dot(cfg_.fused, &counts);
}

} // namespace voxl_b200
