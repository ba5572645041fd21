// block_probe.cuh -- probe_field (lbm.cpp:116-138) over block storage in
// storage order, for the block-sparse and multires engines.
//
// The parity surface (canonical_state) orders cells by pack_coord with z
// fastest (sparse.cpp:416-438), i.e. consecutive canonical cells are E*E
// slots apart inside a block: walking the state in that order touches one
// 32-byte sector per population per cell (8x the useful bytes at fp32). The
// probe's sums do not depend on that order beyond rounding (fixed order
// here, so run-to-run deterministic), so it walks each block's slots
// contiguously instead -- coalesced loads, one pass over the state. Only the
// index of the first unstable cell is order-sensitive; the engines recover it
// from the canonical-order kernel in the (rare) unstable case.
#pragma once

#include "canon_io.cuh"
#include "lattice.cuh"

#include <cstdint>

namespace voxl_b200 {

constexpr int kBlockProbeCtas = 592;  // 4 x 148 SMs

/// Per-CTA (sum f, max |u|^2) over the active slots (mask bit set) of blocks
/// [0, nblocks); any unstable cell (|f| > 1e3, non-finite, rho <= 0) sets
/// *bad_any. |u|^2 = (m_x/rho)^2 + (m_y/rho)^2 + (m_z/rho)^2 exactly as
/// macroscopic + probe_field form it, so sqrt(max) is the reference's max.
template <class L, class R>
__global__ void __launch_bounds__(256) block_probe_kernel(const R* buf, const std::uint64_t* masks, int words, int lb,
                                                          long long nblocks, const __grid_constant__ ShiftQ<L::Q> sh,
                                                          double* partial, unsigned int* bad_any) {
    constexpr int Q = L::Q;
    const int bv = 1 << lb;
    double mass = 0.0, vmax = 0.0;
    bool bad = false;
    for (long long b = blockIdx.x; b < nblocks; b += gridDim.x) {
        const R* base = buf + b * Q * (long long)bv;
        for (int t = threadIdx.x; t < bv; t += blockDim.x) {
            if (!((masks[b * words + (t >> 6)] >> (t & 63)) & 1ull)) continue;
            R raw[Q];
            static_for<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                raw[i] = base[(long long)i * bv + t];
            });
            double r = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
            bool b_here = false;
            static_for<Q>([&](auto I) {
                constexpr int i = decltype(I)::value;
                const double fi = double(raw[i]) + sh.v[i];
                b_here = b_here || !(fabs(fi) <= 1e3);
                r += fi;
                mx = acc_term<double, false, L::ex(i)>(mx, fi);
                my = acc_term<double, false, L::ey(i)>(my, fi);
                mz = acc_term<double, false, L::ez(i)>(mz, fi);
            });
            mass += r;
            if (b_here || !(r > 0.0)) {
                bad = true;
            } else {
                const double ux = mx / r, uy = my / r, uz = mz / r;
                vmax = fmax(vmax, ux * ux + uy * uy + uz * uz);
            }
        }
    }
    if (bad) atomicOr(bad_any, 1u);
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

/// out[0] += sum of the partial masses, out[1] = max(out[1], max |u|^2), in
/// a fixed order (one thread: a few hundred partials).
__global__ inline void block_probe_final(const double* partial, int n, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double m = 0.0, v = 0.0;
    for (int i = 0; i < n; ++i) {
        m += partial[2 * i];
        v = fmax(v, partial[2 * i + 1]);
    }
    out[0] += m;
    out[1] = fmax(out[1], v);
}

/// Fixed-order first stage over n (mass, |u|^2) pairs (the fused probes'
/// per-warp partials): CTA j reduces the contiguous slice j into stage[j].
__global__ inline void __launch_bounds__(256) partials_reduce_kernel(const double* p, long long n, double* stage) {
    __shared__ double sm[256], sv[256];
    const long long per = (n + gridDim.x - 1) / gridDim.x;
    const long long lo = (long long)blockIdx.x * per, hi = min(n, lo + per);
    double m = 0.0, v = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        m += p[2 * i];
        v = fmax(v, p[2 * i + 1]);
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
    if (threadIdx.x == 0) {
        stage[2 * blockIdx.x] = sm[0];
        stage[2 * blockIdx.x + 1] = sv[0];
    }
}

template <class L, class R>
void launch_block_probe(const R* buf, const std::uint64_t* masks, int words, int bv, long long nblocks,
                        const double* shift, double* partial, double* out, unsigned int* bad_any, cudaStream_t st) {
    if (nblocks <= 0) return;
    ShiftQ<L::Q> sh{};
    for (int i = 0; i < L::Q; ++i) sh.v[i] = shift[i];
    const int ctas = int(std::min<long long>(kBlockProbeCtas, nblocks));
    block_probe_kernel<L, R><<<ctas, 256, 0, st>>>(buf, masks, words, log2_exact(bv), nblocks, sh, partial, bad_any);
    block_probe_final<<<1, 32, 0, st>>>(partial, ctas, out);
    VOXL_CUDA(cudaGetLastError());
}

} // namespace voxl_b200
