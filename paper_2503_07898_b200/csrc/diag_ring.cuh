// diag_ring.cuh -- run()'s per-step probe_field rows (solver.cpp:245-255,
// lbm.cpp:116-138), accumulated on the device by the fused step kernels and
// read back once per batch of steps.
//
// No partial arrays: one lane per warp adds the warp's mass partial into one
// of kDiagLanes accumulator lanes as a 128-bit fixed-point number (64
// fraction bits, split over three 64-bit words so plain `red.add` never needs
// a carry) and folds max |u|^2 in with an integer max of its fp64 bits
// (non-negative doubles order like their bit patterns). Integer addition is
// associative, so the per-step sums do not depend on the order the warps
// retire or on how a step is cut into launches: deterministic, and a step
// probed in plane chunks (the streamed run) gives the same row bit for bit.
// The fixed point rounds each warp partial to 2^-64 (the reference's own
// sequential fp64 sum is ~1e-8 off the exact sum at 512^3).
//
// Per step: kDiagLanes x 4 words (32 KB) + one "first bad voxel" word
// ((canonical voxel << 5) | population, atomicMin: the reference's first
// offender, voxel-major then population; population kBadDensity = 31 marks a
// non-positive density, macroscopic's throw). One kernel reduces a whole batch
// into 32-byte exact sums, one copy brings them and the engine's error flag
// home; the host rounds each sum to fp64 once (diag_compose), after adding the
// sums of every device a multi-device step ran on.
#pragma once

#include "common.cuh"
#include "lattice.cuh"

#include <climits>
#include <cstring>
#include <string>
#include <vector>

namespace voxl_b200 {

constexpr int kDiagLanes = 1024;  // power of two
constexpr int kDiagWords = 4;     // fraction bits [0,32) | fraction bits [32,64) | integer part | max |u|^2 bits
constexpr int kDiagBatch = 256;   // steps per read-back (8 MB of accumulators)

/// Where a step launch writes its fused-probe terms.
struct DiagTarget {
    unsigned long long* acc = nullptr;  // the step's accumulator lanes
    unsigned long long* bad = nullptr;  // the step's first-offender word
};

struct DiagRow {
    double mass;
    double v2;                // max |u|^2 (the host takes the square root)
    unsigned long long bad;   // ~0 = healthy
    long long pad;
};

/// red.add with an L2 evict_last policy: the accumulator lines are hit by
/// every CTA of the step while the step streams its whole state through L2;
/// a normal-priority line gets evicted between hits, and each miss costs a
/// DRAM fill plus a write-back (ncu: 5.5 M missed red sectors, +0.2 GB of
/// DRAM writes per 512^3 step with one reduction per warp).
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v, unsigned long long pol) {
    asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ void red_add_u64_plain(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

/// A warp partial as accumulator words: fraction bits [0,32), fraction bits
/// [32,64), integer part (two's complement), max |u|^2 as fp64 bits. A
/// non-finite partial contributes nothing (its bad voxel is reported by the
/// step's bad word).
__device__ __forceinline__ void diag_words(double mass, double v2, unsigned long long (&w)[kDiagWords]) {
    w[0] = w[1] = w[2] = 0;
    if (fabs(mass) < 4.0e18) {
        const double ip = floor(mass);
        const unsigned long long frac = (unsigned long long)((mass - ip) * 18446744073709551616.0);
        w[0] = frac & 0xffffffffull;
        w[1] = frac >> 32;
        w[2] = (unsigned long long)(long long)ip;
    }
    w[3] = v2 > 0.0 ? (unsigned long long)__double_as_longlong(v2) : 0ull;
}

/// One warp's contribution (called by a single lane). `warp_id` only spreads
/// the accumulators over lanes; any mapping gives the same sums. No CTA
/// barrier: a per-CTA pre-reduction through shared memory was measured
/// slower (512^3 dense step_probe 3.53 vs 3.30 ms under ncu: warps parked at
/// the barrier hold their CTA's slot while the step is HBM-bound).
__device__ __forceinline__ void diag_commit(unsigned long long* acc, unsigned long long warp_id, double mass,
                                            double v2) {
    unsigned long long w[kDiagWords];
    diag_words(mass, v2, w);
    unsigned long long* lane = acc + (warp_id & (kDiagLanes - 1)) * kDiagWords;
    const unsigned long long pol = l2_evict_last_policy();
    if (w[0]) red_add_u64(lane + 0, w[0], pol);
    if (w[1]) red_add_u64(lane + 1, w[1], pol);
    if (w[2]) red_add_u64(lane + 2, w[2], pol);
    if (w[3]) atomicMax(lane + 3, w[3]);
}

/// A warp's probe terms for the fp32 (shifted-storage) kernels, every lane
/// calling with its voxel's dr = rho - 1 and |u|^2 (zeros for a dead or
/// unstable lane; `live` = the warp's live lanes). Each lane's dr becomes a
/// fixed-point integer in 2^-40 units (|dr| < 2^15 for any voxel that passes
/// probe_field's |f_i| <= 1e3 test; larger or non-finite terms only occur on a
/// step the bad word already fails), summed exactly across the warp in three
/// 21-bit chunks by redux.sync; max |u|^2 is a redux.sync max of the fp32 bit
/// patterns (non-negative floats order like their bits). Lane 0 adds the
/// live count (the 1 of each rho) and commits the warp's words. Half the
/// instructions of a shuffle tree plus an fp64 fixed-point conversion, and
/// the per-lane rounding (2^-41) is finer than an fp32 warp sum's.
/// Uncond: add the three mass words without a zero test (no branch per word;
/// adding zero is harmless); Policy: carry the L2 evict_last hint. The dense
/// step uses <true, false> (measured: probed 1000-step batches 3.465 ->
/// 3.445 ms, profiles/r2_diag_commit_variants.txt); the block kernels keep the
/// defaults.
template <bool Uncond = false, bool Policy = true>
__device__ __forceinline__ void diag_warp_commit_f32(unsigned long long* acc, unsigned long long warp_id, float dr,
                                                     float v2, unsigned live) {
    long long fx = 0;
    if (fabsf(dr) < 32768.0f) fx = __float2ll_rn(dr * 1099511627776.0f);  // x 2^40 (exact scaling)
    const unsigned c0 = unsigned(fx) & 0x1FFFFFu, c1 = unsigned(fx >> 21) & 0x1FFFFFu;
    const int c2 = int(fx >> 42);
    const unsigned s0 = __reduce_add_sync(0xffffffffu, c0), s1 = __reduce_add_sync(0xffffffffu, c1);
    const int s2 = __reduce_add_sync(0xffffffffu, c2);
    const unsigned vb = __reduce_max_sync(0xffffffffu, __float_as_uint(v2));
    if ((threadIdx.x & 31) != 0 || !live) return;
    // T = sum of the lanes in 2^-40 units, plus 2^40 per live voxel
    const long long T = ((long long)s2 << 42) + ((long long)s1 << 21) + (long long)s0 +
                        ((long long)__popc(live) << 40);
    const unsigned long long frac40 = (unsigned long long)T & ((1ull << 40) - 1);
    unsigned long long* lane = acc + (warp_id & (kDiagLanes - 1)) * kDiagWords;
    const unsigned long long w0 = (frac40 & 0xffull) << 24, w1 = frac40 >> 8,
                             w2 = (unsigned long long)(T >> 40);  // 64 fraction bits: frac40 << 24
    unsigned long long pol = 0;
    if constexpr (Policy) pol = l2_evict_last_policy();
    auto red = [&](unsigned long long* p, unsigned long long v) {
        if constexpr (Policy) red_add_u64(p, v, pol);
        else red_add_u64_plain(p, v);
    };
    if (Uncond || w0) red(lane + 0, w0);
    if (Uncond || w1) red(lane + 1, w1);
    if (Uncond || w2) red(lane + 2, w2);
    if (vb) atomicMax(lane + 3, (unsigned long long)__double_as_longlong(double(__uint_as_float(vb))));
}

/// A step's exact sums: mass as a 128-bit two's-complement fixed-point number
/// (64 fraction bits), max |u|^2 as fp64 bits, the first-offender word.
/// Raw sums from several rings (one per device) add as integers, so a step
/// split over devices composes to the same row bit for bit.
struct DiagRaw {
    unsigned long long lo, hi, vmax, bad;
};

/// One CTA per step: exact integer sums over the lanes.
__global__ inline void __launch_bounds__(256) diag_rows_kernel(const unsigned long long* acc, const unsigned long long* bad,
                                                        DiagRaw* rows) {
    const unsigned long long* a = acc + (long long)blockIdx.x * kDiagLanes * kDiagWords;
    unsigned long long w0 = 0, w1 = 0, w2 = 0, vm = 0;
    for (int l = threadIdx.x; l < kDiagLanes; l += 256) {
        w0 += a[l * kDiagWords + 0];
        w1 += a[l * kDiagWords + 1];
        w2 += a[l * kDiagWords + 2];
        vm = max(vm, a[l * kDiagWords + 3]);
    }
    __shared__ unsigned long long s0[256], s1[256], s2[256], sv[256];
    s0[threadIdx.x] = w0;
    s1[threadIdx.x] = w1;
    s2[threadIdx.x] = w2;
    sv[threadIdx.x] = vm;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            s0[threadIdx.x] += s0[threadIdx.x + o];
            s1[threadIdx.x] += s1[threadIdx.x + o];
            s2[threadIdx.x] += s2[threadIdx.x + o];
            sv[threadIdx.x] = max(sv[threadIdx.x], sv[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        // T = w2 * 2^64 + w1 * 2^32 + w0 (two's complement, 64 fraction bits)
        const unsigned long long x0 = s0[0], x1 = s1[0];
        const unsigned long long lo = x0 + (x1 << 32);
        DiagRaw r;
        r.lo = lo;
        r.hi = s2[0] + (x1 >> 32) + (lo < x0 ? 1ull : 0ull);
        r.vmax = sv[0];
        r.bad = bad[blockIdx.x];
        rows[blockIdx.x] = r;
    }
}

/// Sum of two rings' raw rows (mod 2^128 fixed point, max, min).
inline void diag_accumulate(DiagRaw& into, const DiagRaw& x) {
    const unsigned long long lo = into.lo + x.lo;
    into.hi += x.hi + (lo < x.lo ? 1ull : 0ull);
    into.lo = lo;
    into.vmax = into.vmax > x.vmax ? into.vmax : x.vmax;
    into.bad = into.bad < x.bad ? into.bad : x.bad;
}

/// The row of a raw sum: one rounding of the exact fixed-point mass to fp64.
inline DiagRow diag_compose(const DiagRaw& r) {
    DiagRow row;
    row.mass = double((long long)r.hi) + double(r.lo) * 0x1p-64;
    double v2;
    std::memcpy(&v2, &r.vmax, sizeof v2);
    row.v2 = v2;
    row.bad = r.bad;
    row.pad = 0;
    return row;
}

/// Device accumulators + pinned rows of up to kDiagBatch probed steps.
class DiagRing {
public:
    DiagRing() = default;
    DiagRing(const DiagRing&) = delete;
    DiagRing& operator=(const DiagRing&) = delete;
    ~DiagRing() {
        if (acc_) cudaFree(acc_);
        if (bad_) cudaFree(bad_);
        if (raw_) cudaFree(raw_);
        if (host_) cudaFreeHost(host_);
    }

    /// Zero the accumulators of n <= kDiagBatch steps on `st`.
    void begin(int n, cudaStream_t st) {
        if (n < 1 || n > kDiagBatch) throw std::invalid_argument("DiagRing: batch size out of range");
        if (!acc_) {
            VOXL_CUDA(cudaMalloc(&acc_, std::size_t(kDiagBatch) * kDiagLanes * kDiagWords * 8));
            VOXL_CUDA(cudaMalloc(&bad_, std::size_t(kDiagBatch) * 8));
            VOXL_CUDA(cudaMalloc(&raw_, std::size_t(kDiagBatch) * sizeof(DiagRaw)));
            VOXL_CUDA(cudaMallocHost(&host_, std::size_t(kDiagBatch) * sizeof(DiagRaw) + 16));
        }
        VOXL_CUDA(cudaMemsetAsync(acc_, 0, std::size_t(n) * kDiagLanes * kDiagWords * 8, st));
        VOXL_CUDA(cudaMemsetAsync(bad_, 0xFF, std::size_t(n) * 8, st));
        n_ = n;
    }
    unsigned long long* acc(int s) const { return acc_ + std::size_t(s) * kDiagLanes * kDiagWords; }
    unsigned long long* bad(int s) const { return bad_ + s; }

    /// Enqueue the batch's reduction and the read-back of the rows and of
    /// `error_flag` (the engine's first non-positive-density step) on `st`.
    void reduce(const int* error_flag, cudaStream_t st) {
        diag_rows_kernel<<<n_, 256, 0, st>>>(acc_, bad_, raw_);
        VOXL_CUDA(cudaGetLastError());
        VOXL_CUDA(cudaMemcpyAsync(host_, raw_, std::size_t(n_) * sizeof(DiagRaw), cudaMemcpyDeviceToHost, st));
        if (error_flag)
            VOXL_CUDA(cudaMemcpyAsync(flag_slot(), error_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
        else
            *flag_slot() = INT_MAX;
    }
    /// After the stream synchronised: the raw sums and the error flag.
    const DiagRaw* raw() const { return host_; }
    /// The composed rows of this ring alone.
    const DiagRow* rows() {
        rows_.resize(std::size_t(n_));
        for (int s = 0; s < n_; ++s) rows_[std::size_t(s)] = diag_compose(host_[s]);
        return rows_.data();
    }
    int error_flag() const { return *flag_slot(); }

private:
    int* flag_slot() const { return reinterpret_cast<int*>(host_ + kDiagBatch); }
    unsigned long long* acc_ = nullptr;
    unsigned long long* bad_ = nullptr;
    DiagRaw* raw_ = nullptr;
    DiagRaw* host_ = nullptr;
    std::vector<DiagRow> rows_;
    int n_ = 0;
};

/// run()'s abort rule over a probed batch whose row s is absolute step
/// step0 + s (solver.cpp:245-255): a step fails on a non-positive density
/// during the collision (bgk_relax -> macroscopic, lattice.cpp:124; the
/// engine's error flag holds the first such step) or on probe_field's
/// instability test (lbm.cpp:124-128; the row's bad word). Returns the index
/// of the first failing row (-1: none) and the reference's message.
inline int first_failure(const DiagRow* rows, int n, int step0, int error_flag, std::string* msg) {
    for (int s = 0; s < n; ++s) {
        const int step = step0 + s;
        const std::string head = "run aborted at step " + std::to_string(step) + ": ";
        if (error_flag == step) {
            *msg = head + "macroscopic: non-positive density";
            return s;
        }
        if (rows[s].bad != ~0ull) {
            const int pop = int(rows[s].bad & 31u);
            if (pop == kBadDensity) *msg = head + "macroscopic: non-positive density";
            else
                *msg = head + "instability at step " + std::to_string(step) + ", voxel " +
                       std::to_string((long long)(rows[s].bad >> 5)) + ", population " + std::to_string(pop);
            return s;
        }
    }
    if (error_flag != INT_MAX && error_flag < step0) {
        *msg = "run aborted at step " + std::to_string(error_flag) + ": macroscopic: non-positive density";
        return 0;
    }
    return -1;
}

} // namespace voxl_b200
