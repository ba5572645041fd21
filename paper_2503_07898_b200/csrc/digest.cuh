// digest.cuh -- position-sensitive digest of a canonical fp64 state, on the device.
//
// Full-size parity (512^3 and up) cannot ship the canonical state to the host
// for an element-wise compare, so the engines reduce it to two 64-bit words:
//   h(i, x) = splitmix64(bits(x) ^ splitmix64(i)),  i = canonical element index
//   sum = sum_i h(i, x_i) mod 2^64,   xr = xor_i rotl(h(i, x_i), 29)
// Integer sum/xor are associative, so the result does not depend on the
// reduction order (deterministic under atomics) and equals the host
// restatement in paper_2503_07898_b200/digest.py bit for bit. Two states
// digest equal iff (up to 2^-64 collisions) they are bitwise equal in the
// reference's canonical order (solver.hpp:56-58; sparse.cpp:416-438;
// multires.cpp:578-598).
#pragma once

#include <cuda_runtime.h>

namespace voxl_b200 {

__host__ __device__ __forceinline__ unsigned long long digest_mix(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static __global__ void digest_kernel(const double* __restrict__ x, long long n, long long base,
                                     unsigned long long* __restrict__ acc) {
    unsigned long long s = 0, r = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(x[i]);
        const unsigned long long h = digest_mix(b ^ digest_mix((unsigned long long)(base + i)));
        s += h;
        r ^= (h << 29) | (h >> 35);
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        r ^= __shfl_xor_sync(0xffffffffu, r, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&acc[0], s);
        atomicXor(&acc[1], r);
    }
}

/// acc (device, 2 words, zeroed by the caller) += digest of x[0, n) at
/// canonical element offset `base`.
inline void digest_accumulate(const double* x, long long n, long long base, unsigned long long* acc,
                              cudaStream_t st) {
    if (n <= 0) return;
    long long blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    digest_kernel<<<unsigned(blocks), 256, 0, st>>>(x, n, base, acc);
}

} // namespace voxl_b200
