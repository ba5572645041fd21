// common.cuh -- error plumbing shared by the engines and the C-ABI.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace voxl_b200 {

/// Status codes of the C-ABI (include/voxl_b200.h).
enum Status : int {
    kOk = 0,
    kInvalidArgument = 1,  // std::invalid_argument in the reference
    kOutOfRange = 2,       // std::out_of_range
    kRuntime = 3,          // std::runtime_error (structure errors, asymmetric links)
    kInstability = 4,      // "instability at step N" / "run aborted at step N"
    kCuda = 5,             // CUDA runtime failure
    kDomain = 6,           // std::domain_error (non-finite equilibrium input)
};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct InstabilityError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

#define VOXL_CUDA(call) ::voxl_b200::cuda_check((call), #call)

/// log2 of a power of two (block volumes E^3, E in {1, 2, 4, 8}): device
/// slot arithmetic uses shifts instead of 64-bit division.
inline int log2_exact(long long v) {
    int l = 0;
    while ((1ll << l) < v) ++l;
    if ((1ll << l) != v) throw std::invalid_argument("block volume is not a power of two");
    return l;
}

/// Resident 256-thread CTAs per SM requested from ptxas for the fp32 8^3-block
/// kernels (block-sparse light kernel, multires pull kernel): 6 caps D3Q19 at
/// 40 registers. D3Q27 (27 live populations) spills at 40; measured at 512^3
/// (a -DVOXL_BLOCK_MINB27 sweep, tools/build_lib_variant.sh + gpu_lib_variants.sh;
/// GLUPS sparse disag_mem / multires fused):
/// 6 CTAs 26.1 / 27.1, 5 CTAs 27.9 / 27.8, 4 CTAs 25.9 / 27.7.
#ifndef VOXL_BLOCK_MINB19
#define VOXL_BLOCK_MINB19 6
#endif
#ifndef VOXL_BLOCK_MINB27
#define VOXL_BLOCK_MINB27 5
#endif
constexpr int block_min_ctas(int q) { return q == 27 ? VOXL_BLOCK_MINB27 : VOXL_BLOCK_MINB19; }

} // namespace voxl_b200
