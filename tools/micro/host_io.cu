// host_io.cu -- what bounds the canonical host I/O of the e2e path?
//
// Measures on the GPU box (nvcc -O3 -std=c++17 -Ipaper_2503_07898_b200/csrc):
//   narrow  : fp64 canonical -> fp32 wire on the host pool (HostPool, AVX2 streaming stores)
//   widen   : fp32 wire -> fp64 canonical
//   both    : narrow and widen at the same time, half the pool each
//   h2d/d2h : pinned fp32 copies alone and at the same time (full duplex?)
//   h2d+narrow : DMA of one slot while the pool narrows the next
// Prints one JSON line of GB/s figures (fp64-equivalent bytes for the conversions).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "host_pool.hpp"

using namespace voxl_b200;
using clk = std::chrono::steady_clock;

static double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e = (x);                                                       \
        if (e != cudaSuccess) {                                                    \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));           \
            std::exit(1);                                                          \
        }                                                                          \
    } while (0)

int main(int argc, char** argv) {
    const std::size_t gib = argc > 1 ? std::atoll(argv[1]) : 4;  // fp64 canonical GiB
    const std::size_t n = (gib << 30) / 8;
    const int q = 19;
    double shift[27];
    for (int i = 0; i < 27; ++i) shift[i] = 1.0 / (i + 3);
    double *h64, *h64b;
    float *w32, *w32b;
    CK(cudaMallocHost(&h64, n * 8));
    CK(cudaMallocHost(&h64b, n * 8));
    CK(cudaMallocHost(&w32, n * 4));
    CK(cudaMallocHost(&w32b, n * 4));
    float* d32;
    float* d32b;
    CK(cudaMalloc(&d32, n * 4));
    CK(cudaMalloc(&d32b, n * 4));
    HostPool& pool = HostPool::get();
    pool.parallel_for((long long)(n / q), [&](long long lo, long long hi) {
        for (long long e = lo * q; e < hi * q; ++e) h64[e] = 1.0 / 19, h64b[e] = 0.0;
    });
    const long long cells = (long long)(n / q);
    auto narrow = [&](double* h, float* w) {
        pool.parallel_for(cells, [&](long long lo, long long hi) { io_detail::convert<true>(h, w, lo, hi, shift, q); });
    };
    auto widen = [&](double* h, float* w) {
        pool.parallel_for(cells, [&](long long lo, long long hi) { io_detail::convert<false>(h, w, lo, hi, shift, q); });
    };
    const double gb64 = double(n) * 8 / 1e9, gb32 = double(n) * 4 / 1e9;
    narrow(h64, w32);  // warm
    auto t0 = clk::now();
    narrow(h64, w32);
    auto t1 = clk::now();
    widen(h64b, w32);
    auto t2 = clk::now();
    const double narrow_gbs = gb64 / secs(t0, t1), widen_gbs = gb64 / secs(t1, t2);

    // both at once: two raw thread groups (the pool serialises callers)
    const int T = pool.threads();
    auto both = [&]() {
        std::vector<std::thread> th;
        const int half = std::max(1, T / 2);
        for (int i = 0; i < half; ++i)
            th.emplace_back([&, i] {
                const long long lo = cells * i / half, hi = cells * (i + 1) / half;
                io_detail::convert<true>(h64, w32b, lo, hi, shift, q);
            });
        for (int i = 0; i < half; ++i)
            th.emplace_back([&, i] {
                const long long lo = cells * i / half, hi = cells * (i + 1) / half;
                io_detail::convert<false>(h64b, w32, lo, hi, shift, q);
            });
        for (auto& t : th) t.join();
    };
    auto t3 = clk::now();
    both();
    auto t4 = clk::now();
    const double both_gbs = 2 * gb64 / secs(t3, t4);

    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaMemcpyAsync(d32, w32, n * 4, cudaMemcpyHostToDevice, s1));
    CK(cudaStreamSynchronize(s1));
    auto t5 = clk::now();
    CK(cudaMemcpyAsync(d32, w32, n * 4, cudaMemcpyHostToDevice, s1));
    CK(cudaStreamSynchronize(s1));
    auto t6 = clk::now();
    CK(cudaMemcpyAsync(w32b, d32b, n * 4, cudaMemcpyDeviceToHost, s1));
    CK(cudaStreamSynchronize(s1));
    auto t7 = clk::now();
    CK(cudaMemcpyAsync(d32, w32, n * 4, cudaMemcpyHostToDevice, s1));
    CK(cudaMemcpyAsync(w32b, d32b, n * 4, cudaMemcpyDeviceToHost, s2));
    CK(cudaStreamSynchronize(s1));
    CK(cudaStreamSynchronize(s2));
    auto t8 = clk::now();
    const double h2d = gb32 / secs(t5, t6), d2h = gb32 / secs(t6, t7), duplex = 2 * gb32 / secs(t7, t8);

    // DMA of w32 while the pool narrows into w32b (the pipeline's steady state)
    auto t9 = clk::now();
    CK(cudaMemcpyAsync(d32, w32, n * 4, cudaMemcpyHostToDevice, s1));
    narrow(h64, w32b);
    auto t10 = clk::now();
    CK(cudaStreamSynchronize(s1));
    auto t11 = clk::now();
    // D2H of d32b into w32b while the pool widens w32 into h64b
    CK(cudaMemcpyAsync(w32b, d32b, n * 4, cudaMemcpyDeviceToHost, s1));
    widen(h64b, w32);
    auto t12 = clk::now();
    CK(cudaStreamSynchronize(s1));
    auto t13 = clk::now();
    // fp64 straight over the link
    double* d64 = reinterpret_cast<double*>(d32);  // n*4 bytes: copy half of h64
    auto t14 = clk::now();
    CK(cudaMemcpyAsync(d64, h64, n * 4, cudaMemcpyHostToDevice, s1));
    CK(cudaStreamSynchronize(s1));
    auto t15 = clk::now();
    std::printf(
        "{\"gib_fp64\": %zu, \"threads\": %d, \"narrow_GBs64\": %.1f, \"widen_GBs64\": %.1f, \"narrow+widen_GBs64\": "
        "%.1f, \"h2d_GBs\": %.1f, \"d2h_GBs\": %.1f, \"duplex_GBs\": %.1f, \"h2d_with_narrow\": {\"narrow_s\": %.3f, "
        "\"dma_s\": %.3f, \"alone_narrow_s\": %.3f, \"alone_dma_s\": %.3f}, \"d2h_with_widen\": {\"widen_s\": %.3f, "
        "\"dma_s\": %.3f, \"alone_widen_s\": %.3f, \"alone_dma_s\": %.3f}, \"h2d_fp64_GBs\": %.1f}\n",
        gib, T, narrow_gbs, widen_gbs, both_gbs, h2d, d2h, duplex, secs(t9, t10), secs(t9, t11), secs(t0, t1),
        secs(t5, t6), secs(t11, t12), secs(t11, t13), secs(t1, t2), secs(t6, t7), gb32 / secs(t14, t15));
    return 0;
}
