// membw.cu -- attainable HBM bandwidth on this B200 for streaming patterns
// relevant to the LBM step (not part of the product; roofline context).
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        b[i] = __ldg(a + i);
}
__global__ void copy1(const float* __restrict__ a, float* __restrict__ b, size_t n) {
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i < n) b[i] = __ldg(a + i);
}
// 19 planes read + 19 planes written per thread (the SoA LBM access pattern)
__global__ void planes19(const float* __restrict__ a, float* __restrict__ b, size_t plane) {
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= plane) return;
    float v[19];
#pragma unroll
    for (int c = 0; c < 19; ++c) v[c] = __ldg(a + c * plane + i);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < 19; ++c) s += v[c];
#pragma unroll
    for (int c = 0; c < 19; ++c) b[c * plane + i] = v[c] * 0.999f + s * 1e-6f;
}
__global__ void planes19_cs(const float* __restrict__ a, float* __restrict__ b, size_t plane) {
    size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= plane) return;
    float v[19];
#pragma unroll
    for (int c = 0; c < 19; ++c) v[c] = __ldcs(a + c * plane + i);
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < 19; ++c) s += v[c];
#pragma unroll
    for (int c = 0; c < 19; ++c) __stcs(b + c * plane + i, v[c] * 0.999f + s * 1e-6f);
}

int main() {
    const size_t plane = size_t(512) * 512 * 512;  // 134M voxels
    const size_t n = plane * 19;                    // 10.2 GB per buffer
    float *a, *b;
    cudaMalloc(&a, n * 4);
    cudaMalloc(&b, n * 4);
    cudaMemset(a, 0, n * 4);
    cudaMemset(b, 0, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(e0);
        const int R = 10;
        for (int r = 0; r < R; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s %8.1f GB/s  (%.3f ms)\n", name, 2.0 * n * 4 * R / (ms * 1e-3) / 1e9, ms / R);
    };
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int g : {1, 2, 4, 8, 16})
        run((std::string("copy4 grid=") + std::to_string(g) + "xSM x1024").c_str(),
            [&] { copy4<<<sms * g, 1024>>>((const float4*)a, (float4*)b, n / 4); });
    run("copy1 (1 elem/thread)", [&] { copy1<<<unsigned((n + 255) / 256), 256>>>(a, b, n); });
    run("copy4 one-pass", [&] { copy4<<<unsigned((n / 4 + 255) / 256), 256>>>((const float4*)a, (float4*)b, n / 4); });
    for (int bs : {128, 256, 512})
        run((std::string("planes19 block=") + std::to_string(bs)).c_str(),
            [&] { planes19<<<unsigned((plane + bs - 1) / bs), bs>>>(a, b, plane); });
    run("planes19 ld/st .cs block=128", [&] { planes19_cs<<<unsigned((plane + 127) / 128), 128>>>(a, b, plane); });
    cudaMemcpy(b, a, n * 4, cudaMemcpyDeviceToDevice);
    run("cudaMemcpy D2D", [&] { cudaMemcpy(b, a, n * 4, cudaMemcpyDeviceToDevice); });
    return 0;
}
