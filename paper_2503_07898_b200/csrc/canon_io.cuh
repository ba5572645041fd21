// canon_io.cuh -- host <-> device transfer of a canonical fp64 state, shared by
// the dense, block-sparse and multires engines (fill_canonical / to_canonical
// partition.cpp:111-161, set_state / canonical_state sparse.cpp:416-453,
// multires.cpp:578-598).
//
// The canonical state is cut into chunks of whole "rows" (planes for dense,
// runs of cells for sparse/multires). Two device staging slots and, for fp32
// engines, two pinned host slots form a pipeline on a dedicated copy stream:
// while one chunk crosses PCIe, the engine stream runs the layout kernel of the
// other and the host pool converts the next. fp32 engines put the fp32 storage
// format on the wire (host: R(f - w_i) in, double(g) + w_i out -- the same
// fp64 operation and rounding the device kernels apply), so the link carries
// half the bytes; the resulting field is bitwise the same either way.
#pragma once

#include "common.cuh"
#include "host_pool.hpp"

#include <algorithm>
#include <cstdint>

namespace voxl_b200 {

template <int Q>
struct ShiftQ {
    double v[Q];  // w_i for shifted fp32 storage, 0 otherwise
};

/// Slot-indexed block storage <-> canonical staging (BlockField layout
/// data[((b*Q)+c)*bv + local], sparse.hpp:62-86): canonical cell v lives at
/// slot slots[v] = b*bv + local. S = double: fp64 staging (shift applied
/// here); S = R: fp32 wire staging (shift applied on the host).
template <int Q, class R, bool ToDevice, class S>
__global__ void slot_io_kernel(R* buf, S* staging, const std::int64_t* slots, long long n, int lb,
                               const __grid_constant__ ShiftQ<Q> sh) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    const long long slot = slots[v], bv = 1ll << lb;
    const long long base = ((slot >> lb) * Q << lb) + (slot & (bv - 1));
    for (int c = 0; c < Q; ++c) {
        R* p = buf + base + c * bv;
        if constexpr (std::is_same_v<S, double>) {
            if constexpr (ToDevice) *p = R(staging[v * Q + c] - sh.v[c]);
            else staging[v * Q + c] = double(*p) + sh.v[c];
        } else {
            if constexpr (ToDevice) *p = staging[v * Q + c];
            else staging[v * Q + c] = *p;
        }
    }
}

template <int Q, class R>
void launch_slot_io(R* buf, void* staging, bool wire32, const std::int64_t* slots, long long n, int bv,
                    const double* shift, bool to_device, cudaStream_t st) {
    if (n <= 0) return;
    ShiftQ<Q> sh{};
    for (int c = 0; c < Q; ++c) sh.v[c] = shift[c];
    const int lb = log2_exact(bv);
    const unsigned blocks = unsigned((n + 255) / 256);
    if (wire32) {
        if constexpr (sizeof(R) == 4) {
            auto* s = static_cast<R*>(staging);
            if (to_device) slot_io_kernel<Q, R, true, R><<<blocks, 256, 0, st>>>(buf, s, slots, n, lb, sh);
            else slot_io_kernel<Q, R, false, R><<<blocks, 256, 0, st>>>(buf, s, slots, n, lb, sh);
        } else {
            throw std::logic_error("fp32 wire format on an fp64 engine");
        }
    } else {
        auto* s = static_cast<double*>(staging);
        if (to_device) slot_io_kernel<Q, R, true, double><<<blocks, 256, 0, st>>>(buf, s, slots, n, lb, sh);
        else slot_io_kernel<Q, R, false, double><<<blocks, 256, 0, st>>>(buf, s, slots, n, lb, sh);
    }
    VOXL_CUDA(cudaGetLastError());
}

class CanonPipe {
public:
    CanonPipe() = default;
    CanonPipe(const CanonPipe&) = delete;
    CanonPipe& operator=(const CanonPipe&) = delete;
    ~CanonPipe() {
        if (copy_) {
            cudaStreamSynchronize(copy_);
            for (int i = 0; i < 2; ++i) {
                cudaEventDestroy(copied_[i]);
                cudaEventDestroy(laid_[i]);
            }
            cudaStreamDestroy(copy_);
        }
        if (dev_) cudaFree(dev_);
        if (host_) cudaFreeHost(host_);
    }

    /// Move `rows` rows of `row_cells` canonical cells (q values each) between
    /// `host` (fp64, canonical order; nullptr for a device-only gather) and the
    /// engine. layout(r0, r1, slot, wire32) enqueues on `stream` the kernel
    /// that scatters (to_device) or gathers rows [r0, r1) from/to `slot`.
    /// consume(r0, r1, slot), if given, runs on `stream` after each gather
    /// instead of the D2H copy (device-side digests and reductions; fp64
    /// staging). wire32 selects the fp32 wire format (fp32 engines only).
    template <class Layout, class Consume>
    void run(double* host, long long rows, long long row_cells, int q, bool to_device, bool wire32,
             const double* shift, cudaStream_t stream, Layout&& layout, Consume&& consume,
             bool has_consume) {
        if (rows <= 0) return;
        if (host == nullptr) wire32 = false;
        const std::size_t wsize = wire32 ? sizeof(float) : sizeof(double);
        const std::size_t row_bytes = std::size_t(row_cells) * q * wsize;
        long long chunk = (long long)std::max<std::size_t>(1, (std::size_t(64) << 20) / std::max<std::size_t>(1, row_bytes));
        chunk = std::min(chunk, rows);
        const std::size_t slot_elems = std::size_t(chunk) * row_cells * q;
        const std::size_t need = 2 * slot_elems * wsize;
        if (dev_bytes_ < need) {
            if (dev_) VOXL_CUDA(cudaFree(dev_));
            VOXL_CUDA(cudaMalloc(&dev_, need));
            dev_bytes_ = need;
        }
        if (wire32 && host_bytes_ < need) {
            if (host_) VOXL_CUDA(cudaFreeHost(host_));
            VOXL_CUDA(cudaMallocHost(&host_, need));
            host_bytes_ = need;
        }
        if (!copy_) {
            VOXL_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                VOXL_CUDA(cudaEventCreateWithFlags(&copied_[i], cudaEventDisableTiming));
                VOXL_CUDA(cudaEventCreateWithFlags(&laid_[i], cudaEventDisableTiming));
            }
        }
        auto convert = [&](double* h, float* w, std::size_t elems, bool in) {
            HostPool::get().parallel_for((long long)(elems / q), [&](long long lo, long long hi) {
                if (in) io_detail::convert<true>(h, w, lo, hi, shift, q);
                else io_detail::convert<false>(h, w, lo, hi, shift, q);
            });
        };
        const bool copies = host != nullptr;
        if (copies) {  // the copy stream starts after everything already queued on the engine stream
            VOXL_CUDA(cudaEventRecord(laid_[0], stream));
            VOXL_CUDA(cudaStreamWaitEvent(copy_, laid_[0], 0));
        }
        auto host_slot = [&](int slot) { return static_cast<float*>(host_) + slot * slot_elems; };
        int pending = -1;  // fp32 wire gather: slot whose host widening is still due
        double* pending_host = nullptr;
        std::size_t pending_elems = 0;
        int i = 0;
        for (long long r0 = 0; r0 < rows; r0 += chunk, ++i) {
            const long long r1 = std::min(rows, r0 + chunk);
            const int slot = i & 1;
            void* dslot = static_cast<char*>(dev_) + slot * slot_elems * wsize;
            double* hchunk = host ? host + std::size_t(r0) * row_cells * q : nullptr;
            const std::size_t elems = std::size_t(r1 - r0) * row_cells * q;
            const std::size_t bytes = elems * wsize;
            if (to_device) {
                const void* src = hchunk;
                if (wire32) {
                    if (i >= 2) VOXL_CUDA(cudaEventSynchronize(copied_[slot]));  // pinned slot free again
                    convert(hchunk, host_slot(slot), elems, true);
                    src = host_slot(slot);
                }
                if (i >= 2) VOXL_CUDA(cudaStreamWaitEvent(copy_, laid_[slot], 0));  // device slot consumed
                VOXL_CUDA(cudaMemcpyAsync(dslot, src, bytes, cudaMemcpyHostToDevice, copy_));
                VOXL_CUDA(cudaEventRecord(copied_[slot], copy_));
                VOXL_CUDA(cudaStreamWaitEvent(stream, copied_[slot], 0));
                layout(r0, r1, dslot, wire32);
                VOXL_CUDA(cudaEventRecord(laid_[slot], stream));
                continue;
            }
            if (copies && i >= 2) VOXL_CUDA(cudaStreamWaitEvent(stream, copied_[slot], 0));  // slot drained
            layout(r0, r1, dslot, wire32);
            if (!copies) {
                if (has_consume) consume(r0, r1, dslot);
                continue;
            }
            VOXL_CUDA(cudaEventRecord(laid_[slot], stream));
            VOXL_CUDA(cudaStreamWaitEvent(copy_, laid_[slot], 0));
            void* dst = wire32 ? static_cast<void*>(host_slot(slot)) : static_cast<void*>(hchunk);
            VOXL_CUDA(cudaMemcpyAsync(dst, dslot, bytes, cudaMemcpyDeviceToHost, copy_));
            VOXL_CUDA(cudaEventRecord(copied_[slot], copy_));
            if (wire32) {  // widen the previous chunk while this one is gathered and copied
                if (pending >= 0) {
                    VOXL_CUDA(cudaEventSynchronize(copied_[pending]));
                    convert(pending_host, host_slot(pending), pending_elems, false);
                }
                pending = slot;
                pending_host = hchunk;
                pending_elems = elems;
            }
        }
        if (pending >= 0) {
            VOXL_CUDA(cudaEventSynchronize(copied_[pending]));
            convert(pending_host, host_slot(pending), pending_elems, false);
        }
        if (copies) VOXL_CUDA(cudaStreamSynchronize(copy_));
        VOXL_CUDA(cudaStreamSynchronize(stream));
    }

    template <class Layout>
    void run(double* host, long long rows, long long row_cells, int q, bool to_device, bool wire32,
             const double* shift, cudaStream_t stream, Layout&& layout) {
        run(host, rows, row_cells, q, to_device, wire32, shift, stream, layout,
            [](long long, long long, void*) {}, false);
    }

private:
    void* dev_ = nullptr;
    std::size_t dev_bytes_ = 0;
    void* host_ = nullptr;
    std::size_t host_bytes_ = 0;
    cudaStream_t copy_ = nullptr;
    cudaEvent_t copied_[2] = {nullptr, nullptr};
    cudaEvent_t laid_[2] = {nullptr, nullptr};
};

} // namespace voxl_b200
