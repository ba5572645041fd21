// Persistent host worker pool for the I/O boundary's type conversions
// (fp64 canonical <-> fp32 wire format). Host code only: it converts the
// caller's buffers while the PCIe copies and the layout kernels run; the
// step operator itself never runs here.
#pragma once

#include <algorithm>
#include <cstdint>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace voxl_b200 {

class HostPool {
public:
    static HostPool& get() {
        // never destroyed: workers sleep on the condition variable until exit
        // (and a forked child, which has none of them, must not join them)
        static HostPool* pool = new HostPool;
        return *pool;
    }

    int threads() const { return int(workers_.size()) + 1; }

    /// f(lo, hi) over [0, n) split into threads() contiguous slices; returns
    /// when every slice is done. The calling thread takes slice 0.
    void parallel_for(long long n, const std::function<void(long long, long long)>& f) {
        const int t = threads();
        if (n <= 0) return;
        // a forked child inherits the pool object but not its threads
        if (t == 1 || n < 4096 || getpid() != owner_) {
            f(0, n);
            return;
        }
        std::lock_guard<std::mutex> one_job(call_m_);  // callers on other threads queue here
        {
            std::unique_lock<std::mutex> lk(m_);
            job_ = &f;
            n_ = n;
            pending_ = t - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0, n / t);
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

private:
    HostPool() : owner_(getpid()) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const int t = int(std::min(hw, 32u));
        for (int i = 1; i < t; ++i) workers_.emplace_back([this, i] { run(i); });
    }

    void run(int i) {
        long long seen = 0;
        for (;;) {
            const std::function<void(long long, long long)>* job;
            long long n;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                job = job_;
                n = n_;
            }
            const int t = threads();
            (*job)(n * i / t, n * (i + 1) / t);
            std::lock_guard<std::mutex> lk(m_);
            if (--pending_ == 0) done_.notify_one();
        }
    }

    pid_t owner_;
    std::vector<std::thread> workers_;
    std::mutex call_m_, m_;
    std::condition_variable cv_, done_;
    const std::function<void(long long, long long)>* job_ = nullptr;
    long long n_ = 0;
    long long gen_ = 0;
    int pending_ = 0;
};

/// Canonical I/O conversions of voxels [lo, hi) (q populations each):
///   narrow: w[e] = float(h[e] - shift[e % q])   (fp64 canonical -> fp32 wire)
///   widen:  h[e] = double(w[e]) + shift[e % q]  (fp32 wire -> fp64 canonical)
/// The same single IEEE subtraction / addition and round-to-nearest as the
/// device-side staging kernels. The AVX2 paths use streaming stores (no
/// read-for-ownership of the destination lines): host memory traffic, not
/// arithmetic, bounds these loops.
namespace io_detail {

template <bool Narrow>
inline void convert_scalar(double* h, float* w, long long e, long long end, int j, const double* shift, int q) {
    for (; e < end; ++e) {
        if constexpr (Narrow) w[e] = float(h[e] - shift[j]);
        else h[e] = double(w[e]) + shift[j];
        if (++j == q) j = 0;
    }
}

#if defined(__x86_64__)
template <bool Narrow>
__attribute__((target("avx2"))) inline void convert_avx2(double* h, float* w, long long e, long long end,
                                                          const double* shift, int q) {
    double rep[27 + 4];
    for (int j = 0; j < q + 4; ++j) rep[j] = shift[j % q];
    int j = 0;
    // scalar head until the destination is aligned for streaming stores
    const std::uintptr_t align = Narrow ? 15 : 31;
    while (e < end && (reinterpret_cast<std::uintptr_t>(Narrow ? static_cast<void*>(w + e)
                                                              : static_cast<void*>(h + e)) & align)) {
        if constexpr (Narrow) w[e] = float(h[e] - rep[j]);
        else h[e] = double(w[e]) + rep[j];
        ++e;
        if (++j == q) j = 0;
    }
    for (; e + 4 <= end; e += 4) {
        const __m256d sh = _mm256_loadu_pd(rep + j);
        if constexpr (Narrow) {
            _mm_stream_ps(w + e, _mm256_cvtpd_ps(_mm256_sub_pd(_mm256_loadu_pd(h + e), sh)));
        } else {
            _mm256_stream_pd(h + e, _mm256_add_pd(_mm256_cvtps_pd(_mm_loadu_ps(w + e)), sh));
        }
        j += 4;
        while (j >= q) j -= q;
    }
    _mm_sfence();
    convert_scalar<Narrow>(h, w, e, end, j, shift, q);
}
#endif

template <bool Narrow>
inline void convert(double* h, float* w, long long lo, long long hi, const double* shift, int q) {
#if defined(__x86_64__)
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2 && q <= 27) {
        convert_avx2<Narrow>(h, w, lo * q, hi * q, shift, q);
        return;
    }
#endif
    convert_scalar<Narrow>(h, w, lo * q, hi * q, 0, shift, q);
}

} // namespace io_detail

} // namespace voxl_b200
