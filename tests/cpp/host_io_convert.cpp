// The host side of the fp32 canonical wire format (csrc/host_pool.hpp):
// AVX2 streaming-store conversions and the worker pool must give exactly the
// scalar IEEE results for every lattice width, alignment and slice split.
#include "host_pool.hpp"

#include <cstdio>
#include <random>
#include <vector>

using namespace voxl_b200;

int main() {
    std::mt19937_64 g(1);
    std::uniform_real_distribution<double> U(-1, 1);
    int bad = 0;
    for (int q : {2, 9, 19, 27})
        for (int off = 0; off < 8; ++off) {
            const long long vox = 5000 + off * 37, n = vox * q;
            std::vector<double> hbuf(n + 8), obuf(n + 8);
            std::vector<float> wbuf(n + 8);
            double* h = hbuf.data() + off % 4;
            float* w = wbuf.data() + off / 4;
            double* o = obuf.data() + off % 3;
            double sh[27];
            for (int c = 0; c < q; ++c) sh[c] = 1.0 / (c + 3);
            for (long long e = 0; e < n; ++e) h[e] = U(g);
            HostPool::get().parallel_for(vox, [&](long long lo, long long hi) {
                io_detail::convert<true>(h, w, lo, hi, sh, q);
            });
            HostPool::get().parallel_for(vox, [&](long long lo, long long hi) {
                io_detail::convert<false>(o, w, lo, hi, sh, q);
            });
            for (long long e = 0; e < n; ++e) {
                const float ref = float(h[e] - sh[e % q]);
                if (w[e] != ref || o[e] != double(ref) + sh[e % q]) {
                    std::printf("mismatch q=%d off=%d e=%lld\n", q, off, e);
                    ++bad;
                    break;
                }
            }
        }
    std::printf("host_io_convert: %s (%d threads)\n", bad ? "FAIL" : "ok", HostPool::get().threads());
    return bad ? 1 : 0;
}
