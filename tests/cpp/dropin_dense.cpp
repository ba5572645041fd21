// Drop-in check: a reference-style driver (solver.cpp run_dense shape) on the
// C++ binding include/voxl_b200.hpp. Writes the final canonical field as raw
// doubles to argv[1]; tests/test_capi.py compares it with the oracle.
#include <cstdio>
#include <vector>

#include "voxl_b200.hpp"

int main(int argc, char** argv) {
    voxl_dense_desc d{};
    d.lattice = VOXL_D3Q19;
    d.nx = d.ny = d.nz = 16;
    d.tau = 0.56;
    d.scenario = VOXL_CAVITY;
    d.velocity[0] = 0.05;
    d.layout = VOXL_DISAG_SOA;
    d.partitions = 2;
    d.precision = VOXL_F64;
    d.halo_mode = VOXL_HALO_ZERO_COPY;
    d.first_partition = 0;
    d.local_partitions = -1;
    const std::size_t vq = std::size_t(16 * 16 * 16) * 19;
    // initial_canonical_state (solver.cpp:165-187): rest equilibrium f_i = w_i
    std::vector<double> init(vq);
    for (std::size_t v = 0; v < vq / 19; ++v)
        for (int i = 0; i < 19; ++i) init[v * 19 + i] = i == 0 ? 1.0 / 3.0 : (i < 7 ? 1.0 / 18.0 : 1.0 / 36.0);
    try {
        voxl::b200::DenseEngine a(d);
        a.fill_canonical(init);
        for (int step = 0; step < 20; ++step) {
            a.step();
            a.probe(step);  // run_dense probes every step (solver.cpp:249)
        }
        const std::vector<double> out = a.to_canonical(vq);
        if (argc > 1) {
            std::FILE* f = std::fopen(argv[1], "wb");
            std::fwrite(out.data(), sizeof(double), out.size(), f);
            std::fclose(f);
        }
        // the binding maps statuses back to the reference's exception types
        try {
            voxl_dense_desc bad = d;
            bad.tau = 0.4;
            voxl::b200::DenseEngine b(bad);
            return 3;
        } catch (const std::invalid_argument&) {
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    std::puts("dropin ok");
    return 0;
}
