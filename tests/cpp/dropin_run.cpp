// Drop-in check of voxl::b200::run (the reference's run(), solver.cpp:369-375)
// through the C++ binding: a dense cavity over 2 partitions, the block-sparse
// wind tunnel and a 2-level multires cavity, fp64. For each run it writes
// <prefix>_<name>.bin (final field) and <prefix>_<name>.csv (step,mass,max_speed)
// and prints the report strings' sizes; tests/test_capi.py compares the fields
// with the oracle and the diagnostics with the Python front-end. A final
// unstable run must fail with the reference's "run aborted at step" text.
#include <cstdio>
#include <string>

#include "voxl_b200.hpp"

static void dump(const std::string& prefix, const char* name, const voxl::b200::RunResult& r) {
    std::FILE* f = std::fopen((prefix + "_" + name + ".bin").c_str(), "wb");
    std::fwrite(r.field.data(), sizeof(double), r.field.size(), f);
    std::fclose(f);
    f = std::fopen((prefix + "_" + name + ".csv").c_str(), "w");
    for (const auto& d : r.diagnostics) std::fprintf(f, "%d,%.17g,%.17g\n", d.step, d.mass, d.max_speed);
    std::fclose(f);
    std::printf("%s: field %zu, diag %zu, ledger %zu, dispatch %zu, dot %zu, distribution %s", name,
                r.field.size(), r.diagnostics.size(), r.ledger.size(), r.dispatch_json.size(), r.graph_dot.size(),
                r.distribution.empty() ? "-\n" : r.distribution.c_str());
}

int main(int argc, char** argv) {
    const std::string prefix = argc > 1 ? argv[1] : "dropin";
    try {
        voxl::b200::SolverConfig c;
        c.nx = c.ny = c.nz = 16;
        c.steps = 12;
        c.partitions = 2;
        c.precision = VOXL_F64;
        dump(prefix, "dense", voxl::b200::run(c));

        voxl::b200::SolverConfig s = c;
        s.scenario = VOXL_OBSTACLE;
        s.tau = 0.7;
        s.velocity = {0.04, 0.0, 0.0};
        s.steps = 5;
        s.partitions = 1;
        s.strategy = VOXL_DISAG_MEM;
        dump(prefix, "sparse", voxl::b200::run(s));

        voxl::b200::SolverConfig m = c;
        m.levels = 2;
        m.steps = 2;
        m.partitions = 1;
        dump(prefix, "multires", voxl::b200::run(m));

        voxl::b200::SolverConfig m2 = m;  // run_multires with a D2Q9 config
        m2.lattice = VOXL_D2Q9;
        m2.nx = 32;
        m2.ny = 32;
        m2.nz = 1;
        m2.tau = 0.6;
        m2.levels = 3;
        m2.steps = 3;
        dump(prefix, "multires2d", voxl::b200::run(m2));

        // a configuration that passes validate() and still blows up: the
        // periodic box at tau -> 1/2 with the largest allowed perturbation
        voxl::b200::SolverConfig bad = c;
        bad.nx = bad.ny = bad.nz = 12;
        bad.scenario = VOXL_PERIODIC;
        bad.velocity = {0.0, 0.0, 0.0};
        bad.tau = 0.5000001;
        bad.perturbation = 0.5;
        bad.seed = 3;
        bad.partitions = 2;
        bad.steps = 200;
        try {
            voxl::b200::run(bad);
            std::puts("unstable run did not abort");
            return 3;
        } catch (const std::runtime_error& e) {
            std::printf("abort: %s\n", e.what());
            if (std::string(e.what()).rfind("run aborted at step ", 0) != 0) return 4;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
    std::puts("dropin run ok");
    return 0;
}
