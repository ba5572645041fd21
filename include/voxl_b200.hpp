// voxl_b200.hpp -- header-only C++ binding of the C-ABI (voxl_b200.h) that
// keeps the reference's names, value semantics and exception types, so a
// reference driver (proj/src/solver.cpp run_dense / run_sparse / run_multires)
// can switch engines by changing a type:
//
//   voxl::PartitionedField + step_occ + lbm::GatherKernel  -> voxl::b200::DenseEngine
//   voxl::sparse::SparseLbmEngine                          -> voxl::b200::SparseLbmEngine
//   voxl::mres::MultiResLbm                                -> voxl::b200::MultiResLbm
//
// voxl::b200::run(SolverConfig) is run() (solver.cpp:369-375) on these
// engines: same routing, initial state, per-step probe_field diagnostics,
// ledger, report / graph / distribution strings and "run aborted at step N:"
// error text.
//
// Status codes map back to the reference's exceptions (solver.hpp, lbm.cpp,
// layout.cpp): VOXL_INVALID_ARGUMENT -> std::invalid_argument, VOXL_OUT_OF_RANGE
// -> std::out_of_range, VOXL_DOMAIN -> std::domain_error, VOXL_INSTABILITY and
// VOXL_RUNTIME -> std::runtime_error (message text preserved, e.g. "run
// aborted at step N: ..."), VOXL_CUDA_ERROR -> voxl::b200::cuda_error.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxl_b200.h"

namespace voxl {
namespace b200 {

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int status) {
    if (status == VOXL_OK) return;
    const std::string msg = voxl_last_error();
    switch (status) {
        case VOXL_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case VOXL_OUT_OF_RANGE: throw std::out_of_range(msg);
        case VOXL_DOMAIN: throw std::domain_error(msg);
        case VOXL_CUDA_ERROR: throw cuda_error(msg);
        default: throw std::runtime_error(msg);
    }
}

struct Diagnostics {  // lbm::Diagnostics (lbm.hpp:137-141)
    double mass = 0.0;
    double max_speed = 0.0;
};

/// Dense partitioned engine: PartitionedField a/b + step_occ<GatherKernel>.
class DenseEngine {
public:
    explicit DenseEngine(const voxl_dense_desc& d) { check(voxl_dense_create(&d, &h_)); }
    ~DenseEngine() { voxl_dense_destroy(h_); }
    DenseEngine(const DenseEngine&) = delete;
    DenseEngine& operator=(const DenseEngine&) = delete;

    /// PartitionedField::fill_canonical (partition.cpp:143)
    void fill_canonical(const std::vector<double>& values) { check(voxl_dense_set_canonical(h_, values.data())); }
    /// PartitionedField::to_canonical (partition.cpp:123); `volume_q` = voxels * q
    std::vector<double> to_canonical(std::size_t volume_q) const {
        std::vector<double> out(volume_q);
        check(voxl_dense_get_canonical(h_, out.data()));
        return out;
    }
    /// step_occ x n (partition.hpp:173)
    void step(int n = 1) { check(voxl_dense_step(h_, n)); }
    /// lbm::probe_field on the current state; throws like the reference.
    Diagnostics probe(int step_index) const {
        voxl_diag d{};
        check(voxl_dense_probe(h_, &d));
        if (d.unstable)
            throw std::runtime_error("instability at step " + std::to_string(step_index) + ", voxel " +
                                     std::to_string(d.bad_voxel) + ", population " + std::to_string(d.bad_population));
        return {d.mass, d.max_speed};
    }
    /// The step's TransferLedger records (partition.cpp:163-206).
    std::vector<voxl_transfer_record> ledger(int step) const {
        int n = 0;
        check(voxl_dense_ledger(h_, step, nullptr, 0, &n));
        std::vector<voxl_transfer_record> r(std::size_t(n > 0 ? n : 1));
        check(voxl_dense_ledger(h_, step, r.data(), n, &n));
        r.resize(std::size_t(n));
        return r;
    }
    voxl_dense* handle() const { return h_; }

private:
    voxl_dense* h_ = nullptr;
};

/// sparse::SparseLbmEngine (sparse.hpp:175-213).
class SparseLbmEngine {
public:
    SparseLbmEngine(const voxl_sparse_desc& d, const std::vector<std::uint8_t>& active_mask) {
        check(voxl_sparse_create(&d, active_mask.data(), &h_));
    }
    ~SparseLbmEngine() { voxl_sparse_destroy(h_); }
    SparseLbmEngine(const SparseLbmEngine&) = delete;
    SparseLbmEngine& operator=(const SparseLbmEngine&) = delete;

    void step() { check(voxl_sparse_step(h_, 1)); }
    /// step_identity (sparse.cpp:396-404)
    void step_identity() { check(voxl_sparse_step_identity(h_, 1)); }
    std::int64_t num_active() const {
        std::int64_t n = 0;
        check(voxl_sparse_info(h_, &n, nullptr, nullptr, nullptr));
        return n;
    }
    /// canonical_state (sparse.cpp:416-438)
    std::vector<double> canonical_state(int q) const {
        std::vector<double> out(std::size_t(num_active()) * q);
        check(voxl_sparse_get_state(h_, out.data()));
        return out;
    }
    /// ExecutionReport::to_json (sparse.cpp:240-251)
    std::string report_json() const {
        std::int64_t n = 0;
        check(voxl_sparse_report_json(h_, nullptr, 0, &n));
        std::string s(std::size_t(n) + 1, '\0');
        check(voxl_sparse_report_json(h_, &s[0], n + 1, &n));
        s.resize(std::size_t(n));
        return s;
    }
    voxl_sparse* handle() const { return h_; }

private:
    voxl_sparse* h_ = nullptr;
};

/// mres::MultiResLbm (multires.hpp:138-190).
class MultiResLbm {
public:
    MultiResLbm(const voxl_mres_desc& d, const std::vector<std::int32_t>& level_of_cell) {
        check(voxl_mres_create(&d, level_of_cell.data(), &h_));
    }
    ~MultiResLbm() { voxl_mres_destroy(h_); }
    MultiResLbm(const MultiResLbm&) = delete;
    MultiResLbm& operator=(const MultiResLbm&) = delete;

    void coarse_step() { check(voxl_mres_step(h_, 1)); }
    std::vector<double> canonical_state() const {
        std::int64_t n = 0;
        check(voxl_mres_state_len(h_, &n));
        std::vector<double> out(static_cast<std::size_t>(n));
        check(voxl_mres_get_state(h_, out.data()));
        return out;
    }
    double total_mass() const {
        double m = 0;
        check(voxl_mres_total_mass(h_, &m));
        return m;
    }
    std::string distribution_report() const { return text(1); }
    std::string graph_dot() const { return text(0); }
    voxl_mres* handle() const { return h_; }

private:
    std::string text(int what) const {
        std::int64_t n = 0;
        check(voxl_mres_text(h_, what, nullptr, 0, &n));
        std::string s(std::size_t(n) + 1, '\0');
        check(voxl_mres_text(h_, what, &s[0], n + 1, &n));
        s.resize(std::size_t(n));
        return s;
    }
    voxl_mres* h_ = nullptr;
};

/// SolverConfig (solver.hpp:27-46) plus the two B200 choices the reference
/// does not have: the arithmetic precision (fp32 production, fp64 bitwise
/// parity) and the block edge of the sparse / multires engines.
struct SolverConfig {
    int lattice = VOXL_D3Q19;
    int nx = 32, ny = 32, nz = 32;
    double tau = 0.56;
    int scenario = VOXL_CAVITY;
    std::array<double, 3> velocity{0.05, 0.0, 0.0};
    int steps = 200;
    int layout = VOXL_DISAG_SOA;
    int partitions = 1;
    int strategy = VOXL_NAIVE;
    double obstacle_radius = 0.0;
    int levels = 1;
    bool fused = true;
    unsigned long seed = 42;
    double perturbation = 0.0;
    int precision = VOXL_F32;
    int block_edge = 8;

    int dim() const { return lattice == VOXL_D2Q9 ? 2 : 3; }
    int partition_axis() const { return dim() == 2 ? 1 : 2; }
    std::int64_t volume() const { return std::int64_t(nx) * ny * nz; }
    int q() const { return lattice == VOXL_D2Q9 ? 9 : (lattice == VOXL_D3Q19 ? 19 : 27); }
};

/// RunResult (solver.hpp:54-74).
struct RunResult {
    SolverConfig config;
    std::vector<double> field;
    struct DiagRow {
        int step;
        double mass;
        double max_speed;
    };
    std::vector<DiagRow> diagnostics;
    std::vector<voxl_transfer_record> ledger;  // dense partitioned runs
    std::string dispatch_json;                 // sparse runs
    std::string graph_dot;                     // multires runs
    std::string distribution;                  // multires runs
};

namespace detail {

inline void abort_if_unstable(const voxl_diag& d, int step) {
    if (!d.unstable) return;
    const std::string head = "run aborted at step " + std::to_string(step) + ": ";
    if (d.bad_population == VOXL_BAD_DENSITY)  // macroscopic's throw inside probe_field (lattice.cpp:124)
        throw std::runtime_error(head + "macroscopic: non-positive density");
    // probe_field's throw (lbm.cpp:124-128), rewrapped as run() does (solver.cpp:251-254)
    throw std::runtime_error(head + "instability at step " + std::to_string(step) + ", voxel " +
                             std::to_string(d.bad_voxel) + ", population " + std::to_string(d.bad_population));
}

inline std::string text_of(int (*get)(void*, char*, std::int64_t, std::int64_t*), void* h) {
    std::int64_t n = 0;
    check(get(h, nullptr, 0, &n));
    std::string s(std::size_t(n) + 1, '\0');
    check(get(h, &s[0], n + 1, &n));
    s.resize(std::size_t(n));
    return s;
}

/// run_dense (solver.cpp:225-266): step_occ + probe_field per step, fused on
/// the device (voxl_dense_step_probe).
inline RunResult run_dense(const SolverConfig& c) {
    RunResult r;
    r.config = c;
    voxl_dense_desc d{};
    d.lattice = c.lattice;
    d.nx = c.nx;
    d.ny = c.ny;
    d.nz = c.nz;
    d.tau = c.tau;
    d.scenario = c.scenario;
    for (int a = 0; a < 3; ++a) d.velocity[a] = c.velocity[a];
    d.layout = c.layout;
    d.partitions = c.partitions;
    d.precision = c.precision;
    d.halo_mode = VOXL_HALO_ZERO_COPY;
    d.first_partition = 0;
    d.local_partitions = -1;
    d.op = VOXL_OP_LBM;
    DenseEngine e(d);
    std::vector<double> state(std::size_t(c.volume()) * c.q());
    check(voxl_initial_state(c.lattice, c.scenario, c.nx, c.ny, c.nz, c.seed, c.perturbation, state.data()));
    e.fill_canonical(state);
    // step_occ + probe_field per step; the rows come back once per batch and
    // the first failing step aborts with run()'s text (voxl_dense_step_probe_n)
    std::vector<voxl_diag> rows(std::size_t(std::max(c.steps, 0)));
    int done = 0;
    const int status = voxl_dense_step_probe_n(e.handle(), c.steps, rows.data(), &done);
    for (int step = 0; step < done; ++step) {
        r.diagnostics.push_back({step, rows[std::size_t(step)].mass, rows[std::size_t(step)].max_speed});
        const auto recs = e.ledger(step);
        r.ledger.insert(r.ledger.end(), recs.begin(), recs.end());
    }
    check(status);
    r.field = e.to_canonical(state.size());
    return r;
}

/// run_sparse (solver.cpp:268-310): box minus sphere, wind tunnel, step +
/// probe_field per step; the dispatch report is the reference's edge-4 plan.
inline RunResult run_sparse(const SolverConfig& c) {
    RunResult r;
    r.config = c;
    std::vector<std::uint8_t> mask(std::size_t(c.volume()));
    std::int64_t active = 0;
    check(voxl_obstacle_mask(c.nx, c.ny, c.nz, c.obstacle_radius, mask.data(), &active));
    voxl_sparse_desc d{};
    d.lattice = c.lattice;
    d.nx = c.nx;
    d.ny = c.ny;
    d.nz = c.nz;
    d.tau = c.tau;
    for (int a = 0; a < 3; ++a) d.u_bc[a] = c.velocity[a];
    d.block_edge = c.block_edge;
    d.strategy = c.strategy;
    d.precision = c.precision;
    SparseLbmEngine e(d, mask);
    for (int step = 0; step < c.steps; ++step) {
        voxl_diag g{};
        check(voxl_sparse_step_probe(e.handle(), &g));  // step + probe_field, fused on the device
        abort_if_unstable(g, step);
        r.diagnostics.push_back({step, g.mass, g.max_speed});
    }
    r.field = e.canonical_state(c.q());
    voxl_sparse_desc d4 = d;
    d4.block_edge = 4;
    voxl_sparse_plan* plan = nullptr;
    check(voxl_sparse_plan_create(&d4, mask.data(), &plan));
    try {
        r.dispatch_json = text_of([](void* h, char* o, std::int64_t cap, std::int64_t* n) {
            return voxl_sparse_plan_report_json(static_cast<voxl_sparse_plan*>(h), o, cap, n);
        }, plan) + "\n";
    } catch (...) {
        voxl_sparse_plan_destroy(plan);
        throw;
    }
    voxl_sparse_plan_destroy(plan);
    return r;
}

/// run_multires (solver.cpp:312-367): band level map, coarse_step + probe_field
/// per step, graph and distribution strings.
inline RunResult run_multires(const SolverConfig& c) {
    RunResult r;
    r.config = c;
    std::vector<std::int32_t> level_map(std::size_t(c.volume()));
    check(voxl_band_level_map(c.nx, c.ny, c.nz, c.levels, c.partition_axis(), level_map.data()));
    voxl_mres_desc d{};
    d.lattice = c.lattice;
    d.nx = c.nx;
    d.ny = c.ny;
    d.nz = c.nz;
    d.levels = c.levels;
    d.tau = c.tau;
    for (int a = 0; a < 3; ++a) d.lid_u[a] = c.velocity[a];
    d.fused = c.fused ? 1 : 0;
    d.precision = c.precision;
    d.block_edge = c.block_edge;
    MultiResLbm e(d, level_map);
    for (int step = 0; step < c.steps; ++step) {
        e.coarse_step();
        voxl_diag g{};
        check(voxl_mres_probe(e.handle(), &g));
        abort_if_unstable(g, step);
        r.diagnostics.push_back({step, g.mass, g.max_speed});
    }
    r.field = e.canonical_state();
    r.graph_dot = e.graph_dot();
    r.distribution = e.distribution_report() + "\n";
    return r;
}

}  // namespace detail

/// run (solver.cpp:369-375): multires when levels > 1, block-sparse for flow
/// over an obstacle, the partitioned dense engine otherwise.
inline RunResult run(const SolverConfig& c) {
    if (c.levels > 1) return detail::run_multires(c);
    if (c.scenario == VOXL_OBSTACLE) return detail::run_sparse(c);
    return detail::run_dense(c);
}

}  // namespace b200
}  // namespace voxl
