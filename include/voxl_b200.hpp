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
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxl_b200.h"

namespace voxl {
namespace b200 {

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// ConfigError (solver.hpp:22-25): a configuration that fails validation.
struct ConfigError : std::runtime_error {
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
    /// Partition p on devices[p] (voxl_dense_create_multi); empty = current device.
    DenseEngine(const voxl_dense_desc& d, const std::vector<int>& devices, int graph_steps = 8) {
        if (devices.empty()) check(voxl_dense_create(&d, &h_));
        else check(voxl_dense_create_multi(&d, devices.data(), graph_steps, &h_));
    }
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
    // Dense runs: device of partition p (the single-process multi-device
    // engine). Empty: one partition per visible device when several are
    // visible (round robin), else every partition on the current device.
    std::vector<int> devices;
    int halo_mode = VOXL_HALO_ZERO_COPY;
    int graph_steps = 8;
    // Dense runs: also record the executed step schedule (voxl_dense_trace_json)
    bool observed_trace = false;

    int dim() const { return lattice == VOXL_D2Q9 ? 2 : 3; }
    int partition_axis() const { return dim() == 2 ? 1 : 2; }
    std::int64_t volume() const { return std::int64_t(nx) * ny * nz; }
    int q() const { return lattice == VOXL_D2Q9 ? 9 : (lattice == VOXL_D3Q19 ? 19 : 27); }
    int extent(int axis) const { return axis == 0 ? nx : (axis == 1 ? ny : nz); }

    /// SolverConfig::validate (solver.cpp:27-60): same checks, same message
    /// ("invalid configuration: " + every failed check), ConfigError.
    void validate() const {
        std::string err;
        const double speed =
            std::sqrt(velocity[0] * velocity[0] + velocity[1] * velocity[1] + velocity[2] * velocity[2]);
        if (!(tau > 0.5)) err += "tau must be > 0.5; ";
        if (speed > 0.1) err += "|velocity| must be <= 0.1 (stability envelope); ";
        if (steps < 0) err += "steps must be >= 0; ";
        if (nx < 2 || ny < 2) err += "domain extents must be >= 2; ";
        if (dim() == 2 && nz != 1) err += "D2Q9 requires nz == 1; ";
        if (dim() == 3 && nz < 2) err += "3D lattices require nz >= 2; ";
        if (partitions < 1) err += "partitions must be >= 1; ";
        if (partitions > 1 && extent(partition_axis()) < 2 * partitions)
            err += "partition axis too small for the partition count; ";
        if (levels < 1 || levels > 4) err += "levels must be in [1, 4]; ";
        if (levels > 1 && scenario != VOXL_CAVITY)
            err += "multi-level runs support the lid_driven_cavity scenario only; ";
        if (levels > 1 && partitions > 1) err += "multi-level runs are single-partition; ";
        if (levels > 1 && levels <= 4) {
            const int scale = 1 << (levels - 1);
            if (nx % scale || ny % scale || (dim() == 3 && nz % scale))
                err += "domain extents must divide the coarsest cell size; ";
        }
        if (perturbation < 0.0 || perturbation > 0.5) err += "perturbation must be in [0, 0.5]; ";
        if (scenario == VOXL_OBSTACLE) {
            const int min_extent = std::min(nx, std::min(ny, nz));
            const double r = obstacle_radius > 0.0 ? obstacle_radius : min_extent / 5.0;
            if (2.0 * r >= min_extent - 4) err += "obstacle does not fit the domain; ";
        }
        if (!err.empty()) throw ConfigError("invalid configuration: " + err);
    }
};

inline const char* lattice_name(int k) { return k == VOXL_D2Q9 ? "D2Q9" : (k == VOXL_D3Q19 ? "D3Q19" : "D3Q27"); }
inline const char* layout_name(int s) { return s == VOXL_AOS ? "AoS" : (s == VOXL_SOA ? "SoA" : "DisagSoA"); }
inline const char* strategy_name(int s) {
    return s == VOXL_NAIVE ? "naive" : (s == VOXL_DISAG_BITMASK ? "disag_bitmask" : "disag_mem");
}
inline const char* scenario_name(int s) {
    return s == VOXL_CAVITY ? "lid_driven_cavity" : (s == VOXL_OBSTACLE ? "flow_over_obstacle" : "periodic_box");
}

/// RunResult (solver.hpp:54-74).
struct RunResult {
    SolverConfig config;
    std::vector<double> field;
    struct DiagRow {
        int step;
        double mass;
        double max_speed;
    };
    std::string field_header_json;
    std::vector<DiagRow> diagnostics;
    std::vector<voxl_transfer_record> ledger;  // dense partitioned runs
    struct TraceEvent {                        // TraceLog::Event (partition.hpp:79-84)
        int step;
        int stage;
        std::string phase;
        int partition;
    };
    std::vector<TraceEvent> trace;             // dense runs: the OCC schedule's logical order
    std::string observed_trace_json;           // dense runs with config.observed_trace: the executed schedule
    std::string dispatch_json;                 // sparse runs
    std::string graph_dot;                     // multires runs
    std::string distribution;                  // multires runs

    /// RunResult::diagnostics_csv (solver.cpp:137-146).
    std::string diagnostics_csv() const {
        std::string out = "step,mass,max_u\n";
        char buf[80];
        for (const DiagRow& r : diagnostics) {
            std::snprintf(buf, sizeof buf, "%d,%.17g,%.17g\n", r.step, r.mass, r.max_speed);
            out += buf;
        }
        return out;
    }
    /// TransferLedger::to_csv (partition.cpp:90-97).
    std::string ledger_csv() const {
        std::string out = "step,src,dst,base_src,base_dst,elements\n";
        for (const auto& r : ledger)
            out += std::to_string(r.step) + "," + std::to_string(r.src) + "," + std::to_string(r.dst) + "," +
                   std::to_string(r.src_base) + "," + std::to_string(r.dst_base) + "," + std::to_string(r.elements) +
                   "\n";
        return out;
    }
    /// TraceLog::to_json (partition.cpp:98-109).
    std::string trace_json() const {
        std::string out = "[\n";
        for (std::size_t i = 0; i < trace.size(); ++i) {
            const TraceEvent& e = trace[i];
            out += "  {\"step\": " + std::to_string(e.step) + ", \"stage\": " + std::to_string(e.stage) +
                   ", \"phase\": \"" + e.phase + "\", \"partition\": " + std::to_string(e.partition) + "}" +
                   (i + 1 < trace.size() ? "," : "") + "\n";
        }
        return out + "]\n";
    }
};

namespace detail {

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
    d.halo_mode = c.halo_mode;
    d.first_partition = 0;
    d.local_partitions = -1;
    d.op = VOXL_OP_LBM;
    // the in-process PartitionedField over several GPUs (partition.hpp:92-126)
    std::vector<int> devices = c.devices;
    int visible = 1;
    check(voxl_device_count(&visible));
    if (devices.empty() && visible > 1 && c.partitions > 1)
        for (int p = 0; p < c.partitions; ++p) devices.push_back(p % visible);
    DenseEngine e(d, devices, c.graph_steps);
    std::vector<double> state(std::size_t(c.volume()) * c.q());
    check(voxl_initial_state(c.lattice, c.scenario, c.nx, c.ny, c.nz, c.seed, c.perturbation, state.data()));
    e.fill_canonical(state);
    // step_occ + probe_field per step; the rows come back once per batch and
    // the first failing step aborts with run()'s text (voxl_dense_step_probe_n)
    std::vector<voxl_diag> rows(std::size_t(std::max(c.steps, 0)));
    int done = 0;
    if (c.observed_trace) check(voxl_dense_trace_enable(e.handle(), 1));
    const int status = voxl_dense_step_probe_n(e.handle(), c.steps, rows.data(), &done);
    if (c.observed_trace) {
        r.observed_trace_json = text_of([](void* h, char* o, std::int64_t cap, std::int64_t* n) {
            return voxl_dense_trace_json(static_cast<voxl_dense*>(h), o, cap, n);
        }, e.handle());
        check(voxl_dense_trace_enable(e.handle(), 0));
    }
    for (int step = 0; step < done; ++step) {
        r.diagnostics.push_back({step, rows[std::size_t(step)].mass, rows[std::size_t(step)].max_speed});
        const auto recs = e.ledger(step);
        r.ledger.insert(r.ledger.end(), recs.begin(), recs.end());
    }
    // step_occ's logical schedule per step (partition.hpp:186-213,
    // partition.cpp:193): halo sends by partition, then private, then shared
    for (int step = 0; step < done; ++step) {
        for (int p = 0; p < c.partitions; ++p) r.trace.push_back({step, 1, "halo", p});
        for (int p = 0; p < c.partitions; ++p) r.trace.push_back({step, 1, "private", p});
        for (int p = 0; p < c.partitions; ++p) r.trace.push_back({step, 2, "shared", p});
    }
    check(status);
    r.field = e.to_canonical(state.size());
    r.field_header_json = "{\"shape\": [" + std::to_string(c.nx) + ", " + std::to_string(c.ny) + ", " +
                          std::to_string(c.nz) + "], \"lattice\": \"" + lattice_name(c.lattice) +
                          "\", \"representation\": \"dense\", \"layout\": \"" + layout_name(c.layout) +
                          "\", \"cardinality\": " + std::to_string(c.q()) +
                          ", \"order\": \"voxel-major (x fastest), component innermost\"}\n";
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
    // step + probe_field per step, fused on the device; the rows come back
    // once per batch and the first failing step aborts with run()'s text
    std::vector<voxl_diag> rows(std::size_t(std::max(c.steps, 0)));
    int done = 0;
    const int status = voxl_sparse_step_probe_n(e.handle(), c.steps, rows.data(), &done);
    for (int step = 0; step < done; ++step)
        r.diagnostics.push_back({step, rows[std::size_t(step)].mass, rows[std::size_t(step)].max_speed});
    check(status);
    r.field = e.canonical_state(c.q());
    r.field_header_json = "{\"shape\": [" + std::to_string(c.nx) + ", " + std::to_string(c.ny) + ", " +
                          std::to_string(c.nz) + "], \"lattice\": \"" + lattice_name(c.lattice) +
                          "\", \"representation\": \"block_sparse\", \"strategy\": \"" +
                          strategy_name(c.strategy) + "\", \"cardinality\": " + std::to_string(c.q()) +
                          ", \"active_voxels\": " + std::to_string(e.num_active()) +
                          ", \"order\": \"active cells sorted by (z, y, x), component innermost\"}\n";
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
    // coarse_step + probe_field per step, the probe fused into each level's
    // last sub-step; rows once per batch, run()'s text at the first failure
    std::vector<voxl_diag> rows(std::size_t(std::max(c.steps, 0)));
    int done = 0;
    const int status = voxl_mres_step_probe_n(e.handle(), c.steps, rows.data(), &done);
    for (int step = 0; step < done; ++step)
        r.diagnostics.push_back({step, rows[std::size_t(step)].mass, rows[std::size_t(step)].max_speed});
    check(status);
    r.field = e.canonical_state();
    // the execution graph and the distribution at the reference's block
    // granularity (edge 4, multires.cpp:54-365), whatever edge the engine runs
    voxl_mres_desc d4 = d;
    d4.block_edge = 4;
    d4.reference_tables = 1;
    d4.precision = VOXL_F64;
    voxl_mres_plan* plan = nullptr;
    check(voxl_mres_plan_create(&d4, level_map.data(), &plan));
    try {
        std::int64_t n = 0;
        for (int what : {c.fused ? 0 : 1, 2}) {
            check(voxl_mres_plan_text(plan, what, nullptr, 0, &n));
            std::string s(std::size_t(n) + 1, '\0');
            check(voxl_mres_plan_text(plan, what, &s[0], n + 1, &n));
            s.resize(std::size_t(n));
            if (what == 2) r.distribution = s + "\n";
            else r.graph_dot = s;
        }
    } catch (...) {
        voxl_mres_plan_destroy(plan);
        throw;
    }
    voxl_mres_plan_destroy(plan);
    r.field_header_json = "{\"shape\": [" + std::to_string(c.nx) + ", " + std::to_string(c.ny) + ", " +
                          std::to_string(c.nz) + "], \"lattice\": \"" + lattice_name(c.lattice) +
                          "\", \"representation\": \"multires\", \"levels\": " + std::to_string(c.levels) +
                          ", \"cardinality\": " + std::to_string(c.q()) +
                          ", \"order\": \"levels finest to coarsest, cells sorted by (z, y, x), component "
                          "innermost\"}\n";
    return r;
}

}  // namespace detail

/// run (solver.cpp:369-375): multires when levels > 1, block-sparse for flow
/// over an obstacle, the partitioned dense engine otherwise.
inline RunResult run(const SolverConfig& c) {
    c.validate();
    if (c.levels > 1) return detail::run_multires(c);
    if (c.scenario == VOXL_OBSTACLE) return detail::run_sparse(c);
    return detail::run_dense(c);
}

}  // namespace b200
}  // namespace voxl
