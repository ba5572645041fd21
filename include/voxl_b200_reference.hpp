// voxl_b200_reference.hpp -- the drop-in on the reference's own types.
//
// A caller of the reference library (proj/include/voxl/solver.hpp) switches
// engines by calling voxl::b200::run instead of voxl::run: same argument
// (voxl::SolverConfig), same result type (voxl::RunResult with its
// TransferLedger, TraceLog, field header, diagnostics_csv(), dispatch /
// graph / distribution strings), same exceptions (voxl::ConfigError from
// SolverConfig::validate, std::runtime_error "run aborted at step N: ..."),
// and the same artifact bytes when fp64 is selected (tests/test_dropin_reference.py:
// all six shipped proj/configs/*.json, byte-equal fields.bin, fields.json,
// config.json, ledger.csv, trace.json, dispatch.json, graph.dot,
// distribution.txt; diagnostics.csv within 1e-11 -- the B200 probe sums
// exactly, the reference sequentially).
//
// Needs the reference's headers on the include path and its library at link
// time (TransferLedger::append / to_csv, TraceLog::to_json,
// RunResult::diagnostics_csv and SolverConfig::validate live there); the
// computation runs on libvoxl_b200 through voxl_b200.hpp.
//
//   solver.hpp:70  RunResult run(const SolverConfig&)  ->  voxl::b200::run(config [, precision])
#pragma once

#include "voxl/solver.hpp"
#include "voxl_b200.hpp"

namespace voxl {
namespace b200 {

/// voxl::SolverConfig (solver.hpp:27-46) -> the binding's config. The enum
/// values of the C-ABI are the reference's enum order.
inline SolverConfig from_reference(const voxl::SolverConfig& c, int precision = VOXL_F64) {
    SolverConfig b;
    b.lattice = static_cast<int>(c.lattice);
    b.nx = c.domain.nx;
    b.ny = c.domain.ny;
    b.nz = c.domain.nz;
    b.tau = c.tau;
    b.scenario = static_cast<int>(c.scenario);
    b.velocity = c.velocity;
    b.steps = c.steps;
    b.layout = static_cast<int>(c.layout);
    b.partitions = c.partitions;
    b.strategy = static_cast<int>(c.strategy);
    b.obstacle_radius = c.obstacle_radius;
    b.levels = c.levels;
    b.fused = c.fused;
    b.seed = c.seed;
    b.perturbation = c.perturbation;
    b.precision = precision;
    return b;
}

/// voxl::run (solver.cpp:369-375) on the B200 engines. precision VOXL_F64 is
/// bitwise the reference's arithmetic; VOXL_F32 is the production mode
/// (<= 1e-5 per population after 1000 steps).
inline voxl::RunResult run(const voxl::SolverConfig& config, int precision = VOXL_F64) {
    config.validate();  // the reference's own checks and ConfigError
    RunResult r = run(from_reference(config, precision));
    voxl::RunResult out;
    out.config = config;
    out.field = std::move(r.field);
    out.field_header_json = std::move(r.field_header_json);
    out.diagnostics.reserve(r.diagnostics.size());
    for (const auto& d : r.diagnostics) out.diagnostics.push_back({d.step, d.mass, d.max_speed});
    for (const auto& rec : r.ledger) {
        voxl::TransferRecord t;
        t.step = rec.step;
        t.src = rec.src;
        t.dst = rec.dst;
        t.src_span = {rec.src_base, rec.elements};
        t.dst_span = {rec.dst_base, rec.elements};
        t.elements = rec.elements;
        out.ledger.append(t);
    }
    for (const auto& e : r.trace) out.trace.append({e.step, e.stage, e.phase, e.partition});
    out.dispatch_json = std::move(r.dispatch_json);
    out.graph_dot = std::move(r.graph_dot);
    out.distribution = std::move(r.distribution);
    return out;
}

}  // namespace b200
}  // namespace voxl
