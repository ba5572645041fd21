// voxl_b200 -- the C++ driver of the B200 engines (proj/tools/main.cpp's `run`
// and `verify` subcommands), built on the header-only binding voxl_b200.hpp.
//
//   voxl_b200 run --config FILE [--out DIR] [--precision fp64|fp32] [--devices 0,1,..] [--observed-trace]
//   voxl_b200 verify
//
// `run` parses the configuration with the reference's rules (config_from_json,
// solver.cpp:62-99: the same keys, defaults, validation and messages; nlohmann
// json as in the reference), executes voxl::b200::run and writes the
// reference's artifact set (main.cpp:30-55): fields.bin, fields.json,
// diagnostics.csv, config.json and, when present, ledger.csv, trace.json,
// dispatch.json, graph.dot, distribution.txt. fp64 (the default) is bitwise
// the reference's arithmetic, so the artifacts are byte-equal to the
// reference's (diagnostics.csv to 1e-11: the B200 probe sums exactly).
// Exit codes as main.cpp:248-268: 0 ok, 1 error / failed verification, 2
// configuration error.
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>

#include "json.hpp"
#include "voxl_b200.hpp"

namespace fs = std::filesystem;
using voxl::b200::ConfigError;
using voxl::b200::RunResult;
using voxl::b200::SolverConfig;

namespace {

int lattice_from(const std::string& s) {
    if (s == "D2Q9") return VOXL_D2Q9;
    if (s == "D3Q19") return VOXL_D3Q19;
    if (s == "D3Q27") return VOXL_D3Q27;
    throw std::invalid_argument("unknown lattice kind: " + s);  // lattice_kind_from_string (lattice.cpp)
}
int layout_from(const std::string& s) {
    if (s == "AoS") return VOXL_AOS;
    if (s == "SoA") return VOXL_SOA;
    if (s == "DisagSoA") return VOXL_DISAG_SOA;
    throw std::invalid_argument("unknown layout scheme: " + s);  // layout.cpp
}
int strategy_from(const std::string& s) {
    if (s == "naive") return VOXL_NAIVE;
    if (s == "disag_bitmask") return VOXL_DISAG_BITMASK;
    if (s == "disag_mem") return VOXL_DISAG_MEM;
    throw std::invalid_argument("unknown sparse strategy: " + s);  // sparse.cpp
}
int scenario_from(const std::string& s) {
    if (s == "lid_driven_cavity") return VOXL_CAVITY;
    if (s == "flow_over_obstacle") return VOXL_OBSTACLE;
    if (s == "periodic_box") return VOXL_PERIODIC;
    throw ConfigError("unknown scenario: " + s);  // scenario_from_string (solver.cpp:20-25)
}

/// config_from_json (solver.cpp:62-99).
SolverConfig config_from_json(const std::string& text) {
    nlohmann::json j;
    try {
        j = nlohmann::json::parse(text);
    } catch (const nlohmann::json::exception& e) {
        throw ConfigError(std::string("configuration is not valid JSON: ") + e.what());
    }
    SolverConfig c;
    c.precision = VOXL_F64;
    try {
        if (j.contains("lattice")) c.lattice = lattice_from(j.at("lattice"));
        if (j.contains("domain")) {
            const auto& d = j.at("domain");
            if (!d.is_array() || d.size() < 2 || d.size() > 3)
                throw ConfigError("domain must be [nx, ny] or [nx, ny, nz]");
            c.nx = d[0];
            c.ny = d[1];
            c.nz = d.size() == 3 ? int(d[2]) : 1;
        }
        if (j.contains("tau")) c.tau = j.at("tau");
        if (j.contains("scenario")) c.scenario = scenario_from(j.at("scenario"));
        if (j.contains("velocity")) {
            const auto& u = j.at("velocity");
            for (std::size_t a = 0; a < 3 && a < u.size(); ++a) c.velocity[a] = u[a];
        }
        if (j.contains("steps")) c.steps = j.at("steps");
        if (j.contains("layout")) c.layout = layout_from(j.at("layout"));
        if (j.contains("partitions")) c.partitions = j.at("partitions");
        if (j.contains("strategy")) c.strategy = strategy_from(j.at("strategy"));
        if (j.contains("obstacle_radius")) c.obstacle_radius = j.at("obstacle_radius");
        if (j.contains("levels")) c.levels = j.at("levels");
        if (j.contains("fused")) c.fused = j.at("fused");
        if (j.contains("seed")) c.seed = j.at("seed");
        if (j.contains("perturbation")) c.perturbation = j.at("perturbation");
    } catch (const ConfigError&) {
        throw;
    } catch (const std::exception& e) {
        throw ConfigError(std::string("configuration error: ") + e.what());
    }
    c.validate();
    return c;
}

/// config_to_json (solver.cpp:101-118).
std::string config_to_json(const SolverConfig& c) {
    nlohmann::json j;
    j["lattice"] = voxl::b200::lattice_name(c.lattice);
    j["domain"] = c.dim() == 2 ? nlohmann::json::array({c.nx, c.ny}) : nlohmann::json::array({c.nx, c.ny, c.nz});
    j["tau"] = c.tau;
    j["scenario"] = voxl::b200::scenario_name(c.scenario);
    j["velocity"] = {c.velocity[0], c.velocity[1], c.velocity[2]};
    j["steps"] = c.steps;
    j["layout"] = voxl::b200::layout_name(c.layout);
    j["partitions"] = c.partitions;
    j["strategy"] = voxl::b200::strategy_name(c.strategy);
    j["levels"] = c.levels;
    j["fused"] = c.fused;
    j["seed"] = c.seed;
    j["perturbation"] = c.perturbation;
    if (c.obstacle_radius > 0.0) j["obstacle_radius"] = c.obstacle_radius;
    return j.dump(2) + "\n";
}

std::string config_schema() {  // solver.cpp:120-135
    return "configuration keys (JSON object):\n"
           "  lattice          \"D2Q9\" | \"D3Q19\" | \"D3Q27\"\n"
           "  domain           [nx, ny] or [nx, ny, nz]\n"
           "  tau              relaxation time, > 0.5 (coarsest level for multires)\n"
           "  scenario         \"lid_driven_cavity\" | \"flow_over_obstacle\" | \"periodic_box\"\n"
           "  velocity         [ux, uy, uz]; lid velocity or inflow velocity, |u| <= 0.1\n"
           "  steps            time steps (coarse steps for multires)\n"
           "  layout           \"AoS\" | \"SoA\" | \"DisagSoA\" (dense runs)\n"
           "  partitions       1D partition count (dense runs)\n"
           "  strategy         \"naive\" | \"disag_bitmask\" | \"disag_mem\" (sparse runs)\n"
           "  obstacle_radius  sphere radius in voxels (flow_over_obstacle)\n"
           "  levels           resolution levels, 1-4 (lid_driven_cavity)\n"
           "  fused            multires kernel fusion on uniform blocks (bool)\n"
           "  seed             RNG seed for the periodic_box initial state\n"
           "  perturbation     relative amplitude of the initial perturbation\n";
}

std::string read_file(const fs::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ConfigError("cannot open config file: " + path.string());
    std::ostringstream os;
    os << in.rdbuf();
    return os.str();
}

void write_file(const fs::path& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary);
    out << text;
}

int cmd_run(const std::string& config_path, const std::string& out_dir, int precision, const std::vector<int>& devs,
            bool observed_trace) {
    SolverConfig config = config_from_json(read_file(config_path));
    config.precision = precision;
    config.devices = devs;
    config.observed_trace = observed_trace;
    RunResult result = voxl::b200::run(config);

    fs::create_directories(out_dir);
    const fs::path base(out_dir);
    {
        std::ofstream bin(base / "fields.bin", std::ios::binary);
        bin.write(reinterpret_cast<const char*>(result.field.data()),
                  std::streamsize(result.field.size() * sizeof(double)));
    }
    write_file(base / "fields.json", result.field_header_json);
    write_file(base / "diagnostics.csv", result.diagnostics_csv());
    write_file(base / "config.json", config_to_json(config));
    if (!result.ledger.empty()) write_file(base / "ledger.csv", result.ledger_csv());
    if (!result.trace.empty()) write_file(base / "trace.json", result.trace_json());
    if (!result.observed_trace_json.empty()) write_file(base / "trace_observed.json", result.observed_trace_json);
    if (!result.dispatch_json.empty()) write_file(base / "dispatch.json", result.dispatch_json);
    if (!result.graph_dot.empty()) write_file(base / "graph.dot", result.graph_dot);
    if (!result.distribution.empty()) write_file(base / "distribution.txt", result.distribution);

    if (!result.diagnostics.empty()) {
        const auto& last = result.diagnostics.back();
        std::cout << "run complete: " << config.steps << " steps, final mass " << last.mass << ", max |u| "
                  << last.max_speed << "\n";
    } else {
        std::cout << "run complete: 0 steps\n";
    }
    std::cout << "outputs written to " << out_dir << "\n";
    return 0;
}

int report_divergence(const std::vector<double>& a, const std::vector<double>& b, const std::string& what) {
    if (a.size() != b.size()) {
        std::cout << "FAIL " << what << ": size mismatch " << a.size() << " vs " << b.size() << "\n";
        return 1;
    }
    for (std::size_t i = 0; i < a.size(); ++i)
        if (std::memcmp(&a[i], &b[i], sizeof(double)) != 0) {
            std::cout << "FAIL " << what << ": first divergence at flat index " << i << " (" << a[i] << " vs "
                      << b[i] << ")\n";
            return 1;
        }
    std::cout << "PASS " << what << "\n";
    return 0;
}

/// cmd_verify (main.cpp:73-134) on the B200 engines, fp64: partition and
/// layout invariance against the one-partition engine (the reference checks
/// against reference_dense_run, which the one-partition engine is bitwise --
/// tests/test_dense_gpu.py), both multi-device schedules, the three sparse
/// strategies, fused vs staged multires.
int cmd_verify() {
    int failures = 0;
    {
        SolverConfig config;
        config.precision = VOXL_F64;
        config.lattice = VOXL_D3Q19;
        config.nx = config.ny = config.nz = 16;
        config.scenario = VOXL_CAVITY;
        config.tau = 0.56;
        config.velocity = {0.05, 0.0, 0.0};
        config.steps = 20;
        const std::vector<double> reference = voxl::b200::run(config).field;
        for (int layout : {VOXL_AOS, VOXL_SOA, VOXL_DISAG_SOA})
            for (int parts : {1, 2, 4}) {
                config.layout = layout;
                config.partitions = parts;
                config.devices.clear();
                failures += report_divergence(reference, voxl::b200::run(config).field,
                                              std::string("partition_invariance ") +
                                                  voxl::b200::layout_name(layout) + " x" + std::to_string(parts));
                config.devices.assign(std::size_t(parts), 0);
                failures += report_divergence(reference, voxl::b200::run(config).field,
                                              std::string("multi_stream_schedule ") +
                                                  voxl::b200::layout_name(layout) + " x" + std::to_string(parts));
            }
    }
    {
        SolverConfig config;
        config.precision = VOXL_F64;
        config.lattice = VOXL_D3Q19;
        config.nx = config.ny = config.nz = 16;
        config.scenario = VOXL_OBSTACLE;
        config.tau = 0.7;
        config.velocity = {0.04, 0.0, 0.0};
        config.steps = 10;
        config.strategy = VOXL_NAIVE;
        const RunResult naive = voxl::b200::run(config);
        for (int s : {VOXL_DISAG_BITMASK, VOXL_DISAG_MEM}) {
            config.strategy = s;
            failures += report_divergence(naive.field, voxl::b200::run(config).field,
                                          std::string("sparse_equivalence ") + voxl::b200::strategy_name(s));
        }
    }
    {
        SolverConfig config;
        config.precision = VOXL_F64;
        config.lattice = VOXL_D3Q19;
        config.nx = config.ny = config.nz = 16;
        config.scenario = VOXL_CAVITY;
        config.tau = 0.56;
        config.velocity = {0.05, 0.0, 0.0};
        config.steps = 5;
        config.levels = 2;
        config.fused = false;
        const RunResult staged = voxl::b200::run(config);
        config.fused = true;
        failures += report_divergence(staged.field, voxl::b200::run(config).field, "fusion_soundness 2-level");
    }
    if (failures == 0) std::cout << "all verification suites passed\n";
    return failures == 0 ? 0 : 1;
}

void usage() {
    std::cerr << "usage: voxl_b200 run --config FILE [--out DIR] [--precision fp64|fp32] [--devices 0,1,...] "
                 "[--observed-trace]\n"
                 "       voxl_b200 verify\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "run") {
            std::string config_path, out_dir = "out";
            int precision = VOXL_F64;
            std::vector<int> devices;
            bool observed_trace = false;
            for (int i = 2; i < argc; ++i) {
                const std::string a = argv[i];
                if (a == "--observed-trace") {
                    observed_trace = true;
                    continue;
                }
                if (i + 1 >= argc) {
                    usage();
                    return 2;
                }
                const std::string v = argv[++i];
                if (a == "--config") config_path = v;
                else if (a == "--out") out_dir = v;
                else if (a == "--precision") {
                    if (v != "fp64" && v != "fp32") {
                        usage();
                        return 2;
                    }
                    precision = v == "fp64" ? VOXL_F64 : VOXL_F32;
                } else if (a == "--devices") {
                    std::stringstream ss(v);
                    std::string tok;
                    while (std::getline(ss, tok, ',')) devices.push_back(std::stoi(tok));
                } else {
                    usage();
                    return 2;
                }
            }
            if (config_path.empty()) {
                usage();
                return 2;
            }
            return cmd_run(config_path, out_dir, precision, devices, observed_trace);
        }
        if (cmd == "verify") return cmd_verify();
        usage();
        return 2;
    } catch (const ConfigError& e) {
        std::cerr << "configuration error: " << e.what() << "\n" << config_schema();
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
