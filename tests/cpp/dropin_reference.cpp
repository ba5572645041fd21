// dropin_reference -- TEST DRIVER (built by oracle/Makefile `make dropin`,
// links the reference library oracle/_ref/libvoxl_ref.so and libvoxl_b200.so).
//
//   dropin_reference OUT_ROOT CONFIG.json...
//
// For each configuration: parse it with the reference's config_from_json,
// run the reference's voxl::run and the drop-in voxl::b200::run (fp64, the
// reference's own types, include/voxl_b200_reference.hpp), and write both
// artifact sets exactly as the reference CLI's `run` does (main.cpp:30-55)
// into OUT_ROOT/<name>/ref and OUT_ROOT/<name>/b200. The Python test compares
// the bytes.
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>

#include "voxl_b200_reference.hpp"

namespace fs = std::filesystem;

namespace {

std::string read_file(const fs::path& path) {
    std::ifstream in(path, std::ios::binary);
    std::ostringstream os;
    os << in.rdbuf();
    return os.str();
}

void write_file(const fs::path& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary);
    out << text;
}

void write_artifacts(const voxl::SolverConfig& config, const voxl::RunResult& result, const fs::path& base) {
    fs::create_directories(base);
    {
        std::ofstream bin(base / "fields.bin", std::ios::binary);
        bin.write(reinterpret_cast<const char*>(result.field.data()),
                  std::streamsize(result.field.size() * sizeof(double)));
    }
    write_file(base / "fields.json", result.field_header_json);
    write_file(base / "diagnostics.csv", result.diagnostics_csv());
    write_file(base / "config.json", voxl::config_to_json(config));
    if (!result.ledger.records().empty()) write_file(base / "ledger.csv", result.ledger.to_csv());
    if (!result.trace.events().empty()) write_file(base / "trace.json", result.trace.to_json());
    if (!result.dispatch_json.empty()) write_file(base / "dispatch.json", result.dispatch_json);
    if (!result.graph_dot.empty()) write_file(base / "graph.dot", result.graph_dot);
    if (!result.distribution.empty()) write_file(base / "distribution.txt", result.distribution);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::cerr << "usage: dropin_reference OUT_ROOT CONFIG.json...\n";
        return 2;
    }
    const fs::path root(argv[1]);
    try {
        for (int i = 2; i < argc; ++i) {
            const fs::path cfg_path(argv[i]);
            const voxl::SolverConfig config = voxl::config_from_json(read_file(cfg_path));
            const fs::path out = root / cfg_path.stem();
            write_artifacts(config, voxl::run(config), out / "ref");
            write_artifacts(config, voxl::b200::run(config), out / "b200");
            std::cout << "done " << cfg_path.stem().string() << "\n";
        }
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
