// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference library (libvoxl built
// from /root/reference/proj/src by oracle/Makefile).
//
// TEST INFRASTRUCTURE ONLY. This file is part of the oracle: it lets the Python
// tests, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// leg call the reference's own public C++ API (voxl::run, reference_dense_run,
// SparseLbmEngine, MultiResLbm, LayoutMap, classify_voxels) through ctypes.
// Nothing in the product path (paper_2503_07898_b200/) links or loads it.
//
// Entry points used (reference file:line):
//   voxl::config_from_json        proj/src/solver.cpp:59
//   voxl::run                     proj/src/solver.cpp:369
//   voxl::reference_dense_run     proj/src/solver.cpp:189
//   voxl::initial_canonical_state proj/src/solver.cpp:165
//   voxl::LayoutMap::build/to_json proj/src/layout.cpp:72,203
//   voxl::decompose/classify_voxels proj/src/partition.cpp:20,43
//   voxl::sparse::SparseLbmEngine proj/src/sparse.cpp:253
//   voxl::mres::MultiResGrid::build / MultiResLbm proj/src/multires.cpp:54,367
#include <algorithm>
#include <cstdint>
#include <unordered_map>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "voxl/commodel.hpp"
#include "voxl/layout.hpp"
#include "voxl/multires.hpp"
#include "voxl/partition.hpp"
#include "voxl/solver.hpp"
#include "voxl/sparse.hpp"

using namespace voxl;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}

int copy_text(const std::string& s, char* out, std::int64_t cap) {
    if (out && cap > 0) {
        std::size_t n = std::min<std::size_t>(s.size(), std::size_t(cap - 1));
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
    return int(s.size());
}

// Active set of run_sparse (solver.cpp:272-283), restated so the shim can hand
// the same voxels to SparseLbmEngine with a caller-chosen block edge.
std::vector<Vec3i> obstacle_active(const SolverConfig& config) {
    const int min_extent = std::min(config.domain.nx, std::min(config.domain.ny, config.domain.nz));
    const double radius = config.obstacle_radius > 0.0 ? config.obstacle_radius : min_extent / 5.0;
    const double cx = config.domain.nx / 2.0 - 0.5, cy = config.domain.ny / 2.0 - 0.5,
                 cz = config.domain.nz / 2.0 - 0.5;
    std::vector<Vec3i> active;
    Vec3i v;
    for (v.z = 0; v.z < config.domain.nz; ++v.z)
        for (v.y = 0; v.y < config.domain.ny; ++v.y)
            for (v.x = 0; v.x < config.domain.nx; ++v.x) {
                const double dx = v.x - cx, dy = v.y - cy, dz = v.z - cz;
                if (dx * dx + dy * dy + dz * dz > radius * radius) active.push_back(v);
            }
    return active;
}

// Band level map of run_multires (solver.cpp:319-335).
std::vector<int> band_level_map(const SolverConfig& config) {
    const int axis = config.partition_axis();
    const Extents dom = config.domain;
    std::vector<int> level_map(std::size_t(dom.volume()));
    Vec3i v;
    for (v.z = 0; v.z < dom.nz; ++v.z)
        for (v.y = 0; v.y < dom.ny; ++v.y)
            for (v.x = 0; v.x < dom.nx; ++v.x) {
                const int k = v[axis];
                int level = config.levels - 1;
                for (int l = 0; l < config.levels - 1; ++l)
                    if (k >= (dom[axis] >> (l + 1))) {
                        level = l;
                        break;
                    }
                level_map[std::size_t(linear_index(v, dom))] = level;
            }
    return level_map;
}

struct RunHandle {
    RunResult result;
};

struct SparseHandle {
    std::unique_ptr<sparse::SparseLbmEngine> engine;
    LatticeKind kind = LatticeKind::D3Q19;
};

struct MresHandle {
    std::unique_ptr<mres::MultiResLbm> engine;
    LatticeKind kind = LatticeKind::D3Q19;
};

} // namespace

extern "C" {

const char* vref_last_error() { return g_err.c_str(); }

// ---- solver-level API -------------------------------------------------------

/// voxl::run(config_from_json(json)). Returns an opaque handle or null.
void* vref_run(const char* json) {
    try {
        auto h = new RunHandle;
        h->result = run(config_from_json(json));
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}
std::int64_t vref_run_field_len(void* h) { return std::int64_t(((RunHandle*)h)->result.field.size()); }
void vref_run_field(void* h, double* out) {
    const auto& f = ((RunHandle*)h)->result.field;
    std::memcpy(out, f.data(), f.size() * sizeof(double));
}
int vref_run_diag_rows(void* h) { return int(((RunHandle*)h)->result.diagnostics.size()); }
void vref_run_diag(void* h, double* out) {
    const auto& d = ((RunHandle*)h)->result.diagnostics;
    for (std::size_t i = 0; i < d.size(); ++i) {
        out[3 * i] = d[i].step;
        out[3 * i + 1] = d[i].mass;
        out[3 * i + 2] = d[i].max_speed;
    }
}
/// what: 0 ledger csv, 1 trace json, 2 dispatch json, 3 graph dot, 4 distribution,
/// 5 field header json, 6 diagnostics csv.
int vref_run_text(void* h, int what, char* out, std::int64_t cap) {
    const RunResult& r = ((RunHandle*)h)->result;
    switch (what) {
        case 0: return copy_text(r.ledger.to_csv(), out, cap);
        case 1: return copy_text(r.trace.to_json(), out, cap);
        case 2: return copy_text(r.dispatch_json, out, cap);
        case 3: return copy_text(r.graph_dot, out, cap);
        case 4: return copy_text(r.distribution, out, cap);
        case 5: return copy_text(r.field_header_json, out, cap);
        case 6: return copy_text(r.diagnostics_csv(), out, cap);
    }
    return -1;
}
void vref_run_free(void* h) { delete (RunHandle*)h; }

/// reference_dense_run (solver.cpp:189); `out` must hold volume*q doubles.
int vref_reference_dense_run(const char* json, double* out) {
    try {
        const SolverConfig c = config_from_json(json);
        const std::vector<double> f = reference_dense_run(c);
        std::memcpy(out, f.data(), f.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// The same dense reference loop, with a caller-supplied initial canonical
/// state (fused_stream_collide, lbm.cpp:104-114, driven as solver.cpp:189-206).
int vref_dense_steps_from(const char* json, const double* init, double* out) {
    try {
        const SolverConfig c = config_from_json(json);
        const Lattice lat = build_lattice(c.lattice);
        const lbm::FlowRules rules = rules_for(c);
        lbm::DenseState a(c.domain, lat.q), b(c.domain, lat.q);
        std::memcpy(a.f.data(), init, a.f.size() * sizeof(double));
        const double inv_tau = 1.0 / c.tau;
        for (int s = 0; s < c.steps; ++s) {
            lbm::fused_stream_collide(lat, rules, inv_tau, a, b);
            std::swap(a, b);
        }
        std::memcpy(out, a.f.data(), a.f.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// A resident reference_dense_run state (solver.cpp:189-206 split into create /
/// step / read): the timed loop is the reference's own fused_stream_collide
/// sweep with A/B swap, without per-call allocation or copies (the CPU
/// baseline and bench.py's reference arm time this).
struct DenseHandle {
    Lattice lat;
    lbm::FlowRules rules;
    double inv_tau;
    lbm::DenseState a, b;
    DenseHandle(const SolverConfig& c)
        : lat(build_lattice(c.lattice)), rules(rules_for(c)), inv_tau(1.0 / c.tau), a(c.domain, lat.q),
          b(c.domain, lat.q) {}
};

void* vref_dense_create(const char* json, const double* init) {
    try {
        const SolverConfig c = config_from_json(json);
        auto* h = new DenseHandle(c);
        std::memcpy(h->a.f.data(), init, h->a.f.size() * sizeof(double));
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

int vref_dense_step(void* hv, int n) {
    auto* h = static_cast<DenseHandle*>(hv);
    try {
        for (int s = 0; s < n; ++s) {
            lbm::fused_stream_collide(h->lat, h->rules, h->inv_tau, h->a, h->b);
            std::swap(h->a, h->b);
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void vref_dense_read(void* hv, double* out) {
    auto* h = static_cast<DenseHandle*>(hv);
    std::memcpy(out, h->a.f.data(), h->a.f.size() * sizeof(double));
}

void vref_dense_free(void* hv) { delete static_cast<DenseHandle*>(hv); }

/// step_occ (partition.hpp:173) with the reference tests' generic kernels over a
/// PartitionedField pair: op 1 = identity (partition_test.cpp:189-191, lattice
/// q and TransferSets::for_lattice), op 2 = five-point Jacobi on a 2-component
/// field (partition_test.cpp:234-247, TransferSets::all(2)). `init`/`out` are
/// canonical (x fastest, component innermost). Returns step 0's ledger (alpha, beta).
int vref_occ_run(int op, int lattice, int nx, int ny, int nz, int parts, int axis, int scheme, int steps,
                 const double* init, double* out, std::int64_t* alpha, std::int64_t* beta) {
    try {
        const Extents domain{nx, ny, nz};
        const Decomposition d = decompose(domain, parts, axis);
        int card = 2;
        TransferSets transfer = TransferSets::all(2);
        if (op == 1) {
            const Lattice lat = build_lattice(LatticeKind(lattice));
            card = lat.q;
            transfer = TransferSets::for_lattice(lat, axis);
        }
        PartitionedField a(d, LayoutScheme(scheme), card, transfer);
        PartitionedField b(d, LayoutScheme(scheme), card, transfer);
        a.fill_canonical(std::vector<double>(init, init + std::size_t(domain.volume()) * card));
        auto identity = [&](const PartView& view, Vec3i v, double* o) {
            for (int c = 0; c < card; ++c) o[c] = view(v, c);
        };
        auto jacobi = [&](const PartView& view, Vec3i v, double* o) {
            const Vec3i offsets[4] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}};
            for (int c = 0; c < 2; ++c) {
                double sum = 0.0;
                int n = 0;
                for (const Vec3i& off : offsets) {
                    const Vec3i s = v + off;
                    if (s.x < 0 || s.x >= domain.nx || s.y < 0 || s.y >= domain.ny) continue;
                    sum += view(s, c);
                    ++n;
                }
                o[c] = 0.5 * view(v, c) + 0.5 * (n ? sum / n : 0.0);
            }
        };
        TransferLedger ledger;
        for (int s = 0; s < steps; ++s) {
            if (op == 1) step_occ(a, b, identity, &ledger, nullptr, s);
            else step_occ(a, b, jacobi, &ledger, nullptr, s);
            std::swap(a, b);
        }
        const std::vector<double> res = a.to_canonical();
        std::memcpy(out, res.data(), res.size() * sizeof(double));
        const auto st = ledger.step_stats(0);
        if (alpha) *alpha = st.alpha;
        if (beta) *beta = st.beta;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int vref_initial_state(const char* json, double* out) {
    try {
        const std::vector<double> f = initial_canonical_state(config_from_json(json));
        std::memcpy(out, f.data(), f.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int vref_probe(int lattice, const double* canonical, std::int64_t n, double* mass, double* max_u) {
    try {
        const Lattice lat = build_lattice(LatticeKind(lattice));
        std::vector<double> v(canonical, canonical + n);
        const lbm::Diagnostics d = lbm::probe_field(lat, v, 0);
        *mass = d.mass;
        *max_u = d.max_speed;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// config_to_json(config_from_json(json)) (solver.cpp:59-119), or the
/// ConfigError message (returned negative length).
int vref_config_roundtrip(const char* json, char* out, std::int64_t cap) {
    try {
        return copy_text(config_to_json(config_from_json(json)), out, cap);
    } catch (const std::exception& e) {
        g_err = e.what();
        copy_text(g_err, out, cap);
        return -int(g_err.size()) - 1;
    }
}

/// commodel tables (commodel.cpp:50-75) as `voxl model` prints them.
int vref_model_text(char* out, std::int64_t cap) {
    return copy_text(vector_field_table_csv() + lbm_table_csv(), out, cap);
}

// ---- lattice / layout / partition tables -------------------------------------

int vref_lattice_json(int lattice, char* out, std::int64_t cap) {
    return copy_text(lattice_to_json(build_lattice(LatticeKind(lattice))), out, cap);
}

/// LayoutMap::build + to_json. lattice >= 0 selects TransferSets::for_lattice
/// with cardinality q; lattice < 0 uses the generic build with `cardinality`.
int vref_layout_json(int scheme, int nx, int ny, int nz, int lattice, int cardinality, int axis,
                     char* out, std::int64_t cap) {
    try {
        LayoutMap m;
        if (lattice >= 0) {
            const Lattice lat = build_lattice(LatticeKind(lattice));
            m = LayoutMap::build(LayoutScheme(scheme), {nx, ny, nz}, lat.q, axis,
                                 TransferSets::for_lattice(lat, axis));
        } else {
            m = LayoutMap::build(LayoutScheme(scheme), {nx, ny, nz}, cardinality, axis);
        }
        return copy_text(m.to_json(), out, cap);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// Every address of the layout in (k from -1..n, then cross-section row-major,
/// component innermost) order, written as int64.
int vref_layout_addresses(int scheme, int nx, int ny, int nz, int lattice, int axis,
                          std::int64_t* out) {
    try {
        const Lattice lat = build_lattice(LatticeKind(lattice));
        const Extents shape{nx, ny, nz};
        const LayoutMap m = LayoutMap::build(LayoutScheme(scheme), shape, lat.q, axis,
                                             TransferSets::for_lattice(lat, axis));
        std::int64_t n = 0;
        const int a0 = axis == 0 ? 1 : 0, a1 = axis == 2 ? 1 : 2;
        for (int k = -1; k <= shape[axis]; ++k)
            for (int j = 0; j < shape[a1]; ++j)
                for (int i = 0; i < shape[a0]; ++i) {
                    Vec3i v;
                    v[axis] = k;
                    v[a0] = i;
                    v[a1] = j;
                    for (int c = 0; c < lat.q; ++c) out[n++] = m.address(v, c);
                }
        return int(n);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int vref_decompose(int nx, int ny, int nz, int parts, int axis, int periodic, int* slabs) {
    try {
        const Decomposition d = decompose({nx, ny, nz}, parts, axis, periodic != 0);
        for (int p = 0; p < parts; ++p) {
            slabs[2 * p] = d.slabs[p].first;
            slabs[2 * p + 1] = d.slabs[p].second;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int vref_classify_voxels(int nx, int ny, int nz, int parts, int axis, int periodic, int p,
                         std::uint8_t* out) {
    try {
        const Decomposition d = decompose({nx, ny, nz}, parts, axis, periodic != 0);
        const auto cls = classify_voxels(d, p);
        for (std::size_t i = 0; i < cls.size(); ++i) out[i] = std::uint8_t(cls[i]);
        return int(cls.size());
    } catch (const std::exception& e) {
        return fail(e);
    }
}

/// commodel layout_params (commodel.cpp:19-42): alpha, beta coefficient of s.
int vref_layout_params(int lattice, int scheme, std::int64_t s, std::int64_t* alpha,
                       std::int64_t* beta) {
    try {
        const CommParams p = layout_params(LatticeKind(lattice), LayoutScheme(scheme), s);
        *alpha = p.alpha;
        *beta = p.beta;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- block-sparse engine ------------------------------------------------------

/// SparseLbmEngine over run_sparse's obstacle active set (solver.cpp:268-299)
/// with an explicit block edge (the reference allows 1..4).
void* vref_sparse_create(const char* json, int block_edge) {
    try {
        const SolverConfig c = config_from_json(json);
        const Lattice lat = build_lattice(c.lattice);
        auto h = new SparseHandle;
        h->kind = c.lattice;
        h->engine = std::make_unique<sparse::SparseLbmEngine>(
            lat, sparse::SparseScenario::wind_tunnel(c.domain, c.tau, c.velocity),
            obstacle_active(c), block_edge, c.strategy);
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}
void vref_sparse_free(void* h) { delete (SparseHandle*)h; }
int vref_sparse_step(void* h, int n) {
    try {
        for (int i = 0; i < n; ++i) ((SparseHandle*)h)->engine->step();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
std::int64_t vref_sparse_num_active(void* h) { return ((SparseHandle*)h)->engine->grid().num_active(); }
int vref_sparse_num_blocks(void* h) { return ((SparseHandle*)h)->engine->grid().num_blocks(); }
/// Blocks in current list order: origin (3 int) + mask (uint64) + class (int).
void vref_sparse_blocks(void* h, int* origins, std::uint64_t* masks, int* classes) {
    const auto& e = *((SparseHandle*)h)->engine;
    const auto& blocks = e.grid().blocks();
    for (std::size_t b = 0; b < blocks.size(); ++b) {
        origins[3 * b] = blocks[b].origin.x;
        origins[3 * b + 1] = blocks[b].origin.y;
        origins[3 * b + 2] = blocks[b].origin.z;
        masks[b] = blocks[b].mask;
        classes[b] = int(e.classes().classes[b]);
    }
}
/// Arrangement (sparse.cpp:144-185): permutation, bitmask, voxel_meta_index.
std::int64_t vref_sparse_arrangement(void* h, int* permutation, std::uint8_t* bitmask,
                                     std::int32_t* meta_index) {
    const auto& a = ((SparseHandle*)h)->engine->arrangement();
    std::memcpy(permutation, a.permutation.data(), a.permutation.size() * sizeof(int));
    if (bitmask && !a.boundary_bitmask.empty())
        std::memcpy(bitmask, a.boundary_bitmask.data(), a.boundary_bitmask.size());
    if (meta_index && !a.voxel_meta_index.empty())
        std::memcpy(meta_index, a.voxel_meta_index.data(),
                    a.voxel_meta_index.size() * sizeof(std::int32_t));
    return a.boundary_voxel_count;
}
int vref_sparse_report_json(void* h, char* out, std::int64_t cap) {
    return copy_text(((SparseHandle*)h)->engine->report().to_json(), out, cap);
}
void vref_sparse_state(void* h, double* out) {
    const auto s = ((SparseHandle*)h)->engine->canonical_state();
    std::memcpy(out, s.data(), s.size() * sizeof(double));
}
/// set_state from a canonical (pack_coord-sorted) array.
void vref_sparse_set_state(void* h, const double* canonical) {
    auto& e = *((SparseHandle*)h)->engine;
    // Sorted active voxel list, identical to canonical_state's order.
    std::vector<std::pair<std::uint64_t, int>> order;
    const auto vox = e.grid().active_voxels();
    for (std::size_t i = 0; i < vox.size(); ++i) order.emplace_back(pack_coord(vox[i]), int(i));
    std::sort(order.begin(), order.end());
    std::unordered_map<std::uint64_t, std::int64_t> rank;
    for (std::size_t r = 0; r < order.size(); ++r) rank[order[r].first] = std::int64_t(r);
    const int qq = int(e.canonical_state().size() / vox.size());
    e.set_state([&](Vec3i v, double* vals) {
        const std::int64_t r = rank.at(pack_coord(v));
        for (int i = 0; i < qq; ++i) vals[i] = canonical[r * qq + i];
    });
}

// ---- multi-resolution engine --------------------------------------------------

/// MultiResLbm over run_multires's band level map (solver.cpp:312-340).
void* vref_mres_create(const char* json) {
    try {
        const SolverConfig c = config_from_json(json);
        const Lattice lat = build_lattice(c.lattice);
        mres::MultiResGrid grid =
            mres::MultiResGrid::build(c.domain, c.levels, lat, band_level_map(c), c.tau);
        auto h = new MresHandle;
        h->kind = c.lattice;
        h->engine = std::make_unique<mres::MultiResLbm>(lat, std::move(grid), rules_for(c), c.fused);
        return h;
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}
void vref_mres_free(void* h) { delete (MresHandle*)h; }
int vref_mres_step(void* h, int n) {
    try {
        for (int i = 0; i < n; ++i) ((MresHandle*)h)->engine->coarse_step();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}
int vref_mres_levels(void* h) { return ((MresHandle*)h)->engine->grid().num_levels(); }
std::int64_t vref_mres_num_active(void* h, int l) {
    return ((MresHandle*)h)->engine->grid().level(l).blocks.num_active();
}
int vref_mres_num_blocks(void* h, int l) {
    return ((MresHandle*)h)->engine->grid().level(l).blocks.num_blocks();
}
double vref_mres_tau(void* h, int l) { return ((MresHandle*)h)->engine->grid().level(l).tau; }
void vref_mres_blocks(void* h, int l, int* origins, std::uint64_t* masks, int* fusion_class) {
    const auto& e = *((MresHandle*)h)->engine;
    const auto& blocks = e.grid().level(l).blocks.blocks();
    for (std::size_t b = 0; b < blocks.size(); ++b) {
        origins[3 * b] = blocks[b].origin.x;
        origins[3 * b + 1] = blocks[b].origin.y;
        origins[3 * b + 2] = blocks[b].origin.z;
        masks[b] = blocks[b].mask;
        fusion_class[b] = int(e.fusion().block_class[l][b]);
    }
}
int vref_mres_num_ghosts(void* h, int l) { return int(((MresHandle*)h)->engine->grid().ghosts(l).size()); }
void vref_mres_ghosts(void* h, int l, int* out) {
    const auto& g = ((MresHandle*)h)->engine->grid().ghosts(l);
    for (std::size_t i = 0; i < g.size(); ++i) {
        out[6 * i] = g[i].cell.x;
        out[6 * i + 1] = g[i].cell.y;
        out[6 * i + 2] = g[i].cell.z;
        out[6 * i + 3] = g[i].parent.x;
        out[6 * i + 4] = g[i].parent.y;
        out[6 * i + 5] = g[i].parent.z;
    }
}
int vref_mres_num_pulls(void* h, int l) { return int(((MresHandle*)h)->engine->grid().pulls(l).size()); }
void vref_mres_pulls(void* h, int l, int* out) {
    const auto& p = ((MresHandle*)h)->engine->grid().pulls(l);
    for (std::size_t i = 0; i < p.size(); ++i) {
        out[7 * i] = p[i].voxel.x;
        out[7 * i + 1] = p[i].voxel.y;
        out[7 * i + 2] = p[i].voxel.z;
        out[7 * i + 3] = p[i].direction;
        out[7 * i + 4] = p[i].refined.x;
        out[7 * i + 5] = p[i].refined.y;
        out[7 * i + 6] = p[i].refined.z;
    }
}
std::int64_t vref_mres_state_len(void* h) {
    return std::int64_t(((MresHandle*)h)->engine->canonical_state().size());
}
void vref_mres_state(void* h, double* out) {
    const auto s = ((MresHandle*)h)->engine->canonical_state();
    std::memcpy(out, s.data(), s.size() * sizeof(double));
}
double vref_mres_total_mass(void* h) { return ((MresHandle*)h)->engine->total_mass(); }
int vref_mres_text(void* h, int what, char* out, std::int64_t cap) {
    const auto& e = *((MresHandle*)h)->engine;
    if (what == 0) return copy_text(e.graph().to_dot(), out, cap);
    return copy_text(e.distribution_report(), out, cap);
}

/// MultiResLbm::set_state (multires.hpp:158) per level from a canonical array in
/// canonical_state's order (levels finest first, cells by pack_coord).
void vref_mres_set_state(void* h, const double* canonical) {
    auto& e = *((MresHandle*)h)->engine;
    const int q = build_lattice(((MresHandle*)h)->kind).q;
    std::int64_t base = 0;
    for (int l = 0; l < e.grid().num_levels(); ++l) {
        const auto& blocks = e.grid().level(l).blocks;
        const int edge = blocks.edge();
        std::vector<std::uint64_t> keys;
        for (int b = 0; b < blocks.num_blocks(); ++b) {
            const sparse::Block& blk = blocks.blocks()[b];
            for (int local = 0; local < blocks.block_volume(); ++local) {
                if (!((blk.mask >> local) & 1)) continue;
                const Vec3i v{blk.origin.x + local % edge, blk.origin.y + (local / edge) % edge,
                              blk.origin.z + local / (edge * edge)};
                keys.push_back(pack_coord(v));
            }
        }
        std::sort(keys.begin(), keys.end());
        std::unordered_map<std::uint64_t, std::int64_t> rank;
        for (std::size_t r = 0; r < keys.size(); ++r) rank[keys[r]] = base + std::int64_t(r);
        e.set_state(l, [&](Vec3i v, double* vals) {
            const std::int64_t r = rank.at(pack_coord(v));
            for (int i = 0; i < q; ++i) vals[i] = canonical[r * q + i];
        });
        base += std::int64_t(keys.size());
    }
}

// ---- run()'s per-step loop on a resident engine --------------------------------

/// The loop body of run_dense / run_sparse / run_multires (solver.cpp:245-255,
/// 285-293, 341-349): step, then probe_field over the canonical state; the
/// first failure is rewrapped exactly as run() does ("run aborted at step N: "
/// + what()). kind 0 = a vref_dense_create handle (reference_dense_run's
/// fused_stream_collide step, whose bgk_relax throws the same
/// "macroscopic: non-positive density" as step_occ's), 1 = sparse, 2 =
/// multires. diag gets (mass, max_speed) per completed step; returns the
/// number of completed steps, msg the abort text ("" if none).
int vref_probed_steps(int kind, void* h, int steps, double* diag, char* msg, std::int64_t cap) {
    int step = 0;
    std::string text;
    for (; step < steps; ++step) {
        try {
            LatticeKind lk;
            std::vector<double> canonical;
            if (kind == 0) {
                auto* d = static_cast<DenseHandle*>(h);
                lbm::fused_stream_collide(d->lat, d->rules, d->inv_tau, d->a, d->b);
                std::swap(d->a, d->b);
                lk = d->lat.kind;
                canonical = d->a.f;
            } else if (kind == 1) {
                auto* s = static_cast<SparseHandle*>(h);
                s->engine->step();
                lk = s->kind;
                canonical = s->engine->canonical_state();
            } else {
                auto* m = static_cast<MresHandle*>(h);
                m->engine->coarse_step();
                lk = m->kind;
                canonical = m->engine->canonical_state();
            }
            const lbm::Diagnostics dg = lbm::probe_field(build_lattice(lk), canonical, step);
            diag[2 * step] = dg.mass;
            diag[2 * step + 1] = dg.max_speed;
        } catch (const std::runtime_error& e) {
            text = "run aborted at step " + std::to_string(step) + ": " + e.what();
            break;
        }
    }
    copy_text(text, msg, cap);
    return step;
}

} // extern "C"
