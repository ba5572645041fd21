// capi.cu -- the extern "C" boundary (include/voxl_b200.h).
#include "../../include/voxl_b200.h"

#include <cstring>
#include <numeric>
#include <random>
#include <string>

#include "common.cuh"
#include "dense.cuh"
#include "grid.hpp"
#include "lattice.cuh"
#include "multires.cuh"
#include "sparse.cuh"

using namespace voxl_b200;

struct voxl_dense {
    DenseEngine* eng;
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return VOXL_OK;
    } catch (const InstabilityError& e) {
        g_last_error = e.what();
        return VOXL_INSTABILITY;
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return VOXL_CUDA_ERROR;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return VOXL_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return VOXL_OUT_OF_RANGE;
    } catch (const std::domain_error& e) {
        g_last_error = e.what();
        return VOXL_DOMAIN;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return VOXL_RUNTIME;
    }
}

void put_text(const std::string& s, char* out, int64_t cap, int64_t* len) {
    if (len) *len = int64_t(s.size());
    if (out && cap > 0) {
        const std::size_t n = std::min<std::size_t>(s.size(), std::size_t(cap - 1));
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
}

void require(bool c, const char* msg) {
    if (!c) throw std::invalid_argument(msg);
}

/// Null handle / pointer arguments of an entry point -> VOXL_INVALID_ARGUMENT.
template <class... P>
void need(const char* fn, const P*... p) {
    const bool ok = ((p != nullptr) && ...);
    if (!ok) throw std::invalid_argument(std::string(fn) + ": null argument");
}

} // namespace

extern "C" {

const char* voxl_last_error(void) { return g_last_error.c_str(); }

int voxl_version(void) { return 1; }

int voxl_device_count(int* count) {
    return guarded([&] {
        require(count != nullptr, "voxl_device_count: null argument");
        VOXL_CUDA(cudaGetDeviceCount(count));
    });
}

int voxl_lattice_json(int lattice, char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        require(lattice >= 0 && lattice <= 2, "unknown lattice kind");
        const LatticeTable t = make_lattice(lattice);
        static const char* names[] = {"D2Q9", "D3Q19", "D3Q27"};
        std::string s = "{\n  \"kind\": \"" + std::string(names[lattice]) + "\",\n";
        s += "  \"dim\": " + std::to_string(t.dim) + ",\n  \"q\": " + std::to_string(t.q) + ",\n";
        s += "  \"velocities\": [";
        for (int i = 0; i < t.q; ++i)
            s += std::string(i ? ", " : "") + "[" + std::to_string(t.e[i][0]) + ", " + std::to_string(t.e[i][1]) +
                 ", " + std::to_string(t.e[i][2]) + "]";
        s += "],\n  \"weights\": [";
        for (int i = 0; i < t.q; ++i)
            s += std::string(i ? ", " : "") + "[" + std::to_string(t.wnum[i]) + ", " + std::to_string(t.wden[i]) + "]";
        s += "],\n  \"opposite\": [";
        for (int i = 0; i < t.q; ++i) s += std::string(i ? ", " : "") + std::to_string(t.opp[i]);
        s += "]\n}\n";
        put_text(s, out, cap, len);
    });
}

int voxl_layout_json(int scheme, int nx, int ny, int nz, int lattice, int cardinality, int axis, char* out,
                     int64_t cap, int64_t* len) {
    return guarded([&] {
        require(scheme >= 0 && scheme <= 2, "unknown layout scheme");
        LayoutMap m;
        if (lattice >= 0) {
            require(lattice <= 2, "unknown lattice kind");
            const LatticeTable t = make_lattice(lattice);
            m = LayoutMap::build(LayoutScheme(scheme), {nx, ny, nz}, t.q, axis,
                                 TransferSets::for_lattice(lattice, axis));
        } else {
            m = LayoutMap::build(LayoutScheme(scheme), {nx, ny, nz}, cardinality, axis,
                                 TransferSets::all(cardinality));
        }
        put_text(m.to_json(), out, cap, len);
    });
}

int voxl_layout_addresses(int scheme, int nx, int ny, int nz, int lattice, int axis, int64_t* out, int64_t cap,
                          int64_t* count) {
    return guarded([&] {
        require(lattice >= 0 && lattice <= 2, "unknown lattice kind");
        const LatticeTable t = make_lattice(lattice);
        const std::array<int, 3> shape{nx, ny, nz};
        const LayoutMap m =
            LayoutMap::build(LayoutScheme(scheme), shape, t.q, axis, TransferSets::for_lattice(lattice, axis));
        const int a0 = axis == 0 ? 1 : 0, a1 = axis == 2 ? 1 : 2;
        int64_t n = 0;
        for (int k = -1; k <= shape[axis]; ++k)
            for (int j = 0; j < shape[a1]; ++j)
                for (int i = 0; i < shape[a0]; ++i) {
                    std::array<int, 3> v{};
                    v[axis] = k;
                    v[a0] = i;
                    v[a1] = j;
                    for (int c = 0; c < t.q; ++c, ++n)
                        if (out && n < cap) out[n] = m.address(v, c);
                }
        if (count) *count = n;
    });
}

int voxl_decompose(int nx, int ny, int nz, int parts, int axis, int periodic, int* slabs) {
    return guarded([&] {
        const Decomposition d = decompose({nx, ny, nz}, parts, axis, periodic != 0);
        for (int p = 0; p < parts; ++p) {
            slabs[2 * p] = d.slabs[p].first;
            slabs[2 * p + 1] = d.slabs[p].second;
        }
    });
}

int voxl_classify_voxels(int nx, int ny, int nz, int parts, int axis, int periodic, int p, uint8_t* out,
                         int64_t cap) {
    return guarded([&] {
        const Decomposition d = decompose({nx, ny, nz}, parts, axis, periodic != 0);
        const auto cls = classify_voxels(d, p);
        require(int64_t(cls.size()) <= cap, "classify_voxels: output too small");
        std::memcpy(out, cls.data(), cls.size());
    });
}

namespace {
DenseConfig config_of(const voxl_dense_desc* desc) {
    require(desc != nullptr, "null descriptor");
    DenseConfig c;
    c.lattice = desc->lattice;
    c.domain = {desc->nx, desc->ny, desc->nz};
    c.tau = desc->tau;
    require(desc->scenario >= 0 && desc->scenario <= 2, "unknown scenario");
    c.scenario = Scenario(desc->scenario);
    c.velocity = {desc->velocity[0], desc->velocity[1], desc->velocity[2]};
    require(desc->layout >= 0 && desc->layout <= 2, "unknown layout scheme");
    c.layout = LayoutScheme(desc->layout);
    c.partitions = desc->partitions;
    require(desc->precision == VOXL_F32 || desc->precision == VOXL_F64, "unknown precision");
    c.precision = Precision(desc->precision);
    require(desc->halo_mode >= VOXL_HALO_ZERO_COPY && desc->halo_mode <= VOXL_HALO_NCCL, "unknown halo mode");
    c.halo = HaloMode(desc->halo_mode);
    c.first_partition = desc->first_partition;
    c.local_partitions = desc->local_partitions;
    require(desc->op >= VOXL_OP_LBM && desc->op <= VOXL_OP_JACOBI2, "unknown operator");
    c.op = Operator(desc->op);
    return c;
}
} // namespace

int voxl_dense_create(const voxl_dense_desc* desc, voxl_dense** out) {
    return guarded([&] {
        require(desc && out, "voxl_dense_create: null argument");
        *out = new voxl_dense{new DenseEngine(config_of(desc))};
    });
}

int voxl_dense_create_multi(const voxl_dense_desc* desc, const int* devices, int graph_steps, voxl_dense** out) {
    return guarded([&] {
        require(desc && devices && out, "voxl_dense_create_multi: null argument");
        DenseConfig c = config_of(desc);
        require(c.partitions >= 1, "voxl_dense_create_multi: partitions must be >= 1");
        c.devices.assign(devices, devices + c.partitions);
        c.graph_steps = graph_steps;
        *out = new voxl_dense{new DenseEngine(c)};
    });
}

int voxl_dense_device(voxl_dense* h, int p, int* device) {
    return guarded([&] {
        need("voxl_dense_device", h, device);
        require(p >= 0 && p < h->eng->config().partitions, "voxl_dense_device: no such partition");
        *device = h->eng->device_of(p);
    });
}

int voxl_dense_neighbors(voxl_dense* h, int p, int* upper, int* lower) {
    return guarded([&] {
        need("voxl_dense_neighbors", h, upper, lower);
        require(p >= 0 && p < h->eng->config().partitions, "voxl_dense_neighbors: no such partition");
        const auto l = h->eng->neighbors(p);
        *upper = l.first;
        *lower = l.second;
    });
}

int voxl_dense_set_neighbor_links(voxl_dense* h, int p, int upper, int lower) {
    return guarded([&] {
        need("voxl_dense_set_neighbor_links", h);
        h->eng->set_neighbor_links(p, upper, lower);
    });
}

int voxl_dense_destroy(voxl_dense* h) {
    return guarded([&] {
        if (!h) return;
        delete h->eng;
        delete h;
    });
}

int voxl_dense_set_canonical(voxl_dense* h, const double* host) {
    return guarded([&] {
        need("voxl_dense_set_canonical", h, host);
        h->eng->set_canonical(host);
    });
}

int voxl_dense_set_equilibrium(voxl_dense* h, double rho, const double* u) {
    return guarded([&] {
        need("voxl_dense_set_equilibrium", h, u);
        h->eng->set_equilibrium(rho, u);
    });
}

int voxl_dense_get_canonical(voxl_dense* h, double* host) {
    return guarded([&] {
        need("voxl_dense_get_canonical", h, host);
        h->eng->get_canonical(host);
    });
}

int voxl_dense_digest(voxl_dense* h, uint64_t* out2) {
    return guarded([&] {
        need("voxl_dense_digest", h, out2);
        unsigned long long d[2];
        h->eng->digest(d);
        out2[0] = d[0];
        out2[1] = d[1];
    });
}

int voxl_dense_set_planes(voxl_dense* h, const double* host, int k0, int k1) {
    return guarded([&] {
        need("voxl_dense_set_planes", h, host);
        h->eng->set_canonical_planes(host, k0, k1);
    });
}

int voxl_dense_get_planes(voxl_dense* h, double* host, int k0, int k1) {
    return guarded([&] {
        need("voxl_dense_get_planes", h, host);
        h->eng->get_canonical_planes(host, k0, k1);
    });
}

int voxl_dense_step(voxl_dense* h, int n) {
    return guarded([&] {
        need("voxl_dense_step", h);
        h->eng->step(n);
    });
}

int voxl_dense_enqueue(voxl_dense* h, int n) {
    return guarded([&] {
        need("voxl_dense_enqueue", h);
        h->eng->enqueue_steps(n);
    });
}

int voxl_dense_timed_steps(voxl_dense* h, int n, double* total_ms, double* kernel_ms) {
    return guarded([&] {
        need("voxl_dense_timed_steps", h, total_ms);
        *total_ms = h->eng->timed_steps(n, kernel_ms);
    });
}

int voxl_dense_synchronize(voxl_dense* h) {
    return guarded([&] {
        need("voxl_dense_synchronize", h);
        h->eng->check_errors();
    });
}

int voxl_dense_step_probe(voxl_dense* h, voxl_diag* out) {
    return guarded([&] {
        need("voxl_dense_step_probe", h, out);
        const DenseDiag d = h->eng->step_probe();
        out->mass = d.mass;
        out->max_speed = d.max_speed;
        out->unstable = d.unstable;
        out->bad_population = d.bad_population;
        out->bad_voxel = d.bad_voxel;
    });
}

namespace {
/// The healthy rows of a probed batch in the C-ABI's row type.
void fill_rows(const DenseDiag* r, int done, voxl_diag* rows) {
    for (int s = 0; s < done; ++s) {
        rows[s] = voxl_diag{};
        rows[s].mass = r[s].mass;
        rows[s].max_speed = r[s].max_speed;
        rows[s].bad_population = -1;
        rows[s].bad_voxel = -1;
    }
}
} // namespace

int voxl_dense_step_probe_n(voxl_dense* h, int n, voxl_diag* rows, int* completed) {
    if (completed) *completed = 0;
    return guarded([&] {
        need("voxl_dense_step_probe_n", h);
        if (n > 0) need("voxl_dense_step_probe_n", rows);
        std::vector<DenseDiag> r(std::size_t(std::max(n, 0)));
        std::string msg;
        const int done = h->eng->step_probe_n(n, r.data(), &msg);
        fill_rows(r.data(), done, rows);
        if (completed) *completed = done;
        if (done < n) throw InstabilityError(msg);
    });
}

int voxl_dense_trace_enable(voxl_dense* h, int on) {
    return guarded([&] {
        need("voxl_dense_trace_enable", h);
        h->eng->trace_enable(on != 0);
    });
}

int voxl_dense_trace_json(voxl_dense* h, char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        need("voxl_dense_trace_json", h);
        put_text(h->eng->trace_json(), out, cap, len);
    });
}

int voxl_dense_probe(voxl_dense* h, voxl_diag* out) {
    return guarded([&] {
        need("voxl_dense_probe", h, out);
        const DenseDiag d = h->eng->probe();
        out->mass = d.mass;
        out->max_speed = d.max_speed;
        out->unstable = d.unstable;
        out->bad_population = d.bad_population;
        out->bad_voxel = d.bad_voxel;
    });
}

int voxl_dense_ledger(voxl_dense* h, int step, voxl_transfer_record* out, int cap, int* count) {
    return guarded([&] {
        need("voxl_dense_ledger", h);
        const auto recs = h->eng->ledger_records(step);
        if (count) *count = int(recs.size());
        for (int i = 0; i < int(recs.size()) && i < cap; ++i)
            out[i] = {recs[i].step, recs[i].src, recs[i].dst, recs[i].src_span.base, recs[i].dst_span.base,
                      recs[i].elements};
    });
}

int voxl_dense_plan_ledger(const voxl_dense_desc* desc, int step, voxl_transfer_record* out, int cap,
                           int* count) {
    return guarded([&] {
        const DenseConfig c = config_of(desc);
        const OperatorShape os = operator_shape(c);
        const Decomposition d = decompose(c.domain, c.partitions, os.axis, c.scenario == Scenario::PeriodicBox);
        std::vector<LayoutMap> maps;
        for (int p = 0; p < c.partitions; ++p) {
            std::array<int, 3> shape = c.domain;
            shape[os.axis] = d.thickness(p);
            maps.push_back(LayoutMap::build(c.layout, shape, os.q, os.axis, os.transfer));
        }
        const auto recs = halo_records(d, maps, step);
        if (count) *count = int(recs.size());
        for (int i = 0; i < int(recs.size()) && i < cap; ++i)
            out[i] = {recs[i].step, recs[i].src, recs[i].dst, recs[i].src_span.base, recs[i].dst_span.base,
                      recs[i].elements};
    });
}

int voxl_dense_layout_json(voxl_dense* h, int p, char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        need("voxl_dense_layout_json", h);
        require(p >= 0 && p < h->eng->config().partitions, "bad partition");
        put_text(h->eng->layout(p).to_json(), out, cap, len);
    });
}

int voxl_dense_steps_done(voxl_dense* h, int* steps) {
    return guarded([&] {
        need("voxl_dense_steps_done", h);
        *steps = h->eng->steps_done();
    });
}

int voxl_dense_buffer(voxl_dense* h, int p, int which, void** ptr, size_t* bytes) {
    return guarded([&] {
        need("voxl_dense_buffer", h);
        require(p >= 0 && p < h->eng->config().partitions, "bad partition");
        *ptr = h->eng->buffer(p, which);
        if (bytes) *bytes = h->eng->buffer_bytes(p);
    });
}

int voxl_dense_stream(voxl_dense* h, void** stream) {
    return guarded([&] {
        need("voxl_dense_stream", h);
        *stream = (void*)h->eng->stream();
    });
}

int voxl_dense_shared_stream(voxl_dense* h, void** stream) {
    return guarded([&] {
        need("voxl_dense_shared_stream", h);
        require(h->eng->shared_stream() != nullptr, "shared_stream: call voxl_dense_enable_distributed first");
        *stream = (void*)h->eng->shared_stream();
    });
}

int voxl_dense_attach_peer(voxl_dense* h, int p, void* b0, void* b1) {
    return guarded([&] {
        need("voxl_dense_attach_peer", h);
        h->eng->attach_peer(p, b0, b1);
    });
}

int voxl_dense_raw_buffer(voxl_dense* h, int p, int w, void** ptr) {
    return guarded([&] {
        need("voxl_dense_raw_buffer", h);
        require(p >= 0 && p < h->eng->config().partitions && (w == 0 || w == 1), "bad partition/buffer");
        *ptr = h->eng->raw_buffer(p, w);
    });
}

int voxl_dense_enable_distributed(voxl_dense* h, void** flags) {
    return guarded([&] {
        need("voxl_dense_enable_distributed", h);
        h->eng->enable_distributed();
        if (flags) *flags = h->eng->flag_words();
    });
}

int voxl_dense_attach_flags(voxl_dense* h, void* upper_slot, void* lower_slot) {
    return guarded([&] {
        need("voxl_dense_attach_flags", h);
        h->eng->attach_flags(static_cast<std::uint32_t*>(upper_slot), static_cast<std::uint32_t*>(lower_slot));
    });
}

int voxl_dense_halo_push(voxl_dense* h) {
    return guarded([&] {
        need("voxl_dense_halo_push", h);
        h->eng->halo_push();
    });
}

int voxl_dense_owned_voxels(voxl_dense* h, int64_t* voxels) {
    return guarded([&] {
        need("voxl_dense_owned_voxels", h, voxels);
        *voxels = h->eng->owned_voxels();
    });
}

int voxl_obstacle_mask(int nx, int ny, int nz, double radius, uint8_t* out, int64_t* active) {
    return guarded([&] {
        // solver.cpp:272-283 (same double arithmetic)
        const int mn = std::min(nx, std::min(ny, nz));
        const double r = radius > 0.0 ? radius : mn / 5.0;
        const double cx = nx / 2.0 - 0.5, cy = ny / 2.0 - 0.5, cz = nz / 2.0 - 0.5;
        int64_t n = 0;
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    const double dx = x - cx, dy = y - cy, dz = z - cz;
                    const bool a = dx * dx + dy * dy + dz * dz > r * r;
                    out[(int64_t(z) * ny + y) * nx + x] = a;
                    n += a;
                }
        if (active) *active = n;
    });
}

int voxl_sparse_create(const voxl_sparse_desc* d, const uint8_t* active, voxl_sparse** out) {
    return guarded([&] {
        require(d && active && out, "voxl_sparse_create: null argument");
        SparseConfig c;
        c.lattice = d->lattice;
        c.domain = {d->nx, d->ny, d->nz};
        c.tau = d->tau;
        c.u_bc = {d->u_bc[0], d->u_bc[1], d->u_bc[2]};
        c.edge = d->block_edge;
        require(d->strategy >= 0 && d->strategy <= 2, "unknown sparse strategy");
        c.strategy = Strategy(d->strategy);
        require(d->precision == VOXL_F32 || d->precision == VOXL_F64, "unknown precision");
        c.precision = Precision(d->precision);
        *out = reinterpret_cast<voxl_sparse*>(new SparseEngine(c, active));
    });
}

int voxl_sparse_destroy(voxl_sparse* h) {
    return guarded([&] { delete reinterpret_cast<SparseEngine*>(h); });
}

static SparseEngine* SP(voxl_sparse* h) { return reinterpret_cast<SparseEngine*>(h); }
static SparseTables* PL(voxl_sparse_plan* p) { return reinterpret_cast<SparseTables*>(p); }

int voxl_sparse_plan_create(const voxl_sparse_desc* d, const uint8_t* active, voxl_sparse_plan** out) {
    return guarded([&] {
        require(d && active && out, "voxl_sparse_plan_create: null argument");
        require(d->strategy >= 0 && d->strategy <= 2, "unknown sparse strategy");
        require(d->lattice >= 0 && d->lattice <= 2, "unknown lattice kind");
        auto* t = new SparseTables(SparseTables::build({d->nx, d->ny, d->nz}, active, d->block_edge,
                                                       Strategy(d->strategy), make_lattice(d->lattice).q));
        *out = reinterpret_cast<voxl_sparse_plan*>(t);
    });
}

int voxl_sparse_plan_destroy(voxl_sparse_plan* p) {
    return guarded([&] { delete PL(p); });
}

int voxl_sparse_plan_of(voxl_sparse* h, voxl_sparse_plan** out) {
    return guarded([&] {
        need("voxl_sparse_plan_of", h);
        *out = reinterpret_cast<voxl_sparse_plan*>(&SP(h)->tables());
    });
}

int voxl_sparse_plan_info(voxl_sparse_plan* p, int64_t* na, int* nb, int64_t* nbd, int64_t* nnb) {
    return guarded([&] {
        if (na) *na = PL(p)->grid.num_active();
        if (nb) *nb = PL(p)->grid.num_blocks();
        if (nbd) *nbd = PL(p)->classes.n_boundary;
        if (nnb) *nnb = PL(p)->classes.n_non_boundary;
    });
}

int voxl_sparse_plan_blocks(voxl_sparse_plan* p, int* origins, uint64_t* masks, uint8_t* classes) {
    return guarded([&] {
        const BlockGrid& g = PL(p)->grid;
        for (int b = 0; b < g.num_blocks(); ++b) {
            if (origins)
                for (int a = 0; a < 3; ++a) origins[3 * b + a] = g.blocks()[b].origin[a];
            if (masks)
                for (int w = 0; w < g.mask_words(); ++w) masks[std::size_t(b) * g.mask_words() + w] = g.mask(b, w);
            if (classes) classes[b] = PL(p)->classes.classes[b];
        }
    });
}

int voxl_sparse_plan_arrangement(voxl_sparse_plan* p, int* perm, uint8_t* bitmask, int32_t* meta, int64_t* count) {
    return guarded([&] {
        const Arrangement& a = PL(p)->arr;
        if (perm) std::memcpy(perm, a.permutation.data(), a.permutation.size() * sizeof(int));
        if (bitmask && !a.boundary_bitmask.empty())
            std::memcpy(bitmask, a.boundary_bitmask.data(), a.boundary_bitmask.size());
        if (meta && !a.voxel_meta_index.empty())
            std::memcpy(meta, a.voxel_meta_index.data(), a.voxel_meta_index.size() * sizeof(int32_t));
        if (count) *count = a.boundary_voxel_count;
    });
}

int voxl_sparse_plan_report_json(voxl_sparse_plan* p, char* out, int64_t cap, int64_t* len) {
    return guarded([&] { put_text(PL(p)->plan.to_json(true), out, cap, len); });
}

int voxl_sparse_plan_neighbours(voxl_sparse_plan* p, int32_t* out) {
    return guarded([&] {
        const auto t = PL(p)->grid.neighbour_table();
        std::memcpy(out, t.data(), t.size() * sizeof(int32_t));
    });
}

int voxl_sparse_info(voxl_sparse* h, int64_t* na, int* nb, int64_t* nbd, int64_t* nnb) {
    return voxl_sparse_plan_info(reinterpret_cast<voxl_sparse_plan*>(&SP(h)->tables()), na, nb, nbd, nnb);
}

int voxl_sparse_blocks(voxl_sparse* h, int* origins, uint64_t* masks, uint8_t* classes) {
    return voxl_sparse_plan_blocks(reinterpret_cast<voxl_sparse_plan*>(&SP(h)->tables()), origins, masks, classes);
}

int voxl_sparse_arrangement(voxl_sparse* h, int* perm, uint8_t* bitmask, int32_t* meta, int64_t* count) {
    return voxl_sparse_plan_arrangement(reinterpret_cast<voxl_sparse_plan*>(&SP(h)->tables()), perm, bitmask, meta,
                                        count);
}

int voxl_sparse_report_json(voxl_sparse* h, char* out, int64_t cap, int64_t* len) {
    return voxl_sparse_plan_report_json(reinterpret_cast<voxl_sparse_plan*>(&SP(h)->tables()), out, cap, len);
}

int voxl_sparse_get_state(voxl_sparse* h, double* canonical) {
    return guarded([&] {
        need("voxl_sparse_get_state", h, canonical);
        SP(h)->get_state(canonical);
    });
}

int voxl_sparse_digest(voxl_sparse* h, uint64_t* out2) {
    return guarded([&] {
        need("voxl_sparse_digest", h, out2);
        unsigned long long d[2];
        SP(h)->digest(d);
        out2[0] = d[0];
        out2[1] = d[1];
    });
}

int voxl_sparse_set_state(voxl_sparse* h, const double* canonical) {
    return guarded([&] {
        need("voxl_sparse_set_state", h, canonical);
        SP(h)->set_state(canonical);
    });
}

int voxl_sparse_set_equilibrium(voxl_sparse* h, double rho, const double* u) {
    return guarded([&] {
        need("voxl_sparse_set_equilibrium", h, u);
        SP(h)->set_equilibrium(rho, u);
    });
}

int voxl_sparse_step(voxl_sparse* h, int n) {
    return guarded([&] {
        need("voxl_sparse_step", h);
        SP(h)->step(n);
    });
}

int voxl_sparse_step_identity(voxl_sparse* h, int n) {
    return guarded([&] {
        need("voxl_sparse_step_identity", h);
        require(n >= 0, "step_identity: n must be >= 0");
        SP(h)->step_identity(n);
    });
}

int voxl_sparse_timed_steps(voxl_sparse* h, int n, double* total, double* bms, double* lms) {
    return guarded([&] {
        need("voxl_sparse_timed_steps", h, total);
        *total = SP(h)->timed_steps(n, bms, lms);
    });
}

int voxl_sparse_probe(voxl_sparse* h, voxl_diag* out) {
    return guarded([&] {
        need("voxl_sparse_probe", h, out);
        const DenseDiag d = SP(h)->probe();
        out->mass = d.mass;
        out->max_speed = d.max_speed;
        out->unstable = d.unstable;
        out->bad_population = d.bad_population;
        out->bad_voxel = d.bad_voxel;
    });
}

int voxl_sparse_step_probe_n(voxl_sparse* h, int n, voxl_diag* rows, int* completed) {
    if (completed) *completed = 0;
    return guarded([&] {
        need("voxl_sparse_step_probe_n", h);
        if (n > 0) need("voxl_sparse_step_probe_n", rows);
        std::vector<DenseDiag> r(std::size_t(std::max(n, 0)));
        std::string msg;
        const int done = SP(h)->step_probe_n(n, r.data(), &msg);
        fill_rows(r.data(), done, rows);
        if (completed) *completed = done;
        if (done < n) throw InstabilityError(msg);
    });
}

int voxl_sparse_step_probe(voxl_sparse* h, voxl_diag* out) {
    return guarded([&] {
        need("voxl_sparse_step_probe", h, out);
        const DenseDiag d = SP(h)->step_probe();
        out->mass = d.mass;
        out->max_speed = d.max_speed;
        out->unstable = d.unstable;
        out->bad_population = d.bad_population;
        out->bad_voxel = d.bad_voxel;
    });
}

int voxl_dispatch_plan_json(int strategy, int64_t n_b, int64_t n_nb, int q, int bs, int s_w, int s_i, int full,
                            char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        require(strategy >= 0 && strategy <= 2, "unknown sparse strategy");
        put_text(dispatch_plan(Strategy(strategy), n_b, n_nb, q, bs, s_w, s_i, full != 0).to_json(false), out, cap,
                 len);
    });
}

int voxl_initial_state(int lattice, int scenario, int nx, int ny, int nz, uint64_t seed, double perturbation,
                       double* out) {
    return guarded([&] {
        // initial_canonical_state (solver.cpp:165-187): the same libstdc++
        // mt19937_64 / uniform_real_distribution sequence as the reference.
        require(lattice >= 0 && lattice <= 2, "unknown lattice kind");
        const LatticeTable t = make_lattice(lattice);
        auto eq = [&](double rho, const double u[3], double* f) {
            const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
            for (int i = 0; i < t.q; ++i) {
                const double eu = double(t.e[i][0]) * u[0] + double(t.e[i][1]) * u[1] + double(t.e[i][2]) * u[2];
                const double w = double(t.wnum[i]) / double(t.wden[i]);
                f[i] = w * rho * (1.0 + 3.0 * eu + 4.5 * eu * eu - 1.5 * uu);
            }
        };
        const int64_t vol = int64_t(nx) * ny * nz;
        if (scenario == VOXL_PERIODIC && perturbation > 0.0) {
            std::mt19937_64 rng(seed);
            std::uniform_real_distribution<double> unit(-1.0, 1.0);
            for (int64_t v = 0; v < vol; ++v) {
                const double rho = 1.0 + perturbation * unit(rng);
                const double a = 0.1 * perturbation * unit(rng);
                const double b = 0.1 * perturbation * unit(rng);
                const double c = t.dim == 3 ? 0.1 * perturbation * unit(rng) : 0.0;
                const double u[3] = {a, b, c};
                eq(rho, u, out + v * t.q);
            }
        } else {
            const double u0[3] = {0.0, 0.0, 0.0};
            double f[27];
            eq(1.0, u0, f);
            for (int64_t v = 0; v < vol; ++v) std::memcpy(out + v * t.q, f, sizeof(double) * t.q);
        }
    });
}

int voxl_band_level_map(int nx, int ny, int nz, int levels, int axis, int32_t* out) {
    return guarded([&] {
        // solver.cpp:319-335
        const int n[3] = {nx, ny, nz};
        for (int z = 0; z < nz; ++z)
            for (int y = 0; y < ny; ++y)
                for (int x = 0; x < nx; ++x) {
                    const int v[3] = {x, y, z};
                    const int k = v[axis];
                    int level = levels - 1;
                    for (int l = 0; l < levels - 1; ++l)
                        if (k >= (n[axis] >> (l + 1))) {
                            level = l;
                            break;
                        }
                    out[(int64_t(z) * ny + y) * nx + x] = level;
                }
    });
}

static MresConfig mres_config(const voxl_mres_desc* d) {
    require(d != nullptr, "null descriptor");
    MresConfig c;
    c.lattice = d->lattice;
    c.domain = {d->nx, d->ny, d->nz};
    c.levels = d->levels;
    c.tau = d->tau;
    c.lid_u = {d->lid_u[0], d->lid_u[1], d->lid_u[2]};
    c.fused = d->fused != 0;
    require(d->precision == VOXL_F32 || d->precision == VOXL_F64, "unknown precision");
    c.precision = Precision(d->precision);
    c.edge = d->block_edge;
    c.reference_tables = d->reference_tables != 0;
    c.allow_solid = d->solid_cells != 0;
    return c;
}

static MultiResEngine* MR(voxl_mres* h) { return reinterpret_cast<MultiResEngine*>(h); }
static MresGrid* MP(voxl_mres_plan* p) { return reinterpret_cast<MresGrid*>(p); }

int voxl_mres_create(const voxl_mres_desc* d, const int32_t* map, voxl_mres** out) {
    return guarded([&] {
        require(map && out, "voxl_mres_create: null argument");
        *out = reinterpret_cast<voxl_mres*>(new MultiResEngine(mres_config(d), map));
    });
}

int voxl_mres_destroy(voxl_mres* h) {
    return guarded([&] { delete MR(h); });
}

int voxl_mres_step(voxl_mres* h, int n) {
    return guarded([&] {
        need("voxl_mres_step", h);
        MR(h)->coarse_step(n);
    });
}

int voxl_mres_timed_steps(voxl_mres* h, int n, double* o) {
    return guarded([&] {
        need("voxl_mres_timed_steps", h, o);
        const MresTimes t = MR(h)->timed_steps(n);
        o[0] = t.total;
        o[1] = t.collide;
        o[2] = t.stream;
        o[3] = t.fused;
        o[4] = t.transition;
    });
}

int voxl_mres_state_len(voxl_mres* h, int64_t* len) {
    return guarded([&] {
        need("voxl_mres_state_len", h, len);
        *len = MR(h)->state_len();
    });
}

int voxl_mres_get_state(voxl_mres* h, double* c) {
    return guarded([&] {
        need("voxl_mres_get_state", h, c);
        MR(h)->get_state(c);
    });
}

int voxl_mres_digest(voxl_mres* h, uint64_t* out2) {
    return guarded([&] {
        need("voxl_mres_digest", h, out2);
        unsigned long long d[2];
        MR(h)->digest(d);
        out2[0] = d[0];
        out2[1] = d[1];
    });
}

int voxl_mres_set_state(voxl_mres* h, const double* c) {
    return guarded([&] {
        need("voxl_mres_set_state", h, c);
        MR(h)->set_state(c);
    });
}

int voxl_mres_set_equilibrium(voxl_mres* h, double rho, const double* u) {
    return guarded([&] {
        need("voxl_mres_set_equilibrium", h, u);
        MR(h)->set_equilibrium(rho, u);
    });
}

int voxl_mres_probe(voxl_mres* h, voxl_diag* out) {
    return guarded([&] {
        need("voxl_mres_probe", h, out);
        const DenseDiag d = MR(h)->probe();
        out->mass = d.mass;
        out->max_speed = d.max_speed;
        out->unstable = d.unstable;
        out->bad_population = d.bad_population;
        out->bad_voxel = d.bad_voxel;
    });
}

int voxl_mres_step_probe_n(voxl_mres* h, int n, voxl_diag* rows, int* completed) {
    if (completed) *completed = 0;
    return guarded([&] {
        need("voxl_mres_step_probe_n", h);
        if (n > 0) need("voxl_mres_step_probe_n", rows);
        std::vector<DenseDiag> r(std::size_t(std::max(n, 0)));
        std::string msg;
        const int done = MR(h)->step_probe_n(n, r.data(), &msg);
        fill_rows(r.data(), done, rows);
        if (completed) *completed = done;
        if (done < n) throw InstabilityError(msg);
    });
}

int voxl_mres_total_mass(voxl_mres* h, double* m) {
    return guarded([&] {
        need("voxl_mres_total_mass", h, m);
        *m = MR(h)->total_mass();
    });
}

int voxl_mres_text(voxl_mres* h, int what, char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        need("voxl_mres_text", h);
        put_text(what == 0 ? MR(h)->graph_dot() : MR(h)->grid().distribution_report(), out, cap, len);
    });
}

int voxl_mres_level_info(voxl_mres* h, int l, int64_t* na, double* tau, int64_t* uni, int64_t* jmp) {
    return guarded([&] {
        need("voxl_mres_level_info", h);
        require(l >= 0 && l < MR(h)->grid().num_levels(), "bad level");
        if (na) *na = MR(h)->grid().level(l).num_active;
        if (tau) *tau = MR(h)->grid().level(l).tau;
        const auto c = MR(h)->fusion_counts(l);
        if (uni) *uni = c[0];
        if (jmp) *jmp = c[1];
    });
}

int voxl_mres_lup_per_coarse_step(voxl_mres* h, int64_t* lup) {
    return guarded([&] {
        need("voxl_mres_lup_per_coarse_step", h, lup);
        *lup = MR(h)->grid().lup_per_coarse_step();
    });
}

int voxl_mres_plan_create(const voxl_mres_desc* d, const int32_t* map, voxl_mres_plan** out) {
    return guarded([&] {
        require(d && map && out, "voxl_mres_plan_create: null argument");
        require(d->lattice >= 0 && d->lattice <= 2, "unknown lattice kind");
        *out = reinterpret_cast<voxl_mres_plan*>(
            new MresGrid(MresGrid::build({d->nx, d->ny, d->nz}, d->levels, d->lattice, map, d->tau, true,
                                         d->solid_cells != 0)));
    });
}

int voxl_mres_plan_destroy(voxl_mres_plan* p) {
    return guarded([&] { delete MP(p); });
}

int voxl_mres_plan_level(voxl_mres_plan* p, int l, int64_t* na, double* tau, int* nb, int* ng, int* np) {
    return guarded([&] {
        require(l >= 0 && l < MP(p)->num_levels(), "bad level");
        const MresLevel& L = MP(p)->level(l);
        if (na) *na = L.num_active;
        if (tau) *tau = L.tau;
        if (nb) *nb = L.ref_blocks.num_blocks();
        if (ng) *ng = int(L.ghosts.size());
        if (np) *np = int(L.pulls.size());
    });
}

int voxl_mres_plan_ref_blocks(voxl_mres_plan* p, int l, int* origins, uint64_t* masks, uint8_t* jump) {
    return guarded([&] {
        const MresLevel& L = MP(p)->level(l);
        for (int b = 0; b < L.ref_blocks.num_blocks(); ++b) {
            if (origins)
                for (int a = 0; a < 3; ++a) origins[3 * b + a] = L.ref_blocks.blocks()[b].origin[a];
            if (masks) masks[b] = L.ref_blocks.mask(b, 0);
            if (jump) jump[b] = L.fusion_jump[b];
        }
    });
}

int voxl_mres_plan_ghosts(voxl_mres_plan* p, int l, int* out) {
    return guarded([&] {
        const auto& g = MP(p)->level(l).ghosts;
        for (std::size_t i = 0; i < g.size(); ++i)
            for (int a = 0; a < 3; ++a) {
                out[6 * i + a] = g[i].cell[a];
                out[6 * i + 3 + a] = g[i].parent[a];
            }
    });
}

int voxl_mres_plan_pulls(voxl_mres_plan* p, int l, int* out) {
    return guarded([&] {
        const auto& g = MP(p)->level(l).pulls;
        for (std::size_t i = 0; i < g.size(); ++i) {
            for (int a = 0; a < 3; ++a) {
                out[7 * i + a] = g[i].voxel[a];
                out[7 * i + 4 + a] = g[i].refined[a];
            }
            out[7 * i + 3] = g[i].direction;
        }
    });
}

int voxl_mres_plan_jump_distance(voxl_mres_plan* p, int l, int x, int y, int z, int* out) {
    return guarded([&] { *out = MP(p)->jump_distance(l, x, y, z); });
}

int voxl_mres_plan_text(voxl_mres_plan* p, int what, char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        put_text(what == 2 ? MP(p)->distribution_report() : MP(p)->graph_dot(what == 0), out, cap, len);
    });
}

int voxl_ipc_export(void* dev_ptr, char* handle64) {
    return guarded([&] {
        cudaIpcMemHandle_t hd;
        VOXL_CUDA(cudaIpcGetMemHandle(&hd, dev_ptr));
        static_assert(sizeof(hd) == 64, "IPC handle size");
        std::memcpy(handle64, &hd, 64);
    });
}

int voxl_ipc_open(const char* handle64, void** dev_ptr) {
    return guarded([&] {
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, handle64, 64);
        VOXL_CUDA(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    });
}

int voxl_ipc_close(void* dev_ptr) {
    return guarded([&] { VOXL_CUDA(cudaIpcCloseMemHandle(dev_ptr)); });
}

int voxl_enable_peer_access(int peer_device) {
    return guarded([&] {
        int cur = 0;
        VOXL_CUDA(cudaGetDevice(&cur));
        if (cur == peer_device) return;
        int can = 0;
        VOXL_CUDA(cudaDeviceCanAccessPeer(&can, cur, peer_device));
        if (!can) throw CudaError("peer access not supported between devices");
        const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
            cudaGetLastError();
            return;
        }
        VOXL_CUDA(e);
    });
}

} // extern "C"
