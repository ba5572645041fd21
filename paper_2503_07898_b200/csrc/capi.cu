// capi.cu -- the extern "C" boundary (include/voxl_b200.h).
#include "../../include/voxl_b200.h"

#include <cstring>
#include <numeric>
#include <string>

#include "common.cuh"
#include "dense.cuh"
#include "grid.hpp"
#include "lattice.cuh"

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

} // namespace

extern "C" {

const char* voxl_last_error(void) { return g_last_error.c_str(); }

int voxl_version(void) { return 1; }

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

int voxl_dense_create(const voxl_dense_desc* desc, voxl_dense** out) {
    return guarded([&] {
        require(desc && out, "voxl_dense_create: null argument");
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
        require(desc->halo_mode == 0 || desc->halo_mode == 1, "unknown halo mode");
        c.halo = HaloMode(desc->halo_mode);
        c.first_partition = desc->first_partition;
        c.local_partitions = desc->local_partitions;
        *out = new voxl_dense{new DenseEngine(c)};
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
    return guarded([&] { h->eng->set_canonical(host); });
}

int voxl_dense_set_equilibrium(voxl_dense* h, double rho, const double* u) {
    return guarded([&] { h->eng->set_equilibrium(rho, u); });
}

int voxl_dense_get_canonical(voxl_dense* h, double* host) {
    return guarded([&] { h->eng->get_canonical(host); });
}

int voxl_dense_set_planes(voxl_dense* h, const double* host, int k0, int k1) {
    return guarded([&] { h->eng->set_canonical_planes(host, k0, k1); });
}

int voxl_dense_get_planes(voxl_dense* h, double* host, int k0, int k1) {
    return guarded([&] { h->eng->get_canonical_planes(host, k0, k1); });
}

int voxl_dense_step(voxl_dense* h, int n) {
    return guarded([&] { h->eng->step(n); });
}

int voxl_dense_enqueue(voxl_dense* h, int n) {
    return guarded([&] { h->eng->enqueue_steps(n); });
}

int voxl_dense_timed_steps(voxl_dense* h, int n, double* total_ms, double* kernel_ms) {
    return guarded([&] { *total_ms = h->eng->timed_steps(n, kernel_ms); });
}

int voxl_dense_synchronize(voxl_dense* h) {
    return guarded([&] { h->eng->check_errors(); });
}

int voxl_dense_probe(voxl_dense* h, voxl_diag* out) {
    return guarded([&] {
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
        require(desc != nullptr, "null descriptor");
        require(desc->lattice >= 0 && desc->lattice <= 2, "unknown lattice kind");
        require(desc->layout >= 0 && desc->layout <= 2, "unknown layout scheme");
        const LatticeTable t = make_lattice(desc->lattice);
        const int axis = t.dim == 2 ? 1 : 2;
        const Decomposition d =
            decompose({desc->nx, desc->ny, desc->nz}, desc->partitions, axis, desc->scenario == VOXL_PERIODIC);
        std::vector<LayoutMap> maps;
        const TransferSets ts = TransferSets::for_lattice(desc->lattice, axis);
        for (int p = 0; p < desc->partitions; ++p) {
            std::array<int, 3> shape{desc->nx, desc->ny, desc->nz};
            shape[axis] = d.thickness(p);
            maps.push_back(LayoutMap::build(LayoutScheme(desc->layout), shape, t.q, axis, ts));
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
        require(p >= 0 && p < h->eng->config().partitions, "bad partition");
        put_text(h->eng->layout(p).to_json(), out, cap, len);
    });
}

int voxl_dense_steps_done(voxl_dense* h, int* steps) {
    return guarded([&] { *steps = h->eng->steps_done(); });
}

int voxl_dense_buffer(voxl_dense* h, int p, int which, void** ptr, size_t* bytes) {
    return guarded([&] {
        require(p >= 0 && p < h->eng->config().partitions, "bad partition");
        *ptr = h->eng->buffer(p, which);
        if (bytes) *bytes = h->eng->buffer_bytes(p);
    });
}

int voxl_dense_stream(voxl_dense* h, void** stream) {
    return guarded([&] { *stream = (void*)h->eng->stream(); });
}

int voxl_dense_attach_peer(voxl_dense* h, int p, void* b0, void* b1) {
    return guarded([&] { h->eng->attach_peer(p, b0, b1); });
}

int voxl_dense_raw_buffer(voxl_dense* h, int p, int w, void** ptr) {
    return guarded([&] {
        require(p >= 0 && p < h->eng->config().partitions && (w == 0 || w == 1), "bad partition/buffer");
        *ptr = h->eng->raw_buffer(p, w);
    });
}

int voxl_dense_enable_distributed(voxl_dense* h, void** flags) {
    return guarded([&] {
        h->eng->enable_distributed();
        if (flags) *flags = h->eng->flag_words();
    });
}

int voxl_dense_attach_flags(voxl_dense* h, void* upper_slot, void* lower_slot) {
    return guarded([&] {
        h->eng->attach_flags(static_cast<std::uint32_t*>(upper_slot), static_cast<std::uint32_t*>(lower_slot));
    });
}

int voxl_dense_halo_push(voxl_dense* h) {
    return guarded([&] { h->eng->halo_push(); });
}

int voxl_dense_owned_voxels(voxl_dense* h, int64_t* voxels) {
    return guarded([&] { *voxels = h->eng->owned_voxels(); });
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
