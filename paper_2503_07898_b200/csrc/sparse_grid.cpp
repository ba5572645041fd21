// sparse_grid.cpp -- see sparse_grid.hpp. Reference: proj/src/sparse.cpp.
#include "sparse_grid.hpp"

#include <algorithm>
#include <numeric>
#include <sstream>
#include <stdexcept>

namespace voxl_b200 {

const char* to_string(Strategy s) {
    switch (s) {
        case Strategy::Naive: return "naive";
        case Strategy::DisagBitmask: return "disag_bitmask";
        case Strategy::DisagMem: return "disag_mem";
    }
    return "?";
}

BlockGrid BlockGrid::build(std::array<int, 3> domain, const std::uint8_t* active, int edge) {
    // sparse.cpp:20-59 (edge generalised: any power-of-two edge up to 8)
    if (edge != 1 && edge != 2 && edge != 4 && edge != 8)
        throw std::invalid_argument("block sparse: edge must be 1, 2, 4 or 8");
    BlockGrid g;
    g.edge_ = edge;
    g.words_ = std::max(1, edge * edge * edge / 64);
    g.domain_ = domain;
    for (int a = 0; a < 3; ++a) g.nblk_[a] = (domain[a] + edge - 1) / edge;
    const std::int64_t nb = std::int64_t(g.nblk_[0]) * g.nblk_[1] * g.nblk_[2];
    std::vector<std::uint64_t> dense_masks(std::size_t(nb) * g.words_, 0);
    std::int64_t n_active = 0;
    for (int z = 0; z < domain[2]; ++z)
        for (int y = 0; y < domain[1]; ++y) {
            const std::uint8_t* row = active + (std::int64_t(z) * domain[1] + y) * domain[0];
            for (int x = 0; x < domain[0]; ++x) {
                if (!row[x]) continue;
                const std::int64_t bi = (std::int64_t(z / edge) * g.nblk_[1] + y / edge) * g.nblk_[0] + x / edge;
                const int local = ((z % edge) * edge + (y % edge)) * edge + (x % edge);
                dense_masks[std::size_t(bi) * g.words_ + (local >> 6)] |= std::uint64_t(1) << (local & 63);
                ++n_active;
            }
        }
    if (n_active == 0) throw std::invalid_argument("block sparse: empty active set");
    g.index_.assign(std::size_t(nb), -1);
    // block coordinates ascending in (z, y, x): the dense index order itself
    for (std::int64_t bi = 0; bi < nb; ++bi) {
        bool any = false;
        for (int w = 0; w < g.words_; ++w) any |= dense_masks[std::size_t(bi) * g.words_ + w] != 0;
        if (!any) continue;
        SparseBlock blk;
        const int bx = int(bi % g.nblk_[0]), by = int((bi / g.nblk_[0]) % g.nblk_[1]),
                  bz = int(bi / (std::int64_t(g.nblk_[0]) * g.nblk_[1]));
        blk.origin = {bx * edge, by * edge, bz * edge};
        blk.offset = std::int64_t(g.blocks_.size());
        g.index_[std::size_t(bi)] = int(g.blocks_.size());
        g.blocks_.push_back(blk);
        for (int w = 0; w < g.words_; ++w) g.masks_.push_back(dense_masks[std::size_t(bi) * g.words_ + w]);
    }
    g.num_active_ = n_active;
    return g;
}

int BlockGrid::find_block(int bx, int by, int bz) const {
    if (bx < 0 || by < 0 || bz < 0 || bx >= nblk_[0] || by >= nblk_[1] || bz >= nblk_[2]) return -1;
    return index_[std::size_t((std::int64_t(bz) * nblk_[1] + by) * nblk_[0] + bx)];
}

void BlockGrid::permute(const std::vector<int>& perm) {
    // permute_blocks (sparse.cpp:74-86)
    if (perm.size() != blocks_.size()) throw std::invalid_argument("permute_blocks: size mismatch");
    std::vector<SparseBlock> nb;
    std::vector<std::uint64_t> nm;
    nb.reserve(blocks_.size());
    nm.reserve(masks_.size());
    for (int old : perm) {
        nb.push_back(blocks_[old]);
        for (int w = 0; w < words_; ++w) nm.push_back(masks_[std::size_t(old) * words_ + w]);
    }
    blocks_ = std::move(nb);
    masks_ = std::move(nm);
    for (int i = 0; i < int(blocks_.size()); ++i) {
        blocks_[i].offset = i;
        const auto& o = blocks_[i].origin;
        index_[std::size_t((std::int64_t(o[2] / edge_) * nblk_[1] + o[1] / edge_) * nblk_[0] + o[0] / edge_)] = i;
    }
}

std::vector<std::int32_t> BlockGrid::neighbour_table() const {
    std::vector<std::int32_t> t(blocks_.size() * 27, -1);
    for (std::size_t b = 0; b < blocks_.size(); ++b) {
        const auto& o = blocks_[b].origin;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx)
                    t[b * 27 + (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)] =
                        find_block(o[0] / edge_ + dx, o[1] / edge_ + dy, o[2] / edge_ + dz);
    }
    return t;
}

ClassifyResult classify_blocks(const BlockGrid& g) {
    // sparse.cpp:109-126 with the wind-tunnel predicate x == 0 || x == nx - 1
    ClassifyResult r;
    const int e = g.edge(), nx = g.domain()[0];
    for (int b = 0; b < g.num_blocks(); ++b) {
        bool boundary = false;
        const int ox = g.blocks()[b].origin[0];
        for (int local = 0; local < g.block_volume() && !boundary; ++local) {
            if (!g.bit(b, local)) continue;
            const int x = ox + local % e;
            boundary = x == 0 || x == nx - 1;
        }
        r.classes.push_back(boundary ? 1 : 0);
        (boundary ? r.n_boundary : r.n_non_boundary) += 1;
    }
    return r;
}

Arrangement arrange(Strategy s, BlockGrid& g, ClassifyResult& classes) {
    // sparse.cpp:144-185
    Arrangement a;
    a.strategy = s;
    a.permutation.resize(g.num_blocks());
    std::iota(a.permutation.begin(), a.permutation.end(), 0);
    if (s == Strategy::DisagMem) {
        std::stable_sort(a.permutation.begin(), a.permutation.end(),
                         [&](int x, int y) { return int(classes.classes[x]) > int(classes.classes[y]); });
        g.permute(a.permutation);
        std::vector<std::uint8_t> cls;
        for (int old : a.permutation) cls.push_back(classes.classes[old]);
        classes.classes = std::move(cls);
    } else if (s == Strategy::DisagBitmask) {
        a.boundary_bitmask = classes.classes;
        a.voxel_meta_index.assign(std::size_t(g.num_blocks()) * g.block_volume(), -1);
        const int e = g.edge(), nx = g.domain()[0];
        std::int32_t next = 0;
        for (int b = 0; b < g.num_blocks(); ++b)
            for (int local = 0; local < g.block_volume(); ++local) {
                if (!g.bit(b, local)) continue;
                const int x = g.blocks()[b].origin[0] + local % e;
                if (x == 0 || x == nx - 1) a.voxel_meta_index[std::size_t(b) * g.block_volume() + local] = next++;
            }
        a.boundary_voxel_count = next;
    }
    return a;
}

std::string DispatchPlan::to_json(bool with_peak) const {
    // DispatchPlan / ExecutionReport::to_json (sparse.cpp:187-197, :240-251)
    std::ostringstream os;
    os << "{\"strategy\": \"" << to_string(strategy) << "\", \"kernels\": [";
    std::int64_t peak = 0;
    for (std::size_t i = 0; i < kernels.size(); ++i) {
        os << (i ? ", " : "") << "{\"name\": \"" << kernels[i].name << "\", \"blocks\": " << kernels[i].blocks
           << ", \"cost\": " << kernels[i].cost << "}";
        peak = std::max(peak, kernels[i].cost);
    }
    os << "], \"extra_storage_bytes\": " << extra_storage_bytes << ", \"indexing\": \""
       << (indirect ? "indirect" : "direct") << "\"";
    if (with_peak) os << ", \"peak_cost\": " << peak;
    os << "}";
    return os.str();
}

DispatchPlan dispatch_plan(Strategy s, std::int64_t n_b, std::int64_t n_nb, int q, int bs, int s_w, int s_i,
                           bool full) {
    // sparse.cpp:199-225 (Table 2)
    if (n_b < 0 || n_nb < 0) throw std::invalid_argument("dispatch_plan: negative block counts");
    const std::int64_t rb = 3 * std::int64_t(q), rnb = 2 * std::int64_t(q);
    DispatchPlan p;
    p.strategy = s;
    switch (s) {
        case Strategy::Naive:
            p.kernels = {{"combined", n_b + n_nb, rb}};
            p.extra_storage_bytes = std::int64_t(s_w) * (full ? n_b + n_nb : n_nb) * bs;
            break;
        case Strategy::DisagBitmask:
            p.kernels = {{"boundary", n_b + n_nb, rb}, {"non_boundary", n_b + n_nb, rnb}};
            p.extra_storage_bytes = std::int64_t(s_i) * (n_b + n_nb) * bs;
            p.indirect = true;
            break;
        case Strategy::DisagMem:
            p.kernels = {{"boundary", n_b, rb}, {"non_boundary", n_nb, rnb}};
            break;
    }
    return p;
}

SparseTables SparseTables::build(std::array<int, 3> domain, const std::uint8_t* active, int edge, Strategy s,
                                 int q) {
    SparseTables t;
    t.grid = BlockGrid::build(domain, active, edge);
    t.classes = classify_blocks(t.grid);
    t.arr = arrange(s, t.grid, t.classes);
    // s_w = sizeof(double) * dim, s_i = sizeof(int32) (sparse.cpp:263-266)
    t.plan = dispatch_plan(s, t.classes.n_boundary, t.classes.n_non_boundary, q, t.grid.block_volume(), 8 * 3, 4);
    return t;
}

std::vector<std::int64_t> canonical_slots(const BlockGrid& g) {
    const auto d = g.domain();
    const int e = g.edge();
    std::vector<std::int64_t> out;
    out.reserve(std::size_t(g.num_active()));
    for (int x = 0; x < d[0]; ++x)
        for (int y = 0; y < d[1]; ++y)
            for (int z = 0; z < d[2]; ++z) {
                const int b = g.find_block(x / e, y / e, z / e);
                if (b < 0) continue;
                const int local = ((z % e) * e + (y % e)) * e + (x % e);
                if (g.bit(b, local)) out.push_back(std::int64_t(b) * g.block_volume() + local);
            }
    return out;
}

} // namespace voxl_b200
