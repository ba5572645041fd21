// multires_grid.cpp -- see multires_grid.hpp. Reference: proj/src/multires.cpp.
#include "multires_grid.hpp"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <stdexcept>

#include "lattice.cuh"

namespace voxl_b200 {

namespace {

inline std::int64_t lin3(const std::array<int, 3>& d, int x, int y, int z) {
    return (std::int64_t(z) * d[1] + y) * d[0] + x;
}

inline bool inside(const std::array<int, 3>& d, int x, int y, int z) {
    return x >= 0 && y >= 0 && z >= 0 && x < d[0] && y < d[1] && z < d[2];
}

// Box neighbourhood offsets in the reference's scan order (dz, dy, dx),
// multires.cpp:14-22; 2D keeps dz = 0.
std::vector<std::array<int, 3>> box_offsets(int dim) {
    std::vector<std::array<int, 3>> out;
    const int zlo = dim == 3 ? -1 : 0, zhi = dim == 3 ? 1 : 0;
    for (int dz = zlo; dz <= zhi; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx)
                if (dx || dy || dz) out.push_back({dx, dy, dz});
    return out;
}

} // namespace

bool MresGrid::active(int l, int x, int y, int z) const {
    const auto& L = levels_[l];
    return inside(L.domain, x, y, z) && L.active[std::size_t(lin3(L.domain, x, y, z))];
}

bool MresGrid::crosses_level(int l, int x, int y, int z) const {
    const auto& L = levels_[l];
    for (const auto& d : box_offsets(dim_)) {
        const int a = x + d[0], b = y + d[1], c = z + d[2];
        if (!inside(L.domain, a, b, c)) continue;
        const std::size_t i = std::size_t(lin3(L.domain, a, b, c));
        if (L.active[i]) continue;
        if (L.refined[i] || L.under_coarse[i]) return true;
    }
    return false;
}

int MresGrid::jump_distance(int l, int x, int y, int z) const {
    if (!active(l, x, y, z)) throw std::invalid_argument("jump_distance: inactive voxel");
    const auto& L = levels_[l];
    int best = INT_MAX;
    for (int c = 0; c < L.domain[2]; ++c)
        for (int b = 0; b < L.domain[1]; ++b)
            for (int a = 0; a < L.domain[0]; ++a) {
                if (!L.active[std::size_t(lin3(L.domain, a, b, c))] || !crosses_level(l, a, b, c)) continue;
                best = std::min(best, std::max({std::abs(a - x), std::abs(b - y), std::abs(c - z)}));
            }
    return best;
}

MresGrid MresGrid::build(std::array<int, 3> vdom, int levels, int lattice, const std::int32_t* map, double tau,
                         bool reference_tables, bool allow_solid) {
    // multires.cpp:54-192
    const LatticeTable lat = make_lattice(lattice);
    const int dim = lat.dim;
    if (levels < 1 || levels > 4) throw std::invalid_argument("multires: 1 to 4 levels supported");
    if (dim == 2 && vdom[2] != 1) throw std::invalid_argument("multires: 2D grids must have nz == 1");
    if (std::int64_t(map ? 1 : 0) == 0) throw std::invalid_argument("multires: level map size mismatch");
    const int top = 1 << (levels - 1);
    if (vdom[0] % top || vdom[1] % top || (dim == 3 && vdom[2] % top))
        throw std::invalid_argument("multires: domain extents must divide the coarsest cell size");
    MresGrid g;
    g.ref_tables_ = reference_tables;
    g.vdom_ = vdom;
    g.dim_ = dim;
    g.lattice_ = lattice;
    g.levels_.resize(levels);
    const auto offsets = box_offsets(dim);
    std::int64_t n_solid = 0;
    for (int z = 0; z < vdom[2]; ++z)
        for (int y = 0; y < vdom[1]; ++y)
            for (int x = 0; x < vdom[0]; ++x) {
                const int l = map[lin3(vdom, x, y, z)];
                if (allow_solid && l == kSolidCell) {
                    ++n_solid;
                    continue;
                }
                if (l < 0 || l >= levels) throw std::invalid_argument("multires: level id out of range");
                for (const auto& d : offsets) {
                    const int a = x + d[0], b = y + d[1], c = z + d[2];
                    if (!inside(vdom, a, b, c)) continue;
                    const int ln = map[lin3(vdom, a, b, c)];
                    if (allow_solid && ln == kSolidCell) continue;
                    if (std::abs(ln - l) > 1) throw std::invalid_argument("multires: resolution jump skips a level");
                }
            }
    if (n_solid) {
        // every cell within kSolidMargin of a solid cell is finest-level or solid
        const int m = kSolidMargin, mz = dim == 3 ? m : 0;
        for (int z = 0; z < vdom[2]; ++z)
            for (int y = 0; y < vdom[1]; ++y)
                for (int x = 0; x < vdom[0]; ++x) {
                    if (map[lin3(vdom, x, y, z)] != kSolidCell) continue;
                    for (int c = std::max(0, z - mz); c <= std::min(vdom[2] - 1, z + mz); ++c)
                        for (int b = std::max(0, y - m); b <= std::min(vdom[1] - 1, y + m); ++b)
                            for (int a = std::max(0, x - m); a <= std::min(vdom[0] - 1, x + m); ++a) {
                                const int ln = map[lin3(vdom, a, b, c)];
                                if (ln != 0 && ln != kSolidCell)
                                    throw std::invalid_argument(
                                        "multires: solid cells must lie inside the finest level, 3 cells from any "
                                        "coarser cell");
                            }
                }
    }
    for (int l = 0; l < levels; ++l) {
        MresLevel& L = g.levels_[l];
        const int s = 1 << l;
        L.domain = {vdom[0] / s, vdom[1] / s, dim == 3 ? vdom[2] / s : vdom[2]};
        const std::size_t vol = std::size_t(L.domain[0]) * L.domain[1] * L.domain[2];
        L.active.assign(vol, 0);
        const int zs = dim == 3 ? s : 1;
        for (int z = 0; z < L.domain[2]; ++z)
            for (int y = 0; y < L.domain[1]; ++y)
                for (int x = 0; x < L.domain[0]; ++x) {
                    int cnt = 0, tot = 0;
                    for (int dz = 0; dz < zs; ++dz)
                        for (int dy = 0; dy < s; ++dy)
                            for (int dx = 0; dx < s; ++dx) {
                                ++tot;
                                const int fz = dim == 3 ? z * s + dz : z;
                                if (map[lin3(vdom, x * s + dx, y * s + dy, fz)] == l) ++cnt;
                            }
                    if (cnt == tot) {
                        L.active[std::size_t(lin3(L.domain, x, y, z))] = 1;
                        ++L.num_active;
                    } else if (cnt != 0) {
                        throw std::invalid_argument("multires: level region not aligned to its cell size");
                    }
                }
        if (L.num_active == 0) throw std::invalid_argument("multires: every level must have active cells");
        L.ref_blocks = BlockGrid::build(L.domain, L.active.data(), 4);
        if (l == 0 && n_solid) {
            L.solid.assign(vol, 0);
            for (std::size_t i = 0; i < vol; ++i) L.solid[i] = map[i] == kSolidCell;
            L.num_solid = n_solid;
        }
    }
    g.levels_[levels - 1].tau = tau;
    for (int l = levels - 2; l >= 0; --l) g.levels_[l].tau = 2.0 * g.levels_[l + 1].tau - 0.5;
    for (int l = 0; l < levels; ++l) {
        MresLevel& L = g.levels_[l];
        const std::size_t vol = L.active.size();
        L.refined.assign(vol, 0);
        L.under_coarse.assign(vol, 0);
        for (int z = 0; z < L.domain[2]; ++z)
            for (int y = 0; y < L.domain[1]; ++y)
                for (int x = 0; x < L.domain[0]; ++x) {
                    const std::size_t i = std::size_t(lin3(L.domain, x, y, z));
                    const int pz = dim == 3 ? z >> 1 : z;
                    if (l + 1 < levels && g.levels_[l + 1].active[std::size_t(lin3(g.levels_[l + 1].domain, x >> 1, y >> 1, pz))])
                        L.under_coarse[i] = 1;
                    if (l > 0) {
                        const MresLevel& F = g.levels_[l - 1];
                        const int zhi = dim == 3 ? 1 : 0;
                        for (int dz = 0; dz <= zhi; ++dz)
                            for (int dy = 0; dy <= 1; ++dy)
                                for (int dx = 0; dx <= 1; ++dx) {
                                    const int cz = dim == 3 ? 2 * z + dz : z;
                                    if (F.active[std::size_t(lin3(F.domain, 2 * x + dx, 2 * y + dy, cz))]) L.refined[i] = 1;
                                }
                    }
                    if (L.active[i] && L.under_coarse[i]) throw std::invalid_argument("multires: levels overlap in space");
                }
    }
    // Ghost ring and coalesced pulls in the reference's deterministic scan
    // order: active voxels in edge-4 block-list order, then local order.
    for (int l = 0; l < levels && reference_tables; ++l) {
        MresLevel& L = g.levels_[l];
        const BlockGrid& bg = L.ref_blocks;
        std::vector<std::uint8_t> seen(l + 1 < levels ? L.active.size() : 0, 0);
        for (int b = 0; b < bg.num_blocks(); ++b)
            for (int local = 0; local < bg.block_volume(); ++local) {
                if (!bg.bit(b, local)) continue;
                const auto& o = bg.blocks()[b].origin;
                const int x = o[0] + local % 4, y = o[1] + (local / 4) % 4, z = o[2] + local / 16;
                if (l + 1 < levels)
                    for (const auto& d : offsets) {
                        const int a = x + d[0], bb = y + d[1], c = z + d[2];
                        if (!inside(L.domain, a, bb, c)) continue;
                        const std::size_t i = std::size_t(lin3(L.domain, a, bb, c));
                        if (L.active[i] || (!L.solid.empty() && L.solid[i])) continue;
                        if (L.under_coarse[i]) {
                            if (seen[i]) continue;
                            seen[i] = 1;
                            const int pz = dim == 3 ? c >> 1 : c;
                            L.ghosts.push_back({{a, bb, c}, {a >> 1, bb >> 1, pz}});
                        } else if (!L.refined[i]) {
                            throw std::invalid_argument("multires: active region has an uncovered neighbor");
                        }
                    }
                if (l > 0)
                    for (int q = 0; q < lat.q; ++q) {
                        const int a = x - lat.e[q][0], bb = y - lat.e[q][1], c = z - lat.e[q][2];
                        if (!inside(L.domain, a, bb, c)) continue;
                        const std::size_t i = std::size_t(lin3(L.domain, a, bb, c));
                        if (L.active[i] || !L.refined[i]) continue;
                        const MresLevel& F = g.levels_[l - 1];
                        const int zhi = dim == 3 ? 1 : 0;
                        for (int dz = 0; dz <= zhi; ++dz)
                            for (int dy = 0; dy <= 1; ++dy)
                                for (int dx = 0; dx <= 1; ++dx) {
                                    const int cz = dim == 3 ? 2 * c + dz : c;
                                    if (!F.active[std::size_t(lin3(F.domain, 2 * a + dx, 2 * bb + dy, cz))])
                                        throw std::invalid_argument("multires: refined cell with inactive children");
                                }
                        L.pulls.push_back({{x, y, z}, q, {a, bb, c}});
                    }
            }
        // classify_fusion (multires.cpp:225-247) at edge-4 granularity
        L.fusion_jump.assign(bg.num_blocks(), 0);
        for (int b = 0; b < bg.num_blocks(); ++b)
            for (int local = 0; local < bg.block_volume(); ++local) {
                if (!bg.bit(b, local)) continue;
                const auto& o = bg.blocks()[b].origin;
                const int x = o[0] + local % 4, y = o[1] + (local / 4) % 4, z = o[2] + local / 16;
                if (g.crosses_level(l, x, y, z)) {
                    L.fusion_jump[b] = 1;
                    L.distance0.push_back({x, y, z});
                }
            }
    }
    return g;
}

std::string MresGrid::graph_dot(bool fused, const std::vector<std::array<std::int64_t, 2>>* counts) const {
    // build_execution_graph + ExecutionGraph::to_dot (multires.cpp:287-365)
    struct Node {
        int level;
        const char* group;
        const char* op;
        std::int64_t blocks;
    };
    std::vector<Node> nodes;
    std::vector<std::pair<int, int>> edges;
    const int L = num_levels();
    std::vector<int> collide(L, -1), stream(L, -1);
    for (int l = 0; l < L; ++l) {
        std::int64_t total = levels_[l].ref_blocks.num_blocks();
        std::int64_t jump = 0;
        for (auto c : levels_[l].fusion_jump) jump += c;
        if (counts) {  // (uniform, jump) block counts of another block granularity
            jump = (*counts)[l][1];
            total = (*counts)[l][0] + jump;
        }
        const std::int64_t uniform = total - jump;
        if (!fused) {
            collide[l] = int(nodes.size());
            nodes.push_back({l, "all", "Collide", total});
            stream[l] = int(nodes.size());
            nodes.push_back({l, "all", "Stream", total});
            edges.emplace_back(collide[l], stream[l]);
        } else {
            if (uniform > 0) nodes.push_back({l, "uniform", "FusedCollideStream", uniform});
            if (jump > 0) {
                collide[l] = int(nodes.size());
                nodes.push_back({l, "jump", "Collide", jump});
                stream[l] = int(nodes.size());
                nodes.push_back({l, "jump", "Stream", jump});
                edges.emplace_back(collide[l], stream[l]);
            }
        }
    }
    for (int l = 1; l < L; ++l) {
        const int ex = int(nodes.size());
        nodes.push_back({l - 1, "transition", "Explosion", 0});
        const int co = int(nodes.size());
        nodes.push_back({l, "transition", "Coalescence", 0});
        if (collide[l] >= 0) edges.emplace_back(collide[l], ex);
        if (stream[l - 1] >= 0) {
            edges.emplace_back(ex, stream[l - 1]);
            edges.emplace_back(stream[l - 1], co);
        }
        if (stream[l] >= 0) edges.emplace_back(co, stream[l]);
    }
    std::ostringstream os;
    os << "digraph execution {\n";
    for (std::size_t i = 0; i < nodes.size(); ++i) {
        os << "  n" << i << " [label=\"L" << nodes[i].level << " " << nodes[i].op << " (" << nodes[i].group << ")";
        if (nodes[i].blocks > 0) os << " x" << nodes[i].blocks;
        os << "\"];\n";
    }
    for (const auto& e : edges) os << "  n" << e.first << " -> n" << e.second << ";\n";
    os << "}\n";
    return os.str();
}

std::string MresGrid::distribution_report() const {
    // multires.cpp:611-622
    std::ostringstream os;
    const double total = double(vdom_[0]) * vdom_[1] * vdom_[2];
    for (int l = 0; l < num_levels(); ++l) {
        if (l) os << ", ";
        char buf[32];
        std::snprintf(buf, sizeof buf, "%.3g", 100.0 * double(levels_[l].num_active) / total);
        os << buf;
    }
    return os.str();
}

std::int64_t MresGrid::lup_per_coarse_step() const {
    std::int64_t lup = 0;
    const int L = num_levels();
    for (int l = 0; l < L; ++l) lup += levels_[l].num_active << (L - 1 - l);
    return lup;
}

} // namespace voxl_b200
