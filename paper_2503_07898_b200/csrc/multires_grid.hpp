// multires_grid.hpp -- host side of the multi-resolution path.
//
// Mirrors mres::MultiResGrid::build / classify_fusion / jump_distance /
// build_execution_graph (proj/include/voxl/multires.hpp:24-132,
// proj/src/multires.cpp:54-365). Two products:
//   * reference tables at the reference's edge-4 granularity (ghost list,
//     coalesced pulls, fusion classes, graph), bit-identical to the reference;
//   * the device layout: per level an "extended" block grid covering the
//     active cells plus the ghost ring (fine cells under an active parent) and
//     the refined ring (cells covered by the finer level that an active cell
//     pulls from). The post-collision buffer's ghost / ring slots carry the
//     exploded parent populations / coalesced child averages, so every
//     in-domain pull of the stream kernels is a plain load.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "sparse_grid.hpp"

namespace voxl_b200 {

struct MresGhost {
    std::array<int, 3> cell, parent;
};
struct MresPull {
    std::array<int, 3> voxel;
    int direction;
    std::array<int, 3> refined;
};

struct MresLevel {
    std::array<int, 3> domain{1, 1, 1};
    double tau = 0.6;
    std::vector<std::uint8_t> active;        // level cells, x fastest
    std::vector<std::uint8_t> refined;       // covered by the finer level
    std::vector<std::uint8_t> under_coarse;  // parent active at the coarser level
    std::vector<std::uint8_t> solid;         // obstacle cells (extension; level 0 only, else empty)
    std::int64_t num_active = 0;
    std::int64_t num_solid = 0;
    // reference tables (edge-4 block order)
    BlockGrid ref_blocks;                 // edge 4, active cells only
    std::vector<MresGhost> ghosts;        // multires.cpp:350-368
    std::vector<MresPull> pulls;          // multires.cpp:369-383
    std::vector<std::uint8_t> fusion_jump;  // per ref block: 1 = Jump (classify_fusion)
    std::vector<std::array<int, 3>> distance0;
};

class MresGrid {
public:
    /// level_of_cell: virtual finest domain, x fastest, values in [0, levels).
    /// reference_tables: also build the edge-4 ghost / pull / fusion tables in
    /// the reference's scan order (O(active x 26); off for large grids).
    /// allow_solid (extension beyond the reference, whose build rejects any id
    /// outside [0, levels), multires.cpp:84-85): kSolidCell marks obstacle
    /// cells. They must sit inside the finest level with a margin of
    /// kSolidMargin finest cells to every coarser cell, so no coarse cell,
    /// ghost or coalesced pull ever covers one; fluid cells pulling from a
    /// solid cell bounce back (halfway, like the domain walls).
    static constexpr int kSolidCell = -1;
    static constexpr int kSolidMargin = 3;
    static MresGrid build(std::array<int, 3> virtual_domain, int levels, int lattice, const std::int32_t* level_of_cell,
                          double tau_coarsest, bool reference_tables = true, bool allow_solid = false);
    bool has_reference_tables() const { return ref_tables_; }

    int num_levels() const { return int(levels_.size()); }
    int dim() const { return dim_; }
    int lattice() const { return lattice_; }
    std::array<int, 3> virtual_domain() const { return vdom_; }
    const MresLevel& level(int l) const { return levels_[l]; }

    bool active(int l, int x, int y, int z) const;
    bool crosses_level(int l, int x, int y, int z) const;  // multires.cpp:196-212
    int jump_distance(int l, int x, int y, int z) const;   // multires.cpp:214-223 (kNoJump = INT_MAX)
    /// build_execution_graph + to_dot; block counts from the edge-4 reference
    /// tables, or per level (uniform, jump) counts when given.
    std::string graph_dot(bool fused, const std::vector<std::array<std::int64_t, 2>>* counts = nullptr) const;
    std::string distribution_report() const;               // multires.cpp:611-622
    /// LUP per coarse step: sum_l N_l * 2^(L-1-l).
    std::int64_t lup_per_coarse_step() const;

private:
    std::array<int, 3> vdom_{1, 1, 1};
    bool ref_tables_ = true;
    int dim_ = 3;
    int lattice_ = 1;
    std::vector<MresLevel> levels_;
};

} // namespace voxl_b200
