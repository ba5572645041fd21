// sparse_grid.hpp -- host side of the block-sparse path: block cover,
// classification, arrangement and dispatch accounting.
//
// Mirrors proj/include/voxl/sparse.hpp / proj/src/sparse.cpp (build :20-59,
// classify_blocks :109-126, arrange :144-185, dispatch_plan :199-251),
// generalised from the reference's 64-bit mask (edge <= 4) to a multi-word
// mask so 8^3 blocks (512 bits) use the same code. For edge <= 4 every table
// is bit-identical to the reference's (tests/test_sparse.py).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace voxl_b200 {

enum class Strategy : int { Naive = 0, DisagBitmask = 1, DisagMem = 2 };
const char* to_string(Strategy s);

struct SparseBlock {
    std::array<int, 3> origin{0, 0, 0};
    std::int64_t offset = 0;
};

/// Block cover of an activity mask over a domain, blocks ordered by block
/// coordinate (z, y, x ascending) until permuted.
class BlockGrid {
public:
    /// `active` holds nx*ny*nz bytes, x fastest (1 = active).
    static BlockGrid build(std::array<int, 3> domain, const std::uint8_t* active, int edge);

    int edge() const { return edge_; }
    int block_volume() const { return edge_ * edge_ * edge_; }
    int mask_words() const { return words_; }
    int num_blocks() const { return int(blocks_.size()); }
    std::int64_t num_active() const { return num_active_; }
    std::array<int, 3> domain() const { return domain_; }
    const std::vector<SparseBlock>& blocks() const { return blocks_; }
    /// mask word w of block b (bit local % 64 of word local / 64; local = (lz*E+ly)*E+lx)
    std::uint64_t mask(int b, int w) const { return masks_[std::size_t(b) * words_ + w]; }
    const std::vector<std::uint64_t>& masks() const { return masks_; }
    bool bit(int b, int local) const { return (mask(b, local >> 6) >> (local & 63)) & 1u; }
    /// Index into blocks() for a block coordinate, or -1.
    int find_block(int bx, int by, int bz) const;
    void permute(const std::vector<int>& permutation);
    /// 27-neighbour block table (d = (dx+1) + 3(dy+1) + 9(dz+1)), -1 when absent.
    std::vector<std::int32_t> neighbour_table() const;

private:
    int edge_ = 4, words_ = 1;
    std::array<int, 3> domain_{1, 1, 1};
    std::array<int, 3> nblk_{1, 1, 1};
    std::int64_t num_active_ = 0;
    std::vector<SparseBlock> blocks_;
    std::vector<std::uint64_t> masks_;
    std::vector<std::int32_t> index_;  // dense block-coordinate index -> position
};

struct ClassifyResult {
    std::vector<std::uint8_t> classes;  // 1 = Boundary, 0 = NonBoundary
    std::int64_t n_boundary = 0, n_non_boundary = 0;
};

/// Boundary iff some active voxel lies on the regularized faces x == 0 or
/// x == nx-1 (wind tunnel predicate, sparse.cpp:227-238).
ClassifyResult classify_blocks(const BlockGrid& g);

struct Arrangement {
    Strategy strategy = Strategy::Naive;
    std::vector<int> permutation;
    std::vector<std::uint8_t> boundary_bitmask;
    std::vector<std::int32_t> voxel_meta_index;
    std::int64_t boundary_voxel_count = 0;
};

Arrangement arrange(Strategy s, BlockGrid& g, ClassifyResult& classes);

struct KernelPlan {
    std::string name;
    std::int64_t blocks = 0;
    std::int64_t cost = 0;
};

struct DispatchPlan {
    Strategy strategy = Strategy::Naive;
    std::vector<KernelPlan> kernels;
    std::int64_t extra_storage_bytes = 0;
    bool indirect = false;
    std::string to_json(bool with_peak) const;
};

DispatchPlan dispatch_plan(Strategy s, std::int64_t n_b, std::int64_t n_nb, int q, int block_size, int s_w, int s_i,
                           bool naive_full_domain_storage = false);

/// Everything the engine derives from (domain, mask, edge, strategy) on the
/// host: SparseLbmEngine's constructor steps (sparse.cpp:253-266).
struct SparseTables {
    BlockGrid grid;
    ClassifyResult classes;
    Arrangement arr;
    DispatchPlan plan;
    static SparseTables build(std::array<int, 3> domain, const std::uint8_t* active, int edge, Strategy s, int q);
};

/// Slot (b * block_volume + local) of every active voxel in the reference's
/// canonical order: sorted by pack_coord, i.e. x slowest, z fastest
/// (sparse.cpp:416-438).
std::vector<std::int64_t> canonical_slots(const BlockGrid& g);

} // namespace voxl_b200
