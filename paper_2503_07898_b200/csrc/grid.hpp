// grid.hpp -- host-side dense grid layer: layout maps, slab decomposition,
// voxel classification, transfer ledger and trace.
//
// B200-native mirror of the reference's classification -> mapping steps for the
// dense path (proj/include/voxl/layout.hpp, partition.hpp). The maps here are
// the addressing the CUDA kernels use verbatim (as per-group plane tables), so
// a GPU buffer is bit-for-bit the reference's PartitionedField buffer.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace voxl_b200 {

enum class LayoutScheme : int { AoS = 0, SoA = 1, DisagSoA = 2 };
enum class GroupTag : int { UpperHalo = 0, UpperShared = 1, Interior = 2, LowerShared = 3, LowerHalo = 4 };
constexpr int kGroupCount = 5;

const char* to_string(LayoutScheme s);
const char* to_string(GroupTag g);

struct Span {
    std::int64_t base = 0;
    std::int64_t len = 0;
};

/// Face-crossing component sets (layout.hpp:33-40, layout.cpp:37-49).
struct TransferSets {
    std::vector<int> up;
    std::vector<int> down;
    static TransferSets all(int cardinality);
    static TransferSets for_lattice(int lattice_kind, int axis);
};

/// Address map of one partition plus its two one-deep halo slabs
/// (layout.hpp:42-101, layout.cpp:72-201). Extents are (nx, ny, nz); `axis` is
/// the partition axis.
class LayoutMap {
public:
    static LayoutMap build(LayoutScheme scheme, std::array<int, 3> owned, int cardinality, int axis,
                           const TransferSets& transfer);

    std::int64_t address(std::array<int, 3> v, int component) const;
    GroupTag group_of(int k) const;
    std::pair<int, int> group_slab(GroupTag g) const;
    std::vector<Span> contiguous_spans(GroupTag g, const std::vector<int>& comps) const;
    std::string to_json() const;

    /// Per-(group, component) element offset such that
    ///   address(v, c) = plane_offset(g, c) + extended_linear(v) * voxel_stride()
    /// for every voxel v of group g. This is the form the kernels consume.
    std::int64_t plane_offset(int g, int c) const;
    std::int64_t voxel_stride() const { return scheme_ == LayoutScheme::AoS ? cardinality_ : 1; }
    std::int64_t extended_linear(std::array<int, 3> v) const;

    LayoutScheme scheme() const { return scheme_; }
    std::array<int, 3> shape() const { return shape_; }
    int cardinality() const { return cardinality_; }
    int axis() const { return axis_; }
    std::int64_t total_len() const { return total_len_; }
    std::int64_t cross_section() const { return cross_section_; }
    std::int64_t group_offset(GroupTag g) const { return group_offset_[int(g)]; }
    std::int64_t group_voxels(GroupTag g) const { return group_voxels_[int(g)]; }
    const std::vector<int>& component_order(GroupTag g) const { return order_[int(g)]; }
    const TransferSets& transfer() const { return transfer_; }

private:
    LayoutScheme scheme_ = LayoutScheme::DisagSoA;
    std::array<int, 3> shape_{1, 1, 1};
    int cardinality_ = 1;
    int axis_ = 2;
    TransferSets transfer_;
    std::int64_t cross_section_ = 0;
    std::int64_t extended_voxels_ = 0;
    std::int64_t total_len_ = 0;
    std::array<std::int64_t, kGroupCount> group_offset_{};
    std::array<std::int64_t, kGroupCount> group_voxels_{};
    std::array<std::vector<int>, kGroupCount> order_;
};

/// Balanced 1D slab decomposition (partition.hpp:15-32, partition.cpp:10-41).
struct Decomposition {
    std::array<int, 3> domain{1, 1, 1};
    int num_partitions = 1;
    int axis = 2;
    bool periodic = false;
    std::vector<std::pair<int, int>> slabs;
    int thickness(int p) const { return slabs[p].second - slabs[p].first; }
    int upper_neighbor(int p) const;
    int lower_neighbor(int p) const;
};

Decomposition decompose(std::array<int, 3> domain, int num_partitions, int axis, bool periodic);

/// Private (0) / Shared (1) per owned voxel, canonical local order
/// (partition.cpp:43-61).
std::vector<std::uint8_t> classify_voxels(const Decomposition& d, int p);

/// One contiguous copy (partition.hpp:35-41).
struct TransferRecord {
    int step = 0;
    int src = 0;
    int dst = 0;
    Span src_span;
    Span dst_span;
    std::int64_t elements = 0;
};

/// The halo-update records one step produces, in the reference's order:
/// partitions ascending, upper neighbour then lower (partition.cpp:163-206).
/// AoS carries every component; SoA/DisagSoA the face-crossing set.
std::vector<TransferRecord> halo_records(const Decomposition& d, const std::vector<LayoutMap>& maps,
                                         int step);

} // namespace voxl_b200
