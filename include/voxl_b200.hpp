// voxl_b200.hpp -- header-only C++ binding of the C-ABI (voxl_b200.h) that
// keeps the reference's names, value semantics and exception types, so a
// reference driver (proj/src/solver.cpp run_dense / run_sparse / run_multires)
// can switch engines by changing a type:
//
//   voxl::PartitionedField + step_occ + lbm::GatherKernel  -> voxl::b200::DenseEngine
//   voxl::sparse::SparseLbmEngine                          -> voxl::b200::SparseLbmEngine
//   voxl::mres::MultiResLbm                                -> voxl::b200::MultiResLbm
//
// Status codes map back to the reference's exceptions (solver.hpp, lbm.cpp,
// layout.cpp): VOXL_INVALID_ARGUMENT -> std::invalid_argument, VOXL_OUT_OF_RANGE
// -> std::out_of_range, VOXL_DOMAIN -> std::domain_error, VOXL_INSTABILITY and
// VOXL_RUNTIME -> std::runtime_error (message text preserved, e.g. "run
// aborted at step N: ..."), VOXL_CUDA_ERROR -> voxl::b200::cuda_error.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxl_b200.h"

namespace voxl {
namespace b200 {

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int status) {
    if (status == VOXL_OK) return;
    const std::string msg = voxl_last_error();
    switch (status) {
        case VOXL_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case VOXL_OUT_OF_RANGE: throw std::out_of_range(msg);
        case VOXL_DOMAIN: throw std::domain_error(msg);
        case VOXL_CUDA_ERROR: throw cuda_error(msg);
        default: throw std::runtime_error(msg);
    }
}

struct Diagnostics {  // lbm::Diagnostics (lbm.hpp:137-141)
    double mass = 0.0;
    double max_speed = 0.0;
};

/// Dense partitioned engine: PartitionedField a/b + step_occ<GatherKernel>.
class DenseEngine {
public:
    explicit DenseEngine(const voxl_dense_desc& d) { check(voxl_dense_create(&d, &h_)); }
    ~DenseEngine() { voxl_dense_destroy(h_); }
    DenseEngine(const DenseEngine&) = delete;
    DenseEngine& operator=(const DenseEngine&) = delete;

    /// PartitionedField::fill_canonical (partition.cpp:143)
    void fill_canonical(const std::vector<double>& values) { check(voxl_dense_set_canonical(h_, values.data())); }
    /// PartitionedField::to_canonical (partition.cpp:123); `volume_q` = voxels * q
    std::vector<double> to_canonical(std::size_t volume_q) const {
        std::vector<double> out(volume_q);
        check(voxl_dense_get_canonical(h_, out.data()));
        return out;
    }
    /// step_occ x n (partition.hpp:173)
    void step(int n = 1) { check(voxl_dense_step(h_, n)); }
    /// lbm::probe_field on the current state; throws like the reference.
    Diagnostics probe(int step_index) const {
        voxl_diag d{};
        check(voxl_dense_probe(h_, &d));
        if (d.unstable)
            throw std::runtime_error("instability at step " + std::to_string(step_index) + ", voxel " +
                                     std::to_string(d.bad_voxel) + ", population " + std::to_string(d.bad_population));
        return {d.mass, d.max_speed};
    }
    /// The step's TransferLedger records (partition.cpp:163-206).
    std::vector<voxl_transfer_record> ledger(int step) const {
        int n = 0;
        check(voxl_dense_ledger(h_, step, nullptr, 0, &n));
        std::vector<voxl_transfer_record> r(std::size_t(n > 0 ? n : 1));
        check(voxl_dense_ledger(h_, step, r.data(), n, &n));
        r.resize(std::size_t(n));
        return r;
    }
    voxl_dense* handle() const { return h_; }

private:
    voxl_dense* h_ = nullptr;
};

/// sparse::SparseLbmEngine (sparse.hpp:175-213).
class SparseLbmEngine {
public:
    SparseLbmEngine(const voxl_sparse_desc& d, const std::vector<std::uint8_t>& active_mask) {
        check(voxl_sparse_create(&d, active_mask.data(), &h_));
    }
    ~SparseLbmEngine() { voxl_sparse_destroy(h_); }
    SparseLbmEngine(const SparseLbmEngine&) = delete;
    SparseLbmEngine& operator=(const SparseLbmEngine&) = delete;

    void step() { check(voxl_sparse_step(h_, 1)); }
    /// step_identity (sparse.cpp:396-404)
    void step_identity() { check(voxl_sparse_step_identity(h_, 1)); }
    std::int64_t num_active() const {
        std::int64_t n = 0;
        check(voxl_sparse_info(h_, &n, nullptr, nullptr, nullptr));
        return n;
    }
    /// canonical_state (sparse.cpp:416-438)
    std::vector<double> canonical_state(int q) const {
        std::vector<double> out(std::size_t(num_active()) * q);
        check(voxl_sparse_get_state(h_, out.data()));
        return out;
    }
    /// ExecutionReport::to_json (sparse.cpp:240-251)
    std::string report_json() const {
        std::int64_t n = 0;
        check(voxl_sparse_report_json(h_, nullptr, 0, &n));
        std::string s(std::size_t(n) + 1, '\0');
        check(voxl_sparse_report_json(h_, &s[0], n + 1, &n));
        s.resize(std::size_t(n));
        return s;
    }

private:
    voxl_sparse* h_ = nullptr;
};

/// mres::MultiResLbm (multires.hpp:138-190).
class MultiResLbm {
public:
    MultiResLbm(const voxl_mres_desc& d, const std::vector<std::int32_t>& level_of_cell) {
        check(voxl_mres_create(&d, level_of_cell.data(), &h_));
    }
    ~MultiResLbm() { voxl_mres_destroy(h_); }
    MultiResLbm(const MultiResLbm&) = delete;
    MultiResLbm& operator=(const MultiResLbm&) = delete;

    void coarse_step() { check(voxl_mres_step(h_, 1)); }
    std::vector<double> canonical_state() const {
        std::int64_t n = 0;
        check(voxl_mres_state_len(h_, &n));
        std::vector<double> out(static_cast<std::size_t>(n));
        check(voxl_mres_get_state(h_, out.data()));
        return out;
    }
    double total_mass() const {
        double m = 0;
        check(voxl_mres_total_mass(h_, &m));
        return m;
    }
    std::string distribution_report() const { return text(1); }
    std::string graph_dot() const { return text(0); }

private:
    std::string text(int what) const {
        std::int64_t n = 0;
        check(voxl_mres_text(h_, what, nullptr, 0, &n));
        std::string s(std::size_t(n) + 1, '\0');
        check(voxl_mres_text(h_, what, &s[0], n + 1, &n));
        s.resize(std::size_t(n));
        return s;
    }
    voxl_mres* h_ = nullptr;
};

}  // namespace b200
}  // namespace voxl
