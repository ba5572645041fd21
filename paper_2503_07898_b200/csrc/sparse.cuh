// sparse.cuh -- block-sparse wind-tunnel LBM engine on B200.
//
// Drop-in for sparse::SparseLbmEngine (proj/include/voxl/sparse.hpp:175-213,
// proj/src/sparse.cpp:253-453): the same three dispatch strategies (Table 2),
// with real kernels behind them:
//   Naive        one "combined" kernel over every block; the regularized path
//                is compiled in for all voxels (3Q register footprint) and the
//                boundary velocity comes from an inline per-slot table.
//   DisagBitmask two kernels over every block, each skipping the other class
//                by the per-block bitmask; boundary velocity through the
//                indirect voxel_meta_index into a compact buffer.
//   DisagMem     boundary blocks stored first: a heavy kernel over [0, n_b)
//                and a light bounce-back + BGK kernel (2Q) over [n_b, n);
//                boundary velocity derived from geometry, zero extra storage.
// Storage is the reference's BlockField: SoA within each block,
// data[((b*Q)+c)*E^3 + local], local = (lz*E + ly)*E + lx.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "dense.cuh"
#include "sparse_grid.hpp"
#include "diag_ring.cuh"

namespace voxl_b200 {

struct SparseConfig {
    int lattice = 1;
    std::array<int, 3> domain{32, 32, 32};
    double tau = 0.7;
    std::array<double, 3> u_bc{0.04, 0.0, 0.0};
    int edge = 8;
    Strategy strategy = Strategy::DisagMem;
    Precision precision = Precision::F32;
};

class SparseEngine {
public:
    SparseEngine(const SparseConfig& cfg, const std::uint8_t* active);
    ~SparseEngine();
    SparseEngine(const SparseEngine&) = delete;
    SparseEngine& operator=(const SparseEngine&) = delete;

    const SparseConfig& config() const { return cfg_; }
    const BlockGrid& grid() const { return T_.grid; }
    const ClassifyResult& classes() const { return T_.classes; }
    const Arrangement& arrangement() const { return T_.arr; }
    const DispatchPlan& plan() const { return T_.plan; }
    SparseTables& tables() { return T_; }
    int q() const { return q_; }

    void set_equilibrium(double rho, const double u[3]);
    /// Canonical state: active voxels sorted by pack_coord (x slowest, z
    /// fastest), q populations each (sparse.cpp:416-453).
    void set_state(const double* canonical);
    void get_state(double* canonical);
    /// Device digest (digest.cuh) of the canonical state.
    void digest(unsigned long long out[2]);
    void step(int n);
    /// Identity sweeps (sparse.cpp:396-404): state unchanged, report unchanged.
    void step_identity(int n);
    /// n steps timed with CUDA events per launch: returns total ms, and the
    /// summed boundary-kernel and non-boundary-kernel ms.
    double timed_steps(int n, double* boundary_ms, double* light_ms);
    DenseDiag probe();
    DenseDiag step_probe();  // one step with probe_field fused into the step kernels
    /// n x (step + probe_field), run_sparse's per-step loop (solver.cpp:287-291),
    /// rows accumulated on the device (diag_ring.cuh), one host
    /// synchronisation per kDiagBatch steps. Returns the rows filled; on the
    /// first failing step *abort_msg = run()'s text.
    int step_probe_n(int n, DenseDiag* rows, std::string* abort_msg);
    void check_errors();

private:
    SparseConfig cfg_;
    int q_ = 19;
    SparseTables T_;
    BlockGrid& grid_ = T_.grid;
    ClassifyResult& classes_ = T_.classes;
    Arrangement& arr_ = T_.arr;
    int esize_ = 4;
    void* buf_[2] = {nullptr, nullptr};
    int cur_ = 0;
    int steps_done_ = 0;
    int sm_count_ = 0;  // the DisagMem boundary kernel runs one CTA pair per SM
    bool tma_ = false;  // one block per CTA staged by a bulk copy (E = 8, fp32; VOXL_SPARSE_TMA=1)
    std::int32_t* d_nbr_ = nullptr;
    std::uint64_t* d_masks_ = nullptr;
    std::uint8_t* d_full_ = nullptr;
    int* d_origins_ = nullptr;
    std::uint8_t* d_bitmask_ = nullptr;
    int* d_bitmask_spans_ = nullptr;  // DisagBitmask boundary sweep: bitmask_pairs_ + 1 span starts
    int bitmask_pairs_ = 0;
    std::int32_t* d_meta_index_ = nullptr;
    void* d_compact_meta_ = nullptr;
    void* d_naive_meta_ = nullptr;
    std::int64_t* d_slots_ = nullptr;
    std::unique_ptr<CanonPipe> io_;  // canonical host <-> device pipeline (canon_io.cuh)
    int* d_error_ = nullptr;
    double* d_diag_ = nullptr;
    cudaStream_t stream_ = nullptr;
    // DisagMem: the boundary (regularized) kernel runs on a high-priority side
    // stream concurrently with the light kernel (disjoint output blocks, shared
    // read-only input), so its low-occupancy tail hides under the light sweep.
    cudaStream_t side_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;

    void launch(int which, cudaEvent_t* ev_b, cudaEvent_t* ev_l, const DiagTarget* diag = nullptr);
    std::unique_ptr<DiagRing> ring_;       // step_probe_n's accumulators
    std::int32_t* d_canon_ = nullptr;      // slot -> canonical index (the fused probe's offender)
    unsigned long long last_bad_ = ~0ull;  // first-offender word of the last failing probed step
    void ensure_slots();
    void transfer(double* host, bool to_device, unsigned long long* digest);
};

} // namespace voxl_b200
