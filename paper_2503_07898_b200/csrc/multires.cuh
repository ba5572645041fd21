// multires.cuh -- multi-resolution LBM engine on B200.
//
// Drop-in for mres::MultiResLbm (proj/include/voxl/multires.hpp:138-190,
// proj/src/multires.cpp:367-598). Each level is an edge-E block-sparse grid
// (E = 8 production, 4 reference granularity) extended by its ghost ring and
// refined ring; per level three populations buffers: cur (pre-collision, the
// reference's state), nxt, and post (post-collision of jump-block / staged
// cells, exploded parent values on ghost cells, coalesced child averages on
// ring cells). One coarse step is the reference's recursive schedule
// (advance, multires.cpp:563-576) as a launch sequence:
//   collide(l) [jump blocks | all] ; explode(l) ; advance(l-1) x2 ;
//   coalesce(l) ; fused(l) [uniform blocks] ; stream(l) [jump | all]
// Fused mode: uniform blocks run ONE kernel that reads cur once, collides in
// registers and pushes the post-collision populations to their destinations
// (pulling only from jump-block sources) -- 152 B/LUP instead of the staged
// 304 B/LUP -- while jump blocks keep the staged collide -> stream pair that
// the explosion / coalescence operators need. Results are bitwise equal to
// the staged schedule (fp64) as in the reference (multires_test.cpp:381-455).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"
#include "dense.cuh"
#include "multires_grid.hpp"
#include "diag_ring.cuh"

namespace voxl_b200 {

struct MresConfig {
    int lattice = 1;
    std::array<int, 3> domain{32, 32, 32};
    int levels = 3;
    double tau = 0.56;  // coarsest level
    std::array<double, 3> lid_u{0.05, 0.0, 0.0};
    bool fused = true;
    Precision precision = Precision::F32;
    int edge = 8;
    bool reference_tables = false;
    /// Obstacle extension (not in the reference): level-map entries of
    /// MresGrid::kSolidCell are solid, bounce-back cells inside the finest level.
    bool allow_solid = false;
};

struct MresTimes {
    double total = 0, collide = 0, stream = 0, fused = 0, transition = 0;
};

class MultiResEngine {
public:
    MultiResEngine(const MresConfig& cfg, const std::int32_t* level_map);
    ~MultiResEngine();
    MultiResEngine(const MultiResEngine&) = delete;
    MultiResEngine& operator=(const MultiResEngine&) = delete;

    const MresConfig& config() const { return cfg_; }
    const MresGrid& grid() const { return grid_; }
    int q() const { return q_; }
    std::int64_t state_len() const;
    void set_equilibrium(double rho, const double u[3]);
    void set_state(const double* canonical);
    void get_state(double* canonical);
    /// Device digest (digest.cuh) of the canonical state (levels finest first).
    void digest(unsigned long long out[2]);
    void coarse_step(int n);
    MresTimes timed_steps(int n);
    DenseDiag probe();
    /// n x (coarse_step + probe_field), run_multires's per-step loop
    /// (solver.cpp:343-345), with the probe fused into each level's last
    /// sub-step kernels and the rows accumulated on the device (diag_ring.cuh):
    /// one host synchronisation per kDiagBatch steps. Returns the rows filled;
    /// on the first failing step *abort_msg = run()'s text.
    int step_probe_n(int n, DenseDiag* rows, std::string* abort_msg);
    double total_mass();
    std::string graph_dot() const;
    /// Device-grid (uniform, jump) block counts per level.
    std::array<std::int64_t, 2> fusion_counts(int l) const;
    int edge() const { return cfg_.edge; }
    void check_errors();

    struct Level;
    void read_state(double* canonical, unsigned long long* digest);
    void device_probe(double out[3], DenseDiag* d);
    void transfer(double* host, bool to_device, unsigned long long* digest);

private:
    MresConfig cfg_;
    std::unique_ptr<CanonPipe> io_;  // canonical host <-> device pipeline (canon_io.cuh)
    int q_ = 19;
    int esize_ = 4;
    MresGrid grid_;
    std::vector<Level*> lv_;
    cudaStream_t stream_ = nullptr;
    // fused mode: the jump-block stream runs on a high-priority side stream
    // concurrently with the fused uniform kernel (both read post[parity]; they
    // write disjoint buffers: nxt of jump blocks vs post[parity ^ 1]).
    cudaStream_t side_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    int* d_error_ = nullptr;
    std::unique_ptr<DiagRing> ring_;     // step_probe_n's accumulators
    const DiagTarget* diag_ = nullptr;   // the probed step's target while step_probe_n enqueues it
    double* d_diag_ = nullptr;
    double* probe_scratch_ = nullptr;  // fused-mode pull probe: per-CTA partials of the uniform blocks
    std::size_t probe_scratch_len_ = 0;
    std::size_t diag_len_ = 0;
    int steps_done_ = 0;
    // Fused mode collides ahead: the fused uniform kernel and the jump-block
    // stream compute the NEXT sub-step's collide_level of their blocks. A
    // non-positive density found there belongs to that sub-step, which is the
    // next coarse step after a level's last sub-step of this one (sub_[l]
    // counts the level's sub-steps within the coarse step).
    std::vector<int> sub_;
    int ahead_step_ = 0;
    // timing (events around each launch class) when non-null
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>>* events_ = nullptr;

    bool cur_valid_ = true;  // fused mode: uniform cells' cur reconstructed?
    bool side_transitions_ = false;  // fused mode: explode / coalesce on side_ (see advance)

    void advance(int l);
    void gather_uniform(int l);
    void sync_state();         // cur of every cell valid (fused mode gathers uniform cells)
    void load_uniform_post();  // uniform cells' post = BGK(cur) after a host-side state change
    void launch_collide(int l, bool jump_only);
    void launch_stream(int l, bool jump_only, cudaStream_t s = nullptr, const DiagTarget* diag = nullptr);
    void launch_fused(int l, const DiagTarget* diag = nullptr);
    void build_canon_maps();   // Level::canon (slot -> canonical index), for the fused probe's offender
    void launch_explode(int coarse, cudaStream_t st);
    void launch_coalesce(int coarse, cudaStream_t st);
    void mark_begin(int cls, cudaEvent_t* b, cudaStream_t s = nullptr);
    void mark_end(int cls, cudaEvent_t b, cudaStream_t s = nullptr);
};

} // namespace voxl_b200
