// dense.cuh -- dense z-slab (y-slab in 2D) LBM engine on B200.
//
// Drop-in for the reference's dense path: PartitionedField + step_occ +
// GatherKernel (proj/include/voxl/partition.hpp:95-214, lbm.hpp:123-133) and the
// single-grid oracle loop reference_dense_run (proj/src/solver.cpp:189-206).
//
// One DenseEngine owns P partitions. Each partition is a pair of device buffers
// laid out EXACTLY as the reference's LayoutMap (AoS / SoA / DisagSoA) over the
// owned slab plus one-deep halos. A step is one fused pull + BGK kernel per
// partition; in zero-copy mode the shared-layer voxels also store their
// face-crossing populations straight into the neighbour partition's halo
// group of the output buffer (one contiguous 5*s span in DisagSoA), so no halo
// copy exists at all. Partitions may live on different devices (peer pointers)
// or in different processes (IPC pointers, see attach_peer()).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "grid.hpp"
#include "phase_trace.cuh"

namespace voxl_b200 {

class CanonPipe;
class DiagRing;

struct DiagTarget;
enum class Precision : int { F32 = 0, F64 = 1 };
/// ZeroCopy: the shared-layer kernel stores the crossing populations into the
/// neighbour's halo (peer memory). Copy: span copies after the shared layers
/// (halo_update's copies, device to device). Nccl: the same spans moved by
/// grouped ncclSend/ncclRecv (multi-device engines with one device per
/// partition; the measured comparison of the paper's zero-copy scheme).
enum class HaloMode : int { ZeroCopy = 0, Copy = 1, Nccl = 2 };
enum class Scenario : int { LidDrivenCavity = 0, FlowOverObstacle = 1, PeriodicBox = 2 };

/// The closed operator set behind the step_occ plugin point
/// (partition.hpp:169-174 takes any `kernel(view, v, out)`; device code needs
/// a closed set): the LBM GatherKernel (lbm.hpp:123-133), and the two generic
/// kernels the reference's partition tests drive through step_occ -- the
/// identity copy (partition_test.cpp:189-191) and the five-point Jacobi on a
/// 2-component vector field (partition_test.cpp:234-247).
enum class Operator : int { Lbm = 0, Identity = 1, Jacobi2 = 2 };

struct DenseConfig {
    int lattice = 1;  // LatticeKind
    std::array<int, 3> domain{32, 32, 32};
    double tau = 0.56;
    Scenario scenario = Scenario::LidDrivenCavity;
    std::array<double, 3> velocity{0.05, 0.0, 0.0};
    LayoutScheme layout = LayoutScheme::DisagSoA;
    int partitions = 1;
    Precision precision = Precision::F32;
    HaloMode halo = HaloMode::ZeroCopy;
    // Partitions owned by this engine: [first_partition, first_partition + local_partitions).
    // The default (-1) owns all of them (single process).
    int first_partition = 0;
    int local_partitions = -1;
    Operator op = Operator::Lbm;
    // Single-process multi-device placement: partition p lives on devices[p]
    // (the reference's in-process PartitionedField, partition.hpp:92-126, over
    // several GPUs). Empty: every partition on the current device, launched
    // back to back on one stream. Non-empty (even all equal): the two-stream
    // OCC schedule per partition with cross-device event ordering.
    std::vector<int> devices;
    // Multi-device engines: steps per captured CUDA graph (even, 0 = launch
    // every step from the host).
    int graph_steps = 8;
};

/// Field geometry an operator implies: cardinality, partition axis and the
/// face-crossing component sets. LBM / identity: the lattice's Q and
/// TransferSets::for_lattice along z (y in 2D). Jacobi2: 2 components, every
/// component crosses (TransferSets::all(2)), partitioned along y when nz == 1
/// (the reference test's decompose(domain, parts, 1)) else along z.
struct OperatorShape {
    int q = 19;
    int axis = 2;
    TransferSets transfer;
};
OperatorShape operator_shape(const DenseConfig& cfg);

struct DenseDiag {
    double mass = 0.0;
    double max_speed = 0.0;
    int unstable = 0;            // 1 if some |f| > 1e3 or non-finite
    std::int64_t bad_voxel = -1; // canonical voxel index of the first offender
    int bad_population = -1;
};

class DenseEngine {
public:
    explicit DenseEngine(const DenseConfig& cfg);
    ~DenseEngine();
    DenseEngine(const DenseEngine&) = delete;
    DenseEngine& operator=(const DenseEngine&) = delete;

    const DenseConfig& config() const { return cfg_; }
    const Decomposition& decomposition() const { return decomp_; }
    const LayoutMap& layout(int p) const { return maps_[p]; }
    int q() const { return q_; }
    std::int64_t owned_voxels() const;  // voxels of the locally owned partitions
    int steps_done() const { return steps_done_; }
    /// The executed schedule (phase_trace.cuh): record phases of the steps
    /// enqueued while enabled; json() waits for them.
    void trace_enable(bool on) { trace_.enable(on); }
    std::string trace_json() { return trace_.json(); }

    /// Canonical fp64 state (x fastest, component innermost) for the whole
    /// domain (fill_canonical / to_canonical, partition.cpp:123-161). With a
    /// partial engine only the owned slabs are read/written.
    void set_canonical(const double* host);
    /// Every voxel (halos included, both buffers) at equilibrium(rho, u):
    /// the reference's rest-state initialisation, done on the device.
    void set_equilibrium(double rho, const double u[3]);
    void get_canonical(double* host);
    /// Same, over global axis planes [k_begin, k_end) only (chunked I/O).
    void set_canonical_planes(const double* host, int k_begin, int k_end);
    void get_canonical_planes(double* host, int k_begin, int k_end);
    /// Digest (digest.cuh) of the canonical state of the owned slabs,
    /// computed on the device: full-size parity without a host copy.
    void digest(unsigned long long out[2]);

    /// Advance n steps (step_occ x n). Throws InstabilityError if the device
    /// reported a non-positive density / non-finite moment.
    void step(int n);
    /// Enqueue n steps without any host synchronisation or error check.
    void enqueue_steps(int n);
    /// n steps bracketed by CUDA events on the engine stream; returns the
    /// first-to-last event span (ms) and the summed per-step spans.
    double timed_steps(int n, double* kernel_ms);
    /// probe_field on the current state (lbm.cpp:116-138), on the device.
    DenseDiag probe();
    /// One step with the probe fused into the step kernel (run()'s per-step
    /// diagnostics row, solver.cpp:245-255) -- no extra pass over the field.
    /// A probe_field instability is returned in the row; a non-positive
    /// density throws InstabilityError.
    DenseDiag step_probe();
    /// n probed steps with one host synchronisation per kDiagBatch steps
    /// (diag_ring.cuh). Fills rows[0, r) and returns r: r == n, or r is the
    /// first failing step (relative) and *abort_msg holds run()'s text
    /// ("run aborted at step N: ...", solver.cpp:251-254).
    int step_probe_n(int n, DenseDiag* rows, std::string* abort_msg);
    /// Checks the device error flag; throws InstabilityError on a set flag.
    void check_errors();

    /// Halo refresh of the current buffers by span copies (halo_update).
    void halo_copy(int which);

    /// Records the halo exchange of steps [0, steps_done) as the reference's
    /// TransferLedger would hold them.
    std::vector<TransferRecord> ledger_records(int step) const;

    cudaStream_t stream() const { return stream_; }
    cudaStream_t shared_stream() const { return shared_stream_; }
    /// Raw device buffer of partition p (current if which == 0 else next).
    void* buffer(int p, int which) const;
    std::size_t buffer_bytes(int p) const;
    /// Multi-process: register a neighbour partition's device buffers (both
    /// parities, IPC- or peer-mapped) so the shared-layer kernel stores into it.
    void attach_peer(int p, void* buf0, void* buf1);
    /// Multi-process: allocate this rank's flag words (zeroed). flags[0] is
    /// written by the upper neighbour, flags[1] by the lower neighbour, each
    /// with the number of steps whose shared-layer stores it has completed.
    void enable_distributed();
    /// Multi-process: the neighbours' flag slots this rank signals
    /// (upper neighbour's flags[1], lower neighbour's flags[0]); null at a
    /// domain end.
    void attach_flags(std::uint32_t* upper_flag_remote, std::uint32_t* lower_flag_remote);
    std::uint32_t* flag_words() const { return flags_; }
    /// Raw buffer w (0/1, allocation order, not parity) of partition p.
    void* raw_buffer(int p, int w) const { return parts_[p].buf[w]; }
    bool distributed() const { return distributed_; }
    /// Push this engine's shared slabs into the neighbours' halos (peer
    /// copies), for a canonical state loaded in multi-process mode.
    void halo_push();
    /// PartitionedField::neighbors / set_neighbor_links (partition.hpp:110-113):
    /// (upper, lower) neighbour of partition p. Links are derived from the
    /// decomposition; the setter is the reference's fault-injection hook, and
    /// a step on asymmetric links throws "halo_update: asymmetric neighbor
    /// links" (partition.cpp:165-171).
    std::pair<int, int> neighbors(int p) const { return links_.at(std::size_t(p)); }
    void set_neighbor_links(int p, int upper, int lower);
    /// Device of partition p.
    int device_of(int p) const { return parts_.at(std::size_t(p)).device; }
    bool multi_device() const { return multi_; }

private:
    PhaseTrace trace_;
    static int cur_device() {
        int d = 0;
        VOXL_CUDA(cudaGetDevice(&d));
        return d;
    }
    DenseConfig cfg_;
    int q_ = 19;
    int axis_ = 2;
    int esize_ = 4;
    Decomposition decomp_;
    std::vector<LayoutMap> maps_;
    struct Part {
        void* buf[2] = {nullptr, nullptr};  // owned or attached
        bool owned = false;
        int device = 0;
    };
    std::vector<Part> parts_;
    int cur_ = 0;  // parity of the current buffer
    int steps_done_ = 0;
    cudaStream_t stream_ = nullptr;
    int* error_flag_ = nullptr;
    double* diag_scratch_ = nullptr;
    double* diag_row_host_ = nullptr;
    unsigned long long halo_timeout_ns_ = 120ull * 1000 * 1000 * 1000;  // zero-copy flag wait limit  // pinned: step_probe's diagnostics row
    std::unique_ptr<DiagRing> ring_;  // per-step probe rows (diag_ring.cuh)
    unsigned long long last_bad_ = ~0ull;
    std::size_t diag_scratch_len_ = 0;
    std::unique_ptr<CanonPipe> io_;  // canonical host <-> device pipeline (canon_io.cuh)
    std::uint32_t* flags_ = nullptr;
    std::uint32_t* remote_flag_up_ = nullptr;
    std::uint32_t* remote_flag_low_ = nullptr;
    bool distributed_ = false;
    // multi-process OCC schedule (launch_step_distributed)
    cudaStream_t shared_stream_ = nullptr;
    cudaEvent_t ev_shared_[2] = {nullptr, nullptr};
    cudaEvent_t ev_interior_[2] = {nullptr, nullptr};
    cudaEvent_t ev_join_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr;
    bool occ_ready_ = false;
    void join_streams();

    // single-process multi-device schedule (launch_step_multi)
    struct PartExec {
        cudaStream_t interior = nullptr;  // planes 1 .. n-2
        cudaStream_t shared = nullptr;    // planes 0, n-1 + halo transfer (high priority)
        cudaEvent_t ev_i[2] = {nullptr, nullptr};
        cudaEvent_t ev_s[2] = {nullptr, nullptr};
        cudaEvent_t ev_ready = nullptr;   // batch start (fork) on this partition's device
    };
    struct DevExec {
        int device = 0;
        cudaStream_t aux = nullptr;  // fork / join / diagnostics of this device
        cudaEvent_t ev = nullptr;
        std::unique_ptr<DiagRing> ring;
    };
    bool multi_ = false;
    std::vector<PartExec> px_;
    std::vector<DevExec> dx_;  // distinct devices, dx_[0] = the engine stream's device
    std::vector<std::pair<int, int>> links_;
    struct NcclHalo;
    std::unique_ptr<NcclHalo> nccl_;
    int* step_base_ = nullptr;  // graph replays: device-side step counter for the error flag
    cudaGraphExec_t graph_[2] = {nullptr, nullptr};  // per starting parity
    int dev_index(int device) const;
    void setup_multi();
    void check_links() const;
    std::string graph_note_;  // why graph replay was turned off, if it was
    void enqueue_multi(int n, const DiagTarget* dev_diag, bool use_graph);
    void launch_step_multi(int step_off, bool first, const DiagTarget* dev_diag, bool capturing);
    void fork_multi();
    void join_multi();
    void capture_graph(int parity);
    int step_probe_n_multi(int n, DenseDiag* rows, std::string* abort_msg);

    bool local(int p) const {
        return p >= cfg_.first_partition && p < cfg_.first_partition + cfg_.local_partitions;
    }
    void launch_step(struct DiagTarget* diag = nullptr);
    void launch_step_distributed(struct DiagTarget* diag);
    void scatter_gather(double* host, int k_begin, int k_end, bool to_device, unsigned long long* digest = nullptr);
    void check_plane_range(const char* who, int k_begin, int k_end) const;
};

} // namespace voxl_b200
