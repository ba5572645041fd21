/* voxl_b200.h -- C-ABI of the B200-native disaggregated LBM engines.
 *
 * Plain C: opaque handles, plain pointers and sizes, int status codes. No torch
 * or CUDA types cross this boundary (a stream is exposed as void*).
 *
 * Each entry point names the reference interface it replaces (paths relative to
 * /root/reference/proj). The reference is a C++20 library with no FFI of its
 * own; these are the symbols a maintainer binds from the reference-side
 * drivers (see INTEGRATION.md for the C++ binding that keeps the reference's
 * class names and exceptions).
 *
 * Errors: every call returns VOXL_OK (0) or a status; voxl_last_error() gives
 * the message of the calling thread's last failure, with the reference's
 * message text (e.g. "run aborted at step N: ..."). A null handle or a null
 * state / output buffer is VOXL_INVALID_ARGUMENT ("<entry point>: null argument").
 * Canonical buffers are sized by the engine (voxels * q, state_len); the
 * caller owns them and the callee copies (no pointer is retained).
 */
#ifndef VOXL_B200_H
#define VOXL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror the reference's exception types) ------------------- */
#define VOXL_OK 0
#define VOXL_INVALID_ARGUMENT 1 /* std::invalid_argument / ConfigError        */
#define VOXL_OUT_OF_RANGE 2     /* std::out_of_range (layout.cpp:156)          */
#define VOXL_RUNTIME 3          /* std::runtime_error (structure / links)      */
#define VOXL_INSTABILITY 4      /* instability / run aborted at step N         */
#define VOXL_CUDA_ERROR 5       /* CUDA runtime failure                        */
#define VOXL_DOMAIN 6           /* std::domain_error (lattice.cpp:106)         */

/* ---- enums (values equal the reference's enum order) ------------------------- */
#define VOXL_D2Q9 0  /* LatticeKind (lattice.hpp:10) */
#define VOXL_D3Q19 1
#define VOXL_D3Q27 2
#define VOXL_AOS 0   /* LayoutScheme (layout.hpp:14) */
#define VOXL_SOA 1
#define VOXL_DISAG_SOA 2
#define VOXL_CAVITY 0   /* Scenario (solver.hpp:16) */
#define VOXL_OBSTACLE 1
#define VOXL_PERIODIC 2
#define VOXL_F32 0
#define VOXL_F64 1      /* bitwise parity mode */
#define VOXL_HALO_ZERO_COPY 0 /* shared-layer kernel stores into the neighbour halo */
#define VOXL_HALO_COPY 1      /* span copies after the step (halo_update)          */
#define VOXL_HALO_NCCL 2      /* the same spans by grouped ncclSend/ncclRecv (multi-device engines,
                                 one distinct device per partition): the measured comparison */
#define VOXL_NAIVE 0          /* sparse::Strategy (sparse.hpp:117) */
#define VOXL_DISAG_BITMASK 1
#define VOXL_DISAG_MEM 2
#define VOXL_OP_LBM 0         /* closed step_occ operator set (see voxl_dense_desc::op) */
#define VOXL_OP_IDENTITY 1
#define VOXL_OP_JACOBI2 2
#define VOXL_BAD_DENSITY 31   /* voxl_diag::bad_population of a non-positive density (macroscopic's
                                 throw, lattice.cpp:124) rather than a population out of range */

const char* voxl_last_error(void);
int voxl_version(void);
/** Visible CUDA devices (the multi-device engine places partitions on them). */
int voxl_device_count(int* count);
/** Lattice descriptor as the reference's lattice_to_json (lattice.cpp:140-158). */
int voxl_lattice_json(int lattice, char* out, int64_t cap, int64_t* len);

/* ---- dense grid layer (layout.hpp / partition.hpp) ----------------------------- */

/** LayoutMap::build(scheme, shape, q, axis, TransferSets::for_lattice).to_json()
 *  (layout.cpp:72, :203). lattice < 0: generic build with `cardinality`. */
int voxl_layout_json(int scheme, int nx, int ny, int nz, int lattice, int cardinality, int axis, char* out,
                     int64_t cap, int64_t* len);
/** LayoutMap::address for every (voxel, component), voxels k = -1..n (partition
 *  axis), cross-section row-major, component innermost (layout.cpp:149). */
int voxl_layout_addresses(int scheme, int nx, int ny, int nz, int lattice, int axis, int64_t* out, int64_t cap,
                          int64_t* count);
/** decompose (partition.cpp:20): slabs[2p], slabs[2p+1] = [begin, end). */
int voxl_decompose(int nx, int ny, int nz, int parts, int axis, int periodic, int* slabs);
/** classify_voxels (partition.cpp:43): 0 Private / 1 Shared per owned voxel. */
int voxl_classify_voxels(int nx, int ny, int nz, int parts, int axis, int periodic, int p, uint8_t* out,
                         int64_t cap);

/** initial_canonical_state (solver.cpp:165-187): rest equilibrium, or the
 *  periodic box's mt19937_64-perturbed state; volume * q doubles, canonical. */
int voxl_initial_state(int lattice, int scenario, int nx, int ny, int nz, uint64_t seed, double perturbation,
                       double* out);

/* ---- dense engine (PartitionedField + step_occ + GatherKernel) ------------------ */

typedef struct voxl_dense voxl_dense;

typedef struct {
    int lattice;          /* VOXL_D2Q9 | VOXL_D3Q19 | VOXL_D3Q27 */
    int nx, ny, nz;       /* SolverConfig::domain (solver.hpp:29) */
    double tau;
    int scenario;         /* VOXL_CAVITY | VOXL_PERIODIC */
    double velocity[3];   /* lid velocity */
    int layout;           /* VOXL_AOS | VOXL_SOA | VOXL_DISAG_SOA */
    int partitions;       /* 1D slab count along z (y in 2D) */
    int precision;        /* VOXL_F32 | VOXL_F64 */
    int halo_mode;        /* VOXL_HALO_ZERO_COPY | VOXL_HALO_COPY */
    int first_partition;  /* owned range for multi-process use ... */
    int local_partitions; /* ... -1 = all partitions in this process */
    int op;               /* step_occ kernel (partition.hpp:173): VOXL_OP_LBM (GatherKernel,
                             lbm.hpp:123) | VOXL_OP_IDENTITY (partition_test.cpp:189) |
                             VOXL_OP_JACOBI2 (five-point, 2 components, partition_test.cpp:234);
                             0 = LBM for zero-initialised descriptors */
} voxl_dense_desc;

typedef struct {
    double mass;          /* lbm::Diagnostics (lbm.hpp:137-141) */
    double max_speed;
    int unstable;         /* probe_field would throw (lbm.cpp:124-128) */
    int bad_population;
    int64_t bad_voxel;
} voxl_diag;

typedef struct {
    int step, src, dst;   /* TransferRecord (partition.hpp:35-41) */
    int64_t src_base, dst_base, elements;
} voxl_transfer_record;

/** PartitionedField x2 (partition.cpp:111) on the current device. */
int voxl_dense_create(const voxl_dense_desc* desc, voxl_dense** out);
/** The reference's in-process PartitionedField over several GPUs (partition.hpp:92-126):
 *  partition p lives on devices[p] (`partitions` entries; repeats allowed, e.g. all 0).
 *  Peer access is enabled between the devices; each partition runs the two-stream
 *  OCC schedule (interior stream + high-priority shared-layer stream) and the
 *  streams of neighbouring partitions are ordered by cross-device events, so the
 *  zero-copy halo stores overlap the interior. graph_steps (even, 0 = off): steps
 *  per captured CUDA graph replayed by voxl_dense_step / enqueue / timed_steps.
 *  halo_mode VOXL_HALO_NCCL needs one distinct device per partition. */
int voxl_dense_create_multi(const voxl_dense_desc* desc, const int* devices, int graph_steps, voxl_dense** out);
/** Device of partition p. */
int voxl_dense_device(voxl_dense* h, int partition, int* device);
/** PartitionedField::neighbors (partition.hpp:110): (upper, lower), -1 at a domain end. */
int voxl_dense_neighbors(voxl_dense* h, int partition, int* upper, int* lower);
/** PartitionedField::set_neighbor_links (partition.hpp:111-113), the fault-injection
 *  hook: the next step or halo refresh on asymmetric links fails with VOXL_RUNTIME
 *  "halo_update: asymmetric neighbor links" (partition.cpp:165-171). */
int voxl_dense_set_neighbor_links(voxl_dense* h, int partition, int upper, int lower);
int voxl_dense_destroy(voxl_dense* h);
/** fill_canonical (partition.cpp:143): canonical fp64, x fastest, component innermost. */
int voxl_dense_set_canonical(voxl_dense* h, const double* host);
/** make_equilibrium_state (lbm.cpp:72): every voxel at equilibrium(rho, u), on the device. */
int voxl_dense_set_equilibrium(voxl_dense* h, double rho, const double* u);
/** to_canonical (partition.cpp:123). */
int voxl_dense_get_canonical(voxl_dense* h, double* host);
/** Planes [k_begin, k_end) of the partition axis only (chunked I/O). */
int voxl_dense_set_planes(voxl_dense* h, const double* host, int k_begin, int k_end);
int voxl_dense_get_planes(voxl_dense* h, double* host, int k_begin, int k_end);
/** Digest of to_canonical() computed on the device (no host copy of the field):
 *  out[0] = sum_i h(i, bits(x_i)) mod 2^64, out[1] = xor_i rotl(h, 29),
 *  h(i, b) = splitmix64(b ^ splitmix64(i)), i = canonical element index.
 *  Equal digests <=> bitwise-equal canonical states (full-size parity checks). */
int voxl_dense_digest(voxl_dense* h, uint64_t* out2);
/** n x step_occ(a, b, GatherKernel) (partition.hpp:173) then error check. */
int voxl_dense_step(voxl_dense* h, int n);
/** Enqueue n steps on the engine stream; no host synchronisation. */
int voxl_dense_enqueue(voxl_dense* h, int n);
int voxl_dense_synchronize(voxl_dense* h);
/** n steps timed with CUDA events on the engine stream: total span and the
 *  sum of per-step (kernel) spans, in milliseconds. */
int voxl_dense_timed_steps(voxl_dense* h, int n, double* total_ms, double* kernel_ms);
/** probe_field on the current state (lbm.cpp:116), on the device. */
int voxl_dense_probe(voxl_dense* h, voxl_diag* out);
/** One step_occ with probe_field fused into the step kernel: the per-step
 *  diagnostics row of voxl::run (solver.cpp:245-255) without a second pass. */
int voxl_dense_step_probe(voxl_dense* h, voxl_diag* out);
/** n x (step_occ + probe_field), the per-step loop of run_dense (solver.cpp:245-255),
 *  with the probe fused into the step kernel and the diagnostics rows accumulated
 *  on the device: one host synchronisation per 256 steps instead of one per step.
 *  rows[s] = diagnostics of the s-th step. On the first failing step the call
 *  returns VOXL_INSTABILITY with run()'s text ("run aborted at step N:
 *  macroscopic: non-positive density" / "... instability at step N, voxel V,
 *  population I", N = the engine's step index) and *completed = the rows filled. */
int voxl_dense_step_probe_n(voxl_dense* h, int n, voxl_diag* rows, int* completed);
/** Observed counterpart of TraceLog (partition.hpp:76-90): while enabled, every
 *  phase the engine launches (per partition: "step", or "interior" + "shared" on
 *  two streams in the multi-device / multi-process schedules, "halo_copy" in copy
 *  mode) is bracketed by CUDA events; disabling clears the record. NVTX ranges
 *  name every phase launch regardless. */
int voxl_dense_trace_enable(voxl_dense* h, int on);
/** The record as JSON: [{"step", "stage", "phase", "partition", "device", "stream",
 *  "begin_ms", "end_ms"}, ...] in launch order, times from the first event on the
 *  same device (waits for the recorded steps). */
int voxl_dense_trace_json(voxl_dense* h, char* out, int64_t cap, int64_t* len);
/** Ledger records of one step in the reference's order (partition.cpp:163-206). */
int voxl_dense_ledger(voxl_dense* h, int step, voxl_transfer_record* out, int cap, int* count);
/** The same records from a descriptor alone (no device needed). */
int voxl_dense_plan_ledger(const voxl_dense_desc* desc, int step, voxl_transfer_record* out, int cap, int* count);
int voxl_dense_layout_json(voxl_dense* h, int partition, char* out, int64_t cap, int64_t* len);
int voxl_dense_steps_done(voxl_dense* h, int* steps);
/** Device buffer of a partition: which 0 = current, 1 = next. */
int voxl_dense_buffer(voxl_dense* h, int partition, int which, void** ptr, size_t* bytes);
/** cudaStream_t of the engine, as void*. */
int voxl_dense_stream(voxl_dense* h, void** stream);
/** Multi-process: the shared-layer stream of the OCC step (after
 *  voxl_dense_enable_distributed). In copy halo mode the caller enqueues the
 *  halo exchange of each step here, so it overlaps the interior kernel
 *  (the OCC schedule, partition.hpp:173-214, with NCCL as the transport). */
int voxl_dense_shared_stream(voxl_dense* h, void** stream);
/** Multi-process: map a neighbour partition's buffers (IPC/peer pointers, both parities). */
int voxl_dense_attach_peer(voxl_dense* h, int partition, void* buf0, void* buf1);
/** Allocation-order buffer w (0/1) of an owned partition (for IPC export). */
int voxl_dense_raw_buffer(voxl_dense* h, int partition, int w, void** ptr);
/** Multi-process zero-copy: allocate the step-flag words (returned, for IPC export). */
int voxl_dense_enable_distributed(voxl_dense* h, void** flags);
/** The neighbours' flag slots this rank signals after its shared layers
 *  (upper neighbour's flags + 1 word, lower neighbour's flags + 0); NULL at a domain end. */
int voxl_dense_attach_flags(voxl_dense* h, void* upper_slot, void* lower_slot);
/** Peer-copy this rank's shared slabs into the neighbours' halos (after set_canonical). */
int voxl_dense_halo_push(voxl_dense* h);
int voxl_dense_owned_voxels(voxl_dense* h, int64_t* voxels);

/* ---- block-sparse engine (sparse::SparseLbmEngine, sparse.hpp:175-213) --------- */

typedef struct voxl_sparse voxl_sparse;

typedef struct {
    int lattice;        /* VOXL_D3Q19 | VOXL_D3Q27 */
    int nx, ny, nz;
    double tau;
    double u_bc[3];     /* regularized inflow/outflow velocity (SparseScenario::wind_tunnel) */
    int block_edge;     /* 4 (reference tables) or 8 (B200 production) */
    int strategy;       /* VOXL_NAIVE | VOXL_DISAG_BITMASK | VOXL_DISAG_MEM */
    int precision;      /* VOXL_F32 | VOXL_F64 */
} voxl_sparse_desc;

/** Active set of run_sparse (solver.cpp:272-283): box minus sphere of `radius`
 *  (<= 0: min extent / 5) centred at (n/2 - 0.5); x fastest bytes. */
int voxl_obstacle_mask(int nx, int ny, int nz, double radius, uint8_t* out, int64_t* active);
/** BlockSparseGrid::build + classify_blocks + arrange + dispatch_plan
 *  (sparse.cpp:20, :109, :144, :199) and device buffers at rest equilibrium. */
int voxl_sparse_create(const voxl_sparse_desc* desc, const uint8_t* active, voxl_sparse** out);
int voxl_sparse_destroy(voxl_sparse* h);
/** The same grid, classification, arrangement and plan with no device
 *  allocation (host tables only); the getters below accept either handle
 *  kind through voxl_sparse_plan_of. */
typedef struct voxl_sparse_plan voxl_sparse_plan;
int voxl_sparse_plan_create(const voxl_sparse_desc* desc, const uint8_t* active, voxl_sparse_plan** out);
int voxl_sparse_plan_destroy(voxl_sparse_plan* p);
/** Host tables of an engine (owned by the engine). */
int voxl_sparse_plan_of(voxl_sparse* h, voxl_sparse_plan** out);
int voxl_sparse_plan_info(voxl_sparse_plan* p, int64_t* num_active, int* num_blocks, int64_t* n_boundary,
                          int64_t* n_non_boundary);
int voxl_sparse_plan_blocks(voxl_sparse_plan* p, int* origins, uint64_t* masks, uint8_t* classes);
int voxl_sparse_plan_arrangement(voxl_sparse_plan* p, int* permutation, uint8_t* bitmask, int32_t* meta_index,
                                 int64_t* boundary_voxels);
int voxl_sparse_plan_report_json(voxl_sparse_plan* p, char* out, int64_t cap, int64_t* len);
/** 27-neighbour block table, d = (dx+1) + 3(dy+1) + 9(dz+1), -1 when absent. */
int voxl_sparse_plan_neighbours(voxl_sparse_plan* p, int32_t* out);
int voxl_sparse_info(voxl_sparse* h, int64_t* num_active, int* num_blocks, int64_t* n_boundary,
                     int64_t* n_non_boundary);
/** Blocks in list order: origins (3 ints), masks (block_edge^3/64 words, >= 1), class (1 = boundary). */
int voxl_sparse_blocks(voxl_sparse* h, int* origins, uint64_t* masks, uint8_t* classes);
/** Arrangement (sparse.hpp:101-107): permutation, bitmask, voxel_meta_index (any may be NULL). */
int voxl_sparse_arrangement(voxl_sparse* h, int* permutation, uint8_t* bitmask, int32_t* meta_index,
                            int64_t* boundary_voxels);
/** ExecutionReport::to_json (sparse.cpp:240-251). */
int voxl_sparse_report_json(voxl_sparse* h, char* out, int64_t cap, int64_t* len);
/** canonical_state / set_state (sparse.cpp:416-453): pack_coord order, q per voxel. */
int voxl_sparse_get_state(voxl_sparse* h, double* canonical);
int voxl_sparse_set_state(voxl_sparse* h, const double* canonical);
/** Digest of canonical_state() on the device (see voxl_dense_digest). */
int voxl_sparse_digest(voxl_sparse* h, uint64_t* out2);
int voxl_sparse_set_equilibrium(voxl_sparse* h, double rho, const double* u);
/** n x SparseLbmEngine::step (sparse.cpp:386-394). */
int voxl_sparse_step(voxl_sparse* h, int n);
/** SparseLbmEngine::step_identity (sparse.cpp:396-404): state unchanged. */
int voxl_sparse_step_identity(voxl_sparse* h, int n);
int voxl_sparse_timed_steps(voxl_sparse* h, int n, double* total_ms, double* boundary_ms, double* light_ms);
int voxl_sparse_probe(voxl_sparse* h, voxl_diag* out);
/** One SparseLbmEngine::step with probe_field fused into the step kernels:
 *  run_sparse's per-step diagnostics row (solver.cpp:287-291). */
int voxl_sparse_step_probe(voxl_sparse* h, voxl_diag* out);
/** n x (step + probe_field), run_sparse's per-step loop (solver.cpp:287-291),
 *  rows accumulated on the device (one host synchronisation per 256 steps).
 *  Same contract as voxl_dense_step_probe_n. */
int voxl_sparse_step_probe_n(voxl_sparse* h, int n, voxl_diag* rows, int* completed);
/** dispatch_plan(...).to_json() (sparse.cpp:199-225; Table 2). */
int voxl_dispatch_plan_json(int strategy, int64_t n_b, int64_t n_nb, int q, int block_size, int s_w, int s_i,
                            int naive_full_domain_storage, char* out, int64_t cap, int64_t* len);

/* ---- multi-resolution engine (mres::MultiResLbm, multires.hpp:138-190) ---------- */

typedef struct voxl_mres voxl_mres;
typedef struct voxl_mres_plan voxl_mres_plan;

typedef struct {
    int lattice;          /* VOXL_D2Q9 (nz = 1) | VOXL_D3Q19 | VOXL_D3Q27 */
    int nx, ny, nz;       /* virtual finest domain */
    int levels;           /* 1..4 */
    double tau;           /* coarsest level; tau_l = 2 tau_{l+1} - 1/2 */
    double lid_u[3];      /* lid velocity (cavity, lid on the max-z face; max-y in 2D) */
    int fused;            /* FusedCollideStream on uniform blocks (multires.cpp:541) */
    int precision;        /* VOXL_F32 | VOXL_F64 */
    int block_edge;       /* 8 (production) or 4 (reference granularity) */
    int reference_tables; /* also build the edge-4 ghost / pull / fusion tables */
    int solid_cells;      /* extension beyond the reference (whose build rejects ids outside
                             [0, levels), multires.cpp:84-85): level-map value -1 marks solid
                             bounce-back cells inside the finest level (>= 3 cells from any
                             coarser cell); 0 = reference semantics */
} voxl_mres_desc;

/** Band level map of run_multires (solver.cpp:319-335), x fastest int32. */
int voxl_band_level_map(int nx, int ny, int nz, int levels, int axis, int32_t* out);
/** MultiResGrid::build + MultiResLbm (multires.cpp:54, :367), rest equilibrium. */
int voxl_mres_create(const voxl_mres_desc* desc, const int32_t* level_map, voxl_mres** out);
int voxl_mres_destroy(voxl_mres* h);
/** n x coarse_step (multires.cpp:576). */
int voxl_mres_step(voxl_mres* h, int n);
/** n coarse steps timed with CUDA events: out[5] = total, collide, stream, fused, transition ms. */
int voxl_mres_timed_steps(voxl_mres* h, int n, double* out5);
int voxl_mres_state_len(voxl_mres* h, int64_t* len);
/** canonical_state / set_state (multires.cpp:578-598, :396-410): levels finest
 *  first, cells sorted by pack_coord, q populations each. */
int voxl_mres_get_state(voxl_mres* h, double* canonical);
int voxl_mres_set_state(voxl_mres* h, const double* canonical);
/** Digest of canonical_state() on the device (see voxl_dense_digest). */
int voxl_mres_digest(voxl_mres* h, uint64_t* out2);
int voxl_mres_set_equilibrium(voxl_mres* h, double rho, const double* u);
/** probe_field over canonical_state (solver.cpp:345). */
int voxl_mres_probe(voxl_mres* h, voxl_diag* out);
/** n x (coarse_step + probe_field), run_multires's per-step loop (solver.cpp:343-345),
 *  with the probe fused into each level's last sub-step kernels and the rows
 *  accumulated on the device (one host synchronisation per 256 steps). Same
 *  contract as voxl_dense_step_probe_n: rows[s] = diagnostics of the s-th step;
 *  VOXL_INSTABILITY with run()'s text at the first failing step, *completed =
 *  the rows filled. */
int voxl_mres_step_probe_n(voxl_mres* h, int n, voxl_diag* rows, int* completed);
/** total_mass (multires.cpp:600-609): per-level sums weighted by 8^l. */
int voxl_mres_total_mass(voxl_mres* h, double* mass);
/** what: 0 = execution graph DOT, 1 = distribution report. */
int voxl_mres_text(voxl_mres* h, int what, char* out, int64_t cap, int64_t* len);
/** Per level: active cells, tau, ghost cells, ring cells, uniform / jump blocks (device grid). */
int voxl_mres_level_info(voxl_mres* h, int level, int64_t* num_active, double* tau, int64_t* uniform_blocks,
                         int64_t* jump_blocks);
int voxl_mres_lup_per_coarse_step(voxl_mres* h, int64_t* lup);
/** Host tables only (no device): MultiResGrid::build with reference tables. */
int voxl_mres_plan_create(const voxl_mres_desc* desc, const int32_t* level_map, voxl_mres_plan** out);
int voxl_mres_plan_destroy(voxl_mres_plan* p);
int voxl_mres_plan_level(voxl_mres_plan* p, int level, int64_t* num_active, double* tau, int* ref_blocks,
                         int* n_ghosts, int* n_pulls);
/** Edge-4 blocks of a level: origins, 64-bit masks, fusion class (1 = Jump). */
int voxl_mres_plan_ref_blocks(voxl_mres_plan* p, int level, int* origins, uint64_t* masks, uint8_t* jump);
/** Ghost list: 6 ints each (cell xyz, parent xyz); pulls: 7 ints each (voxel xyz, direction, refined xyz). */
int voxl_mres_plan_ghosts(voxl_mres_plan* p, int level, int* out);
int voxl_mres_plan_pulls(voxl_mres_plan* p, int level, int* out);
/** jump_distance (multires.cpp:214-223); INT_MAX = no interface. */
int voxl_mres_plan_jump_distance(voxl_mres_plan* p, int level, int x, int y, int z, int* out);
/** what: 0 = DOT (fused graph), 1 = DOT (staged graph), 2 = distribution report. */
int voxl_mres_plan_text(voxl_mres_plan* p, int what, char* out, int64_t cap, int64_t* len);

/* ---- CUDA IPC helpers (64-byte cudaIpcMemHandle_t as bytes) ------------------- */
int voxl_ipc_export(void* dev_ptr, char* handle64);
int voxl_ipc_open(const char* handle64, void** dev_ptr);
int voxl_ipc_close(void* dev_ptr);
int voxl_enable_peer_access(int peer_device);

#ifdef __cplusplus
}
#endif
#endif
