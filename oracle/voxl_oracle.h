/* voxl_oracle.h -- plain-C restatement of the reference's LBM hot path.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the thing measured or shipped).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * oracle/_ref/libvoxl_oracle.so. Parity of this restatement is pinned against the
 * reference library itself (oracle/_ref/libvoxl_ref.so, built from
 * /root/reference/proj/src by oracle/Makefile) and the reference's golden files
 * (tests/golden/lattice_d2q9.json, layout_disag_d2q9.json) by tests/test_oracle.py.
 *
 * Every arithmetic sequence follows the reference's IEEE double evaluation order
 * (compiled with -ffp-contract=off), so results are bitwise comparable.
 */
#ifndef VOXL_ORACLE_H
#define VOXL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { VO_D2Q9 = 0, VO_D3Q19 = 1, VO_D3Q27 = 2 };

typedef struct {
    int kind, dim, q;
    int e[27][3];
    double w[27];
    long long wnum[27], wden[27];
    int opp[27];
} vo_lattice;

/* build_lattice (proj/src/lattice.cpp:59-102) */
void vo_build_lattice(int kind, vo_lattice* lat);

/* Dense flow rules (proj/include/voxl/lbm.hpp:23-31). */
typedef struct {
    int n[3];
    int periodic[3];
    int wrap[3];
    int has_lid, lid_axis, lid_at_max;
    double lid_u[3];
} vo_rules;

/* rules_for (proj/src/solver.cpp:150-163); scenario 0 cavity, 1 obstacle, 2 periodic. */
void vo_rules_for(int kind, int scenario, int nx, int ny, int nz, const double vel[3], vo_rules* r);

/* initial_canonical_state (proj/src/solver.cpp:165-187), mt19937_64 + libstdc++
 * uniform_real_distribution<double>(-1, 1) restated. */
void vo_initial_state(int kind, int scenario, int nx, int ny, int nz, uint64_t seed,
                      double perturbation, double* out);

/* reference_dense_run loop body: `steps` x fused_stream_collide (lbm.cpp:104-114)
 * starting from `state` (canonical: x fastest voxels, component innermost). The
 * result is written back into `state`. Returns 0, or -1 on a runtime error that
 * the reference would throw (non-positive density / non-finite input). */
int vo_dense_run(int kind, const vo_rules* r, double tau, int steps, double* state);

/* regularized_reconstruct (proj/src/lbm.cpp:10-59) */
int vo_regularized(const vo_lattice* lat, int axis, int sign, const double u_bc[3], double* f);

/* probe_field (proj/src/lbm.cpp:116-138); returns 0 or -1 (instability). */
int vo_probe(int kind, const double* canonical, int64_t voxels, double* mass, double* max_speed,
             int64_t* bad_voxel, int* bad_pop);

/* Block-sparse wind tunnel (SparseLbmEngine semantics, proj/src/sparse.cpp:321-394)
 * restated over a dense activity mask: the per-voxel update does not depend on
 * the block decomposition or the dispatch strategy (sparse_test.cpp:228-302).
 * `state` holds nx*ny*nz*q doubles (x fastest; inactive voxels ignored). */
int vo_sparse_run(int kind, int nx, int ny, int nz, const uint8_t* active, double tau,
                  const double u_bc[3], int steps, double* state);

/* Sphere-obstacle active set of run_sparse (proj/src/solver.cpp:272-283). */
int64_t vo_obstacle_mask(int nx, int ny, int nz, double radius, uint8_t* active);

/* Multires band cavity (MultiResLbm, proj/src/multires.cpp:367-576) restated over
 * dense per-level arrays. level_map: virtual-finest canonical order. The state
 * out is the reference's canonical_state (levels finest->coarsest, cells sorted
 * by pack_coord (x slowest, z fastest), component innermost). Returns the number
 * of doubles written, or -1.
 * Extension beyond the reference (PARITY UNPINNED for it: the reference's build
 * rejects such maps, multires.cpp:84-85): level_map value -1 marks solid cells
 * inside the finest level; a fluid cell pulling from one bounces back (own
 * post-collision opposite population, as at the domain walls). */
int64_t vo_mres_run(int kind, int nx, int ny, int nz, int levels, const int* level_map, double tau,
                    const double lid_u[3], int steps, double* out, int64_t cap);

/* Band level map of run_multires (proj/src/solver.cpp:319-335). */
void vo_band_level_map(int nx, int ny, int nz, int levels, int axis, int* map);

/* `steps` x the five-point Jacobi of proj/tests/partition_test.cpp:234-247 on a
 * 2-component field (canonical, x fastest, component innermost), each z plane
 * independently. step_occ is partition-invariant for it (the same test), so the
 * single-grid restatement is the oracle for every partitioning. In place. */
void vo_jacobi2_run(int nx, int ny, int nz, int steps, double* state);

#ifdef __cplusplus
}
#endif
#endif
