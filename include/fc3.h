/* fc3.h -- C ABI of libfc's forest-of-OCTREES path (3D).
 *
 * PAPER.md:22-24 [abstract] (a forest of octrees, each leaf a patch of m^d cells)
 * [Fig. 1 caption] ("The situation in 3D (octrees) is analogous"), SURVEY §8(f) #4.  Scope
 * (reading 26): a brick of Tx x Ty x Tz octrees with aligned orientation, each tree face
 * linked to the opposite face of a neighbour (a self-link = periodic) or physical (outflow);
 * 2:1 balance across faces, edges and corners; m even >= 4 (m <= 32), mbc = 2, meqn = 1;
 * constant-velocity scalar advection by LeVeque's wave propagation (PAPER.md:168-182 [§3]) with
 * Godunov dimensional splitting (x, y, z sweeps); one GPU.  The ghost fill, the step and the CFL
 * are bitwise the oracle's (oracle/forest3.c): same operations in the same order, no contraction.
 *
 * Layout: q[P][m][m][m] (index [p][k][j][i], x fastest), patches in global Morton order (trees in
 * order; within a tree x in bits 3k, y in 3k+1, z in 3k+2).  Device state: natural padded blocks
 * [P][m+4][m+4][m+4].  Return codes and fc_last_error() as in fc.h.
 */
#ifndef FC3_H
#define FC3_H
#include <stdint.h>

#include "fc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fc3_forest fc3_forest;

typedef struct {
  int64_t num_patches;
  const int8_t* levels;          /* [P] */
  const int32_t* tree_ids;       /* [P] non-decreasing */
  int32_t m;                     /* cells per patch side, even, 4..32 */
  int32_t num_trees;
  const int32_t* tree_to_tree;   /* [6T] tree across face f = 0..5 (-x, +x, -y, +y, -z, +z) */
  const int8_t* face_bc;         /* [6T] 1 = physical (outflow), 0 = linked (to the opposite face) */
  double tree_dx0;               /* tree edge length */
  int32_t device;                /* CUDA device, or -1: host-only planning handle (tables only) */
} fc3_forest_desc;

/* Decode (Morton order per tree; FC_ETILING), check the connectivity (a linked face f of tree t
 * must be linked back through face f^1; FC_ECONN), locate every ghost cell's source (26
 * directions; FC_EBALANCE if a neighbour is more than one level off), build the typed device lists
 * and allocate the state.  Copies all inputs; *out NULL on failure. */
int fc3_forest_create(const fc3_forest_desc* desc, fc3_forest** out);
int fc3_forest_destroy(fc3_forest* f);

/* velocity (u, v, w), limiter FC_LIM_NONE / MINMOD / MC, method2 1 (first order) or 2,
 * cfl_reject (fc3_step commits only when max CFL <= it).  FC_EINVAL out of range. */
int fc3_set_problem(fc3_forest* f, double u, double v, double w, int limiter, int method2, double cfl_reject);

/* q[P][m][m][m] (host or device by `where`, caller-owned) -> interiors of q_old; FC_ESTATE before
 * fc3_set_problem or on a host-only handle. */
int fc3_set_q(fc3_forest* f, const double* q, int where);

/* Ghost fill of q_old: A (copy, 2x2x2 average) -> C (outflow x, y, z writers) -> per level
 * ascending B (limited interpolation) -> C.  PAPER.md:193-201 [§3]. */
int fc3_ghost_fill(fc3_forest* f);

/* Ghost fill + split update of every patch + max CFL (dt/dx max over the sweeps of |u_d|).
 * Commits iff max_cfl <= cfl_reject, else FC_ECFL with q unchanged; FC_EINVAL for dt <= 0. */
int fc3_step(fc3_forest* f, double dt, double* max_cfl);

/* Use the caller's cudaStream_t for all subsequent work (NULL = the handle's own stream). */
int fc3_set_stream(fc3_forest* f, void* stream);

/* interiors of q_old -> q[P][m][m][m]; padded blocks -> q[P][n][n][n] (n = m + 4).  Synchronous. */
int fc3_get_q(fc3_forest* f, double* q, int where);
int fc3_get_q_padded(fc3_forest* f, double* q, int where);

/* Canonical ghost records: per patch, per ring cell in storage order (k = -1..m+2 outer, then j,
 * i inner, interior skipped), 8 int32 {op, src_patch, si, sj, sk, a, b, c}: 1 COPY (source cell),
 * 2 AVG8 (lower corner cell of the 2x2x2 fine block), 3 INTERP (coarse cell; a, b, c = +-1 the
 * half of it the ghost centre lies in), 4 / 5 / 6 outflow BC along x / y / z (own cell with that
 * axis clamped; the last physical axis).  *len = P (n^3 - m^3) 8; FC_EINVAL if cap < *len.  Works
 * on host-only handles. */
int fc3_get_ghost_table(fc3_forest* f, int32_t* buf, int64_t cap, int64_t* len);

#ifdef __cplusplus
}
#endif
#endif
