/* oracle.h -- plain, slow, obviously-correct CPU oracle for the ForestClaw hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load liboracle.so.  The product path (paper_1308_1472_b200/) never
 * includes, links or calls anything here, and this oracle shares no source with it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, SURVEY.md §8(c) readings):
 *   - forest decode: leaves in Morton order -> (tree, level, x, y)        PAPER.md:240-245 [§4]
 *   - ghost-source classification by brute-force geometry (point location of every ghost-cell
 *     centre, crossing tree faces through the connectivity)               PAPER.md:137-146 [§2], 258-260 [§4]
 *   - ghost fill: copy / average / limited interpolation / physical BC / CORNER3
 *                                                                          PAPER.md:187-201 [§3]
 *   - Clawpack wave-propagation patch update (normal + transverse Riemann solves, wave limiter,
 *     second-order corrections) and the CFL number                       PAPER.md:168-182 [§3]
 * All floating point is IEEE fp64, compiled with -ffp-contract=off.
 *
 * Parity pins: see DESIGN.md "Oracle pins".  Functions without a pin say so in DESIGN.md.
 */
#ifndef FC_ORACLE_H
#define FC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ETILING = -2, ORC_ECONN = -3, ORC_EBALANCE = -4,
       ORC_ENOMEM = -5, ORC_EUNSUP = -6, ORC_EPHYS = -7 };

/* ghost-table record ops (canonical EXPANDED table) */
enum { ORC_OP_NONE = 0, ORC_OP_COPY = 1, ORC_OP_AVG4 = 2, ORC_OP_INTERP = 3, ORC_OP_BCX = 4,
       ORC_OP_BCY = 5, ORC_OP_CORNER3 = 6 };

enum { ORC_ADV_CONST = 0, ORC_ADV_EDGEVEL_CAPA = 1, ORC_SWE_ROE = 2, ORC_EULER_ROE = 3, ORC_EULER_HLLE = 4 };
enum { ORC_LIM_NONE = 0, ORC_LIM_MINMOD = 1, ORC_LIM_MC = 2 };
enum { ORC_BC_OUTFLOW = 0, ORC_BC_WALL = 1 };

typedef struct orc_forest orc_forest;

typedef struct {
  int kind;        /* ORC_ADV_CONST ... */
  double p0, p1;   /* (u, v) | unused | (g, -) | (gamma, efix) */
  int limiter;     /* ORC_LIM_* */
  int method2;     /* 1: first order, 2: + limited second-order corrections */
  int method3;     /* 0: none, 1: transverse of A+-dq, 2: transverse of A+-dq -+ F~ */
  int reflux;      /* 1: conservative coarse/fine flux correction after the update (orc_reflux) */
} orc_problem;

int orc_forest_create(int64_t num_patches, const int8_t* levels, const int32_t* tree_ids,
                      int32_t num_trees, const int32_t* tree_to_tree, const int8_t* tree_to_face,
                      const int8_t* face_bc, int m, orc_forest** out);
void orc_forest_destroy(orc_forest* f);
/* decoded leaf coordinates in units of level-Lmax leaves */
int orc_forest_coords(const orc_forest* f, int64_t* x, int64_t* y, int* lmax);

/* ring cells per patch and the record width */
int orc_ring_count(int m);
#define ORC_REC 8
/* canonical ghost records of patch p: ring cells in storage order (j = -1..m+2 outer,
 * i = -1..m+2 inner, interior skipped); each record {op, src_patch, src_i, src_j, a, b, c, d} */
int orc_ghost_records(const orc_forest* f, int64_t p, int32_t* rec);
int orc_ghost_table(const orc_forest* f, int32_t* rec /* [P][G][8] */);

/* Fill the ghost rings of all patches of qpad[P][meqn][n][n] (n = m+4) in the phase order
 * A (copy, average) -> C (BC x then y) -> for each level ascending: B (interpolate) -> C -> CORNER3 */
int orc_ghost_fill(const orc_forest* f, double* qpad, int meqn);

/* One step on every patch: ghost fill of qpad (rings overwritten), then the wave-propagation
 * update written into the interiors of qout (same layout).  aux: [P][maux][n][n] or NULL.
 * *cfl = max over patches.  nthreads <= 1 runs single-threaded (bitwise identical). */
int orc_step(const orc_forest* f, const orc_problem* pr, double* qpad, const double* aux,
             double dt, double dx0, double* qout, double* cfl, int nthreads);
/* dx0 = cell width of a level-0 patch (tree edge / m); a level-l patch has dx = dx0 2^-l */

/* One step from interior-only data q[P][meqn][m][m] for the listed patches only (sampled
 * parity at full size): rings are built from the neighbours' interiors.  out[ns][meqn][m][m]. */
int orc_step_sample(const orc_forest* f, const orc_problem* pr, const double* q,
                    const double* aux, double dt, double dx0,
                    const int64_t* ids, int64_t ns, double* out, double* cfl_out);
/* padded array [meqn][n][n] of patch p with its ring filled from interior-only data q */
int orc_build_padded_sample(const orc_forest* f, const double* q, int meqn, int64_t p, double* out);

/* single-patch update on a padded patch (ring already filled) -> patch CFL */
double orc_step_patch(const orc_problem* pr, int m, int meqn, const double* qp, const double* auxp,
                      double dt, double dx, double dy, double* qnew);

/* orc_step_patch plus the applied boundary-edge fluxes face[4][m][meqn] (faces -x, +x, -y, +y;
 * edge e = cell row / column e+1 of the face), in outward form (see claw.c); face may be NULL */
double orc_step_patch_faces(const orc_problem* pr, int m, int meqn, const double* qp, const double* auxp,
                            double dt, double dx, double dy, double* qnew, double* face);
/* Conservative coarse/fine flux correction ("reflux"; PAPER.md:279-282 [§4]):
 * every coarse cell C adjacent to a face whose neighbour is one level finer gets, per such face,
 *   Q_C += dt / (kappa_C dx_C) (out_C + (out_f1 + out_f2) / 2)
 * -- its own applied flux replaced by the mean of the two fine fluxes through the same face
 * (fine edges found by point location across the connectivity), all in outward form.  faces =
 * [P][4][m][meqn] from orc_step_patch_faces of the same step; qout updated in place.  Systems
 * (meqn > 1) across non-aligned tree links are not supported (ORC_EUNSUP). */
int orc_reflux(const orc_forest* f, const orc_problem* pr, const double* faces, const double* aux,
               double dt, double dx0, double* qout);
/* general form (coarse patches of one level, weighted records), see forest.c */
int orc_reflux_ex(const orc_forest* f, const orc_problem* pr, const double* faces, const double* faces_f,
                  double wc, double dtr, int level, const double* aux, double dx0, double* qout);
/* Sub-cycled step (PAPER.md:201-202 [§3] "when sub-cycling, time accurate data between coarse grids
 * is used to fill in ghost cells for fine grids"; PAPER.md:277-290 [§4] one exchange per level,
 * coarse-to-fine recursion, correction factors propagated back): level l advances with
 * dt_l = dt_coarse 2^-(l - lmin); advance(l, t): ghost fill at time t of a snapshot in which every
 * patch of level >= l holds its current state and every coarser patch the linear interpolation in
 * time between its last two states, update of the level-l patches, then two advances of level
 * l+1 at t and t + dt_{l+1}, then (reflux on) the level-l / level-(l+1) flux correction with the
 * coarse flux x dt_l against the fine fluxes x dt_{l+1} summed over both sub-steps.  Times are
 * integer ticks of the finest sub-step, so the interpolation weights are exact dyadic numbers.
 * qpad [P][meqn][n][n] in (interiors used), qout interiors out; *cfl = max over all updates. */
int orc_step_subcycled(const orc_forest* f, const orc_problem* pr, const double* qpad, const double* aux,
                       double dt_coarse, double dx0, double* qout, double* cfl);
/* Dynamic regrid of the forest (regrid.c): tag by
 * max - min of component 0, refine above refine_threshold (level < max_level), 2:1 balance by
 * refinement, coarsen complete families below coarsen_threshold (level > min_level) whose
 * neighbours allow it; new leaves in Morton order with the data interpolated (limited, minmod,
 * from the ghost-filled qpad) or averaged.  Outputs (capacity 4P): new_levels, new_trees,
 * qout[new_P][meqn][m][m], and if src != NULL src[new_P][6] = {kind (1 copy, 2 child, 3 parent),
 * old patch (first child for a parent), child index, 0, 0, 0}. */
int orc_regrid(const orc_forest* f, const double* qpad, int meqn, double refine_threshold,
               double coarsen_threshold, int min_level, int max_level, int64_t* new_P, int8_t* new_levels,
               int32_t* new_trees, double* qout, int32_t* src);
/* physical flux along axis ixy of state q (uedge: edge velocity, advective form) */
void orc_flux(const orc_problem* pr, int ixy, const double* q, double uedge, double* f);

/* pieces exposed for the pin tests */
double orc_limiter(int limiter, double theta);
int orc_meqn(int kind);
int orc_mwaves(int kind);
/* normal Riemann solve at one edge: waves[mwaves][meqn], s[mwaves], amdq[meqn], apdq[meqn] */
int orc_rpn2(const orc_problem* pr, int ixy, const double* ql, const double* qr,
             const double* auxl, const double* auxr, double* waves, double* s, double* amdq,
             double* apdq);
/* transverse split of asdq at the edge between ql and qr (ixy = direction of the edge normal);
 * aux_recv = aux of the receiving cell (3 values) and aux_recv_next = aux of the cell above
 * (ixy = 1) / to the right (ixy = 2) of it, for ADV_EDGEVEL_CAPA */
int orc_rpt2(const orc_problem* pr, int ixy, const double* ql, const double* qr,
             const double* aux_recv, const double* aux_recv_next, const double* asdq,
             double* bmasdq, double* bpasdq);


/* ---- forests of octrees (forest3.c): aligned bricks, meqn = 1 constant-velocity advection with
 * Godunov dimensional splitting (reading 26) ---------------------------------------- */
typedef struct orc3_forest orc3_forest;
int orc3_forest_create(int64_t P, const int8_t* levels, const int32_t* tree_ids, int32_t T,
                       const int32_t* t2t /* [6T] */, const int8_t* fbc /* [6T] 1 = outflow */, int m,
                       orc3_forest** out);
void orc3_forest_destroy(orc3_forest* f);
int orc3_forest_coords(const orc3_forest* f, int64_t* x, int64_t* y, int64_t* z, int* lmax);
int orc3_ring_count(int m);
int orc3_ghost_records(const orc3_forest* f, int64_t p, int32_t* rec);
int orc3_ghost_table(const orc3_forest* f, int32_t* rec);
int orc3_ghost_fill(const orc3_forest* f, double* qpad);
double orc3_step_patch(const orc3_forest* f, const double* qp, double u, double v, double w, int limiter,
                       int method2, double dt, double dx, double* qnew);
int orc3_step(const orc3_forest* f, double* qpad, double u, double v, double w, int limiter, int method2,
              double dt, double dx0, double* qout, double* cfl);

#ifdef __cplusplus
}
#endif
#endif
