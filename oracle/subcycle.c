/* subcycle.c -- oracle: sub-cycled (per-level dt) stepping (TEST INFRASTRUCTURE ONLY, see oracle.h).
 *
 * PAPER.md:201-202 [§3]: "When sub-cycling, time accurate data between coarse grids is used to
 * fill in ghost cells for fine grids."  PAPER.md:277-290 [§4]: "one exchange per discretization
 * level per time step if dt is chosen per-patch depending on its size (this is sometimes called
 * sub-cycling) ... interaction between neighbor patches is done in a hierarchy from coarse to fine
 * levels, and then correction factors are propagated back from fine to coarse levels".
 *
 * Written out plainly (readings in DESIGN.md):
 *   level l has dt_l = dt_coarse / 2^(l - lmin) (2:1 balance: the CFL is the same on every level);
 *   advance(l, t):
 *     snapshot: every patch of level >= l holds its current state, every coarser patch
 *       (1 - a) Q_old + a Q_new with a = (t - t_old) / (t_new - t_old) of its own level;
 *     ghost fill of the whole snapshot (orc_ghost_fill: copy / average / interpolate / BC);
 *     update of the level-l patches from the snapshot by dt_l (their Q_old := current first);
 *     if a finer level exists: advance(l+1, t), advance(l+1, t + dt_{l+1});
 *     reflux (pr->reflux): coarse cells of level l next to level l+1 get
 *       Q_C += (dt_l out_C + (F_1 + F_2)/2) / (kappa dx), F = sum over the two fine sub-steps of
 *       dt_{l+1} out_f.
 * Times are integer ticks (one tick = the finest sub-step), so the weights a are exact.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"
#include "oracle_internal.h"

typedef struct {
  const orc_forest* f;
  const orc_problem* pr;
  const double* aux;
  double dx0, dt0;          /* dt0 = dt of level lmin */
  int meqn, m, lmin, lmax;
  size_t S, SA, FS;
  double *cur, *old, *snap; /* [P][meqn][n][n] (interiors used in cur / old) */
  double *faces, *acc;      /* [P][4][m][meqn]: last applied face fluxes; dt-weighted fine sums */
  int64_t tick_old[64], tick_new[64];
  double cfl;
  int err;
} sub_ctx;

static void copy_interior(int m, int meqn, const double* src, double* dst) {
  for (int k = 0; k < meqn; ++k)
    for (int j = 1; j <= m; ++j)
      for (int i = 1; i <= m; ++i) {
        const size_t o = (size_t)k * ORC_N(m) * ORC_N(m) + ORC_IDX(m, i, j);
        dst[o] = src[o];
      }
}

static void advance(sub_ctx* c, int l, int64_t tick, int sub) {
  const orc_forest* f = c->f;
  const int m = c->m, meqn = c->meqn;
  const int64_t len = 1ll << (c->lmax - l);             /* ticks per level-l step */
  const double dt = ldexp(c->dt0, -(l - c->lmin));
  /* snapshot at time `tick` */
  for (int64_t p = 0; p < f->P; ++p) {
    const int lp = f->level[p];
    double* sp = c->snap + p * c->S;
    if (lp >= l) {
      copy_interior(m, meqn, c->cur + p * c->S, sp);
    } else {
      const double a = (double)(tick - c->tick_old[lp]) / (double)(c->tick_new[lp] - c->tick_old[lp]);
      const double* o = c->old + p * c->S;
      const double* q = c->cur + p * c->S;
      for (int k = 0; k < meqn; ++k)
        for (int j = 1; j <= m; ++j)
          for (int i = 1; i <= m; ++i) {
            const size_t x = (size_t)k * ORC_N(m) * ORC_N(m) + ORC_IDX(m, i, j);
            sp[x] = (1.0 - a) * o[x] + a * q[x];
          }
    }
  }
  int rc = orc_ghost_fill(f, c->snap, meqn);
  if (rc && !c->err) c->err = rc;
  /* update of level l */
  for (int64_t p = 0; p < f->P; ++p) {
    if (f->level[p] != l) continue;
    copy_interior(m, meqn, c->cur + p * c->S, c->old + p * c->S);
    const double h = ldexp(c->dx0, -l);
    const double cf = orc_step_patch_faces(c->pr, m, meqn, c->snap + p * c->S, c->aux ? c->aux + p * c->SA : NULL,
                                           dt, h, h, c->cur + p * c->S, c->faces + p * c->FS);
    if (cf > c->cfl || cf != cf) c->cfl = cf;
    if (c->pr->reflux) {                               /* fine-side sums over the parent's sub-steps */
      double* a = c->acc + p * c->FS;
      const double* fc = c->faces + p * c->FS;
      for (size_t x = 0; x < c->FS; ++x) a[x] = sub == 0 ? dt * fc[x] : a[x] + dt * fc[x];
    }
  }
  rc = orc_take_step_error();
  if (rc && !c->err) c->err = rc;
  c->tick_old[l] = tick;
  c->tick_new[l] = tick + len;
  if (l < c->lmax) {
    advance(c, l + 1, tick, 0);
    advance(c, l + 1, tick + len / 2, 1);
    if (c->pr->reflux) {
      rc = orc_reflux_ex(f, c->pr, c->faces, c->acc, dt, 1.0, l, c->aux, c->dx0, c->cur);
      if (rc && !c->err) c->err = rc;
    }
  }
}

int orc_step_subcycled(const orc_forest* f, const orc_problem* pr, const double* qpad, const double* aux,
                       double dt_coarse, double dx0, double* qout, double* cfl) {
  sub_ctx c;
  memset(&c, 0, sizeof(c));
  c.f = f; c.pr = pr; c.aux = aux; c.dx0 = dx0; c.dt0 = dt_coarse;
  c.m = f->m; c.meqn = orc_meqn(pr->kind);
  const int n = ORC_N(c.m);
  c.S = (size_t)c.meqn * n * n; c.SA = (size_t)3 * n * n; c.FS = (size_t)4 * c.m * c.meqn;
  c.lmin = 127; c.lmax = -1;
  for (int64_t p = 0; p < f->P; ++p) {
    if (f->level[p] < c.lmin) c.lmin = f->level[p];
    if (f->level[p] > c.lmax) c.lmax = f->level[p];
  }
  if (c.lmax - c.lmin > 30) return ORC_EINVAL;
  c.cur = (double*)calloc(f->P * c.S, sizeof(double));
  c.old = (double*)calloc(f->P * c.S, sizeof(double));
  c.snap = (double*)calloc(f->P * c.S, sizeof(double));
  c.faces = (double*)calloc(f->P * c.FS, sizeof(double));
  c.acc = (double*)calloc(f->P * c.FS, sizeof(double));
  if (!c.cur || !c.old || !c.snap || !c.faces || !c.acc) {
    free(c.cur); free(c.old); free(c.snap); free(c.faces); free(c.acc);
    return ORC_ENOMEM;
  }
  memcpy(c.cur, qpad, f->P * c.S * sizeof(double));
  orc_take_step_error();
  advance(&c, c.lmin, 0, 0);
  memcpy(qout, c.cur, f->P * c.S * sizeof(double));
  *cfl = c.cfl;
  free(c.cur); free(c.old); free(c.snap); free(c.faces); free(c.acc);
  return c.err;
}
