/* claw.c -- oracle: Clawpack-style wave-propagation patch update (TEST INFRASTRUCTURE ONLY).
 *
 * PAPER.md:168-182 [§3]: "we integrate the solution on a single uniform patch ... using the wave
 * propagation algorithm described by R. J. LeVeque and implemented in Clawpack ... At each edge,
 * we solve Riemann problems to obtain left and right going waves ... For scalar advection, the
 * speed of each wave is simply the local advection speed at the cell interface.  For non-linear
 * problems and systems, an approximate Riemann solver, such as a Roe solver ... Wave limiters are
 * used to supress spurious oscillations".  The algorithm is written from LeVeque's textbook form
 * (unsplit 2D, method = (., 2, 2)) step by step, in the order of SURVEY §8(c.5):
 *   x-sweep over rows j = 0..m+1: normal solves at edges i = 0..m+2 (edge i between cells i-1
 *   and i); for edges i = 1..m+1: CFL, limiter from the *unlimited* upwind neighbour wave,
 *   F~ = 1/2 sum_p |s|(1 - |s| dt/dx_avg) phi W, transverse splitting of
 *   L = A-dq + F~ and R = A+dq - F~ into G~ at the y-edges of cells i-1 and i;
 *   y-sweep likewise; then
 *   Q_ij -= r_ij [A+dq_{i-1/2} + A-dq_{i+1/2} + F~_{i+1/2} - F~_{i-1/2}]
 *         + s_ij [B+dq_{j-1/2} + B-dq_{j+1/2} + G~_{j+1/2} - G~_{j-1/2}],  r = dt/(kappa dx).
 * Solvers: scalar advection (constant / edge velocities with capacity), shallow-water Roe,
 * Euler Roe with the Harten-Hyman entropy fix (SURVEY §8(c.5) "Solvers"); Euler HLLE (SURVEY §8(f)
 * #4: Einfeldt's two-wave solver, LeVeque 2002 §15.3.7) with the Roe transverse solver.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"
#include "oracle_internal.h"

int orc_meqn(int kind) {
  switch (kind) {
    case ORC_ADV_CONST: case ORC_ADV_EDGEVEL_CAPA: return 1;
    case ORC_SWE_ROE: return 3;
    case ORC_EULER_ROE: case ORC_EULER_HLLE: return 4;
  }
  return 0;
}
int orc_mwaves(int kind) {
  switch (kind) {
    case ORC_ADV_CONST: case ORC_ADV_EDGEVEL_CAPA: return 1;
    case ORC_SWE_ROE: return 3;
    case ORC_EULER_ROE: return 4;
    case ORC_EULER_HLLE: return 2;
  }
  return 0;
}

static double dmin(double a, double b) { return a < b ? a : b; }
static double dmax(double a, double b) { return a > b ? a : b; }

/* wave limiters: minmod max(0, min(1, t)); MC max(0, min((1+t)/2, 2, 2t)) */
double orc_limiter(int limiter, double theta) {
  switch (limiter) {
    case ORC_LIM_MINMOD: return dmax(0.0, dmin(1.0, theta));
    case ORC_LIM_MC: return dmax(0.0, dmin(dmin((1.0 + theta) / 2.0, 2.0), 2.0 * theta));
  }
  return 1.0;
}

/* ---- Roe states ---------------------------------------------------------------------------- */
typedef struct { double u, v, H, c, c2; } roe_t;   /* u, v = velocity components 1, 2 */

static int swe_roe(double g, const double* ql, const double* qr, roe_t* R) {
  if (!(ql[0] > 0.0) || !(qr[0] > 0.0)) return ORC_EPHYS;
  double sl = sqrt(ql[0]), sr = sqrt(qr[0]);
  double ul = ql[1] / ql[0], vl = ql[2] / ql[0];
  double ur = qr[1] / qr[0], vr = qr[2] / qr[0];
  R->u = (sl * ul + sr * ur) / (sl + sr);
  R->v = (sl * vl + sr * vr) / (sl + sr);
  R->c2 = 0.5 * g * (ql[0] + qr[0]);
  R->c = sqrt(R->c2);
  R->H = 0.0;
  return ORC_OK;
}

static double euler_p(double gam, const double* q) {
  double rho = q[0], u = q[1] / rho, v = q[2] / rho;
  return (gam - 1.0) * (q[3] - 0.5 * rho * (u * u + v * v));
}

static int euler_roe(double gam, const double* ql, const double* qr, roe_t* R) {
  if (!(ql[0] > 0.0) || !(qr[0] > 0.0)) return ORC_EPHYS;
  double pl = euler_p(gam, ql), pr = euler_p(gam, qr);
  if (!(pl > 0.0) || !(pr > 0.0)) return ORC_EPHYS;
  double sl = sqrt(ql[0]), sr = sqrt(qr[0]);
  double ul = ql[1] / ql[0], vl = ql[2] / ql[0], Hl = (ql[3] + pl) / ql[0];
  double ur = qr[1] / qr[0], vr = qr[2] / qr[0], Hr = (qr[3] + pr) / qr[0];
  R->u = (sl * ul + sr * ur) / (sl + sr);
  R->v = (sl * vl + sr * vr) / (sl + sr);
  R->H = (sl * Hl + sr * Hr) / (sl + sr);
  R->c2 = (gam - 1.0) * (R->H - 0.5 * (R->u * R->u + R->v * R->v));
  if (!(R->c2 > 0.0)) return ORC_EPHYS;
  R->c = sqrt(R->c2);
  return ORC_OK;
}

/* Eigen-decomposition of a vector X for the flux Jacobian in direction `nd` (1 = x, 2 = y) at a
 * Roe state.  nd is the component index of the momentum in that direction, td the other.
 *   SWE:   b1 = ((vn+c)Xh - Xn)/(2c), b2 = Xt - vt Xh, b3 = ((c-vn)Xh + Xn)/(2c);
 *          r1 = (1, vn-c, vt), r2 = (0, 0, 1)_t, r3 = (1, vn+c, vt); speeds vn-c, vn, vn+c.
 *   Euler: b3 = Xt - vt Xrho; b2 = (gam-1)/c^2 [(H - vn^2 - vt^2)Xrho + vn Xn + vt Xt - XE];
 *          b4 = (Xn + (c - vn)Xrho - c b2)/(2c); b1 = Xrho - b2 - b4;
 *          r1 = (1, vn-c, vt, H - vn c), r2 = (1, vn, vt, (vn^2+vt^2)/2), r3 = (0, 0, 1, vt)_t,
 *          r4 = (1, vn+c, vt, H + vn c); speeds vn-c, vn, vn, vn+c.
 * (components written as (density, normal momentum, tangential momentum, energy)) */
static void eig_swe(const roe_t* R, int nd, const double* X, double b[3], double r[3][3], double lam[3]) {
  int td = 3 - nd;
  double vn = nd == 1 ? R->u : R->v, vt = nd == 1 ? R->v : R->u, c = R->c;
  b[0] = ((vn + c) * X[0] - X[nd]) / (2.0 * c);
  b[1] = X[td] - vt * X[0];
  b[2] = ((c - vn) * X[0] + X[nd]) / (2.0 * c);
  memset(r, 0, 9 * sizeof(double));
  r[0][0] = 1.0; r[0][nd] = vn - c; r[0][td] = vt;
  r[1][td] = 1.0;
  r[2][0] = 1.0; r[2][nd] = vn + c; r[2][td] = vt;
  lam[0] = vn - c; lam[1] = vn; lam[2] = vn + c;
}

static void eig_euler(double gam, const roe_t* R, int nd, const double* X, double b[4],
                      double r[4][4], double lam[4]) {
  int td = 3 - nd;
  double vn = nd == 1 ? R->u : R->v, vt = nd == 1 ? R->v : R->u, c = R->c, H = R->H;
  b[2] = X[td] - vt * X[0];
  b[1] = (gam - 1.0) / R->c2 * ((H - vn * vn - vt * vt) * X[0] + vn * X[nd] + vt * X[td] - X[3]);
  b[3] = (X[nd] + (c - vn) * X[0] - c * b[1]) / (2.0 * c);
  b[0] = X[0] - b[1] - b[3];
  memset(r, 0, 16 * sizeof(double));
  r[0][0] = 1.0; r[0][nd] = vn - c; r[0][td] = vt; r[0][3] = H - vn * c;
  r[1][0] = 1.0; r[1][nd] = vn; r[1][td] = vt; r[1][3] = 0.5 * (vn * vn + vt * vt);
  r[2][td] = 1.0; r[2][3] = vt;
  r[3][0] = 1.0; r[3][nd] = vn + c; r[3][td] = vt; r[3][3] = H + vn * c;
  lam[0] = vn - c; lam[1] = vn; lam[2] = vn; lam[3] = vn + c;
}

/* ---- Euler HLLE -------------------------------------------------------------
 * Einfeldt's HLLE solver in LeVeque's wave form (Finite Volume Methods for Hyperbolic Problems,
 * 2002, §15.3.7): two waves through one middle state Q*, with speeds
 *   s1 = min(u_l - c_l, u^ - c^),   s2 = max(u_r + c_r, u^ + c^)
 * (u^, c^ the Roe-averaged normal velocity and sound speed, u_l, c_l / u_r, c_r those of the two
 * states), and Q* fixed by conservation, s1 (Q* - Q_l) + s2 (Q_r - Q*) = f(Q_r) - f(Q_l):
 *   W1 = Q* - Q_l = (f(Q_r) - f(Q_l) - s2 (Q_r - Q_l)) / (s1 - s2),   W2 = (Q_r - Q_l) - W1,
 * A-dq = min(s1,0) W1 + min(s2,0) W2, A+dq = max(s1,0) W1 + max(s2,0) W2 (reading 25). */
static int rp_hlle(const orc_problem* pr, int ixy, const double* ql, const double* qr, double* waves,
                   double* s, double* amdq, double* apdq) {
  const double gam = pr->p0;
  const int nd = ixy;
  roe_t R;
  int rc = euler_roe(gam, ql, qr, &R);
  if (rc) return rc;
  const double un = (nd == 1) ? R.u : R.v;
  const double ul = ql[nd] / ql[0], cl = sqrt(gam * euler_p(gam, ql) / ql[0]);
  const double ur = qr[nd] / qr[0], cr = sqrt(gam * euler_p(gam, qr) / qr[0]);
  const double s1 = dmin(ul - cl, un - R.c);
  const double s2 = dmax(ur + cr, un + R.c);
  double fl[4], fr[4];
  orc_flux(pr, ixy, ql, 0.0, fl);
  orc_flux(pr, ixy, qr, 0.0, fr);
  for (int k = 0; k < 4; ++k) {
    const double dq = qr[k] - ql[k];
    const double w1 = ((fr[k] - fl[k]) - s2 * dq) / (s1 - s2);
    waves[k] = w1;
    waves[4 + k] = dq - w1;
  }
  s[0] = s1;
  s[1] = s2;
  for (int k = 0; k < 4; ++k) {
    amdq[k] = dmin(s1, 0.0) * waves[k] + dmin(s2, 0.0) * waves[4 + k];
    apdq[k] = dmax(s1, 0.0) * waves[k] + dmax(s2, 0.0) * waves[4 + k];
  }
  return ORC_OK;
}

/* ---- normal Riemann solver -------------------------------------------------------------------- */
int orc_rpn2(const orc_problem* pr, int ixy, const double* ql, const double* qr,
             const double* auxl, const double* auxr, double* waves, double* s, double* amdq,
             double* apdq) {
  const int meqn = orc_meqn(pr->kind), mw = orc_mwaves(pr->kind);
  (void)auxl;
  if (pr->kind == ORC_ADV_CONST || pr->kind == ORC_ADV_EDGEVEL_CAPA) {
    double sp;
    if (pr->kind == ORC_ADV_CONST) sp = (ixy == 1) ? pr->p0 : pr->p1;
    else sp = (ixy == 1) ? auxr[1] : auxr[2];   /* the edge velocity stored with the right cell */
    waves[0] = qr[0] - ql[0];
    s[0] = sp;
    amdq[0] = dmin(sp, 0.0) * waves[0];
    apdq[0] = dmax(sp, 0.0) * waves[0];
    return ORC_OK;
  }
  roe_t R;
  double d[4];
  for (int k = 0; k < meqn; ++k) d[k] = qr[k] - ql[k];
  if (pr->kind == ORC_SWE_ROE) {
    int rc = swe_roe(pr->p0, ql, qr, &R);
    if (rc) return rc;
    double b[3], r[3][3], lam[3];
    eig_swe(&R, ixy, d, b, r, lam);
    for (int p = 0; p < 3; ++p) {
      s[p] = lam[p];
      for (int k = 0; k < 3; ++k) waves[p * meqn + k] = b[p] * r[p][k];
    }
    for (int k = 0; k < 3; ++k) {
      amdq[k] = 0.0; apdq[k] = 0.0;
      for (int p = 0; p < 3; ++p) {
        amdq[k] += dmin(s[p], 0.0) * waves[p * meqn + k];
        apdq[k] += dmax(s[p], 0.0) * waves[p * meqn + k];
      }
    }
    return ORC_OK;
  }
  if (pr->kind == ORC_EULER_HLLE) return rp_hlle(pr, ixy, ql, qr, waves, s, amdq, apdq);
  /* Euler */
  const double gam = pr->p0;
  int rc = euler_roe(gam, ql, qr, &R);
  if (rc) return rc;
  double b[4], r[4][4], lam[4];
  eig_euler(gam, &R, ixy, d, b, r, lam);
  for (int p = 0; p < 4; ++p) {
    s[p] = lam[p];
    for (int k = 0; k < 4; ++k) waves[p * meqn + k] = b[p] * r[p][k];
  }
  if (pr->p1 == 0.0) {
    for (int k = 0; k < 4; ++k) {
      amdq[k] = 0.0; apdq[k] = 0.0;
      for (int p = 0; p < mw; ++p) {
        amdq[k] += dmin(s[p], 0.0) * waves[p * meqn + k];
        apdq[k] += dmax(s[p], 0.0) * waves[p * meqn + k];
      }
    }
    return ORC_OK;
  }
  /* Harten-Hyman entropy fix, in this fixed order */
  const int nd = ixy;
  for (int k = 0; k < 4; ++k) amdq[k] = 0.0;
  double rhol = ql[0], ul = ql[nd] / rhol, pl = euler_p(gam, ql);
  double s0 = ul - sqrt(gam * pl / rhol);                 /* lambda_1(Q_l) */
  if (!(s0 >= 0.0 && s[0] > 0.0)) {                        /* (i) fully supersonic: A-dq = 0 */
    double q1[4];
    for (int k = 0; k < 4; ++k) q1[k] = ql[k] + waves[0 * meqn + k];
    if (!(q1[0] > 0.0)) return ORC_EPHYS;
    double p1 = euler_p(gam, q1);
    if (!(p1 > 0.0)) return ORC_EPHYS;
    double s1 = q1[nd] / q1[0] - sqrt(gam * p1 / q1[0]);  /* lambda_1(Q_l + W1) */
    double beta;                                           /* (ii) */
    if (s0 < 0.0 && s1 > 0.0) beta = s0 * (s1 - s[0]) / (s1 - s0);
    else if (s[0] < 0.0) beta = s[0];
    else beta = 0.0;
    for (int k = 0; k < 4; ++k) amdq[k] = beta * waves[0 * meqn + k];
    if (s[1] < 0.0) {                                      /* (iii) */
      for (int k = 0; k < 4; ++k)
        amdq[k] += s[1] * (waves[1 * meqn + k] + waves[2 * meqn + k]);
      double q3[4];                                        /* (iv) */
      for (int k = 0; k < 4; ++k) q3[k] = qr[k] - waves[3 * meqn + k];
      if (!(q3[0] > 0.0)) return ORC_EPHYS;
      double p3 = euler_p(gam, q3), pr_ = euler_p(gam, qr);
      if (!(p3 > 0.0)) return ORC_EPHYS;
      double s2 = q3[nd] / q3[0] + sqrt(gam * p3 / q3[0]);           /* lambda_4(Q_r - W4) */
      double s3 = qr[nd] / qr[0] + sqrt(gam * pr_ / qr[0]);          /* lambda_4(Q_r) */
      double b4;
      int add = 1;
      if (s2 < 0.0 && s3 > 0.0) b4 = s2 * (s3 - s[3]) / (s3 - s2);
      else if (s[3] < 0.0) b4 = s[3];
      else { b4 = 0.0; add = 0; }
      if (add)
        for (int k = 0; k < 4; ++k) amdq[k] += b4 * waves[3 * meqn + k];
    }
  }

  for (int k = 0; k < 4; ++k) {                            /* A+dq = sum_p s W - A-dq */
    double df = 0.0;
    for (int p = 0; p < 4; ++p) df += s[p] * waves[p * meqn + k];
    apdq[k] = df - amdq[k];
  }
  return ORC_OK;
}

/* ---- transverse Riemann solver ---------------------------------------------------------------- */
int orc_rpt2(const orc_problem* pr, int ixy, const double* ql, const double* qr,
             const double* aux_recv, const double* aux_recv_next, const double* asdq,
             double* bm, double* bp) {
  const int meqn = orc_meqn(pr->kind);
  if (pr->kind == ORC_ADV_CONST) {
    double w = (ixy == 1) ? pr->p1 : pr->p0;            /* the other velocity component */
    bm[0] = dmin(w, 0.0) * asdq[0];
    bp[0] = dmax(w, 0.0) * asdq[0];
    return ORC_OK;
  }
  if (pr->kind == ORC_ADV_EDGEVEL_CAPA) {
    /* receiving cell's own low/high transverse edge velocities (v~ bottom/top for ixy = 1,
     * u~ left/right for ixy = 2) */
    int comp = (ixy == 1) ? 2 : 1;
    bm[0] = dmin(aux_recv[comp], 0.0) * asdq[0];
    bp[0] = dmax(aux_recv_next[comp], 0.0) * asdq[0];
    return ORC_OK;
  }
  const int td = (ixy == 1) ? 2 : 1;   /* transverse direction of this sweep */
  roe_t R;
  int rc = pr->kind == ORC_SWE_ROE ? swe_roe(pr->p0, ql, qr, &R) : euler_roe(pr->p0, ql, qr, &R);
  if (rc) return rc;
  if (pr->kind == ORC_SWE_ROE) {
    double b[3], r[3][3], lam[3];
    eig_swe(&R, td, asdq, b, r, lam);
    for (int k = 0; k < meqn; ++k) {
      bm[k] = 0.0; bp[k] = 0.0;
      for (int p = 0; p < 3; ++p) {
        bm[k] += dmin(lam[p], 0.0) * b[p] * r[p][k];
        bp[k] += dmax(lam[p], 0.0) * b[p] * r[p][k];
      }
    }
    return ORC_OK;
  }
  double b[4], r[4][4], lam[4];
  eig_euler(pr->p0, &R, td, asdq, b, r, lam);
  for (int k = 0; k < meqn; ++k) {
    bm[k] = 0.0; bp[k] = 0.0;
    for (int p = 0; p < 4; ++p) {
      bm[k] += dmin(lam[p], 0.0) * b[p] * r[p][k];
      bp[k] += dmax(lam[p], 0.0) * b[p] * r[p][k];
    }
  }
  return ORC_OK;
}

/* ---- physical flux ------------------------------------------------------------------------------ */
/* f(q) along axis ixy (1: x, 2: y) of the conservation law q_t + f(q)_x + g(q)_y = 0 that the
 * wave-propagation method discretises (PAPER.md:168-178 [§3]; LeVeque 2002 ch. 4, 13-14).  For the
 * advective (colour-equation) form with edge velocities the flux through an edge is the edge
 * velocity times the state ("u_e+ Q_l + u_e- Q_r + F~").  Used by the reflux. */
void orc_flux(const orc_problem* pr, int ixy, const double* q, double uedge, double* f) {
  const int nd = ixy, td = 3 - ixy;
  switch (pr->kind) {
    case ORC_ADV_CONST: f[0] = (ixy == 1 ? pr->p0 : pr->p1) * q[0]; return;
    case ORC_ADV_EDGEVEL_CAPA: f[0] = uedge * q[0]; return;
    case ORC_SWE_ROE: {
      const double un = q[nd] / q[0];
      f[0] = q[nd];
      f[nd] = q[nd] * un + 0.5 * pr->p0 * q[0] * q[0];
      f[td] = q[td] * un;
      return;
    }
    default: {
      const double p = euler_p(pr->p0, q), un = q[nd] / q[0];
      f[0] = q[nd];
      f[nd] = q[nd] * un + p;
      f[td] = q[td] * un;
      f[3] = (q[3] + p) * un;
      return;
    }
  }
}

/* ---- one patch -------------------------------------------------------------------------------- */
static int g_step_error = 0;   /* first solver error seen by orc_step_patch (physical guard) */
int orc_take_step_error(void) {
  int e = g_step_error;
  g_step_error = 0;
  return e;
}

double orc_step_patch(const orc_problem* pr, int m, int meqn, const double* qp, const double* auxp,
                      double dt, double dx, double dy, double* qnew) {
  return orc_step_patch_faces(pr, m, meqn, qp, auxp, dt, dx, dy, qnew, NULL);
}

double orc_step_patch_faces(const orc_problem* pr, int m, int meqn, const double* qp, const double* auxp,
                            double dt, double dx, double dy, double* qnew, double* face) {
  const int n = ORC_N(m), nn = n * n, mw = orc_mwaves(pr->kind);
  const size_t A = (size_t)meqn * nn;
  double* amx = (double*)calloc(6 * A, sizeof(double));
  double *apx = amx + A, *fx = apx + A, *amy = fx + A, *apy = amy + A, *gy = apy + A;
  double* wave = (double*)malloc((size_t)n * mw * meqn * sizeof(double));
  double* spd = (double*)malloc((size_t)n * mw * sizeof(double));
  double one_aux[3] = {1.0, 0.0, 0.0};
  double cfl = 0.0;
#define Q(k, i, j) qp[(size_t)(k) * nn + ORC_IDX(m, i, j)]
#define E(arr, k, i, j) arr[(size_t)(k) * nn + ORC_IDX(m, i, j)]
#define AUXP(i, j, tmp) (auxp ? (tmp[0] = auxp[ORC_IDX(m, i, j)], tmp[1] = auxp[nn + ORC_IDX(m, i, j)], \
                                 tmp[2] = auxp[2 * nn + ORC_IDX(m, i, j)], tmp) : one_aux)
#define KAPPA(i, j) (auxp ? auxp[ORC_IDX(m, i, j)] : 1.0)
  double ql[4], qr[4], amdq[4], apdq[4], Ft[4], L[4], R[4], bm[4], bp[4];
  double ta[3], tb[3];
  /* x-sweep */
  for (int j = 0; j <= m + 1; ++j) {
    for (int i = 0; i <= m + 2; ++i) {
      for (int k = 0; k < meqn; ++k) { ql[k] = Q(k, i - 1, j); qr[k] = Q(k, i, j); }
      const double* al = AUXP(i - 1, j, ta);
      const double* ar = AUXP(i, j, tb);
      int rc = orc_rpn2(pr, 1, ql, qr, al, ar, wave + (size_t)i * mw * meqn, spd + (size_t)i * mw, amdq, apdq);
      if (rc && !g_step_error) g_step_error = rc;
      for (int k = 0; k < meqn; ++k) { E(amx, k, i, j) = amdq[k]; E(apx, k, i, j) = apdq[k]; }
    }
    for (int i = 1; i <= m + 1; ++i) {
      const double rl = dt / (KAPPA(i - 1, j) * dx), rr = dt / (KAPPA(i, j) * dx);
      const double* W = wave + (size_t)i * mw * meqn;
      const double* S = spd + (size_t)i * mw;
      for (int p = 0; p < mw; ++p) cfl = dmax(cfl, dmax(rr * S[p], -rl * S[p]));
      for (int k = 0; k < meqn; ++k) Ft[k] = 0.0;
      if (pr->method2 == 2) {
        const double rav = 0.5 * (rl + rr);
        for (int p = 0; p < mw; ++p) {
          double wn2 = 0.0;
          for (int k = 0; k < meqn; ++k) wn2 += W[p * meqn + k] * W[p * meqn + k];
          if (wn2 == 0.0) continue;
          int I = (S[p] > 0.0) ? i - 1 : i + 1;
          const double* WI = wave + (size_t)I * mw * meqn;
          double dot = 0.0;
          for (int k = 0; k < meqn; ++k) dot += WI[p * meqn + k] * W[p * meqn + k];
          double phi = orc_limiter(pr->limiter, dot / wn2);
          double as = fabs(S[p]);
          for (int k = 0; k < meqn; ++k) {
            double wl = phi * W[p * meqn + k];
            Ft[k] += 0.5 * as * (1.0 - as * rav) * wl;
          }
        }
      }
      for (int k = 0; k < meqn; ++k) E(fx, k, i, j) += Ft[k];
      if (pr->method3 >= 1) {
        for (int k = 0; k < meqn; ++k) {
          ql[k] = Q(k, i - 1, j); qr[k] = Q(k, i, j);
          L[k] = E(amx, k, i, j) + (pr->method3 == 2 ? Ft[k] : 0.0);
          R[k] = E(apx, k, i, j) - (pr->method3 == 2 ? Ft[k] : 0.0);
        }
        int rc = orc_rpt2(pr, 1, ql, qr, AUXP(i - 1, j, ta), AUXP(i - 1, j + 1, tb), L, bm, bp);
        if (rc && !g_step_error) g_step_error = rc;
        for (int k = 0; k < meqn; ++k) {
          E(gy, k, i - 1, j) -= 0.5 * rl * bm[k];
          E(gy, k, i - 1, j + 1) -= 0.5 * rl * bp[k];
        }
        rc = orc_rpt2(pr, 1, ql, qr, AUXP(i, j, ta), AUXP(i, j + 1, tb), R, bm, bp);
        if (rc && !g_step_error) g_step_error = rc;
        for (int k = 0; k < meqn; ++k) {
          E(gy, k, i, j) -= 0.5 * rr * bm[k];
          E(gy, k, i, j + 1) -= 0.5 * rr * bp[k];
        }
      }
    }
  }
  /* y-sweep */
  for (int i = 0; i <= m + 1; ++i) {
    for (int j = 0; j <= m + 2; ++j) {
      for (int k = 0; k < meqn; ++k) { ql[k] = Q(k, i, j - 1); qr[k] = Q(k, i, j); }
      const double* al = AUXP(i, j - 1, ta);
      const double* ar = AUXP(i, j, tb);
      int rc = orc_rpn2(pr, 2, ql, qr, al, ar, wave + (size_t)j * mw * meqn, spd + (size_t)j * mw, amdq, apdq);
      if (rc && !g_step_error) g_step_error = rc;
      for (int k = 0; k < meqn; ++k) { E(amy, k, i, j) = amdq[k]; E(apy, k, i, j) = apdq[k]; }
    }
    for (int j = 1; j <= m + 1; ++j) {
      const double sl = dt / (KAPPA(i, j - 1) * dy), sr = dt / (KAPPA(i, j) * dy);
      const double* W = wave + (size_t)j * mw * meqn;
      const double* S = spd + (size_t)j * mw;
      for (int p = 0; p < mw; ++p) cfl = dmax(cfl, dmax(sr * S[p], -sl * S[p]));
      for (int k = 0; k < meqn; ++k) Ft[k] = 0.0;
      if (pr->method2 == 2) {
        const double sav = 0.5 * (sl + sr);
        for (int p = 0; p < mw; ++p) {
          double wn2 = 0.0;
          for (int k = 0; k < meqn; ++k) wn2 += W[p * meqn + k] * W[p * meqn + k];
          if (wn2 == 0.0) continue;
          int J = (S[p] > 0.0) ? j - 1 : j + 1;
          const double* WJ = wave + (size_t)J * mw * meqn;
          double dot = 0.0;
          for (int k = 0; k < meqn; ++k) dot += WJ[p * meqn + k] * W[p * meqn + k];
          double phi = orc_limiter(pr->limiter, dot / wn2);
          double as = fabs(S[p]);
          for (int k = 0; k < meqn; ++k) {
            double wl = phi * W[p * meqn + k];
            Ft[k] += 0.5 * as * (1.0 - as * sav) * wl;
          }
        }
      }
      for (int k = 0; k < meqn; ++k) E(gy, k, i, j) += Ft[k];
      if (pr->method3 >= 1) {
        for (int k = 0; k < meqn; ++k) {
          ql[k] = Q(k, i, j - 1); qr[k] = Q(k, i, j);
          L[k] = E(amy, k, i, j) + (pr->method3 == 2 ? Ft[k] : 0.0);
          R[k] = E(apy, k, i, j) - (pr->method3 == 2 ? Ft[k] : 0.0);
        }
        int rc = orc_rpt2(pr, 2, ql, qr, AUXP(i, j - 1, ta), AUXP(i + 1, j - 1, tb), L, bm, bp);
        if (rc && !g_step_error) g_step_error = rc;
        for (int k = 0; k < meqn; ++k) {
          E(fx, k, i, j - 1) -= 0.5 * sl * bm[k];
          E(fx, k, i + 1, j - 1) -= 0.5 * sl * bp[k];
        }
        rc = orc_rpt2(pr, 2, ql, qr, AUXP(i, j, ta), AUXP(i + 1, j, tb), R, bm, bp);
        if (rc && !g_step_error) g_step_error = rc;
        for (int k = 0; k < meqn; ++k) {
          E(fx, k, i, j) -= 0.5 * sr * bm[k];
          E(fx, k, i + 1, j) -= 0.5 * sr * bp[k];
        }
      }
    }
  }
  /* update */
  for (int k = 0; k < meqn; ++k)
    for (int j = 1; j <= m; ++j)
      for (int i = 1; i <= m; ++i) {
        const double r = dt / (KAPPA(i, j) * dx), s = dt / (KAPPA(i, j) * dy);
        double a = E(apx, k, i, j) + E(amx, k, i + 1, j) + E(fx, k, i + 1, j) - E(fx, k, i, j);
        double b = E(apy, k, i, j) + E(amy, k, i, j + 1) + E(gy, k, i, j + 1) - E(gy, k, i, j);
        qnew[(size_t)k * nn + ORC_IDX(m, i, j)] = Q(k, i, j) - r * a - s * b;
      }
  /* face fluxes for the coarse/fine reflux, per face (0: -x, 1: +x, 2: -y,
   * 3: +y) and boundary edge, in outward form: the total flux the update applied through the
   * edge, F = f(Q_l) + A-dq + F~ = f(Q_r) - A+dq + F~ (F~ including the other sweep's transverse
   * terms), signed along the face's outward normal.  With Q_own the adjacent interior cell:
   *   high faces (+x, +y):  out = f(Q_own) + A-dq + F~;   low faces (-x, -y):  out = A+dq - F~ - f(Q_own). */
  if (face) {
    double fq[4], tmp[3];
    for (int e = 0; e < m; ++e) {
      const int c = e + 1;
      double* o0 = face + ((size_t)0 * m + e) * meqn;
      double* o1 = face + ((size_t)1 * m + e) * meqn;
      double* o2 = face + ((size_t)2 * m + e) * meqn;
      double* o3 = face + ((size_t)3 * m + e) * meqn;
      double ql_[4], qh_[4];
      for (int k = 0; k < meqn; ++k) { ql_[k] = Q(k, 1, c); qh_[k] = Q(k, m, c); }
      orc_flux(pr, 1, ql_, AUXP(1, c, tmp)[1], fq);
      for (int k = 0; k < meqn; ++k) o0[k] = (E(apx, k, 1, c) - E(fx, k, 1, c)) - fq[k];
      orc_flux(pr, 1, qh_, AUXP(m + 1, c, tmp)[1], fq);
      for (int k = 0; k < meqn; ++k) o1[k] = fq[k] + (E(amx, k, m + 1, c) + E(fx, k, m + 1, c));
      for (int k = 0; k < meqn; ++k) { ql_[k] = Q(k, c, 1); qh_[k] = Q(k, c, m); }
      orc_flux(pr, 2, ql_, AUXP(c, 1, tmp)[2], fq);
      for (int k = 0; k < meqn; ++k) o2[k] = (E(apy, k, c, 1) - E(gy, k, c, 1)) - fq[k];
      orc_flux(pr, 2, qh_, AUXP(c, m + 1, tmp)[2], fq);
      for (int k = 0; k < meqn; ++k) o3[k] = fq[k] + (E(amy, k, c, m + 1) + E(gy, k, c, m + 1));
    }
  }
#undef Q
#undef E
#undef AUXP
#undef KAPPA
  free(amx); free(wave); free(spd);
  return cfl;
}

/* ---- whole forest ---------------------------------------------------------------------------- */
int orc_step(const orc_forest* f, const orc_problem* pr, double* qpad, const double* aux,
             double dt, double dx0, double* qout, double* cfl_out, int nthreads) {
  const int m = f->m, meqn = orc_meqn(pr->kind);
  const size_t S = (size_t)meqn * ORC_N(m) * ORC_N(m), SA = (size_t)3 * ORC_N(m) * ORC_N(m);
  int rc = orc_ghost_fill(f, qpad, meqn);
  if (rc) return rc;
  g_step_error = 0;
  double cfl = 0.0;
  (void)nthreads;
  double* faces = NULL;
  const size_t FS = (size_t)4 * m * meqn;
  if (pr->reflux) {
    faces = (double*)malloc((size_t)f->P * FS * sizeof(double));
    if (!faces) return ORC_ENOMEM;
  }
#ifdef _OPENMP
#pragma omp parallel for schedule(static) reduction(max : cfl) num_threads(nthreads > 0 ? nthreads : 1)
#endif
  for (int64_t p = 0; p < f->P; ++p) {
    double h = ldexp(dx0, -f->level[p]);
    double c = orc_step_patch_faces(pr, m, meqn, qpad + p * S, aux ? aux + p * SA : NULL, dt, h, h,
                                    qout + p * S, faces ? faces + p * FS : NULL);
    if (c > cfl || c != c) cfl = c;
  }
  *cfl_out = cfl;
  if (faces) {
    int rr = g_step_error ? g_step_error : orc_reflux(f, pr, faces, aux, dt, dx0, qout);
    free(faces);
    return rr;
  }
  return g_step_error;
}

int orc_build_padded_sample(const orc_forest* f, const double* q, int meqn, int64_t p, double* out);

int orc_step_sample(const orc_forest* f, const orc_problem* pr, const double* q,
                    const double* aux, double dt, double dx0, const int64_t* ids, int64_t ns,
                    double* out, double* cfl_out) {
  const int m = f->m, n = ORC_N(m), meqn = orc_meqn(pr->kind);
  const size_t S = (size_t)meqn * n * n, SA = (size_t)3 * n * n;
  double* pad = (double*)malloc(2 * S * sizeof(double));
  if (!pad) return ORC_ENOMEM;
  g_step_error = 0;
  for (int64_t s = 0; s < ns; ++s) {
    int64_t p = ids[s];
    if (p < 0 || p >= f->P) { free(pad); return ORC_EINVAL; }
    int rc = orc_build_padded_sample(f, q, meqn, p, pad);
    if (rc) { free(pad); return rc; }
    double h = ldexp(dx0, -f->level[p]);
    cfl_out[s] = orc_step_patch(pr, m, meqn, pad, aux ? aux + p * SA : NULL, dt, h, h, pad + S);
    for (int k = 0; k < meqn; ++k)
      for (int j = 1; j <= m; ++j)
        for (int i = 1; i <= m; ++i)
          out[(((size_t)s * meqn + k) * m + (j - 1)) * m + (i - 1)] =
              pad[S + (size_t)k * n * n + ORC_IDX(m, i, j)];
  }
  free(pad);
  return g_step_error;
}
