// solvers.cuh -- device Riemann solvers for the fused step kernel (libfc, sm_100a, fp64).
//
// PAPER.md:171-180 [§3]: "At each edge, we solve Riemann problems to obtain left and right going
// waves propagating at speeds determined from the solution to the Riemann problem.  For scalar
// advection, the speed of each wave is simply the local advection speed at the cell interface.
// For non-linear problems and systems, an approximate Riemann solver, such as a Roe solver ...".
//
// Interface used by k_step (step.cu):
//   NC          per-cell derived fields precomputed once per staged cell (shared by the 4 edges
//               of the cell in both sweeps): Euler {sqrt(rho), u, v, H, c}; SWE {sqrt(h), u, v}
//   NS          per-edge scratch written by the normal solve (phase 1) and read in phase 2
//               (NSA >= NS allocated: slots PB..PB+MEQN-1 receive the edge's L part in phase 2):
//               AdvConst / AdvEdgeCapa {dq}; SweRoe {a1..a3, u, v, c, 1/c};
//               EulerRoe {a1..a4, u, v, H, c, 1/c, A-dq (Harten-Hyman fixed)} (A+dq = sum s W - A-dq)
//   riemann<D>  normal solve on one edge (D = 1: x, normal momentum = component 1; D = 2: y)
//   wave<D>     wave p of an edge from its scratch;  speed<D>, fluct<D>, transverse<D>
// Divisions and square roots use the SFU approximations refined by Newton steps to ~1 ulp
// (fast_rcp / fast_rsqrt): results agree with the oracle's IEEE-rounded operations to rounding
// level (tolerance 1e-12 max|q|), not bitwise.
#pragma once
#include <cuda_runtime.h>

namespace fc {

struct SolverParams {
  double p0, p1;  // (u, v) | - | (g, -) | (gamma, efix)
};

// cell aux view: kappa, u~ (left edge), v~ (bottom edge) of one cell (smem window, stride WW)
struct AuxCell {
  const double* a;
  int WW;
  __device__ double kappa() const { return a[0]; }
  __device__ double ut() const { return a[WW]; }
  __device__ double vt() const { return a[2 * WW]; }
};

__device__ __forceinline__ double dmin0(double s) { return s < 0.0 ? s : 0.0; }
__device__ __forceinline__ double dmax0(double s) { return s > 0.0 ? s : 0.0; }
// (min(s,0), max(s,0)) with one compare: the negative part is s - max(s,0), exact
__device__ __forceinline__ void split0(double s, double& sm, double& sp) {
  sp = s > 0.0 ? s : 0.0;
  sm = s - sp;
}

// 1/x: SFU seed y0 (MUFU.RCP64H, relative error e ~ 2^-22) + one third-order step:
// with e = 1 - x y0, 1/x = y0 / (1 - e) = y0 (1 + e + e^2) + O(e^3 ~ 2^-66) -> ~1 ulp (x normal,
// nonzero); 3 DFMA (two Newton steps took 4)
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}

// 1/sqrt(x): SFU seed y0 + one third-order step: with e = 1 - x y0^2,
// 1/sqrt(x) = y0 (1 - e)^(-1/2) = y0 (1 + e/2 + 3 e^2/8) + O(5 e^3/16 ~ 2^-67) -> ~1 ulp (x > 0
// normal); 5 fp64 ops (two Newton steps took 7)
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);
  return fma(y, e * fma(0.375, e, 0.5), y);
}

// ----------------------------------------------------------------------------------------------
// CFL of a tile whose staged window holds one uniform state q (component stride qs): the max over
// the tile's edges of max(r s, -r s) over the waves, which for a uniform state is r (|u_n| + c).
// Block-uniform result (every thread returns the same value, or its share for AdvEdgeCapa).
struct AdvConst {
  static constexpr int MEQN = 1, MW = 1, NS = 1, NC = 0, PB = NS, NSA = PB + MEQN;
  static constexpr bool CAPA = false, AM_STORED = false;
  __device__ static double quiescent_cfl(const double*, int, const SolverParams& P, const double*, double dtdx,
                                         int, int, int, int) {
    return dtdx * fmax(fabs(P.p0), fabs(P.p1));
  }
  // physical flux along axis D (coarse/fine reflux records)
  template <int D>
  __device__ static void flux(const double* q, int, double, const SolverParams& P, double* f) {
    f[0] = (D == 1 ? P.p0 : P.p1) * q[0];
  }
  __device__ static void precompute(const double*, int, const SolverParams&, double*, int) {}
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, const double*, const double*,
                                 int, AuxCell, AuxCell, const SolverParams&, double* sc, int) {
    sc[0] = qr[0] - ql[0];
  }
  template <int D>
  __device__ static double speed(const double*, int, int, const SolverParams& P, AuxCell) {
    return D == 1 ? P.p0 : P.p1;
  }
  template <int D>
  __device__ static void wave(const double* sc, int, int, const SolverParams&, double* W) {
    W[0] = sc[0];
  }
  template <int D>
  __device__ static void fluct(const double* sc, int st, const SolverParams& P, AuxCell ar,
                               double* am, double* ap) {
    const double s = speed<D>(sc, st, 0, P, ar);
    am[0] = dmin0(s) * sc[0];
    ap[0] = dmax0(s) * sc[0];
  }
  template <int D>
  __device__ static void transverse(const double*, int, const SolverParams& P, const double* X,
                                    AuxCell, AuxCell, double* bm, double* bp) {
    const double w = D == 1 ? P.p1 : P.p0;
    bm[0] = dmin0(w) * X[0];
    bp[0] = dmax0(w) * X[0];
  }
};

// ----------------------------------------------------------------------------------------------
struct AdvEdgeCapa {
  static constexpr int MEQN = 1, MW = 1, NS = 1, NC = 0, PB = NS, NSA = PB + MEQN;
  static constexpr bool CAPA = true, AM_STORED = false;
  // edge velocities vary per edge: each thread scans a share of the tile's x- and y-edges
  __device__ static double quiescent_cfl(const double*, int WW, const SolverParams&, const double* sa,
                                         double dtdx, int T, int W, int tid, int NT) {
    double c = 0.0;
    for (int e = tid; e < (T + 1) * (T + 2); e += NT) {
      const int i = 1 + e % (T + 1), j = e / (T + 1);          // x-edge i of row j
      const int r = (j + 1) * W + (i + 1);
      const double s = sa[WW + r];
      c = fmax(c, fmax(dtdx / sa[r] * s, -dtdx / sa[r - 1] * s));
      const int ii = e % (T + 2), jj = 1 + e / (T + 2);          // y-edge jj of column ii
      const int rr = (jj + 1) * W + (ii + 1);
      const double sy = sa[2 * WW + rr];
      c = fmax(c, fmax(dtdx / sa[rr] * sy, -dtdx / sa[rr - W] * sy));
    }
    return c;
  }
  // advective form: the flux through an edge is its normal velocity times the state
  template <int D>
  __device__ static void flux(const double* q, int, double uedge, const SolverParams&, double* f) {
    f[0] = uedge * q[0];
  }
  __device__ static void precompute(const double*, int, const SolverParams&, double*, int) {}
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, const double*, const double*,
                                 int, AuxCell, AuxCell, const SolverParams&, double* sc, int) {
    sc[0] = qr[0] - ql[0];
  }
  // the edge velocity is stored with the cell to the right of / above the edge
  template <int D>
  __device__ static double speed(const double*, int, int, const SolverParams&, AuxCell ar) {
    return D == 1 ? ar.ut() : ar.vt();
  }
  template <int D>
  __device__ static void wave(const double* sc, int, int, const SolverParams&, double* W) {
    W[0] = sc[0];
  }
  template <int D>
  __device__ static void fluct(const double* sc, int st, const SolverParams& P, AuxCell ar,
                               double* am, double* ap) {
    const double s = speed<D>(sc, st, 0, P, ar);
    am[0] = dmin0(s) * sc[0];
    ap[0] = dmax0(s) * sc[0];
  }
  // receiving cell's own low / high transverse edge velocities (reading 3)
  template <int D>
  __device__ static void transverse(const double*, int, const SolverParams&, const double* X,
                                    AuxCell recv, AuxCell next, double* bm, double* bp) {
    const double lo = D == 1 ? recv.vt() : recv.ut();
    const double hi = D == 1 ? next.vt() : next.ut();
    bm[0] = dmin0(lo) * X[0];
    bp[0] = dmax0(hi) * X[0];
  }
};

// ----------------------------------------------------------------------------------------------
// Shallow water, Roe linearisation: ubar, vbar = sqrt(h)-weighted, cbar = sqrt(g (hl + hr) / 2);
// a1 = ((u+c) dh - dn)/(2c), a2 = dt - vt dh, a3 = ((c-u) dh + dn)/(2c); r1 = (1, u-c, v),
// r2 = (0, 0, 1)_t, r3 = (1, u+c, v); speeds u-c, u, u+c (normal/tangential per direction).
struct SweRoe {
  static constexpr int MEQN = 3, MW = 3, NS = 7, NC = 3, PB = NS, NSA = PB + MEQN;
  static constexpr bool CAPA = false, AM_STORED = false;
  __device__ static double quiescent_cfl(const double* q, int qs, const SolverParams& P, const double*,
                                         double dtdx, int, int, int, int) {
    const double h = q[0], ih = 1.0 / h;
    const double c = sqrt(P.p0 * h);
    return dtdx * (fmax(fabs(q[qs] * ih), fabs(q[2 * qs] * ih)) + c);
  }
  template <int D>
  __device__ static void flux(const double* q, int qs, double, const SolverParams& P, double* f) {
    constexpr int nd = D, td = 3 - D;
    const double un = q[nd * qs] / q[0];
    f[0] = q[nd * qs];
    f[nd] = q[nd * qs] * un + 0.5 * P.p0 * q[0] * q[0];
    f[td] = q[td * qs] * un;
  }
  // cell fields: sqrt(h), u, v
  __device__ static void precompute(const double* q, int qs, const SolverParams&, double* c, int cs) {
    const double h = q[0];
    const double rs = fast_rsqrt(h);
    const double ih = rs * rs;
    c[0] = h * rs;
    c[cs] = q[qs] * ih;
    c[2 * cs] = q[2 * qs] * ih;
  }
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, const double* cl, const double* cr,
                                 int cs, AuxCell, AuxCell, const SolverParams& P, double* sc, int st) {
    constexpr int nd = D, td = 3 - D;
    const double wl = cl[0], wr = cr[0];
    const double inv = fast_rcp(wl + wr);
    const double al = wl * inv, ar = wr * inv;
    const double u = al * cl[cs] + ar * cr[cs];
    const double v = al * cl[2 * cs] + ar * cr[2 * cs];
    const double c2 = 0.5 * P.p0 * (ql[0] + qr[0]);
    const double ic = fast_rsqrt(c2);
    const double c = c2 * ic;
    const double un = nd == 1 ? u : v, ut = nd == 1 ? v : u;
    const double dh = qr[0] - ql[0], dn = qr[nd] - ql[nd], dtg = qr[td] - ql[td];
    const double i2c = 0.5 * ic;
    sc[0] = ((un + c) * dh - dn) * i2c;
    sc[st] = dtg - ut * dh;
    sc[2 * st] = ((c - un) * dh + dn) * i2c;
    sc[3 * st] = u;
    sc[4 * st] = v;
    sc[5 * st] = c;
    sc[6 * st] = ic;
  }
  template <int D>
  __device__ static double speed(const double* sc, int st, int p, const SolverParams&, AuxCell) {
    const double un = D == 1 ? sc[3 * st] : sc[4 * st], c = sc[5 * st];
    return p == 0 ? un - c : (p == 1 ? un : un + c);
  }
  template <int D>
  __device__ static void wave(const double* sc, int st, int p, const SolverParams&, double* W) {
    constexpr int nd = D, td = 3 - D;
    const double u = sc[3 * st], v = sc[4 * st], c = sc[5 * st];
    const double un = nd == 1 ? u : v, ut = nd == 1 ? v : u;
    const double a = sc[p * st];
    if (p == 1) { W[0] = 0.0; W[nd] = 0.0; W[td] = a; return; }
    W[0] = a;
    W[nd] = a * (p == 0 ? un - c : un + c);
    W[td] = a * ut;
  }
  template <int D>
  __device__ static void fluct(const double* sc, int st, const SolverParams& P, AuxCell ar,
                               double* am, double* ap) {
    am[0] = am[1] = am[2] = 0.0;
    ap[0] = ap[1] = ap[2] = 0.0;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      double W[3];
      wave<D>(sc, st, p, P, W);
      const double s = speed<D>(sc, st, p, P, ar);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        am[k] += dmin0(s) * W[k];
        ap[k] += dmax0(s) * W[k];
      }
    }
  }
  template <int D>
  __device__ static void transverse(const double* sc, int st, const SolverParams&, const double* X,
                                    AuxCell, AuxCell, double* bm, double* bp) {
    constexpr int nd = 3 - D, td = D;   // eigen-decomposition along the transverse direction
    const double u = sc[3 * st], v = sc[4 * st], c = sc[5 * st], ic = sc[6 * st];
    const double vn = nd == 1 ? u : v, vt = nd == 1 ? v : u;
    const double i2c = 0.5 * ic;
    const double b1 = ((vn + c) * X[0] - X[nd]) * i2c;
    const double b2 = X[td] - vt * X[0];
    const double b3 = ((c - vn) * X[0] + X[nd]) * i2c;
    double l1m, l1p, l2m, l2p, l3m, l3p;
    split0(vn - c, l1m, l1p);
    split0(vn, l2m, l2p);
    split0(vn + c, l3m, l3p);
    const double m1 = l1m * b1, m2 = l2m * b2, m3 = l3m * b3;
    const double p1 = l1p * b1, p2 = l2p * b2, p3 = l3p * b3;
    bm[0] = m1 + m3;
    bm[nd] = m1 * (vn - c) + m3 * (vn + c);
    bm[td] = (m1 + m3) * vt + m2;
    bp[0] = p1 + p3;
    bp[nd] = p1 * (vn - c) + p3 * (vn + c);
    bp[td] = (p1 + p3) * vt + p2;
  }
};

// ----------------------------------------------------------------------------------------------
// Euler, Roe linearisation with the Harten-Hyman entropy fix:
// a3 = d(mt) - vt drho; a2 = (g-1)/c^2 [(H - un^2 - vt^2) drho + un d(mn) + vt d(mt) - dE];
// a4 = (d(mn) + (c - un) drho - c a2)/(2c); a1 = drho - a2 - a4;
// r1 = (1, un-c, vt, H - un c), r2 = (1, un, vt, (un^2+vt^2)/2), r3 = (0, 0, 1, vt)_t,
// r4 = (1, un+c, vt, H + un c); speeds un-c, un, un, un+c.
struct EulerRoe {
  // PB: the edge's L part (A-dq + F~) overwrites its A-dq slots once they are consumed
  static constexpr int MEQN = 4, MW = 4, NS = 13, NC = 5, PB = 9, NSA = NS;
  static constexpr bool CAPA = false, AM_STORED = true;
  __device__ static double quiescent_cfl(const double* q, int qs, const SolverParams& P, const double*,
                                         double dtdx, int, int, int, int) {
    const double rho = q[0], ir = 1.0 / rho;
    const double u = q[qs] * ir, v = q[2 * qs] * ir;
    const double p = (P.p0 - 1.0) * (q[3 * qs] - 0.5 * rho * (u * u + v * v));
    const double c = sqrt(P.p0 * p * ir);
    return dtdx * (fmax(fabs(u), fabs(v)) + c);
  }
  template <int D>
  __device__ static void flux(const double* q, int qs, double, const SolverParams& P, double* f) {
    constexpr int nd = D, td = 3 - D;
    const double rho = q[0], mx = q[qs], my = q[2 * qs], E = q[3 * qs];
    const double p = (P.p0 - 1.0) * (E - 0.5 * (mx * mx + my * my) / rho);
    const double un = q[nd * qs] / rho;
    f[0] = q[nd * qs];
    f[nd] = q[nd * qs] * un + p;
    f[td] = q[td * qs] * un;
    f[3] = (E + p) * un;
  }
  // cell fields: sqrt(rho), u, v, H, c
  __device__ static void precompute(const double* q, int qs, const SolverParams& P, double* c, int cs) {
    const double gam = P.p0, gm1 = gam - 1.0;
    const double rho = q[0];
    const double rs = fast_rsqrt(rho);
    const double ir = rs * rs;
    const double u = q[qs] * ir, v = q[2 * qs] * ir;
    const double p = gm1 * (q[3 * qs] - 0.5 * rho * (u * u + v * v));
    c[0] = rho * rs;
    c[cs] = u;
    c[2 * cs] = v;
    c[3 * cs] = (q[3 * qs] + p) * ir;
    const double c2 = gam * p * ir;
    c[4 * cs] = c2 * fast_rsqrt(c2);
  }
  // sign test of lambda = m/rho -+ c at a conserved state without divisions:
  // (m/rho)^2 > c^2  <=>  m^2 > gam (gam-1) (E rho - (m^2 + t^2)/2)   (rho > 0)
  __device__ static bool supersonic(double rho, double mn, double mt, double E, double gam) {
    return mn * mn > gam * (gam - 1.0) * (E * rho - 0.5 * (mn * mn + mt * mt));
  }
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, const double* cl, const double* cr,
                                 int cs, AuxCell, AuxCell, const SolverParams& P, double* sc, int st) {
    constexpr int nd = D, td = 3 - D;
    const double gam = P.p0, gm1 = gam - 1.0;
    const double wl = cl[0], wr = cr[0];
    const double inv = fast_rcp(wl + wr);
    const double al = wl * inv, ar = wr * inv;
    const double u = al * cl[cs] + ar * cr[cs];
    const double v = al * cl[2 * cs] + ar * cr[2 * cs];
    const double H = al * cl[3 * cs] + ar * cr[3 * cs];
    const double c2 = gm1 * (H - 0.5 * (u * u + v * v));
    const double ic = fast_rsqrt(c2);
    const double c = c2 * ic;
    const double un = nd == 1 ? u : v, vt = nd == 1 ? v : u;
    double d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = qr[k] - ql[k];
    const double a3 = d[td] - vt * d[0];
    const double a2 = gm1 * (ic * ic) * ((H - un * un - vt * vt) * d[0] + un * d[nd] + vt * d[td] - d[3]);
    const double a4 = (d[nd] + (c - un) * d[0] - c * a2) * (0.5 * ic);
    const double a1 = d[0] - a2 - a4;
    sc[0] = a1; sc[st] = a2; sc[2 * st] = a3; sc[3 * st] = a4;
    sc[4 * st] = u; sc[5 * st] = v; sc[6 * st] = H; sc[7 * st] = c; sc[8 * st] = ic;
    // waves 1 and 4 (2 and 3 move with un)
    double W1[4], W4[4], W23[4];
    W1[0] = a1; W1[nd] = a1 * (un - c); W1[td] = a1 * vt; W1[3] = a1 * (H - un * c);
    W4[0] = a4; W4[nd] = a4 * (un + c); W4[td] = a4 * vt; W4[3] = a4 * (H + un * c);
    W23[0] = a2; W23[nd] = a2 * un; W23[td] = a2 * vt + a3;
    W23[3] = a2 * 0.5 * (un * un + vt * vt) + a3 * vt;
    const double s1 = un - c, s2 = un, s4 = un + c;
    double am[4];
    if (P.p1 == 0.0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) am[k] = dmin0(s1) * W1[k] + dmin0(s2) * W23[k] + dmin0(s4) * W4[k];
    } else {
      // Harten-Hyman; transonic tests are division-free sign tests,
      // the exact eigenvalues are only formed in the (rare) transonic case
      const double s0 = (nd == 1 ? cl[cs] : cl[2 * cs]) - cl[4 * cs];      // lambda_1(Q_l)
#pragma unroll
      for (int k = 0; k < 4; ++k) am[k] = 0.0;
      if (!(s0 >= 0.0 && s1 > 0.0)) {
        double beta = s1 < 0.0 ? s1 : 0.0;
        if (s0 < 0.0) {
          double q1[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) q1[k] = ql[k] + W1[k];
          // lambda_1(Q_l + W1) > 0  <=>  q1n > 0 and supersonic
          if (q1[nd] > 0.0 && supersonic(q1[0], q1[nd], q1[td], q1[3], gam)) {
            const double ir = fast_rcp(q1[0]);
            const double un1 = q1[nd] * ir, ut1 = q1[td] * ir;
            const double p1 = gm1 * (q1[3] - 0.5 * q1[0] * (un1 * un1 + ut1 * ut1));
            const double cc = gam * p1 * ir;
            const double lr = un1 - cc * fast_rsqrt(cc);
            beta = s0 * (lr - s1) * fast_rcp(lr - s0);
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) am[k] = beta * W1[k];
        if (s2 < 0.0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) am[k] += s2 * W23[k];
          const double s4r = (nd == 1 ? cr[cs] : cr[2 * cs]) + cr[4 * cs];  // lambda_4(Q_r)
          double b4 = s4 < 0.0 ? s4 : 0.0;
          if (s4r > 0.0) {
            double q3[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) q3[k] = qr[k] - W4[k];
            // lambda_4(Q_r - W4) < 0  <=>  q3n < 0 and supersonic
            if (q3[nd] < 0.0 && supersonic(q3[0], q3[nd], q3[td], q3[3], gam)) {
              const double ir = fast_rcp(q3[0]);
              const double un3 = q3[nd] * ir, ut3 = q3[td] * ir;
              const double p3 = gm1 * (q3[3] - 0.5 * q3[0] * (un3 * un3 + ut3 * ut3));
              const double cc = gam * p3 * ir;
              const double ll = un3 + cc * fast_rsqrt(cc);
              b4 = ll * (s4r - s4) * fast_rcp(s4r - ll);
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) am[k] += b4 * W4[k];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) sc[(9 + k) * st] = am[k];
  }
  template <int D>
  __device__ static double speed(const double* sc, int st, int p, const SolverParams&, AuxCell) {
    const double un = D == 1 ? sc[4 * st] : sc[5 * st], c = sc[7 * st];
    return p == 0 ? un - c : (p == 3 ? un + c : un);
  }
  template <int D>
  __device__ static void wave(const double* sc, int st, int p, const SolverParams&, double* W) {
    constexpr int nd = D, td = 3 - D;
    const double u = sc[4 * st], v = sc[5 * st], H = sc[6 * st], c = sc[7 * st];
    const double un = nd == 1 ? u : v, vt = nd == 1 ? v : u;
    const double a = sc[p * st];
    if (p == 2) { W[0] = 0.0; W[nd] = 0.0; W[td] = a; W[3] = a * vt; return; }
    if (p == 1) { W[0] = a; W[nd] = a * un; W[td] = a * vt; W[3] = a * 0.5 * (un * un + vt * vt); return; }
    const double sg = p == 0 ? -1.0 : 1.0;
    W[0] = a; W[nd] = a * (un + sg * c); W[td] = a * vt; W[3] = a * (H + sg * un * c);
  }
  // A-dq from the scratch (Harten-Hyman fixed), A+dq = sum_p s_p W_p - A-dq
  template <int D>
  __device__ static void fluct_w(const double* sc, int st, const double (*W)[4], const double* s,
                                 double* am, double* ap) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      am[k] = sc[(9 + k) * st];
      ap[k] = s[0] * W[0][k] + s[1] * W[1][k] + s[2] * W[2][k] + s[3] * W[3][k] - am[k];
    }
  }
  template <int D>
  __device__ static void fluct(const double* sc, int st, const SolverParams& P, AuxCell ar,
                               double* am, double* ap) {
    double df[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      double W[4];
      wave<D>(sc, st, p, P, W);
      const double s = speed<D>(sc, st, p, P, ar);
#pragma unroll
      for (int k = 0; k < 4; ++k) df[k] += s * W[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      am[k] = sc[(9 + k) * st];
      ap[k] = df[k] - am[k];
    }
  }
  template <int D>
  __device__ static void transverse(const double* sc, int st, const SolverParams& P, const double* X,
                                    AuxCell, AuxCell, double* bm, double* bp) {
    roe_transverse<D>(sc[4 * st], sc[5 * st], sc[6 * st], sc[7 * st], sc[8 * st], P.p0 - 1.0, X, bm, bp);
  }
  // B-X and B+X of the Roe matrix (u, v, H, c, 1/c) along the transverse direction of sweep D
  template <int D>
  __device__ static void roe_transverse(double u, double v, double H, double c, double ic, double gm1,
                                        const double* X, double* bm, double* bp) {
    constexpr int nd = 3 - D, td = D;
    const double vn = nd == 1 ? u : v, vt = nd == 1 ? v : u;
    const double b3 = X[td] - vt * X[0];
    const double b2 = gm1 * (ic * ic) * ((H - vn * vn - vt * vt) * X[0] + vn * X[nd] + vt * X[td] - X[3]);
    const double b4 = (X[nd] + (c - vn) * X[0] - c * b2) * (0.5 * ic);
    const double b1 = X[0] - b2 - b4;
    const double ek = 0.5 * (vn * vn + vt * vt);
    // B-X and B+X: sum over waves of min/max(lambda, 0) b r
    double l1m, l1p, l2m, l2p, l4m, l4p;
    split0(vn - c, l1m, l1p);
    split0(vn, l2m, l2p);
    split0(vn + c, l4m, l4p);
    const double m1 = l1m * b1, m2 = l2m * b2, m3 = l2m * b3, m4 = l4m * b4;
    const double p1 = l1p * b1, p2 = l2p * b2, p3 = l2p * b3, p4 = l4p * b4;
    bm[0] = m1 + m2 + m4;
    bm[nd] = m1 * (vn - c) + m2 * vn + m4 * (vn + c);
    bm[td] = (m1 + m2 + m4) * vt + m3;
    bm[3] = m1 * (H - vn * c) + m2 * ek + m3 * vt + m4 * (H + vn * c);
    bp[0] = p1 + p2 + p4;
    bp[nd] = p1 * (vn - c) + p2 * vn + p4 * (vn + c);
    bp[td] = (p1 + p2 + p4) * vt + p3;
    bp[3] = p1 * (H - vn * c) + p2 * ek + p3 * vt + p4 * (H + vn * c);
  }
};

// ----------------------------------------------------------------------------------------------
// Euler, HLLE (Einfeldt; LeVeque 2002 §15.3.7; the oracle's rp_hlle): two waves
// through one middle state, s1 = min(u_l - c_l, u^ - c^), s2 = max(u_r + c_r, u^ + c^),
// W1 = (f(Q_r) - f(Q_l) - s2 dQ) / (s1 - s2), W2 = dQ - W1; the transverse solve is the Roe one
// (reading 25).  Scratch: W1, W2, s1, s2, Roe u, v, H, c, 1/c.
struct EulerHlle {
  static constexpr int MEQN = 4, MW = 2, NS = 15, NC = 5, PB = NS, NSA = PB + MEQN;
  static constexpr bool CAPA = false, AM_STORED = false;
  __device__ static double quiescent_cfl(const double* q, int qs, const SolverParams& P, const double* a,
                                         double dtdx, int i0, int i1, int i2, int i3) {
    return EulerRoe::quiescent_cfl(q, qs, P, a, dtdx, i0, i1, i2, i3);
  }
  template <int D>
  __device__ static void flux(const double* q, int qs, double ue, const SolverParams& P, double* f) {
    EulerRoe::flux<D>(q, qs, ue, P, f);
  }
  __device__ static void precompute(const double* q, int qs, const SolverParams& P, double* c, int cs) {
    EulerRoe::precompute(q, qs, P, c, cs);   // sqrt(rho), u, v, H, c
  }
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, const double* cl, const double* cr,
                                 int cs, AuxCell, AuxCell, const SolverParams& P, double* sc, int st) {
    constexpr int nd = D;
    const double gm1 = P.p0 - 1.0;
    const double wl = cl[0], wr = cr[0];
    const double inv = fast_rcp(wl + wr);
    const double al = wl * inv, ar = wr * inv;
    const double u = al * cl[cs] + ar * cr[cs];
    const double v = al * cl[2 * cs] + ar * cr[2 * cs];
    const double H = al * cl[3 * cs] + ar * cr[3 * cs];
    const double c2 = gm1 * (H - 0.5 * (u * u + v * v));
    const double ic = fast_rsqrt(c2);
    const double c = c2 * ic;
    const double un = nd == 1 ? u : v;
    const double s1 = fmin(cl[nd * cs] - cl[4 * cs], un - c);
    const double s2 = fmax(cr[nd * cs] + cr[4 * cs], un + c);
    double fl[4], fr[4];
    EulerRoe::flux<D>(ql, 1, 0.0, P, fl);
    EulerRoe::flux<D>(qr, 1, 0.0, P, fr);
    const double r12 = fast_rcp(s1 - s2);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double dq = qr[k] - ql[k];
      const double w1 = ((fr[k] - fl[k]) - s2 * dq) * r12;
      sc[k * st] = w1;
      sc[(4 + k) * st] = dq - w1;
    }
    sc[8 * st] = s1; sc[9 * st] = s2;
    sc[10 * st] = u; sc[11 * st] = v; sc[12 * st] = H; sc[13 * st] = c; sc[14 * st] = ic;
  }
  template <int D>
  __device__ static double speed(const double* sc, int st, int p, const SolverParams&, AuxCell) {
    return sc[(8 + p) * st];
  }
  template <int D>
  __device__ static void wave(const double* sc, int st, int p, const SolverParams&, double* W) {
#pragma unroll
    for (int k = 0; k < 4; ++k) W[k] = sc[(4 * p + k) * st];
  }
  template <int D>
  __device__ static void fluct(const double* sc, int st, const SolverParams&, AuxCell, double* am, double* ap) {
    double m1, p1, m2, p2;
    split0(sc[8 * st], m1, p1);
    split0(sc[9 * st], m2, p2);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      am[k] = m1 * sc[k * st] + m2 * sc[(4 + k) * st];
      ap[k] = p1 * sc[k * st] + p2 * sc[(4 + k) * st];
    }
  }
  template <int D>
  __device__ static void transverse(const double* sc, int st, const SolverParams& P, const double* X,
                                    AuxCell, AuxCell, double* bm, double* bp) {
    EulerRoe::roe_transverse<D>(sc[10 * st], sc[11 * st], sc[12 * st], sc[13 * st], sc[14 * st], P.p0 - 1.0, X,
                                bm, bp);
  }
};

}  // namespace fc
