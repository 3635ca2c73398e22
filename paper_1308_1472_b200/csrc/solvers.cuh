// solvers.cuh -- device Riemann solvers for the fused step kernel (libfc, sm_100a, fp64).
//
// PAPER.md:171-180 [§3]: "At each edge, we solve Riemann problems to obtain left and right going
// waves propagating at speeds determined from the solution to the Riemann problem.  For scalar
// advection, the speed of each wave is simply the local advection speed at the cell interface.
// For non-linear problems and systems, an approximate Riemann solver, such as a Roe solver ...".
// Each solver stores a compact per-edge state in shared memory during the normal solve (phase 1)
// and reconstructs waves / fluctuations / transverse splittings from it in phase 2:
//   AdvConst      scratch {dq}                         speed from the problem (u or v)
//   AdvEdgeCapa   scratch {dq}                         speed = edge velocity in aux (capacity form)
//   SweRoe        scratch {a1..a3, u, v, c}            Roe state shared by normal + transverse solves
//   EulerRoe      scratch {a1..a4, u, v, H, c, A-dq}   A-dq carries the Harten-Hyman entropy fix
// Directions: D = 1 (x-sweep, normal momentum = component 1) or D = 2 (y-sweep, component 2).
#pragma once
#include <cuda_runtime.h>

namespace fc {

struct SolverParams {
  double p0, p1;  // (u, v) | - | (g, -) | (gamma, efix)
};

// cell aux view: kappa, u~ (left edge), v~ (bottom edge) of one cell (smem window, stride WW)
struct AuxCell {
  const double* a;  // pointer to kappa of the cell; u~ at a[WW], v~ at a[2 WW]
  int WW;
  __device__ double kappa() const { return a[0]; }
  __device__ double ut() const { return a[WW]; }
  __device__ double vt() const { return a[2 * WW]; }
};

__device__ __forceinline__ double dmin0(double s) { return s < 0.0 ? s : 0.0; }
__device__ __forceinline__ double dmax0(double s) { return s > 0.0 ? s : 0.0; }

// ----------------------------------------------------------------------------------------------
struct AdvConst {
  static constexpr int MEQN = 1, MW = 1, NS = 1;
  static constexpr bool CAPA = false;
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, AuxCell, AuxCell,
                                 const SolverParams&, double* sc, int st) {
    sc[0] = qr[0] - ql[0];
    (void)st;
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
  // transverse split of X for the part entering `recv` (next = the cell after it transversally)
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
  static constexpr int MEQN = 1, MW = 1, NS = 1;
  static constexpr bool CAPA = true;
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, AuxCell, AuxCell,
                                 const SolverParams&, double* sc, int) {
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
  static constexpr int MEQN = 3, MW = 3, NS = 6;
  static constexpr bool CAPA = false;
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, AuxCell, AuxCell,
                                 const SolverParams& P, double* sc, int st) {
    constexpr int nd = D, td = 3 - D;
    const double hl = ql[0], hr = qr[0];
    const double sl = sqrt(hl), sr = sqrt(hr);
    const double inv = 1.0 / (sl + sr);
    const double u = (ql[1] / sl + qr[1] / sr) * inv;   // (sqrt(h) (hu/h)) summed
    const double v = (ql[2] / sl + qr[2] / sr) * inv;
    const double c = sqrt(0.5 * P.p0 * (hl + hr));
    const double un = nd == 1 ? u : v, ut = nd == 1 ? v : u;
    const double dh = hr - hl, dn = qr[nd] - ql[nd], dtg = qr[td] - ql[td];
    const double i2c = 0.5 / c;
    sc[0] = ((un + c) * dh - dn) * i2c;
    sc[st] = dtg - ut * dh;
    sc[2 * st] = ((c - un) * dh + dn) * i2c;
    sc[3 * st] = u;
    sc[4 * st] = v;
    sc[5 * st] = c;
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
  // transverse direction td of this sweep, same Roe state
  template <int D>
  __device__ static void transverse(const double* sc, int st, const SolverParams&, const double* X,
                                    AuxCell, AuxCell, double* bm, double* bp) {
    constexpr int nd = 3 - D, td = D;   // eigen-decomposition along the transverse direction
    const double u = sc[3 * st], v = sc[4 * st], c = sc[5 * st];
    const double vn = nd == 1 ? u : v, vt = nd == 1 ? v : u;
    const double i2c = 0.5 / c;
    const double b1 = ((vn + c) * X[0] - X[nd]) * i2c;
    const double b2 = X[td] - vt * X[0];
    const double b3 = ((c - vn) * X[0] + X[nd]) * i2c;
    const double l1 = vn - c, l2 = vn, l3 = vn + c;
    double r1[3], r3[3];
    r1[0] = 1.0; r1[nd] = vn - c; r1[td] = vt;
    r3[0] = 1.0; r3[nd] = vn + c; r3[td] = vt;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double w2 = (k == td) ? b2 : 0.0;
      bm[k] = dmin0(l1) * b1 * r1[k] + dmin0(l2) * w2 + dmin0(l3) * b3 * r3[k];
      bp[k] = dmax0(l1) * b1 * r1[k] + dmax0(l2) * w2 + dmax0(l3) * b3 * r3[k];
    }
  }
};

// ----------------------------------------------------------------------------------------------
// Euler, Roe linearisation with the Harten-Hyman entropy fix:
// a3 = d(mt) - vt drho; a2 = (g-1)/c^2 [(H - un^2 - vt^2) drho + un d(mn) + vt d(mt) - dE];
// a4 = (d(mn) + (c - un) drho - c a2)/(2c); a1 = drho - a2 - a4;
// r1 = (1, un-c, vt, H - un c), r2 = (1, un, vt, (un^2+vt^2)/2), r3 = (0, 0, 1, vt)_t,
// r4 = (1, un+c, vt, H + un c); speeds un-c, un, un, un+c.
struct EulerRoe {
  static constexpr int MEQN = 4, MW = 4, NS = 12;
  static constexpr bool CAPA = false;
  __device__ static double pressure(const double* q, double gm1) {
    const double ir = 1.0 / q[0];
    return gm1 * (q[3] - 0.5 * (q[1] * q[1] + q[2] * q[2]) * ir);
  }
  template <int D>
  __device__ static void riemann(const double* ql, const double* qr, AuxCell, AuxCell,
                                 const SolverParams& P, double* sc, int st) {
    constexpr int nd = D, td = 3 - D;
    const double gam = P.p0, gm1 = gam - 1.0;
    const double pl = pressure(ql, gm1), pr = pressure(qr, gm1);
    const double sl = sqrt(ql[0]), sr = sqrt(qr[0]);
    const double inv = 1.0 / (sl + sr);
    const double u = (ql[1] / sl + qr[1] / sr) * inv;
    const double v = (ql[2] / sl + qr[2] / sr) * inv;
    const double H = ((ql[3] + pl) / sl + (qr[3] + pr) / sr) * inv;
    const double c2 = gm1 * (H - 0.5 * (u * u + v * v));
    const double c = sqrt(c2);
    const double un = nd == 1 ? u : v, vt = nd == 1 ? v : u;
    double d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = qr[k] - ql[k];
    const double a3 = d[td] - vt * d[0];
    const double a2 = gm1 / c2 * ((H - un * un - vt * vt) * d[0] + un * d[nd] + vt * d[td] - d[3]);
    const double a4 = (d[nd] + (c - un) * d[0] - c * a2) * (0.5 / c);
    const double a1 = d[0] - a2 - a4;
    sc[0] = a1; sc[st] = a2; sc[2 * st] = a3; sc[3 * st] = a4;
    sc[4 * st] = u; sc[5 * st] = v; sc[6 * st] = H; sc[7 * st] = c;
    // A-dq
    double am[4];
    const double s1 = un - c, s2 = un, s4 = un + c;
    double W1[4], W2[4], W3[4], W4[4];
    W1[0] = a1; W1[nd] = a1 * (un - c); W1[td] = a1 * vt; W1[3] = a1 * (H - un * c);
    W2[0] = a2; W2[nd] = a2 * un; W2[td] = a2 * vt; W2[3] = a2 * 0.5 * (un * un + vt * vt);
    W3[0] = 0.0; W3[nd] = 0.0; W3[td] = a3; W3[3] = a3 * vt;
    W4[0] = a4; W4[nd] = a4 * (un + c); W4[td] = a4 * vt; W4[3] = a4 * (H + un * c);
    if (P.p1 == 0.0) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        am[k] = dmin0(s1) * W1[k] + dmin0(s2) * (W2[k] + W3[k]) + dmin0(s4) * W4[k];
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) am[k] = 0.0;
      const double s0 = ql[nd] / ql[0] - sqrt(gam * pl / ql[0]);      // lambda_1(Q_l)
      if (!(s0 >= 0.0 && s1 > 0.0)) {
        double q1[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) q1[k] = ql[k] + W1[k];
        const double p1 = pressure(q1, gm1);
        const double s1r = q1[nd] / q1[0] - sqrt(gam * p1 / q1[0]);    // lambda_1(Q_l + W1)
        double beta;
        if (s0 < 0.0 && s1r > 0.0) beta = s0 * (s1r - s1) / (s1r - s0);
        else if (s1 < 0.0) beta = s1;
        else beta = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) am[k] = beta * W1[k];
        if (s2 < 0.0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) am[k] += s2 * (W2[k] + W3[k]);
          double q3[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) q3[k] = qr[k] - W4[k];
          const double p3 = pressure(q3, gm1);
          const double s4l = q3[nd] / q3[0] + sqrt(gam * p3 / q3[0]);  // lambda_4(Q_r - W4)
          const double s4r = qr[nd] / qr[0] + sqrt(gam * pr / qr[0]);  // lambda_4(Q_r)
          if (s4l < 0.0 && s4r > 0.0) {
            const double b4 = s4l * (s4r - s4) / (s4r - s4l);
#pragma unroll
            for (int k = 0; k < 4; ++k) am[k] += b4 * W4[k];
          } else if (s4 < 0.0) {
#pragma unroll
            for (int k = 0; k < 4; ++k) am[k] += s4 * W4[k];
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) sc[(8 + k) * st] = am[k];
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
      am[k] = sc[(8 + k) * st];
      ap[k] = df[k] - am[k];
    }
  }
  template <int D>
  __device__ static void transverse(const double* sc, int st, const SolverParams& P, const double* X,
                                    AuxCell, AuxCell, double* bm, double* bp) {
    constexpr int nd = 3 - D, td = D;
    const double gm1 = P.p0 - 1.0;
    const double u = sc[4 * st], v = sc[5 * st], H = sc[6 * st], c = sc[7 * st];
    const double vn = nd == 1 ? u : v, vt = nd == 1 ? v : u;
    const double c2 = c * c;
    const double b3 = X[td] - vt * X[0];
    const double b2 = gm1 / c2 * ((H - vn * vn - vt * vt) * X[0] + vn * X[nd] + vt * X[td] - X[3]);
    const double b4 = (X[nd] + (c - vn) * X[0] - c * b2) * (0.5 / c);
    const double b1 = X[0] - b2 - b4;
    double r1[4], r2[4], r3[4], r4[4];
    r1[0] = 1.0; r1[nd] = vn - c; r1[td] = vt; r1[3] = H - vn * c;
    r2[0] = 1.0; r2[nd] = vn; r2[td] = vt; r2[3] = 0.5 * (vn * vn + vt * vt);
    r3[0] = 0.0; r3[nd] = 0.0; r3[td] = 1.0; r3[3] = vt;
    r4[0] = 1.0; r4[nd] = vn + c; r4[td] = vt; r4[3] = H + vn * c;
    const double l1 = vn - c, l2 = vn, l4 = vn + c;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bm[k] = dmin0(l1) * b1 * r1[k] + dmin0(l2) * (b2 * r2[k] + b3 * r3[k]) + dmin0(l4) * b4 * r4[k];
      bp[k] = dmax0(l1) * b1 * r1[k] + dmax0(l2) * (b2 * r2[k] + b3 * r3[k]) + dmax0(l4) * b4 * r4[k];
    }
  }
};

}  // namespace fc
