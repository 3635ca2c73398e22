// step_ws.cuh -- register-resident solver views of the warp-sweep systems kernel (step_ws.cu),
// shared with the quiescent filter (step.cu) so that a quiescent patch's CFL is computed with the
// full update's own arithmetic.  libfc only; nothing shared with oracle/.
#pragma once
#include <cuda_runtime.h>

#include "solvers.cuh"

namespace fc {

// full-warp shuffles of a double as one non-volatile PTX block (the two 32-bit halves of the
// register pair; the header's versions split and rejoin through volatile movs, which cost real
// moves in the sweep loop).  Every caller runs with the whole warp converged.
__device__ __forceinline__ double ws_shfl_idx(double x, int src) {
  double y;
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\t"
      "shfl.sync.idx.b32 lo, lo, %2, 0x1f, 0xffffffff;\n\t"
      "shfl.sync.idx.b32 hi, hi, %2, 0x1f, 0xffffffff;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=d"(y) : "d"(x), "r"(src));
  return y;
}
__device__ __forceinline__ double ws_shfl_down(double x, int d) {
  double y;
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\t"
      "shfl.sync.down.b32 lo, lo, %2, 0x1f, 0xffffffff;\n\t"
      "shfl.sync.down.b32 hi, hi, %2, 0x1f, 0xffffffff;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=d"(y) : "d"(x), "r"(d));
  return y;
}

// ------------------------------------------------------------------------------------------------
// register-resident views of the solvers (the same formulas as solvers.cuh / SURVEY §8(c.5))
struct WsEuler {
  static constexpr int MEQN = 4, MW = 4;
  // components of wave p along sweep D that can be nonzero (the shear wave moves only the
  // tangential momentum and the energy): the others are skipped at compile time
  __host__ __device__ static constexpr bool wave_nz(int D, int p, int k) { return p != 2 || k == 3 - D || k == 3; }
  struct Cell {
    double q[4];
    double sr, u, v, H, c2;   // sqrt(rho), velocity, enthalpy, sound speed squared
  };
  struct Edge {
    double a[4];              // wave strengths
    double u, v, H, c, ic;    // Roe state
    double am[4];             // A-dq (Harten-Hyman fixed)
  };
  __device__ static void cell(Cell& C, const SolverParams& P) {
    const double gam = P.p0, gm1 = gam - 1.0;
    const double rho = C.q[0];
    const double rs = fast_rsqrt(rho);
    const double ir = rs * rs;
    C.sr = rho * rs;
    C.u = C.q[1] * ir;
    C.v = C.q[2] * ir;
    const double p = gm1 * (C.q[3] - 0.5 * rho * (C.u * C.u + C.v * C.v));
    C.H = (C.q[3] + p) * ir;
    C.c2 = gam * p * ir;
  }
  // lambda = m/rho -+ c of a conserved state is beyond 0 (division-free: m^2 > gam (gam-1) (E rho - |m|^2/2))
  __device__ static bool supersonic(double rho, double mn, double mt, double E, double gam) {
    return mn * mn > gam * (gam - 1.0) * (E * rho - 0.5 * (mn * mn + mt * mt));
  }
  template <int D>
  __device__ static void riemann(const Cell& L, const Cell& R, const SolverParams& P, Edge& E) {
    constexpr int nd = D, td = 3 - D;
    const double gam = P.p0, gm1 = gam - 1.0;
    const double inv = fast_rcp(L.sr + R.sr);
    const double al = L.sr * inv, ar = R.sr * inv;
    const double u = al * L.u + ar * R.u;
    const double v = al * L.v + ar * R.v;
    const double H = al * L.H + ar * R.H;
    const double c2 = gm1 * (H - 0.5 * (u * u + v * v));
    const double ic = fast_rsqrt(c2);
    const double c = c2 * ic;
    const double un = nd == 1 ? u : v, vt = nd == 1 ? v : u;
    double d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) d[k] = R.q[k] - L.q[k];
    const double a3 = d[td] - vt * d[0];
    const double a2 = gm1 * (ic * ic) * ((H - un * un - vt * vt) * d[0] + un * d[nd] + vt * d[td] - d[3]);
    const double a4 = (d[nd] + (c - un) * d[0] - c * a2) * (0.5 * ic);
    const double a1 = d[0] - a2 - a4;
    E.a[0] = a1; E.a[1] = a2; E.a[2] = a3; E.a[3] = a4;
    E.u = u; E.v = v; E.H = H; E.c = c; E.ic = ic;
    double W1[4], W4[4], W23[4];
    W1[0] = a1; W1[nd] = a1 * (un - c); W1[td] = a1 * vt; W1[3] = a1 * (H - un * c);
    W4[0] = a4; W4[nd] = a4 * (un + c); W4[td] = a4 * vt; W4[3] = a4 * (H + un * c);
    W23[0] = a2; W23[nd] = a2 * un; W23[td] = a2 * vt + a3;
    W23[3] = a2 * 0.5 * (un * un + vt * vt) + a3 * vt;
    const double s1 = un - c, s2 = un, s4 = un + c;
    if (P.p1 == 0.0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) E.am[k] = dmin0(s1) * W1[k] + dmin0(s2) * W23[k] + dmin0(s4) * W4[k];
      return;
    }
    // Harten-Hyman; the signs of lambda_1(Q_l) and lambda_4(Q_r) by
    // division-free tests, their values only in the (rare) transonic case
    const double unl = nd == 1 ? L.u : L.v, unr = nd == 1 ? R.u : R.v;
    const bool s0_nonneg = unl >= 0.0 && unl * unl >= L.c2;          // lambda_1(Q_l) >= 0
#pragma unroll
    for (int k = 0; k < 4; ++k) E.am[k] = 0.0;
    if (s0_nonneg && s1 > 0.0) return;                                // (i) supersonic to the right
    double beta = s1 < 0.0 ? s1 : 0.0;                                // (ii)
    if (!s0_nonneg) {
      double q1[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) q1[k] = L.q[k] + W1[k];
      if (q1[nd] > 0.0 && supersonic(q1[0], q1[nd], q1[td], q1[3], gam)) {   // lambda_1(Q_l + W1) > 0
        const double s0 = unl - L.c2 * fast_rsqrt(L.c2);
        const double ir = fast_rcp(q1[0]);
        const double un1 = q1[nd] * ir, ut1 = q1[td] * ir;
        const double p1 = gm1 * (q1[3] - 0.5 * q1[0] * (un1 * un1 + ut1 * ut1));
        const double cc = gam * p1 * ir;
        const double lr = un1 - cc * fast_rsqrt(cc);
        beta = s0 * (lr - s1) * fast_rcp(lr - s0);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) E.am[k] = beta * W1[k];
    if (s2 < 0.0) {                                                   // (iii)
#pragma unroll
      for (int k = 0; k < 4; ++k) E.am[k] += s2 * W23[k];
      double b4 = s4 < 0.0 ? s4 : 0.0;                                // (iv)
      const bool s4r_pos = !(unr < 0.0 && unr * unr >= R.c2);         // lambda_4(Q_r) > 0
      if (s4r_pos) {
        double q3[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) q3[k] = R.q[k] - W4[k];
        if (q3[nd] < 0.0 && supersonic(q3[0], q3[nd], q3[td], q3[3], gam)) {   // lambda_4(Q_r - W4) < 0
          const double s4r = unr + R.c2 * fast_rsqrt(R.c2);
          const double ir = fast_rcp(q3[0]);
          const double un3 = q3[nd] * ir, ut3 = q3[td] * ir;
          const double p3 = gm1 * (q3[3] - 0.5 * q3[0] * (un3 * un3 + ut3 * ut3));
          const double cc = gam * p3 * ir;
          const double ll = un3 + cc * fast_rsqrt(cc);
          b4 = ll * (s4r - s4) * fast_rcp(s4r - ll);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) E.am[k] += b4 * W4[k];
    }
  }
  template <int D>
  __device__ static double speed(const Edge& E, int p) {
    const double un = D == 1 ? E.u : E.v;
    return p == 0 ? un - E.c : (p == 3 ? un + E.c : un);
  }
  // max_p |s_p| = |un| + c (bitwise the larger of |un - c|, |un + c|)
  template <int D>
  __device__ static double max_speed(const Edge& E) { return fabs(D == 1 ? E.u : E.v) + E.c; }
  template <int D>
  __device__ static void wave(const Edge& E, int p, double* W) {
    constexpr int nd = D, td = 3 - D;
    const double un = nd == 1 ? E.u : E.v, vt = nd == 1 ? E.v : E.u;
    const double a = E.a[p];
    if (p == 2) { W[0] = 0.0; W[nd] = 0.0; W[td] = a; W[3] = a * vt; return; }
    if (p == 1) { W[0] = a; W[nd] = a * un; W[td] = a * vt; W[3] = a * 0.5 * (un * un + vt * vt); return; }
    const double sg = p == 0 ? -1.0 : 1.0;
    W[0] = a; W[nd] = a * (un + sg * E.c); W[td] = a * vt; W[3] = a * (E.H + sg * un * E.c);
  }
  // the Roe state an edge's transverse splits need
  struct Roe {
    double u, v, H, c, ic;
  };
  __device__ static Roe roe(const Edge& E) { return {E.u, E.v, E.H, E.c, E.ic}; }
  // 2 B-X, 2 B+X of the Roe matrix along the transverse direction of sweep D for two inputs X = XA,
  // XB (EulerRoe::roe_transverse's formulas; the eigenvalue split as lambda -+ |lambda|, i.e. twice
  // its halves, the caller scaling by 1/2: exact; the terms of the Roe state alone -- gm1/c^2,
  // H - |v|^2, the eigenvalue halves -- once for both).  With the eigenvectors r1 = (1, vn - c, vt,
  // H - vn c), r2 = (1, vn, vt, ek), r3 = (0, 0, 1, vt), r4 = (1, vn + c, vt, H + vn c) and weights
  // m_p, sum_p m_p r_p = (S + m2, vn (S + m2) + D, vt (S + m2) + m3, H S + vn D + ek m2 + vt m3)
  // with S = m1 + m4, D = c (m4 - m1): the same sum, regrouped.
  template <int D>
  __device__ static void transverse2(const Roe& r, const SolverParams& P, const double* XA, const double* XB,
                                     double* bmA, double* bpA, double* bmB, double* bpB) {
    constexpr int nd = 3 - D, td = D;
    const double gm1 = P.p0 - 1.0, c = r.c, ic = r.ic, H = r.H;
    const double vn = nd == 1 ? r.u : r.v, vt = nd == 1 ? r.v : r.u;
    const double K = gm1 * (ic * ic), E = H - vn * vn - vt * vt, cv = c - vn, hic = 0.5 * ic;
    const double ek = 0.5 * (vn * vn + vt * vt);
    const double l1 = vn - c, l4 = vn + c;
    const double w1m = l1 - fabs(l1), w2m = vn - fabs(vn), w4m = l4 - fabs(l4);
    const double w1p = l1 + fabs(l1), w2p = vn + fabs(vn), w4p = l4 + fabs(l4);
    auto one = [&](const double* X, double* bm, double* bp) {
      const double b3 = X[td] - vt * X[0];
      const double b2 = K * (E * X[0] + vn * X[nd] + vt * X[td] - X[3]);
      const double b4 = (X[nd] + cv * X[0] - c * b2) * hic;
      const double b1 = X[0] - b2 - b4;
      auto set = [&](double w1, double w2, double w4, double* o) {
        const double m1 = w1 * b1, m2 = w2 * b2, m3 = w2 * b3, m4 = w4 * b4;
        const double S = m1 + m4, Dd = c * (m4 - m1), o0 = S + m2;
        o[0] = o0;
        o[nd] = fma(vn, o0, Dd);
        o[td] = fma(vt, o0, m3);
        o[3] = fma(H, S, fma(vn, Dd, fma(ek, m2, vt * m3)));
      };
      set(w1m, w2m, w4m, bm);
      set(w1p, w2p, w4p, bp);
    };
    one(XA, bmA, bpA);
    one(XB, bmB, bpB);
  }
  __device__ static double quiescent_cfl(const double* q, int qs, const SolverParams& P, double dtdx) {
    return EulerRoe::quiescent_cfl(q, qs, P, nullptr, dtdx, 0, 0, 0, 0);
  }
};

struct WsSwe {
  static constexpr int MEQN = 3, MW = 3;
  __host__ __device__ static constexpr bool wave_nz(int D, int p, int k) { return p != 1 || k == 3 - D; }
  struct Cell {
    double q[3];
    double sr, u, v;
  };
  struct Edge {
    double a[3];
    double u, v, c, ic;
    double am[3];
  };
  __device__ static void cell(Cell& C, const SolverParams&) {
    const double h = C.q[0];
    const double rs = fast_rsqrt(h);
    const double ih = rs * rs;
    C.sr = h * rs;
    C.u = C.q[1] * ih;
    C.v = C.q[2] * ih;
  }
  template <int D>
  __device__ static void riemann(const Cell& L, const Cell& R, const SolverParams& P, Edge& E) {
    constexpr int nd = D, td = 3 - D;
    const double inv = fast_rcp(L.sr + R.sr);
    const double al = L.sr * inv, ar = R.sr * inv;
    const double u = al * L.u + ar * R.u;
    const double v = al * L.v + ar * R.v;
    const double c2 = 0.5 * P.p0 * (L.q[0] + R.q[0]);
    const double ic = fast_rsqrt(c2);
    const double c = c2 * ic;
    const double un = nd == 1 ? u : v, ut = nd == 1 ? v : u;
    const double dh = R.q[0] - L.q[0], dn = R.q[nd] - L.q[nd], dtg = R.q[td] - L.q[td];
    const double i2c = 0.5 * ic;
    E.a[0] = ((un + c) * dh - dn) * i2c;
    E.a[1] = dtg - ut * dh;
    E.a[2] = ((c - un) * dh + dn) * i2c;
    E.u = u; E.v = v; E.c = c; E.ic = ic;
#pragma unroll
    for (int k = 0; k < 3; ++k) E.am[k] = 0.0;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      double W[3];
      wave<D>(E, p, W);
      const double s = speed<D>(E, p);
#pragma unroll
      for (int k = 0; k < 3; ++k) E.am[k] += dmin0(s) * W[k];
    }
  }
  template <int D>
  __device__ static double speed(const Edge& E, int p) {
    const double un = D == 1 ? E.u : E.v;
    return p == 0 ? un - E.c : (p == 1 ? un : un + E.c);
  }
  template <int D>
  __device__ static double max_speed(const Edge& E) { return fabs(D == 1 ? E.u : E.v) + E.c; }
  template <int D>
  __device__ static void wave(const Edge& E, int p, double* W) {
    constexpr int nd = D, td = 3 - D;
    const double un = nd == 1 ? E.u : E.v, ut = nd == 1 ? E.v : E.u;
    const double a = E.a[p];
    if (p == 1) { W[0] = 0.0; W[nd] = 0.0; W[td] = a; return; }
    W[0] = a;
    W[nd] = a * (p == 0 ? un - E.c : un + E.c);
    W[td] = a * ut;
  }
  struct Roe {
    double u, v, c, ic;
  };
  __device__ static Roe roe(const Edge& E) { return {E.u, E.v, E.c, E.ic}; }
  // 2 B-X, 2 B+X for two inputs (as WsEuler::transverse2): sum_p m_p r_p with r1 = (1, vn - c, vt),
  // r2 = (0, 0, 1), r3 = (1, vn + c, vt) is (S, vn S + c (m3 - m1), vt S + m2), S = m1 + m3
  template <int D>
  __device__ static void transverse2(const Roe& r, const SolverParams&, const double* XA, const double* XB,
                                     double* bmA, double* bpA, double* bmB, double* bpB) {
    constexpr int nd = 3 - D, td = D;
    const double vn = nd == 1 ? r.u : r.v, vt = nd == 1 ? r.v : r.u, c = r.c;
    const double i2c = 0.5 * r.ic, pc = vn + c, mc = c - vn;
    const double l1 = vn - c, l3 = vn + c;
    const double w1m = l1 - fabs(l1), w2m = vn - fabs(vn), w3m = l3 - fabs(l3);
    const double w1p = l1 + fabs(l1), w2p = vn + fabs(vn), w3p = l3 + fabs(l3);
    auto one = [&](const double* X, double* bm, double* bp) {
      const double b1 = (pc * X[0] - X[nd]) * i2c;
      const double b2 = X[td] - vt * X[0];
      const double b3 = (mc * X[0] + X[nd]) * i2c;
      auto set = [&](double w1, double w2, double w3, double* o) {
        const double m1 = w1 * b1, m2 = w2 * b2, m3 = w3 * b3;
        const double S = m1 + m3;
        o[0] = S;
        o[nd] = fma(vn, S, c * (m3 - m1));
        o[td] = fma(vt, S, m2);
      };
      set(w1m, w2m, w3m, bm);
      set(w1p, w2p, w3p, bp);
    };
    one(XA, bmA, bpA);
    one(XB, bmB, bpB);
  }
  __device__ static double quiescent_cfl(const double* q, int qs, const SolverParams& P, double dtdx) {
    return SweRoe::quiescent_cfl(q, qs, P, nullptr, dtdx, 0, 0, 0, 0);
  }
};

// an opaque copy of a double: two loads of one value stay two values for the compiler (no CSE), so
// the expressions below are contracted exactly like the general two-state case
__device__ __forceinline__ double opaque_d(double x) {
  double y;
  asm volatile("mov.b64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// CFL of a quiescent (uniform) window: the full update's per-edge value r (|u_n| + c) of the Roe
// state of two equal cells, x and y edges, computed by the same solver code (bitwise the full
// update's CFL of that window; the shortcut then follows the same dt sequence)
template <class S>
__device__ __forceinline__ double ws_quiescent_cfl(const double* q, int qs, const SolverParams& P, double r) {
  typename S::Cell L, R;
#pragma unroll
  for (int k = 0; k < S::MEQN; ++k) {
    L.q[k] = opaque_d(q[k * qs]);
    R.q[k] = opaque_d(q[k * qs]);
  }
  S::cell(L, P);
  S::cell(R, P);
  typename S::Edge E1, E2;
  S::template riemann<1>(L, R, P, E1);
  S::template riemann<2>(L, R, P, E2);
  const double m1 = S::template max_speed<1>(E1), m2 = S::template max_speed<2>(E2);
  return r * (m1 > m2 ? m1 : m2);
}

}  // namespace fc
