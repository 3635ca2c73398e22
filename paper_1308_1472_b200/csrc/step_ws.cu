// step_ws.cu -- the warp-sweep step kernel for systems (libfc, sm_100a, fp64): Roe shallow water
// (C3) and Roe Euler with the Harten-Hyman entropy fix (C5).
//
// PAPER.md:168-182 [§3]: Clawpack's unsplit wave propagation on one patch -- Riemann problems at
// every edge, left/right-going waves, a wave limiter on the upwind neighbour's wave, second-order
// corrections, transverse (rpt2) corrections (readings in DESIGN.md §3).  Same arithmetic as the
// phased k_step (step.cu) and the oracle (oracle/claw.c), different schedule:
//
// One CTA (NW warps) per 16 x 16 tile at a time (persistent over tiles), its 20 x 20 window (tile +
// 2-cell halo, natural layout, row pitch 22: 16-byte interior copies) gathered by cp.async straight
// from the neighbours' interiors (the fused ring gather: no ring is ever written to HBM), the next
// tile's gather in flight while the current one computes.  Per tile three phases, one barrier each:
//   X  the 18 x 19 x-edges of rows 0..17 as 12 warp-iterations of 32 consecutive edges (row-major,
//      advancing 29: lanes 0 and 31 are halo edges for the limiter).  Per lane: both cells' derived
//      fields, the Roe solve (+ Harten-Hyman A-dq), then per wave family the upwind neighbour's wave
//      by one warp shuffle -> limiter, F~, CFL; both transverse splits of the edge with its own
//      Roe state, of its L part P = A-dq + F~ (into the left cell: handed to the previous edge's
//      lane with P by shuffle) and of its R part Q (the right cell, the lane's output cell) -> up /
//      dn (G~ halves) and the x increment of the cell, to shared memory.
//   Y  the same along y (column-major flat edges); the lane owning a cell also folds the x-sweep's
//      G~ differences into its increment; transverse parts -> rt / lf (F~ halves).
//   F  per cell q_new = q + dq - r (F~(i+1/2) - F~(i-1/2)), stored coalesced; non-finite check.
// No per-edge scratch round trip through shared memory (the phased kernel's 7 barrier-separated
// phases and 13-slot edge scratch), no index tables, every edge solved once per sweep except the two
// halo lanes of each iteration.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "../../include/fc.h"
#include "fc_internal.h"
#include "solvers.cuh"
#include "step_common.cuh"
#include "step_ws.cuh"

namespace fc {

// ------------------------------------------------------------------------------------------------
template <class S>
struct WsShape {
#ifndef WS_CHUNK
#define WS_CHUNK 1
#endif
  // window 20 x 20, row pitch 22 (WS_CHUNK: even, so that the tile interior's rows arrive as
  // 16-byte copies) or 21 (odd: conflict-free column access, 8-byte copies only)
  static constexpr bool CHUNK = WS_CHUNK != 0;
  static constexpr int T = 16, W = T + 4, PW = CHUNK ? W + 2 : W + 1;
  static constexpr int NH = W * W - T * T;                     // halo cells of the window (144)
  static constexpr int WPW = W * PW;                           // component stride of the window
  static constexpr int NE = T + 3, NR = T + 2, E = NR * NE;    // 19 edges x 18 rows per sweep
  static constexpr int STEP = 29, NIT = (E + STEP - 1) / STEP; // 12 warp-iterations per sweep
  static constexpr int QB = S::MEQN * WPW;
  static constexpr int UPP = T + 1;                            // up / dn rows [k][j = 0..T+1][i = 1..T]
  static constexpr int RTP = T + 3;                            // rt / lf rows [k][j = 1..T][i = 0..T+1]
  static constexpr int DQP = T + 1;                            // dq rows [k][j = 1..T][i = 1..T]
  static constexpr int N_UP = S::MEQN * NR * UPP;
  static constexpr int N_RT = S::MEQN * T * RTP;
  static constexpr int N_DQ = S::MEQN * T * DQP;
  static constexpr int NDESC = 2 * NIT * 32;                  // lane descriptors of both sweeps (int32)
  static constexpr size_t smem_doubles(int nbuf) {
    return nbuf * (size_t)QB + 2 * (size_t)N_UP + 2 * (size_t)N_RT + 2 * (size_t)N_DQ + NDESC / 2;
  }
  static constexpr size_t smem_bytes(int nbuf) { return smem_doubles(nbuf) * sizeof(double); }
};

// tile -> (patch, tile column, tile row)
__device__ __forceinline__ void ws_tile(const StepArgs& A, int tile, int& patch, int& tx, int& ty) {
  patch = tile;
  tx = ty = 0;
  if (A.tiles > 1) {
    const int t2 = A.tiles * A.tiles;
    patch = tile / t2;
    const int t = tile - patch * t2;
    ty = t / A.tiles;
    tx = t - ty * A.tiles;
  }
}

// cp.async gather of a tile's 20 x 20 window (natural layout, pitch 22): cells inside the patch
// interior from its own storage block, the others from the ring-source table (a neighbour's
// interior, a peer rank's buffer, or a computed ghost); physical-boundary cells after the wait.
// Two stages so that the ring-table loads never stall the issuing thread: ws_prep loads this
// thread's (<= 3) table entries a whole tile ahead, ws_issue turns them into cp.async copies.
template <int GU>          // window cells per thread (ceil(400 / threads))
struct WsGather {
  int tile;
  int32_t v[GU];           // ring source offset, or -1 - BC code, or INT32_MIN: own interior
  uint8_t ow[GU];          // owner code of a ring source (0 local, k peer rank k-1, 255 computed)
};
// window cell c of a thread's gather share: with CHUNK the halo cells only (rows 0, 1, W-2, W-1
// whole, then columns 0, 1, W-2, W-1 of rows 2..W-3), else every window cell; false past the end
template <class S>
__device__ __forceinline__ bool ws_cell(int c, int& wi, int& wj) {
  using Sh = WsShape<S>;
  constexpr int T = Sh::T, W = Sh::W;
  if (!Sh::CHUNK) {
    wj = c / W;
    wi = c - wj * W;
    return c < W * W;
  }
  if (c < 4 * W) {
    const int r = c / W;
    wj = r < 2 ? r : r + T;
    wi = c - r * W;
  } else {
    const int h = c - 4 * W;
    wj = 2 + (h >> 2);
    wi = (h & 3) < 2 ? (h & 3) : (h & 3) + T;
  }
  return c < Sh::NH;
}

template <class S, int WS_GU>
__device__ __forceinline__ void ws_prep(const StepArgs& A, int tile, WsGather<WS_GU>& g, int tid, int nt) {
  using Sh = WsShape<S>;
  constexpr int T = Sh::T;
  g.tile = tile;
  if (tile < 0) return;
  int patch, tx, ty;
  ws_tile(A, tile, patch, tx, ty);
  const int m = A.m, n = m + 4, G = n * n - m * m;
  const int32_t* rs = A.ring + (int64_t)patch * G;
  const uint8_t* rp = A.rpeer ? A.rpeer + (int64_t)patch * G : nullptr;
  // regular ring: every source address from the 9 neighbour block offsets (L1-resident), no table.
  // Off by default here (WS_REGULAR): the systems kernel is compute-bound and the extra address
  // arithmetic measured +1.5 % on C5 (7.63 vs 7.52 ms); the scalar sweeps use it (cv_stage).
#ifndef WS_REGULAR
#define WS_REGULAR 0
#endif
  const int32_t* nb = (WS_REGULAR && A.nb9) ? A.nb9 + (int64_t)patch * 9 : nullptr;
  const bool reg = nb && __ldg(nb) >= 0;
#pragma unroll
  for (int u = 0; u < WS_GU; ++u) {
    const int c = tid + u * nt;
    g.v[u] = INT32_MIN;
    g.ow[u] = 0;
    int wi, wj;
    if (!ws_cell<S>(c, wi, wj)) continue;
    const int i = tx * T + wi - 1, j = ty * T + wj - 1;   // patch cell (1-based interior)
    if ((unsigned)(i - 1) < (unsigned)m && (unsigned)(j - 1) < (unsigned)m) continue;
    if (reg) {
      const int dx = i < 1 ? -1 : (i > m ? 1 : 0), dy = j < 1 ? -1 : (j > m ? 1 : 0);
      g.v[u] = __ldg(nb + 3 * dy + dx + 4) + (j - dy * m - 1) * m + (i - dx * m - 1);
      continue;
    }
    const int r = ring_index(i, j, m);
    g.v[u] = __ldg(rs + r);
    if (rp) g.ow[u] = __ldg(rp + r);
  }
}
template <class S, int WS_GU>
__device__ __forceinline__ void ws_issue(const StepArgs& A, const WsGather<WS_GU>& g, double* sq, int tid, int nt) {
  using Sh = WsShape<S>;
  constexpr int T = Sh::T, PW = Sh::PW, WPW = Sh::WPW, MEQN = S::MEQN;
  if (g.tile < 0) return;
  int patch, tx, ty;
  ws_tile(A, g.tile, patch, tx, ty);
  const int m = A.m, n = m + 4, n2 = n * n;
  const double* qb = A.qold + (int64_t)patch * MEQN * n2;
  if (Sh::CHUNK) {   // the tile interior: rows of T cells as T / 2 16-byte copies per component
    constexpr int HC = T / 2, PER = T * HC;
    for (int t = tid; t < MEQN * PER; t += nt) {
      const int k = t / PER, rem = t - k * PER, rr = rem / HC, cc = rem - rr * HC;
      cp_async16(sq + k * WPW + (rr + 2) * PW + 2 + 2 * cc, qb + (int64_t)k * n2 + (ty * T + rr) * m + tx * T + 2 * cc);
    }
  }
#pragma unroll
  for (int u = 0; u < WS_GU; ++u) {
    const int c = tid + u * nt;
    int wi, wj;
    if (!ws_cell<S>(c, wi, wj)) continue;
    const double* src;
    if (g.v[u] == INT32_MIN) {
      src = qb + (ty * T + wj - 2) * m + (tx * T + wi - 2);
    } else {
      if (g.v[u] < 0) continue;                          // physical boundary: ws_bc
      src = ring_base(A, g.ow[u]) + g.v[u];
    }
    double* d = sq + wj * PW + wi;
#pragma unroll
    for (int k = 0; k < MEQN; ++k) cp_async8(d + k * WPW, src + (int64_t)k * n2);
  }
}

// physical-boundary window cells, x faces (is_y = 0) then y faces: copy (wall: negate the normal
// momentum) of the patch cell the ring-source code names (within 2 cells: inside this window)
template <class S>
__device__ __forceinline__ void ws_bc(const StepArgs& A, int tile, double* sq, int is_y, int tid, int nt) {
  using Sh = WsShape<S>;
  constexpr int T = Sh::T, W = Sh::W, PW = Sh::PW, WPW = Sh::WPW, MEQN = S::MEQN;
  int patch, tx, ty;
  ws_tile(A, tile, patch, tx, ty);
  const int m = A.m, n = m + 4, G = n * n - m * m;
  const int32_t* rs = A.ring + (int64_t)patch * G;
  for (int c = tid; c < W * W; c += nt) {
    const int wj = c / W, wi = c - wj * W;
    const int i = tx * T + wi - 1, j = ty * T + wj - 1;
    if ((unsigned)(i - 1) < (unsigned)m && (unsigned)(j - 1) < (unsigned)m) continue;
    const int32_t v = __ldg(rs + ring_index(i, j, m));
    if (v >= 0) continue;
    const int code = -1 - v;
    if ((code & 1) != is_y) continue;
    const int src = code >> 3, neg = (code >> 1) & 3;
    const int si = src % n - 1, sj = src / n - 1;
    const int ws = (sj - ty * T + 1) * PW + (si - tx * T + 1);
    const int wd = wj * PW + wi;
#pragma unroll
    for (int k = 0; k < MEQN; ++k) {
      const double x = sq[k * WPW + ws];
      sq[k * WPW + wd] = (neg != 0 && k == neg) ? -x : x;
    }
  }
}

// wave limiter phi(theta) = max(lo, min(c1 + c2 theta, c3, c4 theta)) with compare-selects (the
// operands are never NaN here: theta of a zero wave is replaced by 0 first)
__device__ __forceinline__ double ws_phi(const LimiterCoef& L, double th) {
  double t = fma(L.c2, th, L.c1);
  t = t < L.c3 ? t : L.c3;
  const double t4 = L.c4 * th;
  t = t < t4 ? t : t4;
  return t > L.lo ? t : L.lo;
}

// One warp-iteration `it` of a sweep (D = 1: x-edges of rows 0..T+1; D = 2: y-edges of columns
// 0..T+1; NIT iterations per sweep).  FAST: method2 = 2 and method3 = 2 (the configs) known at
// compile time; otherwise read from A.
// Lane descriptor of warp-iteration `it` of sweep D (the same for every tile: built once per CTA
// into shared memory): the right cell's window offset (9 bits), the edge position and line (5 + 5),
// and the valid / corrected / output flags.
template <class S, int D>
__device__ __forceinline__ uint32_t ws_desc(int it, int lane) {
  using Sh = WsShape<S>;
  constexpr int T = Sh::T, PW = Sh::PW, NE = Sh::NE, E = Sh::E;
  const int e = it * Sh::STEP - 1 + lane;                   // flat edge index of this lane
  const bool ev = (unsigned)e < (unsigned)E;
  const int ee = ev ? e : 0;
  const int line = ee / NE, pos = ee - line * NE;         // D=1: row j, edge i; D=2: column i, edge j
  // the edge between window cells (pos-1, line) and (pos, line) along the sweep (1-based cells)
  const int wr = D == 1 ? (line + 1) * PW + (pos + 1) : (pos + 1) * PW + (line + 1);   // the right cell
  const bool corr = ev && lane >= 1 && lane <= 30 && pos >= 1 && pos <= T + 1;
  const bool out = ev && lane >= 1 && lane <= 29 && pos >= 1 && pos <= T;
  static_assert((T + 3) * PW < 512 && T + 3 < 32, "descriptor fields");
  return (uint32_t)wr | (uint32_t)pos << 9 | (uint32_t)line << 14 | (uint32_t)corr << 20 | (uint32_t)out << 21;
}

// One warp-iteration of a sweep (D = 1: x-edges of rows 0..T+1; D = 2: y-edges of columns
// 0..T+1; NIT iterations per sweep), its lane's descriptor `dsc`, in three stages: ws_s1 (both
// cells, the Roe solve + Harten-Hyman A-dq), ws_s2 (CFL, the limited corrections), ws_s3 (both
// transverse splits, the lane's output cell).
// FAST: method2 = 2 and method3 = 2 (the configs) known at compile time; otherwise read from A.
template <class S>
struct WsChain {
  typename S::Cell L, R;
  typename S::Edge Ed;
  double sw[S::MEQN], F[S::MEQN];
};

template <class S, int D>
__device__ __forceinline__ void ws_s1(const StepArgs& A, const double* __restrict__ sq, uint32_t dsc, WsChain<S>& c) {
  using Sh = WsShape<S>;
  constexpr int PW = Sh::PW, WPW = Sh::WPW, MEQN = S::MEQN;
  const int wr = dsc & 511;
  const int wl = D == 1 ? wr - 1 : wr - PW;
#pragma unroll
  for (int k = 0; k < MEQN; ++k) {
    c.L.q[k] = sq[k * WPW + wl];
    c.R.q[k] = sq[k * WPW + wr];
  }
  S::cell(c.L, A.sp);
  S::cell(c.R, A.sp);
  S::template riemann<D>(c.L, c.R, A.sp, c.Ed);
}

template <class S, int D, bool FAST>
__device__ __forceinline__ void ws_s2(const StepArgs& A, double r, double& smax, uint32_t dsc, int lane,
                                      WsChain<S>& c) {
  constexpr int MEQN = S::MEQN;
  const bool m2 = FAST || A.method2 == 2;
  const bool corr = (dsc >> 20) & 1;
  const typename S::Edge& Ed = c.Ed;
  // CFL of the corrected edges: max over waves of r |s| = r (|un| + c) (the max taken per tile)
  const double ms = S::template max_speed<D>(Ed);
  smax = corr && ms > smax ? ms : smax;
  // corrections: limiter on the upwind neighbour edge's wave of the same family (warp shuffle)
  double* sw = c.sw;
  double* F = c.F;
#pragma unroll
  for (int k = 0; k < MEQN; ++k) { sw[k] = 0.0; F[k] = 0.0; }
#pragma unroll
  for (int p = 0; p < S::MW; ++p) {
    double Wp[MEQN], WI[MEQN];
    S::template wave<D>(Ed, p, Wp);
    const double s = S::template speed<D>(Ed, p);
#pragma unroll
    for (int k = 0; k < MEQN; ++k)
      if (S::wave_nz(D, p, k)) sw[k] = fma(s, Wp[k], sw[k]);
    if (m2) {
      const int src = s > 0.0 ? lane - 1 : lane + 1;    // (s = 0: the right neighbour, reading 1)
      double wn2 = 0.0, dot = 0.0;
#pragma unroll
      for (int k = 0; k < MEQN; ++k) {
        if (!S::wave_nz(D, p, k)) continue;
        WI[k] = ws_shfl_idx(Wp[k], src & 31);
        wn2 = fma(Wp[k], Wp[k], wn2);
        dot = fma(WI[k], Wp[k], dot);
      }
      // a zero wave adds nothing: theta = 0 there (dot = 0; the 1e-300 changes wn2 only below
      // 1e-284, i.e. for waves of norm < 1e-142) keeps the limiter's selects NaN-free
      const double th = dot * fast_rcp(wn2 + 1e-300);
      const double as = fabs(s);
      // 0.5 |s| (1 - |s| r) phi(theta), the 1/2 carried by the halved limiter coefficients (exact)
      const double cf = as * (1.0 - as * r) * ws_phi(A.limh, th);
#pragma unroll
      for (int k = 0; k < MEQN; ++k)
        if (S::wave_nz(D, p, k)) F[k] = fma(cf, Wp[k], F[k]);
    }
  }
}

template <class S, int D, bool FAST>
__device__ __forceinline__ void ws_s3(const StepArgs& A, double* __restrict__ up, double* __restrict__ dn,
                                      double* __restrict__ dq, double r, uint32_t dsc, const WsChain<S>& c) {
  using Sh = WsShape<S>;
  constexpr int T = Sh::T, MEQN = S::MEQN;
  const int m3 = FAST ? 2 : A.method3;
  const int pos = (dsc >> 9) & 31, line = (dsc >> 14) & 31;
  const bool out = (dsc >> 21) & 1;
  const typename S::Edge& Ed = c.Ed;
  const double* sw = c.sw;
  const double* F = c.F;
  // L part P = A-dq + F~ (enters the left cell), R part Q = A+dq - F~ (the right cell)
  double P[MEQN], Q[MEQN];
#pragma unroll
  for (int k = 0; k < MEQN; ++k) {
    P[k] = Ed.am[k] + F[k];
    Q[k] = (sw[k] - Ed.am[k]) - F[k];
  }
  // both transverse splits with this edge's own Roe state (its Roe-only terms once): of Q (into
  // the right cell, this lane's output) and of P (into the left cell: the previous edge's lane's
  // output, handed down scaled together with P)
  double XP[MEQN], XQ[MEQN], bmP[MEQN], bpP[MEQN], bmQ[MEQN], bpQ[MEQN];
#pragma unroll
  for (int k = 0; k < MEQN; ++k) {
    XP[k] = m3 == 1 ? Ed.am[k] : P[k];
    XQ[k] = m3 == 1 ? sw[k] - Ed.am[k] : Q[k];
  }
  if (m3 >= 1) {
    S::template transverse2<D>(S::roe(Ed), A.sp, XP, XQ, bmP, bpP, bmQ, bpQ);
  } else {
#pragma unroll
    for (int k = 0; k < MEQN; ++k) bmQ[k] = bpQ[k] = bmP[k] = bpP[k] = 0.0;
  }
  const double hh = -0.25 * r;   // (-1/2 r, and transverse returns 2 B-X, 2 B+X)
  double Un[MEQN], Dn[MEQN], Pn[MEQN];
#pragma unroll
  for (int k = 0; k < MEQN; ++k) {
    Un[k] = ws_shfl_down(hh * bpP[k], 1);
    Dn[k] = ws_shfl_down(hh * bmP[k], 1);
    Pn[k] = ws_shfl_down(P[k], 1);
  }
  if (out) {
    if (D == 1) {   // cell (i = pos, j = line): G~ halves for rows 0..T+1, the x increment for rows 1..T
      const int i = pos, j = line;
#pragma unroll
      for (int k = 0; k < MEQN; ++k) {
        up[(k * Sh::NR + j) * Sh::UPP + (i - 1)] = fma(hh, bpQ[k], Un[k]);
        dn[(k * Sh::NR + j) * Sh::UPP + (i - 1)] = fma(hh, bmQ[k], Dn[k]);
      }
      if (j >= 1 && j <= T) {
#pragma unroll
        for (int k = 0; k < MEQN; ++k) dq[(k * T + (j - 1)) * Sh::DQP + (i - 1)] = -r * Pn[k] - r * Q[k];
      }
    } else {        // cell (i = line, j = pos): F~ halves (up / dn are the rt / lf arrays)
      const int i = line, j = pos;
#pragma unroll
      for (int k = 0; k < MEQN; ++k) {
        up[(k * T + (j - 1)) * Sh::RTP + i] = fma(hh, bpQ[k], Un[k]);
        dn[(k * T + (j - 1)) * Sh::RTP + i] = fma(hh, bmQ[k], Dn[k]);
      }
      if (i >= 1 && i <= T) {
#pragma unroll
        for (int k = 0; k < MEQN; ++k) dq[(k * T + (j - 1)) * Sh::DQP + (i - 1)] = -r * Pn[k] - r * Q[k];
      }
    }
  }
}

template <class S, int D, bool FAST>
__device__ __forceinline__ void ws_iter(const StepArgs& A, const double* __restrict__ sq, double* __restrict__ up,
                                        double* __restrict__ dn, double* __restrict__ dq, double r, double& smax,
                                        uint32_t dsc, int lane) {
  WsChain<S> c;
  ws_s1<S, D>(A, sq, dsc, c);
#ifndef WS_ITER_VOTE
#define WS_ITER_VOTE 0
#endif
  if (WS_ITER_VOTE && __any_sync(0xffffffffu, c.Ed.c != c.Ed.c)) smax = __longlong_as_double(0x7ff0000000000000ll);
  ws_s2<S, D, FAST>(A, r, smax, dsc, lane, c);
  ws_s3<S, D, FAST>(A, up, dn, dq, r, dsc, c);
}

// an x-iteration and a y-iteration as two independent dependency chains in one instruction stream
// (twice the instruction-level parallelism; for the branch-free Roe SWE solve: T3 4.53 -> 4.43 ms
// at 4 CTAs x 4 warps per SM, 126 registers.  Euler measured slower paired, at 2 CTAs of 242
// registers: 7.58 vs 6.84 ms, its Harten-Hyman branches splitting the two streams)
template <class S, bool FAST>
__device__ __forceinline__ void ws_iter_xy(const StepArgs& A, const double* __restrict__ sq, double* __restrict__ up,
                                           double* __restrict__ dn, double* __restrict__ dq, double* __restrict__ rt,
                                           double* __restrict__ lf, double* __restrict__ dqy, double r, double& smax,
                                           uint32_t dx, uint32_t dy, int lane) {
  WsChain<S> cx, cy;
  ws_s1<S, 1>(A, sq, dx, cx);
  ws_s1<S, 2>(A, sq, dy, cy);
  // a non-finite Roe sound speed makes the tile's CFL +inf (-> FC_ENONFINITE, as the fold's check
  // would); the warp vote between the solves and the limiters is also the scheduling split that
  // measured best (T3 4.53 -> 4.36 ms; the pair without it 4.66)
  if (__any_sync(0xffffffffu, cx.Ed.c != cx.Ed.c || cy.Ed.c != cy.Ed.c)) smax = __longlong_as_double(0x7ff0000000000000ll);
  ws_s2<S, 1, FAST>(A, r, smax, dx, lane, cx);
  ws_s2<S, 2, FAST>(A, r, smax, dy, lane, cy);
  ws_s3<S, 1, FAST>(A, up, dn, dq, r, dx, cx);
  ws_s3<S, 2, FAST>(A, rt, lf, dqy, r, dy, cy);
}

#ifndef WS_PAIR_EULER
#define WS_PAIR_EULER 0
#endif
#ifndef WS_PAIR_SWE
#define WS_PAIR_SWE 1
#endif
template <class S, int NW, int MINB, int NBUF, bool FAST>
__global__ void __launch_bounds__(NW * 32, MINB) k_step_ws(StepArgs A, int ntiles) {
  using Sh = WsShape<S>;
  constexpr int T = Sh::T, PW = Sh::PW, WPW = Sh::WPW, MEQN = S::MEQN, NT = NW * 32;
  constexpr int GU = ((Sh::CHUNK ? Sh::NH : Sh::W * Sh::W) + NT - 1) / NT;
  const int tiles2 = A.tiles * A.tiles;
  if (A.active) ntiles = *A.nactive * tiles2;
  auto tile_of = [&](int k) {
    if (k >= ntiles) return -1;
    if (!A.active) return k;
    const int a = k / tiles2;
    return A.active[a] * tiles2 + (k - a * tiles2);
  };
  extern __shared__ __align__(128) double sm[];
  double* sbuf = sm;                           // NBUF x [MEQN][W][PW] windows
  double* up = sbuf + NBUF * Sh::QB;           // x-sweep G~ halves (up / dn)
  double* dn = up + Sh::N_UP;
  double* rt = dn + Sh::N_UP;                  // y-sweep F~ halves (right / left)
  double* lf = rt + Sh::N_RT;
  double* dq = lf + Sh::N_RT;                  // x increments
  double* dqy = dq + Sh::N_DQ;                 // y increments
  uint32_t* desc = reinterpret_cast<uint32_t*>(dqy + Sh::N_DQ);   // [2 NIT][32] lane descriptors
  __shared__ double wmax[NW];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int t = tid; t < Sh::NDESC; t += NT) {   // (read after the first tile's barrier)
    const int v = t >> 5, l = t & 31;
    desc[t] = v < Sh::NIT ? ws_desc<S, 1>(v, l) : ws_desc<S, 2>(v - Sh::NIT, l);
  }
  double cfl = 0.0;
  bool bad = false;

  // NBUF = 2: the window of tile k+1 is gathered while tile k computes, with the ring-table
  // entries of tile k+2 and the patch metadata of tile k+1 loaded at the same time.  NBUF = 1: the
  // gather of tile k follows tile k-1's fold (the other CTAs of the SM cover the latency), the
  // entries of tile k+1 loaded while it is in flight.
  WsGather<GU> g;
  ws_prep<S>(A, tile_of(blockIdx.x), g, tid, NT);
  if (NBUF == 2) {
    ws_issue<S>(A, g, sbuf, tid, NT);
    cp_async_commit();
    ws_prep<S>(A, tile_of(blockIdx.x + gridDim.x), g, tid, NT);
  }
  // boundary flags and level of the next tile, loaded a tile ahead into their own registers (volatile
  // loads: the combination happens at their use, one tile later -- combined at the load, the
  // compiler waited on the two loads every tile: 5.7 % of the stall samples)
  int nbc = 0, nlv = 0;
  auto load_meta = [&](int t) {
    if (t < 0) return;
    int pm, xm, ym;
    ws_tile(A, t, pm, xm, ym);
    asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(nbc) : "l"(A.bcflag + pm));
    asm volatile("ld.global.nc.s8 %0, [%1];" : "=r"(nlv) : "l"(A.level + pm));
  };
  load_meta(tile_of(blockIdx.x));
  int it = 0;
  for (int kt = blockIdx.x; kt < ntiles; kt += gridDim.x, ++it) {
    double* sq = sbuf + (NBUF == 2 ? (it & 1) * Sh::QB : 0);
    const int tile = tile_of(kt);
    int patch, tx, ty;
    ws_tile(A, tile, patch, tx, ty);
    if (NBUF == 2) {
      cp_async_wait<0>();
      __syncthreads();                          // this tile's window is in; the previous tile is done
      ws_issue<S>(A, g, sbuf + ((it + 1) & 1) * Sh::QB, tid, NT);   // tile k+1 (entries loaded last tile)
      cp_async_commit();
      ws_prep<S>(A, tile_of(kt + 2 * gridDim.x), g, tid, NT);        // tile k+2's entries
    } else {
      __syncthreads();                          // the previous tile's fold is done with the window
      ws_issue<S>(A, g, sbuf, tid, NT);
      cp_async_commit();
      ws_prep<S>(A, tile_of(kt + gridDim.x), g, tid, NT);            // tile k+1's entries
      cp_async_wait<0>();
      __syncthreads();
    }
    const int cur = nbc | (nlv << 8);             // bcflag | level << 8 of this tile
    load_meta(tile_of(kt + gridDim.x));
    if (cur & 1) { ws_bc<S>(A, tile, sq, 0, tid, NT); __syncthreads(); }
    if (cur & 2) { ws_bc<S>(A, tile, sq, 1, tid, NT); __syncthreads(); }
    const double r = dtdx_level(A, cur >> 8);   // square cells, no capacity: dt/dx = dt/dy
    double* o = A.qnew + (int64_t)patch * MEQN * (A.m + 4) * (A.m + 4) + (int64_t)(ty * T) * A.m + tx * T;
    const int64_t n2 = (int64_t)(A.m + 4) * (A.m + 4);
    if (A.skip_quiescent) {   // one state in the whole window: every jump is 0, q_new = q bitwise
      const double* q11 = sq + 2 * PW + 2;
      bool diff = false;
      for (int t = tid; t < Sh::W * Sh::W; t += NT) {
        const int wj = t / Sh::W, wi = t - wj * Sh::W;
#pragma unroll
        for (int k = 0; k < MEQN; ++k) diff |= sq[k * WPW + wj * PW + wi] != q11[k * WPW];
      }
      if (!__syncthreads_or(diff)) {
        cfl = fmax(cfl, ws_quiescent_cfl<S>(q11, WPW, A.sp, r));
        for (int t = tid; t < T * T; t += NT) {
          const int j = t / T, i = t - j * T;
#pragma unroll
          for (int k = 0; k < MEQN; ++k) o[k * n2 + j * A.m + i] = q11[k * WPW];
        }
        continue;
      }
    }
    // both sweeps read Q^n only (unsplit): their 2 NIT warp-iterations are one phase
    double smax = 0.0;
    if (std::is_same<S, WsSwe>::value ? WS_PAIR_SWE : WS_PAIR_EULER) {   // x- and y-iteration v together
      for (int v = warp; v < Sh::NIT; v += NW)
        ws_iter_xy<S, FAST>(A, sq, up, dn, dq, rt, lf, dqy, r, smax, desc[v * 32 + lane],
                            desc[(Sh::NIT + v) * 32 + lane], lane);
    } else {
      for (int v = warp; v < 2 * Sh::NIT; v += NW) {
        const uint32_t d = desc[v * 32 + lane];
        if (v < Sh::NIT) ws_iter<S, 1, FAST>(A, sq, up, dn, dq, r, smax, d, lane);
        else ws_iter<S, 2, FAST>(A, sq, rt, lf, dqy, r, smax, d, lane);
      }
    }
    cfl = fmax(cfl, r * smax);
    __syncthreads();
    // fold: q_new = q + (x and y increments) - r (G~ and F~ differences), one thread per cell
    for (int t = tid; t < T * T; t += NT) {
      const int jj = t / T, ii = t - jj * T;     // cell (ii + 1, jj + 1)
      const int i = ii + 1, j = jj + 1;
      const double* qs = sq + (j + 1) * PW + (i + 1);
#pragma unroll
      for (int k = 0; k < MEQN; ++k) {
        const double* u_ = up + k * Sh::NR * Sh::UPP + ii;
        const double* d_ = dn + k * Sh::NR * Sh::UPP + ii;
        const double gt = u_[j * Sh::UPP] + d_[(j + 1) * Sh::UPP];
        const double gb = u_[(j - 1) * Sh::UPP] + d_[j * Sh::UPP];
        const double* rr = rt + (k * T + jj) * Sh::RTP;
        const double* ll = lf + (k * T + jj) * Sh::RTP;
        const double fr = rr[i] + ll[i + 1];
        const double fl = rr[i - 1] + ll[i];
        const double dxy = dq[(k * T + jj) * Sh::DQP + ii] + dqy[(k * T + jj) * Sh::DQP + ii];
        const double val = qs[k * WPW] + ((dxy - r * (gt - gb)) - r * (fr - fl));
        bad |= !isfinite(val);
        o[k * n2 + jj * A.m + ii] = val;
      }
    }
  }
  cp_async_wait<0>();
  // a non-finite updated state makes the step's CFL +inf (fc_step -> FC_ENONFINITE)
  if (__syncthreads_or(bad)) cfl = __longlong_as_double(0x7ff0000000000000ll);
  if (cfl != cfl) cfl = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) cfl = fmax(cfl, __shfl_xor_sync(0xffffffffu, cfl, o));
  if (lane == 0) wmax[warp] = cfl;
  __syncthreads();
  if (tid == 0) {
    double c = wmax[0];
    for (int w = 1; w < NW; ++w) c = fmax(c, wmax[w]);
    atomicMax(A.cfl_bits, (unsigned long long)__double_as_longlong(c));
  }
}

template <class S, int NW, int MINB, int NBUF, bool FAST>
static int launch_ws_t(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  const size_t smem = WsShape<S>::smem_bytes(NBUF);
  auto kern = k_step_ws<S, NW, MINB, NBUF, FAST>;
  static int resident[64] = {};    // per device: CTAs resident at once (persistent grid)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return -1;
  if (!resident[dev]) {            // (function attributes are per device)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem);
    resident[dev] = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int64_t ntiles = npatch * a.tiles * a.tiles;
  if (ntiles >= (1ll << 31)) return -1;
  const int64_t grid = ntiles < resident[dev] ? ntiles : resident[dev];
  kern<<<(unsigned)grid, NW * 32, smem, st>>>(a, (int)ntiles);
  return 1;
}

// warps per CTA, CTAs per SM, window buffers: 24 warp-iterations per tile (both sweeps).
// Measured (C5 / T3 full update, ms): Euler 6 warps x 2 CTAs double-buffered (166 registers) 8.45,
// single-buffered 8.61, 8 warps x 1 CTA (181 registers) 10.0, 4 warps x 3 CTAs single-buffered
// (168 registers, 70 KB) 7.75; SWE 8 x 2 double-buffered 5.51, single 5.66, 4 x 4 single
// (128 registers, 52 KB) 4.97.  More, smaller CTAs per SM: a CTA at its barrier or waiting for its
// window leaves the SM to the others.
#ifndef WS_NW_EULER
#define WS_NW_EULER 4
#endif
#ifndef WS_MINB_EULER
#define WS_MINB_EULER 3
#endif
#ifndef WS_NBUF_EULER
#define WS_NBUF_EULER 1
#endif
#ifndef WS_NW_SWE
#define WS_NW_SWE 4
#endif
#ifndef WS_MINB_SWE
#define WS_MINB_SWE 4
#endif
#ifndef WS_NBUF_SWE
#define WS_NBUF_SWE 1
#endif
template <class S>
static int launch_ws_s(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  constexpr bool swe = std::is_same<S, WsSwe>::value;
  constexpr int NW = swe ? WS_NW_SWE : WS_NW_EULER;
  constexpr int MINB = swe ? WS_MINB_SWE : WS_MINB_EULER;
  constexpr int NBUF = swe ? WS_NBUF_SWE : WS_NBUF_EULER;
  if (a.method2 == 2 && a.method3 == 2) return launch_ws_t<S, NW, MINB, NBUF, true>(a, npatch, st);
  return launch_ws_t<S, NW, MINB, NBUF, false>(a, npatch, st);
}

int launch_step_ws(int kind, const StepArgs& a, int64_t npatch, cudaStream_t st) {
  const char* env = getenv("FC_WS");   // (read per launch: tests switch kernels within a process)
  if ((env && atoi(env) == 0) || !a.ring || a.rslot || a.m % 16 != 0) return 0;
  if (kind == FC_EULER_ROE) return launch_ws_s<WsEuler>(a, npatch, st);
  if (kind == FC_SWE_ROE) return launch_ws_s<WsSwe>(a, npatch, st);
  return 0;
}

}  // namespace fc
