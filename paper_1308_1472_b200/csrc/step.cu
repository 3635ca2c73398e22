// step.cu -- the fused wave-propagation step kernel (libfc, sm_100a, fp64).
//
// PAPER.md:168-182 [§3]: Clawpack's wave propagation on one uniform patch -- Riemann problems at
// every edge, left/right-going waves, a wave limiter, second-order corrections; transverse
// (rpt2) corrections of the unsplit 2D method (readings in DESIGN.md).
//
// Layout: one CTA per T x T tile of a patch (T = 16 for m = 16, 32, ...; 8 for m = 8, ...); the
// update of a cell reads only its 2-cell neighbourhood, so tiles of a patch are independent and
// exact.  The tile plus its 2-cell halo (W = T + 4) is staged in shared memory from the padded
// patch (ring filled by the ghost kernels).  Phases (one barrier between each):
//   P   per-cell derived fields (sqrt(rho), u, v, H, c ...) for all W^2 staged cells
//   X1  normal Riemann solve on all (T+3)(T+2) x-edges -> compact per-edge scratch
//   X2  for the (T+1)(T+2) x-edges with corrections: limiter (upwind neighbour's unlimited wave),
//       F~, CFL, L = A-dq + F~ / R = A+dq - F~, transverse splits B-+(L), B-+(R).  Each cell
//       receives exactly one L part (from its right edge) and one R part (its left edge): L parts
//       are stored with '=', then after a barrier R parts with '+=' -- no atomics, no zero fill.
//   X3  fold G~ (transverse of the x-sweep) into the cell increments
//   Y1/Y2 the same along y (reading Q^n: unsplit), transverse into F~ at x-edges
//   Y3  fold F~ transverse, q_new = q + dq, non-finite check, CFL block max -> one atomicMax.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "../../include/fc.h"
#include "fc_internal.h"
#include "solvers.cuh"
#include "step_common.cuh"
#include "step_ws.cuh"

namespace fc {

template <class S, int T>
struct StepShape {
  static constexpr int W = T + 4;
  static constexpr int WW = W * W;
  static constexpr int EX = (T + 3) * (T + 2);   // edges per sweep (incl. limiter neighbours)
  static constexpr int E2 = (T + 1) * (T + 2);   // edges with corrections / transverse
  static constexpr int NTR = S::MEQN * T * (T + 2);
  // one staged tile: q [MEQN][W][W] (+2 doubles: the single-copy whole-patch staging lands at +2,
  // see stage_tile) then aux [3][W][W] at offset MEQN WW + 2
  static constexpr int BUF = S::MEQN * WW + 2 + (S::CAPA ? 3 : 0) * WW;
  static constexpr size_t smem_doubles = (size_t)2 * BUF + (size_t)S::NC * WW + (size_t)S::NSA * EX +
                                         (size_t)S::MEQN * E2 + S::MEQN * T * T + 2 * NTR;
  static constexpr size_t smem_bytes = smem_doubles * sizeof(double);
};

// Phase 2a of a sweep, one correction edge: fluctuations A-+dq, second-order correction F~ (MC /
// minmod limiter on the upwind neighbour's *unlimited* wave) and the edge CFL.
// Waves are reconstructed one at a time from the compact scratch (no wave array stays live):
// A-dq = sum_p min(s_p,0) W_p, A+dq = sum_p max(s_p,0) W_p, or, for Euler, A-dq is the Harten-Hyman
// fixed value stored by the normal solve and A+dq = sum_p s_p W_p - A-dq.  Out: P = A-dq + F~ (the
// edge's L part, entering the cell on its low side), Q = A+dq - F~ (R part), F = F~.
template <class S, int D>
__device__ __forceinline__ void edge_correction(const double* sc, const double* scm, const double* scp,
                                                int st, const StepArgs& A, AuxCell ar, double rl, double rr,
                                                double& cfl, double* P, double* Q, double* F) {
  constexpr int MEQN = S::MEQN;
  if constexpr (MEQN == 1 && S::MW == 1) {
    // scalar: the limited correction phi(W_I / W) W evaluated division-free as
    // sign(W) min(|c1 W + c2 W_I|, c3 |W|, c4 |W_I|) when W and W_I share a sign (else lo W) --
    // equal in exact arithmetic; the phased kernel is issue-bound on scalars, so the reciprocal's
    // MUFU + Newton steps per edge are worth removing
    const double W = sc[0];
    const double s = S::template speed<D>(sc, st, 0, A.sp, ar);
    cfl = fmax(cfl, fmax(rr * s, -rl * s));
    double sm, sp;
    split0(s, sm, sp);
    double f = 0.0;
    if (A.method2 == 2 && W != 0.0) {
      const double WI = (s > 0.0 ? scm : scp)[0];
      const LimiterCoef& L = A.lim;
      double phiw;
      if (L.lo == 1.0) {
        phiw = W;
      } else if ((W > 0.0 && WI > 0.0) || (W < 0.0 && WI < 0.0)) {
        const double mag = fmin(fmin(fabs(fma(L.c1, W, L.c2 * WI)), L.c3 * fabs(W)), L.c4 * fabs(WI));
        phiw = W > 0.0 ? mag : -mag;
      } else {
        phiw = 0.0;
      }
      const double as = fabs(s), rav = 0.5 * (rl + rr);
      f = 0.5 * as * (1.0 - as * rav) * phiw;
    }
    F[0] = f;
    P[0] = sm * W + f;
    Q[0] = sp * W - f;
    return;
  }
  double am[MEQN], ap[MEQN];
#pragma unroll
  for (int k = 0; k < MEQN; ++k) {
    am[k] = 0.0;   // (Euler: the stored A-dq is read after the wave loop, fewer live registers)
    ap[k] = 0.0;
    F[k] = 0.0;
  }
  const double rav = 0.5 * (rl + rr);
#pragma unroll
  for (int p = 0; p < S::MW; ++p) {
    double W[MEQN];
    S::template wave<D>(sc, st, p, A.sp, W);
    const double s = S::template speed<D>(sc, st, p, A.sp, ar);
    cfl = fmax(cfl, fmax(rr * s, -rl * s));
    if (S::AM_STORED) {
#pragma unroll
      for (int k = 0; k < MEQN; ++k) ap[k] = fma(s, W[k], ap[k]);
    } else {
      double sm, sp;
      split0(s, sm, sp);
#pragma unroll
      for (int k = 0; k < MEQN; ++k) { am[k] = fma(sm, W[k], am[k]); ap[k] = fma(sp, W[k], ap[k]); }
    }
    if (A.method2 == 2) {
      double WI[MEQN];
      S::template wave<D>(s > 0.0 ? scm : scp, st, p, A.sp, WI);
      double wn2 = W[0] * W[0], dot = WI[0] * W[0];
#pragma unroll
      for (int k = 1; k < MEQN; ++k) { wn2 = fma(W[k], W[k], wn2); dot = fma(WI[k], W[k], dot); }
      if (wn2 != 0.0) {   // a zero wave adds nothing (also skips the limiter in quiescent flow)
        const double phi = limiter_phi(A.lim, dot * fast_rcp(wn2));
        const double as = fabs(s);
        const double c = 0.5 * as * (1.0 - as * rav) * phi;
#pragma unroll
        for (int k = 0; k < MEQN; ++k) F[k] = fma(c, W[k], F[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < MEQN; ++k) {
    if (S::AM_STORED) {
      am[k] = sc[(S::PB + k) * st];
      ap[k] -= am[k];
    }
    P[k] = am[k] + F[k];
    Q[k] = ap[k] - F[k];
  }
}

// transverse split of X = A-+dq (+-F~ for method3 = 2) entering `recv`
template <class S, int D>
__device__ __forceinline__ void edge_transverse(const double* sc, int st, const StepArgs& A, const double* X,
                                                AuxCell recv, AuxCell next, double* bm, double* bp) {
  if (A.method3 >= 1) {
    S::template transverse<D>(sc, st, A.sp, X, recv, next, bm, bp);
  } else {
#pragma unroll
    for (int k = 0; k < S::MEQN; ++k) bm[k] = bp[k] = 0.0;
  }
}

// issue the bulk copies staging tile `tile` (q window + aux window) into buf, on barrier bar.
// Called by all 32 lanes of warp 0: lane 0 arms the barrier, the lanes split the row copies.
// Issued by `nthr` threads (thread `lane` of them): one warp for the single-copy staging, the whole
// CTA when the window comes in many row pieces (multi-tile patches, fused ring rows) -- a lone warp
// issuing ~60-180 row copies per tile held the CTA at its next barrier (T3: 55 % barrier stalls).
// Thread 0 arms the barrier with the window's bytes; the copies may complete before or after.
template <class S, int T>
__device__ __forceinline__ void stage_tile(const StepArgs& A, int tile, double* buf, uint64_t* bar,
                                           int lane, int nthr = 32) {
  using Sh = StepShape<S, T>;
  constexpr int MEQN = S::MEQN, W = Sh::W, WW = Sh::WW;
  int patch = tile, tx = 0, ty = 0;
  if (A.tiles > 1) {
    const int tiles2 = A.tiles * A.tiles;
    patch = tile / tiles2;
    const int t = tile - patch * tiles2;
    ty = t / A.tiles;
    tx = t - ty * A.tiles;
  }
  const int n = A.m + 4, n2 = n * n;
  if (A.ring && A.tiles > 1) {   // fused ring gather, multi-tile patch: the window's part inside the
                                 // patch interior by row copies (16-byte aligned: m, T even), the
                                 // rest by gather_ring_tiles (constant-aux forms only)
    const int m = A.m;
    const int i_lo = max(1, tx * T - 1), i_hi = min(m, tx * T + T + 2);
    const int j_lo = max(1, ty * T - 1), j_hi = min(m, ty * T + T + 2);
    const int L = i_hi - i_lo + 1, R = j_hi - j_lo + 1;
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)(MEQN * R * L) * (uint32_t)sizeof(double));
    const double* qb = A.qold + (int64_t)patch * MEQN * n2;
#pragma unroll 1
    for (int r = lane; r < MEQN * R; r += nthr) {
      const int k = r / R, j = j_lo + (r - k * R);
      bulk_g2s(buf + k * WW + (j - ty * T + 1) * W + (i_lo - tx * T + 1), qb + (int64_t)k * n2 + (j - 1) * m + (i_lo - 1),
               L * sizeof(double), bar);
    }
    return;
  }
  if (A.ring) {              // fused ring gather: the TMA brings the m x m interior rows only
    constexpr uint32_t qbytes = (uint32_t)MEQN * T * T * sizeof(double);
    constexpr uint32_t abytes = S::CAPA ? (uint32_t)3 * WW * sizeof(double) : 0u;
    if (lane == 0) mbar_expect_tx(bar, qbytes + abytes);
    const double* qb = A.qold + (int64_t)patch * MEQN * n2;
#pragma unroll 1
    for (int r = lane; r < MEQN * T; r += nthr) {
      const int k = r / T, row = r - k * T;
      // storage (qcell): the interior is dense, row `row` at row * m
      bulk_g2s(buf + k * WW + (row + 2) * W + 2, qb + (int64_t)k * n2 + row * T, T * sizeof(double), bar);
    }
    if (S::CAPA && lane == 0) bulk_g2s(buf + MEQN * WW + 2, A.aux + (int64_t)patch * 3 * n2, abytes, bar);
    return;
  }
  constexpr uint32_t bytes = (uint32_t)(Sh::BUF - 2) * sizeof(double);
  if (lane == 0) mbar_expect_tx(bar, bytes);
  if (A.tiles == 1) {        // the window is the whole padded patch: one contiguous copy of its
                             // storage blocks (dense interior + ring, qcell); the kernel reads them
                             // through qidx
    if (lane == 0) bulk_g2s(buf, A.qold + patch * (int64_t)MEQN * n2, MEQN * WW * sizeof(double), bar);
  } else {                   // q: per (component, window row): a ghost row is one piece of the ring
                             // area; an interior row is its interior run plus the ghost pair of an
                             // edge tile (ring area) -- into the natural window
    const int m = A.m, mm = m * m;
    const double* qb = A.qold + patch * (int64_t)MEQN * n2;
#pragma unroll 1
    for (int r = lane; r < MEQN * W; r += nthr) {
      const int k = r / W, b = r - k * W;
      const int j = ty * T + b - 1, i0 = tx * T - 1;
      const double* blk = qb + (int64_t)k * n2;
      double* dst = buf + r * W;
      if (j <= 0 || j > m) {
        bulk_g2s(dst, blk + mm + ring_index(i0, j, m), W * sizeof(double), bar);
      } else {
        const int ia = i0 < 1 ? 1 : i0, ib = i0 + W - 1 > m ? m : i0 + W - 1;   // interior run
        bulk_g2s(dst + (ia - i0), blk + (j - 1) * m + (ia - 1), (ib - ia + 1) * sizeof(double), bar);
        if (i0 < 1) bulk_g2s(dst, blk + mm + ring_index(-1, j, m), 2 * sizeof(double), bar);
        if (i0 + W - 1 > m) bulk_g2s(dst + (m + 1 - i0), blk + mm + ring_index(m + 1, j, m), 2 * sizeof(double), bar);
      }
    }
  }
  if (A.tiles == 1) {        // aux (natural layout): the window is the whole padded patch
    if (S::CAPA && lane == 1) bulk_g2s(buf + MEQN * WW + 2, A.aux + patch * 3ll * n2, 3 * WW * sizeof(double), bar);
  } else {
    if (S::CAPA) {
      const double* ab = A.aux + patch * 3ll * n2 + (int64_t)(ty * T) * n + tx * T;
#pragma unroll 1
      for (int r = lane; r < 3 * W; r += nthr) {
        const int k = r / W, b = r - k * W;
        bulk_g2s(buf + MEQN * WW + 2 + r * W, ab + (int64_t)k * n2 + b * n, W * sizeof(double), bar);
      }
    }
  }
}

template <class S, int T, int NT>
__device__ __forceinline__ void gather_ring_tiles(const StepArgs& A, int tile, double* buf);
template <class S, int T, int NT>
__device__ __forceinline__ void window_bc_tiles(const StepArgs& A, int tile, double* sq, int is_y);

// issue the cp.async copies of the ring cells of `tile` (COPY sources) into buf; one group
template <class S, int T, int NT>
__device__ __forceinline__ void gather_ring(const StepArgs& A, int tile, double* buf) {
  if (A.tiles > 1) { gather_ring_tiles<S, T, NT>(A, tile, buf); return; }
  using Sh = StepShape<S, T>;
  constexpr int MEQN = S::MEQN, WW = Sh::WW, G = WW - T * T;
  const int n2 = WW;
  const int32_t* rs = A.ring + (int64_t)tile * G;
  const uint8_t* rp = A.rpeer ? A.rpeer + (int64_t)tile * G : nullptr;
  for (int e = opaque(threadIdx.x); e < G * MEQN; e += NT) {
    const int k = e / G, r = e - k * G;
    const int32_t v = __ldg(rs + r);
    if (v >= 0) {
      // peer-memory halo: a cell of another rank is copied straight from its buffer over NVLink
      const int ow = rp ? __ldg(rp + r) : 0;
      const double* base = ring_base(A, ow);
      cp_async8(buf + k * WW + ring_window_index<T>(r), base + v + (int64_t)k * n2);
    }
  }
}

// multi-tile patches (m = tiles x T): the window cells outside the patch interior are ring cells of
// the patch; copy their sources (the patch's ring table), physical-boundary ones after the gather
template <class S, int T, int NT>
__device__ __forceinline__ void gather_ring_tiles(const StepArgs& A, int tile, double* buf) {
  constexpr int MEQN = S::MEQN, W = T + 4, WW = W * W;
  const int m = A.m, n = m + 4, n2 = n * n, G = n2 - m * m, tiles2 = A.tiles * A.tiles;
  const int patch = tile / tiles2, tt = tile - patch * tiles2, ty = tt / A.tiles, tx = tt - ty * A.tiles;
  const int32_t* rs = A.ring + (int64_t)patch * G;
  const uint8_t* rp = A.rpeer ? A.rpeer + (int64_t)patch * G : nullptr;
  for (int e = opaque(threadIdx.x); e < WW; e += NT) {
    const int i = tx * T + e % W - 1, j = ty * T + e / W - 1;
    if (i >= 1 && i <= m && j >= 1 && j <= m) continue;        // (row copies)
    const int r = ring_index(i, j, m);
    const int32_t v = __ldg(rs + r);
    if (v < 0) continue;                                        // (physical boundary: window_bc_tiles)
    const double* base = ring_base(A, rp ? __ldg(rp + r) : 0);
#pragma unroll
    for (int k = 0; k < MEQN; ++k) cp_async8(buf + k * WW + e, base + v + (int64_t)k * n2);
  }
}

template <class S, int T, int NT>
__device__ __forceinline__ void window_bc_tiles(const StepArgs& A, int tile, double* sq, int is_y) {
  constexpr int MEQN = S::MEQN, W = T + 4, WW = W * W;
  const int m = A.m, n = m + 4, n2 = n * n, G = n2 - m * m, tiles2 = A.tiles * A.tiles;
  const int patch = tile / tiles2, tt = tile - patch * tiles2, ty = tt / A.tiles, tx = tt - ty * A.tiles;
  const int32_t* rs = A.ring + (int64_t)patch * G;
  for (int e = opaque(threadIdx.x); e < WW; e += NT) {
    const int i = tx * T + e % W - 1, j = ty * T + e / W - 1;
    if (i >= 1 && i <= m && j >= 1 && j <= m) continue;
    const int32_t v = __ldg(rs + ring_index(i, j, m));
    if (v >= 0) continue;
    const int code = -1 - v;
    if ((code & 1) != is_y) continue;
    const int src = code >> 3, neg = (code >> 1) & 3;
    const int si = src % n - 1, sj = src / n - 1;               // the patch cell it copies (natural)
    const int ws = (sj - ty * T + 1) * W + (si - tx * T + 1);   // (within 2 cells: inside this window)
#pragma unroll
    for (int k = 0; k < MEQN; ++k) {
      const double x = sq[k * WW + ws];
      sq[k * WW + e] = (neg != 0 && k == neg) ? -x : x;
    }
  }
}

// physical-boundary ring cells of the staged window, x faces (is_y = 0) then y faces (is_y = 1)
template <class S, int T, int NT>
__device__ __forceinline__ void window_bc(const StepArgs& A, int tile, double* sq, int is_y) {
  if (A.tiles > 1) { window_bc_tiles<S, T, NT>(A, tile, sq, is_y); return; }
  using Sh = StepShape<S, T>;
  constexpr int MEQN = S::MEQN, WW = Sh::WW, G = WW - T * T;
  const int32_t* rs = A.ring + (int64_t)tile * G;
  for (int r = opaque(threadIdx.x); r < G; r += NT) {
    const int32_t v = __ldg(rs + r);
    if (v >= 0) continue;
    const int code = -1 - v;
    if ((code & 1) != is_y) continue;
    const int src = code >> 3, neg = (code >> 1) & 3, dst = ring_window_index<T>(r);
#pragma unroll
    for (int k = 0; k < MEQN; ++k) {
      const double x = sq[k * WW + src];
      sq[k * WW + dst] = (neg != 0 && k == neg) ? -x : x;
    }
  }
}

// Persistent CTAs: each loops over tiles blockIdx.x, + gridDim.x, ...; the next tile's window is
// bulk-copied (TMA engine) into the other staging buffer while the current one is computed.
// register cap for MINB resident CTAs of NT threads.  Registers are split between the 4 SM
// sub-partitions: the one holding ceil(warps / 4) warps bounds the per-thread count (8-register units)
constexpr int step_maxnreg(int nt, int minb) {
  return (16384 / (((nt * minb / 32) + 3) / 4 * 32)) / 8 * 8 > 255 ? 255
                                                                 : (16384 / (((nt * minb / 32) + 3) / 4 * 32)) / 8 * 8;
}

template <class S, int T, int NT, int MINB, bool RF>
__global__ void __launch_bounds__(NT) __maxnreg__(step_maxnreg(NT, MINB)) k_step(StepArgs A, int ntiles) {
  using Sh = StepShape<S, T>;
  constexpr int MEQN = S::MEQN, W = Sh::W, WW = Sh::WW, EX = Sh::EX, E2 = Sh::E2;
  static_assert(E2 <= NT && T * (T + 2) <= NT, "one round of edges / receiving cells per phase");
  const int tiles2_ = A.tiles * A.tiles;
  if (A.active) ntiles = *A.nactive * tiles2_;   // the tiles of the active patches only
  auto tile_of = [&](int k) {
    if (!A.active) return k;
    const int a = k / tiles2_;
    return A.active[a] * tiles2_ + (k - a * tiles2_);
  };
  extern __shared__ __align__(128) double sm[];
  double* sbuf = sm;                                 // 2 x [MEQN + 3 aux][W][W] staging buffers
  double* scl = sbuf + 2 * Sh::BUF;                  // [NC][W][W] per-cell derived fields
  double* scr = scl + S::NC * WW;                    // [NSA][EX] per-edge scratch
  double* qrp = scr + S::NSA * EX;                   // [MEQN][E2] per-edge R part (A+dq - F~)
  double* dq = qrp + MEQN * E2;                      // [MEQN][T][T]
  double* ta = dq + MEQN * T * T;                    // x: up / y: right
  double* tb = ta + Sh::NTR;                         // x: down / y: left
  double* fb = A.fbuf ? A.fbuf + (int64_t)blockIdx.x * MEQN * E2 : nullptr;
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ double wmax[(NT + 31) / 32];

  const int tid = threadIdx.x;
  const int tiles2 = A.tiles * A.tiles;
  const int n = A.m + 4, n2 = n * n;
  const bool dense = !A.ring && A.tiles == 1;   // staged window = storage blocks (see stage_tile)
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_proxy_async();
  }
  __syncthreads();
  const bool wide = A.ring || A.tiles > 1;          // many row pieces: the whole CTA issues them,
  const int sid = wide ? (tid & 31) * (NT / 32) + (tid >> 5) : tid;   // consecutive rows on different warps
  if ((tid < 32 || wide) && (int)blockIdx.x < ntiles)
    stage_tile<S, T>(A, tile_of(blockIdx.x), sbuf, &bars[0], sid, wide ? NT : 32);
  if (A.ring) {
    if ((int)blockIdx.x < ntiles) gather_ring<S, T, NT>(A, tile_of(blockIdx.x), sbuf);
    cp_async_commit();
  }
  uint32_t phase = 0;   // bit b = parity to wait for on buffer b
  double cfl = 0.0;
  bool bad = false;

  int it = 0;
  for (int kt = blockIdx.x; kt < ntiles; kt += gridDim.x, ++it) {
    const int b = it & 1;
    const int tile = tile_of(kt);
    const int knext = kt + gridDim.x;
    // Staging of the next tile into the other buffer.  That buffer was read by the previous tile up
    // to its last phase, so this is issued right after this tile's first barrier (every thread has
    // left the previous tile by then); no end-of-tile barrier is needed.
    bool issued = false;
    auto issue_next = [&]() {
      if (issued) return;
      issued = true;
      if ((tid < 32 || wide) && knext < ntiles) {
        fence_proxy_async();
        stage_tile<S, T>(A, tile_of(knext), sbuf + (b ^ 1) * Sh::BUF, &bars[b ^ 1], sid, wide ? NT : 32);
      }
      if (A.ring) {                    // this thread's ring cells of the next tile: one cp.async group
        if (knext < ntiles) gather_ring<S, T, NT>(A, tile_of(knext), sbuf + (b ^ 1) * Sh::BUF);
        cp_async_commit();
      }
    };
    double* sq = sbuf + b * Sh::BUF;                 // [MEQN][W][W]
    double* sa = sq + MEQN * WW + 2;                 // [3][W][W] aux (capacity form)
    int patch = tile, tx = 0, ty = 0;
    if (A.tiles > 1) {
      patch = tile / tiles2;
      const int tt = tile - patch * tiles2;
      ty = tt / A.tiles;
      tx = tt - ty * A.tiles;
    }
    const double dx = ldexp(A.dx0, -(int)A.level[patch]);
    // coarse/fine reflux: this patch records the fluxes it applies through its 4 faces
    const int slot = RF ? A.rslot[patch] : -1;   // RF: compiled with the reflux records
    auto reg = [&](int face, int e) { return A.freg + (((int64_t)slot * 4 + face) * A.m + e) * MEQN; };
    const double dtdx = A.dt / dx;   // square cells: dt/dy = dt/dx
    mbar_wait(&bars[b], (phase >> b) & 1u);
    phase ^= 1u << b;
    if (A.ring) {                      // this tile's ring: wait for this thread's copies, make every
      cp_async_wait<0>();              // thread's copies visible, then the BCs
      __syncthreads();
      issue_next();
      const uint8_t bc = A.bcflag[patch];
      if (bc & 1) { window_bc<S, T, NT>(A, tile, sq, 0); __syncthreads(); }
      if (bc & 2) { window_bc<S, T, NT>(A, tile, sq, 1); __syncthreads(); }
    }

    auto widx = [](int i, int j) { return (j + 1) * W + (i + 1); };   // tile-local 1-based cell
    // staged-q index: the single-copy staging (dense) keeps the storage blocks (qcell)
    auto qidx = [&](int i, int j) {
      if (!dense) return widx(i, j);
      if ((unsigned)(i - 1) < (unsigned)T && (unsigned)(j - 1) < (unsigned)T) return (j - 1) * T + (i - 1);
      return T * T + ring_index(i, j, T);
    };
    auto auxc = [&](int i, int j) { return AuxCell{sa + widx(i, j), WW}; };
    auto rcell = [&](int i, int j) { return S::CAPA ? dtdx / sa[widx(i, j)] : dtdx; };

    // Quiescent tile: if every staged cell (interior + 2-cell halo) holds the same state, every
    // Riemann problem of the tile has a zero jump, so all waves, fluctuations, corrections and
    // transverse terms are exactly 0 and q_new = q bitwise (the oracle computes q - 0 - 0).  Only
    // the CFL remains: the max over the tile's edges of the wave speeds, taken from the state.
    if (A.skip_quiescent && !(RF && slot >= 0)) {
      bool diff = false;
      for (int t = opaque(threadIdx.x); t < MEQN * WW; t += NT) diff |= sq[t] != sq[(t / WW) * WW + qidx(1, 1)];
      const bool uniform = !__syncthreads_or(diff);
      issue_next();
      if (uniform) {
        cfl = fmax(cfl, S::quiescent_cfl(sq + qidx(1, 1), WW, A.sp, sa, dtdx, T, W, opaque(threadIdx.x), NT));
        const int t = opaque(threadIdx.x);
        if (t < T * T) {
          const int i = 1 + t % T, j = 1 + t / T;
          double* o = A.qnew + patch * (int64_t)MEQN * n2 + (int64_t)(ty * T + j - 1) * A.m + tx * T + i - 1;
#pragma unroll
          for (int k = 0; k < MEQN; ++k) o[(int64_t)k * n2] = sq[k * WW + qidx(1, 1)];
        }
        continue;
      }
    }

    if (S::NC > 0) {
      const int tid = opaque(threadIdx.x);
      for (int t = tid; t < WW; t += NT) S::precompute(sq + qidx(t % W - 1, t / W - 1), WW, A.sp, scl + t, WW);
      __syncthreads();
      issue_next();
    }
    // =============================== x-sweep ===============================
    for (int e = opaque(threadIdx.x); e < EX; e += NT) {       // edge i (cells i-1 | i), row j
      const int i = e % (T + 3), j = e / (T + 3);
      double ql[MEQN], qr[MEQN];
#pragma unroll
      for (int k = 0; k < MEQN; ++k) { ql[k] = sq[k * WW + qidx(i - 1, j)]; qr[k] = sq[k * WW + qidx(i, j)]; }
      S::template riemann<1>(ql, qr, scl + widx(i - 1, j), scl + widx(i, j), WW, auxc(i - 1, j), auxc(i, j),
                             A.sp, scr + e, EX);
    }
    __syncthreads();
    issue_next();                      // (solvers without per-cell precompute)
    // X2a: fluctuations, limited correction F~ and CFL per correction edge (i in 1..T+1, row j)
    {
      const int e2 = opaque(threadIdx.x);
      if (e2 < E2) {
        const int i = 1 + e2 % (T + 1), j = e2 / (T + 1);
        const int e = j * (T + 3) + i;
        double P[MEQN], Q[MEQN], F[MEQN];
        edge_correction<S, 1>(scr + e, scr + e - 1, scr + e + 1, EX, A, auxc(i, j), rcell(i - 1, j), rcell(i, j),
                              cfl, P, Q, F);
#pragma unroll
        for (int k = 0; k < MEQN; ++k) { scr[(S::PB + k) * EX + e] = P[k]; qrp[k * E2 + e2] = Q[k]; }
        if (A.method3 == 1) {   // transverse of A-+dq alone: keep F~ (CTA-private global scratch)
#pragma unroll
          for (int k = 0; k < MEQN; ++k) fb[k * E2 + e2] = F[k];
        }
      }
    }
    __syncthreads();
    // X2b: one thread per receiving cell (i in 1..T, row j in 0..T+1): the L part of its right edge
    // and the R part of its left edge -> dq (interior rows) and the transverse split of both into
    // the y-edge accumulators up (ta) / down (tb).  Single writer per cell: no atomics, no zero fill.
    {
      const int t = opaque(threadIdx.x);
      if (t < T * (T + 2)) {
        const int i = 1 + t % T, j = t / T;
        const int er = j * (T + 3) + i + 1, el = er - 1, e2l = j * (T + 1) + (i - 1);
        const double r = rcell(i, j);
        double XL[MEQN], XR[MEQN], bm[MEQN], bp[MEQN], bmR[MEQN], bpR[MEQN];
#pragma unroll
        for (int k = 0; k < MEQN; ++k) { XL[k] = scr[(S::PB + k) * EX + er]; XR[k] = qrp[k * E2 + e2l]; }
        if (j >= 1 && j <= T) {
#pragma unroll
          for (int k = 0; k < MEQN; ++k) {
            double d = -r * XL[k];
            d -= r * XR[k];
            dq[(k * T + (j - 1)) * T + (i - 1)] = d;
          }
          if (RF && slot >= 0) {   // x faces, part 1: A+dq - F~ (low face) / A-dq + F~ (high face)
            if (tx == 0 && i == 1) {
              double* g = reg(0, ty * T + j - 1);
#pragma unroll
              for (int k = 0; k < MEQN; ++k) g[k] = XR[k];
            }
            if (tx == A.tiles - 1 && i == T) {
              double* g = reg(1, ty * T + j - 1);
#pragma unroll
              for (int k = 0; k < MEQN; ++k) g[k] = XL[k];
            }
          }
        }
        if (A.method3 == 1) {
#pragma unroll
          for (int k = 0; k < MEQN; ++k) { XL[k] -= fb[k * E2 + e2l + 1]; XR[k] += fb[k * E2 + e2l]; }
        }
        edge_transverse<S, 1>(scr + er, EX, A, XL, auxc(i, j), auxc(i, j + 1), bm, bp);
        edge_transverse<S, 1>(scr + el, EX, A, XR, auxc(i, j), auxc(i, j + 1), bmR, bpR);
#pragma unroll
        for (int k = 0; k < MEQN; ++k) {
          double u = -0.5 * r * bp[k], d = -0.5 * r * bm[k];
          u -= 0.5 * r * bpR[k];
          d -= 0.5 * r * bmR[k];
          ta[(k * (T + 2) + j) * T + (i - 1)] = u;
          tb[(k * (T + 2) + j) * T + (i - 1)] = d;
        }
      }
    }
    __syncthreads();
    // =============================== y-sweep ===============================
    // X3 (fold the x-sweep's transverse G~ into dq) shares this phase with the y Riemann solves:
    // it reads ta/tb and updates dq, Y1 reads sq/scl and writes scr, so no barrier between them.
    // X3: G~(i, j+1/2) = up(i, j) + dn(i, j+1)
    for (int t = opaque(threadIdx.x); t < T * T; t += NT) {
      const int i = 1 + t % T, j = 1 + t / T;
      const double s = rcell(i, j);
      double* gl = nullptr;
      double* gh = nullptr;
      if (RF && slot >= 0) {   // y faces, part 1: the x-sweep's transverse flux at the face
        if (ty == 0 && j == 1) gl = reg(2, tx * T + i - 1);
        if (ty == A.tiles - 1 && j == T) gh = reg(3, tx * T + i - 1);
      }
#pragma unroll
      for (int k = 0; k < MEQN; ++k) {
        const double* up = ta + k * (T + 2) * T;
        const double* dn = tb + k * (T + 2) * T;
        const double gt = up[j * T + (i - 1)] + dn[(j + 1) * T + (i - 1)];
        const double gb = up[(j - 1) * T + (i - 1)] + dn[j * T + (i - 1)];
        dq[(k * T + (j - 1)) * T + (i - 1)] -= s * (gt - gb);
        if (gl) gl[k] = -gb;
        if (gh) gh[k] = gt;
      }
    }
    for (int e = opaque(threadIdx.x); e < EX; e += NT) {       // column i, edge j (cells j-1 | j)
      const int i = e % (T + 2), j = e / (T + 2);
      double ql[MEQN], qr[MEQN];
#pragma unroll
      for (int k = 0; k < MEQN; ++k) { ql[k] = sq[k * WW + qidx(i, j - 1)]; qr[k] = sq[k * WW + qidx(i, j)]; }
      S::template riemann<2>(ql, qr, scl + widx(i, j - 1), scl + widx(i, j), WW, auxc(i, j - 1), auxc(i, j),
                             A.sp, scr + e, EX);
    }
    __syncthreads();
    // Y2a: per correction edge j in 1..T+1 of column i in 0..T+1
    {
      const int e2 = opaque(threadIdx.x);
      if (e2 < E2) {
        const int i = e2 % (T + 2), j = 1 + e2 / (T + 2);
        const int e = j * (T + 2) + i;
        double P[MEQN], Q[MEQN], F[MEQN];
        edge_correction<S, 2>(scr + e, scr + e - (T + 2), scr + e + (T + 2), EX, A, auxc(i, j), rcell(i, j - 1),
                              rcell(i, j), cfl, P, Q, F);
#pragma unroll
        for (int k = 0; k < MEQN; ++k) { scr[(S::PB + k) * EX + e] = P[k]; qrp[k * E2 + e2] = Q[k]; }
        if (A.method3 == 1) {
#pragma unroll
          for (int k = 0; k < MEQN; ++k) fb[k * E2 + e2] = F[k];
        }
      }
    }
    __syncthreads();
    // Y2b: one thread per receiving cell (column i in 0..T+1, j in 1..T): L part of its top edge, R
    // part of its bottom edge -> dq (interior columns), transverse into the x-edge accumulators
    // right (ta) / left (tb)
    {
      const int t = opaque(threadIdx.x);
      if (t < T * (T + 2)) {
        const int i = t % (T + 2), j = 1 + t / (T + 2);
        const int et = (j + 1) * (T + 2) + i, eb = et - (T + 2), e2b = (j - 1) * (T + 2) + i;
        const double r = rcell(i, j);
        double XL[MEQN], XR[MEQN], bm[MEQN], bp[MEQN], bmR[MEQN], bpR[MEQN];
#pragma unroll
        for (int k = 0; k < MEQN; ++k) { XL[k] = scr[(S::PB + k) * EX + et]; XR[k] = qrp[k * E2 + e2b]; }
        if (i >= 1 && i <= T) {
#pragma unroll
          for (int k = 0; k < MEQN; ++k) {
            double d = dq[(k * T + (j - 1)) * T + (i - 1)];
            d -= r * XL[k];
            d -= r * XR[k];
            dq[(k * T + (j - 1)) * T + (i - 1)] = d;
          }
          if (RF && slot >= 0) {   // y faces, part 2: fluctuation + F~ and the physical flux (outward)
            if (ty == 0 && j == 1) {
              double fq[MEQN];
              S::template flux<2>(sq + qidx(i, 1), WW, S::CAPA ? sa[2 * WW + widx(i, 1)] : 0.0, A.sp, fq);
              double* g = reg(2, tx * T + i - 1);
#pragma unroll
              for (int k = 0; k < MEQN; ++k) g[k] = (g[k] + XR[k]) - fq[k];
            }
            if (ty == A.tiles - 1 && j == T) {
              double fq[MEQN];
              S::template flux<2>(sq + qidx(i, T), WW, S::CAPA ? sa[2 * WW + widx(i, T + 1)] : 0.0, A.sp, fq);
              double* g = reg(3, tx * T + i - 1);
#pragma unroll
              for (int k = 0; k < MEQN; ++k) g[k] = fq[k] + (XL[k] + g[k]);
            }
          }
        }
        if (A.method3 == 1) {
#pragma unroll
          for (int k = 0; k < MEQN; ++k) { XL[k] -= fb[k * E2 + e2b + (T + 2)]; XR[k] += fb[k * E2 + e2b]; }
        }
        edge_transverse<S, 2>(scr + et, EX, A, XL, auxc(i, j), auxc(i + 1, j), bm, bp);
        edge_transverse<S, 2>(scr + eb, EX, A, XR, auxc(i, j), auxc(i + 1, j), bmR, bpR);
#pragma unroll
        for (int k = 0; k < MEQN; ++k) {
          double u = -0.5 * r * bp[k], d = -0.5 * r * bm[k];
          u -= 0.5 * r * bpR[k];
          d -= 0.5 * r * bmR[k];
          ta[(k * T + (j - 1)) * (T + 2) + i] = u;
          tb[(k * T + (j - 1)) * (T + 2) + i] = d;
        }
      }
    }
    __syncthreads();
    // Y3: F~(i+1/2, j) = right(i, j) + left(i+1, j); q_new = q + dq  (one thread per cell)
    {
      const int t = opaque(threadIdx.x);
      if (t < T * T) {
        const int i = 1 + t % T, j = 1 + t / T;
        const double rc = rcell(i, j);
        double* o = A.qnew + patch * (int64_t)MEQN * n2 + (int64_t)(ty * T + j - 1) * A.m + tx * T + i - 1;
        const double* rt = ta + (j - 1) * (T + 2) + i;   // right(i, j) of component 0
        const double* lf = tb + (j - 1) * (T + 2) + i;   // left(i, j)
        const double* qs = sq + qidx(i, j);
        const double* d = dq + (j - 1) * T + (i - 1);
#pragma unroll
        double* gl = nullptr;
        double* gh = nullptr;
        double fql[MEQN], fqh[MEQN];
        if (RF && slot >= 0) {   // x faces, part 2: the y-sweep's transverse flux and the physical flux
          if (tx == 0 && i == 1) {
            gl = reg(0, ty * T + j - 1);
            S::template flux<1>(qs, WW, S::CAPA ? sa[WW + widx(1, j)] : 0.0, A.sp, fql);
          }
          if (tx == A.tiles - 1 && i == T) {
            gh = reg(1, ty * T + j - 1);
            S::template flux<1>(qs, WW, S::CAPA ? sa[WW + widx(T + 1, j)] : 0.0, A.sp, fqh);
          }
        }
#pragma unroll
        for (int k = 0; k < MEQN; ++k) {
          const int c = k * T * (T + 2);
          const double fr = rt[c] + lf[c + 1];
          const double fl = rt[c - 1] + lf[c];
          const double val = qs[k * WW] + (d[k * T * T] - rc * (fr - fl));
          bad |= !isfinite(val);
          o[(int64_t)k * n2] = val;
          if (gl) gl[k] = (gl[k] - fl) - fql[k];
          if (gh) gh[k] = fqh[k] + (gh[k] + fr);
        }
      }
    }
    // no barrier: the next tile's phases touch ta/tb/dq (read above) only after two barriers, and
    // this buffer is re-staged only after the next tile's first barrier (issue_next)
  }

  // a non-finite updated state makes the step's CFL +inf (fc_step -> FC_ENONFINITE)
  if (__syncthreads_or(bad)) cfl = __longlong_as_double(0x7ff0000000000000ll);
  if (cfl != cfl) cfl = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) cfl = fmax(cfl, __shfl_xor_sync(0xffffffffu, cfl, o));
  if ((tid & 31) == 0) wmax[tid >> 5] = cfl;
  __syncthreads();
  if (tid == 0) {
    double c = wmax[0];
    for (int w = 1; w < (NT + 31) / 32; ++w) c = fmax(c, wmax[w]);
    atomicMax(A.cfl_bits, (unsigned long long)__double_as_longlong(c));
  }
}

// ---------------------------------------------------------------------------------------------
// Scalar advection (AdvConst, AdvEdgeCapa): two phases per tile.  For a scalar the wave is the jump
// and the limiter's upwind wave is another jump, so every edge computes everything it needs straight
// from the staged window -- no separate Riemann phase -- and writes its L part (A-dq + F~, entering
// the low cell), R part (A+dq - F~) and the four pre-scaled transverse contributions of those parts;
// then every cell gathers its 2 x 2 edges' parts and the 8 transverse contributions around it.
// 2 barriers per tile (3 with the window), each edge computed once: the phased k_step spent ~750
// thread-instructions per scalar cell-update on 7 barrier-separated phases (issue-bound).
// staging depth of the scalar kernel: NB - 1 tiles in flight ahead.  Constant-velocity tiles are
// 3.2 KB and quick to update, so more are kept in flight; capacity-form tiles carry 3 aux fields
// and deeper staging would cost CTAs per SM (measured: T2 -4 % time at 4, T4 +18 % at 4)
template <class S>
__host__ __device__ constexpr int sc_nbuf() { return S::CAPA ? 2 : 4; }
template <class S, int T, int NT, bool RF>
__global__ void __launch_bounds__(NT) k_step_sc(StepArgs A, int ntiles) {
  using Sh = StepShape<S, T>;
  constexpr int W = Sh::W, WW = Sh::WW;
  constexpr int NXE = (T + 1) * (T + 2), NE = 2 * NXE;   // x-edges a-1/2 (a = 1..T+1) of rows 0..T+1; y likewise
  const int tiles2 = A.tiles * A.tiles;
  if (A.active) ntiles = *A.nactive * tiles2;
  auto tile_of = [&](int k) {
    if (!A.active) return k;
    const int a = k / tiles2;
    return A.active[a] * tiles2 + (k - a * tiles2);
  };
  constexpr int NB = sc_nbuf<S>();          // staging depth: NB - 1 tiles in flight ahead
  extern __shared__ __align__(128) double sm[];
  double* sbuf = sm;                        // NB staging buffers
  double* win = sbuf + NB * Sh::BUF;        // natural window (dense single-copy staging only)
  double* rr = win + WW;                    // dt / (kappa dx) per window cell (capacity form)
  double* ex = rr + WW;                     // [6][NXE]: dqL, dqR, L->up, L->down, R->up, R->down
  double* ey = ex + 6 * NXE;                // [6][NXE]: dqL, dqR, L->left, L->right, R->left, R->right
  __shared__ __align__(8) uint64_t bars[NB];
  __shared__ double wmax[(NT + 31) / 32];
  __shared__ int16_t umap[WW];              // natural window index -> dense storage index (qcell)
  const int tid = threadIdx.x;
  const int n = A.m + 4, n2 = n * n;
  const bool dense = !A.ring && A.tiles == 1;
  const bool wide = A.ring || A.tiles > 1;          // many row pieces: the whole CTA issues them,
  const int sid = wide ? (tid & 31) * (NT / 32) + (tid >> 5) : tid;   // consecutive rows on different warps
  for (int t = tid; t < WW; t += NT) {
    const int i = t % W - 1, j = t / W - 1;
    umap[t] = (int16_t)(((unsigned)(i - 1) < (unsigned)T && (unsigned)(j - 1) < (unsigned)T)
                            ? (j - 1) * T + (i - 1) : T * T + ring_index(i, j, T));
  }
  if (tid == 0) {
    for (int q = 0; q < NB; ++q) mbar_init(&bars[q], 1);
    fence_proxy_async();
  }
  __syncthreads();
  for (int q = 0; q < NB - 1; ++q) {
    const int k0 = blockIdx.x + q * gridDim.x;
    if ((tid < 32 || wide) && k0 < ntiles) stage_tile<S, T>(A, tile_of(k0), sbuf + q * Sh::BUF, &bars[q], sid, wide ? NT : 32);
    if (A.ring) {
      if (k0 < ntiles) gather_ring<S, T, NT>(A, tile_of(k0), sbuf + q * Sh::BUF);
      cp_async_commit();
    }
  }
  double cfl = 0.0;
  bool bad = false;
  const double m3 = A.method3 == 2 ? 1.0 : 0.0;
  const bool trans = A.method3 >= 1, second = A.method2 == 2;
  const bool nolim = A.lim.lo == 1.0;
  const double lc1 = A.lim.c1, lc2 = A.lim.c2, lc3 = A.lim.c3, lc4 = A.lim.c4;
  const double u0 = A.sp.p0, v0 = A.sp.p1;
  int it = 0;
  for (int kt = blockIdx.x; kt < ntiles; kt += gridDim.x, ++it) {
    const int b = it % NB, bn = (it + NB - 1) % NB;
    const int tile = tile_of(kt);
    const int knext = kt + (NB - 1) * gridDim.x;
    bool issued = false;
    auto issue_next = [&]() {
      if (issued) return;
      issued = true;
      if ((tid < 32 || wide) && knext < ntiles) {
        fence_proxy_async();
        stage_tile<S, T>(A, tile_of(knext), sbuf + bn * Sh::BUF, &bars[bn], sid, wide ? NT : 32);
      }
      if (A.ring) {
        if (knext < ntiles) gather_ring<S, T, NT>(A, tile_of(knext), sbuf + bn * Sh::BUF);
        cp_async_commit();
      }
    };
    double* sq = sbuf + b * Sh::BUF;
    double* sa = sq + WW + 2;
    int patch = tile, tx = 0, ty = 0;
    if (A.tiles > 1) {
      patch = tile / tiles2;
      const int tt = tile - patch * tiles2;
      ty = tt / A.tiles;
      tx = tt - ty * A.tiles;
    }
    const double dtdx = dtdx_level(A, (int)A.level[patch]);
    const int slot = RF ? A.rslot[patch] : -1;
    auto reg = [&](int face, int e) { return A.freg + (((int64_t)slot * 4 + face) * A.m + e); };
    mbar_wait(&bars[b], (uint32_t)((it / NB) & 1));
    if (A.ring) {
      cp_async_wait<NB - 2>();
      __syncthreads();
      issue_next();
      const uint8_t bc = A.bcflag[patch];
      if (bc & 1) { window_bc<S, T, NT>(A, tile, sq, 0); __syncthreads(); }
      if (bc & 2) { window_bc<S, T, NT>(A, tile, sq, 1); __syncthreads(); }
    }
    // phase 0: natural window (un-permuting the dense staging), r per cell, uniformity
    const double* wq = dense ? win : sq;
    const double ref = dense ? sq[0] : sq[2 * W + 2];     // interior cell (1, 1)
    bool diff = false;
    for (int t = opaque(threadIdx.x); t < WW; t += NT) {
      double v;
      if (dense) {
        v = sq[umap[t]];
        win[t] = v;
      } else {
        v = sq[t];
      }
      if (S::CAPA) rr[t] = dtdx / sa[t];
      diff |= v != ref;
    }
    const bool may_skip = A.skip_quiescent && !(RF && slot >= 0);
    bool uniform = false;
    if (may_skip) uniform = !__syncthreads_or(diff);
    else __syncthreads();
    issue_next();
    if (uniform) {   // every jump is zero: q_new = q, CFL from the state
      cfl = fmax(cfl, S::quiescent_cfl(sq, WW, A.sp, sa, dtdx, T, W, opaque(threadIdx.x), NT));
      for (int t = opaque(threadIdx.x); t < T * T; t += NT) {
        const int i = 1 + t % T, j = 1 + t / T;
        A.qnew[patch * (int64_t)n2 + (int64_t)(ty * T + j - 1) * A.m + tx * T + i - 1] = ref;
      }
      __syncthreads();
      continue;
    }
    auto Q = [&](int a, int c) { return wq[(c + 1) * W + (a + 1)]; };
    auto R = [&](int a, int c) { return S::CAPA ? rr[(c + 1) * W + (a + 1)] : dtdx; };
    auto UX = [&](int a, int c) { return S::CAPA ? sa[WW + (c + 1) * W + (a + 1)] : u0; };
    auto VY = [&](int a, int c) { return S::CAPA ? sa[2 * WW + (c + 1) * W + (a + 1)] : v0; };
    // phi(w_i / w) w, division-free and branch-free (lo = 1: no limiter)
    auto limited = [&](double w, double wi) {
      const bool same = (w > 0.0 && wi > 0.0) || (w < 0.0 && wi < 0.0);
      const double mag = fmin(fmin(fabs(fma(lc1, w, lc2 * wi)), lc3 * fabs(w)), lc4 * fabs(wi));
      return nolim ? w : (same ? copysign(mag, w) : 0.0);
    };
    // per-tile constants of the constant-velocity solver
    const double spx = u0 > 0.0 ? u0 : 0.0, snx = u0 - spx, spy = v0 > 0.0 ? v0 : 0.0, sny = v0 - spy;
    const double cfx = second ? 0.5 * fabs(u0) * (1.0 - fabs(u0) * dtdx) : 0.0;
    const double cfy = second ? 0.5 * fabs(v0) * (1.0 - fabs(v0) * dtdx) : 0.0;
    const double ht = trans ? -0.5 * dtdx : 0.0;
    const double kup = ht * (v0 > 0.0 ? v0 : 0.0), kdown = ht * (v0 < 0.0 ? v0 : 0.0);
    const double kleft = ht * (u0 < 0.0 ? u0 : 0.0), kright = ht * (u0 > 0.0 ? u0 : 0.0);
    // phase A: every edge once (x-edges then y-edges; the branch is warp-uniform but for one warp)
    auto edge = [&](auto dir, int u) {
      constexpr int D = decltype(dir)::value;
      constexpr int dla = D == 1 ? -1 : 0, dlc = D == 1 ? 0 : -1;
      const int a = D == 1 ? 1 + u % (T + 1) : u % (T + 2);
      const int c = D == 1 ? u / (T + 1) : 1 + u / (T + 2);
      // the edge joins cells lo = (a-1, c) | hi = (a, c) (x) or lo = (a, c-1) | hi = (a, c) (y)
      const double* qh_p = wq + (c + 1) * W + (a + 1);
      constexpr int step = D == 1 ? 1 : W;
      const double qh = qh_p[0], ql = qh_p[-step];
      const double w = qh - ql;
      double s, sp, sn, cf, rl, rh;
      if (S::CAPA) {
        s = D == 1 ? UX(a, c) : VY(a, c);
        rl = R(a + dla, c + dlc);
        rh = R(a, c);
        sp = s > 0.0 ? s : 0.0;
        sn = s - sp;
        const double as = fabs(s);
        cf = second ? 0.5 * as * (1.0 - as * (0.5 * (rl + rh))) : 0.0;
        cfl = fmax(cfl, fmax(rh * s, -rl * s));
      } else {   // per-tile constants
        s = D == 1 ? u0 : v0;
        sp = D == 1 ? spx : spy;
        sn = D == 1 ? snx : sny;
        cf = D == 1 ? cfx : cfy;
        rl = rh = dtdx;
      }
      const double wi = s > 0.0 ? ql - qh_p[-2 * step] : qh_p[step] - qh;
      const double f = cf * limited(w, wi);
      double* E = D == 1 ? ex : ey;
      E[u] = sn * w + f;                 // dqL: enters the low cell
      E[NXE + u] = sp * w - f;           // dqR: enters the high cell
      const double xl = sn * w + m3 * f, xr = sp * w - m3 * f;
      double k0, k1, k2, k3;             // -1/2 r B+- of the receiving cells, 0 without transverse
      if (S::CAPA) {
        const double h = trans ? -0.5 : 0.0;
        if (D == 1) {    // into G~ at the y-edges of the receiving cells (own bottom / top velocities)
          k0 = h * rl * fmax(VY(a - 1, c + 1), 0.0);   // L -> up of (a-1, c)
          k1 = h * rl * fmin(VY(a - 1, c), 0.0);       // L -> down
          k2 = h * rh * fmax(VY(a, c + 1), 0.0);       // R -> up of (a, c)
          k3 = h * rh * fmin(VY(a, c), 0.0);           // R -> down
        } else {         // into F~ at the x-edges of the receiving cells (own left / right velocities)
          k0 = h * rl * fmin(UX(a, c - 1), 0.0);       // L -> left of (a, c-1)
          k1 = h * rl * fmax(UX(a + 1, c - 1), 0.0);   // L -> right
          k2 = h * rh * fmin(UX(a, c), 0.0);           // R -> left of (a, c)
          k3 = h * rh * fmax(UX(a + 1, c), 0.0);       // R -> right
        }
      } else {
        k0 = D == 1 ? kup : kleft;
        k1 = D == 1 ? kdown : kright;
        k2 = k0;
        k3 = k1;
      }
      E[2 * NXE + u] = k0 * xl;
      E[3 * NXE + u] = k1 * xl;
      E[4 * NXE + u] = k2 * xr;
      E[5 * NXE + u] = k3 * xr;
    };
    if (!S::CAPA)   // constant velocities: the CFL is r max(|u|, |v|) on every edge
      cfl = fmax(cfl, fmax(fmax(dtdx * u0, -dtdx * u0), fmax(dtdx * v0, -dtdx * v0)));
    for (int t = opaque(threadIdx.x); t < NE; t += NT) {
      if (t < NXE) edge(std::integral_constant<int, 1>{}, t);
      else edge(std::integral_constant<int, 2>{}, t - NXE);
    }
    __syncthreads();
    // phase B: every cell gathers its edges
    for (int t = opaque(threadIdx.x); t < T * T; t += NT) {
      const int i = 1 + t % T, j = 1 + t / T;
      auto xi = [](int a, int c) { return c * (T + 1) + (a - 1); };
      auto yi = [](int a, int c) { return (c - 1) * (T + 2) + a; };
      const double Gt = ex[4 * NXE + xi(i, j)] + ex[2 * NXE + xi(i + 1, j)] + ex[5 * NXE + xi(i, j + 1)] +
                        ex[3 * NXE + xi(i + 1, j + 1)];
      const double Gb = ex[4 * NXE + xi(i, j - 1)] + ex[2 * NXE + xi(i + 1, j - 1)] + ex[5 * NXE + xi(i, j)] +
                        ex[3 * NXE + xi(i + 1, j)];
      const double Fr = ey[3 * NXE + yi(i, j + 1)] + ey[5 * NXE + yi(i, j)] + ey[2 * NXE + yi(i + 1, j + 1)] +
                        ey[4 * NXE + yi(i + 1, j)];
      const double Fl = ey[3 * NXE + yi(i - 1, j + 1)] + ey[5 * NXE + yi(i - 1, j)] + ey[2 * NXE + yi(i, j + 1)] +
                        ey[4 * NXE + yi(i, j)];
      const double dxR = ex[NXE + xi(i, j)], dxL = ex[xi(i + 1, j)];
      const double dyR = ey[NXE + yi(i, j)], dyL = ey[yi(i, j + 1)];
      const double r0 = R(i, j), q0 = Q(i, j);
      const double val = q0 - r0 * (dxR + dxL + Fr - Fl) - r0 * (dyR + dyL + Gt - Gb);
      bad |= !isfinite(val);
      A.qnew[patch * (int64_t)n2 + (int64_t)(ty * T + j - 1) * A.m + tx * T + i - 1] = val;
      if (RF && slot >= 0) {   // applied face fluxes, outward (reflux records)
        if (tx == 0 && i == 1) *reg(0, ty * T + j - 1) = (dxR - Fl) - UX(1, j) * q0;
        if (tx == A.tiles - 1 && i == T) *reg(1, ty * T + j - 1) = UX(T + 1, j) * q0 + (dxL + Fr);
        if (ty == 0 && j == 1) *reg(2, tx * T + i - 1) = (dyR - Gb) - VY(i, 1) * q0;
        if (ty == A.tiles - 1 && j == T) *reg(3, tx * T + i - 1) = VY(i, T + 1) * q0 + (dyL + Gt);
      }
    }
    __syncthreads();   // the window, r and the edge arrays are rewritten by the next tile
  }
  if (__syncthreads_or(bad)) cfl = __longlong_as_double(0x7ff0000000000000ll);
  if (cfl != cfl) cfl = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) cfl = fmax(cfl, __shfl_xor_sync(0xffffffffu, cfl, o));
  if ((tid & 31) == 0) wmax[tid >> 5] = cfl;
  __syncthreads();
  if (tid == 0) {
    double c = wmax[0];
    for (int w = 1; w < (NT + 31) / 32; ++w) c = fmax(c, wmax[w]);
    atomicMax(A.cfl_bits, (unsigned long long)__double_as_longlong(c));
  }
}

// ---------------------------------------------------------------------------------------------
// Constant-velocity scalar advection (the C1/C2/T1/T2 physics), register sweep.  With the same
// speeds (u, v) on every edge, the parts k_step_sc gathers per cell regroup as
//   q_new = q - r [ Xf + Yf + k_right (Y - Y_{i-1}) + k_left (Y_{i+1} - Y)
//                           + k_up (X - X_{j-1}) + k_down (X_{j+1} - X) ]
// where, per cell, Xf = dqR(i-1/2) + dqL(i+1/2) are the parts of its two x-edges that enter it
// (A+dq - F~ from the left edge, A-dq + F~ from the right one), X the same with the correction
// weighted by (method3 == 2) (what the transverse solve splits), Yf / Y along y, r = dt / dx and
// k_* = -r/2 max/min(u or v, 0) (0 without transverse terms): the same sums, re-associated
// (reading 24).  A warp holds PW = 32 / LP patches, LP = T/2 + 1 lanes each; lane k of a
// patch owns columns 2k, 2k+1 (0..T+1) and sweeps rows 0..T+1 once with its columns' 4-row windows,
// the X of the two rows below and the last y-edge's parts in registers; a neighbouring column's
// parts come by shuffle.  Every edge is computed once, by one lane; no shared-memory scratch and
// no barrier in the sweep.  Each CTA is one warp with its own double-buffered staging (whole
// padded patches by one bulk copy each, or, on the fused ring path, the interior rows by bulk copy
// and the ring by cp.async from the sources) into the natural (T+4)^2 window, so that a lane's
// reads are fixed offsets from its columns' base addresses.
#ifndef CV_UNROLL
#define CV_UNROLL 0
#endif
template <int T>
struct CvShape {
  static constexpr int W = T + 4, WW = W * W, LP = T / 2 + 1, PW = 32 / LP;
};

// staging of one group of PW patches into natural (T+4)^2 windows for the register sweeps: the
// padded patch (dense interior + ring) by row bulk copies and 16-byte side pairs, or, on the fused
// ring path, the interior rows by bulk copy and the ring cells by cp.async from their sources (all
// of the group's source offsets loaded first: one latency, not one per patch)
#ifndef CV_STAGE_INLINE
#define CV_STAGE_INLINE __forceinline__
#endif
// regular-ring neighbour offsets of a group of PW patches (plan_ring_regular): entry q 9 + d in
// lane (q 9 + d) mod 32 of lo (< 32) or hi; -1 for a patch that reads the ring table.  Loaded a
// group ahead of its staging (the loads complete under the current group's sweep).
struct CvNb {
  int32_t lo, hi;
};
// Quad blocks (QD): a 2 x 2 sibling family of regular m = 8 patches (local patches 4b .. 4b+3, x in
// the low bit: child c = cx + 2 cy) staged as one 16 x 16 window and swept as one T = 16 patch.
// Each edge of the family is computed once instead of once per patch it borders, from the same cell
// values the patches' rings hold (aligned same-level copies): every patch's update is the one the
// m = 8 sweep computes.  The block's ring reads the 12 same-level neighbours around it, entry k of
// the block = neighbour d (3 (dy + 1) + dx + 1) of child c in plan_ring_regular's table:
__device__ __forceinline__ int quad_child(int k) { return (int)((0x332232101100ull >> (4 * k)) & 15); }
__device__ __forceinline__ int quad_dir(int k) { return (int)((0x877653532110ull >> (4 * k)) & 15); }

template <int T, bool QD = false>
__device__ __forceinline__ CvNb cv_nb_load(const StepArgs& A, int i0, int cnt, int lane) {
  constexpr int PW = CvShape<T>::PW, NE = QD ? 12 : 9;
  CvNb r{-1, -1};
  if (!A.nb9 || cnt <= 0) return r;
  auto entry = [&](int e) {
    const int q = e / NE;
    if (q >= cnt || q >= PW) return -1;
    int64_t at;
    if (QD) {
      const int k = e - NE * q;
      at = (int64_t)(4 * (i0 + q) + quad_child(k)) * 9 + quad_dir(k);
    } else {
      at = (int64_t)(A.active ? A.active[i0 + q] : i0 + q) * 9 + (e - 9 * q);
    }
    // (a volatile load: issued here, not sunk to its use after the sweep)
    int32_t v;
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(A.nb9 + at));
    return v;
  };
  r.lo = entry(lane);
  if (PW * NE > 32) r.hi = entry(lane + 32);
  return r;
}

// staging of a group of PW quad blocks (T = 16 windows): the 4 children's interiors as 16-byte
// chunks, the ring as 16-byte pairs from the 12 neighbours (every pair lies in one neighbour's
// interior row, aligned: the patch boundaries fall between odd and even window columns)
template <int T>
__device__ __forceinline__ void cv_stage_quad(const StepArgs& A, double* buf, uint64_t* bar, int lane, int i0,
                                              int cnt, const CvNb& nbv) {
  static_assert(T == 16, "quad blocks are 16 x 16");
  using C = CvShape<T>;
  constexpr int W = C::W, WW = C::WW, PW = C::PW, S8 = 12 * 12;   // (m = 8 storage block, meqn = 1)
  if (lane == 0) mbar_expect_tx(bar, 0u);
  __syncwarp();
  auto nb_of = [&](int e) {
    const int lo = __shfl_sync(0xffffffffu, nbv.lo, e & 31);
    const int hi = __shfl_sync(0xffffffffu, nbv.hi, e & 31);
    return e < 32 ? lo : hi;
  };
  constexpr int RCH = 2 * W + 2 * T, RU = (RCH + 31) / 32;
  int rdst[RU], rk[RU], rsrc[RU];
#pragma unroll
  for (int u = 0; u < RU; ++u) {
    const int c = lane + 32 * u;
    int wi, wj;
    if (c < 2 * W) {
      const int rr = c / (W / 2);
      wj = rr < 2 ? rr : T + rr;
      wi = 2 * (c - rr * (W / 2));
    } else {
      wj = 2 + ((c - 2 * W) >> 1);
      wi = (c & 1) ? T + 2 : 0;
    }
    const int i = wi - 1, j = wj - 1;                       // block cell (1-based interior 1..16)
    const int cx = i <= 8 ? 0 : 1, cy = j <= 8 ? 0 : 1;     // the child it borders
    const int ii = i - 8 * cx, jj = j - 8 * cy;             // in that child's frame (-1 .. 10)
    const int dx = ii < 1 ? -1 : (ii > 8 ? 1 : 0), dy = jj < 1 ? -1 : (jj > 8 ? 1 : 0);
    const int child = cx + 2 * cy, d = 3 * (dy + 1) + dx + 1;
    int k = 0;
#pragma unroll
    for (int t = 0; t < 12; ++t) k = (quad_child(t) == child && quad_dir(t) == d) ? t : k;
    rdst[u] = c < RCH ? wj * W + wi : -1;
    rk[u] = k;
    rsrc[u] = (jj - dy * 8 - 1) * 8 + (ii - dx * 8 - 1);
  }
#pragma unroll
  for (int q = 0; q < PW; ++q) {
    if (q >= cnt) break;
    double* b = buf + q * WW;
    const double* qc = A.qold + (int64_t)4 * (i0 + q) * S8;
#pragma unroll
    for (int c = lane; c < T * T / 2; c += 32) {
      const int row = c >> 3, cp = c & 7;
      const double* src = qc + ((row >> 3) * 2 + (cp >> 2)) * S8 + (row & 7) * 8 + 2 * (cp & 3);
      cp_async16(b + (row + 2) * W + 2 + 2 * cp, src);
    }
#pragma unroll
    for (int u = 0; u < RU; ++u) {
      const int off = nb_of(12 * q + rk[u]);
      if (rdst[u] >= 0) cp_async16(b + rdst[u], A.qold + off + rsrc[u]);
    }
  }
  cp_async_commit();
}

template <int T>
__device__ CV_STAGE_INLINE void cv_stage(const StepArgs& A, double* buf, uint64_t* bar, int lane, int i0, int cnt,
                                         const CvNb& nbv) {
  using C = CvShape<T>;
  constexpr int W = C::W, WW = C::WW, PW = C::PW, G = WW - T * T;
  const bool ring = A.ring != nullptr;
  auto patch_of = [&](int idx) { return A.active ? A.active[idx] : idx; };
  // (the ring path stages by cp.async only: the barrier just completes its phase)
  if (lane == 0) mbar_expect_tx(bar, ring ? 0u : (uint32_t)cnt * (T * T + 4 * W) * (uint32_t)sizeof(double));
  __syncwarp();
  if (!ring) {
    const int mp = lane < cnt ? patch_of(i0 + lane) : 0;
#pragma unroll
    for (int q = 0; q < PW; ++q) {
      const int patch = __shfl_sync(0xffffffffu, mp, q);
      if (q >= cnt) break;
      const double* qb = A.qold + (int64_t)patch * WW;
      double* b = buf + q * WW;
      if (lane < T) bulk_g2s(b + (lane + 2) * W + 2, qb + lane * T, T * sizeof(double), bar);
      else if (lane == T) bulk_g2s(b, qb + T * T, 2 * W * sizeof(double), bar);
      else if (lane == T + 1) bulk_g2s(b + (T + 2) * W, qb + T * T + 2 * W + 4 * T, 2 * W * sizeof(double), bar);
      if (lane < 2 * T) {
        const int j = 1 + (lane >> 1), side = lane & 1;
        cp_async16(b + (j + 1) * W + (side ? T + 2 : 0), qb + T * T + 2 * W + 4 * (j - 1) + 2 * side);
      }
    }
    cp_async_commit();
    return;
  }
  // the neighbour offset of entry e = q 9 + d from the prefetched registers
  auto nb_of = [&](int e) {
    const int lo = __shfl_sync(0xffffffffu, nbv.lo, e & 31);
    if (PW * 9 <= 32) return lo;
    const int hi = __shfl_sync(0xffffffffu, nbv.hi, e & 31);
    return e < 32 ? lo : hi;
  };
  // the ring as 16-byte pairs (regular patches): rows -1, 0, T+1, T+2 whole (W / 2 pairs each),
  // then the two side pairs of rows 1..T; every pair lies in one neighbour's interior row (m even:
  // aligned).  Per lane: the window offset, the direction and the offset within the neighbour of
  // its pairs, the same for every patch.
  constexpr int RCH = 2 * W + 2 * T, RU = (RCH + 31) / 32;
  int rdst[RU], rdir[RU], rsrc[RU];
#pragma unroll
  for (int u = 0; u < RU; ++u) {
    const int c = lane + 32 * u;
    int wi, wj;
    if (c < 2 * W) {
      const int rr = c / (W / 2);
      wj = rr < 2 ? rr : T + rr;
      wi = 2 * (c - rr * (W / 2));
    } else {
      wj = 2 + ((c - 2 * W) >> 1);
      wi = (c & 1) ? T + 2 : 0;
    }
    const int i = wi - 1, j = wj - 1;   // patch cell (1-based interior)
    const int dx = i < 1 ? -1 : (i > T ? 1 : 0), dy = j < 1 ? -1 : (j > T ? 1 : 0);
    rdst[u] = c < RCH ? wj * W + wi : -1;
    rdir[u] = 3 * dy + dx + 4;
    rsrc[u] = (j - dy * T - 1) * T + (i - dx * T - 1);
  }
  constexpr int NR = (G + 31) / 32;
  int pt[PW];
  bool rg[PW];                             // (warp-uniform)
  int32_t src[PW][NR];
  uint8_t own[PW][NR];
  const bool peers = A.rpeer != nullptr;   // (uniform: only peer-memory / AMR forests carry owners)
#pragma unroll
  for (int q = 0; q < PW; ++q) {
    pt[q] = q < cnt ? patch_of(i0 + q) : -1;
    rg[q] = pt[q] >= 0 && nb_of(9 * q) >= 0;
  }
  // the other patches' ring-table entries, all loaded first: one latency, not one per patch
  // (skipped as a whole -- a warp-uniform branch -- when every patch of the group is regular)
  bool table = false;
#pragma unroll
  for (int q = 0; q < PW; ++q) table |= pt[q] >= 0 && !rg[q];
#pragma unroll
  for (int q = 0; q < PW; ++q)
#pragma unroll
    for (int t = 0; t < NR; ++t) { src[q][t] = -1; own[q][t] = 0; }
  if (table) {
#pragma unroll
    for (int q = 0; q < PW; ++q)
#pragma unroll
      for (int t = 0; t < NR; ++t) {
        const int r = lane + 32 * t;
        const bool ok = pt[q] >= 0 && !rg[q] && r < G;
        if (ok) src[q][t] = __ldg(A.ring + (int64_t)pt[q] * G + r);
        if (ok && peers) own[q][t] = __ldg(A.rpeer + (int64_t)pt[q] * G + r);
      }
  }
  // the interior as 16-byte cp.async chunks (two cells) into the natural window: every lane issues
  // its own (a per-row bulk copy from per-lane addresses is serialised over the lanes)
  constexpr int CH = T * T / 2;
#pragma unroll
  for (int q = 0; q < PW; ++q) {
    if (pt[q] < 0) continue;
    double* b = buf + q * WW;
    const double* qi = A.qold + (int64_t)pt[q] * WW;
#pragma unroll
    for (int c = lane; c < CH; c += 32) {
      const int row = c / (T / 2), cp = c - row * (T / 2);
      cp_async16(b + (row + 2) * W + 2 + 2 * cp, qi + row * T + 2 * cp);
    }
    if (rg[q]) {
#pragma unroll
      for (int u = 0; u < RU; ++u) {
        const int off = nb_of(9 * q + rdir[u]);
        if (rdst[u] >= 0) cp_async16(b + rdst[u], A.qold + off + rsrc[u]);
      }
      continue;
    }
#pragma unroll
    for (int t = 0; t < NR; ++t) {
      const int r = lane + 32 * t;
      if (src[q][t] >= 0)
        cp_async8(b + ring_window_index<T>(r), (peers ? ring_base(A, own[q][t]) : A.qold) + src[q][t]);
    }
  }
  cp_async_commit();
}

// fused ring path: the physical-boundary ring cells of the group's windows (x faces, then y faces)
template <int T>
__device__ __forceinline__ void cv_bcs(const StepArgs& A, double* gbuf, int mypatch, int mybc, int lane) {
  constexpr int WW = CvShape<T>::WW, G = WW - T * T;
  for (unsigned todo = __ballot_sync(0xffffffffu, mybc != 0); todo; todo &= todo - 1) {
    const int q = __ffs(todo) - 1;
    const int patch = __shfl_sync(0xffffffffu, mypatch, q);
    const int bc = __shfl_sync(0xffffffffu, mybc, q);
    const int32_t* rs = A.ring + (int64_t)patch * G;
    double* sq = gbuf + q * WW;
    for (int is_y = 0; is_y < 2; ++is_y) {
      if (!(bc & (1 << is_y))) continue;
      for (int r = lane; r < G; r += 32) {
        const int32_t v = __ldg(rs + r);
        if (v >= 0) continue;
        const int code = -1 - v;
        if ((code & 1) != is_y) continue;
        sq[ring_window_index<T>(r)] = sq[code >> 3];   // (one component: no momentum to negate)
      }
      __syncwarp();
    }
  }
}

// CV_EXACT: the sums and products of the sweep rounded on their own (no contraction left to the
// compiler, whose choice may differ between instantiations)
#ifndef CV_EXACT
#define CV_EXACT 1
#endif
#if CV_EXACT
#define CV_ADD(x, y) __dadd_rn(x, y)
#define CV_MUL(x, y) __dmul_rn(x, y)
#else
#define CV_ADD(x, y) ((x) + (y))
#define CV_MUL(x, y) ((x) * (y))
#endif
template <int T, int SX, int SY, bool MT2, int NB, bool RF, bool QD = false>
#ifndef CV_MINB
#define CV_MINB 20
#endif
__global__ void __launch_bounds__(32, CV_MINB) k_step_cv(StepArgs A, int npatch) {
  using C = CvShape<T>;
  constexpr int W = C::W, WW = C::WW, LP = C::LP, PW = C::PW, G = WW - T * T;
  extern __shared__ __align__(128) double sm[];     // [NB][PW][WW]
  __shared__ __align__(8) uint64_t bars[NB];
  const int lane = threadIdx.x;
  if (A.active) npatch = *A.nactive;
  const int ngroups = (npatch + PW - 1) / PW;
  const bool ring = A.ring != nullptr;
  // (QD: npatch counts quad blocks, unit b = local patches 4b .. 4b + 3; no active list)
  auto patch_of = [&](int idx) { return QD ? 4 * idx : (A.active ? A.active[idx] : idx); };
  auto nbload = [&](int g) { return g < ngroups ? cv_nb_load<T, QD>(A, g * PW, min(PW, npatch - g * PW), lane) : CvNb{-1, -1}; };
  auto stage = [&](int g, int s, const CvNb& nb) {
    if constexpr (QD) cv_stage_quad<T>(A, sm + (size_t)s * PW * WW, &bars[s], lane, g * PW, min(PW, npatch - g * PW), nb);
    else cv_stage<T>(A, sm + (size_t)s * PW * WW, &bars[s], lane, g * PW, min(PW, npatch - g * PW), nb);
  };
  if (lane == 0) {
    for (int q = 0; q < NB; ++q) mbar_init(&bars[q], 1);
    fence_proxy_async();
  }
  __syncwarp();
  for (int q = 0; q < (NB > 1 ? NB - 1 : 1); ++q) {
    const int g = blockIdx.x + q * gridDim.x;
    if (g < ngroups) stage(g, q, nbload(g));
    else cp_async_commit();
  }
  // lane -> (patch slot, columns c0 = 2k, c0 + 1); the 5 columns it reads: c0 - 1 .. c0 + 3 (the
  // last clamped into the window: it only feeds the unused edge T + 3/2)
  const int p = lane / LP, k = lane - p * LP, c0 = 2 * k;
  const double u0 = A.sp.p0, v0 = A.sp.p1;
  const bool trans = A.method3 >= 1, second = A.method2 == 2;
  // phi(wi / w) w of the MC / minmod limiter (launched for those only): cv_limited
  const double lp1 = A.lp1, lp2 = A.lp2, lk3 = A.lk3;
  auto limited = [&](double w, double wi) { return cv_limited(w, wi, lp1, lp2, lk3); };
  double cfl = 0.0;
  double chk = 0.0;                     // sum of 0 * q_new: NaN iff some q_new is not finite
  // a group's levels and boundary flags, loaded a group ahead into their own registers (volatile:
  // issued here, consumed one group later -- loaded at the group's start, the boundary ballot after
  // the staging wait stalled on them)
  int nlev = 0, nbc = 0;
  auto meta_load = [&](int gg) {
    if (gg >= ngroups) return;
    const int c = min(PW, npatch - gg * PW);
    const int pt = lane < c ? patch_of(gg * PW + lane) : 0;
    asm volatile("ld.global.nc.s8 %0, [%1];" : "=r"(nlev) : "l"(A.level + pt));
    if (ring) asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(nbc) : "l"(A.bcflag + pt));
  };
  meta_load(blockIdx.x);
  int it = 0;
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
    const int b = it % NB;
    const int cnt = min(PW, npatch - g * PW);
    // this group's patch ids (the reflux slots load during the wait)
    const int mypatch = lane < cnt ? patch_of(g * PW + lane) : 0;
    const int mylevel = nlev;
    const int myslot = RF ? A.rslot[mypatch] : -1;
    const int mybc = (ring && lane < cnt) ? nbc : 0;
    meta_load(g + gridDim.x);
    // the next staged group's regular-ring offsets (in flight during this group's sweep)
    const CvNb nbn = ring ? nbload(g + (NB > 1 ? NB - 1 : 1) * gridDim.x) : CvNb{-1, -1};
    mbar_wait(&bars[b], (uint32_t)((it / NB) & 1));
    cp_async_wait<(NB > 1 ? NB - 2 : 0)>();
    __syncwarp();
    // the next group's staging: NB - 1 groups ahead, or (NB = 1) after this group's sweep
    auto issue_next = [&]() {
      const int gn = g + (NB > 1 ? NB - 1 : 1) * gridDim.x, bn = (it + NB - 1) % NB;
      if (gn < ngroups) {
        fence_proxy_async();
        stage(gn, bn, nbn);
      } else {
        cp_async_commit();
      }
    };
    if (NB > 1) issue_next();
    double* gbuf = sm + (size_t)b * PW * WW;
    if (ring) cv_bcs<T>(A, gbuf, mypatch, mybc, lane);
    const bool live = p < cnt;
    const int patch = __shfl_sync(0xffffffffu, mypatch, live ? p : 0);
    const int level = __shfl_sync(0xffffffffu, mylevel, live ? p : 0);
    const int slot = RF ? __shfl_sync(0xffffffffu, myslot, live ? p : 0) : -1;
    const bool rec = RF && live && slot >= 0;   // reflux records: applied face fluxes, outward
    double* reg = RF ? A.freg + (int64_t)(slot < 0 ? 0 : slot) * 4 * T : nullptr;   // [face][T]
    const double* sq = gbuf + (live ? p : 0) * WW;
    const double* col[5];   // column c0 - 1 + e of window row -1
#pragma unroll
    for (int e = 0; e < 5; ++e) col[e] = sq + min(c0 - 1 + e, T + 2) + 1;
    auto ld = [&](int e, int j) { return col[e][(j + 1) * W]; };
    const double r = dtdx_level(A, level);
    if (live) cfl = fmax(cfl, fmax(fmax(r * u0, -r * u0), fmax(r * v0, -r * v0)));
    const double cfx = second ? __dmul_rn(0.5 * fabs(u0), __dsub_rn(1.0, __dmul_rn(fabs(u0), r))) : 0.0;
    const double cfy = second ? __dmul_rn(0.5 * fabs(v0), __dsub_rn(1.0, __dmul_rn(fabs(v0), r))) : 0.0;
    const double ht = trans ? -0.5 * r : 0.0;
    // k_up / k_down / k_left / k_right with the signs fixed by SX, SY
    const double kx = ht * u0, ky = ht * v0;   // (SX > 0: k_right = kx, k_left = 0; SX < 0: k_left = kx)
    const double m3 = A.method3 == 2 ? 1.0 : 0.0;
    double* out = A.qnew + (int64_t)patch * (QD ? 144 : WW);
    // interior cell (x, y) of the unit -> its offset from out (QD: in child (x / 8, y / 8))
    auto oidx = [&](int x, int y) {
      return QD ? ((y >> 3) * 2 + (x >> 3)) * 144 + (y & 7) * 8 + (x & 7) : y * T + x;
    };
    // edge parts: dqL (into the low cell), dqR (into the high cell), xl / xr (their transverse
    // parts: the correction weighted by m3)
    auto edge = [&](double w, double wi, double s, double cf, double& dL, double& dR, double& xl, double& xr,
                    auto sgn) {
      constexpr int SG = decltype(sgn)::value;
      // (every product and sum rounded on its own or as an explicit fma: the same bits in every
      // instantiation -- the m = 8 patch sweep and the quad blocks' T = 16 sweep)
      const double f = CV_MUL(cf, limited(w, wi));
      if (SG > 0) {
        dL = f;
        dR = fma(s, w, -f);
        if (MT2) { xl = dL; xr = dR; }
        else { xl = CV_MUL(m3, f); xr = fma(s, w, -CV_MUL(m3, f)); }
      } else {
        dL = fma(s, w, f);
        dR = -f;
        if (MT2) { xl = dL; xr = dR; }
        else { xl = fma(s, w, CV_MUL(m3, f)); xr = -CV_MUL(m3, f); }
      }
    };
    using SXc = std::integral_constant<int, SX>;
    using SYc = std::integral_constant<int, SY>;
    double qa[4], qb[4];                  // columns c0, c0 + 1: rows j-1 .. j+2
    qa[1] = ld(1, -1); qa[2] = ld(1, 0); qa[3] = ld(1, 1);
    qb[1] = ld(2, -1); qb[2] = ld(2, 0); qb[3] = ld(2, 1);
    qa[0] = qb[0] = 0.0;
    double Xa1 = 0, Xa2 = 0, Xb1 = 0, Xb2 = 0;       // X(c, j-1), X(c, j-2)
    double Xfa = 0, Xfb = 0;                         // Xf(c, j-1)
    double Ya = 0, Yb = 0, Yl = 0, Yr = 0, Yfa = 0, Yfb = 0;   // Y(c0 / c0+1 / c0-1 / c0+2, j-1), Yf
    double yra = 0, yrb = 0, dRya = 0, dRyb = 0, wya = 0, wyb = 0;   // last y-edge's parts, its jump
    double dR0p = 0, dL0p = 0, dRh_a = 0, dRh_b = 0, dLt_a = 0, dLt_b = 0;   // (reflux records only)
    // one row j of the sweep; F: which parts exist at this j (peeled first / last rows)
    constexpr int LD = 1, UPD = 2, YE = 4, YS = 8, J0 = 16;
    auto iter = [&](int j, auto flags) {
      constexpr int F = decltype(flags)::value;
      qa[0] = qa[1]; qa[1] = qa[2]; qa[2] = qa[3];
      qb[0] = qb[1]; qb[1] = qb[2]; qb[2] = qb[3];
      if (F & LD) { qa[3] = ld(1, j + 2); qb[3] = ld(2, j + 2); }
      // x-edges c0 + 1/2 and c0 + 3/2 of row j
      const double qm = ld(0, j), qc = ld(3, j), qd = ld(4, j);
      const double w0 = qb[1] - qa[1], w1 = qc - qb[1];
      const double wi0 = SX > 0 ? qa[1] - qm : w1, wi1 = SX > 0 ? w0 : qd - qc;
      double dL0, dR0, xl0, xr0, dL1, dR1, xl1, xr1;
      edge(w0, wi0, u0, cfx, dL0, dR0, xl0, xr0, SXc{});
      edge(w1, wi1, u0, cfx, dL1, dR1, xl1, xr1, SXc{});
      const double xrL = __shfl_up_sync(0xffffffffu, xr1, 1);
      const double dRL = MT2 ? xrL : __shfl_up_sync(0xffffffffu, dR1, 1);
      const double Xa = CV_ADD(xrL, xl0), Xb = CV_ADD(xr0, xl1);
      const double Xfa0 = MT2 ? Xa : CV_ADD(dRL, dL0), Xfb0 = MT2 ? Xb : CV_ADD(dR0, dL1);
      if (F & UPD) {   // update of row j - 1
        const int jr = j - 1;
        const double ta = fma(ky, SY > 0 ? Xa1 - Xa2 : Xa - Xa1,
                              fma(kx, SX > 0 ? Ya - Yl : Yb - Ya, CV_ADD(Xfa, Yfa)));
        const double tb = fma(ky, SY > 0 ? Xb1 - Xb2 : Xb - Xb1,
                              fma(kx, SX > 0 ? Yb - Ya : Yr - Yb, CV_ADD(Xfb, Yfb)));
        const double va = fma(-r, ta, qa[0]), vb = fma(-r, tb, qb[0]);
        const bool sa_ = live && c0 >= 1, sb_ = live && c0 + 1 <= T;
        if (sa_) out[oidx(c0 - 1, jr - 1)] = va;
        if (sb_) out[oidx(c0, jr - 1)] = vb;
        chk = fma(sa_ ? va : 0.0, 0.0, fma(sb_ ? vb : 0.0, 0.0, chk));
        if (RF && rec) {   // the same face fluxes k_step_sc records (F~ / G~ transverse at the face)
          if (k == 0) reg[jr - 1] = (dR0p - kx * (SX > 0 ? Ya : Yb)) - u0 * qb[0];                 // x-low, i = 1
          if (k == LP - 1) reg[T + jr - 1] = u0 * qa[0] + (dL0p + kx * (SX > 0 ? Ya : Yb));       // x-high, i = T
          if (jr == 1) {                                                                          // y-low, j = 1
            if (c0 >= 1) reg[2 * T + c0 - 1] = (dRh_a - ky * (SY > 0 ? Xa2 : Xa1)) - v0 * qa[0];
            if (c0 + 1 <= T) reg[2 * T + c0] = (dRh_b - ky * (SY > 0 ? Xb2 : Xb1)) - v0 * qb[0];
          }
          if (jr == T) {                                                                          // y-high, j = T
            if (c0 >= 1) reg[3 * T + c0 - 1] = v0 * qa[0] + (dLt_a + ky * (SY > 0 ? Xa1 : Xa));
            if (c0 + 1 <= T) reg[3 * T + c0] = v0 * qb[0] + (dLt_b + ky * (SY > 0 ? Xb1 : Xb));
          }
        }
      }
      if (F & YE) {    // y-edges (c, j + 1/2)
        const double wa = qa[2] - qa[1], wb = qb[2] - qb[1];
        const double wia = SY > 0 ? ((F & J0) ? qa[1] - qa[0] : wya) : qa[3] - qa[2];
        const double wib = SY > 0 ? ((F & J0) ? qb[1] - qb[0] : wyb) : qb[3] - qb[2];
        double dLa, dRa, yla, yra_, dLb, dRb, ylb, yrb_;
        edge(wa, wia, v0, cfy, dLa, dRa, yla, yra_, SYc{});
        edge(wb, wib, v0, cfy, dLb, dRb, ylb, yrb_, SYc{});
        if (F & YS) {
          Ya = CV_ADD(yra, yla); Yb = CV_ADD(yrb, ylb);
          Yfa = MT2 ? Ya : CV_ADD(dRya, dLa); Yfb = MT2 ? Yb : CV_ADD(dRyb, dLb);
          Yl = __shfl_up_sync(0xffffffffu, Yb, 1);
          Yr = __shfl_down_sync(0xffffffffu, Ya, 1);
        }
        yra = yra_; yrb = yrb_; dRya = dRa; dRyb = dRb; wya = wa; wyb = wb;
        if (RF) {
          if (F & J0) { dRh_a = dRa; dRh_b = dRb; }
          dLt_a = dLa; dLt_b = dLb;
        }
      }
      Xa2 = Xa1; Xa1 = Xa; Xb2 = Xb1; Xb1 = Xb; Xfa = Xfa0; Xfb = Xfb0;
      if (RF) { dR0p = dR0; dL0p = dL0; }
    };
    iter(0, std::integral_constant<int, LD | YE | J0>{});
    iter(1, std::integral_constant<int, LD | YE | YS>{});
#if CV_UNROLL == 1
#pragma unroll 1
#elif CV_UNROLL == 2
#pragma unroll 2
#elif CV_UNROLL == 3
#pragma unroll 3
#else
#pragma unroll
#endif
    for (int j = 2; j <= T; ++j) iter(j, std::integral_constant<int, LD | UPD | YE | YS>{});
    iter(T + 1, std::integral_constant<int, UPD>{});
    __syncwarp();   // the staging buffer is refilled by a later group
    if (NB == 1) issue_next();
  }
  const bool bad = __any_sync(0xffffffffu, chk != chk);
  if (bad || cfl != cfl) cfl = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) cfl = fmax(cfl, __shfl_xor_sync(0xffffffffu, cfl, o));
  if (lane == 0) atomicMax(A.cfl_bits, (unsigned long long)__double_as_longlong(cfl));
}

// ---------------------------------------------------------------------------------------------
// Capacity-form advection with edge velocities (C4 / T4 physics), register sweep: the layout of
// k_step_cv (PW patches per warp, lane k owns columns 2k, 2k+1, one pass over rows 0..T+1), with
// per-edge speeds and per-cell r = dt / (kappa dx).  The transverse parts regroup per cell as
//   U = h r max(v_top, 0) X,  D = h r min(v_bot, 0) X,  R = h r max(u_right, 0) Y,  L = h r min(u_left, 0) Y
// (h = -1/2, X / Y as in k_step_cv; the receiving cell's own edge velocities, PAPER.md:168-171 /
// reading 24), and
//   q_new = q - r [Xf + Yf + R + L_{i+1} - R_{i-1} - L + U + D_{j+1} - U_{j-1} - D].
// q is staged in shared memory as in k_step_cv; the three aux fields are read from global memory
// one row ahead (read-only path), kappa's reciprocal is formed once per cell.  CFL: every x-edge
// i - 1/2, i = 1..T+1, of rows 0..T+1 and every y-edge of columns 0..T+1 (k_step_sc's set).
#ifndef CVC_MINB
#define CVC_MINB 12
#endif
#ifndef CVC_UNROLL
#define CVC_UNROLL 1
#endif
template <int T, bool MT2, int NB>
__global__ void __launch_bounds__(32, CVC_MINB) k_step_cvc(StepArgs A, int npatch) {
  using C = CvShape<T>;
  constexpr int W = C::W, WW = C::WW, LP = C::LP, PW = C::PW;
  extern __shared__ __align__(128) double sm[];     // [NB][PW][WW]
  __shared__ __align__(8) uint64_t bars[NB];
  const int lane = threadIdx.x;
  if (A.active) npatch = *A.nactive;
  const int ngroups = (npatch + PW - 1) / PW;
  auto patch_of = [&](int idx) { return A.active ? A.active[idx] : idx; };
  auto nbload = [&](int g) { return g < ngroups ? cv_nb_load<T>(A, g * PW, min(PW, npatch - g * PW), lane) : CvNb{-1, -1}; };
  auto stage = [&](int g, int s, const CvNb& nb) {
    cv_stage<T>(A, sm + (size_t)s * PW * WW, &bars[s], lane, g * PW, min(PW, npatch - g * PW), nb);
  };
  if (lane == 0) {
    for (int q = 0; q < NB; ++q) mbar_init(&bars[q], 1);
    fence_proxy_async();
  }
  __syncwarp();
  for (int q = 0; q < (NB > 1 ? NB - 1 : 1); ++q) {
    const int g = blockIdx.x + q * gridDim.x;
    if (g < ngroups) stage(g, q, nbload(g));
    else cp_async_commit();
  }
  const int p = lane / LP, k = lane - p * LP, c0 = 2 * k;
  const bool trans = A.method3 >= 1, second = A.method2 == 2;
  const double m3 = A.method3 == 2 ? 1.0 : 0.0, h = trans ? -0.5 : 0.0;
  const double lp1 = A.lp1, lp2 = A.lp2, lk3 = A.lk3;
  auto limited = [&](double w, double wi) { return cv_limited(w, wi, lp1, lp2, lk3); };   // as k_step_cv
  double cfl = 0.0, chk = 0.0;
  int it = 0;
  for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
    const int b = it % NB;
    const int cnt = min(PW, npatch - g * PW);
    const int mypatch = lane < cnt ? patch_of(g * PW + lane) : 0;
    const int mylevel = A.level[mypatch];
    const int mybc = (A.ring && lane < cnt) ? A.bcflag[mypatch] : 0;
    const CvNb nbn = A.ring ? nbload(g + (NB > 1 ? NB - 1 : 1) * gridDim.x) : CvNb{-1, -1};
    mbar_wait(&bars[b], (uint32_t)((it / NB) & 1));
    cp_async_wait<(NB > 1 ? NB - 2 : 0)>();
    __syncwarp();
    auto issue_next = [&]() {
      const int gn = g + (NB > 1 ? NB - 1 : 1) * gridDim.x, bn = (it + NB - 1) % NB;
      if (gn < ngroups) {
        fence_proxy_async();
        stage(gn, bn, nbn);
      } else {
        cp_async_commit();
      }
    };
    if (NB > 1) issue_next();
    if (A.ring) cv_bcs<T>(A, sm + (size_t)b * PW * WW, mypatch, mybc, lane);
    const bool live = p < cnt;
    const int patch = __shfl_sync(0xffffffffu, mypatch, live ? p : 0);
    const int level = __shfl_sync(0xffffffffu, mylevel, live ? p : 0);
    const double* sq = sm + ((size_t)b * PW + (live ? p : 0)) * WW;
    const double* col[5];
#pragma unroll
    for (int e = 0; e < 5; ++e) col[e] = sq + min(c0 - 1 + e, T + 2) + 1;
    auto ld = [&](int e, int j) { return col[e][(j + 1) * W]; };
    // aux (natural [3][W][W]): kappa, u~ (left edge of the cell), v~ (bottom edge)
    const double* ax = A.aux + (int64_t)patch * 3 * WW;
    const int ca = c0 + 1, cb = min(c0 + 2, T + 2);   // natural column offsets of c0 and c0 + 1 (+1)
    auto kap = [&](int cc, int j) { return __ldg(ax + (j + 1) * W + cc); };
    auto uu = [&](int cc, int j) { return __ldg(ax + WW + (j + 1) * W + cc); };
    auto vv = [&](int cc, int j) { return __ldg(ax + 2 * WW + (j + 1) * W + cc); };
    const double dtdx = A.dt / ldexp(A.dx0, -level);   // (the table lookup costs this kernel 5 spills, T4 +10 %)
    double* out = A.qnew + (int64_t)patch * WW;
    // edge parts from (w, upwind candidates, speed, r of the low / high cell); CFL when counted
    auto edge = [&](double w, double wup_lo, double wup_hi, double s, double rl, double rh, bool count,
                    double& dL, double& dR, double& xl, double& xr) {
      if (count && live) cfl = fmax(cfl, fmax(rh * s, -rl * s));
      const double as = fabs(s);
      const double cf = second ? 0.5 * as * (1.0 - as * (0.5 * (rl + rh))) : 0.0;
      const double f = cf * limited(w, s > 0.0 ? wup_lo : wup_hi);
      const double sp = s > 0.0 ? s : 0.0, sn = s - sp;
      dL = fma(sn, w, f);
      dR = fma(sp, w, -f);
      if (MT2) { xl = dL; xr = dR; }
      else { xl = fma(sn, w, m3 * f); xr = fma(sp, w, -(m3 * f)); }
    };
    double qa[4], qb[4];
    qa[1] = ld(1, -1); qa[2] = ld(1, 0); qa[3] = ld(1, 1);
    qb[1] = ld(2, -1); qb[2] = ld(2, 0); qb[3] = ld(2, 1);
    qa[0] = qb[0] = 0.0;
    double ra = dtdx * fast_rcp(kap(ca, 0)), rb = dtdx * fast_rcp(kap(cb, 0));   // r at row j (j = 0)
    double Ua1 = 0, Ua2 = 0, Ub1 = 0, Ub2 = 0, Da1 = 0, Db1 = 0;   // U(j-1), U(j-2), D(j-1)
    double Xfa = 0, Xfb = 0, Yfa = 0, Yfb = 0, Ra = 0, Rb = 0, La = 0, Lb = 0, Rl = 0, Lr = 0;
    double yra = 0, yrb = 0, dRya = 0, dRyb = 0, wya = 0, wyb = 0, vba = 0, vbb = 0;   // last y-edge
    double ra1 = 0, rb1 = 0;                                        // r(j - 1)
    vba = vv(ca, 0); vbb = vv(cb, 0);                                // v~ at the bottom of row 0
    // aux one row ahead of its use (global-load latency): u~ of the row, v~ and kappa of the row above
    const int cu2 = min(c0 + 3, T + 3);
    double u1c = uu(ca + 1, 0), u2c = uu(cu2, 0), vtca = vv(ca, 1), vtcb = vv(cb, 1), kca = kap(ca, 1),
           kcb = kap(cb, 1);
    constexpr int LD = 1, UPD = 2, YE = 4, YS = 8, J0 = 16;
    auto iter = [&](int j, auto flags) {
      constexpr int F = decltype(flags)::value;
      qa[0] = qa[1]; qa[1] = qa[2]; qa[2] = qa[3];
      qb[0] = qb[1]; qb[1] = qb[2]; qb[2] = qb[3];
      if (F & LD) { qa[3] = ld(1, j + 2); qb[3] = ld(2, j + 2); }
      const double u1 = u1c, u2 = u2c;
      double vta = 0, vtb = 0, ra_n = 0, rb_n = 0;
      if (F & YE) {
        vta = vtca; vtb = vtcb;
        ra_n = dtdx * fast_rcp(kca); rb_n = dtdx * fast_rcp(kcb);
      }
      if (j + 1 <= T + 1) { u1c = uu(ca + 1, j + 1); u2c = uu(cu2, j + 1); }   // (the next row's)
      if (j + 2 <= T + 1) { vtca = vv(ca, j + 2); vtcb = vv(cb, j + 2); kca = kap(ca, j + 2); kcb = kap(cb, j + 2); }
      const double rc = __shfl_down_sync(0xffffffffu, ra, 1);          // r of column c0 + 2
      const double uL = __shfl_up_sync(0xffffffffu, u2, 1);            // u~ at c0 - 1/2 (left lane)
      // x-edges c0 + 1/2, c0 + 3/2 of row j (the second one of the last lane is outside the set)
      const double qm = ld(0, j), qc = ld(3, j), qd = ld(4, j);
      const double w0 = qb[1] - qa[1], w1 = qc - qb[1];
      double dL0, dR0, xl0, xr0, dL1, dR1, xl1, xr1;
      edge(w0, qa[1] - qm, w1, u1, ra, rb, true, dL0, dR0, xl0, xr0);
      edge(w1, w0, qd - qc, u2, rb, rc, k < LP - 1, dL1, dR1, xl1, xr1);
      const double xrL = __shfl_up_sync(0xffffffffu, xr1, 1);
      const double dRL = MT2 ? xrL : __shfl_up_sync(0xffffffffu, dR1, 1);
      const double Xa = xrL + xl0, Xb = xr0 + xl1;
      const double Xfa0 = MT2 ? Xa : dRL + dL0, Xfb0 = MT2 ? Xb : dR0 + dL1;
      // U(j) needs v~ at the top of row j (the y-edge j + 1/2), D(j) the bottom one
      const double Ua = h * ra * fmax(F & YE ? vta : 0.0, 0.0) * Xa, Ub = h * rb * fmax(F & YE ? vtb : 0.0, 0.0) * Xb;
      const double Da = h * ra * fmin(vba, 0.0) * Xa, Db = h * rb * fmin(vbb, 0.0) * Xb;
      if (F & UPD) {   // row j - 1
        const int jr = j - 1;
        const double ta = Xfa + Yfa + (Ra + Lb - Rl - La) + (Ua1 + Da - Ua2 - Da1);
        const double tb = Xfb + Yfb + (Rb + Lr - Ra - Lb) + (Ub1 + Db - Ub2 - Db1);
        const double va = fma(-ra1, ta, qa[0]), vb = fma(-rb1, tb, qb[0]);
        const bool sa_ = live && c0 >= 1, sb_ = live && c0 + 1 <= T;
        if (sa_) out[(jr - 1) * T + c0 - 1] = va;
        if (sb_) out[(jr - 1) * T + c0] = vb;
        chk = fma(sa_ ? va : 0.0, 0.0, fma(sb_ ? vb : 0.0, 0.0, chk));
      }
      if (F & YE) {    // y-edges (c, j + 1/2)
        const double wa = qa[2] - qa[1], wb = qb[2] - qb[1];
        const double wla = (F & J0) ? qa[1] - qa[0] : wya, wlb = (F & J0) ? qb[1] - qb[0] : wyb;
        double dLa, dRa, yla, yra_, dLb, dRb, ylb, yrb_;
        edge(wa, wla, qa[3] - qa[2], vta, ra, ra_n, true, dLa, dRa, yla, yra_);
        edge(wb, wlb, qb[3] - qb[2], vtb, rb, rb_n, true, dLb, dRb, ylb, yrb_);
        if (F & YS) {
          const double Ya = yra + yla, Yb = yrb + ylb;
          Yfa = MT2 ? Ya : dRya + dLa; Yfb = MT2 ? Yb : dRyb + dLb;
          Ra = h * ra * fmax(u1, 0.0) * Ya; Rb = h * rb * fmax(u2, 0.0) * Yb;
          La = h * ra * fmin(uL, 0.0) * Ya; Lb = h * rb * fmin(u1, 0.0) * Yb;
          Rl = __shfl_up_sync(0xffffffffu, Rb, 1);      // R of column c0 - 1
          Lr = __shfl_down_sync(0xffffffffu, La, 1);    // L of column c0 + 2
        }
        yra = yra_; yrb = yrb_; dRya = dRa; dRyb = dRb; wya = wa; wyb = wb;
      }
      Ua2 = Ua1; Ua1 = Ua; Ub2 = Ub1; Ub1 = Ub; Da1 = Da; Db1 = Db; Xfa = Xfa0; Xfb = Xfb0;
      ra1 = ra; rb1 = rb;
      if (F & YE) { ra = ra_n; rb = rb_n; vba = vta; vbb = vtb; }
    };
    iter(0, std::integral_constant<int, LD | YE | J0>{});
    iter(1, std::integral_constant<int, LD | YE | YS>{});
#if CVC_UNROLL == 1
#pragma unroll 1
#elif CVC_UNROLL == 2
#pragma unroll 2
#else
#pragma unroll
#endif
    for (int j = 2; j <= T; ++j) iter(j, std::integral_constant<int, LD | UPD | YE | YS>{});
    iter(T + 1, std::integral_constant<int, UPD>{});
    __syncwarp();
    if (NB == 1) issue_next();
  }
  const bool bad = __any_sync(0xffffffffu, chk != chk);
  if (bad || cfl != cfl) cfl = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) cfl = fmax(cfl, __shfl_xor_sync(0xffffffffu, cfl, o));
  if (lane == 0) atomicMax(A.cfl_bits, (unsigned long long)__double_as_longlong(cfl));
}

// ---------------------------------------------------------------------------------------------
// Quiescent-patch filter for the fused (ring-gather) path, three kernels per step:
//   k_copy_classify  q_new interior = q_old interior (streaming, 16-byte accesses) and, per patch,
//                    "interior uniform" + its state;
//   k_activity       a patch is quiescent iff it is uniform, every patch its ring reads is uniform
//                    with the same state, and no wall negates a non-zero component of it: then its
//                    staged window is uniform, every wave of its update is exactly 0 and q_new = q
//                    (already copied); its CFL comes from the state.  Others go to the active list;
//   k_step           over the active list only.
#ifndef COPY_V256
#define COPY_V256 1
#endif
// (tuning knobs; measured on C5: 8 x 32-byte loads in flight per lane at 2 CTAs/SM is best --
// 3 CTAs/SM 0.747 ms, 4 loads per lane 0.755 ms, vs 0.714 ms; tools/copy_variants.sh)
#ifndef COPY_MINB
#define COPY_MINB 1
#endif
#ifndef COPY_NC4
#define COPY_NC4 8
#endif
template <int MEQN, int T>
__global__ void __launch_bounds__(256, COPY_MINB) k_copy_classify(const double* __restrict__ qold, double* __restrict__ qnew,
                                                       int npatch, uint8_t* __restrict__ uflag,
                                                       double* __restrict__ uval) {
  // One warp per patch (T = m here).  The storage keeps each (patch, component) interior as one
  // dense m x m block (qcell): exactly the interior is copied, contiguous 16-byte accesses, so DRAM
  // traffic is the compulsory read + write of q.  Each lane issues up to 16 loads before using any.
  constexpr int n = T + 4, n2 = n * n, H = T * T / 2;       // double2 per interior block
  constexpr int E = MEQN * H, NE = (E + 31) / 32, NC = NE < 16 ? NE : 16;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < npatch; p += warps) {
    const double* src = qold + (int64_t)p * MEQN * n2;
    double* dst = qnew + (int64_t)p * MEQN * n2;
    double v0[MEQN];
#pragma unroll
    for (int k = 0; k < MEQN; ++k) v0[k] = __ldg(src + k * n2);
    bool diff = false;
#if COPY_V256
    // 32-byte accesses (LDG/STG.E.ENL2.256 on sm_100a): 4 doubles per lane and access
    constexpr int Q4 = T * T / 4, E4 = MEQN * Q4, NE4 = (E4 + 31) / 32, NC4 = NE4 < COPY_NC4 ? NE4 : COPY_NC4;
#pragma unroll 1
    for (int base = 0; base < E4; base += 32 * NC4) {
      double x[NC4][4];
#pragma unroll
      for (int u = 0; u < NC4; ++u) {
        const int e = base + lane + 32 * u;
        const int k = e / Q4, c4 = e - k * Q4;
        if (e < E4)
          asm volatile("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];"
                       : "=d"(x[u][0]), "=d"(x[u][1]), "=d"(x[u][2]), "=d"(x[u][3])
                       : "l"(src + k * n2 + 4 * c4));
      }
#pragma unroll
      for (int u = 0; u < NC4; ++u) {
        const int e = base + lane + 32 * u;
        if (e < E4) {
          const int k = e / Q4, c4 = e - k * Q4;
          asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst + k * n2 + 4 * c4), "d"(x[u][0]),
                       "d"(x[u][1]), "d"(x[u][2]), "d"(x[u][3])
                       : "memory");
          diff |= (x[u][0] != v0[k]) | (x[u][1] != v0[k]) | (x[u][2] != v0[k]) | (x[u][3] != v0[k]);
        }
      }
    }
    (void)NC;
#else
#pragma unroll 1
    for (int base = 0; base < E; base += 32 * NC) {
      double2 x[NC];
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int e = base + lane + 32 * u;
        const int k = e / H, c2 = e - k * H;
        if (e < E) x[u] = __ldcs(reinterpret_cast<const double2*>(src + k * n2) + c2);
      }
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int e = base + lane + 32 * u;
        if (e < E) {
          const int k = e / H, c2 = e - k * H;
          __stcs(reinterpret_cast<double2*>(dst + k * n2) + c2, x[u]);
          diff |= (x[u].x != v0[k]) | (x[u].y != v0[k]);
        }
      }
    }
#endif
    const bool uni = !__any_sync(0xffffffffu, diff);
    if (lane == 0) uflag[p] = uni ? 1 : 0;
    if (lane < MEQN) uval[(int64_t)p * MEQN + lane] = v0[lane < MEQN ? lane : 0];
  }
}

template <class S>
__global__ void __launch_bounds__(256) k_activity(int npatch, const uint8_t* __restrict__ uflag,
                                                  const double* __restrict__ uval, const int32_t* __restrict__ nbr,
                                                  const uint8_t* __restrict__ negmask, const int8_t* __restrict__ level,
                                                  double dt, double dx0, SolverParams sp, int32_t* __restrict__ active,
                                                  int32_t* __restrict__ nactive, unsigned long long* cfl_bits) {
  constexpr int MEQN = S::MEQN;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double cfl = 0.0;
  bool act = false;
  if (p < npatch) {
    bool q = uflag[p] != 0;
    double v[MEQN];
#pragma unroll
    for (int k = 0; k < MEQN; ++k) v[k] = uval[(int64_t)p * MEQN + k];
    const uint8_t nm = negmask[p];
#pragma unroll
    for (int k = 0; k < MEQN; ++k)
      if (((nm >> k) & 1) && v[k] != 0.0) q = false;
#pragma unroll
    for (int s = 0; s < 8 && q; ++s) {
      const int32_t o = nbr[(int64_t)p * 8 + s];
      if (o == -1) continue;
      if (o < 0 || !uflag[o]) { q = false; break; }
#pragma unroll
      for (int k = 0; k < MEQN; ++k)
        if (uval[(int64_t)o * MEQN + k] != v[k]) q = false;
    }
    if (q) {
      const double dtdx = dt / ldexp(dx0, -(int)level[p]);
      // Roe systems: the warp-sweep kernel's own CFL arithmetic for a uniform window (bitwise the
      // full update's value, so both modes follow the same dt sequence); others: the state's speeds
      if constexpr (std::is_same<S, EulerRoe>::value) cfl = ws_quiescent_cfl<WsEuler>(v, 1, sp, dtdx);
      else if constexpr (std::is_same<S, SweRoe>::value) cfl = ws_quiescent_cfl<WsSwe>(v, 1, sp, dtdx);
      else cfl = S::quiescent_cfl(v, 1, sp, nullptr, dtdx, 0, 0, 0, 1);
    } else {
      act = true;
    }
  }
  // warp-aggregated append to the active list
  const unsigned mask = __ballot_sync(0xffffffffu, act);
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == 0 && mask) base = atomicAdd(nactive, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (act) active[base + __popc(mask & ((1u << lane) - 1u))] = p;
  if (cfl != cfl) cfl = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) cfl = fmax(cfl, __shfl_xor_sync(0xffffffffu, cfl, o));
  __shared__ double wmax[8];
  if (lane == 0) wmax[threadIdx.x >> 5] = cfl;
  __syncthreads();
  if (threadIdx.x == 0) {
    double c = wmax[0];
    for (int w = 1; w < 8; ++w) c = fmax(c, wmax[w]);
    if (c > 0.0) atomicMax(cfl_bits, (unsigned long long)__double_as_longlong(c));
  }
}

template <class S>
static int launch_filter_s(const double* qold, double* qnew, int npatch, int m, uint8_t* uflag, double* uval,
                           const int32_t* nbr, const uint8_t* negmask, const int8_t* level, double dt,
                           double dx0, SolverParams sp, int32_t* active, int32_t* nactive,
                           unsigned long long* cfl_bits, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1) {
  if (npatch <= 0) return 0;
  const int blocks_copy = 148 * 8;
  if (e0) cudaEventRecord(e0, st);
  switch (m) {
    case 32: k_copy_classify<S::MEQN, 32><<<blocks_copy, 256, 0, st>>>(qold, qnew, npatch, uflag, uval); break;
    case 16: k_copy_classify<S::MEQN, 16><<<blocks_copy, 256, 0, st>>>(qold, qnew, npatch, uflag, uval); break;
    case 8: k_copy_classify<S::MEQN, 8><<<blocks_copy, 256, 0, st>>>(qold, qnew, npatch, uflag, uval); break;
    case 4: k_copy_classify<S::MEQN, 4><<<blocks_copy, 256, 0, st>>>(qold, qnew, npatch, uflag, uval); break;
    default: return -1;
  }
  if (e1) cudaEventRecord(e1, st);
  k_activity<S><<<(npatch + 255) / 256, 256, 0, st>>>(npatch, uflag, uval, nbr, negmask, level, dt, dx0, sp,
                                                       active, nactive, cfl_bits);
  return 2;
}

int launch_filter(int kind, const double* qold, double* qnew, int npatch, int m, uint8_t* uflag, double* uval,
                  const int32_t* nbr, const uint8_t* negmask, const int8_t* level, double dt, double dx0,
                  double p0, double p1, int32_t* active, int32_t* nactive, unsigned long long* cfl_bits,
                  cudaStream_t st, cudaEvent_t ev_before_copy, cudaEvent_t ev_after_copy) {
  SolverParams sp;
  sp.p0 = p0;
  sp.p1 = p1;
  switch (kind) {
    case FC_ADV_CONST:
      return launch_filter_s<AdvConst>(qold, qnew, npatch, m, uflag, uval, nbr, negmask, level, dt, dx0, sp,
                                       active, nactive, cfl_bits, st, ev_before_copy, ev_after_copy);
    case FC_SWE_ROE:
      return launch_filter_s<SweRoe>(qold, qnew, npatch, m, uflag, uval, nbr, negmask, level, dt, dx0, sp,
                                     active, nactive, cfl_bits, st, ev_before_copy, ev_after_copy);
    case FC_EULER_ROE:
      return launch_filter_s<EulerRoe>(qold, qnew, npatch, m, uflag, uval, nbr, negmask, level, dt, dx0, sp,
                                       active, nactive, cfl_bits, st, ev_before_copy, ev_after_copy);
    case FC_EULER_HLLE:
      return launch_filter_s<EulerHlle>(qold, qnew, npatch, m, uflag, uval, nbr, negmask, level, dt, dx0, sp,
                                        active, nactive, cfl_bits, st, ev_before_copy, ev_after_copy);
  }
  return -1;   // capacity form: edge-dependent CFL, no patch filter
}

// ---------------------------------------------------------------------------------------------
template <class S, int T, int NT, int MINB, bool RF>
static int launch_step_t(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  const size_t smem = StepShape<S, T>::smem_bytes;
  static int resident_dev[64] = {};   // per device: CTAs that fit at once (persistent grid)
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (dev_ < 0 || dev_ >= 64) return -1;
  int& resident = resident_dev[dev_];
  if (!resident) {   // (function attributes are per device)
    cudaFuncSetAttribute(k_step<S, T, NT, MINB, RF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_step<S, T, NT, MINB, RF>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step<S, T, NT, MINB, RF>, NT, smem);
    resident = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int64_t ntiles = npatch * a.tiles * a.tiles;
  if (ntiles >= (1ll << 31)) return -1;
  const int64_t grid = ntiles < resident ? ntiles : resident;   // (active list: at most ntiles)
  StepArgs b = a;
  b.fbuf = nullptr;
  if (a.method3 == 1) {      // F~ scratch for the (rare) method3 = 1 transverse variant: one per
    // (device, stream) for the process lifetime (resident CTAs x E2), so handles stepping on
    // different streams never share it; launches on one stream are ordered
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, double*> bufs;
    std::lock_guard<std::mutex> lock(mu);
    double*& fb = bufs[std::make_pair(dev_, st)];
    if (!fb && cudaMalloc(&fb, (size_t)resident * S::MEQN * StepShape<S, T>::E2 * sizeof(double)) != cudaSuccess) {
      fb = nullptr;
      return -1;
    }
    b.fbuf = fb;
  }
  k_step<S, T, NT, MINB, RF><<<(unsigned)grid, NT, smem, st>>>(b, (int)ntiles);
  return 1;
}

template <class S, int T, bool RF>
static int launch_sc_t(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  constexpr int NT = T * T < 32 ? 32 : T * T;
  constexpr int NXE = (T + 1) * (T + 2);
  const size_t smem = ((size_t)sc_nbuf<S>() * StepShape<S, T>::BUF + 2 * (size_t)StepShape<S, T>::WW +
                       12 * (size_t)NXE) * sizeof(double);
  static int resident_dev[64] = {};
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (dev_ < 0 || dev_ >= 64) return -1;
  int& resident = resident_dev[dev_];
  if (!resident) {
    cudaFuncSetAttribute(k_step_sc<S, T, NT, RF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_step_sc<S, T, NT, RF>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step_sc<S, T, NT, RF>, NT, smem);
    resident = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int64_t ntiles = npatch * a.tiles * a.tiles;
  if (ntiles >= (1ll << 31)) return -1;
  const int64_t grid = ntiles < resident ? ntiles : resident;
  k_step_sc<S, T, NT, RF><<<(unsigned)grid, NT, smem, st>>>(a, (int)ntiles);
  return 1;
}

#ifndef CV_NB
#define CV_NB 1
#endif
template <int T, int SX, int SY, bool MT2, bool RF = false, bool QD = false>
static int launch_cv_t(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  constexpr int NB = CV_NB;
  using C = CvShape<T>;
  const size_t smem = (size_t)NB * C::PW * C::WW * sizeof(double);
  static int resident_dev[64] = {};
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (dev_ < 0 || dev_ >= 64) return -1;
  int& resident = resident_dev[dev_];
  if (!resident) {
    cudaFuncSetAttribute(k_step_cv<T, SX, SY, MT2, NB, RF, QD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_step_cv<T, SX, SY, MT2, NB, RF, QD>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step_cv<T, SX, SY, MT2, NB, RF, QD>, 32, smem);
    resident = sms * (per_sm > 0 ? per_sm : 1);
  }
  if (npatch >= (1ll << 31)) return -1;
  const int64_t groups = (npatch + C::PW - 1) / C::PW;
  const int64_t grid = groups < resident ? groups : resident;
  k_step_cv<T, SX, SY, MT2, NB, RF, QD><<<(unsigned)grid, 32, smem, st>>>(a, (int)npatch);
  return 1;
}

template <int T, bool MT2>
static int launch_cvc_t(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  constexpr int NB = CV_NB;
  using C = CvShape<T>;
  const size_t smem = (size_t)NB * C::PW * C::WW * sizeof(double);
  static int resident_dev[64] = {};
  int dev_ = 0;
  cudaGetDevice(&dev_);
  if (dev_ < 0 || dev_ >= 64) return -1;
  int& resident = resident_dev[dev_];
  if (!resident) {
    cudaFuncSetAttribute(k_step_cvc<T, MT2, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_step_cvc<T, MT2, NB>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step_cvc<T, MT2, NB>, 32, smem);
    resident = sms * (per_sm > 0 ? per_sm : 1);
  }
  if (npatch >= (1ll << 31)) return -1;
  const int64_t groups = (npatch + C::PW - 1) / C::PW;
  const int64_t grid = groups < resident ? groups : resident;
  k_step_cvc<T, MT2, NB><<<(unsigned)grid, 32, smem, st>>>(a, (int)npatch);
  return 1;
}

// quad blocks (cv_stage_quad): npatch / 4 units of the T = 16 sweep
static int launch_cv_quad(const StepArgs& a, int64_t nblk, cudaStream_t st) {
  const bool px = a.sp.p0 > 0.0, py = a.sp.p1 > 0.0;
  if (a.method3 == 2) {
    if (px) return py ? launch_cv_t<16, 1, 1, true, false, true>(a, nblk, st) : launch_cv_t<16, 1, -1, true, false, true>(a, nblk, st);
    return py ? launch_cv_t<16, -1, 1, true, false, true>(a, nblk, st) : launch_cv_t<16, -1, -1, true, false, true>(a, nblk, st);
  }
  if (px) return py ? launch_cv_t<16, 1, 1, false, false, true>(a, nblk, st) : launch_cv_t<16, 1, -1, false, false, true>(a, nblk, st);
  return py ? launch_cv_t<16, -1, 1, false, false, true>(a, nblk, st) : launch_cv_t<16, -1, -1, false, false, true>(a, nblk, st);
}

template <int T>
static int launch_cv(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  const bool px = a.sp.p0 > 0.0, py = a.sp.p1 > 0.0, mt2 = a.method3 == 2;
  if (a.rslot) {   // reflux records (method3 = 2 only; others go to k_step_sc)
    if (px) return py ? launch_cv_t<T, 1, 1, true, true>(a, npatch, st) : launch_cv_t<T, 1, -1, true, true>(a, npatch, st);
    return py ? launch_cv_t<T, -1, 1, true, true>(a, npatch, st) : launch_cv_t<T, -1, -1, true, true>(a, npatch, st);
  }
  if (mt2) {
    if (px) return py ? launch_cv_t<T, 1, 1, true>(a, npatch, st) : launch_cv_t<T, 1, -1, true>(a, npatch, st);
    return py ? launch_cv_t<T, -1, 1, true>(a, npatch, st) : launch_cv_t<T, -1, -1, true>(a, npatch, st);
  }
  if (px) return py ? launch_cv_t<T, 1, 1, false>(a, npatch, st) : launch_cv_t<T, 1, -1, false>(a, npatch, st);
  return py ? launch_cv_t<T, -1, 1, false>(a, npatch, st) : launch_cv_t<T, -1, -1, false>(a, npatch, st);
}

template <class S, int T>
static int launch_sc(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  return a.rslot ? launch_sc_t<S, T, true>(a, npatch, st) : launch_sc_t<S, T, false>(a, npatch, st);
}

template <class S, int T, int NT, int MINB>
static int launch_step_r(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  return a.rslot ? launch_step_t<S, T, NT, MINB, true>(a, npatch, st) : launch_step_t<S, T, NT, MINB, false>(a, npatch, st);
}

template <class S>
static int launch_step_s(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  // constant-velocity advection on whole 8 x 8 / 16 x 16 patches: the register-sweep kernel
  // (FC_SCALAR_CV=0 keeps k_step_sc; reflux records need method3 = 2 here)
  static const bool cv = !(getenv("FC_SCALAR_CV") && atoi(getenv("FC_SCALAR_CV")) == 0);
  // (the choice may not depend on the local patch count: results must not depend on the sharding)
  if constexpr (std::is_same<S, AdvConst>::value) {
    if (cv && (!a.rslot || a.method3 == 2) && a.tiles == 1 && a.limiter != 0) {
      if (a.m == 16) return launch_cv<16>(a, npatch, st);
      // a forest of complete sibling families of regular patches (the planner's quad flag): 2 x 2
      // blocks through the 16 x 16 sweep (not on active lists or reflux records)
      if (a.m == 8 && a.quad && !a.active && !a.rslot && a.ring && a.nb9 && !a.rpeer && npatch % 4 == 0)
        return launch_cv_quad(a, npatch / 4, st);
      if (a.m == 8) return launch_cv<8>(a, npatch, st);
    }
  }
  if constexpr (std::is_same<S, AdvEdgeCapa>::value) {   // capacity form: the same sweep, aux from global
    if (cv && !a.rslot && a.tiles == 1 && a.limiter != 0) {
      const bool mt2 = a.method3 == 2;
      if (a.m == 16) return mt2 ? launch_cvc_t<16, true>(a, npatch, st) : launch_cvc_t<16, false>(a, npatch, st);
      if (a.m == 8) return mt2 ? launch_cvc_t<8, true>(a, npatch, st) : launch_cvc_t<8, false>(a, npatch, st);
    }
  }
  if constexpr (S::MEQN == 1) {   // scalars: the two-phase kernel
    if (a.m % 16 == 0) return launch_sc<S, 16>(a, npatch, st);
    if (a.m % 8 == 0) return launch_sc<S, 8>(a, npatch, st);
    if (a.m % 4 == 0) return launch_sc<S, 4>(a, npatch, st);
    if (a.m % 2 == 0) return launch_sc<S, 2>(a, npatch, st);
    return -1;
  } else {
    // systems: the phased kernel; CTAs per SM requested from ptxas for the 16 x 16 tile
    // (HLLE's 15-slot edge scratch leaves shared memory for one 16 x 16 CTA per SM)
    constexpr int dmb = std::is_same<S, EulerHlle>::value ? 1 : 2;
    if (a.m % 16 == 0) {
      // 384 threads (12 warps; 2 CTAs keep the 80-register budget): measured on C5 full update
      // 8.58 -> 8.12 ms vs 352; 416 / 448 (72 registers, spills): 8.78 ms (`tools/nt_variants.sh`)
      return launch_step_r<S, 16, 384, dmb>(a, npatch, st);
    }
    if (a.m % 8 == 0) return launch_step_r<S, 8, 128, 4>(a, npatch, st);
    if (a.m % 4 == 0) return launch_step_r<S, 4, 64, 8>(a, npatch, st);
    if (a.m % 2 == 0) return launch_step_r<S, 2, 32, 8>(a, npatch, st);
    return -1;
  }
}

int launch_step(int kind, const double* qold, double* qnew, const double* aux, const int8_t* level,
                int64_t npatch, int m, double dt, double dx0, double p0, double p1, int limiter,
                int method2, int method3, int skip_quiescent, const int32_t* ring, const int32_t* nb9,
                const uint8_t* bcflag,
                const int32_t* active, const int32_t* nactive, unsigned long long* cfl_bits,
                const int32_t* rslot, double* freg, const uint8_t* rpeer, const double* const* peerq,
                const double* cg, cudaStream_t st, int quad) {
  if (npatch <= 0) return 0;
  StepArgs a;
  a.quad = quad;
  a.cg = cg;
  a.rslot = rslot;
  a.freg = freg;
  a.rpeer = rpeer;
  for (int r = 0; r < 16; ++r) a.peerq[r] = peerq ? peerq[r] : nullptr;
  a.qold = qold; a.qnew = qnew; a.aux = aux; a.level = level;
  a.dt = dt; a.dx0 = dx0; a.sp.p0 = p0; a.sp.p1 = p1;
  for (int L = 0; L < 29; ++L) a.dtdx[L] = dt / ldexp(dx0, -L);
  a.limiter = limiter; a.method2 = method2; a.method3 = method3;
  a.skip_quiescent = skip_quiescent;
  a.ring = ring;
  a.nb9 = ring ? nb9 : nullptr;
  a.bcflag = bcflag;
  a.active = active;
  a.nactive = nactive;
  a.lim = limiter_coef(limiter);
  a.limh = {0.5 * a.lim.lo, 0.5 * a.lim.c1, 0.5 * a.lim.c2, 0.5 * a.lim.c3, 0.5 * a.lim.c4};
  a.lp1 = limiter == FC_LIM_MC ? 0.5 : 0.0;     // (cv_limited; the register sweeps run MC / minmod only)
  a.lp2 = limiter == FC_LIM_MC ? 0.0 : 1.0;
  a.lk3 = limiter == FC_LIM_MC ? 1.0 : 0.5;
  a.m = m;
  const int T = (m % 16 == 0) ? 16 : ((m % 8 == 0) ? 8 : ((m % 4 == 0) ? 4 : 2));
  a.tiles = m / T;
  a.cfl_bits = cfl_bits;
  {   // systems on the fused ring gather: the warp-sweep kernel (step_ws.cu) where it applies
    const int r = launch_step_ws(kind, a, npatch, st);
    if (r != 0) return r;
  }
  switch (kind) {
    case FC_ADV_CONST: return launch_step_s<AdvConst>(a, npatch, st);
    case FC_ADV_EDGEVEL_CAPA: return launch_step_s<AdvEdgeCapa>(a, npatch, st);
    case FC_SWE_ROE: return launch_step_s<SweRoe>(a, npatch, st);
    case FC_EULER_ROE: return launch_step_s<EulerRoe>(a, npatch, st);
    case FC_EULER_HLLE: return launch_step_s<EulerHlle>(a, npatch, st);
  }
  return -1;
}

// ---------------------------------------------------------------------------------------------
// Coarse/fine reflux: one thread per coarse cell next to a
// finer face; per face (ascending face order) Q_C += dt / (kappa dx) (out_C + (out_f1 + out_f2)/2),
// i.e. the flux the coarse cell applied is replaced by the mean of the two fine fluxes (all in
// outward form, recorded by k_step).  Runs after k_step on q_new, before the commit.
// General form Q_C += dtr / (kappa dx) (wc out_C + (F_1 + F_2)/2) with the fine F from ffine:
// global dt: ffine = freg, wc = 1, dtr = dt; sub-cycling: ffine = the dt-weighted fine sums over
// the two fine sub-steps, wc = dt of the coarse level, dtr = 1.
__global__ void __launch_bounds__(128) k_reflux(const int32_t* __restrict__ cells, int64_t ncells,
                                                const double* __restrict__ freg, const double* __restrict__ ffine,
                                                double* __restrict__ qnew, const double* __restrict__ aux,
                                                const int8_t* __restrict__ level, double wc, double dtr, double dx0,
                                                int meqn, int n2) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ncells; t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* r = cells + t * RFX;
    const double kap = r[1] >= 0 ? aux[r[1]] : 1.0;
    const double rr = dtr / (kap * ldexp(dx0, -(int)level[r[2]]));
    double* q = qnew + r[0];
    for (int f = 0; f < r[3]; ++f) {
      const double* oc = freg + r[4 + 3 * f];
      const double* f1 = ffine + r[5 + 3 * f];
      const double* f2 = ffine + r[6 + 3 * f];
      for (int k = 0; k < meqn; ++k) {
        const double corr = wc * oc[k] + 0.5 * (f1[k] + f2[k]);
        q[(int64_t)k * n2] += rr * corr;
      }
    }
  }
}

int launch_reflux(const int32_t* cells, int64_t ncells, const double* freg, const double* ffine, double* qnew,
                  const double* aux, const int8_t* level, double wc, double dtr, double dx0, int meqn, int n2,
                  cudaStream_t st) {
  if (ncells <= 0) return 0;
  const int64_t blocks = (ncells + 127) / 128;
  k_reflux<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 128, 0, st>>>(cells, ncells, freg, ffine, qnew, aux,
                                                                              level, wc, dtr, dx0, meqn, n2);
  return 1;
}

// ---------------------------------------------------------------------------------------------
// Sub-cycling, driven by fc_step_subcycled (api.cu).
// Snapshot for the ghost fill of level l at one time: patches of level >= l hold their current
// interior, coarser ones (1 - a) Q_old + a Q_new with a the exact dyadic weight of their level
// (separately rounded products, as the oracle); level-l patches also save Q_old := current.
struct SubAlpha {
  double a[32];
  int lmin;
};
__global__ void k_sub_snapshot(const double* __restrict__ cur, double* __restrict__ old,
                               const double* __restrict__ old0, double* __restrict__ snap,
                               const int8_t* __restrict__ level, const int32_t* __restrict__ list, int64_t P,
                               int meqn, int mm, int n2, int l, SubAlpha al) {
  const int64_t per = (int64_t)meqn * mm, tot = P * per;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / per;
    const int r = (int)(t - i * per), k = r / mm, c = r - k * mm;
    const int64_t p = list ? (int64_t)list[i] : i;
    const int64_t o = (p * meqn + k) * n2 + c;     // dense interior (qcell)
    const int lp = level[p];
    if (lp >= l) {
      const double v = cur[o];
      snap[o] = v;
      if (lp == l) old[o] = v;
    } else {
      const double a = al.a[lp - al.lmin];
      const double ov = lp == al.lmin ? old0[o] : old[o];   // the coarsest level starts at q_old
      snap[o] = __dadd_rn(__dmul_rn(1.0 - a, ov), __dmul_rn(a, cur[o]));
    }
  }
}

// fine-side reflux sums: acc = dt rec (first sub-step of the parent's step) or acc + dt rec
__global__ void k_sub_accumulate(const int32_t* __restrict__ list, int64_t n, const int32_t* __restrict__ rslot,
                                 const double* __restrict__ rec, double* __restrict__ acc, int fs, double dt,
                                 int add) {
  const int64_t tot = n * fs;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / fs;
    const int e = (int)(t - i * fs);
    const int32_t slot = rslot[list[i]];
    if (slot < 0) continue;
    const int64_t o = (int64_t)slot * fs + e;
    const double v = __dmul_rn(dt, rec[o]);
    acc[o] = add ? __dadd_rn(acc[o], v) : v;
  }
}

int launch_sub_snapshot(const double* cur, double* old, const double* old0, double* snap, const int8_t* level,
                        const int32_t* list, int64_t P, int meqn, int m, int n2, int l, const double* alpha, int lmin,
                        cudaStream_t st) {
  if (P <= 0) return 0;
  SubAlpha al;
  for (int i = 0; i < 32; ++i) al.a[i] = alpha[i];
  al.lmin = lmin;
  k_sub_snapshot<<<148 * 8, 256, 0, st>>>(cur, old, old0, snap, level, list, P, meqn, m * m, n2, l, al);
  return 1;
}

int launch_sub_accumulate(const int32_t* list, int64_t n, const int32_t* rslot, const double* rec, double* acc,
                          int fs, double dt, int add, cudaStream_t st) {
  if (n <= 0) return 0;
  const int64_t tot = n * fs, blocks = (tot + 255) / 256;
  k_sub_accumulate<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, st>>>(list, n, rslot, rec, acc, fs, dt, add);
  return 1;
}

}  // namespace fc
