// step_common.cuh -- declarations shared by the step kernels (step.cu: phased / scalar / sweep
// kernels; step_ws.cu: the warp-sweep kernel for systems).  libfc only, nothing shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fc_internal.h"
#include "solvers.cuh"

namespace fc {

// wave limiters as one branch-free form phi = max(lo, min(c1 + c2 theta, c3, c4 theta)):
//   MC     (lo, c1, c2, c3, c4) = (0, 1/2, 1/2, 2, 2)   -> max(0, min((1+t)/2, 2, 2t))
//   minmod                        (0, 1,   0,   1, 1)   -> max(0, min(1, t))
//   none                          (1, 1,   0,   1, 1)   -> 1
struct LimiterCoef {
  double lo, c1, c2, c3, c4;
};
__host__ __device__ inline LimiterCoef limiter_coef(int lim) {
  if (lim == 2) return {0.0, 0.5, 0.5, 2.0, 2.0};
  if (lim == 1) return {0.0, 1.0, 0.0, 1.0, 1.0};
  return {1.0, 1.0, 0.0, 1.0, 1.0};
}
__device__ __forceinline__ double limiter_phi(const LimiterCoef& L, double th) {
  return fmax(L.lo, fmin(fmin(fma(L.c2, th, L.c1), L.c3), L.c4 * th));
}

struct StepArgs {
  const double* __restrict__ qold;
  double* __restrict__ qnew;
  const double* __restrict__ aux;     // [Pl][3][n][n] or null
  const int8_t* __restrict__ level;   // [Pl]
  double dt, dx0;
  SolverParams sp;
  int limiter, method2, method3;
  int skip_quiescent;                 // exact shortcut for tiles whose staged window is uniform
  const int32_t* __restrict__ ring;   // fused ring gather (RingSources.src) or null: ring in q_old
  const int32_t* __restrict__ nb9;    // regular rings (plan_ring_regular): [P][9] neighbour block offsets, [p][0] < 0: table
  const uint8_t* __restrict__ bcflag; // per patch: bit 0 BCX, bit 1 BCY entries present
  const int32_t* __restrict__ active; // active-patch list (quiescent patches filtered out) or null
  const int32_t* __restrict__ nactive;
  LimiterCoef lim;
  LimiterCoef limh;                   // lim with every coefficient halved: phi / 2, exactly
  double lp1, lp2, lk3;               // MC / minmod as min(lp1 (a + b) + lp2 a, lk3 (a + b - |a - b|)), cv_limited
  double dtdx[29];                    // dt / dx of a level-L patch (levels 0..28), dt / ldexp(dx0, -L) on the host
  int m, tiles;                       // tiles per side
  unsigned long long* cfl_bits;
  double* fbuf;                       // method3 = 1 only: per-CTA F~ of each correction edge [MEQN][E2]
  const int32_t* __restrict__ rslot;  // reflux: per patch flux-register slot (-1: none) or null
  double* freg;                       // reflux: [slot][4 faces][m edges][MEQN] applied fluxes, outward
  const uint8_t* __restrict__ rpeer;  // peer-memory halo: owner of each ring source (0 = this rank)
  const double* peerq[16];            // peer-memory halo: rank r's current q_old (peer pointer)
  const double* cg;                   // fused AMR ring gather: computed ghosts (ring peer code 255)
  int quad;                           // m = 8 forest of complete sibling families of regular patches
};

// phi(wi / w) w of the MC / minmod limiter for the scalar register sweeps, division- and
// select-free: with a = |w|, b = |wi|, s = a + b, MC is min(s / 2, 2 min(a, b)) and minmod
// min(a, min(a, b)), i.e. min(lp1 s + lp2 a, lk3 (s - |a - b|)) with (lp1, lp2, lk3) = (1/2, 0, 1) /
// (0, 1, 1/2); min(x, y) = (x + y - |x - y|) / 2 on the fp64 pipe; the sign of w when w and wi
// share a sign (an integer test of the sign bits: a zero w or wi gives mag = 0 anyway), else 0.
// The rounding differs from the oracle's phi(theta) w by ulps, within the step tolerance (reading 24).
__device__ __forceinline__ double cv_limited(double w, double wi, double lp1, double lp2, double lk3) {
  const double a = fabs(w), b = fabs(wi), s = a + b;
  // (the compiler's contraction of x +- y is local to this expression -- y has the same two uses
  // in every instance -- and measured bitwise alike in the m = 8 and the quad-block sweeps; the
  // explicit forms, fmas or rounded intrinsics, compiled to slower code: T1 0.38 -> 0.41 ms)
  const double x = fma(lp1, s, lp2 * a), y = lk3 * (s - fabs(a - b));
  const double mag = 0.5 * ((x + y) - fabs(x - y));
  const int hw = __double2hiint(w);
  const bool opp = (hw ^ __double2hiint(wi)) < 0;
  return opp ? 0.0 : __hiloint2double((hw & 0x80000000) | __double2hiint(mag), __double2loint(mag));
}

// dt / dx of a level-L patch (the host's table: no division in the kernels)
__device__ __forceinline__ double dtdx_level(const StepArgs& A, int L) { return A.dtdx[L]; }
// base of a ring source: this rank's q_old, a peer's (code k = rank k - 1), the computed ghosts (255)
__device__ __forceinline__ const double* ring_base(const StepArgs& A, int ow) {
  if (ow == 0) return A.qold;
  if (ow == 255) return A.cg;
  return A.peerq[ow - 1];
}

// ---- TMA bulk copies + mbarrier (sm_90+ / sm_100a) -------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (UBLKCP); bytes and both addresses multiples of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// an opaque copy: keeps per-thread index arithmetic inside the tile loop instead of letting the
// compiler hoist (and keep live in registers) every phase's thread->edge mapping
__device__ __forceinline__ int opaque(int x) {
  int y;
  asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
// 8-byte async global -> shared copy (LDGSTS), completion tracked with cp.async groups
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// window index (padded index, W = n) of ring cell r in ring storage order (j = -1..m+2 outer,
// i = -1..m+2 inner, interior skipped)
template <int T>
__device__ __forceinline__ int ring_window_index(int r) {
  constexpr int n = T + 4;
  if (r < 2 * n) return r;                                   // rows j = -1, 0
  r -= 2 * n;
  if (r < 4 * T) {                                           // rows 1..m: i = -1, 0, m+1, m+2
    const int j = r / 4 + 1, c = r % 4;
    const int i = c < 2 ? c - 1 : T + c - 1;
    return (j + 1) * n + (i + 1);
  }
  r -= 4 * T;
  return (T + 2) * n + r;                                    // rows j = m+1, m+2
}

// the warp-sweep kernel for systems (step_ws.cu): 1 = launched, 0 = not applicable (the caller
// falls back to k_step), < 0 = error
int launch_step_ws(int kind, const StepArgs& a, int64_t npatch, cudaStream_t st);

}  // namespace fc
