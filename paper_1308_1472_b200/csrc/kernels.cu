// kernels.cu -- libfc device kernels (sm_100a, fp64): ghost fill from typed work lists, halo
// pack/unpack, interior <-> padded transfers, and the fused wave-propagation step.
//
// Ghost fill (PAPER.md:187-201 [§3]; readings in DESIGN.md): one thread per ghost-cell record,
// all meqn components; the arithmetic is exact-order (products by 0.25 / 0.5 are exact, no
// multiply precedes an add that could contract to FMA), so rings are bitwise equal to the oracle's.
//
// Step (PAPER.md:168-182 [§3]): one CTA per T x T tile of a patch (T = m for m <= 16; larger
// patches are split into 16 x 16 tiles -- the update of a cell only reads its 2-cell
// neighbourhood, so tiles are exact).  The tile plus its 2-cell halo is staged in shared memory;
// per sweep: (1) normal Riemann solve on every edge into a compact per-edge scratch; (2) limiter
// from the upwind neighbour's unlimited wave, second-order correction, CFL, transverse splitting
// of A-+dq +- F~, accumulated into per-cell arrays with a two-colour write (no atomics);
// (3) transverse contributions folded into the cell update.  The y-sweep reads Q^n (unsplit).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fc.h"
#include "solvers.cuh"

namespace fc {

// ---------------------------------------------------------------------------------------------
// ghost fill
__global__ void k_ghost_copy(double* __restrict__ q, const int32_t* __restrict__ L, int64_t nrec,
                             int meqn, int n2) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const int32_t d = L[2 * r], s = L[2 * r + 1];
  for (int k = 0; k < meqn; ++k) q[d + k * n2] = q[s + k * n2];
}

__global__ void k_ghost_avg(double* __restrict__ q, const int32_t* __restrict__ L, int64_t nrec,
                            int meqn, int n2) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const int32_t* o = L + 5 * r;
  for (int k = 0; k < meqn; ++k) {
    const int64_t c = (int64_t)k * n2;
    const double a = __dadd_rn(q[o[1] + c], q[o[2] + c]);
    const double b = __dadd_rn(q[o[3] + c], q[o[4] + c]);
    q[o[0] + c] = __dmul_rn(__dadd_rn(a, b), 0.25);
  }
}

__device__ __forceinline__ double minmod(double a, double b) {
  if (a > 0.0 && b > 0.0) return a < b ? a : b;
  if (a < 0.0 && b < 0.0) return a > b ? a : b;
  return 0.0;
}

__global__ void k_ghost_interp(double* __restrict__ q, const int32_t* __restrict__ L, int64_t nrec,
                               int meqn, int n2) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const int32_t* o = L + 8 * r;
  const double sgx = (double)o[6], sgy = (double)o[7];
  for (int k = 0; k < meqn; ++k) {
    const int64_t c = (int64_t)k * n2;
    const double qc = q[o[1] + c];
    const double sx = minmod(__dsub_rn(q[o[3] + c], qc), __dsub_rn(qc, q[o[2] + c]));
    const double sy = minmod(__dsub_rn(q[o[5] + c], qc), __dsub_rn(qc, q[o[4] + c]));
    const double t = __dadd_rn(__dmul_rn(sgx, sx), __dmul_rn(sgy, sy));
    q[o[0] + c] = __dadd_rn(qc, __dmul_rn(0.25, t));
  }
}

__global__ void k_ghost_bc(double* __restrict__ q, const int32_t* __restrict__ L, int64_t nrec,
                           int meqn, int n2) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const int32_t d = L[3 * r], s = L[3 * r + 1], neg = L[3 * r + 2];
  for (int k = 0; k < meqn; ++k) {
    const double v = q[s + k * n2];
    q[d + k * n2] = (k == neg) ? -v : v;
  }
}

__global__ void k_ghost_corner3(double* __restrict__ q, const int32_t* __restrict__ L, int64_t nrec,
                                int meqn, int n2) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const int32_t d = L[3 * r], a = L[3 * r + 1], b = L[3 * r + 2];
  for (int k = 0; k < meqn; ++k)
    q[d + k * n2] = __dmul_rn(0.5, __dadd_rn(q[a + k * n2], q[b + k * n2]));
}

// halo: pack local cells (offset of component 0) into buf[item][meqn]; unpack into halo slots
__global__ void k_pack(const double* __restrict__ q, const int32_t* __restrict__ idx, int64_t cnt,
                       int meqn, int n2, double* __restrict__ buf) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt * meqn) return;
  const int64_t it = t / meqn;
  const int k = (int)(t - it * meqn);
  buf[t] = q[idx[it] + (int64_t)k * n2];
}

__global__ void k_unpack(double* __restrict__ q, const int32_t* __restrict__ idx, int64_t cnt,
                         int meqn, int n2, const double* __restrict__ buf) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt * meqn) return;
  const int64_t it = t / meqn;
  const int k = (int)(t - it * meqn);
  q[idx[it] + (int64_t)k * n2] = buf[t];
}

// interior [P][meqn][m][m] <-> padded [P][meqn][n][n]
__global__ void k_scatter_interior(const double* __restrict__ src, double* __restrict__ q,
                                   int64_t P, int meqn, int m) {
  const int64_t tot = P * meqn * m * m;
  const int n = m + 4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % m);
    const int64_t r = t / m;
    const int j = (int)(r % m);
    const int64_t pk = r / m;
    q[pk * n * n + (int64_t)(j + 2) * n + (i + 2)] = src[t];
  }
}

__global__ void k_gather_interior(const double* __restrict__ q, double* __restrict__ dst,
                                  int64_t P, int meqn, int m) {
  const int64_t tot = P * meqn * m * m;
  const int n = m + 4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(t % m);
    const int64_t r = t / m;
    const int j = (int)(r % m);
    const int64_t pk = r / m;
    dst[t] = q[pk * n * n + (int64_t)(j + 2) * n + (i + 2)];
  }
}

// ---------------------------------------------------------------------------------------------
// fused step
struct StepArgs {
  const double* __restrict__ qold;
  double* __restrict__ qnew;
  const double* __restrict__ aux;     // [Pl][3][n][n] or null
  const int8_t* __restrict__ level;   // [Pl]
  double dt, dx0;
  SolverParams sp;
  int limiter, method2, method3;
  int m, tiles;                       // tiles per side
  unsigned long long* cfl_bits;
};

__device__ __forceinline__ double limiter_phi(int lim, double th) {
  if (lim == 2) return fmax(0.0, fmin(fmin(0.5 * (1.0 + th), 2.0), 2.0 * th));
  if (lim == 1) return fmax(0.0, fmin(1.0, th));
  return 1.0;
}

template <class S, int T>
struct StepShape {
  static constexpr int W = T + 4;
  static constexpr int WW = W * W;
  static constexpr int EX = (T + 3) * (T + 2);   // edges per sweep (incl. limiter neighbours)
  static constexpr int E2 = (T + 1) * (T + 2);   // edges with corrections / transverse
  static constexpr int NTR = S::MEQN * T * (T + 2);
  static constexpr size_t smem_doubles =
      (size_t)S::MEQN * WW + (S::CAPA ? 3 * WW : 0) + (size_t)S::NS * EX + S::MEQN * T * T + 2 * NTR;
  static constexpr size_t smem_bytes = smem_doubles * sizeof(double);
};

template <class S, int T, int NT>
__global__ void __launch_bounds__(NT) k_step(StepArgs A) {
  using Sh = StepShape<S, T>;
  constexpr int MEQN = S::MEQN, W = Sh::W, WW = Sh::WW, EX = Sh::EX, E2 = Sh::E2;
  extern __shared__ double sm[];
  double* sq = sm;                                   // [MEQN][W][W]
  double* sa = sq + MEQN * WW;                       // [3][W][W]
  double* scr = sa + (S::CAPA ? 3 * WW : 0);         // [NS][EX]
  double* dq = scr + S::NS * EX;                     // [MEQN][T][T]
  double* ta = dq + MEQN * T * T;                    // x: up / y: right     [MEQN][..]
  double* tb = ta + Sh::NTR;                         // x: down / y: left

  const int tid = threadIdx.x;
  const int tiles2 = A.tiles * A.tiles;
  const int64_t patch = blockIdx.x / tiles2;
  const int tile = blockIdx.x - (int)(patch * tiles2);
  const int tx = tile % A.tiles, ty = tile / A.tiles;
  const int n = A.m + 4, n2 = n * n;
  const double* qb = A.qold + patch * (int64_t)MEQN * n2 + (int64_t)(ty * T) * n + tx * T;

  for (int t = tid; t < MEQN * WW; t += NT) {
    const int k = t / WW, r = t - k * WW, b = r / W, a = r - b * W;
    sq[t] = qb[(int64_t)k * n2 + b * n + a];
  }
  if (S::CAPA) {
    const double* ab = A.aux + patch * 3ll * n2 + (int64_t)(ty * T) * n + tx * T;
    for (int t = tid; t < 3 * WW; t += NT) {
      const int k = t / WW, r = t - k * WW, b = r / W, a = r - b * W;
      sa[t] = ab[(int64_t)k * n2 + b * n + a];
    }
  }
  for (int t = tid; t < MEQN * T * T; t += NT) dq[t] = 0.0;
  for (int t = tid; t < 2 * Sh::NTR; t += NT) ta[t] = 0.0;
  __syncthreads();

  const double dx = ldexp(A.dx0, -(int)A.level[patch]);
  const double dtdx = A.dt / dx;   // square cells: dt/dy = dt/dx
  // window index of tile-local 1-based cell (i, j)
  auto widx = [](int i, int j) { return (j + 1) * W + (i + 1); };
  auto auxc = [&](int i, int j) { return AuxCell{sa + widx(i, j), WW}; };
  auto rcell = [&](int i, int j) { return S::CAPA ? dtdx / sa[widx(i, j)] : dtdx; };
  double cfl = 0.0;

  // =============================== x-sweep ===============================
  for (int e = tid; e < EX; e += NT) {       // edge i (cells i-1 | i), row j
    const int i = e % (T + 3), j = e / (T + 3);
    double ql[MEQN], qr[MEQN];
#pragma unroll
    for (int k = 0; k < MEQN; ++k) { ql[k] = sq[k * WW + widx(i - 1, j)]; qr[k] = sq[k * WW + widx(i, j)]; }
    S::template riemann<1>(ql, qr, auxc(i - 1, j), auxc(i, j), A.sp, scr + e, EX);
  }
  __syncthreads();
  for (int base = 0; base < E2; base += NT) {
    const int e2 = base + tid;
    const bool v = e2 < E2;
    const int i = v ? 1 + e2 % (T + 1) : 0, j = v ? e2 / (T + 1) : 0;
    double Lv[MEQN], Rv[MEQN], bmL[MEQN], bpL[MEQN], bmR[MEQN], bpR[MEQN];
    double rl = 0.0, rr = 0.0;
    if (v) {
      const int e = j * (T + 3) + i;
      const double* sc = scr + e;
      rl = rcell(i - 1, j); rr = rcell(i, j);
      double am[MEQN], ap[MEQN], F[MEQN];
      S::template fluct<1>(sc, EX, A.sp, auxc(i, j), am, ap);
#pragma unroll
      for (int k = 0; k < MEQN; ++k) F[k] = 0.0;
      const double rav = 0.5 * (rl + rr);
#pragma unroll
      for (int p = 0; p < S::MW; ++p) {
        const double s = S::template speed<1>(sc, EX, p, A.sp, auxc(i, j));
        cfl = fmax(cfl, fmax(rr * s, -rl * s));
        if (A.method2 == 2) {
          double Wp[MEQN], WI[MEQN];
          S::template wave<1>(sc, EX, p, A.sp, Wp);
          double wn2 = 0.0;
#pragma unroll
          for (int k = 0; k < MEQN; ++k) wn2 += Wp[k] * Wp[k];
          if (wn2 != 0.0) {
            const int I = s > 0.0 ? e - 1 : e + 1;
            S::template wave<1>(scr + I, EX, p, A.sp, WI);
            double dot = 0.0;
#pragma unroll
            for (int k = 0; k < MEQN; ++k) dot += WI[k] * Wp[k];
            const double phi = limiter_phi(A.limiter, dot / wn2);
            const double as = fabs(s);
            const double c = 0.5 * as * (1.0 - as * rav) * phi;
#pragma unroll
            for (int k = 0; k < MEQN; ++k) F[k] += c * Wp[k];
          }
        }
      }
      const double m3 = A.method3 == 2 ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < MEQN; ++k) { Lv[k] = am[k] + F[k]; Rv[k] = ap[k] - F[k]; }
      if (A.method3 >= 1) {
        double XL[MEQN], XR[MEQN];
#pragma unroll
        for (int k = 0; k < MEQN; ++k) { XL[k] = am[k] + m3 * F[k]; XR[k] = ap[k] - m3 * F[k]; }
        S::template transverse<1>(sc, EX, A.sp, XL, auxc(i - 1, j), auxc(i - 1, j + 1), bmL, bpL);
        S::template transverse<1>(sc, EX, A.sp, XR, auxc(i, j), auxc(i, j + 1), bmR, bpR);
      } else {
#pragma unroll
        for (int k = 0; k < MEQN; ++k) bmL[k] = bpL[k] = bmR[k] = bpR[k] = 0.0;
      }
    }
    for (int color = 0; color < 2; ++color) {
      __syncthreads();
      if (v && (i & 1) == color) {
        if (i - 1 >= 1) {   // left cell (i-1, j) receives L
#pragma unroll
          for (int k = 0; k < MEQN; ++k) {
            if (j >= 1 && j <= T) dq[(k * T + (j - 1)) * T + (i - 2)] -= rl * Lv[k];
            ta[(k * (T + 2) + j) * T + (i - 2)] -= 0.5 * rl * bpL[k];
            tb[(k * (T + 2) + j) * T + (i - 2)] -= 0.5 * rl * bmL[k];
          }
        }
        if (i <= T) {       // right cell (i, j) receives R
#pragma unroll
          for (int k = 0; k < MEQN; ++k) {
            if (j >= 1 && j <= T) dq[(k * T + (j - 1)) * T + (i - 1)] -= rr * Rv[k];
            ta[(k * (T + 2) + j) * T + (i - 1)] -= 0.5 * rr * bpR[k];
            tb[(k * (T + 2) + j) * T + (i - 1)] -= 0.5 * rr * bmR[k];
          }
        }
      }
    }
  }
  __syncthreads();
  // fold G~ transverse (from the x-sweep) into dq: G~(i, j+1/2) = up(i, j) + dn(i, j+1)
  for (int t = tid; t < T * T; t += NT) {
    const int i = 1 + t % T, j = 1 + t / T;
    const double s = rcell(i, j);
#pragma unroll
    for (int k = 0; k < MEQN; ++k) {
      const double* up = ta + k * (T + 2) * T;
      const double* dn = tb + k * (T + 2) * T;
      const double gt = up[j * T + (i - 1)] + dn[(j + 1) * T + (i - 1)];
      const double gb = up[(j - 1) * T + (i - 1)] + dn[j * T + (i - 1)];
      dq[(k * T + (j - 1)) * T + (i - 1)] -= s * (gt - gb);
    }
  }
  __syncthreads();
  for (int t = tid; t < 2 * Sh::NTR; t += NT) ta[t] = 0.0;

  // =============================== y-sweep ===============================
  for (int e = tid; e < EX; e += NT) {       // column i, edge j (cells j-1 | j)
    const int i = e % (T + 2), j = e / (T + 2);
    double ql[MEQN], qr[MEQN];
#pragma unroll
    for (int k = 0; k < MEQN; ++k) { ql[k] = sq[k * WW + widx(i, j - 1)]; qr[k] = sq[k * WW + widx(i, j)]; }
    S::template riemann<2>(ql, qr, auxc(i, j - 1), auxc(i, j), A.sp, scr + e, EX);
  }
  __syncthreads();
  for (int base = 0; base < E2; base += NT) {
    const int e2 = base + tid;
    const bool v = e2 < E2;
    const int i = v ? e2 % (T + 2) : 0, j = v ? 1 + e2 / (T + 2) : 0;
    double Lv[MEQN], Rv[MEQN], bmL[MEQN], bpL[MEQN], bmR[MEQN], bpR[MEQN];
    double sl = 0.0, sr = 0.0;
    if (v) {
      const int e = j * (T + 2) + i;
      const double* sc = scr + e;
      sl = rcell(i, j - 1); sr = rcell(i, j);
      double am[MEQN], ap[MEQN], F[MEQN];
      S::template fluct<2>(sc, EX, A.sp, auxc(i, j), am, ap);
#pragma unroll
      for (int k = 0; k < MEQN; ++k) F[k] = 0.0;
      const double sav = 0.5 * (sl + sr);
#pragma unroll
      for (int p = 0; p < S::MW; ++p) {
        const double s = S::template speed<2>(sc, EX, p, A.sp, auxc(i, j));
        cfl = fmax(cfl, fmax(sr * s, -sl * s));
        if (A.method2 == 2) {
          double Wp[MEQN], WI[MEQN];
          S::template wave<2>(sc, EX, p, A.sp, Wp);
          double wn2 = 0.0;
#pragma unroll
          for (int k = 0; k < MEQN; ++k) wn2 += Wp[k] * Wp[k];
          if (wn2 != 0.0) {
            const int I = s > 0.0 ? e - (T + 2) : e + (T + 2);
            S::template wave<2>(scr + I, EX, p, A.sp, WI);
            double dot = 0.0;
#pragma unroll
            for (int k = 0; k < MEQN; ++k) dot += WI[k] * Wp[k];
            const double phi = limiter_phi(A.limiter, dot / wn2);
            const double as = fabs(s);
            const double c = 0.5 * as * (1.0 - as * sav) * phi;
#pragma unroll
            for (int k = 0; k < MEQN; ++k) F[k] += c * Wp[k];
          }
        }
      }
      const double m3 = A.method3 == 2 ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < MEQN; ++k) { Lv[k] = am[k] + F[k]; Rv[k] = ap[k] - F[k]; }
      if (A.method3 >= 1) {
        double XL[MEQN], XR[MEQN];
#pragma unroll
        for (int k = 0; k < MEQN; ++k) { XL[k] = am[k] + m3 * F[k]; XR[k] = ap[k] - m3 * F[k]; }
        S::template transverse<2>(sc, EX, A.sp, XL, auxc(i, j - 1), auxc(i + 1, j - 1), bmL, bpL);
        S::template transverse<2>(sc, EX, A.sp, XR, auxc(i, j), auxc(i + 1, j), bmR, bpR);
      } else {
#pragma unroll
        for (int k = 0; k < MEQN; ++k) bmL[k] = bpL[k] = bmR[k] = bpR[k] = 0.0;
      }
    }
    for (int color = 0; color < 2; ++color) {
      __syncthreads();
      if (v && (j & 1) == color) {
        if (j - 1 >= 1) {   // lower cell (i, j-1) receives L
#pragma unroll
          for (int k = 0; k < MEQN; ++k) {
            if (i >= 1 && i <= T) dq[(k * T + (j - 2)) * T + (i - 1)] -= sl * Lv[k];
            ta[(k * T + (j - 2)) * (T + 2) + i] -= 0.5 * sl * bpL[k];
            tb[(k * T + (j - 2)) * (T + 2) + i] -= 0.5 * sl * bmL[k];
          }
        }
        if (j <= T) {       // upper cell (i, j) receives R
#pragma unroll
          for (int k = 0; k < MEQN; ++k) {
            if (i >= 1 && i <= T) dq[(k * T + (j - 1)) * T + (i - 1)] -= sr * Rv[k];
            ta[(k * T + (j - 1)) * (T + 2) + i] -= 0.5 * sr * bpR[k];
            tb[(k * T + (j - 1)) * (T + 2) + i] -= 0.5 * sr * bmR[k];
          }
        }
      }
    }
  }
  __syncthreads();
  // fold F~ transverse (from the y-sweep): F~(i+1/2, j) = right(i, j) + left(i+1, j); write q_new
  double* ob = A.qnew + patch * (int64_t)MEQN * n2 + (int64_t)(ty * T + 2) * n + tx * T + 2;
  for (int t = tid; t < MEQN * T * T; t += NT) {
    const int k = t / (T * T), r = t - k * T * T;
    const int i = 1 + r % T, j = 1 + r / T;
    const double rc = rcell(i, j);
    const double* rt = ta + k * T * (T + 2);
    const double* lf = tb + k * T * (T + 2);
    const double fr = rt[(j - 1) * (T + 2) + i] + lf[(j - 1) * (T + 2) + i + 1];
    const double fl = rt[(j - 1) * (T + 2) + i - 1] + lf[(j - 1) * (T + 2) + i];
    const double val = sq[k * WW + widx(i, j)] + (dq[t] - rc * (fr - fl));
    ob[(int64_t)k * n2 + (int64_t)(j - 1) * n + (i - 1)] = val;
  }

  // CFL: warp max -> block max -> one atomicMax on the IEEE bits (non-negative; NaN -> +inf)
  if (cfl != cfl) cfl = __longlong_as_double(0x7ff0000000000000ll);
  for (int o = 16; o > 0; o >>= 1) cfl = fmax(cfl, __shfl_xor_sync(0xffffffffu, cfl, o));
  __shared__ double wmax[NT / 32];
  if ((tid & 31) == 0) wmax[tid >> 5] = cfl;
  __syncthreads();
  if (tid == 0) {
    double c = wmax[0];
    for (int w = 1; w < NT / 32; ++w) c = fmax(c, wmax[w]);
    atomicMax(A.cfl_bits, (unsigned long long)__double_as_longlong(c));
  }
}

// ---------------------------------------------------------------------------------------------
// host-side launchers (called from api.cu)
static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

int launch_ghost(int op, double* q, const int32_t* list, int64_t nrec, int meqn, int n2,
                 cudaStream_t st) {
  if (nrec <= 0) return 0;
  const int B = 256;
  switch (op) {
    case 1: k_ghost_copy<<<nblk(nrec, B), B, 0, st>>>(q, list, nrec, meqn, n2); break;
    case 2: k_ghost_avg<<<nblk(nrec, B), B, 0, st>>>(q, list, nrec, meqn, n2); break;
    case 3: k_ghost_interp<<<nblk(nrec, B), B, 0, st>>>(q, list, nrec, meqn, n2); break;
    case 4: k_ghost_bc<<<nblk(nrec, B), B, 0, st>>>(q, list, nrec, meqn, n2); break;
    case 6: k_ghost_corner3<<<nblk(nrec, B), B, 0, st>>>(q, list, nrec, meqn, n2); break;
    default: return -1;
  }
  return 1;
}

int launch_pack(const double* q, const int32_t* idx, int64_t cnt, int meqn, int n2, double* buf,
                cudaStream_t st) {
  if (cnt <= 0) return 0;
  k_pack<<<nblk(cnt * meqn, 256), 256, 0, st>>>(q, idx, cnt, meqn, n2, buf);
  return 1;
}

int launch_unpack(double* q, const int32_t* idx, int64_t cnt, int meqn, int n2, const double* buf,
                  cudaStream_t st) {
  if (cnt <= 0) return 0;
  k_unpack<<<nblk(cnt * meqn, 256), 256, 0, st>>>(q, idx, cnt, meqn, n2, buf);
  return 1;
}

int launch_scatter(const double* src, double* q, int64_t P, int meqn, int m, cudaStream_t st) {
  if (P <= 0) return 0;
  k_scatter_interior<<<148 * 8, 256, 0, st>>>(src, q, P, meqn, m);
  return 1;
}

int launch_gather(const double* q, double* dst, int64_t P, int meqn, int m, cudaStream_t st) {
  if (P <= 0) return 0;
  k_gather_interior<<<148 * 8, 256, 0, st>>>(q, dst, P, meqn, m);
  return 1;
}

template <class S, int T, int NT>
static int launch_step_t(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  const size_t smem = StepShape<S, T>::smem_bytes;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_step<S, T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  const int64_t grid = npatch * a.tiles * a.tiles;
  k_step<S, T, NT><<<(unsigned)grid, NT, smem, st>>>(a);
  return 1;
}

template <class S>
static int launch_step_s(const StepArgs& a, int64_t npatch, cudaStream_t st) {
  if (a.m == 4) return launch_step_t<S, 4, 32>(a, npatch, st);
  if (a.m % 16 == 0) return launch_step_t<S, 16, 320>(a, npatch, st);
  if (a.m % 8 == 0) return launch_step_t<S, 8, 96>(a, npatch, st);
  if (a.m % 4 == 0) return launch_step_t<S, 4, 32>(a, npatch, st);
  if (a.m % 2 == 0) return launch_step_t<S, 2, 32>(a, npatch, st);
  return -1;
}

int launch_step(int kind, const double* qold, double* qnew, const double* aux, const int8_t* level,
                int64_t npatch, int m, double dt, double dx0, double p0, double p1, int limiter,
                int method2, int method3, unsigned long long* cfl_bits, cudaStream_t st) {
  if (npatch <= 0) return 0;
  StepArgs a;
  a.qold = qold; a.qnew = qnew; a.aux = aux; a.level = level;
  a.dt = dt; a.dx0 = dx0; a.sp.p0 = p0; a.sp.p1 = p1;
  a.limiter = limiter; a.method2 = method2; a.method3 = method3;
  a.m = m;
  const int T = (m % 16 == 0) ? 16 : ((m % 8 == 0) ? 8 : ((m % 4 == 0) ? 4 : 2));
  a.tiles = m / T;
  a.cfl_bits = cfl_bits;
  switch (kind) {
    case FC_ADV_CONST: return launch_step_s<AdvConst>(a, npatch, st);
    case FC_ADV_EDGEVEL_CAPA: return launch_step_s<AdvEdgeCapa>(a, npatch, st);
    case FC_SWE_ROE: return launch_step_s<SweRoe>(a, npatch, st);
    case FC_EULER_ROE: return launch_step_s<EulerRoe>(a, npatch, st);
  }
  return -1;
}

}  // namespace fc
