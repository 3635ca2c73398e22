// kernels.cu -- libfc device kernels (sm_100a, fp64): ghost fill from typed work lists, halo
// pack/unpack, interior <-> padded transfers, and the fused wave-propagation step.
//
// Ghost fill (PAPER.md:187-201 [§3]; readings in DESIGN.md): one thread per ghost-cell record,
// all meqn components; the arithmetic is exact-order (products by 0.25 / 0.5 are exact, no
// multiply precedes an add that could contract to FMA), so rings are bitwise equal to the oracle's.
//
// The fused wave-propagation step is in step.cu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fc.h"
#include "fc_internal.h"

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

// computed ghosts of the fused AMR ring gather (plan_ring_amr): the same arithmetic as
// k_ghost_avg / k_ghost_interp, written into slots of the computed-ghost buffer cg; a source
// reference v >= 0 is q[v], v < 0 is cg[-1 - v]
__global__ void k_cg_avg(const double* __restrict__ q, double* __restrict__ cg, const int32_t* __restrict__ L,
                         int64_t nrec, int meqn, int n2) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const int32_t* o = L + 5 * r;
  for (int k = 0; k < meqn; ++k) {
    const int64_t c = (int64_t)k * n2;
    const double a = __dadd_rn(q[o[1] + c], q[o[2] + c]);
    const double b = __dadd_rn(q[o[3] + c], q[o[4] + c]);
    cg[o[0] + c] = __dmul_rn(__dadd_rn(a, b), 0.25);
  }
}

__global__ void k_cg_interp(const double* __restrict__ q, double* __restrict__ cg, const int32_t* __restrict__ L,
                            int64_t nrec, int meqn, int n2) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const int32_t* o = L + 8 * r;
  const double sgx = (double)o[6], sgy = (double)o[7];
  for (int k = 0; k < meqn; ++k) {
    const int64_t c = (int64_t)k * n2;
    auto rd = [&](int32_t v) { return v >= 0 ? q[v + c] : cg[(-1 - (int64_t)v) + c]; };
    const double qc = rd(o[1]);
    const double sx = minmod(__dsub_rn(rd(o[3]), qc), __dsub_rn(qc, rd(o[2])));
    const double sy = minmod(__dsub_rn(rd(o[5]), qc), __dsub_rn(qc, rd(o[4])));
    const double t = __dadd_rn(__dmul_rn(sgx, sx), __dmul_rn(sgy, sy));
    cg[o[0] + c] = __dadd_rn(qc, __dmul_rn(0.25, t));
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
    q[pk * n * n + (int64_t)j * m + i] = src[t];   // dense interior first (fc_internal.h qcell)
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
    dst[t] = q[pk * n * n + (int64_t)j * m + i];
  }
}

// storage (interior + ring, qcell) -> natural padded layout, one n x n block per (patch, component)
__global__ void k_unpack_padded(const double* __restrict__ q, double* __restrict__ dst, int64_t nblocks, int n) {
  const int64_t tot = nblocks * n * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % n);                 // natural column = i + 1
    const int64_t rr = t / n;
    const int r = (int)(rr % n);                // natural row = j + 1
    dst[t] = q[(rr - r) * n + qcell(c - 1, r - 1, n)];
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

__global__ void k_cg_corner3(const double* __restrict__ q, double* __restrict__ cg, const int32_t* __restrict__ L,
                             int64_t nrec, int meqn, int n2) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrec) return;
  const int32_t* o = L + 3 * r;
  for (int k = 0; k < meqn; ++k) {
    const int64_t c = (int64_t)k * n2;
    auto rd = [&](int32_t v) { return v >= 0 ? q[v + c] : cg[(-1 - (int64_t)v) + c]; };
    cg[o[0] + c] = __dmul_rn(0.5, __dadd_rn(rd(o[1]), rd(o[2])));   // (k_ghost_corner3's order)
  }
}

int launch_cg(int op, const double* q, double* cg, const int32_t* list, int64_t nrec, int meqn, int n2,
              cudaStream_t st) {
  if (nrec <= 0) return 0;
  const int B = 256;
  if (op == 2) k_cg_avg<<<nblk(nrec, B), B, 0, st>>>(q, cg, list, nrec, meqn, n2);
  else if (op == 6) k_cg_corner3<<<nblk(nrec, B), B, 0, st>>>(q, cg, list, nrec, meqn, n2);
  else k_cg_interp<<<nblk(nrec, B), B, 0, st>>>(q, cg, list, nrec, meqn, n2);
  return 1;
}

// whole padded patch blocks (S doubles each): dst block b = src block ids[b] (regrid migration)
__global__ void k_copy_blocks(const double* __restrict__ src, double* __restrict__ dst,
                              const int32_t* __restrict__ ids, int64_t nb, int64_t S) {
  const int64_t tot = nb * S;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / S;
    dst[t] = src[(int64_t)ids[b] * S + (t - b * S)];
  }
}

int launch_copy_blocks(const double* src, double* dst, const int32_t* ids, int64_t nb, int64_t S, cudaStream_t st) {
  if (nb <= 0) return 0;
  k_copy_blocks<<<148 * 8, 256, 0, st>>>(src, dst, ids, nb, S);
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

int launch_unpack_padded(const double* q, double* dst, int64_t nblocks, int n, cudaStream_t st) {
  if (nblocks <= 0) return 0;
  k_unpack_padded<<<148 * 8, 256, 0, st>>>(q, dst, nblocks, n);
  return 1;
}

int launch_gather(const double* q, double* dst, int64_t P, int meqn, int m, cudaStream_t st) {
  if (P <= 0) return 0;
  k_gather_interior<<<148 * 8, 256, 0, st>>>(q, dst, P, meqn, m);
  return 1;
}

// ---- multi-step runs (fc_run): the step's CFL (IEEE bits from the atomicMax) into a history slot
__global__ void k_cfl_hist(const unsigned long long* __restrict__ cfl_bits, double* __restrict__ hist,
                           int64_t* __restrict__ idx) {
  const int64_t i = *idx;
  hist[i] = __longlong_as_double((long long)*cfl_bits);
  *idx = i + 1;
}

int launch_cfl_hist(const unsigned long long* cfl_bits, double* hist, int64_t* idx, cudaStream_t st) {
  k_cfl_hist<<<1, 1, 0, st>>>(cfl_bits, hist, idx);
  return 1;
}

// ---- dynamic regrid --------------------------------------------------------
// tag: max - min of component 0 over each patch interior (one warp per patch)
__global__ void k_regrid_tag(const double* __restrict__ q, int64_t P, int meqn, int m, double* __restrict__ tag) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int n = m + 4, mm = m * m;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P; p += warps) {
    const double* b = q + p * meqn * n * n;     // dense interior of component 0 (qcell)
    double lo = b[0], hi = b[0];
    for (int c = lane; c < mm; c += 32) { lo = fmin(lo, b[c]); hi = fmax(hi, b[c]); }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) tag[p] = hi - lo;
  }
}

__device__ __forceinline__ double rg_minmod(double a, double b) {
  if (a > 0.0 && b > 0.0) return a < b ? a : b;
  if (a < 0.0 && b < 0.0) return a > b ? a : b;
  return 0.0;
}

// new state from the old one (ghost rings filled): src[np][3] = {kind, old patch, child}
//   1 copy; 2 child k of the old patch: limited (minmod) interpolation, the ghost fill's formula;
//   3 parent of the 4 old patches from the given one: ((a + b) + (c + d)) / 4 per coarse cell
__global__ void k_regrid_transfer(const double* __restrict__ qo, double* __restrict__ qn,
                                  const int32_t* __restrict__ src, int64_t NP, int meqn, int m) {
  const int n = m + 4, n2 = n * n, mm = m * m, h = m / 2;
  const int64_t tot = NP * meqn * mm;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t np = t / ((int64_t)meqn * mm);
    const int r = (int)(t - np * meqn * mm), e = r / mm, c = r - e * mm;
    const int i = 1 + c % m, j = 1 + c / m;
    const int32_t* s = src + np * 3;
    double v;
    if (s[0] == 1) {
      v = qo[((int64_t)s[1] * meqn + e) * n2 + qcell(i, j, n)];
    } else if (s[0] == 2) {
      const double* Q = qo + ((int64_t)s[1] * meqn + e) * n2;
      const int ox = s[2] & 1, oy = s[2] >> 1;
      const int I = ox * h + (i + 1) / 2, J = oy * h + (j + 1) / 2;
      const double sgx = (i & 1) ? -1.0 : 1.0, sgy = (j & 1) ? -1.0 : 1.0;
      const double cc = Q[qcell(I, J, n)];
      const double sx = rg_minmod(Q[qcell(I + 1, J, n)] - cc, cc - Q[qcell(I - 1, J, n)]);
      const double sy = rg_minmod(Q[qcell(I, J + 1, n)] - cc, cc - Q[qcell(I, J - 1, n)]);
      v = __dadd_rn(cc, 0.25 * __dadd_rn(__dmul_rn(sgx, sx), __dmul_rn(sgy, sy)));
    } else {
      const int k = (i > h) + 2 * (j > h);
      const int a = 2 * (i - (i > h) * h), b = 2 * (j - (j > h) * h);
      const double* Q = qo + ((int64_t)(s[1] + k) * meqn + e) * n2;
      v = __dadd_rn(__dadd_rn(Q[qcell(a - 1, b - 1, n)], Q[qcell(a, b - 1, n)]),
                    __dadd_rn(Q[qcell(a - 1, b, n)], Q[qcell(a, b, n)])) * 0.25;
    }
    qn[(np * meqn + e) * n2 + (j - 1) * m + (i - 1)] = v;
  }
}

int launch_regrid_tag(const double* q, int64_t P, int meqn, int m, double* tag, cudaStream_t st) {
  if (P <= 0) return 0;
  const int64_t blocks = (P * 32 + 255) / 256;
  k_regrid_tag<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(q, P, meqn, m, tag);
  return 1;
}

int launch_regrid_transfer(const double* qo, double* qn, const int32_t* src, int64_t NP, int meqn, int m,
                           cudaStream_t st) {
  if (NP <= 0) return 0;
  k_regrid_transfer<<<148 * 8, 256, 0, st>>>(qo, qn, src, NP, meqn, m);
  return 1;
}

}  // namespace fc
