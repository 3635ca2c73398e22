/* forest3.c -- the CPU oracle for forests of OCTREES (3D): plain C, fp64, single-threaded.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): shares no code with the product.
 *
 * PAPER.md:22-24 [abstract] "a forest of octrees ... each leaf a patch of m^d cells",
 * PAPER.md:229-232 [Fig. 1 caption] "The situation in 3D (octrees) is analogous": the 3D analogue
 * of the quadtree path, built to this scope (reading 26):
 *   - a brick of Tx x Ty x Tz octrees with aligned orientation; each tree face either linked to
 *     the opposite face of a neighbour tree (periodic wrap = a self-link) or physical (outflow);
 *   - leaves in Morton order per tree, x in bits 3k, y in 3k+1, z in 3k+2;
 *   - 2:1 balance across faces, edges and corners; mbc = 2, m even >= 4; meqn = 1;
 *   - ghost cells of all 26 directions by brute-force point location of the ghost-cell centre:
 *     COPY (same level), AVG8 (finer: the 2x2x2 block mean, pairwise order), INTERP (coarser:
 *     Q + 1/4 (sx sgx + sy sgy + sz sgz) with minmod slopes of one-sided differences in the coarse
 *     patch's padded array; PAPER.md:193-201 [§3]), outflow BC (zero-order extrapolation, x faces
 *     then y then z: Clawpack's bc3 order);
 *   - phases A (copy, average) -> C (BCs) -> per level ascending [B (interpolate) -> C];
 *   - the update: constant-velocity advection q_t + u q_x + v q_y + w q_z = 0 by LeVeque's wave
 *     propagation (PAPER.md:168-182 [§3]) with Godunov dimensional splitting (Clawpack's
 *     dimensional-split option): an x sweep over rows j, k = -1..m+2, then a y sweep over i = 1..m,
 *     k = -1..m+2, then a z sweep over the interior; each sweep the 1D method: W = dQ, s = u_d,
 *     A-+dQ = min/max(s, 0) W, MC / minmod limiter on W_I / W (I the upwind edge),
 *     F~ = 1/2 |s| (1 - (dt/dx) |s|) phi W;
 *   - CFL = max over the three sweeps of (dt/dx) |u_d|.
 * Readings are listed in DESIGN.md (reading 26). */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"
#include "oracle_internal.h"

struct orc3_forest {
  int64_t P;
  int m, T, lmax;
  int32_t* t2t;      /* [6T] neighbour tree across face f (f = 0..5: -x, +x, -y, +y, -z, +z) */
  int8_t* fbc;       /* [6T] 1: physical (outflow), 0: linked */
  int8_t* level;
  int32_t* tree;
  int64_t *x, *y, *z;   /* origin in units of level-Lmax leaves */
  uint64_t* start;      /* Morton start of the leaf in its tree (8^Lmax index space) */
  int64_t* tree_first;  /* [T+1] */
};

#define N3(m) ((m) + 4)
#define IDX3(m, i, j, k) ((((int64_t)(k) + 1) * N3(m) + ((j) + 1)) * N3(m) + ((i) + 1))

static uint64_t spread3(uint64_t v) {   /* bit b of v -> bit 3b */
  uint64_t r = 0;
  for (int b = 0; b < 21; ++b) r |= ((v >> b) & 1ull) << (3 * b);
  return r;
}
static uint64_t morton3(uint64_t x, uint64_t y, uint64_t z) {
  return spread3(x) | (spread3(y) << 1) | (spread3(z) << 2);
}
static uint64_t compact3(uint64_t c) {   /* bit 3b of c -> bit b */
  uint64_t r = 0;
  for (int b = 0; b < 21; ++b) r |= ((c >> (3 * b)) & 1ull) << b;
  return r;
}

void orc3_forest_destroy(orc3_forest* f) {
  if (!f) return;
  free(f->t2t); free(f->fbc); free(f->level); free(f->tree); free(f->x); free(f->y); free(f->z);
  free(f->start); free(f->tree_first);
  free(f);
}

/* decode: per tree a cursor in the 8^Lmax index space; a leaf of level l covers 8^(Lmax-l) */
int orc3_forest_create(int64_t P, const int8_t* levels, const int32_t* tree_ids, int32_t T,
                       const int32_t* t2t, const int8_t* fbc, int m, orc3_forest** out) {
  *out = NULL;
  if (P <= 0 || T <= 0 || m < 4 || (m & 1)) return ORC_EINVAL;
  orc3_forest* f = (orc3_forest*)calloc(1, sizeof(orc3_forest));
  f->P = P; f->m = m; f->T = T;
  f->t2t = (int32_t*)malloc(6 * (size_t)T * sizeof(int32_t));
  f->fbc = (int8_t*)malloc(6 * (size_t)T);
  memcpy(f->t2t, t2t, 6 * (size_t)T * sizeof(int32_t));
  memcpy(f->fbc, fbc, 6 * (size_t)T);
  for (int t = 0; t < T; ++t)
    for (int fc = 0; fc < 6; ++fc) {   /* linked faces: the neighbour links back through the opposite face */
      if (f->fbc[6 * t + fc]) continue;
      const int nt = f->t2t[6 * t + fc];
      if (nt < 0 || nt >= T || f->fbc[6 * nt + (fc ^ 1)] || f->t2t[6 * nt + (fc ^ 1)] != t) {
        orc3_forest_destroy(f);
        return ORC_ECONN;
      }
    }
  f->level = (int8_t*)malloc(P);
  f->tree = (int32_t*)malloc(P * sizeof(int32_t));
  memcpy(f->level, levels, P);
  memcpy(f->tree, tree_ids, P * sizeof(int32_t));
  int lmax = 0;
  for (int64_t p = 0; p < P; ++p) {
    if (levels[p] < 0 || levels[p] > 20) { orc3_forest_destroy(f); return ORC_EINVAL; }
    if (levels[p] > lmax) lmax = levels[p];
    if (tree_ids[p] < 0 || tree_ids[p] >= T || (p && tree_ids[p] < tree_ids[p - 1])) {
      orc3_forest_destroy(f);
      return ORC_ETILING;
    }
  }
  f->lmax = lmax;
  f->x = (int64_t*)malloc(P * sizeof(int64_t));
  f->y = (int64_t*)malloc(P * sizeof(int64_t));
  f->z = (int64_t*)malloc(P * sizeof(int64_t));
  f->start = (uint64_t*)malloc(P * sizeof(uint64_t));
  f->tree_first = (int64_t*)malloc((T + 1) * sizeof(int64_t));
  const uint64_t total = 1ull << (3 * lmax);
  int64_t p = 0;
  for (int t = 0; t < T; ++t) {
    f->tree_first[t] = p;
    uint64_t c = 0;
    while (p < P && tree_ids[p] == t) {
      const uint64_t size = 1ull << (3 * (lmax - levels[p]));
      if (c % size || c >= total) { orc3_forest_destroy(f); return ORC_ETILING; }
      f->start[p] = c;
      f->x[p] = (int64_t)compact3(c);
      f->y[p] = (int64_t)compact3(c >> 1);
      f->z[p] = (int64_t)compact3(c >> 2);
      c += size;
      ++p;
    }
    if (c != total) { orc3_forest_destroy(f); return ORC_ETILING; }
  }
  f->tree_first[T] = P;
  *out = f;
  return ORC_OK;
}

int orc3_forest_coords(const orc3_forest* f, int64_t* x, int64_t* y, int64_t* z, int* lmax) {
  for (int64_t p = 0; p < f->P; ++p) { x[p] = f->x[p]; y[p] = f->y[p]; z[p] = f->z[p]; }
  *lmax = f->lmax;
  return ORC_OK;
}

/* the leaf of tree t containing the point (X, Y, Z) in fine units (a level-Lmax cell is 2 units,
 * so 2m units per level-Lmax leaf): the leaf whose Morton range holds the point's finest index */
static int64_t locate3(const orc3_forest* f, int t, int64_t X, int64_t Y, int64_t Z) {
  const int64_t w = 2 * (int64_t)f->m;
  const uint64_t c = morton3((uint64_t)(X / w), (uint64_t)(Y / w), (uint64_t)(Z / w));
  int64_t lo = f->tree_first[t], hi = f->tree_first[t + 1] - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (f->start[mid] <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}

/* move a point of tree t across the faces it lies beyond, axis by axis (x, then y, then z);
 * returns 0 if it reaches a physical face (the point is outside the domain) */
static int cross3(const orc3_forest* f, int* t, int64_t P[3]) {
  const int64_t E = (2 * (int64_t)f->m) << f->lmax;
  for (int a = 0; a < 3; ++a) {
    if (P[a] < 0 || P[a] >= E) {
      const int fc = 2 * a + (P[a] >= E);
      if (f->fbc[6 * *t + fc]) return 0;
      *t = f->t2t[6 * *t + fc];
      P[a] += P[a] < 0 ? E : -E;
    }
  }
  return 1;
}

int orc3_ring_count(int m) { const int n = N3(m); return n * n * n - m * m * m; }

/* canonical records of patch p: ring cells in storage order (k = -1..m+2 outer, j, i inner,
 * interior skipped), 8 int32 each {op, src_patch, si, sj, sk, a, b, c}:
 *   1 COPY (source cell), 2 AVG8 (lower corner cell of the 2x2x2 fine block), 3 INTERP (coarse
 *   cell; a, b, c = +-1 the half of it the ghost centre lies in), 4 / 5 / 6 BCX / BCY / BCZ
 *   (outflow: own cell with that axis clamped to 1 or m, the last physical axis of x, y, z) */
int orc3_ghost_records(const orc3_forest* f, int64_t p, int32_t* rec) {
  const int m = f->m, l = f->level[p];
  const int64_t sz = 1ll << (f->lmax - l);        /* leaf size in level-Lmax leaves */
  const int64_t h = sz;                            /* half a cell of p in fine units */
  const int64_t O[3] = {f->x[p] * 2 * m, f->y[p] * 2 * m, f->z[p] * 2 * m};
  int r = 0;
  for (int k = -1; k <= m + 2; ++k)
    for (int j = -1; j <= m + 2; ++j)
      for (int i = -1; i <= m + 2; ++i) {
        if (i >= 1 && i <= m && j >= 1 && j <= m && k >= 1 && k <= m) continue;
        int32_t* o = rec + 8 * (r++);
        memset(o, 0, 8 * sizeof(int32_t));
        const int ijk[3] = {i, j, k};
        int64_t Pt[3];
        for (int a = 0; a < 3; ++a) Pt[a] = O[a] + (2 * ijk[a] - 1) * h;   /* the ghost centre */
        int t = f->tree[p];
        if (!cross3(f, &t, Pt)) {
          /* outflow: the final BC writer is the last physical axis (x, y, z order) */
          int64_t Q[3] = {O[0] + (2 * i - 1) * h, O[1] + (2 * j - 1) * h, O[2] + (2 * k - 1) * h};
          const int64_t E = (2 * (int64_t)m) << f->lmax;
          int last = -1;
          int tt = f->tree[p];
          for (int a = 0; a < 3; ++a) {
            if (Q[a] < 0 || Q[a] >= E) {
              const int fc = 2 * a + (Q[a] >= E);
              if (f->fbc[6 * tt + fc]) last = a;
              else { tt = f->t2t[6 * tt + fc]; Q[a] += Q[a] < 0 ? E : -E; }
            }
          }
          o[0] = 4 + last;
          o[1] = (int32_t)p;
          o[2] = i; o[3] = j; o[4] = k;
          o[2 + last] = ijk[last] < 1 ? 1 : m;
          continue;
        }
        const int64_t L = locate3(f, t, Pt[0], Pt[1], Pt[2]);
        const int lL = f->level[L];
        const int64_t LO[3] = {f->x[L] * 2 * m, f->y[L] * 2 * m, f->z[L] * 2 * m};
        int64_t rel[3];
        for (int a = 0; a < 3; ++a) rel[a] = Pt[a] - LO[a];
        o[1] = (int32_t)L;
        if (lL == l) {                      /* same level: the coinciding cell */
          o[0] = 1;
          for (int a = 0; a < 3; ++a) o[2 + a] = (int32_t)((rel[a] / h + 1) / 2);
        } else if (lL == l + 1) {           /* finer: the 2x2x2 block centred on the ghost centre */
          o[0] = 2;
          for (int a = 0; a < 3; ++a) o[2 + a] = (int32_t)(rel[a] / h);   /* fine cells are h wide */
        } else if (lL == l - 1) {           /* coarser: the containing coarse cell and the half */
          o[0] = 3;
          for (int a = 0; a < 3; ++a) {
            const int64_t I = rel[a] / (4 * h);
            o[2 + a] = (int32_t)(I + 1);
            o[5 + a] = (rel[a] - I * 4 * h > 2 * h) ? 1 : -1;
          }
        } else {
          return ORC_EBALANCE;
        }
      }
  return ORC_OK;
}

int orc3_ghost_table(const orc3_forest* f, int32_t* rec) {
  const int G = orc3_ring_count(f->m);
  for (int64_t p = 0; p < f->P; ++p) {
    int rc = orc3_ghost_records(f, p, rec + (size_t)p * G * 8);
    if (rc) return rc;
  }
  return ORC_OK;
}

static double minmod3(double a, double b) {   /* sign tests, no products */
  if (a > 0.0 && b > 0.0) return a < b ? a : b;
  if (a < 0.0 && b < 0.0) return a > b ? a : b;
  return 0.0;
}

/* ghost fill of qpad[P][n^3], phases A -> C -> per level [B -> C] */
int orc3_ghost_fill(const orc3_forest* f, double* qpad) {
  const int m = f->m, n = N3(m), G = orc3_ring_count(m);
  const int64_t S = (int64_t)n * n * n;
  int32_t* rec = (int32_t*)malloc((size_t)f->P * G * 8 * sizeof(int32_t));
  int rc = orc3_ghost_table(f, rec);
  if (rc) { free(rec); return rc; }
  int64_t* dst = (int64_t*)malloc((size_t)G * sizeof(int64_t));
  { int r = 0;
    for (int k = -1; k <= m + 2; ++k)
      for (int j = -1; j <= m + 2; ++j)
        for (int i = -1; i <= m + 2; ++i)
          if (!(i >= 1 && i <= m && j >= 1 && j <= m && k >= 1 && k <= m)) dst[r++] = IDX3(m, i, j, k); }
  /* A: copy and average (sources are interiors) */
  for (int64_t p = 0; p < f->P; ++p)
    for (int r = 0; r < G; ++r) {
      const int32_t* o = rec + ((size_t)p * G + r) * 8;
      const double* s = qpad + (int64_t)o[1] * S;
      double* g = qpad + p * S + dst[r];
      if (o[0] == 1) {
        *g = s[IDX3(m, o[2], o[3], o[4])];
      } else if (o[0] == 2) {
        const int a = o[2], b = o[3], c = o[4];
        const double lo = (s[IDX3(m, a, b, c)] + s[IDX3(m, a + 1, b, c)]) +
                          (s[IDX3(m, a, b + 1, c)] + s[IDX3(m, a + 1, b + 1, c)]);
        const double hi = (s[IDX3(m, a, b, c + 1)] + s[IDX3(m, a + 1, b, c + 1)]) +
                          (s[IDX3(m, a, b + 1, c + 1)] + s[IDX3(m, a + 1, b + 1, c + 1)]);
        *g = (lo + hi) * 0.125;
      }
    }
  /* C: outflow BCs, x then y then z writers */
  for (int bc = 4; bc <= 6; ++bc)
    for (int64_t p = 0; p < f->P; ++p)
      for (int r = 0; r < G; ++r) {
        const int32_t* o = rec + ((size_t)p * G + r) * 8;
        if (o[0] == bc) qpad[p * S + dst[r]] = qpad[p * S + IDX3(m, o[2], o[3], o[4])];
      }
  /* B per level ascending (the coarse patch's padded array after A and C), then C again */
  int lmin = 99, lmx = -1;
  for (int64_t p = 0; p < f->P; ++p) { if (f->level[p] < lmin) lmin = f->level[p]; if (f->level[p] > lmx) lmx = f->level[p]; }
  for (int lv = lmin; lv <= lmx; ++lv) {
    for (int64_t p = 0; p < f->P; ++p) {
      if (f->level[p] != lv) continue;
      for (int r = 0; r < G; ++r) {
        const int32_t* o = rec + ((size_t)p * G + r) * 8;
        if (o[0] != 3) continue;
        const double* s = qpad + (int64_t)o[1] * S;
        const int I = o[2], J = o[3], K = o[4];
        const double qc = s[IDX3(m, I, J, K)];
        const double sx = minmod3(s[IDX3(m, I + 1, J, K)] - qc, qc - s[IDX3(m, I - 1, J, K)]);
        const double sy = minmod3(s[IDX3(m, I, J + 1, K)] - qc, qc - s[IDX3(m, I, J - 1, K)]);
        const double sz = minmod3(s[IDX3(m, I, J, K + 1)] - qc, qc - s[IDX3(m, I, J, K - 1)]);
        qpad[p * S + dst[r]] = qc + 0.25 * ((o[5] * sx + o[6] * sy) + o[7] * sz);
      }
    }
    for (int bc = 4; bc <= 6; ++bc)
      for (int64_t p = 0; p < f->P; ++p) {
        if (f->level[p] != lv) continue;
        for (int r = 0; r < G; ++r) {
          const int32_t* o = rec + ((size_t)p * G + r) * 8;
          if (o[0] == bc) qpad[p * S + dst[r]] = qpad[p * S + IDX3(m, o[2], o[3], o[4])];
        }
      }
  }
  free(dst);
  free(rec);
  return ORC_OK;
}

/* 1D wave propagation along one pencil of c = 0..N+3 cells (N = m, 2 ghosts each side), updating
 * cells 2..N+1 in place into out; returns max (dt/dx) |s| (LeVeque 2002 §6, scalar advection) */
static double sweep1(const double* q, double* out, int N, double s, double r, int limiter, int method2) {
  double W[64], F[64];
  for (int c = 1; c <= N + 3; ++c) W[c] = q[c] - q[c - 1];
  for (int c = 2; c <= N + 2; ++c) {
    F[c] = 0.0;
    if (method2 == 2 && W[c] != 0.0) {
      const double th = W[s > 0.0 ? c - 1 : c + 1] / W[c];
      const double phi = orc_limiter(limiter, th);
      const double as = fabs(s);
      F[c] = 0.5 * as * (1.0 - r * as) * phi * W[c];
    }
  }
  const double sp = s > 0.0 ? s : 0.0, sm = s < 0.0 ? s : 0.0;
  for (int c = 2; c <= N + 1; ++c)
    out[c] = q[c] - r * (sp * W[c] + sm * W[c + 1]) - r * (F[c + 1] - F[c]);
  return r * fabs(s);
}

/* one Godunov-split step of one padded patch (ring filled): x sweep over j, k = -1..m+2, y sweep
 * over i = 1..m, k = -1..m+2, z sweep over the interior; qnew's interior receives the result */
double orc3_step_patch(const orc3_forest* f, const double* qp, double u, double v, double w, int limiter,
                       int method2, double dt, double dx, double* qnew) {
  const int m = f->m, n = N3(m);
  const int64_t S = (int64_t)n * n * n;
  double* a = (double*)malloc(S * sizeof(double));
  memcpy(a, qp, S * sizeof(double));
  const double r = dt / dx;
  double line[64], res[64], cfl = 0.0;
  for (int k = -1; k <= m + 2; ++k)
    for (int j = -1; j <= m + 2; ++j) {
      for (int c = 0; c < n; ++c) line[c] = a[IDX3(m, c - 1, j, k)];
      cfl = fmax(cfl, sweep1(line, res, m, u, r, limiter, method2));
      for (int c = 2; c <= m + 1; ++c) a[IDX3(m, c - 1, j, k)] = res[c];
    }
  for (int k = -1; k <= m + 2; ++k)
    for (int i = 1; i <= m; ++i) {
      for (int c = 0; c < n; ++c) line[c] = a[IDX3(m, i, c - 1, k)];
      cfl = fmax(cfl, sweep1(line, res, m, v, r, limiter, method2));
      for (int c = 2; c <= m + 1; ++c) a[IDX3(m, i, c - 1, k)] = res[c];
    }
  for (int j = 1; j <= m; ++j)
    for (int i = 1; i <= m; ++i) {
      for (int c = 0; c < n; ++c) line[c] = a[IDX3(m, i, j, c - 1)];
      cfl = fmax(cfl, sweep1(line, res, m, w, r, limiter, method2));
      for (int c = 2; c <= m + 1; ++c) qnew[IDX3(m, i, j, c - 1)] = res[c];
    }
  free(a);
  return cfl;
}

/* ghost fill of qpad, then every patch's split step into qout's interiors; dx0 = level-0 cell */
int orc3_step(const orc3_forest* f, double* qpad, double u, double v, double w, int limiter, int method2,
              double dt, double dx0, double* qout, double* cfl) {
  int rc = orc3_ghost_fill(f, qpad);
  if (rc) return rc;
  const int64_t S = (int64_t)N3(f->m) * N3(f->m) * N3(f->m);
  double c = 0.0;
  for (int64_t p = 0; p < f->P; ++p) {
    memcpy(qout + p * S, qpad + p * S, S * sizeof(double));
    const double dx = ldexp(dx0, -f->level[p]);
    c = fmax(c, orc3_step_patch(f, qpad + p * S, u, v, w, limiter, method2, dt, dx, qout + p * S));
  }
  *cfl = c;
  return ORC_OK;
}
