/* regrid.c -- oracle: dynamic regridding of the forest (TEST INFRASTRUCTURE ONLY, see oracle.h).
 *
 * PAPER.md:148-155 [§2] "refinement ... with the 2:1 balance condition ... the size difference of
 * neighbouring leaves is at most a factor of two"; PAPER.md:207-211 [§3] "Mesh refinement and
 * coarsening requires interpolation from coarse grids to newly created fine grids, and the
 * averaging of fine grid data to a newly created underlying coarse grid"; SURVEY §8(f) #3 "tag
 * (max - min > threshold), refine (interpolate new fine), coarsen (average new coarse), 2:1 balance".
 *
 * Written out plainly (readings in DESIGN.md), one rank:
 *   tag:      d_p = max - min of component 0 over the interior of patch p;
 *   refine:   d_p > refine_threshold and level < max_level;
 *   balance:  repeat until nothing changes: a leaf that will be refined to l+1 forces every face or
 *             corner neighbour whose new level would be <= l-1 to refine as well (point location
 *             just outside each face midpoint and corner, crossing tree faces);
 *   coarsen:  4 consecutive leaves forming a complete family of level l > min_level, none refined,
 *             all with d < coarsen_threshold, and no face or corner neighbour of any of them (outside
 *             the family) with a new level above l;
 *   new leaves in Morton order: refined leaves -> their 4 children (z-order), families -> parent;
 *   data:     copy; new fine cell = parent cell + 1/4 (sx sigma_x + sy sigma_y) with minmod slopes of
 *             the parent's ghost-filled array (the ghost fill's limited interpolation, reading 6);
 *             new coarse cell = ((a + b) + (c + d)) / 4 of its 2 x 2 children cells (reading 7).
 * Point location is a linear search over the leaves: slow and obviously correct.
 */
#include <stdlib.h>
#include <string.h>
#include "oracle.h"
#include "oracle_internal.h"

typedef struct {
  int t, l;
  int64_t X, Y;   /* origin in units of level-U leaves */
} rleaf;

/* leaf containing the point (px, py), in half-units of a level-U leaf, of tree t; -1 if none */
static int64_t rfind(const rleaf* L, int64_t n, int U, int t, int64_t px, int64_t py) {
  for (int64_t i = 0; i < n; ++i) {
    if (L[i].t != t) continue;
    const int64_t s = 2 * (1ll << (U - L[i].l));
    if (px >= 2 * L[i].X && px < 2 * L[i].X + s && py >= 2 * L[i].Y && py < 2 * L[i].Y + s) return i;
  }
  return -1;
}

/* move a point across face `face` of tree *t (tree edge E half-units); 1 if the face is physical */
static int rcross(const orc_forest* f, int64_t E, int* t, int64_t* X, int64_t* Y, int face) {
  const int tt = *t, nt = f->t2t[4 * tt + face], code = f->t2f[4 * tt + face];
  const int nf = code & 3, rev = code >> 2;
  if (nt == tt && nf == face) return 1;
  int64_t d, tau;
  switch (face) {
    case 0: d = -*X; tau = *Y; break;
    case 1: d = *X - E; tau = *Y; break;
    case 2: d = -*Y; tau = *X; break;
    default: d = *Y - E; tau = *X; break;
  }
  if (rev) tau = E - tau;
  switch (nf) {
    case 0: *X = d; *Y = tau; break;
    case 1: *X = E - d; *Y = tau; break;
    case 2: *X = tau; *Y = d; break;
    default: *X = tau; *Y = E - d; break;
  }
  *t = nt;
  return 0;
}

/* leaves at the point (px, py) of tree t, which may lie outside the tree (across one face, or a
 * corner: both routes x-then-y and y-then-x are taken).  Writes up to 2 leaf ids, returns count. */
static int rlocate(const orc_forest* f, const rleaf* L, int64_t n, int U, int t, int64_t px, int64_t py,
                   int64_t out[2]) {
  const int64_t E = 2 * (1ll << U);
  int cnt = 0;
  for (int first = 0; first < 2; ++first) {
    int tt = t;
    int64_t x = px, y = py, phys = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const int axis = pass == 0 ? first : 1 - first;
      int face = -1;
      if (axis == 0) face = x < 0 ? 0 : (x >= E ? 1 : -1);
      else face = y < 0 ? 2 : (y >= E ? 3 : -1);
      if (face >= 0 && rcross(f, E, &tt, &x, &y, face)) { phys = 1; break; }
    }
    if (phys || x < 0 || y < 0 || x >= E || y >= E) continue;
    const int64_t q = rfind(L, n, U, tt, x, y);
    if (q >= 0 && !(cnt == 1 && out[0] == q)) out[cnt++] = q;
  }
  return cnt;
}

static double rminmod(double a, double b) {
  if (a > 0.0 && b > 0.0) return a < b ? a : b;
  if (a < 0.0 && b < 0.0) return a > b ? a : b;
  return 0.0;
}

int orc_regrid(const orc_forest* f, const double* qpad, int meqn, double refine_threshold,
               double coarsen_threshold, int min_level, int max_level, int64_t* new_P, int8_t* new_levels,
               int32_t* new_trees, double* qout, int32_t* src) {
  const int m = f->m, n = ORC_N(m);
  const size_t S = (size_t)meqn * n * n, SI = (size_t)meqn * m * m;
  const int64_t P = f->P;
  const int U = max_level > f->lmax ? max_level : f->lmax;
  if (U > 28 || m % 2) return ORC_EINVAL;
  rleaf* L = (rleaf*)malloc(P * sizeof(rleaf));
  double* d = (double*)malloc(P * sizeof(double));
  int* refine = (int*)calloc(P, sizeof(int));
  int* coarsen = (int*)calloc(P, sizeof(int));   /* 1 on the first leaf of an accepted family */
  if (!L || !d || !refine || !coarsen) { free(L); free(d); free(refine); free(coarsen); return ORC_ENOMEM; }
  for (int64_t p = 0; p < P; ++p) {
    L[p].t = f->tree[p];
    L[p].l = f->level[p];
    L[p].X = f->x[p] << (U - f->lmax);
    L[p].Y = f->y[p] << (U - f->lmax);
    double lo = qpad[p * S + ORC_IDX(m, 1, 1)], hi = lo;
    for (int j = 1; j <= m; ++j)
      for (int i = 1; i <= m; ++i) {
        const double v = qpad[p * S + ORC_IDX(m, i, j)];
        if (v < lo) lo = v;
        if (v > hi) hi = v;
      }
    d[p] = hi - lo;
    refine[p] = d[p] > refine_threshold && f->level[p] < max_level;
  }
  /* 2:1 balance of the refinement */
  for (int changed = 1; changed;) {
    changed = 0;
    for (int64_t p = 0; p < P; ++p) {
      if (!refine[p]) continue;
      const int64_t s = 2 * (1ll << (U - L[p].l));   /* leaf size in half-units */
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!dx && !dy) continue;
          const int64_t px = dx < 0 ? 2 * L[p].X - 1 : (dx > 0 ? 2 * L[p].X + s : 2 * L[p].X + s / 2);
          const int64_t py = dy < 0 ? 2 * L[p].Y - 1 : (dy > 0 ? 2 * L[p].Y + s : 2 * L[p].Y + s / 2);
          int64_t q[2];
          const int c = rlocate(f, L, P, U, L[p].t, px, py, q);
          for (int k = 0; k < c; ++k)
            if (L[q[k]].l + refine[q[k]] <= L[p].l - 1) { refine[q[k]] = 1; changed = 1; }
        }
    }
  }
  /* coarsening of complete families */
  for (int64_t p = 0; p + 3 < P; ++p) {
    const int l = L[p].l;
    if (l <= min_level || l == 0) continue;
    const int64_t cs = 1ll << (U - l);
    if ((L[p].X / cs) % 2 || (L[p].Y / cs) % 2) continue;
    int ok = 1;
    for (int k = 0; k < 4 && ok; ++k) {
      const rleaf* c = &L[p + k];
      ok = c->t == L[p].t && c->l == l && c->X == L[p].X + (k & 1) * cs && c->Y == L[p].Y + (k >> 1) * cs &&
           !refine[p + k] && d[p + k] < coarsen_threshold;
    }
    for (int k = 0; k < 4 && ok; ++k) {   /* no neighbour of a child finer than l after refinement */
      const int64_t s = 2 * cs, X2 = 2 * L[p + k].X, Y2 = 2 * L[p + k].Y;
      for (int dy = -1; dy <= 1 && ok; ++dy)
        for (int dx = -1; dx <= 1 && ok; ++dx) {
          if (!dx && !dy) continue;
          for (int h = 0; h < 2 && ok; ++h) {   /* 1/4 and 3/4 along a face */
            const int64_t along = h ? 3 * s / 4 : s / 4;
            const int64_t px = dx < 0 ? X2 - 1 : (dx > 0 ? X2 + s : X2 + along);
            const int64_t py = dy < 0 ? Y2 - 1 : (dy > 0 ? Y2 + s : Y2 + along);
            int64_t q[2];
            const int c = rlocate(f, L, P, U, L[p].t, px, py, q);
            for (int j = 0; j < c; ++j)
              if (!(q[j] >= p && q[j] < p + 4) && L[q[j]].l + refine[q[j]] > l) ok = 0;
            if (dx && dy) break;                /* a corner has one point */
          }
        }
    }
    if (ok) { coarsen[p] = 1; p += 3; }
  }
  /* new leaves and data */
  int64_t np = 0;
  for (int64_t p = 0; p < P; ++p) {
    const double* qp = qpad + p * S;
    if (refine[p]) {
      for (int k = 0; k < 4; ++k, ++np) {
        new_levels[np] = (int8_t)(L[p].l + 1);
        new_trees[np] = L[p].t;
        if (src) { src[np * 6 + 0] = 2; src[np * 6 + 1] = (int32_t)p; src[np * 6 + 2] = k; }
        const int ox = k & 1, oy = k >> 1;
        for (int e = 0; e < meqn; ++e)
          for (int j = 1; j <= m; ++j)
            for (int i = 1; i <= m; ++i) {
              const int I = ox * (m / 2) + (i + 1) / 2, J = oy * (m / 2) + (j + 1) / 2;
              const double sgx = (i & 1) ? -1.0 : 1.0, sgy = (j & 1) ? -1.0 : 1.0;
              const double* Q = qp + (size_t)e * n * n;
              const double c = Q[ORC_IDX(m, I, J)];
              const double sx = rminmod(Q[ORC_IDX(m, I + 1, J)] - c, c - Q[ORC_IDX(m, I - 1, J)]);
              const double sy = rminmod(Q[ORC_IDX(m, I, J + 1)] - c, c - Q[ORC_IDX(m, I, J - 1)]);
              qout[np * SI + ((size_t)e * m + (j - 1)) * m + (i - 1)] = c + 0.25 * (sgx * sx + sgy * sy);
            }
      }
    } else if (coarsen[p]) {
      new_levels[np] = (int8_t)(L[p].l - 1);
      new_trees[np] = L[p].t;
      if (src) { src[np * 6 + 0] = 3; src[np * 6 + 1] = (int32_t)p; src[np * 6 + 2] = 0; }
      for (int e = 0; e < meqn; ++e)
        for (int J = 1; J <= m; ++J)
          for (int I = 1; I <= m; ++I) {
            const int k = (I > m / 2) + 2 * (J > m / 2);
            const int a = 2 * (I - (I > m / 2) * (m / 2)), b = 2 * (J - (J > m / 2) * (m / 2));
            const double* Q = qpad + (p + k) * S + (size_t)e * n * n;
            const double v = ((Q[ORC_IDX(m, a - 1, b - 1)] + Q[ORC_IDX(m, a, b - 1)]) +
                              (Q[ORC_IDX(m, a - 1, b)] + Q[ORC_IDX(m, a, b)])) * 0.25;
            qout[np * SI + ((size_t)e * m + (J - 1)) * m + (I - 1)] = v;
          }
      ++np;
      p += 3;
    } else {
      new_levels[np] = (int8_t)L[p].l;
      new_trees[np] = L[p].t;
      if (src) { src[np * 6 + 0] = 1; src[np * 6 + 1] = (int32_t)p; src[np * 6 + 2] = 0; }
      for (int e = 0; e < meqn; ++e)
        for (int j = 1; j <= m; ++j)
          for (int i = 1; i <= m; ++i)
            qout[np * SI + ((size_t)e * m + (j - 1)) * m + (i - 1)] = qp[(size_t)e * n * n + ORC_IDX(m, i, j)];
      ++np;
    }
  }
  *new_P = np;
  free(L); free(d); free(refine); free(coarsen);
  return ORC_OK;
}
