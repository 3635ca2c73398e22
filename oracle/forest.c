/* forest.c -- oracle: forest decode and brute-force ghost-source classification.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Shares no code with the product path.
 *
 * Decode (PAPER.md:240-245 [§4] "leaf ordering ... according to a space filling
 * curve"): per tree, a cursor c runs through the 4^Lmax Morton index space; a leaf of level l
 * covers [c, c + 4^(Lmax-l)), must start aligned to its size, and (x, y) = de-interleave(c)
 * with x on the even bits.  The tree must be covered exactly.
 *
 * Ghost sources (PAPER.md:137-146 [§2] neighbour lookup with relative
 * orientation, PAPER.md:258-260 [§4] coordinate transformation across blocks
 * [§3] copy / average / interpolate): every ring-cell centre is taken as an exact integer point
 * in units of 1/(2m 2^Lmax) of the tree edge; if it lies outside its tree it crosses the face
 * through tree_to_tree / tree_to_face (tangential coordinate kept or reflected); corner cells
 * cross x-then-y and y-then-x and disagreeing routes mean a 3-tree corner (CORNER3); any
 * physical face crossed means PHYS.  The leaf containing the point is found by Morton-range
 * search (no neighbour logic), and the op follows from its level.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"
#include "oracle_internal.h"

int orc_ring_count(int m) { return (m + 4) * (m + 4) - m * m; }

static uint64_t interleave(uint64_t x, uint64_t y) {
  uint64_t c = 0;
  for (int b = 0; b < 31; ++b) {
    c |= ((x >> b) & 1ull) << (2 * b);
    c |= ((y >> b) & 1ull) << (2 * b + 1);
  }
  return c;
}

static void deinterleave(uint64_t c, int64_t* x, int64_t* y) {
  int64_t xx = 0, yy = 0;
  for (int b = 0; b < 31; ++b) {
    xx |= (int64_t)((c >> (2 * b)) & 1ull) << b;
    yy |= (int64_t)((c >> (2 * b + 1)) & 1ull) << b;
  }
  *x = xx;
  *y = yy;
}

int orc_forest_create(int64_t P, const int8_t* levels, const int32_t* tree_ids, int32_t T,
                      const int32_t* t2t, const int8_t* t2f, const int8_t* fbc, int m,
                      orc_forest** out) {
  *out = NULL;
  if (P <= 0 || T <= 0 || m < 4 || (m % 2) != 0) return ORC_EINVAL;
  /* connectivity: in range and symmetric */
  for (int t = 0; t < T; ++t)
    for (int f = 0; f < 4; ++f) {
      int32_t nt = t2t[4 * t + f];
      int8_t code = t2f[4 * t + f];
      if (nt < 0 || nt >= T || code < 0 || code > 7) return ORC_ECONN;
      int nf = code & 3, rev = code >> 2;
      if (t2t[4 * nt + nf] != t || t2f[4 * nt + nf] != f + 4 * rev) return ORC_ECONN;
      if (nt == t && nf == f && rev) return ORC_ECONN;
    }
  int lmax = 0;
  for (int64_t p = 0; p < P; ++p) {
    if (levels[p] < 0 || levels[p] > 28) return ORC_EINVAL;
    if (levels[p] > lmax) lmax = levels[p];
    if (tree_ids[p] < 0 || tree_ids[p] >= T) return ORC_ETILING;
    if (p > 0 && tree_ids[p] < tree_ids[p - 1]) return ORC_ETILING;
  }
  orc_forest* f = (orc_forest*)calloc(1, sizeof(orc_forest));
  if (!f) return ORC_ENOMEM;
  f->P = P; f->T = T; f->m = m; f->lmax = lmax;
  f->level = (int8_t*)malloc(P);
  f->tree = (int32_t*)malloc(P * sizeof(int32_t));
  f->x = (int64_t*)malloc(P * sizeof(int64_t));
  f->y = (int64_t*)malloc(P * sizeof(int64_t));
  f->start = (uint64_t*)malloc(P * sizeof(uint64_t));
  f->tree_first = (int64_t*)malloc((T + 1) * sizeof(int64_t));
  f->t2t = (int32_t*)malloc(4 * T * sizeof(int32_t));
  f->t2f = (int8_t*)malloc(4 * T);
  f->bc = (int8_t*)malloc(4 * T);
  if (!f->level || !f->tree || !f->x || !f->y || !f->start || !f->tree_first || !f->t2t ||
      !f->t2f || !f->bc) { orc_forest_destroy(f); return ORC_ENOMEM; }
  memcpy(f->level, levels, P);
  memcpy(f->tree, tree_ids, P * sizeof(int32_t));
  memcpy(f->t2t, t2t, 4 * T * sizeof(int32_t));
  memcpy(f->t2f, t2f, 4 * T);
  memcpy(f->bc, fbc, 4 * T);
  const uint64_t full = 1ull << (2 * lmax);
  int64_t p = 0;
  for (int t = 0; t < T; ++t) {
    f->tree_first[t] = p;
    uint64_t c = 0;
    while (p < P && tree_ids[p] == t) {
      uint64_t size = 1ull << (2 * (lmax - levels[p]));
      if (c % size != 0 || c + size > full) { orc_forest_destroy(f); return ORC_ETILING; }
      f->start[p] = c;
      deinterleave(c, &f->x[p], &f->y[p]);
      c += size;
      ++p;
    }
    if (c != full) { orc_forest_destroy(f); return ORC_ETILING; }
  }
  f->tree_first[T] = p;
  *out = f;
  return ORC_OK;
}

void orc_forest_destroy(orc_forest* f) {
  if (!f) return;
  free(f->level); free(f->tree); free(f->x); free(f->y); free(f->start); free(f->tree_first);
  free(f->t2t); free(f->t2f); free(f->bc); free(f->table);
  free(f);
}

int orc_forest_coords(const orc_forest* f, int64_t* x, int64_t* y, int* lmax) {
  for (int64_t p = 0; p < f->P; ++p) { x[p] = f->x[p]; y[p] = f->y[p]; }
  *lmax = f->lmax;
  return ORC_OK;
}

/* the leaf of tree t containing the point (X, Y) (units of 1/(2m 2^Lmax)): the leaf whose Morton
 * range holds the point's finest-level Morton index */
static int64_t locate(const orc_forest* f, int t, int64_t X, int64_t Y) {
  const int64_t w = 2 * (int64_t)f->m;               /* a level-Lmax leaf is 2m units wide */
  uint64_t c = interleave((uint64_t)(X / w), (uint64_t)(Y / w));
  int64_t lo = f->tree_first[t], hi = f->tree_first[t + 1] - 1;  /* largest start <= c */
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (f->start[mid] <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}

/* move the point across face `face` of tree *t; returns 1 if that face is physical */
static int cross(const orc_forest* f, int* t, int64_t* X, int64_t* Y, int face) {
  const int64_t E = (2 * (int64_t)f->m) << f->lmax;
  int tt = *t;
  int nt = f->t2t[4 * tt + face];
  int code = f->t2f[4 * tt + face];
  int nf = code & 3, rev = code >> 2;
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

static int out_face(const orc_forest* f, int64_t X, int64_t Y, int axis) {
  const int64_t E = (2 * (int64_t)f->m) << f->lmax;
  if (axis == 0) return X < 0 ? 0 : (X >= E ? 1 : -1);
  return Y < 0 ? 2 : (Y >= E ? 3 : -1);
}

/* route: cross the face of axis `first`, then whatever is still outside. 1 = physical, -1 = bad */
static int route(const orc_forest* f, int first, int* t, int64_t* X, int64_t* Y) {
  int face = out_face(f, *X, *Y, first);
  if (cross(f, t, X, Y, face)) return 1;
  for (int axis = 0; axis < 2; ++axis) {
    int g = out_face(f, *X, *Y, axis);
    if (g >= 0) {
      if (cross(f, t, X, Y, g)) return 1;
      break;
    }
  }
  if (out_face(f, *X, *Y, 0) >= 0 || out_face(f, *X, *Y, 1) >= 0) return -1;
  return 0;
}

static int mirror(int k, int m, int lowside, int wall) {
  if (lowside) return wall ? 1 - k : 1;
  return wall ? 2 * m + 1 - k : m;
}

int orc_ghost_records(const orc_forest* f, int64_t p, int32_t* rec) {
  const int m = f->m;
  const int64_t E = (2 * (int64_t)m) << f->lmax;
  const int l = f->level[p];
  const int64_t s = 1ll << (f->lmax - l);          /* half a cell of p */
  const int64_t X0 = f->x[p] * 2 * m, Y0 = f->y[p] * 2 * m;
  const int t0 = f->tree[p];
  int r = 0;
  for (int j = -1; j <= m + 2; ++j)
    for (int i = -1; i <= m + 2; ++i) {
      if (i >= 1 && i <= m && j >= 1 && j <= m) continue;
      int32_t* o = rec + ORC_REC * (r++);
      memset(o, 0, ORC_REC * sizeof(int32_t));
      int64_t X = X0 + (2 * i - 1) * s, Y = Y0 + (2 * j - 1) * s;
      int ox = out_face(f, X, Y, 0), oy = out_face(f, X, Y, 1);
      int t = t0;
      int phys = 0, corner3 = 0;
      if (ox >= 0 && oy >= 0) {
        int ta = t0, tb = t0;
        int64_t Xa = X, Ya = Y, Xb = X, Yb = Y;
        int ra = route(f, 0, &ta, &Xa, &Ya);
        int rb = route(f, 1, &tb, &Xb, &Yb);
        if (ra < 0 || rb < 0) return ORC_ECONN;
        if (ra == 1 || rb == 1) phys = 1;
        else if (ta != tb || Xa != Xb || Ya != Yb) corner3 = 1;
        else { t = ta; X = Xa; Y = Ya; }
      } else if (ox >= 0 || oy >= 0) {
        int rr = route(f, ox >= 0 ? 0 : 1, &t, &X, &Y);
        if (rr < 0) return ORC_ECONN;
        if (rr == 1) phys = 1;
      }
      if (phys) {
        /* Clawpack bc2 order: x faces, then y faces over all columns, so a y-face BC is the
         * final writer wherever p's own y face is physical (SURVEY §8(c.4) phase C) */
        int ylow = (j < 1), yhigh = (j > m), xlow = (i < 1), xhigh = (i > m);
        int fy = ylow ? 2 : 3, fx = xlow ? 0 : 1;
        int yphys = (ylow && Y0 == 0) || (yhigh && Y0 + 2 * m * s == E);
        yphys = yphys && (ylow || yhigh) && f->t2t[4 * t0 + fy] == t0 && (f->t2f[4 * t0 + fy] & 3) == fy;
        int xphys = (xlow && X0 == 0) || (xhigh && X0 + 2 * m * s == E);
        xphys = xphys && (xlow || xhigh) && f->t2t[4 * t0 + fx] == t0 && (f->t2f[4 * t0 + fx] & 3) == fx;
        if (yphys) {
          int wall = f->bc[4 * t0 + fy] == ORC_BC_WALL;
          o[0] = ORC_OP_BCY; o[1] = (int32_t)p; o[2] = i; o[3] = mirror(j, m, ylow, wall);
          o[4] = f->bc[4 * t0 + fy];
        } else if (xphys) {
          int wall = f->bc[4 * t0 + fx] == ORC_BC_WALL;
          o[0] = ORC_OP_BCX; o[1] = (int32_t)p; o[2] = mirror(i, m, xlow, wall); o[3] = j;
          o[4] = f->bc[4 * t0 + fx];
        } else {
          return ORC_EUNSUP;   /* corner outside a non-convex domain: not supported */
        }
        continue;
      }
      if (corner3) {
        /* 0.5 (Q(a, mirror_y b) + Q(mirror_x a, b)) about the patch's own edges (c.4) */
        int my = (j < 1) ? 1 - j : 2 * m + 1 - j;
        int mx = (i < 1) ? 1 - i : 2 * m + 1 - i;
        o[0] = ORC_OP_CORNER3; o[1] = (int32_t)p; o[2] = i; o[3] = my; o[6] = mx; o[7] = j;
        continue;
      }
      int64_t L = locate(f, t, X, Y);
      int lL = f->level[L];
      int64_t XL = X - f->x[L] * 2 * m, YL = Y - f->y[L] * 2 * m;
      o[1] = (int32_t)L;
      if (lL == l) {
        o[0] = ORC_OP_COPY;
        o[2] = (int32_t)((XL / s + 1) / 2);
        o[3] = (int32_t)((YL / s + 1) / 2);
        if (o[2] < 1 || o[2] > m || o[3] < 1 || o[3] > m) return ORC_EBALANCE;
      } else if (lL == l + 1) {
        o[0] = ORC_OP_AVG4;
        o[2] = (int32_t)(XL / s);
        o[3] = (int32_t)(YL / s);
        if (o[2] < 1 || o[2] > m - 1 || o[3] < 1 || o[3] > m - 1) return ORC_EBALANCE;
      } else if (lL == l - 1) {
        o[0] = ORC_OP_INTERP;
        int64_t I = XL / (4 * s), J = YL / (4 * s);
        o[2] = (int32_t)(I + 1);
        o[3] = (int32_t)(J + 1);
        o[4] = (XL - I * 4 * s > 2 * s) ? 1 : -1;
        o[5] = (YL - J * 4 * s > 2 * s) ? 1 : -1;
        if (o[2] < 1 || o[2] > m || o[3] < 1 || o[3] > m) return ORC_EBALANCE;
      } else {
        return ORC_EBALANCE;
      }
    }
  return ORC_OK;
}

int orc_ghost_table(const orc_forest* f, int32_t* rec) {
  const int64_t G = orc_ring_count(f->m);
  for (int64_t p = 0; p < f->P; ++p) {
    int rc = orc_ghost_records(f, p, rec + p * G * ORC_REC);
    if (rc) return rc;
  }
  return ORC_OK;
}

/* lazily cached full table (oracle-internal) */
const int32_t* orc_cached_table(const orc_forest* fc, int* rc) {
  orc_forest* f = (orc_forest*)fc;
  *rc = ORC_OK;
  if (f->table) return f->table;
  const int64_t G = orc_ring_count(f->m);
  f->table = (int32_t*)malloc((size_t)f->P * G * ORC_REC * sizeof(int32_t));
  if (!f->table) { *rc = ORC_ENOMEM; return NULL; }
  *rc = orc_ghost_table(f, f->table);
  if (*rc) { free(f->table); f->table = NULL; return NULL; }
  return f->table;
}

/* ---- coarse/fine reflux (PAPER.md:279-282 [§4]) ------------------------------ */
/* fine cell of the finer neighbour at the point (X, Y) of tree t (a fine-cell centre); -1 if the
 * leaf there is not one level finer than l */
static int fine_cell(const orc_forest* f, int t, int64_t X, int64_t Y, int l, int64_t sh, int64_t* L,
                     int* i, int* j) {
  const int m = f->m;
  *L = locate(f, t, X, Y);
  if (f->level[*L] != l + 1) return -1;
  *i = (int)(((X - f->x[*L] * 2 * m) / sh + 1) / 2);
  *j = (int)(((Y - f->y[*L] * 2 * m) / sh + 1) / 2);
  return 0;
}

int orc_reflux(const orc_forest* f, const orc_problem* pr, const double* faces, const double* aux,
               double dt, double dx0, double* qout) {
  return orc_reflux_ex(f, pr, faces, faces, 1.0, dt, -1, aux, dx0, qout);
}

/* the reflux of coarse patches of level `level` (all levels if < 0), with the coarse records
 * weighted by wc and the fine ones taken from faces_f:
 *   Q_C += dtr / (kappa dx) (wc out_C + (F_1 + F_2) / 2)
 * global dt: faces_f = faces_c, wc = 1, dtr = dt;  sub-cycling: faces_f = dt-weighted fine sums
 * over the fine sub-steps, wc = dt_coarse, dtr = 1 */
int orc_reflux_ex(const orc_forest* f, const orc_problem* pr, const double* faces, const double* faces_f,
                  double wc, double dtr, int level, const double* aux, double dx0, double* qout) {
  const int m = f->m, meqn = orc_meqn(pr->kind), n = ORC_N(m);
  const size_t S = (size_t)meqn * n * n, SA = (size_t)3 * n * n, FS = (size_t)4 * m * meqn;
  for (int64_t p = 0; p < f->P; ++p) {
    const int l = f->level[p];
    if (l >= f->lmax) continue;                       /* no finer neighbour possible */
    if (level >= 0 && l != level) continue;
    const int64_t s = 1ll << (f->lmax - l);           /* half a cell of p; s / 2 = half a fine cell */
    const int64_t sh = s / 2;
    const int64_t X0 = f->x[p] * 2 * m, Y0 = f->y[p] * 2 * m;
    const double dx = ldexp(dx0, -l);
    for (int sf = 0; sf < 4; ++sf) {
      for (int c = 0; c < m; ++c) {
        const double* oc = faces + p * FS + ((size_t)sf * m + c) * meqn;
        const double* of[2];
        int ok = 1;
        for (int h = 0; h < 2 && ok; ++h) {          /* the two fine edges covering coarse edge c */
          const int64_t tau = 2 * s * c + (h ? 3 * sh : sh);
          int64_t Lc[2];
          int ic[2], jc[2];
          for (int d = 0; d < 2 && ok; ++d) {        /* fine cells at depth 1 and 2 behind the face */
            const int64_t dep = d ? 3 * sh : sh;
            int64_t X, Y;
            switch (sf) {
              case 0: X = X0 - dep; Y = Y0 + tau; break;
              case 1: X = X0 + 2 * m * s + dep; Y = Y0 + tau; break;
              case 2: X = X0 + tau; Y = Y0 - dep; break;
              default: X = X0 + tau; Y = Y0 + 2 * m * s + dep; break;
            }
            int t = f->tree[p];
            const int axis = sf < 2 ? 0 : 1, fo = out_face(f, X, Y, axis);
            if (fo >= 0) {
              const int code = f->t2f[4 * t + fo], nf = code & 3, rev = code >> 2;
              const int t_from = t;
              if (cross(f, &t, &X, &Y, fo)) { ok = 0; break; }   /* physical face */
              if (meqn > 1 && t != t_from && !(nf == (fo ^ 1) && !rev)) return ORC_EUNSUP;
            }
            if (fine_cell(f, t, X, Y, l, sh, &Lc[d], &ic[d], &jc[d])) { ok = 0; break; }
          }
          if (!ok) break;
          if (Lc[0] != Lc[1]) return ORC_EBALANCE;
          const int di = ic[1] - ic[0], dj = jc[1] - jc[0];   /* inward normal in the fine frame */
          int ff, fe;
          if (di == 1 && dj == 0 && ic[0] == 1) { ff = 0; fe = jc[0] - 1; }
          else if (di == -1 && dj == 0 && ic[0] == m) { ff = 1; fe = jc[0] - 1; }
          else if (di == 0 && dj == 1 && jc[0] == 1) { ff = 2; fe = ic[0] - 1; }
          else if (di == 0 && dj == -1 && jc[0] == m) { ff = 3; fe = ic[0] - 1; }
          else return ORC_EBALANCE;
          of[h] = faces_f + Lc[0] * FS + ((size_t)ff * m + fe) * meqn;
        }
        if (!ok) continue;                            /* not a coarse/fine edge */
        const int ci = sf == 0 ? 1 : (sf == 1 ? m : c + 1), cj = sf < 2 ? c + 1 : (sf == 2 ? 1 : m);
        const double kap = aux ? aux[p * SA + ORC_IDX(m, ci, cj)] : 1.0;
        const double r = dtr / (kap * dx);
        for (int k = 0; k < meqn; ++k) {
          const double corr = wc * oc[k] + 0.5 * (of[0][k] + of[1][k]);
          qout[p * S + (size_t)k * n * n + ORC_IDX(m, ci, cj)] += r * corr;
        }
      }
    }
  }
  return ORC_OK;
}
