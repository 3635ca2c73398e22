/* ghost.c -- oracle: ghost-cell fill (TEST INFRASTRUCTURE ONLY, see oracle.h).
 *
 * PAPER.md:187-201 [§3]: "Neighboring patches at the same level of refinement simply copy their
 * interior edge values into a neighbors' ghost cells.  Neighboring fine grid patches average their
 * interior edge data to a coarser neighbor's ghost cell values.  And neighboring coarse grid
 * patches interpolate data ... we use a standard conservative, limited interpolation scheme".
 * Readings (DESIGN.md "Readings" 5-9):
 *   COPY    g = Q_src(i', j')
 *   AVG4    g = ((s00 + s10) + (s01 + s11)) * 0.25                  in the source frame
 *   INTERP  g = Q(I,J) + 0.25 (sx*sx_slope + sy*sy_slope),  slopes = minmod of one-sided
 *           differences of the coarse padded array, signs in the coarse frame
 *   BCX/BCY outflow: first interior cell; wall: mirror, normal momentum negated (meqn >= 3)
 *   CORNER3 g = 0.5 (Q(a, mirror b) + Q(mirror a, b))
 * Phase order: A (COPY, AVG4) -> C (BCX then BCY) -> for each level ascending
 * [B (INTERP into patches of that level) -> C (those patches)] -> CORNER3.
 */
#include <stdlib.h>
#include <string.h>
#include "oracle.h"
#include "oracle_internal.h"

static double minmod(double a, double b) {
  if (a > 0.0 && b > 0.0) return a < b ? a : b;
  if (a < 0.0 && b < 0.0) return a > b ? a : b;
  return 0.0;
}

/* accessor: component k of 1-based cell (i, j) of a padded patch array */
#define QP(base, m, k, i, j) ((base)[(size_t)(k) * ORC_N(m) * ORC_N(m) + ORC_IDX(m, i, j)])

/* Apply one record to ring cell (i, j) of destination array dst.  src_of(patch) returns the
 * padded array of a source patch; own is dst itself. */
typedef const double* (*src_fn)(void* ctx, int64_t patch);

static void apply_record(const int32_t* o, int m, int meqn, double* dst, int i, int j,
                         src_fn src_of, void* ctx) {
  const int op = o[0];
  const double* S = (op == ORC_OP_BCX || op == ORC_OP_BCY || op == ORC_OP_CORNER3)
                        ? dst : src_of(ctx, o[1]);
  const int a = o[2], b = o[3];
  for (int k = 0; k < meqn; ++k) {
    double g;
    switch (op) {
      case ORC_OP_COPY:
        g = QP(S, m, k, a, b);
        break;
      case ORC_OP_AVG4:
        g = ((QP(S, m, k, a, b) + QP(S, m, k, a + 1, b)) +
             (QP(S, m, k, a, b + 1) + QP(S, m, k, a + 1, b + 1))) * 0.25;
        break;
      case ORC_OP_INTERP: {
        double c = QP(S, m, k, a, b);
        double sx = minmod(QP(S, m, k, a + 1, b) - c, c - QP(S, m, k, a - 1, b));
        double sy = minmod(QP(S, m, k, a, b + 1) - c, c - QP(S, m, k, a, b - 1));
        g = c + 0.25 * ((double)o[4] * sx + (double)o[5] * sy);
        break;
      }
      case ORC_OP_BCX:
      case ORC_OP_BCY: {
        g = QP(S, m, k, a, b);
        int normal = (op == ORC_OP_BCX) ? 1 : 2;
        if (o[4] == ORC_BC_WALL && meqn >= 3 && k == normal) g = -g;
        break;
      }
      case ORC_OP_CORNER3:
        g = 0.5 * (QP(S, m, k, a, b) + QP(S, m, k, o[6], o[7]));
        break;
      default:
        continue;
    }
    QP(dst, m, k, i, j) = g;
  }
}

/* iterate the ring of one patch in canonical order, applying records whose op is in `mask` */
static void ring_pass(const int32_t* rec, int m, int meqn, double* dst, unsigned mask,
                      src_fn src_of, void* ctx) {
  int r = 0;
  for (int j = -1; j <= m + 2; ++j)
    for (int i = -1; i <= m + 2; ++i) {
      if (i >= 1 && i <= m && j >= 1 && j <= m) continue;
      const int32_t* o = rec + ORC_REC * (r++);
      if (mask & (1u << o[0])) apply_record(o, m, meqn, dst, i, j, src_of, ctx);
    }
}

#define M_A ((1u << ORC_OP_COPY) | (1u << ORC_OP_AVG4))
#define M_BCX (1u << ORC_OP_BCX)
#define M_BCY (1u << ORC_OP_BCY)
#define M_B (1u << ORC_OP_INTERP)
#define M_C3 (1u << ORC_OP_CORNER3)

typedef struct { double* qpad; int m, meqn; } full_ctx;
static const double* full_src(void* ctx, int64_t patch) {
  full_ctx* c = (full_ctx*)ctx;
  return c->qpad + (size_t)patch * c->meqn * ORC_N(c->m) * ORC_N(c->m);
}

int orc_ghost_fill(const orc_forest* f, double* qpad, int meqn) {
  int rc;
  const int32_t* tab = orc_cached_table(f, &rc);
  if (!tab) return rc;
  const int m = f->m;
  const int64_t G = orc_ring_count(m);
  const size_t S = (size_t)meqn * ORC_N(m) * ORC_N(m);
  full_ctx ctx = {qpad, m, meqn};
  for (int64_t p = 0; p < f->P; ++p)          /* A */
    ring_pass(tab + p * G * ORC_REC, m, meqn, qpad + p * S, M_A, full_src, &ctx);
  for (int64_t p = 0; p < f->P; ++p) {        /* C */
    ring_pass(tab + p * G * ORC_REC, m, meqn, qpad + p * S, M_BCX, full_src, &ctx);
    ring_pass(tab + p * G * ORC_REC, m, meqn, qpad + p * S, M_BCY, full_src, &ctx);
  }
  for (int l = 0; l <= f->lmax; ++l) {        /* B, C per level ascending */
    for (int64_t p = 0; p < f->P; ++p)
      if (f->level[p] == l)
        ring_pass(tab + p * G * ORC_REC, m, meqn, qpad + p * S, M_B, full_src, &ctx);
    for (int64_t p = 0; p < f->P; ++p)
      if (f->level[p] == l) {
        ring_pass(tab + p * G * ORC_REC, m, meqn, qpad + p * S, M_BCX, full_src, &ctx);
        ring_pass(tab + p * G * ORC_REC, m, meqn, qpad + p * S, M_BCY, full_src, &ctx);
      }
  }
  for (int64_t p = 0; p < f->P; ++p)          /* CORNER3 */
    ring_pass(tab + p * G * ORC_REC, m, meqn, qpad + p * S, M_C3, full_src, &ctx);
  return ORC_OK;
}

/* ---- sampled mode: build one patch's padded array from interior-only data ---------------- */
typedef struct {
  const orc_forest* f;
  const double* q;       /* [P][meqn][m][m] interiors */
  int meqn;
  double* scratch;       /* padded array of the last built source patch */
  int depth;
  int rc;
} sample_ctx;

static int build_padded(sample_ctx* c, int64_t p, double* out);

static const double* sample_src(void* vctx, int64_t patch) {
  sample_ctx* c = (sample_ctx*)vctx;
  const int m = c->f->m;
  const size_t S = (size_t)c->meqn * ORC_N(m) * ORC_N(m);
  double* buf = c->scratch + (size_t)(c->depth + 1) * S;
  c->depth++;
  int rc = build_padded(c, patch, buf);
  c->depth--;
  if (rc) c->rc = rc;
  return buf;
}

/* interior copy + the ring in phase order (INTERP sources rebuilt recursively) */
static int build_padded(sample_ctx* c, int64_t p, double* out) {
  const int m = c->f->m, meqn = c->meqn;
  const int64_t G = orc_ring_count(m);
  if (c->depth > 40) return ORC_EBALANCE;
  for (int k = 0; k < meqn; ++k)
    for (int j = 1; j <= m; ++j)
      for (int i = 1; i <= m; ++i)
        QP(out, m, k, i, j) = c->q[(((size_t)p * meqn + k) * m + (j - 1)) * m + (i - 1)];
  int32_t* rec = (int32_t*)malloc(G * ORC_REC * sizeof(int32_t));
  if (!rec) return ORC_ENOMEM;
  int rc = orc_ghost_records(c->f, p, rec);
  if (rc) { free(rec); return rc; }
  /* phase A reads neighbour interiors only: serve them from a padded copy built without ring */
  int r = 0;
  for (int j = -1; j <= m + 2; ++j)
    for (int i = -1; i <= m + 2; ++i) {
      if (i >= 1 && i <= m && j >= 1 && j <= m) continue;
      const int32_t* o = rec + ORC_REC * (r++);
      if (o[0] != ORC_OP_COPY && o[0] != ORC_OP_AVG4) continue;
      for (int k = 0; k < meqn; ++k) {
        const double* I = c->q + ((size_t)o[1] * meqn + k) * m * m;
#define QI(ii, jj) I[((jj) - 1) * m + ((ii) - 1)]
        double g;
        if (o[0] == ORC_OP_COPY) g = QI(o[2], o[3]);
        else g = ((QI(o[2], o[3]) + QI(o[2] + 1, o[3])) + (QI(o[2], o[3] + 1) + QI(o[2] + 1, o[3] + 1))) * 0.25;
#undef QI
        QP(out, m, k, i, j) = g;
      }
    }
  ring_pass(rec, m, meqn, out, M_BCX, sample_src, c);
  ring_pass(rec, m, meqn, out, M_BCY, sample_src, c);
  ring_pass(rec, m, meqn, out, M_B, sample_src, c);
  ring_pass(rec, m, meqn, out, M_BCX, sample_src, c);
  ring_pass(rec, m, meqn, out, M_BCY, sample_src, c);
  ring_pass(rec, m, meqn, out, M_C3, sample_src, c);
  free(rec);
  return c->rc;
}

int orc_build_padded_sample(const orc_forest* f, const double* q, int meqn, int64_t p, double* out) {
  const int m = f->m;
  const size_t S = (size_t)meqn * ORC_N(m) * ORC_N(m);
  sample_ctx c = {f, q, meqn, NULL, 0, 0};
  c.scratch = (double*)calloc((size_t)48 * S, sizeof(double));
  if (!c.scratch) return ORC_ENOMEM;
  int rc = build_padded(&c, p, out);
  free(c.scratch);
  return rc;
}
