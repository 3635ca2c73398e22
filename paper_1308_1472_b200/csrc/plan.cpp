// plan.cpp -- libfc host planner: forest decode, per-direction neighbour lookup with inter-tree
// transforms, canonical ghost records, typed GPU work lists and the multi-GPU halo plan.
//
// PAPER.md:137-146 [§2]: "an interface that provides ... the sequence of blocks, the list of
// patches per-block, and a constant-time lookup of neighbor patches (and their relative and, in
// general, nontrivial orientation between blocks)".  PAPER.md:258-260 [§4]: "When ForestClaw
// accesses neighbor patches, they can be on the same or a different block.  In the latter case,
// coordinate transformations are carried out."  PAPER.md:264-272 [§4]: ghost patches of remote
// ranks are exchanged before the local neighbour work.
//
// Unlike the oracle (which locates every ghost-cell centre by a Morton-range search), this planner
// looks up the neighbour region of each of the 8 directions of a patch once, in a hash of
// (tree, level, x, y), after composing face-crossing isometries; cells are then expanded through
// that direction's affine map.  The two must produce bit-identical tables (tests/).
#include <algorithm>
#include <array>
#include <map>
#include <cstring>
#include <tuple>

#include "fc_internal.h"

namespace fc {

static const int NX[4] = {-1, 1, 0, 0}, NY[4] = {0, 0, -1, 1};  // outward normals
static const int TX[4] = {0, 0, 1, 1}, TY[4] = {1, 1, 0, 0};    // tangents

static uint64_t compact_even_bits(uint64_t v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v >> 4)) & 0x00FF00FF00FF00FFull;
  v = (v | (v >> 8)) & 0x0000FFFF0000FFFFull;
  v = (v | (v >> 16)) & 0x00000000FFFFFFFFull;
  return v;
}

static int face_of_normal(int nx, int ny) {
  if (nx < 0) return 0;
  if (nx > 0) return 1;
  if (ny < 0) return 2;
  return 3;
}

static bool is_phys(const Plan& pl, int t, int f) {
  return pl.t2t[4 * t + f] == t && (pl.t2f[4 * t + f] & 3) == f;
}

// isometry carrying points just outside face f of tree t to the neighbour tree's coordinates:
// P' = o_nf + tau'(P) tau_nf - d(P) n_nf with tau = tau_f.(P - o_f), d = n_f.(P - o_f) and
// tau' = tau (aligned) or E - tau (reversed).  Returns false on a physical face.
static bool cross_map(const Plan& pl, int t, int f, int64_t E, Affine& A) {
  const int nt = pl.t2t[4 * t + f], code = pl.t2f[4 * t + f];
  const int nf = code & 3, rev = code >> 2;
  if (nt == t && nf == f) return false;
  const int s = rev ? -1 : 1;
  A.r00 = s * TX[nf] * TX[f] - NX[nf] * NX[f];
  A.r01 = s * TX[nf] * TY[f] - NX[nf] * NY[f];
  A.r10 = s * TY[nf] * TX[f] - NY[nf] * NX[f];
  A.r11 = s * TY[nf] * TY[f] - NY[nf] * NY[f];
  const int64_t ofx = (f == 1) ? E : 0, ofy = (f == 3) ? E : 0;
  const int64_t onx = (nf == 1) ? E : 0, ony = (nf == 3) ? E : 0;
  A.b0 = onx + (rev ? E * TX[nf] : 0) - (A.r00 * ofx + A.r01 * ofy);
  A.b1 = ony + (rev ? E * TY[nf] : 0) - (A.r10 * ofx + A.r11 * ofy);
  A.tree = nt;
  return true;
}

static Affine compose(const Affine& A2, const Affine& A1) {  // A2 o A1
  Affine C;
  C.r00 = A2.r00 * A1.r00 + A2.r01 * A1.r10;
  C.r01 = A2.r00 * A1.r01 + A2.r01 * A1.r11;
  C.r10 = A2.r10 * A1.r00 + A2.r11 * A1.r10;
  C.r11 = A2.r10 * A1.r01 + A2.r11 * A1.r11;
  C.b0 = A2.r00 * A1.b0 + A2.r01 * A1.b1 + A2.b0;
  C.b1 = A2.r10 * A1.b0 + A2.r11 * A1.b1 + A2.b1;
  C.tree = A2.tree;
  return C;
}

static inline void apply(const Affine& A, int64_t X, int64_t Y, int64_t& Xo, int64_t& Yo) {
  Xo = A.r00 * X + A.r01 * Y + A.b0;
  Yo = A.r10 * X + A.r11 * Y + A.b1;
}

static int64_t find_leaf(const Plan& pl, int t, int l, int64_t x, int64_t y) {
  auto it = pl.index.find(std::make_tuple((int32_t)t, (int32_t)l, x, y));
  return it == pl.index.end() ? -1 : it->second;
}

// neighbour region of patch p in direction (di, dj)
static int dir_info(const Plan& pl, int64_t p, int di, int dj, DirInfo& D, std::string& err) {
  const Leaf& L = pl.leaves[p];
  const int64_t m2 = 2 * (int64_t)pl.m;
  const int64_t E = m2 << pl.lmax;
  const int64_t sz = 1ll << (pl.lmax - L.level);  // leaf size in level-Lmax leaves
  const int64_t S = m2 * sz;                      // in fine units
  const int64_t X0 = L.x * m2, Y0 = L.y * m2;
  const bool outx = (di < 0 && X0 == 0) || (di > 0 && X0 + S == E);
  const bool outy = (dj < 0 && Y0 == 0) || (dj > 0 && Y0 + S == E);
  const int fx = di < 0 ? 0 : 1, fy = dj < 0 ? 2 : 3;
  Affine T;
  T.tree = L.tree;
  D.leaf = -1;
  if (outx && outy) {
    Affine a1, a2, b1, b2;
    bool ok = cross_map(pl, L.tree, fx, E, a1);
    if (ok) ok = cross_map(pl, a1.tree, face_of_normal(a1.r01 * dj, a1.r11 * dj), E, a2);
    bool okb = cross_map(pl, L.tree, fy, E, b1);
    if (okb) okb = cross_map(pl, b1.tree, face_of_normal(b1.r00 * di, b1.r10 * di), E, b2);
    if (!ok || !okb) { D.kind = D_PHYS; return FC_OK; }
    Affine ta = compose(a2, a1), tb = compose(b2, b1);
    if (!(ta == tb)) { D.kind = D_CORNER3; return FC_OK; }
    T = ta;
  } else if (outx) {
    if (!cross_map(pl, L.tree, fx, E, T)) { D.kind = D_PHYS; return FC_OK; }
  } else if (outy) {
    if (!cross_map(pl, L.tree, fy, E, T)) { D.kind = D_PHYS; return FC_OK; }
  }
  D.T = T;
  // image of the same-size neighbour region
  int64_t ax, ay, bx, by;
  apply(T, X0 + di * S, Y0 + dj * S, ax, ay);
  apply(T, X0 + di * S + S, Y0 + dj * S + S, bx, by);
  const int64_t ox = std::min(ax, bx), oy = std::min(ay, by);
  if (ox % m2 || oy % m2 || ox < 0 || oy < 0 || ox + S > E || oy + S > E) {
    err = "neighbour region not aligned (connectivity inconsistent)";
    return FC_ECONN;
  }
  const int64_t qx = ox / m2, qy = oy / m2;
  int64_t id = find_leaf(pl, T.tree, L.level, qx, qy);
  if (id >= 0) { D.kind = D_SAME; D.leaf = id; return FC_OK; }
  if (L.level >= 1) {
    const int64_t ps = 2 * sz;
    id = find_leaf(pl, T.tree, L.level - 1, (qx / ps) * ps, (qy / ps) * ps);
    if (id >= 0) { D.kind = D_COARSER; D.leaf = id; return FC_OK; }
  }
  if (L.level < pl.lmax) { D.kind = D_FINER; return FC_OK; }
  err = "2:1 balance violated (coarser-by-two neighbour)";
  return FC_EBALANCE;
}

// canonical expanded records of any patch p (global id); rec[G][8]
static int patch_records(const Plan& pl, int64_t p, int32_t* rec, std::string& err) {
  const Leaf& L = pl.leaves[p];
  const int m = pl.m;
  const int64_t m2 = 2 * (int64_t)m;
  const int64_t E = m2 << pl.lmax;
  const int64_t sz = 1ll << (pl.lmax - L.level);
  const int64_t S = m2 * sz, h = sz;  // h = half a cell of p in fine units
  const int64_t X0 = L.x * m2, Y0 = L.y * m2;
  DirInfo dirs[9];
  for (int dj = -1; dj <= 1; ++dj)
    for (int di = -1; di <= 1; ++di) {
      if (!di && !dj) continue;
      int rc = dir_info(pl, p, di, dj, dirs[(dj + 1) * 3 + (di + 1)], err);
      if (rc) return rc;
    }
  int r = 0;
  for (int j = -1; j <= m + 2; ++j)
    for (int i = -1; i <= m + 2; ++i) {
      if (i >= 1 && i <= m && j >= 1 && j <= m) continue;
      int32_t* o = rec + REC * (r++);
      std::memset(o, 0, REC * sizeof(int32_t));
      const int di = i < 1 ? -1 : (i > m ? 1 : 0), dj = j < 1 ? -1 : (j > m ? 1 : 0);
      const DirInfo& D = dirs[(dj + 1) * 3 + (di + 1)];
      if (D.kind == D_PHYS) {
        const bool yphys = dj != 0 && ((dj < 0 && Y0 == 0) || (dj > 0 && Y0 + S == E)) &&
                           is_phys(pl, L.tree, dj < 0 ? 2 : 3);
        const bool xphys = di != 0 && ((di < 0 && X0 == 0) || (di > 0 && X0 + S == E)) &&
                           is_phys(pl, L.tree, di < 0 ? 0 : 1);
        if (yphys) {
          const int f = dj < 0 ? 2 : 3;
          const bool wall = pl.fbc[4 * L.tree + f] == FC_BC_WALL;
          o[0] = OP_BCY; o[1] = (int32_t)p; o[2] = i;
          o[3] = dj < 0 ? (wall ? 1 - j : 1) : (wall ? 2 * m + 1 - j : m);
          o[4] = pl.fbc[4 * L.tree + f];
        } else if (xphys) {
          const int f = di < 0 ? 0 : 1;
          const bool wall = pl.fbc[4 * L.tree + f] == FC_BC_WALL;
          o[0] = OP_BCX; o[1] = (int32_t)p; o[3] = j;
          o[2] = di < 0 ? (wall ? 1 - i : 1) : (wall ? 2 * m + 1 - i : m);
          o[4] = pl.fbc[4 * L.tree + f];
        } else {
          err = "physical corner outside a non-convex domain is not supported";
          return FC_EUNSUP;
        }
        continue;
      }
      if (D.kind == D_CORNER3) {
        o[0] = OP_CORNER3; o[1] = (int32_t)p;
        o[2] = i; o[3] = (j < 1) ? 1 - j : 2 * m + 1 - j;
        o[6] = (i < 1) ? 1 - i : 2 * m + 1 - i; o[7] = j;
        continue;
      }
      int64_t cx, cy;
      apply(D.T, X0 + (2 * i - 1) * h, Y0 + (2 * j - 1) * h, cx, cy);
      if (D.kind == D_SAME || D.kind == D_COARSER) {
        const Leaf& N = pl.leaves[D.leaf];
        const int64_t xl = cx - N.x * m2, yl = cy - N.y * m2;
        o[1] = (int32_t)D.leaf;
        if (D.kind == D_SAME) {
          o[0] = OP_COPY;
          o[2] = (int32_t)((xl / h + 1) / 2);
          o[3] = (int32_t)((yl / h + 1) / 2);
        } else {
          o[0] = OP_INTERP;
          const int64_t I = xl / (4 * h), J = yl / (4 * h);
          o[2] = (int32_t)(I + 1);
          o[3] = (int32_t)(J + 1);
          o[4] = (xl - I * 4 * h > 2 * h) ? 1 : -1;
          o[5] = (yl - J * 4 * h > 2 * h) ? 1 : -1;
        }
        if (o[2] < 1 || o[2] > m || o[3] < 1 || o[3] > m) { err = "ghost source outside leaf"; return FC_EBALANCE; }
      } else {  // FINER: the child leaf holding the 2x2 block centred on the ghost centre
        const int64_t csz = sz / 2, cw = m2 * csz;
        const int64_t kx = ((cx - 1) / cw) * csz, ky = ((cy - 1) / cw) * csz;
        const int64_t id = find_leaf(pl, D.T.tree, L.level + 1, kx, ky);
        if (id < 0) { err = "2:1 balance violated (finer-by-two neighbour)"; return FC_EBALANCE; }
        const Leaf& N = pl.leaves[id];
        o[0] = OP_AVG4; o[1] = (int32_t)id;
        o[2] = (int32_t)((cx - N.x * m2) / h);
        o[3] = (int32_t)((cy - N.y * m2) / h);
        if (o[2] < 1 || o[2] > m - 1 || o[3] < 1 || o[3] > m - 1) { err = "fine block outside leaf"; return FC_EBALANCE; }
      }
    }
  return FC_OK;
}

// COMPACT ghost table of patch p (include/fc.h, FC_TABLE_COMPACT): per direction d (faces -x, +x,
// -y, +y, then corners (-x,-y), (+x,-y), (-x,+y), (+x,+y)) {kind, nbr0, nbr1, xform, half}, from
// the same per-direction lookup the ghost records use (PAPER.md:141-144 [§2]: constant-time
// neighbour lookup with the relative orientation of the trees)
int plan_compact_patch(const Plan& pl, int64_t p, int32_t* o, std::string& err) {
  static const int DIR[8][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}, {-1, -1}, {1, -1}, {-1, 1}, {1, 1}};
  const Leaf& L = pl.leaves[p];
  const int64_t m2 = 2 * (int64_t)pl.m;
  const int64_t sz = 1ll << (pl.lmax - L.level);
  const int64_t S = m2 * sz;
  const int64_t X0 = L.x * m2, Y0 = L.y * m2;
  for (int d = 0; d < 8; ++d) {
    const int di = DIR[d][0], dj = DIR[d][1];
    DirInfo D;
    int rc = dir_info(pl, p, di, dj, D, err);
    if (rc) return rc;
    int32_t* e = o + 5 * d;
    e[0] = (int32_t)D.kind;
    e[1] = e[2] = e[3] = e[4] = -1;
    if (D.kind == D_PHYS || D.kind == D_CORNER3) continue;
    // orientation of the linear part p-frame -> neighbour frame: 4 swap + 2 [e_x reversed] + [e_y reversed]
    const Affine& T = D.T;
    if (T.r00 != 0) e[3] = 2 * (T.r00 < 0) + (T.r11 < 0);
    else e[3] = 4 + 2 * (T.r10 < 0) + (T.r01 < 0);
    if (D.kind == D_SAME || D.kind == D_COARSER) {
      e[1] = (int32_t)D.leaf;
      if (D.kind == D_COARSER && d < 4)   // which half of the coarse face, along p's tangential axis
        e[4] = (int32_t)(((d < 2 ? L.y : L.x) / sz) & 1);
      continue;
    }
    // FINER: the finer leaves touching p's face (two, lower tangential coordinate first) or corner
    const int64_t csz = sz / 2, cw = m2 * csz;
    const int64_t px = di < 0 ? X0 - 1 : (di > 0 ? X0 + S + 1 : 0);
    const int64_t py = dj < 0 ? Y0 - 1 : (dj > 0 ? Y0 + S + 1 : 0);
    const int nq = d < 4 ? 2 : 1;
    for (int q = 0; q < nq; ++q) {
      int64_t X = px, Y = py;
      if (d < 2) Y = Y0 + (2 * q + 1) * S / 4;
      else if (d < 4) X = X0 + (2 * q + 1) * S / 4;
      int64_t cx, cy;
      apply(T, X, Y, cx, cy);
      const int64_t id = find_leaf(pl, T.tree, L.level + 1, (cx / cw) * csz, (cy / cw) * csz);
      if (id < 0) { err = "2:1 balance violated (finer-by-two neighbour)"; return FC_EBALANCE; }
      e[1 + q] = (int32_t)id;
    }
  }
  return FC_OK;
}

static int64_t owner_of(const Plan& pl, int64_t q) {   // the rank whose [part[r], part[r+1]) holds q
  return (int64_t)(std::upper_bound(pl.part.begin(), pl.part.end(), q) - pl.part.begin()) - 1;
}

static inline bool is_ring(int m, int i, int j) { return !(i >= 1 && i <= m && j >= 1 && j <= m); }

int plan_build(const fc_forest_desc* d, Plan& pl, std::string& err) {
  if (!d || !d->levels || !d->tree_ids || !d->tree_to_tree || !d->tree_to_face || !d->face_bc) {
    err = "null descriptor field"; return FC_EINVAL;
  }
  if (d->num_patches <= 0 || d->num_trees <= 0) { err = "empty forest"; return FC_EINVAL; }
  if (d->m < 4 || (d->m & 1)) { err = "m must be even and >= 4"; return FC_EINVAL; }
  if (d->mbc != 2) { err = "mbc must be 2"; return FC_EINVAL; }
  if (d->meqn < 1 || d->meqn > 4 || d->maux < 0 || d->maux > 3) { err = "meqn/maux out of range"; return FC_EINVAL; }
  if (d->nranks < 1 || d->rank < 0 || d->rank >= d->nranks) { err = "bad rank/nranks"; return FC_EINVAL; }
  if (!(d->tree_dx0 > 0.0)) { err = "tree_dx0 must be positive"; return FC_EINVAL; }
  pl.P = d->num_patches; pl.T = d->num_trees; pl.m = d->m; pl.n = d->m + 4;
  pl.meqn = d->meqn; pl.maux = d->maux; pl.dx0 = d->tree_dx0 / d->m;
  pl.rank = d->rank; pl.nranks = d->nranks;
  pl.t2t.assign(d->tree_to_tree, d->tree_to_tree + 4 * pl.T);
  pl.t2f.assign(d->tree_to_face, d->tree_to_face + 4 * pl.T);
  pl.fbc.assign(d->face_bc, d->face_bc + 4 * pl.T);
  for (int t = 0; t < pl.T; ++t)
    for (int f = 0; f < 4; ++f) {
      const int nt = pl.t2t[4 * t + f], code = pl.t2f[4 * t + f];
      if (nt < 0 || nt >= pl.T || code < 0 || code > 7) { err = "connectivity out of range"; return FC_ECONN; }
      const int nf = code & 3, rev = code >> 2;
      if (pl.t2t[4 * nt + nf] != t || pl.t2f[4 * nt + nf] != f + 4 * rev || (nt == t && nf == f && rev)) {
        err = "connectivity not symmetric"; return FC_ECONN;
      }
    }
  // decode: a Morton cursor per tree, leaves aligned to their size
  int lmax = 0;
  for (int64_t p = 0; p < pl.P; ++p) {
    if (d->levels[p] < 0 || d->levels[p] > 28) { err = "level out of range"; return FC_EINVAL; }
    lmax = std::max(lmax, (int)d->levels[p]);
    if (d->tree_ids[p] < 0 || d->tree_ids[p] >= pl.T || (p && d->tree_ids[p] < d->tree_ids[p - 1])) {
      err = "tree ids must be non-decreasing and in range"; return FC_ETILING;
    }
  }
  pl.lmax = lmax;
  pl.leaves.resize(pl.P);
  pl.index.reserve((size_t)pl.P * 2);
  const uint64_t full = 1ull << (2 * lmax);
  int64_t p = 0;
  for (int t = 0; t < pl.T; ++t) {
    uint64_t c = 0;
    int64_t first = p;
    while (p < pl.P && d->tree_ids[p] == t) {
      const int l = d->levels[p];
      const uint64_t span = 1ull << (2 * (lmax - l));
      if ((c & (span - 1)) != 0 || c + span > full) { err = "leaves do not tile tree in z-order"; return FC_ETILING; }
      Leaf& L = pl.leaves[p];
      L.tree = t; L.level = l;
      L.x = (int64_t)compact_even_bits(c);
      L.y = (int64_t)compact_even_bits(c >> 1);
      pl.index.emplace(std::make_tuple((int32_t)t, (int32_t)l, L.x, L.y), p);
      c += span;
      ++p;
    }
    if (c != full || p == first) { err = "tree not covered exactly"; return FC_ETILING; }
  }
  // local range and expanded table of local patches
  pl.part.assign(pl.nranks + 1, 0);
  for (int r = 0; r <= pl.nranks; ++r)
    pl.part[r] = d->partition ? d->partition[r] : ((int64_t)r * pl.P) / pl.nranks;
  for (int r = 0; r < pl.nranks; ++r)
    if (pl.part[r] > pl.part[r + 1]) { err = "partition not non-decreasing"; return FC_EINVAL; }
  if (pl.part[0] != 0 || pl.part[pl.nranks] != pl.P) { err = "partition must cover 0..num_patches"; return FC_EINVAL; }
  pl.p0 = pl.part[pl.rank];
  pl.p1 = pl.part[pl.rank + 1];
  const int64_t Pl = pl.p1 - pl.p0, G = (int64_t)pl.n * pl.n - (int64_t)pl.m * pl.m;
  pl.table.assign((size_t)Pl * G * REC, 0);
  pl.uniform_same = true;
  pl.lmin_local = 99; pl.lmax_local = 0;
  for (int64_t q = pl.p0; q < pl.p1; ++q) {
    int rc = patch_records(pl, q, pl.table.data() + (q - pl.p0) * G * REC, err);
    if (rc) return rc;
    pl.lmin_local = std::min(pl.lmin_local, pl.leaves[q].level);
    pl.lmax_local = std::max(pl.lmax_local, pl.leaves[q].level);
  }
  for (int64_t k = 0; k < Pl * G; ++k) {
    const int op = pl.table[k * REC];
    if (op != OP_COPY && op != OP_BCX && op != OP_BCY) { pl.uniform_same = false; break; }
  }
  // halo plan: remote sources grouped by owner, round 1 (interior cells) / round 2 (ring cells)
  pl.halo = HaloPlan();
  pl.halo.need1.assign(pl.nranks, {});
  pl.halo.need2.assign(pl.nranks, {});
  if (pl.nranks > 1) {
    const int m = pl.m, n = pl.n;
    const int64_t n2 = (int64_t)n * n;
    std::unordered_map<int64_t, std::vector<int32_t>> remote_cache;
    auto need = [&](int64_t q, int i, int j) -> int {
      if (q >= pl.p0 && q < pl.p1) return FC_OK;
      const int64_t key = q * n2 + (int64_t)(j + 1) * n + (i + 1);
      const int64_t own = owner_of(pl, q);
      if (!is_ring(m, i, j)) { pl.halo.need1[own].push_back(key); return FC_OK; }
      // a remote ring cell read by interpolation: must be final after the owner's phases A + C
      auto it = remote_cache.find(q);
      if (it == remote_cache.end()) {
        std::vector<int32_t> rr((size_t)G * REC);
        int rc = patch_records(pl, q, rr.data(), err);
        if (rc) return rc;
        it = remote_cache.emplace(q, std::move(rr)).first;
      }
      const int32_t* o = it->second.data() + (size_t)ring_index(i, j, m) * REC;
      bool ok = o[0] == OP_COPY || o[0] == OP_AVG4;
      if (o[0] == OP_BCX || o[0] == OP_BCY) ok = !is_ring(m, o[2], o[3]);
      if (!ok) { err = "multi-level interpolation chain across a shard cut"; return FC_EUNSUP; }
      pl.halo.need2[own].push_back(key);
      // the cell's own sources (interior cells) in round 1 as well: the fused AMR gather computes
      // this ghost itself from them (plan_ring_amr) and needs no second round
      auto need1 = [&](int64_t s, int si, int sj) {
        if (s >= pl.p0 && s < pl.p1) return;
        pl.halo.need1[owner_of(pl, s)].push_back(s * n2 + (int64_t)(sj + 1) * n + (si + 1));
      };
      if (o[0] == OP_COPY) need1(o[1], o[2], o[3]);
      else if (o[0] == OP_AVG4) {
        for (int b = 0; b < 2; ++b)
          for (int a = 0; a < 2; ++a) need1(o[1], o[2] + a, o[3] + b);
      } else {
        need1(q, o[2], o[3]);
      }
      return FC_OK;
    };
    for (int64_t k = 0; k < Pl * G; ++k) {
      const int32_t* o = pl.table.data() + k * REC;
      int rc = FC_OK;
      switch (o[0]) {
        case OP_COPY: rc = need(o[1], o[2], o[3]); break;
        case OP_AVG4:
          for (int b = 0; b < 2 && !rc; ++b)
            for (int a = 0; a < 2 && !rc; ++a) rc = need(o[1], o[2] + a, o[3] + b);
          break;
        case OP_INTERP:
          rc = need(o[1], o[2], o[3]);
          if (!rc) rc = need(o[1], o[2] - 1, o[3]);
          if (!rc) rc = need(o[1], o[2] + 1, o[3]);
          if (!rc) rc = need(o[1], o[2], o[3] - 1);
          if (!rc) rc = need(o[1], o[2], o[3] + 1);
          break;
        default: break;
      }
      if (rc) return rc;
    }
    int64_t slot = 0;
    for (int round = 1; round <= 2; ++round)
      for (int r = 0; r < pl.nranks; ++r) {
        auto& v = round == 1 ? pl.halo.need1[r] : pl.halo.need2[r];
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        for (int64_t key : v) pl.halo.slot.emplace(key * 2 + (round - 1), slot++);
        (round == 1 ? pl.halo.n1 : pl.halo.n2) += (int64_t)v.size();
      }
  }
  return FC_OK;
}

int plan_lists(const Plan& pl, int meqn, GhostLists& gl, std::string& err, const std::vector<uint8_t>* dst_mask) {
  const int m = pl.m, n = pl.n;
  const int64_t n2 = (int64_t)n * n, S = (int64_t)meqn * n2;
  const int64_t Pl = pl.p1 - pl.p0, G = n2 - (int64_t)m * m;
  const int64_t nhalo = pl.halo.n1 + pl.halo.n2;
  const int64_t total = (Pl + (nhalo + n2 - 1) / n2) * S;
  if (total >= (1ll << 31)) { err = "state too large for 32-bit offsets"; return FC_EUNSUP; }
  gl = GhostLists();
  gl.interp.assign(pl.lmax + 1, {});
  gl.bcx_l.assign(pl.lmax + 1, {});
  gl.bcy_l.assign(pl.lmax + 1, {});
  bool any_interp = false;
  auto off = [&](int64_t q, int i, int j, int round) -> int32_t {
    const int64_t cell = (int64_t)(j + 1) * n + (i + 1);   // natural index: halo keys
    if (q >= pl.p0 && q < pl.p1) return (int32_t)((q - pl.p0) * S + qcell(i, j, n));
    const int64_t key = (q * n2 + cell) * 2 + (round - 1);
    auto it = pl.halo.slot.find(key);
    if (it == pl.halo.slot.end()) return -1;
    const int64_t h = it->second;
    return (int32_t)((Pl + h / n2) * S + h % n2);
  };
  for (int64_t lp = 0; lp < Pl; ++lp) {
    if (dst_mask && !(*dst_mask)[lp]) continue;   // (sub-cycling: only the rings a level fill needs)
    const int lvl = pl.leaves[pl.p0 + lp].level;
    int r = 0;
    for (int j = -1; j <= m + 2; ++j)
      for (int i = -1; i <= m + 2; ++i) {
        if (!is_ring(m, i, j)) continue;
        const int32_t* o = pl.table.data() + (lp * G + r++) * REC;
        const int32_t dst = (int32_t)(lp * S + qcell(i, j, n));
        switch (o[0]) {
          case OP_COPY: {
            int32_t s = off(o[1], o[2], o[3], 1);
            if (s < 0) { err = "missing halo slot"; return FC_EINVAL; }
            gl.copy.insert(gl.copy.end(), {dst, s});
            break;
          }
          case OP_AVG4: {
            int32_t s[4] = {off(o[1], o[2], o[3], 1), off(o[1], o[2] + 1, o[3], 1),
                            off(o[1], o[2], o[3] + 1, 1), off(o[1], o[2] + 1, o[3] + 1, 1)};
            if (s[0] < 0 || s[1] < 0 || s[2] < 0 || s[3] < 0) { err = "missing halo slot"; return FC_EINVAL; }
            gl.avg.insert(gl.avg.end(), {dst, s[0], s[1], s[2], s[3]});
            break;
          }
          case OP_INTERP: {
            auto rnd = [&](int ii, int jj) { return is_ring(m, ii, jj) ? 2 : 1; };
            const int I = o[2], J = o[3];
            int32_t s[5] = {off(o[1], I, J, rnd(I, J)), off(o[1], I - 1, J, rnd(I - 1, J)),
                            off(o[1], I + 1, J, rnd(I + 1, J)), off(o[1], I, J - 1, rnd(I, J - 1)),
                            off(o[1], I, J + 1, rnd(I, J + 1))};
            for (int k = 0; k < 5; ++k)
              if (s[k] < 0) { err = "missing halo slot"; return FC_EINVAL; }
            gl.interp[lvl].insert(gl.interp[lvl].end(), {dst, s[0], s[1], s[2], s[3], s[4], o[4], o[5]});
            any_interp = true;
            break;
          }
          case OP_BCX:
          case OP_BCY: {
            const int32_t s = (int32_t)(lp * S + qcell(o[2], o[3], n));
            const int32_t neg = (o[4] == FC_BC_WALL && meqn >= 3) ? (o[0] == OP_BCX ? 1 : 2) : -1;
            auto& v = o[0] == OP_BCX ? gl.bcx : gl.bcy;
            v.insert(v.end(), {dst, s, neg});
            auto& vl = o[0] == OP_BCX ? gl.bcx_l[lvl] : gl.bcy_l[lvl];
            vl.insert(vl.end(), {dst, s, neg});
            break;
          }
          case OP_CORNER3: {
            const int32_t a = (int32_t)(lp * S + qcell(o[2], o[3], n));
            const int32_t b = (int32_t)(lp * S + qcell(o[6], o[7], n));
            gl.corner3.insert(gl.corner3.end(), {dst, a, b});
            break;
          }
          default:
            err = "unexpected ghost op";
            return FC_EINVAL;
        }
      }
  }
  if (!any_interp) {  // no per-level B/C passes needed
    for (auto& v : gl.bcx_l) v.clear();
    for (auto& v : gl.bcy_l) v.clear();
  }
  return FC_OK;
}

int plan_activity(const Plan& pl, int meqn, std::vector<int32_t>& nbr, std::vector<uint8_t>& negmask,
                  std::string& err) {
  const int64_t n2 = (int64_t)pl.n * pl.n, G = n2 - (int64_t)pl.m * pl.m;
  const int64_t Pl = pl.p1 - pl.p0;
  nbr.assign((size_t)Pl * 8, -1);
  negmask.assign((size_t)Pl, 0);
  for (int64_t lp = 0; lp < Pl; ++lp) {
    int nn = 0;
    bool always = false;
    for (int64_t r = 0; r < G && !always; ++r) {
      const int32_t* o = pl.table.data() + (lp * G + r) * REC;
      if (o[0] == OP_COPY) {
        const int64_t q = o[1];
        const int32_t id = (q >= pl.p0 && q < pl.p1) ? (int32_t)(q - pl.p0) : -2;
        bool found = false;
        for (int k = 0; k < nn; ++k) found |= nbr[lp * 8 + k] == id;
        if (!found) {
          if (nn >= 8 || id == -2) { always = true; break; }
          nbr[lp * 8 + nn++] = id;
        }
      } else if (o[0] == OP_BCX || o[0] == OP_BCY) {
        if (o[4] == FC_BC_WALL && meqn >= 3) negmask[lp] |= (uint8_t)(1u << (o[0] == OP_BCY ? 2 : 1));
      } else {
        always = true;   // averaged / interpolated / corner ghosts: not tested, always updated
      }
    }
    if (always) {
      for (int k = 0; k < 8; ++k) nbr[lp * 8 + k] = -1;
      nbr[lp * 8] = -2;
    }
  }
  (void)err;
  return FC_OK;
}

int plan_ring_sources(const Plan& pl, int meqn, RingSources& rs, std::string& err, bool p2p) {
  const int m = pl.m, n = pl.n;
  const int64_t n2 = (int64_t)n * n, S = (int64_t)meqn * n2;
  const int64_t Pl = pl.p1 - pl.p0, G = n2 - (int64_t)m * m;
  rs.src.assign((size_t)Pl * G, 0);
  rs.bcflag.assign((size_t)Pl, 0);
  rs.nbr.assign((size_t)Pl * 8, -1);
  rs.negmask.assign((size_t)Pl, 0);
  if (p2p) {
    if (pl.nranks > 255) { err = "peer-memory halo supports at most 255 ranks"; return FC_EUNSUP; }
    rs.peer.assign((size_t)Pl * G, 0);
  }
  for (int64_t lp = 0; lp < Pl; ++lp) {
    int nn = 0;
    auto add_nbr = [&](int32_t id) {
      for (int k = 0; k < nn; ++k)
        if (rs.nbr[lp * 8 + k] == id) return true;
      if (nn >= 8) return false;
      rs.nbr[lp * 8 + nn++] = id;
      return true;
    };
    for (int64_t r = 0; r < G; ++r) {
      const int32_t* o = pl.table.data() + (lp * G + r) * REC;
      int32_t v;
      if (o[0] == OP_COPY) {
        const int64_t cell = (int64_t)(o[3] + 1) * n + (o[2] + 1);   // natural: halo key
        const int64_t q = o[1];
        if (!add_nbr((q >= pl.p0 && q < pl.p1) ? (int32_t)(q - pl.p0) : -2)) { err = "more than 8 ring neighbours"; return FC_EUNSUP; }
        if (q >= pl.p0 && q < pl.p1) {
          v = (int32_t)((q - pl.p0) * S + qcell(o[2], o[3], n));
        } else if (p2p) {   // the owner's own state: its local patch index, same block layout
          const int64_t ow = owner_of(pl, q), first = pl.part[ow];
          v = (int32_t)((q - first) * S + qcell(o[2], o[3], n));
          rs.peer[lp * G + r] = (uint8_t)(ow + 1);
        } else {
          auto it = pl.halo.slot.find((q * n2 + cell) * 2);
          if (it == pl.halo.slot.end()) { err = "missing halo slot"; return FC_EINVAL; }
          const int64_t h = it->second;
          v = (int32_t)((Pl + h / n2) * S + h % n2);
        }
      } else if (o[0] == OP_BCX || o[0] == OP_BCY) {
        const int win = (o[3] + 1) * n + (o[2] + 1);
        const int isy = o[0] == OP_BCY;
        const int neg = (o[4] == FC_BC_WALL && meqn >= 3) ? (isy ? 2 : 1) : 0;
        v = -1 - ((win << 3) | (neg << 1) | isy);
        rs.bcflag[lp] |= (uint8_t)(isy ? 2 : 1);
        if (neg) rs.negmask[lp] |= (uint8_t)(1u << neg);
      } else {
        err = "ring gather needs COPY/BC records only";
        return FC_EUNSUP;
      }
      rs.src[lp * G + r] = v;
    }
  }
  return FC_OK;
}

int64_t plan_ring_regular(const Plan& pl, int meqn, const RingSources& rs, std::vector<int32_t>& nb9) {
  const int m = pl.m, n = pl.n;
  const int64_t S = (int64_t)meqn * n * n, Pl = pl.p1 - pl.p0, G = (int64_t)n * n - (int64_t)m * m;
  nb9.assign((size_t)std::max<int64_t>(1, Pl) * 9, -1);
  int64_t count = 0;
  for (int64_t lp = 0; lp < Pl; ++lp) {
    const int32_t* src = rs.src.data() + lp * G;
    const uint8_t* peer = rs.peer.empty() ? nullptr : rs.peer.data() + lp * G;
    if (!rs.bcflag.empty() && rs.bcflag[lp]) continue;
    int64_t off[9];
    bool ok = true;
    for (int d = 0; d < 9 && ok; ++d) {   // the neighbour from one representative ring cell
      const int dx = d % 3 - 1, dy = d / 3 - 1;
      if (d == 4) { off[d] = lp * S; continue; }
      const int i = dx < 0 ? 0 : (dx > 0 ? m + 1 : 1), j = dy < 0 ? 0 : (dy > 0 ? m + 1 : 1);
      const int32_t v = src[ring_index(i, j, m)];
      if (v < 0) { ok = false; break; }
      off[d] = v - (v % S);
      if (off[d] / S >= Pl) ok = false;   // (a halo slot, not a local patch)
    }
    for (int j = -1; j <= m + 2 && ok; ++j)
      for (int i = -1; i <= m + 2 && ok; ++i) {
        if (i >= 1 && i <= m && j >= 1 && j <= m) continue;
        const int dx = i < 1 ? -1 : (i > m ? 1 : 0), dy = j < 1 ? -1 : (j > m ? 1 : 0);
        const int r = ring_index(i, j, m);
        const int64_t want = off[3 * (dy + 1) + dx + 1] + (int64_t)(j - dy * m - 1) * m + (i - dx * m - 1);
        if (src[r] != want || (peer && peer[r] != 0)) ok = false;
      }
    if (!ok) continue;
    for (int d = 0; d < 9; ++d) nb9[lp * 9 + d] = (int32_t)off[d];
    ++count;
  }
  return count;
}

// Fused two-hop ring gather for AMR forests (one rank, one tile per patch).  The
// rings are never written: COPY ring cells are gathered by the step kernel straight from their
// source cells; AVG4 and INTERP ring cells get a slot in a "computed ghost" buffer (virtual patches
// of n^2 cells, the same component stride as the state) that two small kernels fill first -- the
// averages from the fine interiors, then per level (ascending) the interpolations, whose slope
// stencil reads the coarse patch's interior or, one hop further, the source of the coarse patch's
// ring cell (a COPY source cell, or another computed slot).  Every value is the one the ghost
// kernels would have written into the ring, with the same arithmetic.  Slope stencils that reach a
// physical-boundary ring cell are not supported (FC_EUNSUP: the caller keeps the ghost kernels);
// CORNER3 cells (cube corners) are computed last from the refs of their two face ghosts.  Source references in the lists: >= 0 an offset in q_old, < 0 the
// computed slot offset -1 - v.  In rs.src the computed cells have peer code 255.
int plan_ring_amr(const Plan& pl, int meqn, RingSources& rs, RingAmr& ra, std::string& err) {
  const int m = pl.m, n = pl.n;
  const int64_t n2 = (int64_t)n * n, S = (int64_t)meqn * n2;
  const int64_t Pl = pl.p1 - pl.p0, G = n2 - (int64_t)m * m;
  // several ranks: every remote cell a computed or copied ghost reads is an interior cell of its
  // owner, brought into a round-1 halo slot (plan_build adds the one-hop sources of the remote
  // ring cells that interpolation slopes read), so the gather needs one exchange round only
  rs.src.assign((size_t)Pl * G, 0);
  rs.peer.assign((size_t)Pl * G, 0);
  rs.bcflag.assign((size_t)Pl, 0);
  rs.nbr.clear();
  rs.negmask.clear();
  ra = RingAmr();
  ra.interp.assign(pl.lmax + 1, {});
  std::vector<int64_t> slot((size_t)Pl * G, -1);
  int64_t ncg = 0;
  for (int64_t i = 0; i < Pl * G; ++i) {
    const int op = pl.table[i * REC];
    if (op == OP_AVG4 || op == OP_INTERP || op == OP_CORNER3) slot[i] = ncg++;
  }
  // remote coarse patches' ring cells that slopes read and that are averages: a computed slot
  // each, after the local ones (keyed by remote patch * G + ring index)
  std::map<int64_t, int64_t> rslot;
  std::unordered_map<int64_t, std::vector<int32_t>> rrec;   // records of remote patches
  auto remote_records = [&](int64_t q) -> const int32_t* {
    auto it = rrec.find(q);
    if (it == rrec.end()) {
      std::vector<int32_t> rr((size_t)G * REC);
      if (patch_records(pl, q, rr.data(), err)) return nullptr;
      it = rrec.emplace(q, std::move(rr)).first;
    }
    return it->second.data();
  };
  const int64_t nhalo = pl.halo.n1 + pl.halo.n2, Pv = (nhalo + n2 - 1) / n2;
  if (pl.nranks > 1) {   // count the remote average slots first (the buffer size)
    for (int64_t i = 0; i < Pl * G; ++i) {
      const int32_t* o = pl.table.data() + i * REC;
      if (o[0] != OP_INTERP || (o[1] >= pl.p0 && o[1] < pl.p1)) continue;
      const int dI[4] = {-1, 1, 0, 0}, dJ[4] = {0, 0, -1, 1};
      for (int d = 0; d < 4; ++d) {
        const int I = o[2] + dI[d], J = o[3] + dJ[d];
        if (I >= 1 && I <= m && J >= 1 && J <= m) continue;
        const int32_t* rr = remote_records(o[1]);
        if (!rr) return FC_EINVAL;
        if (rr[(size_t)ring_index(I, J, m) * REC] == OP_AVG4) rslot.emplace(o[1] * G + ring_index(I, J, m), 0);
      }
    }
    for (auto& kv : rslot) kv.second = ncg++;
  }
  ra.ncg_patches = (ncg + n2 - 1) / n2;
  if ((Pl + Pv + ra.ncg_patches) * S >= (1ll << 31)) { err = "AMR ring gather: state too large"; return FC_EUNSUP; }
  auto cgoff = [&](int64_t g) { return (int32_t)((g / n2) * S + g % n2); };
  bool missing = false;
  auto interior = [&](int64_t q, int i, int j) -> int32_t {   // q global, (i, j) interior
    if (q >= pl.p0 && q < pl.p1) return (int32_t)((q - pl.p0) * S + qcell(i, j, n));
    auto it = pl.halo.slot.find((q * n2 + (int64_t)(j + 1) * n + (i + 1)) * 2);   // round-1 slot
    if (it == pl.halo.slot.end()) { missing = true; return 0; }
    return (int32_t)((Pl + it->second / n2) * S + it->second % n2);
  };
  // a cell (I, J) of patch q (interior or ring; local or remote) as a source reference
  auto ref = [&](int64_t q, int I, int J, int32_t& v) -> bool {
    if (I >= 1 && I <= m && J >= 1 && J <= m) { v = interior(q, I, J); return true; }
    const bool local = q >= pl.p0 && q < pl.p1;
    const int64_t i = local ? (q - pl.p0) * G + ring_index(I, J, m) : -1;
    const int32_t* o = local ? pl.table.data() + i * REC : remote_records(q) + (size_t)ring_index(I, J, m) * REC;
    if (o[0] == OP_COPY) {
      if (o[2] < 1 || o[2] > m || o[3] < 1 || o[3] > m) return false;
      v = interior(o[1], o[2], o[3]);
      return true;
    }
    if (local && (o[0] == OP_AVG4 || o[0] == OP_INTERP)) { v = -1 - cgoff(slot[i]); return true; }
    if (!local && o[0] == OP_AVG4) { v = -1 - cgoff(rslot.at(q * G + ring_index(I, J, m))); return true; }
    return false;   // a physical-boundary (or corner) ring cell, or a remote interpolation chain
  };
  for (auto& kv : rslot) {   // the remote averages: their fine sources are interiors (local or halo)
    const int64_t q = kv.first / G;
    const int32_t* o = remote_records(q) + (size_t)(kv.first % G) * REC;
    const int I = o[2], J = o[3];
    ra.avg.insert(ra.avg.end(), {cgoff(kv.second), interior(o[1], I, J), interior(o[1], I + 1, J),
                                 interior(o[1], I, J + 1), interior(o[1], I + 1, J + 1)});
  }
  for (int64_t lp = 0; lp < Pl; ++lp) {
    const int lvl = pl.leaves[pl.p0 + lp].level;
    for (int64_t r = 0; r < G; ++r) {
      const int64_t i = lp * G + r;
      const int32_t* o = pl.table.data() + i * REC;
      int32_t v = 0;
      switch (o[0]) {
        case OP_COPY:
          if (o[2] < 1 || o[2] > m || o[3] < 1 || o[3] > m) { err = "AMR ring gather: copy from a ghost"; return FC_EUNSUP; }
          v = interior(o[1], o[2], o[3]);
          break;
        case OP_BCX:
        case OP_BCY: {
          const int win = (o[3] + 1) * n + (o[2] + 1);
          const int isy = o[0] == OP_BCY;
          const int neg = (o[4] == FC_BC_WALL && meqn >= 3) ? (isy ? 2 : 1) : 0;
          v = -1 - ((win << 3) | (neg << 1) | isy);
          rs.bcflag[lp] |= (uint8_t)(isy ? 2 : 1);
          break;
        }
        case OP_AVG4: {
          const int I = o[2], J = o[3];
          if (I < 1 || I + 1 > m || J < 1 || J + 1 > m) { err = "AMR ring gather: average outside the interior"; return FC_EUNSUP; }
          v = cgoff(slot[i]);
          rs.peer[i] = 255;
          ra.avg.insert(ra.avg.end(), {v, interior(o[1], I, J), interior(o[1], I + 1, J), interior(o[1], I, J + 1),
                                       interior(o[1], I + 1, J + 1)});
          break;
        }
        case OP_INTERP: {
          const int I = o[2], J = o[3];
          int32_t c[5];
          if (!ref(o[1], I, J, c[0]) || !ref(o[1], I - 1, J, c[1]) || !ref(o[1], I + 1, J, c[2]) ||
              !ref(o[1], I, J - 1, c[3]) || !ref(o[1], I, J + 1, c[4])) {
            err = "AMR ring gather: interpolation slope reads a boundary ghost";
            return FC_EUNSUP;
          }
          v = cgoff(slot[i]);
          rs.peer[i] = 255;
          ra.interp[lvl].insert(ra.interp[lvl].end(), {v, c[0], c[1], c[2], c[3], c[4], o[4], o[5]});
          break;
        }
        case OP_CORNER3: {   // (3-tree cube corners) the mean of two of the patch's own face ghosts
          int32_t a, b;
          if (!ref(pl.p0 + lp, o[2], o[3], a) || !ref(pl.p0 + lp, o[6], o[7], b)) {
            err = "AMR ring gather: corner ghost reads a boundary ghost";
            return FC_EUNSUP;
          }
          v = cgoff(slot[i]);
          rs.peer[i] = 255;
          ra.corner3.insert(ra.corner3.end(), {v, a, b});
          break;
        }
        default:
          err = "AMR ring gather: unexpected ghost op";
          return FC_EUNSUP;
      }
      rs.src[i] = v;
    }
  }
  if (missing) { err = "AMR ring gather: a remote source without a halo slot"; return FC_EINVAL; }
  return FC_OK;
}

}  // namespace fc

namespace fc {

// Reflux pairing.  For every local patch p and face direction whose neighbour is
// FINER: each coarse edge c of the face is covered by two fine edges, at tangential positions
// c + 1/4 and c + 3/4 of a coarse cell.  The fine cells at depth 1 and 2 behind those positions are
// located through the face transform of dir_info; their difference is the inward normal of the
// fine patch's face, which gives the fine face and edge index in the fine patch's own frame.
int plan_reflux(const Plan& pl, int meqn, RefluxPlan& rf, std::string& err) {
  const int m = pl.m, n = pl.n;
  const int64_t m2 = 2 * (int64_t)m, n2 = (int64_t)n * n, S = (int64_t)meqn * n2;
  const int64_t Pl = pl.p1 - pl.p0;
  static const int FD[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};
  rf.slot.assign((size_t)Pl, -1);
  rf.nslots = 0;
  rf.cells.clear();
  rf.req.assign(pl.nranks, {});
  rf.nremote = 0;
  std::vector<std::map<int64_t, int64_t>> rmap(pl.nranks);   // per owner: key -> index in its list
  struct Fix { int64_t cell; int pos; int owner; int64_t key; int fe; };
  std::vector<Fix> fixes;                                     // remote references, resolved at the end
  // slots: every local patch with a coarser or finer face neighbour
  std::vector<std::array<DirKind, 4>> kinds((size_t)Pl);
  std::vector<std::array<DirInfo, 4>> dirs((size_t)Pl);
  for (int64_t lp = 0; lp < Pl; ++lp) {
    bool cf = false;
    for (int s = 0; s < 4; ++s) {
      int rc = dir_info(pl, pl.p0 + lp, FD[s][0], FD[s][1], dirs[lp][s], err);
      if (rc) return rc;
      kinds[lp][s] = dirs[lp][s].kind;
      cf |= kinds[lp][s] == D_FINER || kinds[lp][s] == D_COARSER;
    }
    if (cf) rf.slot[lp] = rf.nslots++;
  }
  auto RO = [&](int32_t slot, int face, int e) { return (int32_t)((((int64_t)slot * 4 + face) * m + e) * meqn); };
  std::map<int64_t, std::vector<int32_t>> cells;   // coarse cell (lp, i, j) -> face triples
  for (int64_t lp = 0; lp < Pl; ++lp) {
    const int64_t p = pl.p0 + lp;
    const Leaf& L = pl.leaves[p];
    const int64_t sz = 1ll << (pl.lmax - L.level), h = sz, hh = h / 2;   // half a coarse / fine cell
    const int64_t X0 = L.x * m2, Y0 = L.y * m2, W = m2 * sz;
    for (int s = 0; s < 4; ++s) {
      if (kinds[lp][s] != D_FINER) continue;
      const DirInfo& D = dirs[lp][s];
      if (meqn > 1 && !(D.T.r00 == 1 && D.T.r11 == 1 && D.T.r01 == 0 && D.T.r10 == 0)) {
        err = "reflux of a system across a rotated tree link is not supported";
        return FC_EUNSUP;
      }
      for (int c = 0; c < m; ++c) {
        int32_t ro[2];
        for (int hf = 0; hf < 2; ++hf) {
          const int64_t tau = 2 * h * c + (hf ? 3 * hh : hh);
          int64_t leaf[2];
          int ic[2], jc[2];
          for (int d = 0; d < 2; ++d) {
            const int64_t dep = d ? 3 * hh : hh;
            int64_t X, Y;
            switch (s) {
              case 0: X = X0 - dep; Y = Y0 + tau; break;
              case 1: X = X0 + W + dep; Y = Y0 + tau; break;
              case 2: X = X0 + tau; Y = Y0 - dep; break;
              default: X = X0 + tau; Y = Y0 + W + dep; break;
            }
            int64_t cx, cy;
            apply(D.T, X, Y, cx, cy);
            const int64_t csz = sz / 2, cw = m2 * csz;
            const int64_t id = find_leaf(pl, D.T.tree, L.level + 1, (cx / cw) * csz, (cy / cw) * csz);
            if (id < 0) { err = "reflux: fine neighbour not found"; return FC_EBALANCE; }
            const Leaf& N = pl.leaves[id];
            leaf[d] = id;
            ic[d] = (int)(((cx - N.x * m2) / hh + 1) / 2);
            jc[d] = (int)(((cy - N.y * m2) / hh + 1) / 2);
          }
          if (leaf[0] != leaf[1]) { err = "reflux: fine edge pair split"; return FC_EBALANCE; }
          const int di = ic[1] - ic[0], dj = jc[1] - jc[0];
          int ff, fe;
          if (di == 1 && dj == 0 && ic[0] == 1) { ff = 0; fe = jc[0] - 1; }
          else if (di == -1 && dj == 0 && ic[0] == m) { ff = 1; fe = jc[0] - 1; }
          else if (di == 0 && dj == 1 && jc[0] == 1) { ff = 2; fe = ic[0] - 1; }
          else if (di == 0 && dj == -1 && jc[0] == m) { ff = 3; fe = ic[0] - 1; }
          else { err = "reflux: fine face not found"; return FC_EBALANCE; }
          const int64_t q = leaf[0];
          if (q < pl.p0 || q >= pl.p1) {   // the fine face is another rank's: requested from it
            const int ow = (int)owner_of(pl, q);
            const int64_t key = q * 4 + ff;
            auto it = rmap[ow].find(key);
            if (it == rmap[ow].end()) it = rmap[ow].emplace(key, (int64_t)rmap[ow].size()).first;
            ro[hf] = -1 - (int32_t)fixes.size();
            fixes.push_back({0, 0, ow, key, fe});
            continue;
          }
          const int32_t fs = rf.slot[q - pl.p0];
          if (fs < 0) { err = "reflux: fine patch without a flux slot"; return FC_EINVAL; }
          ro[hf] = RO(fs, ff, fe);
        }
        const int ci = s == 0 ? 1 : (s == 1 ? m : c + 1), cj = s < 2 ? c + 1 : (s == 2 ? 1 : m);
        const int64_t ck = (lp * (m + 2) + cj) * (m + 2) + ci;
        auto& v = cells[ck];
        v.push_back(RO(rf.slot[lp], s, c));
        for (int hf = 0; hf < 2; ++hf) {
          if (ro[hf] < 0) { fixes[-1 - ro[hf]].cell = ck; fixes[-1 - ro[hf]].pos = (int)v.size(); }
          v.push_back(ro[hf]);
        }
      }
    }
  }
  // remote faces: owner-major, each owner's keys in first-reference order
  {
    std::vector<int64_t> base(pl.nranks + 1, 0);
    for (int o = 0; o < pl.nranks; ++o) {
      rf.req[o].assign(rmap[o].size(), 0);
      for (auto& kv : rmap[o]) rf.req[o][kv.second] = kv.first;
      base[o + 1] = base[o] + (int64_t)rmap[o].size();
    }
    rf.nremote = base[pl.nranks];
    if ((4 * (int64_t)rf.nslots + rf.nremote) * m * meqn >= (1ll << 31)) { err = "reflux: too many flux records"; return FC_EUNSUP; }
    for (const Fix& x : fixes) {
      const int64_t r = base[x.owner] + rmap[x.owner].at(x.key);
      cells[x.cell][x.pos] = (int32_t)(((4 * (int64_t)rf.nslots + r) * m + x.fe) * meqn);
    }
  }
  for (auto& kv : cells) {
    const int64_t key = kv.first;
    const int ci = (int)(key % (m + 2)), cj = (int)((key / (m + 2)) % (m + 2));
    const int64_t lp = key / ((int64_t)(m + 2) * (m + 2));
    const int nf = (int)kv.second.size() / 3;
    if (nf < 1 || nf > 2) { err = "reflux: bad face count"; return FC_EINVAL; }
    int32_t r[RFX] = {(int32_t)(lp * S + qcell(ci, cj, n)),
                      pl.maux ? (int32_t)(lp * pl.maux * n2 + (int64_t)(cj + 1) * n + (ci + 1)) : -1,
                      (int32_t)lp, nf, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < 3 * nf; ++k) r[4 + k] = kv.second[k];
    rf.cells.insert(rf.cells.end(), r, r + RFX);
  }
  return FC_OK;
}

}  // namespace fc

namespace fc {

// ---- dynamic regrid ----------------------------
// Leaf containing a point (fine units, possibly outside its tree: crossed through the face maps,
// both orders at a corner).  Up to 2 leaves (3-tree corners); -1 entries otherwise.
static int leaves_at(const Plan& pl, int t, int64_t X, int64_t Y, int64_t out[2]) {
  const int64_t m2 = 2 * (int64_t)pl.m, E = m2 << pl.lmax;
  int cnt = 0;
  for (int first = 0; first < 2; ++first) {
    int tt = t;
    int64_t x = X, y = Y;
    bool phys = false;
    for (int pass = 0; pass < 2 && !phys; ++pass) {
      const int axis = pass == 0 ? first : 1 - first;
      const int face = axis == 0 ? (x < 0 ? 0 : (x >= E ? 1 : -1)) : (y < 0 ? 2 : (y >= E ? 3 : -1));
      if (face < 0) continue;
      Affine A;
      if (!cross_map(pl, tt, face, E, A)) { phys = true; break; }
      int64_t nx, ny;
      apply(A, x, y, nx, ny);
      x = nx; y = ny; tt = A.tree;
    }
    if (phys || x < 0 || y < 0 || x >= E || y >= E) continue;
    int64_t id = -1;
    for (int l = pl.lmax; l >= 0 && id < 0; --l) {
      const int64_t sz = 1ll << (pl.lmax - l);
      id = find_leaf(pl, tt, l, (x / m2) / sz * sz, (y / m2) / sz * sz);
    }
    if (id >= 0 && !(cnt == 1 && out[0] == id)) out[cnt++] = id;
  }
  return cnt;
}

int plan_regrid(const Plan& pl, const double* tag, double refine_threshold, double coarsen_threshold,
                int min_level, int max_level, std::vector<int8_t>& new_levels, std::vector<int32_t>& new_trees,
                std::vector<int32_t>& src, std::string& err) {
  // (the plan is global: every rank runs it on the same leaves and the gathered tags)
  if (max_level > 28 || min_level < 0) { err = "regrid levels out of range"; return FC_EINVAL; }
  const int64_t P = pl.P, m2 = 2 * (int64_t)pl.m;
  std::vector<uint8_t> refine((size_t)P, 0), coarsen((size_t)P, 0);
  for (int64_t p = 0; p < P; ++p) refine[p] = tag[p] > refine_threshold && pl.leaves[p].level < max_level;
  auto newlev = [&](int64_t q) { return pl.leaves[q].level + refine[q]; };
  // refinement until 2:1 balanced: a leaf going to l+1 lifts face / corner neighbours at <= l-1
  for (bool changed = true; changed;) {
    changed = false;
    for (int64_t p = 0; p < P; ++p) {
      if (!refine[p]) continue;
      const Leaf& L = pl.leaves[p];
      const int64_t S = m2 << (pl.lmax - L.level), X0 = L.x * m2, Y0 = L.y * m2;
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          if (!di && !dj) continue;
          const int64_t X = di < 0 ? X0 - 1 : (di > 0 ? X0 + S : X0 + S / 2);
          const int64_t Y = dj < 0 ? Y0 - 1 : (dj > 0 ? Y0 + S : Y0 + S / 2);
          int64_t q[2];
          const int c = leaves_at(pl, L.tree, X, Y, q);
          for (int k = 0; k < c; ++k)
            if (newlev(q[k]) <= L.level - 1) { refine[q[k]] = 1; changed = true; }
        }
    }
  }
  // coarsening of complete families whose outside neighbours all stay at <= l
  for (int64_t p = 0; p + 3 < P; ++p) {
    const Leaf& L = pl.leaves[p];
    if (L.level <= min_level || L.level == 0) continue;
    const int64_t sz = 1ll << (pl.lmax - L.level);
    if ((L.x / sz) % 2 || (L.y / sz) % 2) continue;
    bool ok = true;
    for (int k = 0; k < 4 && ok; ++k) {
      const Leaf& c = pl.leaves[p + k];
      ok = c.tree == L.tree && c.level == L.level && c.x == L.x + (k & 1) * sz && c.y == L.y + (k >> 1) * sz &&
           !refine[p + k] && tag[p + k] < coarsen_threshold;
    }
    for (int k = 0; k < 4 && ok; ++k) {
      const Leaf& c = pl.leaves[p + k];
      const int64_t S = m2 * sz, X0 = c.x * m2, Y0 = c.y * m2;
      for (int dj = -1; dj <= 1 && ok; ++dj)
        for (int di = -1; di <= 1 && ok; ++di) {
          if (!di && !dj) continue;
          for (int h = 0; h < ((di && dj) ? 1 : 2) && ok; ++h) {
            const int64_t along = h ? 3 * S / 4 : S / 4;
            const int64_t X = di < 0 ? X0 - 1 : (di > 0 ? X0 + S : X0 + along);
            const int64_t Y = dj < 0 ? Y0 - 1 : (dj > 0 ? Y0 + S : Y0 + along);
            int64_t q[2];
            const int cnt = leaves_at(pl, L.tree, X, Y, q);
            for (int j = 0; j < cnt; ++j)
              if (!(q[j] >= p && q[j] < p + 4) && newlev(q[j]) > L.level) ok = false;
          }
        }
    }
    if (ok) { coarsen[p] = 1; p += 3; }
  }
  new_levels.clear(); new_trees.clear(); src.clear();
  for (int64_t p = 0; p < P; ++p) {
    const Leaf& L = pl.leaves[p];
    if (refine[p]) {
      for (int k = 0; k < 4; ++k) {
        new_levels.push_back((int8_t)(L.level + 1)); new_trees.push_back(L.tree);
        src.insert(src.end(), {2, (int32_t)p, k});
      }
    } else if (coarsen[p]) {
      new_levels.push_back((int8_t)(L.level - 1)); new_trees.push_back(L.tree);
      src.insert(src.end(), {3, (int32_t)p, 0});
      p += 3;
    } else {
      new_levels.push_back((int8_t)L.level); new_trees.push_back(L.tree);
      src.insert(src.end(), {1, (int32_t)p, 0});
    }
  }
  return FC_OK;
}

}  // namespace fc
