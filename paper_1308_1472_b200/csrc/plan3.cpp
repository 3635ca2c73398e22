// plan3.cpp -- host planner of the octree path (libfc, include/fc3.h): Morton decode of the leaves,
// a leaf hash, and the canonical ghost records of every ring cell.  Not shared with oracle/.
//
// PAPER.md:141-144 [§2]: ghost cells from the neighbour relations of the leaves
// [Fig. 1]: octrees analogous to quadtrees.  The source of a ghost cell: move its centre across the
// tree faces it lies beyond (axis by axis, aligned links), then look the leaf up in a hash of
// (tree, level, x, y, z) at the patch's level (COPY), one coarser (INTERP) or, for the finer case,
// the child that holds the 2x2x2 block (AVG8).  (The oracle instead binary-searches Morton ranges.)
#include <cstdint>
#include <cstring>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "../../include/fc3.h"

namespace fc {

struct Plan3 {
  int64_t P = 0;
  int m = 0, T = 0, lmax = 0;
  std::vector<int32_t> t2t;
  std::vector<int8_t> fbc, level;
  std::vector<int32_t> tree;
  std::vector<int64_t> x, y, z;   // origin in level-Lmax leaves
  struct KeyHash {
    size_t operator()(const std::tuple<int32_t, int32_t, int64_t, int64_t, int64_t>& k) const {
      uint64_t h = (uint64_t)std::get<0>(k) * 0x9E3779B97F4A7C15ull;
      h ^= (uint64_t)std::get<1>(k) + 0x7F4A7C159E3779B9ull + (h << 6) + (h >> 2);
      h ^= (uint64_t)std::get<2>(k) * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
      h ^= (uint64_t)std::get<3>(k) * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
      h ^= (uint64_t)std::get<4>(k) * 0x27D4EB2F165667C5ull + (h << 6) + (h >> 2);
      return (size_t)h;
    }
  };
  std::unordered_map<std::tuple<int32_t, int32_t, int64_t, int64_t, int64_t>, int64_t, KeyHash> index;
  std::vector<int32_t> table;   // [P][G][8]
};

static inline int ring3(int m) { const int n = m + 4; return n * n * n - m * m * m; }

static int64_t find3(const Plan3& pl, int t, int l, int64_t x, int64_t y, int64_t z) {
  auto it = pl.index.find(std::make_tuple((int32_t)t, (int32_t)l, x, y, z));
  return it == pl.index.end() ? -1 : it->second;
}

int plan3_build(const fc3_forest_desc* d, Plan3& pl, std::string& err) {
  if (!d || !d->levels || !d->tree_ids || !d->tree_to_tree || !d->face_bc) { err = "null descriptor field"; return FC_EINVAL; }
  if (d->num_patches <= 0 || d->num_trees <= 0) { err = "empty forest"; return FC_EINVAL; }
  if (d->m < 4 || d->m > 32 || (d->m & 1)) { err = "m must be even, 4..32"; return FC_EINVAL; }
  if (!(d->tree_dx0 > 0.0)) { err = "tree_dx0 must be positive"; return FC_EINVAL; }
  pl.P = d->num_patches; pl.m = d->m; pl.T = d->num_trees;
  pl.t2t.assign(d->tree_to_tree, d->tree_to_tree + 6 * pl.T);
  pl.fbc.assign(d->face_bc, d->face_bc + 6 * pl.T);
  for (int t = 0; t < pl.T; ++t)
    for (int f = 0; f < 6; ++f) {
      if (pl.fbc[6 * t + f]) continue;
      const int nt = pl.t2t[6 * t + f];
      if (nt < 0 || nt >= pl.T || pl.fbc[6 * nt + (f ^ 1)] || pl.t2t[6 * nt + (f ^ 1)] != t) {
        err = "connectivity: a linked face must link back through the opposite face";
        return FC_ECONN;
      }
    }
  pl.level.assign(d->levels, d->levels + pl.P);
  pl.tree.assign(d->tree_ids, d->tree_ids + pl.P);
  int lmax = 0;
  for (int64_t p = 0; p < pl.P; ++p) {
    if (pl.level[p] < 0 || pl.level[p] > 18) { err = "level out of range"; return FC_EINVAL; }
    lmax = std::max(lmax, (int)pl.level[p]);
    if (pl.tree[p] < 0 || pl.tree[p] >= pl.T || (p && pl.tree[p] < pl.tree[p - 1])) {
      err = "tree ids must be non-decreasing and in range"; return FC_ETILING;
    }
  }
  pl.lmax = lmax;
  pl.x.resize(pl.P); pl.y.resize(pl.P); pl.z.resize(pl.P);
  // decode: walk each tree's leaves with a cursor in the 8^Lmax index space
  int64_t p = 0;
  const uint64_t total = 1ull << (3 * lmax);
  for (int t = 0; t < pl.T; ++t) {
    uint64_t c = 0;
    for (; p < pl.P && pl.tree[p] == t; ++p) {
      const uint64_t size = 1ull << (3 * (lmax - pl.level[p]));
      if (c % size != 0 || c >= total) { err = "leaf not aligned to its size in the Morton order"; return FC_ETILING; }
      int64_t X = 0, Y = 0, Z = 0;
      for (int b = 0; b < lmax; ++b) {
        X |= (int64_t)((c >> (3 * b)) & 1) << b;
        Y |= (int64_t)((c >> (3 * b + 1)) & 1) << b;
        Z |= (int64_t)((c >> (3 * b + 2)) & 1) << b;
      }
      pl.x[p] = X; pl.y[p] = Y; pl.z[p] = Z;
      pl.index[std::make_tuple((int32_t)t, (int32_t)pl.level[p], X, Y, Z)] = p;
      c += size;
    }
    if (c != total) { err = "tree not covered by its leaves"; return FC_ETILING; }
  }
  // ghost records
  const int m = pl.m, G = ring3(m);
  const int64_t E = (2 * (int64_t)m) << lmax;   // tree edge in fine units (a level-Lmax cell = 2)
  pl.table.assign((size_t)pl.P * G * 8, 0);
  for (int64_t q = 0; q < pl.P; ++q) {
    const int l = pl.level[q];
    const int64_t sz = 1ll << (lmax - l), h = sz;
    const int64_t O[3] = {pl.x[q] * 2 * m, pl.y[q] * 2 * m, pl.z[q] * 2 * m};
    int r = 0;
    for (int k = -1; k <= m + 2; ++k)
      for (int j = -1; j <= m + 2; ++j)
        for (int i = -1; i <= m + 2; ++i) {
          if (i >= 1 && i <= m && j >= 1 && j <= m && k >= 1 && k <= m) continue;
          int32_t* o = pl.table.data() + ((size_t)q * G + r++) * 8;
          const int ijk[3] = {i, j, k};
          int64_t Pt[3];
          for (int a = 0; a < 3; ++a) Pt[a] = O[a] + (2 * ijk[a] - 1) * h;
          int t = pl.tree[q], last = -1;
          bool inside = true;
          for (int a = 0; a < 3; ++a) {
            if (Pt[a] >= 0 && Pt[a] < E) continue;
            const int fc = 2 * a + (Pt[a] >= E);
            if (pl.fbc[6 * t + fc]) { inside = false; last = a; continue; }
            t = pl.t2t[6 * t + fc];   // (linked crossings continue past a physical one: they decide
            Pt[a] += Pt[a] < 0 ? E : -E;   // which tree's faces the later axes test)
          }
          if (!inside) {   // outflow: the last physical axis writes last (x, y, z order)
            o[0] = 4 + last;
            o[1] = (int32_t)q;
            o[2] = i; o[3] = j; o[4] = k;
            o[2 + last] = ijk[last] < 1 ? 1 : m;
            continue;
          }
          // the leaf containing the point: same level, one coarser, or the finer child
          const int64_t lw = 2 * (int64_t)m;   // level-Lmax leaf width in fine units
          int64_t id = -1;
          for (int dl = 0; dl <= 2 && id < 0; ++dl) {
            const int L = dl == 0 ? l : (dl == 1 ? l - 1 : l + 1);
            if (L < 0 || L > lmax) continue;
            const int64_t s = 1ll << (lmax - L);
            id = find3(pl, t, L, (Pt[0] / lw) / s * s, (Pt[1] / lw) / s * s, (Pt[2] / lw) / s * s);
          }
          if (id < 0) { err = "2:1 balance violated (neighbour more than one level off)"; return FC_EBALANCE; }
          const int lL = pl.level[id];
          const int64_t LO[3] = {pl.x[id] * 2 * m, pl.y[id] * 2 * m, pl.z[id] * 2 * m};
          o[1] = (int32_t)id;
          if (lL == l) {
            o[0] = 1;
            for (int a = 0; a < 3; ++a) o[2 + a] = (int32_t)(((Pt[a] - LO[a]) / h + 1) / 2);
          } else if (lL == l + 1) {
            o[0] = 2;
            for (int a = 0; a < 3; ++a) o[2 + a] = (int32_t)((Pt[a] - LO[a]) / h);
          } else {
            o[0] = 3;
            for (int a = 0; a < 3; ++a) {
              const int64_t rel = Pt[a] - LO[a], I = rel / (4 * h);
              o[2 + a] = (int32_t)(I + 1);
              o[5 + a] = (rel - I * 4 * h > 2 * h) ? 1 : -1;
            }
          }
        }
  }
  return FC_OK;
}

}  // namespace fc
