// fc_internal.h -- libfc private structures (host planner <-> device runtime).
// Nothing here is shared with oracle/ (the oracle has its own sources and header).
#pragma once
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/fc.h"

namespace fc {

#ifdef __CUDACC__
#define FC_HD __host__ __device__
#else
#define FC_HD
#endif

// Storage of a padded patch in device memory, per (patch, component) block of n^2 doubles
// (n = m + 4): the m x m interior first, dense and row-major (cell (i, j), i, j = 1..m, at
// (j - 1) m + (i - 1)), then the 8m + 16 ghost cells in ring order (rows j = -1..m+2 outer, columns
// i = -1..m+2 inner, interior skipped) -- the order of the ring tables.  Interior-only traffic (the
// quiescent copy, interior staging) then streams whole contiguous 2 KB blocks: B200's DRAM fetch
// granule made a strided interior (128 of every 160 bytes) cost the full rows (measured with
// tools/dram_pattern.cu: 16 of 20 doubles per row reads 100% of the bytes).  The ABI's padded
// arrays (fc_get_q_padded, aux) keep the natural layout (j + 1) n + (i + 1).
FC_HD inline int ring_index(int i, int j, int m) {
  const int n = m + 4;
  if (j <= 0) return (j + 1) * n + (i + 1);
  if (j <= m) return 2 * n + 4 * (j - 1) + (i <= 0 ? i + 1 : i - m + 1);
  return 2 * n + 4 * m + (j - m - 1) * n + (i + 1);
}
FC_HD inline int qcell(int i, int j, int n) {
  const int m = n - 4;
  if (i >= 1 && i <= m && j >= 1 && j <= m) return (j - 1) * m + (i - 1);
  return m * m + ring_index(i, j, m);
}
// natural padded index -> storage index
inline int qcell_of_natural(int cell, int n) { return qcell(cell % n - 1, cell / n - 1, n); }

// ghost-record ops (canonical EXPANDED table, include/fc.h)
enum Op : int32_t { OP_NONE = 0, OP_COPY = 1, OP_AVG4 = 2, OP_INTERP = 3, OP_BCX = 4, OP_BCY = 5, OP_CORNER3 = 6 };
constexpr int REC = 8;

struct Leaf {
  int32_t tree;
  int32_t level;
  int64_t x, y;  // origin in units of level-Lmax leaves
};

// Isometry of the plane on "fine units" (1 unit = half a level-Lmax cell; tree edge E = 2 m 2^Lmax):
// P' = R P + b, landing in tree `tree`.
struct Affine {
  int r00 = 1, r01 = 0, r10 = 0, r11 = 1;
  int64_t b0 = 0, b1 = 0;
  int32_t tree = 0;
  bool operator==(const Affine& o) const {
    return r00 == o.r00 && r01 == o.r01 && r10 == o.r10 && r11 == o.r11 && b0 == o.b0 &&
           b1 == o.b1 && tree == o.tree;
  }
};

enum DirKind : int { D_SAME = 0, D_COARSER = 1, D_FINER = 2, D_PHYS = 3, D_CORNER3 = 4 };

struct DirInfo {
  DirKind kind;
  Affine T;        // p's tree coordinates -> neighbour tree coordinates
  int64_t leaf;    // SAME / COARSER: the neighbour leaf; FINER: resolved per cell
};

struct LeafKeyHash {
  size_t operator()(const std::tuple<int32_t, int32_t, int64_t, int64_t>& k) const {
    uint64_t h = (uint64_t)std::get<0>(k) * 0x9E3779B97F4A7C15ull;
    h ^= (uint64_t)std::get<1>(k) + 0x7F4A7C159E3779B9ull + (h << 6) + (h >> 2);
    h ^= (uint64_t)std::get<2>(k) * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
    h ^= (uint64_t)std::get<3>(k) * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
    return (size_t)h;
  }
};

// Typed ghost work lists, offsets in doubles relative to the state base:
// local patch slot s, cell c -> s * S + c (S = meqn n^2); halo cell h -> (Pl + h / n2) * S + h % n2.
struct GhostLists {
  std::vector<int32_t> copy;      // {dst, src}
  std::vector<int32_t> avg;       // {dst, s00, s10, s01, s11}
  std::vector<int32_t> bcx, bcy;  // {dst, src, negated component or -1}  (all patches)
  std::vector<int32_t> corner3;   // {dst, a, b}
  // per level l: INTERP records {dst, c, xm, xp, ym, yp, sigx, sigy} and that level's BC records
  std::vector<std::vector<int32_t>> interp, bcx_l, bcy_l;
};

struct HaloPlan {
  // per peer: requested remote cells (global patch id * n2 + cell), rounds 1 and 2
  std::vector<std::vector<int64_t>> need1, need2;
  int64_t n1 = 0, n2 = 0;   // total halo cells per round
  std::unordered_map<int64_t, int64_t> slot;   // key (gpatch * n2 + cell) * 2 + (round - 1) -> slot
};

struct Plan {
  int64_t P = 0;
  int32_t T = 0, m = 0, n = 0, meqn = 0, maux = 0, lmax = 0;
  double dx0 = 0.0;
  std::vector<Leaf> leaves;
  std::unordered_map<std::tuple<int32_t, int32_t, int64_t, int64_t>, int64_t, LeafKeyHash> index;
  std::vector<int32_t> t2t;
  std::vector<int8_t> t2f, fbc;
  int rank = 0, nranks = 1;
  int64_t p0 = 0, p1 = 0;           // local range [p0, p1)
  std::vector<int64_t> part;        // [nranks + 1] Morton cut points (rank r owns [part[r], part[r+1]))
  std::vector<int32_t> table;       // expanded records of local patches [Pl][G][8]
  HaloPlan halo;
  bool uniform_same = false;        // every ring cell is COPY/BC (no AVG/INTERP/CORNER3)
  int lmin_local = 0, lmax_local = 0;
};

// Fused ring gather (forests whose ghost records are all COPY / BCX / BCY, one tile per patch):
// per local patch, G entries in ring storage order: >= 0 = source offset of component 0 (local or
// halo slot, as in the ghost lists); < 0 = -1 - ((window_src << 3) | (negated_comp << 1) | is_y)
// for a physical-boundary cell filled from the patch's own window.  bcflag[p]: bit 0 BCX, bit 1 BCY.
struct RingSources {
  std::vector<int32_t> src;
  // peer-memory halo (p2p): 0 = src is an offset in this rank's state, k > 0 = in rank k-1's
  // local state (its own patch numbering); empty without p2p (remote cells use halo slots)
  std::vector<uint8_t> peer;
  std::vector<uint8_t> bcflag;
  // activity test: the <= 8 distinct patches the ring reads (local ids; -2 = a remote patch,
  // -1 = unused) and a mask of components a wall negates (they must vanish for a quiescent patch)
  std::vector<int32_t> nbr;     // [Pl][8]
  std::vector<uint8_t> negmask; // [Pl]
};

// planner entry points (plan.cpp); return FC_OK or an FC_E* code with err set
int plan_build(const fc_forest_desc* d, Plan& pl, std::string& err);
// build typed lists for `meqn` (component stride n^2); halo slots from pl.halo
int plan_lists(const Plan& pl, int meqn, GhostLists& gl, std::string& err,
               const std::vector<uint8_t>* dst_mask = nullptr);
int plan_ring_sources(const Plan& pl, int meqn, RingSources& rs, std::string& err, bool p2p = false);
// COMPACT ghost-table rows of patch p (global id): 8 directions x {kind, nbr0, nbr1, xform, half}
int plan_compact_patch(const Plan& pl, int64_t p, int32_t* out40, std::string& err);
// fused two-hop ring gather on AMR forests: computed-ghost (AVG4 / INTERP) lists and slot count
struct RingAmr {
  std::vector<int32_t> avg;                  // {dst slot offset, 4 q_old offsets}
  std::vector<std::vector<int32_t>> interp;  // per level: {dst slot offset, 5 refs, sigx, sigy}
  std::vector<int32_t> corner3;              // {dst slot offset, 2 refs}: after every level
  int64_t ncg_patches = 0;                   // computed-ghost buffer size in n^2-cell virtual patches
};
int plan_ring_amr(const Plan& pl, int meqn, RingSources& rs, RingAmr& ra, std::string& err);
// Regular rings: a local patch whose every ring cell is a COPY of the aligned cell of one of its 8
// same-level neighbours (local, no wall / outflow cell) gets nb9[lp][3 (dy + 1) + dx + 1] = the
// block offset (patch * meqn n^2) of the neighbour in direction (dx, dy) (its own at the centre):
// the step kernels then compute every source address instead of loading it from rs.src.  Checked
// entry by entry against rs.src (the same source cells, bitwise the same gather); -1 at [lp][0]:
// use the table.  Returns the number of regular patches.
int64_t plan_ring_regular(const Plan& pl, int meqn, const RingSources& rs, std::vector<int32_t>& nb9);
// activity tables for the quiescent filter on any forest: nbr [Pl][8] / negmask [Pl] as in
// RingSources; a patch with an AVG4 / INTERP / CORNER3 ghost record is always active (nbr[0] = -2)
int plan_activity(const Plan& pl, int meqn, std::vector<int32_t>& nbr, std::vector<uint8_t>& negmask,
                  std::string& err);

// Coarse/fine reflux.  slot[lp] >= 0 for local patches with a face whose
// neighbour is one level coarser or finer: the step kernel records, for each of their 4 faces and
// m boundary edges, the applied flux in outward form into reg[((slot * 4 + face) * m + edge) *
// meqn + k].  cells: one record per coarse cell next to >= 1 finer face, RFX ints each:
// {q offset (storage, component 0), aux offset of kappa (natural, -1 = none), local patch,
//  number of faces (1 or 2), then per face (ascending face order) {RO_coarse, RO_fine1, RO_fine2}}
// with RO = register offset of component 0 of that (slot, face, edge).
constexpr int RFX = 10;
struct RefluxPlan {
  std::vector<int32_t> slot;
  int32_t nslots = 0;
  std::vector<int32_t> cells;
  // fine faces owned by other ranks: per owner rank the keys (fine patch global id * 4 + face) in
  // remote-face order; remote face r (owner-major) lives at face index 4 nslots + r of freg
  std::vector<std::vector<int64_t>> req;
  int64_t nremote = 0;
};
int plan_reflux(const Plan& pl, int meqn, RefluxPlan& rf, std::string& err);
// Dynamic regrid (one rank): new leaves in Morton order and per new leaf {kind (1 copy, 2 child,
// 3 parent), old patch (first child for a parent), child index}; tag[p] = max - min of component 0
int plan_regrid(const Plan& pl, const double* tag, double refine_threshold, double coarsen_threshold,
                int min_level, int max_level, std::vector<int8_t>& new_levels, std::vector<int32_t>& new_trees,
                std::vector<int32_t>& src, std::string& err);

}  // namespace fc
