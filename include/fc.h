/* fc.h -- C ABI of libfc: the B200-native ForestClaw hot path (arXiv 1308.1472).
 *
 * One global-dt time step on every leaf patch of a static forest of quadtrees
 * (PAPER.md:275-277 [§4] "one such parallel data exchange per time step for a global value of
 * the time step length dt"): ghost-cell fill (PAPER.md:187-201 [§3]: same-level copy, fine->coarse
 * averaging, coarse->fine limited interpolation, tree-boundary index remap PAPER.md:258-260 [§4],
 * physical boundaries), then the Clawpack wave-propagation update (PAPER.md:168-182 [§3]) and the
 * CFL max-reduction.  Hand-written CUDA for sm_100a, fp64 throughout, NCCL between GPUs.
 *
 * Conventions shared by every call:
 *   - All functions return FC_OK (0) or a negative FC_E* code; nothing throws across the ABI.
 *     fc_last_error() returns a thread-local message for the last failure.
 *   - Handles are opaque, owned by the library, not thread-safe: one handle per process/GPU.
 *   - Patches are in global Morton order (trees ascending, z-order inside a tree, x on the even
 *     bits).  Rank r of R owns patches [floor(r P / R), floor((r+1) P / R)) ("local" patches).
 *   - Cell arrays are fp64, structure of arrays per patch, x fastest:
 *       interior  q[P_local][meqn][m][m]
 *       padded    q[P_local][meqn][n][n], n = m + 2 mbc, cell (i, j) (1-based, i, j in
 *                 [-1, m+2]) at [(j+1) n + (i+1)]
 *   - `where` selects the memory space of a user pointer: FC_HOST (pageable or pinned host
 *     memory) or FC_DEVICE (a device pointer on the handle's GPU, e.g. torch data_ptr()).
 *     User buffers are copied; the caller keeps ownership.
 *   - All device work is issued on the handle's stream (fc_set_stream, default: a private
 *     non-blocking stream).  Calls that return data to the host synchronise that stream.
 */
#ifndef FC_H
#define FC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ---------------------------------------------------------------------------- */
#define FC_OK 0
#define FC_EINVAL -1      /* bad argument / descriptor field */
#define FC_ETILING -2     /* leaves do not tile every tree in z-order (Morton decode failed) */
#define FC_ECONN -3       /* connectivity not symmetric or out of range */
#define FC_EBALANCE -4    /* face or corner level jump > 1 (2:1 balance) */
#define FC_ECUDA -5       /* CUDA runtime error */
#define FC_ENCCL -6       /* NCCL error */
#define FC_ENOMEM -7      /* host or device allocation failed */
#define FC_ESTATE -8      /* call out of order (e.g. fc_step before fc_set_problem / fc_set_q) */
#define FC_ECFL -9        /* step rejected: max CFL > cfl_reject; state unchanged */
#define FC_ENONFINITE -10 /* CFL is NaN/Inf; state unchanged */
#define FC_EUNSUP -11     /* configuration outside what this build supports */

/* ---- enums --------------------------------------------------------------------------------- */
#define FC_HOST 0
#define FC_DEVICE 1

#define FC_ADV_CONST 0        /* q_t + u q_x + v q_y = 0, (p0, p1) = (u, v); meqn 1, maux 0 */
#define FC_ADV_EDGEVEL_CAPA 1 /* kappa q_t + (u~ q)_xi + (v~ q)_eta advective form; aux = {kappa, u~ (left edge), v~ (bottom edge)}; meqn 1, maux 3 */
#define FC_SWE_ROE 2          /* shallow water (h, hu, hv), p0 = g; meqn 3 */
#define FC_EULER_ROE 3        /* Euler (rho, rho u, rho v, E), p0 = gamma, p1 != 0: Harten-Hyman entropy fix; meqn 4 */
#define FC_EULER_HLLE 4       /* Euler, HLLE two-wave solver (Roe transverse), p0 = gamma; meqn 4 */

#define FC_LIM_NONE 0
#define FC_LIM_MINMOD 1
#define FC_LIM_MC 2

#define FC_BC_OUTFLOW 0
#define FC_BC_WALL 1

#define FC_TABLE_EXPANDED 1   /* per ghost cell records, see fc_get_ghost_table */
#define FC_TABLE_COMPACT 2    /* per patch direction: kind, neighbours, orientation, see fc_get_ghost_table */

/* ---- descriptors --------------------------------------------------------------------------- */
typedef struct fc_forest fc_forest;

typedef struct {
  int64_t num_patches;          /* P, global */
  const int8_t* levels;         /* [P] leaf levels, global Morton order */
  const int32_t* tree_ids;      /* [P] non-decreasing tree ids */
  int32_t num_trees;            /* T */
  const int32_t* tree_to_tree;  /* [4T] neighbour tree across face f = 0 (-x), 1 (+x), 2 (-y), 3 (+y) */
  const int8_t* tree_to_face;   /* [4T] neighbour face + 4 * reversed; (t, f) -> (t, f) = physical */
  const int8_t* face_bc;        /* [4T] FC_BC_OUTFLOW | FC_BC_WALL on physical faces */
  int32_t m;                    /* cells per patch side, even, >= 4 */
  int32_t mbc;                  /* ghost layers, must be 2 */
  int32_t meqn;                 /* equations (must match the problem kind) */
  int32_t maux;                 /* aux fields (3 for FC_ADV_EDGEVEL_CAPA, else 0) */
  double tree_dx0;              /* tree edge length (a level-l cell is tree_dx0 2^-l / m wide) */
  int32_t device;               /* CUDA device ordinal; -1 = host-only planning handle (tables only) */
  int32_t rank, nranks;         /* this process among nranks (1 = single GPU) */
  const void* nccl_id;          /* 128-byte ncclUniqueId when nranks > 1 (fc_nccl_unique_id on rank 0);
                                   NULL with nranks > 1 selects the manual halo transport (below) */
  int32_t halo_p2p;             /* 1 (nranks > 1, uniform forests, fused ring gather): ring cells owned
                                   by other ranks are read inside the update kernel straight from the
                                   owners' state buffers in peer memory (CUDA IPC over NVLink; in manual
                                   mode wired with fc_p2p_set_peer) -- no pack / ncclSend/Recv / unpack
                                   pass (PAPER.md:264-272's ghost exchange fused into the gather); the
                                   CFL allreduce orders the steps across ranks.  0: halo exchange */
  const int64_t* partition;     /* optional [nranks + 1] Morton cut points (0 = p_0 <= p_1 ... <= p_R =
                                   num_patches; rank r owns [p_r, p_{r+1})), identical on every rank;
                                   NULL: by count, [floor(rP/R), floor((r+1)P/R)) */
} fc_forest_desc;

typedef struct {
  int32_t kind;                 /* FC_ADV_CONST ... */
  double p0, p1;                /* physical parameters, see the kind */
  int32_t limiter;              /* FC_LIM_* (wave limiter) */
  int32_t method2;              /* 1: first order; 2: + limited second-order corrections */
  int32_t method3;              /* 0: no transverse; 1: transverse of A+-dq; 2: also of the corrections */
  double cfl_reject;            /* fc_step rejects (FC_ECFL) when max CFL exceeds this (e.g. 1.0) */
  int32_t skip_quiescent;       /* 1: exact shortcut for tiles whose 2-cell-haloed window holds one
                                   uniform state (all waves are exactly 0, so q_new = q bitwise and only
                                   the CFL is evaluated); 0: always run the full update */
  int32_t reflux;               /* 1: conservative coarse/fine flux correction after the update
                                   (PAPER.md:279-282): every coarse cell next to a
                                   face whose neighbour is one level finer has the flux it applied
                                   through that face replaced by the mean of the two fine fluxes, so
                                   sum kappa q is conserved across coarse/fine faces.  No-op on
                                   conforming meshes.  FC_EUNSUP (at fc_set_problem) for systems
                                   (meqn > 1) across rotated tree links.  Coarse/fine pairs split
                                   between ranks exchange the fine-face records every step
                                   (fc_reflux_* below for the manual transport); only the sub-cycled
                                   step refuses them.  0: off (the paper's global-dt step) */
} fc_problem;

typedef struct {
  int64_t kernel_launches;      /* kernels this handle launched since creation / last reset */
  int64_t steps;                /* committed steps */
  double ms_ghost;              /* accumulated device time in ghost-fill kernels (timing on) */
  double ms_step;               /* accumulated device time in the update kernel (timing on) */
  double ms_comm;               /* accumulated device time in halo pack/NCCL/unpack + allreduce */
  int64_t step_kernel_launches; /* launches of the update kernel counted in ms_step */
  int64_t local_patches;        /* patches owned by this rank */
  int64_t halo_cells;           /* remote cells received per step (all rounds) */
  int32_t uniform_fast_path;    /* fused gather path (no ring writes): 1 uniform forest, 2 AMR forest
                                   (two-hop: computed AVG/INTERP ghosts), 0 ghost kernels */
  int32_t pad_;
  double ms_copy;               /* accumulated device time in the quiescent copy/classify kernel (part of ms_step) */
  int64_t copy_launches;        /* launches counted in ms_copy */
  int64_t regular_patches;      /* local patches with a regular ring (every ring cell a copy of
                                   the aligned cell of a same-level local neighbour): the scalar
                                   sweeps compute their gather addresses and move the ring in
                                   16-byte pairs; other patches (and the systems kernel) read the
                                   ring table.  Bitwise the same gather either way */
  int64_t quad_blocks;          /* m = 8 constant-velocity advection: 2 x 2 sibling families of
                                   regular patches swept as one 16 x 16 window (every local patch
                                   regular, the local list whole families; FC_CV_QUAD=0: off): each
                                   family edge computed once.  Bitwise the per-patch sweep */
} fc_stats;

/* ---- calls --------------------------------------------------------------------------------- */

/* PAPER.md:105-113 [§2] (a forest of quadtrees, one m x m patch per leaf), PAPER.md:132-144 [§2]
 * (multiblock: each tree a reference square with its own orientation; the connectivity; ghost
 * cells from the neighbour relations), PAPER.md:150-155 [§2] (2:1 balance)
 * [Fig. 1, §4] (leaves ordered along a space-filling curve and partitioned among processes, one
 * layer of ghost leaves).
 * Copy and validate the forest, decode Morton order, build the neighbour / ghost tables and the
 * shard + halo plan, allocate device state (q_old, q_new double buffer, aux) and, when
 * nranks > 1, create the NCCL communicator.  Validation: tree ids non-decreasing and every tree
 * tiled exactly (FC_ETILING); connectivity symmetric (FC_ECONN); m even >= 4, mbc == 2
 * (FC_EINVAL); face and corner level jumps <= 1 (FC_EBALANCE).  *out is NULL on failure. */
int fc_forest_create(const fc_forest_desc* desc, fc_forest** out);

/* Free everything the handle owns (device memory, streams, events, communicator). */
int fc_forest_destroy(fc_forest* f);

/* Select the solver (PAPER.md:168-182 [§3]: Clawpack's wave propagation with a problem-specific
 * Riemann solver, wave limiters, second-order and transverse corrections; kinds and readings in
 * DESIGN.md §3).  FC_EINVAL if kind/meqn/maux disagree or parameters are out of range. */
int fc_set_problem(fc_forest* f, const fc_problem* pr);

/* aux[P_local][maux][n][n] including the ghost ring (FC_ADV_EDGEVEL_CAPA only): kappa, u~ at
 * each cell's left edge, v~ at its bottom edge.  Copied into device memory. */
int fc_set_aux(fc_forest* f, const double* aux, int where);

/* PAPER.md:113-125 [§2] (each leaf houses one patch of m^d cells: the numerical data).
 * q[P_local][meqn][m][m] (x fastest; patches in global Morton order; host or device by
 * `where`; caller keeps ownership) -> interior of q_old.  The ghost ring becomes stale until the
 * next fill.  FC_ESTATE before fc_set_problem. */
int fc_set_q(fc_forest* f, const double* q, int where);

/* Fill the ghost rings of q_old (halo exchange included) -- inspection / tests; fc_step does its
 * own fill.  Ring contents are then readable with fc_get_q_padded. */
int fc_ghost_fill(fc_forest* f);

/* One step: ghost fill + wave-propagation update of every local patch + global max CFL
 * (*max_cfl, max over edges and waves of dt |s| / (kappa dx) taken on the upwind side,
 * PAPER.md:276-277).  Commits (swaps q_old / q_new) iff max_cfl <= cfl_reject; otherwise returns
 * FC_ECFL with q unchanged.  FC_EINVAL if dt <= 0 or not finite; FC_ENONFINITE if the CFL is
 * NaN/Inf or the updated state is not finite (state unchanged).  Synchronises the handle's stream (the CFL is returned to the host). */
int fc_step(fc_forest* f, double dt, double* max_cfl);

/* One sub-cycled step (PAPER.md:201-202 [§3] "when sub-cycling, time accurate data between coarse
 * grids is used to fill in ghost cells for fine grids", PAPER.md:277-290 [§4] one exchange per
 * level, coarse-to-fine recursion): the coarsest level of the forest advances by
 * dt_coarse and level l by dt_coarse 2^-(l - lmin), each level after a ghost fill (halo exchange
 * included) in which coarser patches hold their state interpolated linearly in time; with
 * fc_problem.reflux the coarse/fine fluxes are balanced over the fine sub-steps.  *max_cfl = max over
 * all level updates; commit / FC_ECFL / FC_ENONFINITE as fc_step.  On a one-level forest this is
 * fc_step(dt_coarse).  FC_ESTATE on a manual-transport handle.  Extra device memory: two state-sized
 * buffers, allocated at the first call. */
int fc_step_subcycled(fc_forest* f, double dt_coarse, double* max_cfl);

/* nsteps global steps with a fixed dt (the advection configs' policy), as one CUDA graph per step
 * replayed back to back with no host round trip (the per-step CFL goes to a device history;
 * cfls[nsteps] receives it if not NULL, *max_cfl its maximum).  Same kernels and results as
 * nsteps x fc_step(dt).  If any step's CFL exceeds cfl_reject (FC_ECFL) or is not finite
 * (FC_ENONFINITE) the whole run is undone (state restored).  One rank (FC_EUNSUP otherwise).  The
 * graphs are captured at the first call and again when dt or nsteps' capacity changes. */
int fc_run(fc_forest* f, double dt, int64_t nsteps, double* cfls, double* max_cfl);

/* Dynamic regrid (PAPER.md:148-155 [§2] 2:1 balanced refinement, PAPER.md:207-211 [§3] "interpolation
 * from coarse grids to newly created fine grids, and the averaging of fine grid data to a newly
 * created underlying coarse grid").  Tag: max - min of component 0 over each patch.
 * Refine when above refine_threshold (level < max_level), then refine neighbours as needed for the
 * face and corner 2:1 balance; coarsen a complete family of 4 siblings (level > min_level) when all
 * are below coarsen_threshold, none is refined and no outside neighbour would end more than one
 * level finer.  Data: copied, limited (minmod) interpolation from the ghost-filled parent (the ghost
 * fill's formula), or the 2x2 average.  *out is a NEW handle on the new forest (same connectivity,
 * m, meqn, device, problem; q set; aux NOT set: the capacity form needs fc_set_aux on the new mesh,
 * see fc_get_leaves); the old handle is unchanged and stays valid.  One rank only (FC_EUNSUP). */
typedef struct {
  double refine_threshold, coarsen_threshold;
  int32_t min_level, max_level;
  int32_t level_weights;        /* multi-rank: 1 = cut the new Morton order into equal sums of
                                   2^(level - coarsest level) (the work of a sub-cycled step), 0 = by count */
  int32_t pad_;
} fc_regrid_params;
int fc_regrid(fc_forest* f, const fc_regrid_params* rp, fc_forest** out);

/* Multi-rank regrid (SURVEY §8(f) #3 "Morton repartition + NCCL migration").  On NCCL handles
 * fc_regrid is collective: ghost fill with halo, local tags, all-gathered tags, the same global
 * plan on every rank, a new handle partitioned by count over the same ranks (its NCCL id broadcast
 * from rank 0), and migration of the old padded blocks each new patch reads from their old owners
 * (grouped send/recv), then the transfer.  Manual transport, per rank: halo round 1,
 * fc_regrid_fill(1), halo round 2, fc_regrid_fill(2) (rings filled); fc_regrid_tags (the local
 * patches' tags, host); fc_regrid_begin with the concatenation of all ranks' tags (global patch
 * order) -> the new handle; copy recv_g[recv_off[s]..] <- send_s[send_off_s[me]..] between ranks
 * (fc_regrid_buffers(old, new): device pointers, offsets in doubles, [nranks + 1]; the own part is
 * already in place); fc_regrid_finish(new).  The new handle then needs its halo requests (and
 * reflux requests) set as any manual handle. */
int fc_regrid_fill(fc_forest* f, int phase);
int fc_regrid_tags(fc_forest* f, double* tags);
int fc_regrid_begin(fc_forest* f, const double* global_tags, const fc_regrid_params* params, fc_forest** out);
int fc_regrid_buffers(fc_forest* f, fc_forest* g, void** send, void** recv, int64_t* send_off, int64_t* recv_off);
int fc_regrid_finish(fc_forest* g);

/* The forest's leaves in global Morton order: levels[P], tree_ids[P] (either may be NULL; both NULL
 * = size query); *num_patches = P.  FC_EINVAL if cap < P. */
int fc_get_leaves(fc_forest* f, int8_t* levels, int32_t* tree_ids, int64_t cap, int64_t* num_patches);

/* PAPER.md:113-125 [§2] (the per-leaf patch data).  Interior q_old -> q[P_local][meqn][m][m]
 * (layout as fc_set_q; host or device by `where`; caller-owned buffer).  Synchronous on the
 * handle's stream.  FC_ESTATE on a host-only handle. */
int fc_get_q(fc_forest* f, double* q, int where);

/* Padded q_old (ring as left by the last fill) -> q[P_local][meqn][n][n].  Synchronous. */
int fc_get_q_padded(fc_forest* f, double* q, int where);

/* Canonical ghost table of the LOCAL patches (global patch ids, independent of sharding).
 * PAPER.md:141-144 [§2] (constant-time neighbour lookup, with the relative orientation across
 * tree boundaries), PAPER.md:193-201 [§3] (the copy / average / interpolate ghost operations).
 * which = FC_TABLE_COMPACT: for each local patch, 8 directions d (faces -x, +x, -y, +y, then
 * corners (-x,-y), (+x,-y), (-x,+y), (+x,+y)), 5 int32 {kind, nbr0, nbr1, xform, half}:
 *   kind  0 SAME level, 1 COARSER (one level), 2 FINER (one level), 3 PHYS (physical boundary),
 *         4 CORNER3 (three-tree cube corner);
 *   nbr0, nbr1  global ids: SAME / COARSER the neighbour leaf (nbr1 = -1); FINER face the two
 *         finer leaves along the face, lower tangential coordinate of this patch's frame first;
 *         FINER corner the one finer leaf at the corner (nbr1 = -1); PHYS / CORNER3 -1, -1;
 *   xform orientation of this patch's frame in the neighbour's tree, 4 swap + 2 flip_x + flip_y:
 *         e_x -> (-1)^flip_x e_x', e_y -> (-1)^flip_y e_y' (swap = 0) or e_x -> (-1)^flip_x e_y',
 *         e_y -> (-1)^flip_y e_x' (swap = 1); -1 for PHYS / CORNER3;
 *   half  COARSER faces: which half (0 lower, 1 upper, along this patch's tangential coordinate)
 *         of the coarse leaf's face this patch touches; -1 otherwise.
 *   *len = P_local * 40.
 * which = FC_TABLE_EXPANDED: for each local patch, for each ring cell in storage order
 * (j = -1..m+2 outer, i = -1..m+2 inner, interior skipped; G = n^2 - m^2 cells), 8 int32
 * {op, src_patch, src_i, src_j, a, b, c, d} with op 1 COPY (src cell), 2 AVG4 (lower-left cell of
 * the 2x2 fine block, source frame), 3 INTERP (coarse cell; a, b = +-1 offset signs in the coarse
 * frame), 4 BCX / 5 BCY (own cell mirrored or extrapolated; a = bc kind), 6 CORNER3 (average of
 * own cells (src_i, src_j) and (c, d)).  *len = P_local * G * 8; FC_EINVAL if cap < *len
 * (len is still set).  Works on host-only handles (device = -1). */
int fc_get_ghost_table(fc_forest* f, int which, int32_t* buf, int64_t cap, int64_t* len);

/* Use the caller's cudaStream_t for all subsequent work (NULL = the handle's own stream). */
int fc_set_stream(fc_forest* f, void* stream);

/* Enable (1) / disable (0) per-phase CUDA-event timing accumulated into fc_stats. */
int fc_set_timing(fc_forest* f, int on);

/* Counters and timings; fc_reset_stats zeroes the accumulating fields. */
int fc_get_stats(fc_forest* f, fc_stats* out);
int fc_reset_stats(fc_forest* f);

/* First local patch (global id) and count of local patches. */
int fc_local_range(fc_forest* f, int64_t* first, int64_t* count);

/* Halo plan of this rank for tests of the sharded path: per peer the number of remote cells this
 * rank receives per step (counts[nranks]).  Works on host-only handles. */
int fc_halo_counts(fc_forest* f, int64_t* counts);

/* The remote cells this rank requests from `peer` in halo round 1 (interior cells) or 2 (ring cells
 * read by interpolation slopes): keys global_patch * n^2 + padded cell index, ascending.
 * *len = count; FC_EINVAL if cap < count.  Works on host-only handles (multi-rank plan tests). */
int fc_halo_requests(fc_forest* f, int peer, int round, int64_t* buf, int64_t cap, int64_t* len);

/* ---- staged step with a caller-provided halo transport ---------------------------------------
 * A handle created with nranks > 1 and nccl_id == NULL uses a *manual* halo transport: no NCCL
 * communicator is created and fc_step / fc_ghost_fill return FC_ESTATE; the caller instead
 *   (once)  passes every peer's requests (fc_halo_requests of the peer, `peer` = this rank) with
 *           fc_halo_set_requests and calls fc_halo_finalize;
 *   (step)  round 1: fc_halo_pack on every rank, copies recv[recv_off[s]..] <- send_s[send_off_s[me]..]
 *           between ranks (fc_halo_buffers: device pointers, offsets in doubles, [nranks + 1]),
 *           fc_halo_unpack; fc_step_local(phase 1) (ghost phases A, C); round 2 likewise (ring cells
 *           read by interpolation); fc_step_local(phase 2) (ghost phase B, update, this rank's CFL);
 *           fc_commit with the max of the ranks' CFLs.
 *   (split)  uniform forests on the fused path without quiescent filter / reflux (e.g. the full
 *           update): fc_halo_pack, fc_step_local(phase 4) (update of the interior patches -- those
 *           whose ring reads no remote cell -- and the CFL reset), the transport, fc_halo_unpack,
 *           fc_step_local(phase 5) (the boundary patches, this rank's CFL); FC_EUNSUP elsewhere.
 * fc_step on an NCCL handle is exactly this sequence with ncclSend/Recv as the transport and
 * ncclAllReduce(max) for the CFL (PAPER.md:264-272 [§4]: exchange, then local neighbour work);
 * where the split applies it overlaps the exchange (pack, NCCL, unpack on a high-priority
 * stream) with the interior update, the boundary patches waiting on the exchange's event.
 * Used to test the sharded data path with several rank handles in one process. */
int fc_halo_set_requests(fc_forest* f, int round, int peer, const int64_t* keys, int64_t n);
int fc_halo_finalize(fc_forest* f);
int fc_halo_buffers(fc_forest* f, int round, void** send, void** recv, int64_t* send_off, int64_t* recv_off);
int fc_halo_pack(fc_forest* f, int round);      /* synchronous */
int fc_halo_unpack(fc_forest* f, int round);    /* synchronous */
int fc_step_local(fc_forest* f, double dt, int phase, double* local_cfl);
int fc_commit(fc_forest* f, double global_cfl); /* FC_ECFL / FC_ENONFINITE as fc_step */

/* ---- reflux across rank cuts (SURVEY §8(f) #1 on shards) --------------------
 * With reflux = 1 on a sharded forest, a coarse cell whose finer face neighbours live on another
 * rank needs their recorded face fluxes.  fc_set_problem plans it: this rank requests each such
 * fine face from its owner (fc_reflux_requests: keys global_fine_patch * 4 + face, in the order
 * of this rank's remote-face records; works on host-only handles).  NCCL handles exchange the
 * requests inside fc_set_problem (collective: every rank calls it) and the records inside fc_step
 * (after the update kernel, before the correction).  Manual transport: pass every peer's requests
 * with fc_reflux_set_requests (`peer` = the requesting rank) and call fc_reflux_finalize once; per
 * step, after fc_step_local(phase 2) (which packs this rank's served records), copy
 * recv[recv_off[s]..] <- send_s[send_off_s[me]..] between ranks (fc_reflux_buffers: device
 * pointers, offsets in doubles, [nranks + 1]), then fc_step_local(phase 3) applies the correction,
 * then fc_commit.  Sub-cycled steps with cross-rank pairs return FC_EUNSUP. */
int fc_reflux_requests(fc_forest* f, int peer, int64_t* buf, int64_t cap, int64_t* len);
int fc_reflux_set_requests(fc_forest* f, int peer, const int64_t* keys, int64_t n);
int fc_reflux_finalize(fc_forest* f);
int fc_reflux_buffers(fc_forest* f, void** send, void** recv, int64_t* send_off, int64_t* recv_off);

/* Peer-memory halo (halo_p2p = 1).  fc_p2p_buffers: this handle's two state buffers (device
 * pointers, fixed for its lifetime; they alternate as q_old / q_new) and *parity = which one is
 * q_old now (0 or 1; all ranks commit in lockstep, so the parity is global).  fc_p2p_set_peer
 * (manual transport only; NCCL handles exchange CUDA IPC handles at creation): register rank
 * `peer`'s two buffers as mapped in this process. */
int fc_p2p_buffers(fc_forest* f, void** buf0, void** buf1, int32_t* parity);
int fc_p2p_set_peer(fc_forest* f, int32_t peer, void* buf0, void* buf1);

/* Write a fresh 128-byte ncclUniqueId into out (call on rank 0, broadcast to the others). */
int fc_nccl_unique_id(void* out);

/* Thread-local message describing the last error (never NULL). */
const char* fc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
