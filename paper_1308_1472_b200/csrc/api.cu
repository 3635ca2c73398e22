// api.cu -- the libfc C ABI (include/fc.h): handle lifetime, device state, ghost-fill schedule,
// halo exchange over NCCL, the step with its CFL reduction, and instrumentation.
//
// Schedule of one step (PAPER.md:264-277 [§4]: one ghost exchange per global-dt step, before the
// local neighbour work):
//   [halo round 1: pack -> ncclSend/Recv -> unpack]  A: copy, average  ->  C: BC x, BC y
//   [halo round 2]  for each level ascending: B: interpolate -> C of that level  ->  CORNER3
//   step kernel (q_old -> q_new, per-CTA CFL max -> atomicMax)  [ncclAllReduce(max)]
//   CFL -> host; commit (swap) iff CFL <= cfl_reject.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fc_internal.h"

namespace fc {
int launch_ghost(int op, double* q, const int32_t* list, int64_t nrec, int meqn, int n2, cudaStream_t st);
int launch_pack(const double* q, const int32_t* idx, int64_t cnt, int meqn, int n2, double* buf, cudaStream_t st);
int launch_unpack(double* q, const int32_t* idx, int64_t cnt, int meqn, int n2, const double* buf, cudaStream_t st);
int launch_scatter(const double* src, double* q, int64_t P, int meqn, int m, cudaStream_t st);
int launch_gather(const double* q, double* dst, int64_t P, int meqn, int m, cudaStream_t st);
int launch_unpack_padded(const double* q, double* dst, int64_t nblocks, int n, cudaStream_t st);
int launch_step(int kind, const double* qold, double* qnew, const double* aux, const int8_t* level,
                int64_t npatch, int m, double dt, double dx0, double p0, double p1, int limiter,
                int method2, int method3, int skip_quiescent, const int32_t* ring, const int32_t* nb9,
                const uint8_t* bcflag,
                const int32_t* active, const int32_t* nactive, unsigned long long* cfl_bits,
                const int32_t* rslot, double* freg, const uint8_t* rpeer, const double* const* peerq,
                const double* cg, cudaStream_t st, int quad = 0);
int launch_cg(int op, const double* q, double* cg, const int32_t* list, int64_t nrec, int meqn, int n2,
              cudaStream_t st);
int launch_copy_blocks(const double* src, double* dst, const int32_t* ids, int64_t nb, int64_t S, cudaStream_t st);
int launch_reflux(const int32_t* cells, int64_t ncells, const double* freg, const double* ffine, double* qnew,
                  const double* aux, const int8_t* level, double wc, double dtr, double dx0, int meqn, int n2,
                  cudaStream_t st);
int launch_sub_snapshot(const double* cur, double* old, const double* old0, double* snap, const int8_t* level,
                        const int32_t* list, int64_t P, int meqn,
                        int m, int n2, int l, const double* alpha, int lmin, cudaStream_t st);
int launch_sub_accumulate(const int32_t* list, int64_t n, const int32_t* rslot, const double* rec, double* acc,
                          int fs, double dt, int add, cudaStream_t st);
int launch_cfl_hist(const unsigned long long* cfl_bits, double* hist, int64_t* idx, cudaStream_t st);
int launch_regrid_tag(const double* q, int64_t P, int meqn, int m, double* tag, cudaStream_t st);
int launch_regrid_transfer(const double* qo, double* qn, const int32_t* src, int64_t NP, int meqn, int m,
                           cudaStream_t st);
int launch_filter(int kind, const double* qold, double* qnew, int npatch, int m, uint8_t* uflag, double* uval,
                  const int32_t* nbr, const uint8_t* negmask, const int8_t* level, double dt, double dx0,
                  double p0, double p1, int32_t* active, int32_t* nactive, unsigned long long* cfl_bits,
                  cudaStream_t st, cudaEvent_t ev_before_copy, cudaEvent_t ev_after_copy);
}  // namespace fc

using namespace fc;

static thread_local std::string g_err = "no error";
namespace fc {
void set_last_error(const std::string& m) { g_err = m; }   // (the octree ABI, step3.cu)
}

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(FC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)
#define NK(call)                                                                       \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess)                                                             \
      return fail(FC_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));       \
  } while (0)

struct DevList {
  int32_t* d = nullptr;
  int64_t nrec = 0;
};

// the ghost lists of one fill: the whole forest's, or (sub-cycling) the part a level-l fill needs
struct FillLists {
  DevList copy, avg, bcx, bcy, corner3;
  std::vector<DevList> interp, bcx_l, bcy_l;
  int32_t* d_snap = nullptr;           // (sub-cycling) the patches whose snapshot the fill reads
  int64_t n_snap = 0;
};

struct fc_forest {
  Plan pl;
  GhostLists gl;
  bool host_only = true;
  int device = -1;
  int64_t Pl = 0, Pv = 0;        // local patches, + virtual halo patches
  size_t state_doubles = 0;
  cudaStream_t stream = nullptr, own_stream = nullptr;
  double *qold = nullptr, *qnew = nullptr, *aux = nullptr;
  int8_t* d_level = nullptr;
  unsigned long long* d_cfl = nullptr;
  double* h_cfl = nullptr;
  DevList copy, avg, bcx, bcy, corner3;
  // halo overlap (NCCL halo on the fused path, several ranks): interior patches (no remote ring
  // source) are updated while the exchange runs on a high-priority comm stream; the boundary
  // patches after its event (SURVEY §8(e) "Overlap")
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_halo = nullptr;
  int32_t *d_ilist = nullptr, *d_blist = nullptr, *d_icnt = nullptr, *d_bcnt = nullptr;
  int64_t n_int = 0, n_bnd = 0;
  bool split = false;
  // fused ring gather (uniform same-level forests, one tile per patch): ring never written
  bool fused = false;
  int32_t* d_ring = nullptr;
  int32_t* d_nb9 = nullptr;   // regular rings: per local patch the 9 neighbour block offsets (plan_ring_regular)
  int quad = 0;               // m = 8, every local patch regular, complete sibling families 4b .. 4b+3
  uint8_t* d_bcflag = nullptr;
  // quiescent-patch filter (fused path): neighbour table, wall mask, flags, states, active list
  int32_t *d_nbr = nullptr, *d_active = nullptr, *d_nactive = nullptr;
  uint8_t *d_negmask = nullptr, *d_uflag = nullptr;
  double* d_uval = nullptr;
  int32_t h_nactive = 0;
  // adaptive quiescent filter: skipped (the full update runs; both are exact) while most patches
  // are active, re-probed every 16 steps
  int32_t* h_nact = nullptr;           // pinned: active patches of the last filtered step
  double active_frac = 0.0;
  int probe_countdown = 0;
  bool filtered_last = false;
  // coarse/fine reflux (built at the first fc_set_problem asking for it)
  bool reflux_planned = false;
  int32_t* d_rslot = nullptr;          // [Pl] flux-register slot or -1
  int32_t* d_rcells = nullptr;         // [ncells][RFX]
  int64_t nrcells = 0;
  double* d_freg = nullptr;            // [4 slots + remote faces][m][meqn] applied face fluxes (outward)
  int32_t nslots = 0;
  // reflux across rank cuts: fine faces requested from / served to other ranks (keys q * 4 + face)
  std::vector<std::vector<int64_t>> rf_req, rf_serve;
  std::vector<int32_t> h_rslot;
  int64_t rf_nremote = 0, rf_npack = 0;
  int32_t* d_rf_pack = nullptr;        // freg offsets (doubles) of the records this rank sends
  double* d_rf_send = nullptr;
  std::vector<int64_t> rf_send_off, rf_recv_off;   // [R + 1], doubles
  bool rf_ready = true;                // manual transport: false until fc_reflux_finalize
  // multi-rank regrid migration: old side (the blocks this rank sends, per new rank) and new side
  // (the staged old blocks this rank's new patches read, per old owner, and their source records)
  double* d_rg_send = nullptr;
  std::vector<int64_t> rg_send_off;    // [R + 1], doubles
  double* d_rg_stage = nullptr;
  std::vector<int64_t> rg_recv_off;    // [R + 1], doubles
  int32_t* d_rg_src = nullptr;
  bool rg_pending = false;
  std::vector<int64_t> rcell_off;      // reflux cells sorted by coarse level: [level - glmin] offsets
  // sub-cycling (fc_step_subcycled): levels [glmin, glmax] of the whole forest, per-level local lists
  int glmin = 0, glmax = 0;
  bool sub_ready = false;
  double *d_sub_old = nullptr, *d_sub_snap = nullptr, *d_facc = nullptr;
  std::vector<int32_t*> d_lvl;         // per level: local patch ids
  std::vector<int64_t> n_lvl;
  int32_t* d_lvl_cnt = nullptr;        // per level: count (device, for k_step's active list)
  int64_t sub_tick_old[32] = {}, sub_tick_new[32] = {};
  std::vector<FillLists> sub_fill;     // per level (single rank): restricted fills + snapshot lists
  const FillLists* fill_sel = nullptr; // when set, the ghost phases run these lists
  double sub_dt0 = 0.0;
  // fc_run: one CUDA graph per buffer parity for a fixed dt, the CFL history, a rollback copy
  cudaGraphExec_t run_exec[2] = {nullptr, nullptr};
  double run_dt = 0.0;
  double* d_hist = nullptr;
  int64_t hist_cap = 0;
  int64_t* d_hist_idx = nullptr;
  double* d_backup = nullptr;
  int64_t run_launches = 0;            // kernels per captured step
  std::vector<DevList> interp, bcx_l, bcy_l;
  fc_problem prob{};
  bool has_problem = false, has_q = false, has_aux = false;
  // peer-memory halo (halo_p2p, fused path): ring cells of other ranks read from their buffers
  bool p2p = false;
  uint8_t* d_rpeer = nullptr;          // [Pl][G] 0 = local, k = rank k-1, 255 = computed ghost
  bool amr_fused = false;              // fused ring gather on an AMR forest (computed ghosts)
  double* d_cg = nullptr;              // computed ghosts (AVG4 / INTERP ring cells), plan_ring_amr
  DevList cg_avg, cg_c3;
  std::vector<DevList> cg_interp;      // per level
  double* buf[2] = {nullptr, nullptr}; // this rank's two state buffers (q_old = buf[parity])
  int parity = 0;
  std::vector<std::array<double*, 2>> peer_buf;   // per rank: its two buffers mapped here
  std::vector<bool> peer_ipc;          // opened through CUDA IPC (closed on destroy)
  // halo
  ncclComm_t comm = nullptr;
  bool manual = false;                 // nranks > 1 without an NCCL id: the caller moves halo data
  std::vector<std::vector<int64_t>> peer_req[2];   // requests this rank serves, per round and peer
  // per round: concatenated pack / unpack index lists and per-peer counts
  int32_t *d_pack[2] = {nullptr, nullptr}, *d_unpack[2] = {nullptr, nullptr};
  int64_t npack[2] = {0, 0}, nunpack[2] = {0, 0};
  std::vector<int64_t> send_cnt[2], recv_cnt[2];
  double *d_sendbuf = nullptr, *d_recvbuf = nullptr;
  // instrumentation
  fc_stats st{};
  bool timing = false;
  bool capturing = false;              // run_capture: the graphs skip the host read of the active count
  cudaEvent_t ev[6] = {};
  bool copy_timed = false;             // ev[4] / ev[5] bracket the quiescent copy of this step
  // fc_step's timing events are read lazily (fc_get_stats): per step it only records events, so
  // the instrumented loop runs at the uninstrumented pace (elapsed-time queries after each step's
  // synchronisation kept the GPU idle: C5 0.92 -> 1.07 ms per step)
  struct PendingTiming { cudaEvent_t e[6]; bool copy; };
  std::vector<PendingTiming> t_pending;
  std::vector<cudaEvent_t> t_pool, t_all;
};

static int to_dev(fc_forest* f, const std::vector<int32_t>& v, int rec, DevList& out) {
  out.nrec = (int64_t)v.size() / rec;
  if (v.empty()) return FC_OK;
  CK(cudaMalloc(&out.d, v.size() * sizeof(int32_t)));
  CK(cudaMemcpy(out.d, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  (void)f;
  return FC_OK;
}

static void free_list(DevList& l) {
  if (l.d) cudaFree(l.d);
  l.d = nullptr;
}

// pack / unpack lists and buffers from the requests this rank serves (f->peer_req) and its own
// requests (pl.halo.need1/need2); shared by the NCCL and the manual transports
static int build_halo_lists(fc_forest* f) {
  Plan& pl = f->pl;
  const int R = pl.nranks;
  const int64_t n2 = (int64_t)pl.n * pl.n;
  const int64_t S = (int64_t)pl.meqn * n2;
  for (int round = 0; round < 2; ++round) {
    const auto& need = round == 0 ? pl.halo.need1 : pl.halo.need2;
    f->send_cnt[round].assign(R, 0);
    f->recv_cnt[round].assign(R, 0);
    std::vector<int32_t> pack, unpack;
    for (int s = 0; s < R; ++s) {
      f->recv_cnt[round][s] = (int64_t)need[s].size();
      f->send_cnt[round][s] = (int64_t)f->peer_req[round][s].size();
      for (int64_t key : f->peer_req[round][s]) {
        const int64_t q = key / n2, cell = key % n2;
        if (q < pl.p0 || q >= pl.p1) return fail(FC_EINVAL, "halo request for a patch this rank does not own");
        pack.push_back((int32_t)((q - pl.p0) * S + qcell_of_natural((int)cell, pl.n)));
      }
      for (int64_t key : need[s]) {   // my requests, in slot order
        const int64_t h = pl.halo.slot.at(key * 2 + round);
        unpack.push_back((int32_t)((f->Pl + h / n2) * S + h % n2));
      }
    }
    cudaFree(f->d_pack[round]);
    cudaFree(f->d_unpack[round]);
    f->d_pack[round] = f->d_unpack[round] = nullptr;
    f->npack[round] = (int64_t)pack.size();
    f->nunpack[round] = (int64_t)unpack.size();
    if (!pack.empty()) {
      CK(cudaMalloc(&f->d_pack[round], pack.size() * sizeof(int32_t)));
      CK(cudaMemcpy(f->d_pack[round], pack.data(), pack.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    if (!unpack.empty()) {
      CK(cudaMalloc(&f->d_unpack[round], unpack.size() * sizeof(int32_t)));
      CK(cudaMemcpy(f->d_unpack[round], unpack.data(), unpack.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
  }
  cudaFree(f->d_sendbuf);
  cudaFree(f->d_recvbuf);
  const int64_t maxs = std::max(f->npack[0], f->npack[1]), maxr = std::max(f->nunpack[0], f->nunpack[1]);
  CK(cudaMalloc(&f->d_sendbuf, std::max<int64_t>(1, maxs) * pl.meqn * sizeof(double)));
  CK(cudaMalloc(&f->d_recvbuf, std::max<int64_t>(1, maxr) * pl.meqn * sizeof(double)));
  f->st.halo_cells = f->nunpack[0] + f->nunpack[1];
  return FC_OK;
}

// one-time NCCL exchange of halo requests (counts all-gathered, then per-peer send/recv)
static int setup_halo(fc_forest* f, const void* nccl_id) {
  Plan& pl = f->pl;
  const int R = pl.nranks, me = pl.rank;
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  NK(ncclCommInitRank(&f->comm, R, id, me));
  std::vector<int64_t> mine(2 * R), all((size_t)2 * R * R);
  for (int s = 0; s < R; ++s) {
    mine[s] = (int64_t)pl.halo.need1[s].size();
    mine[R + s] = (int64_t)pl.halo.need2[s].size();
  }
  int64_t *d_mine = nullptr, *d_all = nullptr;
  CK(cudaMalloc(&d_mine, mine.size() * sizeof(int64_t)));
  CK(cudaMalloc(&d_all, all.size() * sizeof(int64_t)));
  CK(cudaMemcpy(d_mine, mine.data(), mine.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  NK(ncclAllGather(d_mine, d_all, 2 * R, ncclInt64, f->comm, f->stream));
  CK(cudaMemcpyAsync(all.data(), d_all, all.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(d_mine);
  cudaFree(d_all);
  for (int round = 0; round < 2; ++round) {
    const auto& need = round == 0 ? pl.halo.need1 : pl.halo.need2;
    std::vector<int64_t> cnt_in(R), off_out(R + 1, 0), off_in(R + 1, 0), req_out;
    for (int s = 0; s < R; ++s) {
      cnt_in[s] = all[(size_t)s * 2 * R + round * R + me];   // s needs from me
      off_out[s + 1] = off_out[s] + (int64_t)need[s].size();
      off_in[s + 1] = off_in[s] + cnt_in[s];
      req_out.insert(req_out.end(), need[s].begin(), need[s].end());
    }
    int64_t *d_out = nullptr, *d_in = nullptr;
    CK(cudaMalloc(&d_out, std::max<int64_t>(1, off_out[R]) * sizeof(int64_t)));
    CK(cudaMalloc(&d_in, std::max<int64_t>(1, off_in[R]) * sizeof(int64_t)));
    if (off_out[R])
      CK(cudaMemcpy(d_out, req_out.data(), off_out[R] * sizeof(int64_t), cudaMemcpyHostToDevice));
    NK(ncclGroupStart());
    for (int s = 0; s < R; ++s) {
      if (s == me) continue;
      if (need[s].size()) NK(ncclSend(d_out + off_out[s], need[s].size(), ncclInt64, s, f->comm, f->stream));
      if (cnt_in[s]) NK(ncclRecv(d_in + off_in[s], cnt_in[s], ncclInt64, s, f->comm, f->stream));
    }
    NK(ncclGroupEnd());
    CK(cudaStreamSynchronize(f->stream));
    std::vector<int64_t> req_in(off_in[R]);
    if (off_in[R]) CK(cudaMemcpy(req_in.data(), d_in, off_in[R] * sizeof(int64_t), cudaMemcpyDeviceToHost));
    cudaFree(d_out);
    cudaFree(d_in);
    f->peer_req[round].assign(R, {});
    for (int s = 0; s < R; ++s) f->peer_req[round][s].assign(req_in.begin() + off_in[s], req_in.begin() + off_in[s + 1]);
  }
  return build_halo_lists(f);
}

// peer-memory halo over NCCL ranks: all-gather the CUDA IPC handles of every rank's two state
// buffers, open the other ranks' (peer access over NVLink), then an allreduce as a barrier
static int setup_p2p_ipc(fc_forest* f) {
  const int R = f->pl.nranks, me = f->pl.rank;
  cudaIpcMemHandle_t mine[2];
  CK(cudaIpcGetMemHandle(&mine[0], f->buf[0]));
  CK(cudaIpcGetMemHandle(&mine[1], f->buf[1]));
  const size_t hb = sizeof(mine);
  char *d_mine = nullptr, *d_all = nullptr;
  CK(cudaMalloc(&d_mine, hb));
  CK(cudaMalloc(&d_all, hb * R));
  CK(cudaMemcpy(d_mine, mine, hb, cudaMemcpyHostToDevice));
  NK(ncclAllGather(d_mine, d_all, hb, ncclUint8, f->comm, f->stream));
  std::vector<cudaIpcMemHandle_t> all(2 * R);
  CK(cudaMemcpyAsync(all.data(), d_all, hb * R, cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(d_mine);
  cudaFree(d_all);
  for (int r = 0; r < R; ++r) {
    if (r == me) continue;
    for (int b = 0; b < 2; ++b) {
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, all[2 * r + b], cudaIpcMemLazyEnablePeerAccess));
      f->peer_buf[r][b] = (double*)p;
    }
    f->peer_ipc[r] = true;
  }
  return FC_OK;
}

// ---- halo transfer pieces (round: 0 = interior cells, 1 = ring cells read by interpolation) ----
static int halo_pack(fc_forest* f, int round, cudaStream_t st) {
  f->st.kernel_launches += launch_pack(f->qold, f->d_pack[round], f->npack[round], f->pl.meqn,
                                       f->pl.n * f->pl.n, f->d_sendbuf, st);
  CK(cudaGetLastError());
  return FC_OK;
}
static int halo_unpack(fc_forest* f, int round, cudaStream_t st) {
  f->st.kernel_launches += launch_unpack(f->qold, f->d_unpack[round], f->nunpack[round], f->pl.meqn,
                                         f->pl.n * f->pl.n, f->d_recvbuf, st);
  CK(cudaGetLastError());
  return FC_OK;
}
static int halo_nccl(fc_forest* f, int round, cudaStream_t st) {
  const int R = f->pl.nranks, me = f->pl.rank, meqn = f->pl.meqn;
  NK(ncclGroupStart());
  int64_t so = 0, ro = 0;
  for (int s = 0; s < R; ++s) {
    const int64_t sc = f->send_cnt[round][s], rc = f->recv_cnt[round][s];
    if (s != me && sc) NK(ncclSend(f->d_sendbuf + so * meqn, sc * meqn, ncclDouble, s, f->comm, st));
    if (s != me && rc) NK(ncclRecv(f->d_recvbuf + ro * meqn, rc * meqn, ncclDouble, s, f->comm, st));
    so += sc;
    ro += rc;
  }
  NK(ncclGroupEnd());
  return FC_OK;
}

// one NCCL halo round (pack -> grouped send/recv -> unpack); no-op on one rank
static int halo_round(fc_forest* f, int round, cudaStream_t st = nullptr) {
  if (f->pl.nranks <= 1) return FC_OK;
  if (f->manual) return fail(FC_ESTATE, "manual halo transport: use the staged step calls");
  if (!st) st = f->stream;
  int rc;
  if ((rc = halo_pack(f, round, st)) || (rc = halo_nccl(f, round, st)) || (rc = halo_unpack(f, round, st))) return rc;
  return FC_OK;
}

static bool has_round2(const fc_forest* f) { return f->npack[1] || f->nunpack[1]; }

// the fused ring gather (no ring writes): default mode, and the full-update mode for constant-
// velocity advection (measured: T1 full 1.00 -> 0.67 ms, T2 0.27 -> 0.22 ms; for Euler the gather
// of every patch's ring in the 352-thread k_step costs more than the ghost kernels: C5 full 9.5 ->
// 10.3 ms).  FC_FUSED_RING=0 at creation keeps the ghost kernels; the capacity form always does.
// systems whose update the warp-sweep kernel takes (step_ws.cu): it gathers its windows itself,
// so their full-update mode runs on the fused path too (FC_WS=0: the phased k_step + ghost kernels)
static bool ws_applies(const fc_forest* f) {
  const char* env = getenv("FC_WS");
  return !(env && atoi(env) == 0) && (f->prob.kind == FC_SWE_ROE || f->prob.kind == FC_EULER_ROE) && f->pl.m % 16 == 0 &&
         !f->prob.reflux;
}

static bool use_fused(const fc_forest* f) {
  if (!f->fused) return false;
  if (f->prob.kind == FC_ADV_EDGEVEL_CAPA)   // (aux staging of the fused multi-tile windows: not built)
    return (f->pl.m == 16 || f->pl.m == 8) && (std::getenv("FC_FUSED_CAPA") == nullptr || std::atoi(std::getenv("FC_FUSED_CAPA")) != 0);
  return f->prob.skip_quiescent || f->prob.kind == FC_ADV_CONST || ws_applies(f);
}

static void run_ghost(fc_forest* f, int op, const DevList& l) {
  f->st.kernel_launches += launch_ghost(op, f->qold, l.d, l.nrec, f->pl.meqn, f->pl.n * f->pl.n, f->stream);
}

// ghost phases that only need halo round 1: A (copy, average) -> C (BC x then y)
static int ghost_phase_ac(fc_forest* f) {
  const FillLists* s = f->fill_sel;
  run_ghost(f, OP_COPY, s ? s->copy : f->copy);
  run_ghost(f, OP_AVG4, s ? s->avg : f->avg);
  run_ghost(f, 4, s ? s->bcx : f->bcx);
  run_ghost(f, 4, s ? s->bcy : f->bcy);
  CK(cudaGetLastError());
  return FC_OK;
}

// ghost phases after halo round 2: per level B (interpolate) -> C, then CORNER3
static int ghost_phase_b(fc_forest* f) {
  const FillLists* s = f->fill_sel;
  const auto& interp = s ? s->interp : f->interp;
  const auto& bcx_l = s ? s->bcx_l : f->bcx_l;
  const auto& bcy_l = s ? s->bcy_l : f->bcy_l;
  for (size_t l = 0; l < interp.size(); ++l) {
    if (!interp[l].nrec) continue;
    run_ghost(f, OP_INTERP, interp[l]);
    run_ghost(f, 4, bcx_l[l]);
    run_ghost(f, 4, bcy_l[l]);
  }
  run_ghost(f, 6, s ? s->corner3 : f->corner3);
  CK(cudaGetLastError());
  return FC_OK;
}

static int ghost_fill_internal(fc_forest* f) {
  int rc;
  if ((rc = halo_round(f, 0)) || (rc = ghost_phase_ac(f))) return rc;
  if (has_round2(f) && (rc = halo_round(f, 1))) return rc;
  return ghost_phase_b(f);
}

// coarse cells next to finer faces: applied flux -> mean of the fine fluxes
static int apply_reflux(fc_forest* f, double dt) {
  if (f->nrcells <= 0) return FC_OK;
  f->st.kernel_launches += launch_reflux(f->d_rcells, f->nrcells, f->d_freg, f->d_freg, f->qnew, f->aux, f->d_level,
                                         1.0, dt, f->pl.dx0, f->pl.meqn, f->pl.n * f->pl.n, f->stream);
  CK(cudaGetLastError());
  return FC_OK;
}

// pack the fine-face records other ranks requested; with NCCL send them and receive this rank's
// requests straight into the remote-face region of freg (the manual transport moves them itself)
static int reflux_exchange(fc_forest* f) {
  const int R = f->pl.nranks, me = f->pl.rank;
  const int64_t rec = (int64_t)f->pl.m * f->pl.meqn;
  if (f->rf_npack) {
    f->st.kernel_launches += launch_pack(f->d_freg, f->d_rf_pack, f->rf_npack, 1, 0, f->d_rf_send, f->stream);
    CK(cudaGetLastError());
  }
  if (f->manual) return FC_OK;
  double* remote = f->d_freg + 4 * (int64_t)f->nslots * rec;
  NK(ncclGroupStart());
  for (int s = 0; s < R; ++s) {
    if (s == me) continue;
    const int64_t ns = f->rf_send_off[s + 1] - f->rf_send_off[s], nr = f->rf_recv_off[s + 1] - f->rf_recv_off[s];
    if (ns) NK(ncclSend(f->d_rf_send + f->rf_send_off[s], ns, ncclDouble, s, f->comm, f->stream));
    if (nr) NK(ncclRecv(remote + f->rf_recv_off[s], nr, ncclDouble, s, f->comm, f->stream));
  }
  NK(ncclGroupEnd());
  return FC_OK;
}

// the update after the ghost data are in place: quiescent filter (fused path) + step kernel,
// leaving this rank's CFL max in d_cfl
// the split update applies on the fused NCCL-halo path when no quiescent filter and no reflux
// records are involved (the filter's active list and the records span both patch classes)
static bool overlap_ok(const fc_forest* f) {
  if (!f->split || !use_fused(f) || f->prob.reflux || has_round2(f)) return false;
  const bool want_filter = f->prob.skip_quiescent && f->prob.kind != FC_ADV_EDGEVEL_CAPA && f->Pl >= 512;
  return !want_filter;
}

// part: 0 every local patch; 1 the interior patches only (no remote ring source: may run before
// the halo arrives; resets the CFL); 2 the boundary patches (after the halo; keeps the CFL)
static int update_local(fc_forest* f, double dt, int part = 0) {
  if (part != 2) CK(cudaMemsetAsync(f->d_cfl, 0, sizeof(unsigned long long), f->stream));
  const fc_problem& p = f->prob;
  const bool fused = use_fused(f);
  if (part != 0) {   // split update (halo overlap): fused path, no filter, no reflux records
    const int32_t* lst = part == 1 ? f->d_ilist : f->d_blist;
    const int32_t* cnt = part == 1 ? f->d_icnt : f->d_bcnt;
    if ((part == 1 ? f->n_int : f->n_bnd) == 0) return FC_OK;
    std::array<const double*, 16> pq{};
    int lr = launch_step(p.kind, f->qold, f->qnew, f->aux, f->d_level, f->Pl, f->pl.m, dt, f->pl.dx0, p.p0, p.p1,
                         p.limiter, p.method2, p.method3, p.skip_quiescent, f->d_ring, f->d_nb9, f->d_bcflag, lst, cnt,
                         f->d_cfl, nullptr, nullptr, nullptr, pq.data(), f->d_cg, f->stream);
    if (lr < 0) return fail(FC_EUNSUP, "no step kernel for this m / kind");
    f->st.kernel_launches += lr;
    f->st.step_kernel_launches += lr;
    CK(cudaGetLastError());
    return FC_OK;
  }
  const bool reflux = p.reflux && f->nrcells > 0;          // this rank applies corrections
  const bool records = p.reflux && (f->nrcells > 0 || f->rf_npack > 0);   // and / or serves records
  if (p.reflux && !f->rf_ready) return fail(FC_ESTATE, "reflux requests not finalized (fc_reflux_finalize)");
  std::array<const double*, 16> peerq{};   // peers' current q_old (peer-memory halo)
  if (fused && f->p2p) {
    if (f->pl.nranks > 16) return fail(FC_EUNSUP, "peer-memory halo supports at most 16 ranks");
    for (int r = 0; r < f->pl.nranks; ++r) peerq[r] = f->peer_buf[r][f->parity];
  }
  if (fused && f->amr_fused) {   // computed ghosts of the AMR ring gather: averages, then per level
    const int n2 = f->pl.n * f->pl.n;
    f->st.kernel_launches += launch_cg(2, f->qold, f->d_cg, f->cg_avg.d, f->cg_avg.nrec, f->pl.meqn, n2, f->stream);
    for (auto& l : f->cg_interp)
      f->st.kernel_launches += launch_cg(3, f->qold, f->d_cg, l.d, l.nrec, f->pl.meqn, n2, f->stream);
    f->st.kernel_launches += launch_cg(6, f->qold, f->d_cg, f->cg_c3.d, f->cg_c3.nrec, f->pl.meqn, n2, f->stream);
    CK(cudaGetLastError());
  }
  bool filtered = false;
  // (tiny forests skip the filter: its two extra launches cost more than the tiles they save; the
  // step kernel's own quiescent-window check still applies)
  f->filtered_last = false;
  const bool want_filter = p.skip_quiescent && p.kind != FC_ADV_EDGEVEL_CAPA && f->Pl >= 512;
  const bool probe = f->probe_countdown <= 0;
  if (want_filter && !(f->active_frac >= 0.75 && !probe)) {
    // copy/classify + activity filter, then the step over the active patches' tiles only
    CK(cudaMemsetAsync(f->d_nactive, 0, sizeof(int32_t), f->stream));
    static const bool env_tc = !(getenv("FC_TIME_COPY") && atoi(getenv("FC_TIME_COPY")) == 0);
    const bool time_copy = f->timing && env_tc;
    const int fr = launch_filter(p.kind, f->qold, f->qnew, (int)f->Pl, f->pl.m, f->d_uflag, f->d_uval, f->d_nbr,
                                 f->d_negmask, f->d_level, dt, f->pl.dx0, p.p0, p.p1, f->d_active, f->d_nactive,
                                 f->d_cfl, f->stream, time_copy ? f->ev[4] : nullptr, time_copy ? f->ev[5] : nullptr);
    if (fr > 0) {
      f->st.kernel_launches += fr;
      filtered = true;
      f->copy_timed = time_copy;
    }
  } else if (want_filter) {
    f->probe_countdown -= 1;
  }
  int lr = launch_step(p.kind, f->qold, f->qnew, f->aux, f->d_level, f->Pl, f->pl.m, dt, f->pl.dx0,
                       p.p0, p.p1, p.limiter, p.method2, p.method3, filtered ? 0 : p.skip_quiescent,
                       fused ? f->d_ring : nullptr, f->d_nb9, f->d_bcflag, filtered ? f->d_active : nullptr,
                       filtered ? f->d_nactive : nullptr, f->d_cfl, records ? f->d_rslot : nullptr,
                       records ? f->d_freg : nullptr, (fused && (f->p2p || f->amr_fused)) ? f->d_rpeer : nullptr,
                       peerq.data(), f->d_cg, f->stream, fused ? f->quad : 0);
  if (lr < 0) return fail(FC_EUNSUP, "no step kernel for this m / kind");
  f->st.kernel_launches += lr;
  f->st.step_kernel_launches += lr;
  CK(cudaGetLastError());
  if (filtered && !f->capturing) {   // active count for the adaptive filter (read after the step's sync)
    CK(cudaMemcpyAsync(f->h_nact, f->d_nactive, sizeof(int32_t), cudaMemcpyDeviceToHost, f->stream));
    f->filtered_last = true;
  }
  if (p.reflux && f->pl.nranks > 1) {   // fine-face records for other ranks' coarse cells
    int rc = reflux_exchange(f);
    if (rc) return rc;
  }
  if (reflux && !f->manual) return apply_reflux(f, dt);   // (manual transport: fc_step_local phase 3)
  return FC_OK;
}

// after a step's stream synchronisation: the active fraction seen by the quiescent filter
static void note_activity(fc_forest* f) {
  if (!f->filtered_last) return;
  f->active_frac = f->Pl > 0 ? (double)*f->h_nact / (double)f->Pl : 0.0;
  if (f->active_frac >= 0.75) f->probe_countdown = 16;
  f->filtered_last = false;
}

static int check_step_args(fc_forest* f, double dt) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (f->host_only || !f->has_q || !f->has_problem) return fail(FC_ESTATE, "set problem and q first");
  if (f->pl.maux > 0 && !f->has_aux) return fail(FC_ESTATE, "set aux first");
  if (!(dt > 0.0) || !std::isfinite(dt)) return fail(FC_EINVAL, "dt must be positive and finite");
  return FC_OK;
}

// commit rule shared by fc_step and fc_commit
static int commit(fc_forest* f, double cfl) {
  if (!std::isfinite(cfl)) return fail(FC_ENONFINITE, "CFL is not finite");
  if (cfl > f->prob.cfl_reject) return fail(FC_ECFL, "CFL above cfl_reject; step not committed");
  std::swap(f->qold, f->qnew);
  f->parity ^= 1;
  f->st.steps += 1;
  return FC_OK;
}

static void destroy(fc_forest* f) {
  if (!f) return;
  if (!f->host_only) {
    cudaSetDevice(f->device);
    if (f->stream) cudaStreamSynchronize(f->stream);
    cudaFree(f->qold); cudaFree(f->qnew); cudaFree(f->aux); cudaFree(f->d_level); cudaFree(f->d_cfl);
    cudaFree(f->d_ring); cudaFree(f->d_nb9); cudaFree(f->d_bcflag);
    cudaFree(f->d_nbr); cudaFree(f->d_active); cudaFree(f->d_nactive); cudaFree(f->d_negmask);
    cudaFree(f->d_uflag); cudaFree(f->d_uval);
    cudaFree(f->d_rslot); cudaFree(f->d_rcells); cudaFree(f->d_freg);
    cudaFree(f->d_rf_pack); cudaFree(f->d_rf_send);
    cudaFree(f->d_rg_send); cudaFree(f->d_rg_stage); cudaFree(f->d_rg_src);
    cudaFree(f->d_rpeer);
    cudaFree(f->d_cg);
    free_list(f->cg_avg);
    free_list(f->cg_c3);
    for (auto& l : f->cg_interp) free_list(l);
    for (auto& g : f->run_exec) if (g) cudaGraphExecDestroy(g);
    cudaFree(f->d_hist); cudaFree(f->d_hist_idx); cudaFree(f->d_backup);
    for (size_t r = 0; r < f->peer_ipc.size(); ++r)
      if (f->peer_ipc[r])
        for (double* p : f->peer_buf[r]) if (p) cudaIpcCloseMemHandle(p);
    cudaFree(f->d_sub_old); cudaFree(f->d_sub_snap); cudaFree(f->d_facc); cudaFree(f->d_lvl_cnt);
    for (auto* d : f->d_lvl) cudaFree(d);
    for (auto& s : f->sub_fill) {
      free_list(s.copy); free_list(s.avg); free_list(s.bcx); free_list(s.bcy); free_list(s.corner3);
      for (auto& l : s.interp) free_list(l);
      for (auto& l : s.bcx_l) free_list(l);
      for (auto& l : s.bcy_l) free_list(l);
      cudaFree(s.d_snap);
    }
    if (f->h_cfl) cudaFreeHost(f->h_cfl);
    if (f->h_nact) cudaFreeHost(f->h_nact);
    free_list(f->copy); free_list(f->avg); free_list(f->bcx); free_list(f->bcy); free_list(f->corner3);
    for (auto& l : f->interp) free_list(l);
    for (auto& l : f->bcx_l) free_list(l);
    for (auto& l : f->bcy_l) free_list(l);
    for (int r = 0; r < 2; ++r) { cudaFree(f->d_pack[r]); cudaFree(f->d_unpack[r]); }
    cudaFree(f->d_sendbuf); cudaFree(f->d_recvbuf);
    for (auto& e : f->t_all) cudaEventDestroy(e);
    if (f->comm) ncclCommDestroy(f->comm);
    cudaFree(f->d_ilist); cudaFree(f->d_blist); cudaFree(f->d_icnt); cudaFree(f->d_bcnt);
    if (f->ev_fork) cudaEventDestroy(f->ev_fork);
    if (f->ev_halo) cudaEventDestroy(f->ev_halo);
    if (f->comm_stream) cudaStreamDestroy(f->comm_stream);
    if (f->own_stream) cudaStreamDestroy(f->own_stream);
  }
  delete f;
}

// regular-ring neighbour offsets of the fused gather (plan_ring_regular; FC_REGULAR_RING=0: off)
static int upload_regular(fc_forest* f, const RingSources& rs) {
  const char* env = getenv("FC_REGULAR_RING");
  if (env && atoi(env) == 0) return FC_OK;
  std::vector<int32_t> nb9;
  const int64_t nreg = plan_ring_regular(f->pl, f->pl.meqn, rs, nb9);
  f->st.regular_patches = nreg;
  f->st.quad_blocks = 0;
  f->quad = 0;
  if (nreg == 0) return FC_OK;
  {   // quad blocks for the scalar sweep (cv_stage_quad): every local patch regular and the local
      // list made of whole sibling families in Morton order (FC_CV_QUAD=0: off)
    const char* qe = getenv("FC_CV_QUAD");
    const int64_t Pl = f->pl.p1 - f->pl.p0;
    bool ok = !(qe && atoi(qe) == 0) && f->pl.m == 8 && f->pl.meqn == 1 && nreg == Pl && Pl % 4 == 0;
    for (int64_t b = 0; ok && b < Pl / 4; ++b) {
      const Leaf& l0 = f->pl.leaves[f->pl.p0 + 4 * b];
      const int64_t sz = (int64_t)1 << (f->pl.lmax - l0.level);
      if (l0.level == 0 || (l0.x / sz) % 2 != 0 || (l0.y / sz) % 2 != 0) { ok = false; break; }
      for (int c = 1; c < 4 && ok; ++c) {
        const Leaf& l = f->pl.leaves[f->pl.p0 + 4 * b + c];
        ok = l.tree == l0.tree && l.level == l0.level && l.x == l0.x + sz * (c & 1) && l.y == l0.y + sz * (c >> 1);
      }
    }
    f->quad = ok ? 1 : 0;
    f->st.quad_blocks = ok ? Pl / 4 : 0;
  }
  cudaError_t e = cudaMalloc(&f->d_nb9, nb9.size() * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemcpy(f->d_nb9, nb9.data(), nb9.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    std::string m = std::string("regular ring table: ") + cudaGetErrorString(e);
    destroy(f);
    return fail(FC_ECUDA, m);
  }
  return FC_OK;
}

// accumulate the pending fc_step timing events into the stats and recycle them
static void timing_drain(fc_forest* f) {
  for (auto& p : f->t_pending) {
    float a = 0.f, b = 0.f, c = 0.f;
    cudaEventElapsedTime(&a, p.e[0], p.e[1]);
    cudaEventElapsedTime(&b, p.e[1], p.e[2]);
    cudaEventElapsedTime(&c, p.e[2], p.e[3]);
    f->st.ms_ghost += a;
    f->st.ms_step += b;
    f->st.ms_comm += c;
    if (p.copy) {
      float d = 0.f;
      cudaEventElapsedTime(&d, p.e[4], p.e[5]);
      f->st.ms_copy += d;
      f->st.copy_launches += 1;
    }
    for (int k = 0; k < 6; ++k) f->t_pool.push_back(p.e[k]);
  }
  f->t_pending.clear();
}

// reflux across rank cuts: pack list (freg offsets of the served records) and the per-peer send /
// receive offsets, from rf_serve (requests this rank serves) and rf_req (its own requests)
static int build_reflux_lists(fc_forest* f) {
  const int R = f->pl.nranks;
  const int64_t rec = (int64_t)f->pl.m * f->pl.meqn;
  std::vector<int32_t> pack;
  f->rf_send_off.assign(R + 1, 0);
  f->rf_recv_off.assign(R + 1, 0);
  for (int s = 0; s < R; ++s) {
    for (int64_t key : f->rf_serve[s]) {
      const int64_t q = key / 4, face = key % 4;
      if (q < f->pl.p0 || q >= f->pl.p1) return fail(FC_EINVAL, "reflux request for a patch this rank does not own");
      const int32_t slot = f->h_rslot[q - f->pl.p0];
      if (slot < 0) return fail(FC_EINVAL, "reflux request for a patch without flux records");
      for (int64_t e = 0; e < rec; ++e) pack.push_back((int32_t)((slot * 4 + face) * rec + e));
    }
    f->rf_send_off[s + 1] = (int64_t)pack.size();
    f->rf_recv_off[s + 1] = f->rf_recv_off[s] + (int64_t)f->rf_req[s].size() * rec;
  }
  cudaFree(f->d_rf_pack);
  cudaFree(f->d_rf_send);
  f->d_rf_pack = nullptr;
  f->d_rf_send = nullptr;
  f->rf_npack = (int64_t)pack.size();
  CK(cudaMalloc(&f->d_rf_send, std::max<int64_t>(1, f->rf_npack) * sizeof(double)));
  if (f->rf_npack) {
    CK(cudaMalloc(&f->d_rf_pack, pack.size() * sizeof(int32_t)));
    CK(cudaMemcpy(f->d_rf_pack, pack.data(), pack.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  f->rf_ready = true;
  return FC_OK;
}

// one-time NCCL exchange of the reflux requests (counts all-gathered, then per-peer send/recv)
static int reflux_exchange_requests(fc_forest* f) {
  const int R = f->pl.nranks, me = f->pl.rank;
  std::vector<int64_t> mine(R), all((size_t)R * R);
  for (int s = 0; s < R; ++s) mine[s] = (int64_t)f->rf_req[s].size();
  int64_t *d_mine = nullptr, *d_all = nullptr;
  CK(cudaMalloc(&d_mine, R * sizeof(int64_t)));
  CK(cudaMalloc(&d_all, all.size() * sizeof(int64_t)));
  CK(cudaMemcpy(d_mine, mine.data(), R * sizeof(int64_t), cudaMemcpyHostToDevice));
  NK(ncclAllGather(d_mine, d_all, R, ncclInt64, f->comm, f->stream));
  CK(cudaMemcpyAsync(all.data(), d_all, all.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(d_mine);
  cudaFree(d_all);
  std::vector<int64_t> off_out(R + 1, 0), off_in(R + 1, 0), out;
  for (int s = 0; s < R; ++s) {
    off_out[s + 1] = off_out[s] + (int64_t)f->rf_req[s].size();
    off_in[s + 1] = off_in[s] + all[(size_t)s * R + me];
    out.insert(out.end(), f->rf_req[s].begin(), f->rf_req[s].end());
  }
  int64_t *d_out = nullptr, *d_in = nullptr;
  CK(cudaMalloc(&d_out, std::max<int64_t>(1, off_out[R]) * sizeof(int64_t)));
  CK(cudaMalloc(&d_in, std::max<int64_t>(1, off_in[R]) * sizeof(int64_t)));
  if (off_out[R]) CK(cudaMemcpy(d_out, out.data(), off_out[R] * sizeof(int64_t), cudaMemcpyHostToDevice));
  NK(ncclGroupStart());
  for (int s = 0; s < R; ++s) {
    if (s == me) continue;
    if (off_out[s + 1] > off_out[s]) NK(ncclSend(d_out + off_out[s], off_out[s + 1] - off_out[s], ncclInt64, s, f->comm, f->stream));
    if (off_in[s + 1] > off_in[s]) NK(ncclRecv(d_in + off_in[s], off_in[s + 1] - off_in[s], ncclInt64, s, f->comm, f->stream));
  }
  NK(ncclGroupEnd());
  CK(cudaStreamSynchronize(f->stream));
  std::vector<int64_t> in(off_in[R]);
  if (off_in[R]) CK(cudaMemcpy(in.data(), d_in, off_in[R] * sizeof(int64_t), cudaMemcpyDeviceToHost));
  cudaFree(d_out);
  cudaFree(d_in);
  f->rf_serve.assign(R, {});
  for (int s = 0; s < R; ++s) f->rf_serve[s].assign(in.begin() + off_in[s], in.begin() + off_in[s + 1]);
  return build_reflux_lists(f);
}

extern "C" {

const char* fc_last_error(void) { return g_err.c_str(); }

int fc_nccl_unique_id(void* out) {
  if (!out) return fail(FC_EINVAL, "null output");
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return FC_OK;
}

int fc_forest_create(const fc_forest_desc* d, fc_forest** out) {
  if (!out) return fail(FC_EINVAL, "null output handle");
  *out = nullptr;
  fc_forest* f = new (std::nothrow) fc_forest();
  if (!f) return fail(FC_ENOMEM, "host allocation failed");
  std::string err;
  int rc = plan_build(d, f->pl, err);
  if (rc) { delete f; return fail(rc, err); }
  f->Pl = f->pl.p1 - f->pl.p0;
  f->st.local_patches = f->Pl;
  f->glmin = 127;
  f->glmax = -1;
  for (const Leaf& L : f->pl.leaves) {   // levels of the whole forest (same on every rank)
    f->glmin = std::min(f->glmin, (int)L.level);
    f->glmax = std::max(f->glmax, (int)L.level);
  }
  f->st.uniform_fast_path = 0;
  if (d->device < 0) {           // host-only planning handle: tables and plans, no device work
    f->host_only = true;
    *out = f;
    return FC_OK;
  }
  f->manual = d->nranks > 1 && !d->nccl_id;   // no NCCL id: the caller transports halo data
  f->host_only = false;
  f->device = d->device;
  const Plan& pl = f->pl;
  const int64_t n2 = (int64_t)pl.n * pl.n;
  auto cuda_fail = [&](cudaError_t e, const char* what) {
    std::string m = std::string(what) + ": " + cudaGetErrorString(e);
    destroy(f);
    return fail(e == cudaErrorMemoryAllocation ? FC_ENOMEM : FC_ECUDA, m);
  };
  cudaError_t e;
  if ((e = cudaSetDevice(f->device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  if ((e = cudaStreamCreateWithFlags(&f->own_stream, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_fail(e, "cudaStreamCreate");
  f->stream = f->own_stream;
  const int64_t nhalo = pl.halo.n1 + pl.halo.n2;
  f->Pv = (nhalo + n2 - 1) / n2;
  // (at least one block: an empty rank still has mappable buffers for the peer-memory halo)
  f->state_doubles = (size_t)std::max<int64_t>(1, f->Pl + f->Pv) * pl.meqn * n2;
  if ((e = cudaMalloc(&f->qold, f->state_doubles * sizeof(double))) != cudaSuccess) return cuda_fail(e, "cudaMalloc q_old");
  if ((e = cudaMalloc(&f->qnew, f->state_doubles * sizeof(double))) != cudaSuccess) return cuda_fail(e, "cudaMalloc q_new");
  f->buf[0] = f->qold;
  f->buf[1] = f->qnew;
  cudaMemset(f->qold, 0, f->state_doubles * sizeof(double));
  cudaMemset(f->qnew, 0, f->state_doubles * sizeof(double));
  if (pl.maux > 0) {
    if ((e = cudaMalloc(&f->aux, (size_t)f->Pl * pl.maux * n2 * sizeof(double))) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc aux");
  }
  std::vector<int8_t> lv(f->Pl);
  for (int64_t p = 0; p < f->Pl; ++p) lv[p] = (int8_t)pl.leaves[pl.p0 + p].level;
  if ((e = cudaMalloc(&f->d_level, std::max<int64_t>(1, f->Pl))) != cudaSuccess) return cuda_fail(e, "cudaMalloc level");
  cudaMemcpy(f->d_level, lv.data(), f->Pl, cudaMemcpyHostToDevice);
  if ((e = cudaMalloc(&f->d_cfl, sizeof(unsigned long long))) != cudaSuccess) return cuda_fail(e, "cudaMalloc cfl");
  if ((e = cudaMallocHost(&f->h_cfl, sizeof(double))) != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
  if ((e = cudaMallocHost(&f->h_nact, sizeof(int32_t))) != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
  for (auto& ev : f->ev) {
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    f->t_all.push_back(ev);            // (every event the handle owns, destroyed once)
  }
  rc = plan_lists(f->pl, pl.meqn, f->gl, err);
  if (rc) { destroy(f); return fail(rc, err); }
  if ((rc = to_dev(f, f->gl.copy, 2, f->copy)) || (rc = to_dev(f, f->gl.avg, 5, f->avg)) ||
      (rc = to_dev(f, f->gl.bcx, 3, f->bcx)) || (rc = to_dev(f, f->gl.bcy, 3, f->bcy)) ||
      (rc = to_dev(f, f->gl.corner3, 3, f->corner3))) {
    std::string m = g_err;
    destroy(f);
    return fail(rc, m);
  }
  f->interp.resize(f->gl.interp.size());
  f->bcx_l.resize(f->gl.interp.size());
  f->bcy_l.resize(f->gl.interp.size());
  for (size_t l = 0; l < f->gl.interp.size(); ++l) {
    if ((rc = to_dev(f, f->gl.interp[l], 8, f->interp[l])) || (rc = to_dev(f, f->gl.bcx_l[l], 3, f->bcx_l[l])) ||
        (rc = to_dev(f, f->gl.bcy_l[l], 3, f->bcy_l[l]))) {
      std::string m = g_err;
      destroy(f);
      return fail(rc, m);
    }
  }
  // fused ring gather: every ghost record COPY/BC and one 2-tile-free patch per tile (m <= 16)
  {
    const int T = (pl.m % 16 == 0) ? 16 : ((pl.m % 8 == 0) ? 8 : ((pl.m % 4 == 0) ? 4 : 2));
    const char* env = getenv("FC_FUSED_RING");
    const bool allow = !env || atoi(env) != 0;
    if (allow && pl.uniform_same && pl.m % T == 0) {   // (multi-tile patches: gather_ring_tiles)
      RingSources rs;
      f->p2p = d->halo_p2p != 0 && pl.nranks > 1;
      rc = plan_ring_sources(f->pl, pl.meqn, rs, err, f->p2p);
      if (rc) { destroy(f); return fail(rc, err); }
      if (f->p2p) {
        if ((e = cudaMalloc(&f->d_rpeer, rs.peer.size())) != cudaSuccess) return cuda_fail(e, "cudaMalloc ring peers");
        cudaMemcpy(f->d_rpeer, rs.peer.data(), rs.peer.size(), cudaMemcpyHostToDevice);
        f->peer_buf.assign(pl.nranks, {nullptr, nullptr});
        f->peer_ipc.assign(pl.nranks, false);
      }
      if ((e = cudaMalloc(&f->d_ring, rs.src.size() * sizeof(int32_t))) != cudaSuccess) return cuda_fail(e, "cudaMalloc ring");
      if ((e = cudaMalloc(&f->d_bcflag, std::max<size_t>(1, rs.bcflag.size()))) != cudaSuccess) return cuda_fail(e, "cudaMalloc bcflag");
      cudaMemcpy(f->d_ring, rs.src.data(), rs.src.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
      cudaMemcpy(f->d_bcflag, rs.bcflag.data(), rs.bcflag.size(), cudaMemcpyHostToDevice);
      const size_t Pl1 = std::max<int64_t>(1, f->Pl);
      if ((e = cudaMalloc(&f->d_nbr, Pl1 * 8 * sizeof(int32_t))) != cudaSuccess ||
          (e = cudaMalloc(&f->d_active, Pl1 * sizeof(int32_t))) != cudaSuccess ||
          (e = cudaMalloc(&f->d_nactive, sizeof(int32_t))) != cudaSuccess ||
          (e = cudaMalloc(&f->d_negmask, Pl1)) != cudaSuccess || (e = cudaMalloc(&f->d_uflag, Pl1)) != cudaSuccess ||
          (e = cudaMalloc(&f->d_uval, Pl1 * pl.meqn * sizeof(double))) != cudaSuccess)
        return cuda_fail(e, "cudaMalloc filter");
      cudaMemcpy(f->d_nbr, rs.nbr.data(), rs.nbr.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
      cudaMemcpy(f->d_negmask, rs.negmask.data(), rs.negmask.size(), cudaMemcpyHostToDevice);
      if ((rc = upload_regular(f, rs))) return rc;
      f->fused = true;
      f->st.uniform_fast_path = 1;
      if (pl.nranks > 1 && !f->p2p) {   // halo overlap: interior / boundary patch lists
        std::vector<int32_t> il, bl;
        for (int64_t lp = 0; lp < f->Pl; ++lp) {
          bool remote = false;
          for (int k = 0; k < 8; ++k) remote |= rs.nbr[lp * 8 + k] == -2;
          (remote ? bl : il).push_back((int32_t)lp);
        }
        f->n_int = (int64_t)il.size();
        f->n_bnd = (int64_t)bl.size();
        const int32_t ni = (int32_t)il.size(), nb = (int32_t)bl.size();
        if ((e = cudaMalloc(&f->d_ilist, std::max<size_t>(1, il.size()) * sizeof(int32_t))) != cudaSuccess ||
            (e = cudaMalloc(&f->d_blist, std::max<size_t>(1, bl.size()) * sizeof(int32_t))) != cudaSuccess ||
            (e = cudaMalloc(&f->d_icnt, sizeof(int32_t))) != cudaSuccess ||
            (e = cudaMalloc(&f->d_bcnt, sizeof(int32_t))) != cudaSuccess)
          return cuda_fail(e, "cudaMalloc overlap lists");
        if (ni) cudaMemcpy(f->d_ilist, il.data(), il.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
        if (nb) cudaMemcpy(f->d_blist, bl.data(), bl.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
        cudaMemcpy(f->d_icnt, &ni, sizeof(int32_t), cudaMemcpyHostToDevice);
        cudaMemcpy(f->d_bcnt, &nb, sizeof(int32_t), cudaMemcpyHostToDevice);
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if ((e = cudaStreamCreateWithPriority(&f->comm_stream, cudaStreamNonBlocking, hi)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&f->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&f->ev_halo, cudaEventDisableTiming)) != cudaSuccess)
          return cuda_fail(e, "overlap stream / events");
        f->split = true;
      }
    } else if (allow && !pl.uniform_same && T == pl.m) {
      // AMR forest: fused two-hop gather (plan_ring_amr; on shards with the NCCL / manual halo,
      // one exchange round); unsupported forests keep the ghost kernels
      RingSources rs;
      RingAmr ra;
      std::string why;
      if (plan_ring_amr(f->pl, pl.meqn, rs, ra, why) == FC_OK) {
        const int64_t S = (int64_t)pl.meqn * pl.n * pl.n;
        if ((e = cudaMalloc(&f->d_rpeer, rs.peer.size())) != cudaSuccess ||
            (e = cudaMalloc(&f->d_ring, rs.src.size() * sizeof(int32_t))) != cudaSuccess ||
            (e = cudaMalloc(&f->d_bcflag, std::max<size_t>(1, rs.bcflag.size()))) != cudaSuccess ||
            (e = cudaMalloc(&f->d_cg, (size_t)std::max<int64_t>(1, ra.ncg_patches) * S * sizeof(double))) != cudaSuccess)
          return cuda_fail(e, "cudaMalloc AMR ring");
        cudaMemcpy(f->d_rpeer, rs.peer.data(), rs.peer.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(f->d_ring, rs.src.data(), rs.src.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
        cudaMemcpy(f->d_bcflag, rs.bcflag.data(), rs.bcflag.size(), cudaMemcpyHostToDevice);
        if ((rc = to_dev(f, ra.avg, 5, f->cg_avg)) || (rc = to_dev(f, ra.corner3, 3, f->cg_c3))) {
          destroy(f);
          return fail(rc, g_err);
        }
        f->cg_interp.resize(ra.interp.size());
        for (size_t l = 0; l < ra.interp.size(); ++l)
          if ((rc = to_dev(f, ra.interp[l], 8, f->cg_interp[l]))) { destroy(f); return fail(rc, g_err); }
        if ((rc = upload_regular(f, rs))) return rc;
        f->fused = true;
        f->amr_fused = true;
        f->st.uniform_fast_path = 2;
      }
    }
  }
  if (!f->d_nbr) {   // quiescent-filter tables for the ring (non-fused) path: any forest
    std::vector<int32_t> nbr;
    std::vector<uint8_t> nm;
    rc = plan_activity(f->pl, pl.meqn, nbr, nm, err);
    if (rc) { destroy(f); return fail(rc, err); }
    const size_t Pl1 = std::max<int64_t>(1, f->Pl);
    if ((e = cudaMalloc(&f->d_nbr, Pl1 * 8 * sizeof(int32_t))) != cudaSuccess ||
        (e = cudaMalloc(&f->d_active, Pl1 * sizeof(int32_t))) != cudaSuccess ||
        (e = cudaMalloc(&f->d_nactive, sizeof(int32_t))) != cudaSuccess ||
        (e = cudaMalloc(&f->d_negmask, Pl1)) != cudaSuccess || (e = cudaMalloc(&f->d_uflag, Pl1)) != cudaSuccess ||
        (e = cudaMalloc(&f->d_uval, Pl1 * pl.meqn * sizeof(double))) != cudaSuccess)
      return cuda_fail(e, "cudaMalloc filter");
    if (!nbr.empty()) cudaMemcpy(f->d_nbr, nbr.data(), nbr.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (!nm.empty()) cudaMemcpy(f->d_negmask, nm.data(), nm.size(), cudaMemcpyHostToDevice);
  }
  if (pl.nranks > 1) {
    if (f->manual) {
      for (int r = 0; r < 2; ++r) f->peer_req[r].assign(pl.nranks, {});
      rc = build_halo_lists(f);   // receive side now; send side after fc_halo_set_requests + finalize
    } else {
      rc = setup_halo(f, d->nccl_id);
      if (!rc && f->p2p) rc = setup_p2p_ipc(f);
    }
    if (rc) { std::string m = g_err; destroy(f); return fail(rc, m); }
  }
  *out = f;
  return FC_OK;
}

int fc_forest_destroy(fc_forest* f) {
  destroy(f);
  return FC_OK;
}

int fc_set_problem(fc_forest* f, const fc_problem* pr) {
  if (!f || !pr) return fail(FC_EINVAL, "null argument");
  static const int meqn_of[5] = {1, 1, 3, 4, 4}, maux_of[5] = {0, 3, 0, 0, 0};
  if (pr->kind < 0 || pr->kind > 4) return fail(FC_EINVAL, "unknown problem kind");
  if (meqn_of[pr->kind] != f->pl.meqn || maux_of[pr->kind] != f->pl.maux)
    return fail(FC_EINVAL, "meqn/maux of the forest do not match the problem kind");
  if (pr->limiter < 0 || pr->limiter > 2 || pr->method2 < 1 || pr->method2 > 2 || pr->method3 < 0 ||
      pr->method3 > 2)
    return fail(FC_EINVAL, "limiter/method out of range");
  if ((pr->kind == FC_SWE_ROE || pr->kind == FC_EULER_ROE || pr->kind == FC_EULER_HLLE) && !(pr->p0 > 0.0))
    return fail(FC_EINVAL, "g / gamma must be positive");
  if ((pr->kind == FC_EULER_ROE || pr->kind == FC_EULER_HLLE) && !(pr->p0 > 1.0)) return fail(FC_EINVAL, "gamma must exceed 1");
  if (pr->skip_quiescent != 0 && pr->skip_quiescent != 1) return fail(FC_EINVAL, "skip_quiescent must be 0 or 1");
  if (pr->reflux != 0 && pr->reflux != 1) return fail(FC_EINVAL, "reflux must be 0 or 1");
  if (pr->reflux && !f->reflux_planned) {
    RefluxPlan rf;
    std::string err;
    int rc = plan_reflux(f->pl, f->pl.meqn, rf, err);
    if (rc) return fail(rc, err);
    {   // cells grouped by the coarse patch's level (sub-cycling refluxes one level pair at a time)
      const int64_t nc = (int64_t)rf.cells.size() / RFX;
      std::vector<int64_t> idx(nc);
      for (int64_t i = 0; i < nc; ++i) idx[i] = i;
      auto lev = [&](int64_t i) { return (int)f->pl.leaves[f->pl.p0 + rf.cells[i * RFX + 2]].level; };
      std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return lev(a) < lev(b); });
      std::vector<int32_t> sorted(rf.cells.size());
      for (int64_t i = 0; i < nc; ++i)
        std::copy(rf.cells.begin() + idx[i] * RFX, rf.cells.begin() + (idx[i] + 1) * RFX, sorted.begin() + i * RFX);
      rf.cells.swap(sorted);
      f->rcell_off.assign(f->glmax - f->glmin + 2, 0);
      for (int64_t i = 0; i < nc; ++i) f->rcell_off[lev(i) - f->glmin + 1] += 1;
      for (size_t l = 1; l < f->rcell_off.size(); ++l) f->rcell_off[l] += f->rcell_off[l - 1];
      f->nslots = rf.nslots;
    }
    f->rf_req = rf.req;
    f->rf_nremote = rf.nremote;
    f->h_rslot = rf.slot;
    f->nrcells = (int64_t)rf.cells.size() / RFX;
    if (!f->host_only) {
      CK(cudaSetDevice(f->device));
      const int64_t Pl1 = std::max<int64_t>(1, f->Pl);
      CK(cudaMalloc(&f->d_rslot, Pl1 * sizeof(int32_t)));
      if (f->Pl) CK(cudaMemcpy(f->d_rslot, rf.slot.data(), f->Pl * sizeof(int32_t), cudaMemcpyHostToDevice));
      if (f->nrcells) {
        CK(cudaMalloc(&f->d_rcells, rf.cells.size() * sizeof(int32_t)));
        CK(cudaMemcpy(f->d_rcells, rf.cells.data(), rf.cells.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      }
      const int64_t faces = 4 * (int64_t)rf.nslots + rf.nremote;
      CK(cudaMalloc(&f->d_freg, (size_t)std::max<int64_t>(1, faces) * f->pl.m * f->pl.meqn * sizeof(double)));
      if (f->pl.nranks > 1) {   // who serves whom: NCCL exchange now, or the caller (manual transport)
        if (f->manual) {
          f->rf_serve.assign(f->pl.nranks, {});
          f->rf_ready = false;
        } else {
          int rc2 = reflux_exchange_requests(f);
          if (rc2) return rc2;
        }
      }
    } else {
      f->nrcells = (int64_t)rf.cells.size() / RFX;
    }
    f->reflux_planned = true;
  }
  f->prob = *pr;
  f->has_problem = true;
  // fc_run's captured graphs bake the problem's kernel arguments (kind, limiter, methods, p0/p1,
  // skip_quiescent, reflux): a new problem invalidates them
  for (auto& g : f->run_exec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  return FC_OK;
}

int fc_set_stream(fc_forest* f, void* stream) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (f->host_only) return fail(FC_ESTATE, "host-only handle");
  f->stream = stream ? (cudaStream_t)stream : f->own_stream;
  return FC_OK;
}

int fc_set_timing(fc_forest* f, int on) {
  if (!f) return fail(FC_EINVAL, "null handle");
  f->timing = on != 0;
  return FC_OK;
}

int fc_get_stats(fc_forest* f, fc_stats* out) {
  if (!f || !out) return fail(FC_EINVAL, "null argument");
  if (!f->t_pending.empty()) {
    CK(cudaSetDevice(f->device));
    CK(cudaStreamSynchronize(f->stream));
    timing_drain(f);
  }
  *out = f->st;
  return FC_OK;
}

int fc_reset_stats(fc_forest* f) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (!f->t_pending.empty()) {
    CK(cudaSetDevice(f->device));
    CK(cudaStreamSynchronize(f->stream));
    timing_drain(f);   // (then zeroed below)
  }
  f->st.kernel_launches = 0;
  f->st.steps = 0;
  f->st.ms_ghost = f->st.ms_step = f->st.ms_comm = f->st.ms_copy = 0.0;
  f->st.copy_launches = 0;
  f->st.step_kernel_launches = 0;
  return FC_OK;
}

int fc_local_range(fc_forest* f, int64_t* first, int64_t* count) {
  if (!f || !first || !count) return fail(FC_EINVAL, "null argument");
  *first = f->pl.p0;
  *count = f->Pl;
  return FC_OK;
}

int fc_halo_counts(fc_forest* f, int64_t* counts) {
  if (!f || !counts) return fail(FC_EINVAL, "null argument");
  for (int s = 0; s < f->pl.nranks; ++s)
    counts[s] = (int64_t)(f->pl.halo.need1[s].size() + f->pl.halo.need2[s].size());
  return FC_OK;
}

int fc_halo_requests(fc_forest* f, int peer, int round, int64_t* buf, int64_t cap, int64_t* len) {
  if (!f || !len) return fail(FC_EINVAL, "null argument");
  if (peer < 0 || peer >= f->pl.nranks || (round != 1 && round != 2)) return fail(FC_EINVAL, "bad peer/round");
  const auto& v = round == 1 ? f->pl.halo.need1[peer] : f->pl.halo.need2[peer];
  *len = (int64_t)v.size();
  if (cap < *len || (!buf && *len)) return fail(FC_EINVAL, "buffer too small");
  if (*len) std::memcpy(buf, v.data(), v.size() * sizeof(int64_t));
  return FC_OK;
}

int fc_get_ghost_table(fc_forest* f, int which, int32_t* buf, int64_t cap, int64_t* len) {
  if (!f || !len) return fail(FC_EINVAL, "null argument");
  if (which == FC_TABLE_COMPACT) {
    *len = f->Pl * 40;
    if (!buf || cap < *len) return fail(FC_EINVAL, "buffer too small");
    std::string err;
    for (int64_t lp = 0; lp < f->Pl; ++lp) {
      const int rc = plan_compact_patch(f->pl, f->pl.p0 + lp, buf + 40 * lp, err);
      if (rc) return fail(rc, err);
    }
    return FC_OK;
  }
  if (which != FC_TABLE_EXPANDED) return fail(FC_EINVAL, "unknown table kind");
  *len = (int64_t)f->pl.table.size();
  if (!buf || cap < *len) return fail(FC_EINVAL, "buffer too small");
  std::memcpy(buf, f->pl.table.data(), f->pl.table.size() * sizeof(int32_t));
  return FC_OK;
}

int fc_set_aux(fc_forest* f, const double* aux, int where) {
  if (!f || !aux) return fail(FC_EINVAL, "null argument");
  if (f->host_only) return fail(FC_ESTATE, "host-only handle");
  if (f->pl.maux == 0) return fail(FC_EINVAL, "forest has maux = 0");
  CK(cudaSetDevice(f->device));
  const size_t bytes = (size_t)f->Pl * f->pl.maux * f->pl.n * f->pl.n * sizeof(double);
  CK(cudaMemcpyAsync(f->aux, aux, bytes, where == FC_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  f->has_aux = true;
  return FC_OK;
}

int fc_set_q(fc_forest* f, const double* q, int where) {
  if (!f || !q) return fail(FC_EINVAL, "null argument");
  if (f->host_only) return fail(FC_ESTATE, "host-only handle");
  if (!f->has_problem) return fail(FC_ESTATE, "fc_set_problem first");
  CK(cudaSetDevice(f->device));
  const int m = f->pl.m, meqn = f->pl.meqn;
  const size_t bytes = (size_t)f->Pl * meqn * m * m * sizeof(double);
  const double* src = q;
  if (where != FC_DEVICE) {   // stage through q_new (free between steps)
    CK(cudaMemcpyAsync(f->qnew, q, bytes, cudaMemcpyHostToDevice, f->stream));
    src = f->qnew;
  }
  f->st.kernel_launches += launch_scatter(src, f->qold, f->Pl, meqn, m, f->stream);
  CK(cudaGetLastError());
  if (f->p2p && f->comm)   // peers read this state directly: every rank's upload before any step
    NK(ncclAllReduce(f->d_cfl, f->d_cfl, 1, ncclDouble, ncclMax, f->comm, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  f->has_q = true;
  return FC_OK;
}

int fc_get_q(fc_forest* f, double* q, int where) {
  if (!f || !q) return fail(FC_EINVAL, "null argument");
  if (f->host_only || !f->has_q) return fail(FC_ESTATE, "no state");
  CK(cudaSetDevice(f->device));
  const int m = f->pl.m, meqn = f->pl.meqn;
  const size_t bytes = (size_t)f->Pl * meqn * m * m * sizeof(double);
  double* dst = where == FC_DEVICE ? q : f->qnew;
  f->st.kernel_launches += launch_gather(f->qold, dst, f->Pl, meqn, m, f->stream);
  CK(cudaGetLastError());
  if (where != FC_DEVICE) CK(cudaMemcpyAsync(q, f->qnew, bytes, cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  return FC_OK;
}

int fc_get_q_padded(fc_forest* f, double* q, int where) {
  if (!f || !q) return fail(FC_EINVAL, "null argument");
  if (f->host_only || !f->has_q) return fail(FC_ESTATE, "no state");
  CK(cudaSetDevice(f->device));
  const size_t bytes = (size_t)f->Pl * f->pl.meqn * f->pl.n * f->pl.n * sizeof(double);
  // storage -> natural padded layout (q_new is free scratch between steps)
  double* dst = where == FC_DEVICE ? q : f->qnew;
  f->st.kernel_launches += launch_unpack_padded(f->qold, dst, f->Pl * f->pl.meqn, f->pl.n, f->stream);
  CK(cudaGetLastError());
  if (where != FC_DEVICE) CK(cudaMemcpyAsync(q, f->qnew, bytes, cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  return FC_OK;
}

int fc_ghost_fill(fc_forest* f) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (f->host_only || !f->has_q) return fail(FC_ESTATE, "no state");
  if (f->manual) return fail(FC_ESTATE, "manual halo transport: use the staged calls");
  CK(cudaSetDevice(f->device));
  int rc = ghost_fill_internal(f);
  if (rc) return rc;
  CK(cudaStreamSynchronize(f->stream));
  return FC_OK;
}

int fc_step(fc_forest* f, double dt, double* max_cfl) {
  int rc = check_step_args(f, dt);
  if (rc) return rc;
  if (f->manual) return fail(FC_ESTATE, "manual halo transport: use fc_halo_* / fc_step_local / fc_commit");
  CK(cudaSetDevice(f->device));
  f->copy_timed = false;
  if (f->timing) {   // fresh events for this step (read at fc_get_stats)
    for (int k = 0; k < 6; ++k) {
      if (f->t_pool.empty()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        f->t_all.push_back(e);
        f->t_pool.push_back(e);
      }
      f->ev[k] = f->t_pool.back();
      f->t_pool.pop_back();
    }
  }
  if (f->timing) CK(cudaEventRecord(f->ev[0], f->stream));
  // fused ring gather + quiescent filter when skipping is on (rings never written); otherwise the
  // ghost kernels fill the rings and every tile is bulk-copied whole (faster for the full update)
  // (peer-memory halo: the fused gather reads other ranks' cells itself; no exchange pass)
  if (overlap_ok(f)) {
    // halo exchange on the high-priority comm stream (pack -> NCCL send / recv -> unpack into the
    // halo slots) while the interior patches update; the boundary patches after its event.  The
    // halo slots are only read by boundary patches, and q_old is not written during the step.
    CK(cudaEventRecord(f->ev_fork, f->stream));
    CK(cudaStreamWaitEvent(f->comm_stream, f->ev_fork, 0));
    if ((rc = halo_round(f, 0, f->comm_stream))) return rc;
    CK(cudaEventRecord(f->ev_halo, f->comm_stream));
    if (f->timing) CK(cudaEventRecord(f->ev[1], f->stream));
    if ((rc = update_local(f, dt, 1))) return rc;
    CK(cudaStreamWaitEvent(f->stream, f->ev_halo, 0));
    if ((rc = update_local(f, dt, 2))) return rc;
  } else {
    rc = use_fused(f) ? (f->p2p ? FC_OK : halo_round(f, 0)) : ghost_fill_internal(f);
    if (rc) return rc;
    if (f->timing) CK(cudaEventRecord(f->ev[1], f->stream));
    if ((rc = update_local(f, dt))) return rc;
  }
  if (f->timing) CK(cudaEventRecord(f->ev[2], f->stream));
  if (f->pl.nranks > 1)
    NK(ncclAllReduce(f->d_cfl, f->d_cfl, 1, ncclDouble, ncclMax, f->comm, f->stream));
  if (f->timing) CK(cudaEventRecord(f->ev[3], f->stream));
  CK(cudaMemcpyAsync(f->h_cfl, f->d_cfl, sizeof(double), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  note_activity(f);
  if (f->timing) {
    fc_forest::PendingTiming p;
    for (int k = 0; k < 6; ++k) p.e[k] = f->ev[k];
    p.copy = f->copy_timed;
    f->copy_timed = false;
    f->t_pending.push_back(p);
    if (f->t_pending.size() >= 4096) timing_drain(f);
  }
  const double cfl = *f->h_cfl;
  if (max_cfl) *max_cfl = cfl;
  return commit(f, cfl);
}

// ---- multi-step fixed-dt run in CUDA graphs ---------------------------------------------------------
// (timing_drain: see fc_forest::t_pending)
// The device part of one step (ghost fill or fused gather, quiescent filter, update, CFL into the
// history) is captured once per buffer parity and replayed nsteps times with no host round trip;
// the CFLs are checked at the end.  If any exceeds cfl_reject (or is not finite) the run is undone
// from a copy of the starting state.  Semantics = nsteps x fc_step(dt) without retakes.
static int run_capture(fc_forest* f, double dt) {
  const int64_t kl = f->st.kernel_launches, skl = f->st.step_kernel_launches;   // capture is not a launch
  const bool timing = f->timing;   // no timing events inside the graphs
  f->timing = false;
  for (int par = 0; par < 2; ++par) {
    if (f->run_exec[par]) { cudaGraphExecDestroy(f->run_exec[par]); f->run_exec[par] = nullptr; }
    double* qo = f->buf[par];
    double* qn = f->buf[par ^ 1];
    double* save_o = f->qold;
    double* save_n = f->qnew;
    f->qold = qo;
    f->qnew = qn;
    CK(cudaStreamBeginCapture(f->stream, cudaStreamCaptureModeRelaxed));
    f->capturing = true;
    int rc = use_fused(f) ? FC_OK : ghost_fill_internal(f);
    if (!rc) rc = update_local(f, dt);
    f->capturing = false;
    if (!rc) launch_cfl_hist(f->d_cfl, f->d_hist, f->d_hist_idx, f->stream);
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(f->stream, &g);
    f->qold = save_o;
    f->qnew = save_n;
    if (rc) { if (g) cudaGraphDestroy(g); f->timing = timing; return rc; }
    if (ec != cudaSuccess) { f->timing = timing; return fail(FC_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ec)); }
    const cudaError_t ei = cudaGraphInstantiate(&f->run_exec[par], g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) { f->timing = timing; return fail(FC_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei)); }
  }
  f->timing = timing;
  f->copy_timed = false;
  f->run_launches = (f->st.kernel_launches - kl) / 2 + 1;   // + the CFL history kernel
  f->st.kernel_launches = kl;
  f->st.step_kernel_launches = skl;
  f->run_dt = dt;
  return FC_OK;
}

int fc_run(fc_forest* f, double dt, int64_t nsteps, double* cfls, double* max_cfl) {
  int rc = check_step_args(f, dt);
  if (rc) return rc;
  if (nsteps < 0) return fail(FC_EINVAL, "nsteps < 0");
  if (f->pl.nranks != 1) return fail(FC_EUNSUP, "fc_run runs on one rank");
  if (max_cfl) *max_cfl = 0.0;
  if (nsteps == 0) return FC_OK;
  CK(cudaSetDevice(f->device));
  if (f->hist_cap < nsteps) {
    cudaFree(f->d_hist);
    f->d_hist = nullptr;
    CK(cudaMalloc(&f->d_hist, nsteps * sizeof(double)));
    f->hist_cap = nsteps;
    if (f->run_exec[0]) { cudaGraphExecDestroy(f->run_exec[0]); f->run_exec[0] = nullptr; }   // re-capture
    if (f->run_exec[1]) { cudaGraphExecDestroy(f->run_exec[1]); f->run_exec[1] = nullptr; }
  }
  if (!f->d_hist_idx) CK(cudaMalloc(&f->d_hist_idx, sizeof(int64_t)));
  if (!f->d_backup) CK(cudaMalloc(&f->d_backup, f->state_doubles * sizeof(double)));
  if (!f->run_exec[0] || f->run_dt != dt) {   // (relaxed capture: one-time kernel setup may run inside)
    if ((rc = run_capture(f, dt))) return rc;
  }
  const int par0 = f->parity;
  double* start = f->qold;
  CK(cudaMemcpyAsync(f->d_backup, start, f->state_doubles * sizeof(double), cudaMemcpyDeviceToDevice, f->stream));
  CK(cudaMemsetAsync(f->d_hist_idx, 0, sizeof(int64_t), f->stream));
  for (int64_t i = 0; i < nsteps; ++i) {
    CK(cudaGraphLaunch(f->run_exec[f->parity], f->stream));
    std::swap(f->qold, f->qnew);
    f->parity ^= 1;
  }
  std::vector<double> h(nsteps);
  CK(cudaMemcpyAsync(h.data(), f->d_hist, nsteps * sizeof(double), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  double mx = 0.0;
  bool bad = false, over = false;
  for (int64_t i = 0; i < nsteps; ++i) {
    if (cfls) cfls[i] = h[i];
    if (!std::isfinite(h[i])) bad = true;
    else if (h[i] > f->prob.cfl_reject) over = true;
    if (h[i] > mx || h[i] != h[i]) mx = h[i];
  }
  if (max_cfl) *max_cfl = mx;
  f->st.kernel_launches += nsteps * f->run_launches;
  f->st.step_kernel_launches += nsteps;
  if (bad || over) {   // undo: the starting state back into the buffer that held it
    if (f->parity != par0) { std::swap(f->qold, f->qnew); f->parity = par0; }
    CK(cudaMemcpyAsync(f->qold, f->d_backup, f->state_doubles * sizeof(double), cudaMemcpyDeviceToDevice, f->stream));
    CK(cudaStreamSynchronize(f->stream));
    return bad ? fail(FC_ENONFINITE, "CFL not finite in the run; state restored")
               : fail(FC_ECFL, "CFL above cfl_reject in the run; state restored");
  }
  f->st.steps += nsteps;
  return FC_OK;
}

// ---- sub-cycled step ---------------------------------
// Level l advances with dt_l = dt_coarse 2^-(l - glmin) in a coarse-to-fine recursion; the ghost
// fill of level l at each of its start times runs on a snapshot in which coarser patches hold their
// state interpolated linearly in time (exact dyadic weights from integer ticks).  Buffers: q_old =
// the committed state (untouched until the commit), q_new = the working state (each patch's
// interior written by its level's first step; all levels at their current times), d_sub_old = each level's state at the start of its current step, d_sub_snap = the
// snapshot with its rings (the ghost fill and the halo exchange run on it).
static int sub_prepare(fc_forest* f) {
  if (f->sub_ready) return FC_OK;
  const int NL = f->glmax - f->glmin + 1;
  if (NL > 30) return fail(FC_EUNSUP, "more than 30 refinement levels");
  CK(cudaMalloc(&f->d_sub_old, f->state_doubles * sizeof(double)));
  CK(cudaMalloc(&f->d_sub_snap, f->state_doubles * sizeof(double)));
  CK(cudaMemset(f->d_sub_snap, 0, f->state_doubles * sizeof(double)));
  std::vector<std::vector<int32_t>> lists(NL);
  for (int64_t lp = 0; lp < f->Pl; ++lp) lists[f->pl.leaves[f->pl.p0 + lp].level - f->glmin].push_back((int32_t)lp);
  std::vector<int32_t> cnt(NL);
  f->d_lvl.assign(NL, nullptr);
  f->n_lvl.assign(NL, 0);
  for (int l = 0; l < NL; ++l) {
    f->n_lvl[l] = (int64_t)lists[l].size();
    cnt[l] = (int32_t)lists[l].size();
    CK(cudaMalloc(&f->d_lvl[l], std::max<size_t>(1, lists[l].size()) * sizeof(int32_t)));
    if (!lists[l].empty())
      CK(cudaMemcpy(f->d_lvl[l], lists[l].data(), lists[l].size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  }
  CK(cudaMalloc(&f->d_lvl_cnt, NL * sizeof(int32_t)));
  CK(cudaMemcpy(f->d_lvl_cnt, cnt.data(), NL * sizeof(int32_t), cudaMemcpyHostToDevice));
  // Restricted fills (one rank; a remote coarse patch's ring would need its owner's closure): the
  // level-l fill only has to produce the rings of D_l = the level-l patches plus, recursively, every
  // patch an INTERP record of D_l reads (its ring feeds the slopes), and the snapshot only has to
  // hold N_l = D_l plus every patch a record of D_l reads.  The records kept are exactly the full
  // fill's records for D_l's cells, in the same order, so the rings of D_l are bitwise those of the
  // full fill; other rings and snapshot cells are stale and nothing of level l reads them.
  const char* full = std::getenv("FC_SUB_FULL_FILL");
  if (f->pl.nranks == 1 && !(full && full[0] == '1')) {
    const Plan& pl = f->pl;
    const int64_t Pl = f->Pl, G = (int64_t)pl.n * pl.n - (int64_t)pl.m * pl.m;
    auto sources = [&](int64_t lp, auto&& fn) {       // (op, source local patch) of lp's records
      for (int64_t r = 0; r < G; ++r) {
        const int32_t* o = pl.table.data() + (lp * G + r) * REC;
        if (o[0] == OP_COPY || o[0] == OP_AVG4 || o[0] == OP_INTERP) fn(o[0], (int64_t)o[1] - pl.p0);
      }
    };
    f->sub_fill.resize(NL);
    for (int l = 0; l < NL; ++l) {
      std::vector<uint8_t> D(Pl, 0), N(Pl, 0);
      std::vector<int64_t> work(lists[l].begin(), lists[l].end());
      for (int64_t lp : work) D[lp] = 1;
      while (!work.empty()) {
        const int64_t lp = work.back();
        work.pop_back();
        sources(lp, [&](int op, int64_t q) {
          if (op == OP_INTERP && !D[q]) { D[q] = 1; work.push_back(q); }
        });
      }
      std::vector<int32_t> snap;
      for (int64_t lp = 0; lp < Pl; ++lp)
        if (D[lp]) { N[lp] = 1; sources(lp, [&](int, int64_t q) { N[q] = 1; }); }
      for (int64_t lp = 0; lp < Pl; ++lp) if (N[lp]) snap.push_back((int32_t)lp);
      GhostLists gl;
      std::string err;
      int rc = plan_lists(pl, pl.meqn, gl, err, &D);
      if (rc) return fail(rc, err);
      FillLists& s = f->sub_fill[l];
      if ((rc = to_dev(f, gl.copy, 2, s.copy)) || (rc = to_dev(f, gl.avg, 5, s.avg)) ||
          (rc = to_dev(f, gl.bcx, 3, s.bcx)) || (rc = to_dev(f, gl.bcy, 3, s.bcy)) ||
          (rc = to_dev(f, gl.corner3, 3, s.corner3)))
        return rc;
      s.interp.resize(gl.interp.size());
      s.bcx_l.resize(gl.interp.size());
      s.bcy_l.resize(gl.interp.size());
      for (size_t k = 0; k < gl.interp.size(); ++k)
        if ((rc = to_dev(f, gl.interp[k], 8, s.interp[k])) || (rc = to_dev(f, gl.bcx_l[k], 3, s.bcx_l[k])) ||
            (rc = to_dev(f, gl.bcy_l[k], 3, s.bcy_l[k])))
          return rc;
      s.n_snap = (int64_t)snap.size();
      CK(cudaMalloc(&s.d_snap, std::max<size_t>(1, snap.size()) * sizeof(int32_t)));
      if (!snap.empty())
        CK(cudaMemcpy(s.d_snap, snap.data(), snap.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
  }
  f->sub_ready = true;
  return FC_OK;
}

static int sub_advance(fc_forest* f, int l, int64_t tick, int sub) {
  const fc_problem& p = f->prob;
  const int li = l - f->glmin, m = f->pl.m, meqn = f->pl.meqn, n2 = f->pl.n * f->pl.n;
  const int64_t len = 1ll << (f->glmax - l);
  const double dt = std::ldexp(f->sub_dt0, -li);
  const bool reflux = p.reflux && f->nrcells > 0;
  double alpha[32] = {};
  for (int c = f->glmin; c < l; ++c)
    alpha[c - f->glmin] = (double)(tick - f->sub_tick_old[c - f->glmin]) /
                          (double)(f->sub_tick_new[c - f->glmin] - f->sub_tick_old[c - f->glmin]);
  const FillLists* sel = f->sub_fill.empty() ? nullptr : &f->sub_fill[li];
  // The coarsest level steps once, from the committed state: its fill runs on q_old itself (whose
  // rings are scratch) and q_old doubles as its start-of-step state, so no snapshot is taken.
  // Finer levels: at tick 0 no patch has stepped yet, the current state is the committed one (and
  // the weights of the coarser levels are 0), so q_new is never read before each patch's step has
  // written it.
  const bool coarsest = l == f->glmin;
  if (!coarsest) {
    f->st.kernel_launches += launch_sub_snapshot(tick == 0 ? f->qold : f->qnew, f->d_sub_old, f->qold, f->d_sub_snap,
                                                 f->d_level, sel ? sel->d_snap : nullptr, sel ? sel->n_snap : f->Pl,
                                                 meqn, m, n2, l, alpha, f->glmin, f->stream);
    CK(cudaGetLastError());
  }
  double* committed = f->qold;       // the ghost fill (and its halo exchange) runs on the snapshot
  double* src = coarsest ? f->qold : f->d_sub_snap;
  // fused AMR gather (one rank): no ring writes -- the computed ghosts from this snapshot, and the
  // step gathers every ring cell of the level's patches itself (their sources are all in N_l)
  const bool fused = f->amr_fused && use_fused(f);
  int rc = FC_OK;
  if (fused) {
    if (f->pl.nranks > 1) {   // the remote interior cells of this snapshot into its halo slots
      f->qold = src;
      rc = halo_round(f, 0);
      f->qold = committed;
      if (rc) return rc;
    }
    f->st.kernel_launches += launch_cg(2, src, f->d_cg, f->cg_avg.d, f->cg_avg.nrec, meqn, n2, f->stream);
    for (auto& cl : f->cg_interp)
      f->st.kernel_launches += launch_cg(3, src, f->d_cg, cl.d, cl.nrec, meqn, n2, f->stream);
    f->st.kernel_launches += launch_cg(6, src, f->d_cg, f->cg_c3.d, f->cg_c3.nrec, meqn, n2, f->stream);
    CK(cudaGetLastError());
  } else {
    f->qold = src;
    f->fill_sel = sel;
    rc = ghost_fill_internal(f);
    f->fill_sel = nullptr;
    f->qold = committed;
    if (rc) return rc;
  }
  if (f->n_lvl[li] > 0) {
    int lr = launch_step(p.kind, src, f->qnew, f->aux, f->d_level, f->n_lvl[li], m, dt, f->pl.dx0, p.p0,
                         p.p1, p.limiter, p.method2, p.method3, p.skip_quiescent, fused ? f->d_ring : nullptr,
                         f->d_nb9, f->d_bcflag, f->d_lvl[li], f->d_lvl_cnt + li, f->d_cfl, reflux ? f->d_rslot : nullptr,
                         reflux ? f->d_freg : nullptr, fused ? f->d_rpeer : nullptr, nullptr,
                         fused ? f->d_cg : nullptr, f->stream);
    if (lr < 0) return fail(FC_EUNSUP, "no step kernel for this m / kind");
    f->st.kernel_launches += lr;
    f->st.step_kernel_launches += lr;
    CK(cudaGetLastError());
    if (reflux)
      f->st.kernel_launches += launch_sub_accumulate(f->d_lvl[li], f->n_lvl[li], f->d_rslot, f->d_freg, f->d_facc,
                                                     4 * m * meqn, dt, sub, f->stream);
  }
  f->sub_tick_old[li] = tick;
  f->sub_tick_new[li] = tick + len;
  if (l < f->glmax) {
    if ((rc = sub_advance(f, l + 1, tick, 0))) return rc;
    if ((rc = sub_advance(f, l + 1, tick + len / 2, 1))) return rc;
    if (reflux) {
      const int64_t a = f->rcell_off[li], b = f->rcell_off[li + 1];
      f->st.kernel_launches += launch_reflux(f->d_rcells + a * RFX, b - a, f->d_freg, f->d_facc, f->qnew, f->aux,
                                             f->d_level, dt, 1.0, f->pl.dx0, meqn, n2, f->stream);
      CK(cudaGetLastError());
    }
  }
  return FC_OK;
}

int fc_step_subcycled(fc_forest* f, double dt_coarse, double* max_cfl) {
  int rc = check_step_args(f, dt_coarse);
  if (rc) return rc;
  if (f->manual) return fail(FC_ESTATE, "manual halo transport: sub-cycling needs the NCCL transport");
  if (f->prob.reflux && (f->rf_nremote > 0 || f->rf_npack > 0))
    return fail(FC_EUNSUP, "sub-cycled reflux across rank cuts is not supported");
  if (f->glmin == f->glmax) return fc_step(f, dt_coarse, max_cfl);   // one level: the global step
  CK(cudaSetDevice(f->device));
  if ((rc = sub_prepare(f))) return rc;
  if (f->prob.reflux && f->nrcells > 0 && !f->d_facc)
    CK(cudaMalloc(&f->d_facc, (size_t)std::max<int32_t>(1, f->nslots) * 4 * f->pl.m * f->pl.meqn * sizeof(double)));
  if (f->timing && !f->t_pending.empty()) {   // (f->ev may be pending events of fc_step)
    CK(cudaStreamSynchronize(f->stream));
    timing_drain(f);
  }
  if (f->timing) CK(cudaEventRecord(f->ev[0], f->stream));
  CK(cudaMemsetAsync(f->d_cfl, 0, sizeof(unsigned long long), f->stream));
  f->sub_dt0 = dt_coarse;
  if ((rc = sub_advance(f, f->glmin, 0, 0))) return rc;
  if (f->timing) CK(cudaEventRecord(f->ev[2], f->stream));
  if (f->pl.nranks > 1)
    NK(ncclAllReduce(f->d_cfl, f->d_cfl, 1, ncclDouble, ncclMax, f->comm, f->stream));
  if (f->timing) CK(cudaEventRecord(f->ev[3], f->stream));
  CK(cudaMemcpyAsync(f->h_cfl, f->d_cfl, sizeof(double), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  if (f->timing) {
    float b = 0.f, c = 0.f;
    cudaEventElapsedTime(&b, f->ev[0], f->ev[2]);
    cudaEventElapsedTime(&c, f->ev[2], f->ev[3]);
    f->st.ms_step += b;
    f->st.ms_comm += c;
  }
  const double cfl = *f->h_cfl;
  if (max_cfl) *max_cfl = cfl;
  return commit(f, cfl);
}

// ---- dynamic regrid -------------------------------
static int regrid_nccl(fc_forest* f, const fc_regrid_params* rp, fc_forest** out);

int fc_regrid(fc_forest* f, const fc_regrid_params* rp, fc_forest** out) {
  if (!f || !rp || !out) return fail(FC_EINVAL, "null argument");
  *out = nullptr;
  if (f->host_only || !f->has_q || !f->has_problem) return fail(FC_ESTATE, "set problem and q first");
  if (rp->min_level < 0 || rp->max_level < rp->min_level || rp->max_level > 28)
    return fail(FC_EINVAL, "regrid level bounds out of range");
  if (f->manual) return fail(FC_ESTATE, "manual transport: use fc_regrid_fill / _tags / _begin / _finish");
  CK(cudaSetDevice(f->device));
  if (f->pl.nranks > 1) return regrid_nccl(f, rp, out);
  int rc = ghost_fill_internal(f);                 // the interpolation slopes read the parents' rings
  if (rc) return rc;
  const int m = f->pl.m, meqn = f->pl.meqn;
  double* d_tag = nullptr;
  CK(cudaMalloc(&d_tag, std::max<int64_t>(1, f->Pl) * sizeof(double)));
  f->st.kernel_launches += launch_regrid_tag(f->qold, f->Pl, meqn, m, d_tag, f->stream);
  std::vector<double> tag(f->Pl);
  CK(cudaMemcpyAsync(tag.data(), d_tag, f->Pl * sizeof(double), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(d_tag);
  std::vector<int8_t> lv;
  std::vector<int32_t> tr, src;
  std::string err;
  if ((rc = plan_regrid(f->pl, tag.data(), rp->refine_threshold, rp->coarsen_threshold, rp->min_level,
                        rp->max_level, lv, tr, src, err)))
    return fail(rc, err);
  fc_forest_desc d{};
  d.num_patches = (int64_t)lv.size();
  d.levels = lv.data();
  d.tree_ids = tr.data();
  d.num_trees = f->pl.T;
  d.tree_to_tree = f->pl.t2t.data();
  d.tree_to_face = f->pl.t2f.data();
  d.face_bc = f->pl.fbc.data();
  d.m = m;
  d.mbc = 2;
  d.meqn = meqn;
  d.maux = f->pl.maux;
  d.tree_dx0 = f->pl.dx0 * m;
  d.device = f->device;
  d.rank = 0;
  d.nranks = 1;
  d.nccl_id = nullptr;
  fc_forest* g = nullptr;
  if ((rc = fc_forest_create(&d, &g))) return rc;
  if ((rc = fc_set_problem(g, &f->prob))) { fc_forest_destroy(g); return rc; }
  int32_t* d_src = nullptr;
  if (cudaMalloc(&d_src, src.size() * sizeof(int32_t)) != cudaSuccess ||
      cudaMemcpy(d_src, src.data(), src.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d_src);
    fc_forest_destroy(g);
    return fail(FC_ECUDA, "regrid: source records");
  }
  g->st.kernel_launches += launch_regrid_transfer(f->qold, g->qold, d_src, g->Pl, meqn, m, f->stream);
  cudaError_t e = cudaStreamSynchronize(f->stream);
  cudaFree(d_src);
  if (e != cudaSuccess) { fc_forest_destroy(g); return fail(FC_ECUDA, std::string("regrid transfer: ") + cudaGetErrorString(e)); }
  g->has_q = true;
  *out = g;
  return FC_OK;
}

// ---- multi-rank regrid: the same global plan on every rank, Morton repartition by count of the
// new leaves, migration of the old padded blocks each new patch reads (copy: its old patch; child:
// the ghost-filled parent; parent: the 4 old children) from their old owners ----------------------
static int regrid_local_tags(fc_forest* f, std::vector<double>& tag) {
  const int m = f->pl.m, meqn = f->pl.meqn;
  double* d_tag = nullptr;
  CK(cudaMalloc(&d_tag, std::max<int64_t>(1, f->Pl) * sizeof(double)));
  f->st.kernel_launches += launch_regrid_tag(f->qold, f->Pl, meqn, m, d_tag, f->stream);
  tag.assign(f->Pl, 0.0);
  if (f->Pl) CK(cudaMemcpyAsync(tag.data(), d_tag, f->Pl * sizeof(double), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(d_tag);
  return FC_OK;
}

// plan + new handle + migration buffers (old side packed, self part staged); g's transfer waits
// for the other owners' blocks (regrid_finish)
static int regrid_begin(fc_forest* f, const double* gtag, const fc_regrid_params* rp, const void* nccl_id,
                        fc_forest** out) {
  const int m = f->pl.m, meqn = f->pl.meqn, R = f->pl.nranks, me = f->pl.rank;
  const int64_t S = (int64_t)meqn * f->pl.n * f->pl.n, Pold = f->pl.P;
  std::vector<int8_t> lv;
  std::vector<int32_t> tr, src;
  std::string err;
  int rc = plan_regrid(f->pl, gtag, rp->refine_threshold, rp->coarsen_threshold, rp->min_level, rp->max_level,
                       lv, tr, src, err);
  if (rc) return fail(rc, err);
  const int64_t Pnew = (int64_t)lv.size();
  // new Morton partition: by count, or (level_weights) equal sums of 2^(level - coarsest)
  std::vector<int64_t> part(R + 1, 0);
  if (rp->level_weights && R > 1) {
    int lmin = 127;
    for (int8_t l : lv) lmin = std::min(lmin, (int)l);
    std::vector<double> cum(Pnew + 1, 0.0);
    for (int64_t i = 0; i < Pnew; ++i) cum[i + 1] = cum[i] + std::ldexp(1.0, lv[i] - lmin);
    for (int r = 1; r < R; ++r)   // first patch whose prefix weight reaches r / R of the total
      part[r] = std::lower_bound(cum.begin(), cum.end(), cum[Pnew] * r / R) - cum.begin();
    for (int r = 1; r < R; ++r) part[r] = std::max(part[r], part[r - 1]);
  } else {
    for (int r = 0; r <= R; ++r) part[r] = (int64_t)r * Pnew / R;
  }
  part[R] = Pnew;
  fc_forest_desc d{};
  d.num_patches = Pnew;
  d.levels = lv.data();
  d.tree_ids = tr.data();
  d.num_trees = f->pl.T;
  d.tree_to_tree = f->pl.t2t.data();
  d.tree_to_face = f->pl.t2f.data();
  d.face_bc = f->pl.fbc.data();
  d.m = m;
  d.mbc = 2;
  d.meqn = meqn;
  d.maux = f->pl.maux;
  d.tree_dx0 = f->pl.dx0 * m;
  d.device = f->device;
  d.rank = me;
  d.nranks = R;
  d.nccl_id = nccl_id;
  d.partition = part.data();
  fc_forest* g = nullptr;
  if ((rc = fc_forest_create(&d, &g))) return rc;
  if ((rc = fc_set_problem(g, &f->prob))) { fc_forest_destroy(g); return rc; }
  auto old_first = [&](int r) { return f->pl.part[r]; };
  auto new_first = [&](int r) { return part[r]; };
  auto old_owner = [&](int64_t j) {
    return (int)(std::upper_bound(f->pl.part.begin(), f->pl.part.end(), j) - f->pl.part.begin()) - 1;
  };
  (void)old_first;
  (void)Pold;
  // the old blocks rank rr's new patches read, sorted (the 4 children of a parent are consecutive)
  auto referenced = [&](int rr) {
    std::vector<int32_t> ids;
    for (int64_t i = new_first(rr); i < new_first(rr + 1); ++i) {
      const int32_t* s = src.data() + i * 3;
      if (s[0] == 3) for (int k = 0; k < 4; ++k) ids.push_back(s[1] + k);
      else ids.push_back(s[1]);
    }
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    return ids;
  };
  // new side: staging slots in old-id order = owner-major
  const std::vector<int32_t> mine = referenced(me);
  g->rg_recv_off.assign(R + 1, 0);
  for (int32_t j : mine) g->rg_recv_off[old_owner(j) + 1] += S;
  for (int r = 0; r < R; ++r) g->rg_recv_off[r + 1] += g->rg_recv_off[r];
  std::vector<int32_t> lsrc(src.begin() + new_first(me) * 3, src.begin() + new_first(me + 1) * 3);
  for (size_t i = 0; i < lsrc.size(); i += 3)
    lsrc[i + 1] = (int32_t)(std::lower_bound(mine.begin(), mine.end(), lsrc[i + 1]) - mine.begin());
  CK(cudaSetDevice(f->device));
  CK(cudaMalloc(&g->d_rg_stage, std::max<size_t>(1, mine.size()) * S * sizeof(double)));
  CK(cudaMalloc(&g->d_rg_src, std::max<size_t>(1, lsrc.size()) * sizeof(int32_t)));
  if (!lsrc.empty()) CK(cudaMemcpy(g->d_rg_src, lsrc.data(), lsrc.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  // old side: per new rank the blocks of mine it reads, packed (local ids)
  std::vector<int32_t> ids;
  f->rg_send_off.assign(R + 1, 0);
  int64_t self_off = 0, self_n = 0;
  for (int r = 0; r < R; ++r) {
    const std::vector<int32_t> ref = r == me ? mine : referenced(r);
    if (r == me) self_off = (int64_t)ids.size();
    for (int32_t j : ref)
      if (j >= f->pl.p0 && j < f->pl.p1) ids.push_back((int32_t)(j - f->pl.p0));
    if (r == me) self_n = (int64_t)ids.size() - self_off;
    f->rg_send_off[r + 1] = (int64_t)ids.size() * S;
  }
  cudaFree(f->d_rg_send);
  f->d_rg_send = nullptr;
  CK(cudaMalloc(&f->d_rg_send, std::max<size_t>(1, ids.size()) * S * sizeof(double)));
  int32_t* d_ids = nullptr;
  CK(cudaMalloc(&d_ids, std::max<size_t>(1, ids.size()) * sizeof(int32_t)));
  if (!ids.empty()) CK(cudaMemcpy(d_ids, ids.data(), ids.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  f->st.kernel_launches += launch_copy_blocks(f->qold, f->d_rg_send, d_ids, (int64_t)ids.size(), S, f->stream);
  if (self_n)   // this rank's own blocks go straight to its staging
    CK(cudaMemcpyAsync(g->d_rg_stage + g->rg_recv_off[me], f->d_rg_send + self_off * S, self_n * S * sizeof(double),
                       cudaMemcpyDeviceToDevice, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(d_ids);
  g->rg_pending = true;
  *out = g;
  return FC_OK;
}

static int regrid_finish(fc_forest* g) {
  if (!g->rg_pending) return fail(FC_ESTATE, "no regrid in progress on this handle");
  CK(cudaSetDevice(g->device));
  g->st.kernel_launches += launch_regrid_transfer(g->d_rg_stage, g->qold, g->d_rg_src, g->Pl, g->pl.meqn, g->pl.m,
                                                  g->stream);
  CK(cudaStreamSynchronize(g->stream));
  cudaFree(g->d_rg_stage);
  cudaFree(g->d_rg_src);
  g->d_rg_stage = nullptr;
  g->d_rg_src = nullptr;
  g->rg_pending = false;
  g->has_q = true;
  return FC_OK;
}

// NCCL handles: every step of the above inside one collective call
static int regrid_nccl(fc_forest* f, const fc_regrid_params* rp, fc_forest** out) {
  const int R = f->pl.nranks, me = f->pl.rank;
  int rc = ghost_fill_internal(f);                 // (halo rounds included)
  if (rc) return rc;
  std::vector<double> tag;
  if ((rc = regrid_local_tags(f, tag))) return rc;
  // all-gather the tags (padded to the largest shard)
  int64_t maxpl = 0;
  for (int r = 0; r < R; ++r) maxpl = std::max(maxpl, f->pl.part[r + 1] - f->pl.part[r]);
  double *d_mine = nullptr, *d_all = nullptr;
  CK(cudaMalloc(&d_mine, std::max<int64_t>(1, maxpl) * sizeof(double)));
  CK(cudaMalloc(&d_all, std::max<int64_t>(1, maxpl) * R * sizeof(double)));
  if (f->Pl) CK(cudaMemcpy(d_mine, tag.data(), f->Pl * sizeof(double), cudaMemcpyHostToDevice));
  NK(ncclAllGather(d_mine, d_all, std::max<int64_t>(1, maxpl), ncclDouble, f->comm, f->stream));
  std::vector<double> all((size_t)std::max<int64_t>(1, maxpl) * R), gtag(f->pl.P);
  CK(cudaMemcpyAsync(all.data(), d_all, all.size() * sizeof(double), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(d_mine);
  cudaFree(d_all);
  for (int r = 0; r < R; ++r) {
    const int64_t a = f->pl.part[r], b = f->pl.part[r + 1];
    std::copy(all.begin() + (size_t)r * std::max<int64_t>(1, maxpl), all.begin() + (size_t)r * std::max<int64_t>(1, maxpl) + (b - a),
              gtag.begin() + a);
  }
  // a fresh NCCL id for the new handle's communicator, broadcast from rank 0 over the old one
  char id[128] = {};
  if (me == 0 && (rc = fc_nccl_unique_id(id))) return rc;
  char* d_id = nullptr;
  CK(cudaMalloc(&d_id, sizeof(id)));
  CK(cudaMemcpy(d_id, id, sizeof(id), cudaMemcpyHostToDevice));
  NK(ncclBroadcast(d_id, d_id, sizeof(id), ncclChar, 0, f->comm, f->stream));
  CK(cudaMemcpyAsync(id, d_id, sizeof(id), cudaMemcpyDeviceToHost, f->stream));
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(d_id);
  fc_forest* g = nullptr;
  if ((rc = regrid_begin(f, gtag.data(), rp, id, &g))) return rc;
  NK(ncclGroupStart());
  for (int s = 0; s < R; ++s) {
    if (s == me) continue;
    const int64_t ns = f->rg_send_off[s + 1] - f->rg_send_off[s], nr = g->rg_recv_off[s + 1] - g->rg_recv_off[s];
    if (ns) NK(ncclSend(f->d_rg_send + f->rg_send_off[s], ns, ncclDouble, s, f->comm, f->stream));
    if (nr) NK(ncclRecv(g->d_rg_stage + g->rg_recv_off[s], nr, ncclDouble, s, f->comm, f->stream));
  }
  NK(ncclGroupEnd());
  CK(cudaStreamSynchronize(f->stream));
  cudaFree(f->d_rg_send);
  f->d_rg_send = nullptr;
  if ((rc = regrid_finish(g))) { fc_forest_destroy(g); return rc; }
  *out = g;
  return FC_OK;
}

int fc_regrid_fill(fc_forest* f, int phase) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (!f->manual) return fail(FC_ESTATE, "not a manual-transport handle (fc_regrid does it all)");
  if (f->host_only || !f->has_q) return fail(FC_ESTATE, "no state");
  CK(cudaSetDevice(f->device));
  int rc = phase == 1 ? ghost_phase_ac(f) : (phase == 2 ? ghost_phase_b(f) : fail(FC_EINVAL, "phase must be 1 or 2"));
  if (rc) return rc;
  CK(cudaStreamSynchronize(f->stream));
  return FC_OK;
}

int fc_regrid_tags(fc_forest* f, double* tags) {
  if (!f || !tags) return fail(FC_EINVAL, "null argument");
  if (f->host_only || !f->has_q) return fail(FC_ESTATE, "no state");
  CK(cudaSetDevice(f->device));
  std::vector<double> t;
  int rc = regrid_local_tags(f, t);
  if (rc) return rc;
  std::copy(t.begin(), t.end(), tags);
  return FC_OK;
}

int fc_regrid_begin(fc_forest* f, const double* global_tags, const fc_regrid_params* rp, fc_forest** out) {
  if (!f || !global_tags || !rp || !out) return fail(FC_EINVAL, "null argument");
  *out = nullptr;
  if (!f->manual) return fail(FC_ESTATE, "not a manual-transport handle (fc_regrid does it all)");
  if (f->host_only || !f->has_q || !f->has_problem) return fail(FC_ESTATE, "set problem and q first");
  if (rp->min_level < 0 || rp->max_level < rp->min_level || rp->max_level > 28)
    return fail(FC_EINVAL, "regrid level bounds out of range");
  CK(cudaSetDevice(f->device));
  return regrid_begin(f, global_tags, rp, nullptr, out);
}

int fc_regrid_buffers(fc_forest* f, fc_forest* g, void** send, void** recv, int64_t* send_off, int64_t* recv_off) {
  if (!f || !g || !send || !recv || !send_off || !recv_off) return fail(FC_EINVAL, "null argument");
  if (!g->rg_pending || f->rg_send_off.size() != (size_t)f->pl.nranks + 1) return fail(FC_ESTATE, "no regrid in progress");
  *send = f->d_rg_send;
  *recv = g->d_rg_stage;
  std::copy(f->rg_send_off.begin(), f->rg_send_off.end(), send_off);
  std::copy(g->rg_recv_off.begin(), g->rg_recv_off.end(), recv_off);
  return FC_OK;
}

int fc_regrid_finish(fc_forest* g) {
  if (!g) return fail(FC_EINVAL, "null handle");
  return regrid_finish(g);
}

int fc_get_leaves(fc_forest* f, int8_t* levels, int32_t* tree_ids, int64_t cap, int64_t* num_patches) {
  if (!f || !num_patches) return fail(FC_EINVAL, "null argument");
  *num_patches = f->pl.P;
  if (!levels && !tree_ids) return FC_OK;        // size query
  if (cap < f->pl.P) return fail(FC_EINVAL, "capacity below the number of patches");
  for (int64_t p = 0; p < f->pl.P; ++p) {
    if (levels) levels[p] = (int8_t)f->pl.leaves[p].level;
    if (tree_ids) tree_ids[p] = f->pl.leaves[p].tree;
  }
  return FC_OK;
}

// ---- reflux across rank cuts ----------------------------------------------------------------
int fc_reflux_requests(fc_forest* f, int peer, int64_t* buf, int64_t cap, int64_t* len) {
  if (!f || !len) return fail(FC_EINVAL, "null argument");
  if (peer < 0 || peer >= f->pl.nranks) return fail(FC_EINVAL, "bad peer");
  if (!f->reflux_planned) return fail(FC_ESTATE, "set a problem with reflux = 1 first");
  const auto& v = f->rf_req[peer];
  *len = (int64_t)v.size();
  if (buf && cap >= *len) std::copy(v.begin(), v.end(), buf);
  else if (buf && *len) return fail(FC_EINVAL, "buffer too small");
  return FC_OK;
}

int fc_reflux_set_requests(fc_forest* f, int peer, const int64_t* keys, int64_t n) {
  if (!f || (n && !keys)) return fail(FC_EINVAL, "null argument");
  if (!f->manual) return fail(FC_ESTATE, "not a manual-transport handle");
  if (!f->reflux_planned) return fail(FC_ESTATE, "set a problem with reflux = 1 first");
  if (peer < 0 || peer >= f->pl.nranks) return fail(FC_EINVAL, "bad peer");
  f->rf_serve[peer].assign(keys, keys + n);
  return FC_OK;
}

int fc_reflux_finalize(fc_forest* f) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (!f->manual) return fail(FC_ESTATE, "not a manual-transport handle");
  if (!f->reflux_planned) return fail(FC_ESTATE, "set a problem with reflux = 1 first");
  CK(cudaSetDevice(f->device));
  return build_reflux_lists(f);
}

int fc_reflux_buffers(fc_forest* f, void** send, void** recv, int64_t* send_off, int64_t* recv_off) {
  if (!f || !send || !recv || !send_off || !recv_off) return fail(FC_EINVAL, "null argument");
  if (f->host_only || !f->reflux_planned || f->rf_send_off.size() != (size_t)f->pl.nranks + 1)
    return fail(FC_ESTATE, "no reflux exchange on this handle");
  *send = f->d_rf_send;
  *recv = f->d_freg + 4 * (int64_t)f->nslots * f->pl.m * f->pl.meqn;
  std::copy(f->rf_send_off.begin(), f->rf_send_off.end(), send_off);
  std::copy(f->rf_recv_off.begin(), f->rf_recv_off.end(), recv_off);
  return FC_OK;
}

// ---- staged step for a caller-provided halo transport (manual mode) ---------------------------
int fc_halo_set_requests(fc_forest* f, int round, int peer, const int64_t* keys, int64_t n) {
  if (!f || (n && !keys)) return fail(FC_EINVAL, "null argument");
  if (!f->manual) return fail(FC_ESTATE, "not a manual-transport handle");
  if (round != 1 && round != 2) return fail(FC_EINVAL, "round must be 1 or 2");
  if (peer < 0 || peer >= f->pl.nranks) return fail(FC_EINVAL, "bad peer");
  if (f->peer_req[round - 1].size() != (size_t)f->pl.nranks) f->peer_req[round - 1].assign(f->pl.nranks, {});
  f->peer_req[round - 1][peer].assign(keys, keys + n);
  return FC_OK;
}

int fc_halo_finalize(fc_forest* f) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (!f->manual) return fail(FC_ESTATE, "not a manual-transport handle");
  CK(cudaSetDevice(f->device));
  for (int r = 0; r < 2; ++r)
    if (f->peer_req[r].size() != (size_t)f->pl.nranks) f->peer_req[r].assign(f->pl.nranks, {});
  return build_halo_lists(f);
}

int fc_halo_buffers(fc_forest* f, int round, void** send, void** recv, int64_t* send_off, int64_t* recv_off) {
  if (!f || !send || !recv || !send_off || !recv_off) return fail(FC_EINVAL, "null argument");
  if (f->host_only || f->pl.nranks <= 1) return fail(FC_ESTATE, "no halo on this handle");
  if (round != 1 && round != 2) return fail(FC_EINVAL, "round must be 1 or 2");
  const int r = round - 1, R = f->pl.nranks, meqn = f->pl.meqn;
  *send = f->d_sendbuf;
  *recv = f->d_recvbuf;
  send_off[0] = recv_off[0] = 0;
  for (int s = 0; s < R; ++s) {
    send_off[s + 1] = send_off[s] + (f->send_cnt[r].empty() ? 0 : f->send_cnt[r][s]) * meqn;
    recv_off[s + 1] = recv_off[s] + (f->recv_cnt[r].empty() ? 0 : f->recv_cnt[r][s]) * meqn;
  }
  return FC_OK;
}

int fc_halo_pack(fc_forest* f, int round) {
  if (!f || (round != 1 && round != 2)) return fail(FC_EINVAL, "bad argument");
  if (f->host_only || !f->has_q) return fail(FC_ESTATE, "no state");
  CK(cudaSetDevice(f->device));
  int rc = halo_pack(f, round - 1, f->stream);
  if (rc) return rc;
  CK(cudaStreamSynchronize(f->stream));
  return FC_OK;
}

int fc_halo_unpack(fc_forest* f, int round) {
  if (!f || (round != 1 && round != 2)) return fail(FC_EINVAL, "bad argument");
  if (f->host_only || !f->has_q) return fail(FC_ESTATE, "no state");
  CK(cudaSetDevice(f->device));
  int rc = halo_unpack(f, round - 1, f->stream);
  if (rc) return rc;
  CK(cudaStreamSynchronize(f->stream));
  return FC_OK;
}

int fc_step_local(fc_forest* f, double dt, int phase, double* local_cfl) {
  int rc = check_step_args(f, dt);
  if (rc) return rc;
  CK(cudaSetDevice(f->device));
  if (phase == 1) {
    if (!use_fused(f) && (rc = ghost_phase_ac(f))) return rc;
  } else if (phase == 3) {   // after the caller moved the reflux records: apply the reflux
    if (f->prob.reflux && (rc = apply_reflux(f, dt))) return rc;
  } else if (phase == 4 || phase == 5) {   // split update (the halo overlap's two halves)
    if (!overlap_ok(f)) return fail(FC_EUNSUP, "split update: fused NCCL-halo path without filter / reflux only");
    if ((rc = update_local(f, dt, phase == 4 ? 1 : 2))) return rc;
    if (phase == 5) {
      CK(cudaMemcpyAsync(f->h_cfl, f->d_cfl, sizeof(double), cudaMemcpyDeviceToHost, f->stream));
      if (local_cfl) {
        CK(cudaStreamSynchronize(f->stream));
        *local_cfl = *f->h_cfl;
      }
    }
  } else if (phase == 2) {
    if (!use_fused(f) && (rc = ghost_phase_b(f))) return rc;
    if ((rc = update_local(f, dt))) return rc;
    CK(cudaMemcpyAsync(f->h_cfl, f->d_cfl, sizeof(double), cudaMemcpyDeviceToHost, f->stream));
    if (local_cfl) {
      CK(cudaStreamSynchronize(f->stream));
      *local_cfl = *f->h_cfl;
    }
  } else {
    return fail(FC_EINVAL, "phase must be 1 .. 5");
  }
  CK(cudaStreamSynchronize(f->stream));
  note_activity(f);
  return FC_OK;
}

int fc_p2p_buffers(fc_forest* f, void** buf0, void** buf1, int32_t* parity) {
  if (!f || !buf0 || !buf1 || !parity) return fail(FC_EINVAL, "null argument");
  if (f->host_only) return fail(FC_ESTATE, "host-only handle");
  *buf0 = f->buf[0];
  *buf1 = f->buf[1];
  *parity = f->parity;
  return FC_OK;
}

int fc_p2p_set_peer(fc_forest* f, int32_t peer, void* buf0, void* buf1) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (!f->p2p) return fail(FC_ESTATE, "not a peer-memory-halo handle (halo_p2p = 0 or not the fused path)");
  if (!f->manual) return fail(FC_ESTATE, "NCCL handles map their peers at creation");
  if (peer < 0 || peer >= f->pl.nranks || peer == f->pl.rank || !buf0 || !buf1) return fail(FC_EINVAL, "bad peer");
  f->peer_buf[peer] = {(double*)buf0, (double*)buf1};
  return FC_OK;
}

int fc_commit(fc_forest* f, double global_cfl) {
  if (!f) return fail(FC_EINVAL, "null handle");
  if (f->host_only || !f->has_q) return fail(FC_ESTATE, "no state");
  return commit(f, global_cfl);
}

}  // extern "C"
