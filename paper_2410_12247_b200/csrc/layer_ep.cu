// The EP > 1 forward (Algorithm 1): count exchange (C3), plan,
// all2all layouts, and the chunked dispatch / ComputeMoE / combine over the
// transport (NCCL, the host-collective bootstrap or the in-process test group)
// or the layer's own peer-memory planes (put kernels, copy engines).
//
// Phases (one host wait, for the counts; everything after is stream-ordered):
//   ep_counts        allgather of the histogram, plan, send / recv layouts (R6),
//                    token-sliced counts (R8), per-chunk GEMM row tables
//   ep_lr_layout     local_reduce (R16): dedup permute + unique-row exchange
//   ep_p2p_tables    a2a_p2p: per-(direction, chunk) peer segments and flags
//   Algorithm 1      dispatch(0); for p: dispatch(p), compute(p-1), combine(p-2);
//                    combine(PN-1); then the weighted unpermute (LocalReduce)
#include "layer_impl.h"

#include <nvtx3/nvToolsExt.h>

namespace epsmoe {
namespace {

// NVTX range over one host-side phase (visible in nsys timelines).
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

// Host-side state of one EP forward.  Every rank derives the same tables from
// the same global counts, so a rank can address its peers' buffers directly.
struct Ep {
  Fwd& F;
  moe_layer* L;
  const moe_config_t& c;
  moe_plan_t& plan;
  cudaStream_t st;
  int E, k, H, D, E_loc, me;
  bool fp8, lr;
  // pairs per (rank, expert, token slice): [D][E * S] (R8 extension)
  int S = 1;
  const int32_t* hsl = nullptr;
  std::vector<int64_t> send_off, recv_off, send_pos, recv_pos;
  int32_t *tstart = nullptr, *tcount = nullptr;  // per-chunk GEMM row tables (host mirror)
  // local_reduce (R16): G = PN * D groups, unique rows per (rank, group)
  int G = 0;
  const int32_t* ug = nullptr;
  std::vector<int64_t> usend_off, urecv;
  // peer-memory planes (a2a_p2p)
  bool p2p = false, copy_engine = false;
  uint32_t epoch = 0;
  int comm_ctas = 0;  // CTAs per put direction / 2, NCCL maxCTAs (plan.comm_ctas, NEXT-1)
  int nseg[2][MOE_MAX_CHUNKS] = {};
  int64_t total[2][MOE_MAX_CHUNKS] = {};
  bool fuse_comb[MOE_MAX_CHUNKS] = {};  // the chunk's DownGemm stores its rows at home (fused combine)
  int fuse_nrseg[MOE_MAX_CHUNKS] = {};
  // SM partition (NEXT-1): with a GEMM grid below the SM count, every
  // persistent GEMM of the forward runs on the caller's stream (one grid
  // resident at a time), so the reserved SMs stay free for the all2all
  bool capped = false;
  bool two_streams = false;

  Ep(Fwd& f)
      : F(f), L(f.L), c(f.L->cfg), plan(f.plan), st(f.st), E(c.num_experts), k(c.top_k), H(c.hidden), D(c.ep),
        E_loc(f.L->E_loc), me(c.rank), fp8(f.fp8), lr(f.lr_ep) {}
  int64_t cnt(int src, int ex, int sl) const { return hsl[((int64_t)src * E + ex) * S + sl]; }
  int64_t rpos(int el, int sl, int src) const { return recv_pos[((size_t)el * S + sl) * D + src]; }
  int slice(int ch) const { return ch % S; }
  int g0(int ch) const { return plan.group_begin[ch / S]; }
  int g1(int ch) const { return plan.group_begin[ch / S + 1]; }
  cudaStream_t comp_stream(int ch) const { return (two_streams && (ch & 1)) ? L->s_comp2 : st; }
  size_t row_bytes() const { return (size_t)H * 2; }
  size_t drow() const { return fp8 ? (size_t)L->qpitch : row_bytes(); }  // dispatch payload row
  char* dsend() const { return fp8 ? (char*)L->sendq : (char*)L->send; }
  char* drecv() const { return fp8 ? (char*)L->recvq : (char*)L->recv; }
};

// The one host wait of a forward: the count exchange's device->host copy.
// Polls instead of blocking so that an asynchronous collective error
// (ncclCommGetAsyncError) surfaces as MOE_ERR_NCCL instead of a hang.
moe_status_t wait_counts(moe_layer* L, cudaStream_t st) {
  CUDA_TRY(cudaEventRecord(L->ev_hist, st));
  for (;;) {
    const cudaError_t q = cudaEventQuery(L->ev_hist);
    if (q == cudaSuccess) return MOE_OK;
    if (q != cudaErrorNotReady) {
      set_error(std::string("count exchange: ") + cudaGetErrorString(q));
      return MOE_ERR_CUDA;
    }
    if (int e = L->tr->poll_async()) return (moe_status_t)e;
  }
}

// Count exchange (C3), plan, layouts (R6, R8), per-chunk GEMM row tables.
moe_status_t ep_counts(Ep& X) {
  moe_layer* L = X.L;
  const int E = X.E, D = X.D, E_loc = X.E_loc, me = X.me;
  TR_TRY(L->tr->allgather_i32(L->hist, L->ghist, E, X.st));
  CUDA_TRY(cudaMemcpyAsync(L->ghist_host, L->ghist, sizeof(int32_t) * D * E, cudaMemcpyDeviceToHost, X.st));
  if (moe_status_t r = wait_counts(L, X.st)) return r;
  const int32_t* gh = L->ghist_host;
  if (!X.F.plan_in) {
    int64_t m = 0;
    for (int i = 0; i < D * E; ++i) m += gh[i];
    plan_compute(X.c, L->cost, m / X.k, gh, &X.plan);
    // the planner's SM partition applies to the chunk GEMMs (NEXT-1)
    if (X.plan.sm_gemm > 0) X.F.num_ctas = std::min(X.plan.sm_gemm, L->num_sms);
  }
  X.comm_ctas = X.plan.comm_ctas > 0 ? X.plan.comm_ctas : L->comm_ctas;
  // send offsets (local, expert-major) and recv layout [e_l][src] (R6)
  X.send_off.assign(E + 1, 0);
  X.recv_off.assign((size_t)E_loc * D + 1, 0);
  exchange_layout(X.c, gh, X.send_off.data(), X.recv_off.data());
  if (X.recv_off.back() > L->recv_cap) { set_error("recv rows exceed capacity"); return MOE_ERR_CAPACITY; }
  // Token-sliced chunks (R8 extension, S > 1): chunk c = (expert group c / S,
  // source-token slice c % S); the (expert, slice) counts of every rank take
  // one more exchange.  Send rows stay (e, t), so (e, s) is contiguous; recv
  // rows become (e_l, s, src, t), so each expert's rows of a chunk are.  Every
  // row still meets the same weights and returns to the same send row, so
  // slicing changes no bit of y.
  X.S = X.plan.token_slices;
  const int S = X.S;
  X.hsl = gh;
  if (S > 1) {
    KERNEL_TRY(launch_slice_hist(X.F.topk_idx, (int)X.F.T, X.k, E, S, L->slice_hist, X.st));
    TR_TRY(L->tr->allgather_i32(L->slice_hist, L->gslice, E * S, X.st));
    CUDA_TRY(cudaMemcpyAsync(L->gslice_host, L->gslice, sizeof(int32_t) * D * E * S, cudaMemcpyDeviceToHost, X.st));
    if (moe_status_t r = wait_counts(L, X.st)) return r;
    X.hsl = L->gslice_host;
  }
  X.send_pos.assign((size_t)E * S, 0);
  for (int ex = 0; ex < E; ++ex) {
    int64_t p0 = X.send_off[ex];
    for (int sl = 0; sl < S; ++sl) {
      X.send_pos[(size_t)ex * S + sl] = p0;
      p0 += X.cnt(me, ex, sl);
    }
  }
  X.recv_pos.assign((size_t)E_loc * S * D + 1, 0);  // (e_l, s, src)
  for (int el = 0, i = 0; el < E_loc; ++el)
    for (int sl = 0; sl < S; ++sl)
      for (int src = 0; src < D; ++src, ++i) X.recv_pos[i + 1] = X.recv_pos[i] + X.cnt(src, me * E_loc + el, sl);
  // per-chunk GEMM row tables: chunk c's experts at [c * E_loc + e_l]
  X.tstart = L->tables_host;
  X.tcount = L->tables_host + moe_layer::TBL;
  for (int ch = 0; ch < X.plan.num_chunks; ++ch) {
    const int sl = X.slice(ch);
    for (int el = X.g0(ch); el < X.g1(ch); ++el) {
      X.tstart[ch * E_loc + el] = (int32_t)X.rpos(el, sl, 0);
      X.tcount[ch * E_loc + el] =
          (int32_t)(X.rpos(el, sl, D - 1) + X.cnt(D - 1, me * E_loc + el, sl) - X.rpos(el, sl, 0));
    }
  }
  const size_t tbytes = sizeof(int32_t) * (size_t)X.plan.num_chunks * E_loc;
  CUDA_TRY(cudaMemcpyAsync(L->recv_start_d, X.tstart, tbytes, cudaMemcpyHostToDevice, X.st));
  CUDA_TRY(cudaMemcpyAsync(L->recv_count_d, X.tcount, tbytes, cudaMemcpyHostToDevice, X.st));
  return MOE_OK;
}

// local_reduce (R16): the dedup layout needs the plan's chunks, and the
// unique-row counts per (chunk, peer) need a second (G-int) exchange.
moe_status_t ep_lr_layout(Ep& X) {
  moe_layer* L = X.L;
  const int D = X.D, E_loc = X.E_loc, me = X.me, PN = X.plan.num_chunks;
  const int G = X.G = PN * D;
  X.usend_off.assign(G + 1, 0);       // my send rows of group g = c*D + peer
  X.urecv.assign((size_t)G + 1, 0);   // first unique recv row of (c, src)
  X.ug = L->ughist_host;              // [D][G]
  if (!X.lr) return MOE_OK;
  const int T = (int)X.F.T;
  int q0 = prof_rec(L, X.st);
  LrChunks chs;
  chs.n = PN;
  for (int i = 0; i <= PN; ++i) chs.begin[i] = X.plan.group_begin[i];
  KERNEL_TRY(launch_lr_count(X.F.topk_idx, T, X.k, E_loc, D, chs, L->range_hist, X.st));
  KERNEL_TRY(launch_range_scan(L->range_hist, T, G, L->range_off, L->u_hist, L->u_start, X.st));
  KERNEL_TRY(launch_lr_permute(X.F.x, T, X.H, X.k, X.F.topk_idx, X.F.topk_w, L->pos, L->seg_start, E_loc, D, chs,
                               L->range_off, L->u_start, X.fp8 ? nullptr : L->send, X.fp8 ? L->sendq : nullptr,
                               L->qpitch, L->posg, L->meta_send, X.st));
  prof_mark(L, MOE_STAGE_ROUTE, q0, prof_rec(L, X.st));
  TR_TRY(L->tr->allgather_i32(L->u_hist, L->ughist, G, X.st));
  CUDA_TRY(cudaMemcpyAsync(L->ughist_host, L->ughist, sizeof(int32_t) * D * G, cudaMemcpyDeviceToHost, X.st));
  if (moe_status_t r = wait_counts(L, X.st)) return r;
  const int32_t* ug = X.ug;
  for (int g = 0; g < G; ++g) X.usend_off[g + 1] = X.usend_off[g] + ug[(size_t)me * G + g];
  int64_t row = 0;
  for (int ch = 0; ch < PN; ++ch)
    for (int src = 0; src < D; ++src) {
      X.urecv[(size_t)ch * D + src] = row;
      row += ug[(size_t)src * G + ch * D + me];
    }
  X.urecv[G] = row;
  if (row > L->recv_cap) { set_error("unique recv rows exceed capacity"); return MOE_ERR_CAPACITY; }
  int32_t* tb = L->tables_host + 2 * moe_layer::TBL;  // [E_loc*D+1] recv_off, then [G+1] urecv
  for (int i = 0; i <= E_loc * D; ++i) tb[i] = (int32_t)X.recv_off[i];
  for (int i = 0; i <= G; ++i) tb[MOE_MAX_EXPERTS + 4 + i] = (int32_t)X.urecv[i];
  CUDA_TRY(cudaMemcpyAsync(L->lr_recv_off_d, tb, sizeof(int32_t) * (E_loc * D + 1), cudaMemcpyHostToDevice, X.st));
  CUDA_TRY(cudaMemcpyAsync(L->lr_usrc_d, tb + MOE_MAX_EXPERTS + 4, sizeof(int32_t) * (G + 1), cudaMemcpyHostToDevice,
                           X.st));
  return MOE_OK;
}

}  // namespace

// First p2p use (collective): map every rank's workspace, learn the byte
// offsets of the buffers peers write into (a rank's max_tokens, hence its
// workspace layout, may differ from its peers').
moe_status_t p2p_map_peers(moe_layer* L, cudaStream_t st) {
  if (!L->peer_ws.empty()) return MOE_OK;
  const int D = L->cfg.ep;
  TR_TRY(L->tr->map_peers(L->ws_base, L->peer_ws));
  const void* bufs[moe_layer::P2P_NBUF] = {L->recv, L->recvq, L->recvu, L->meta_recv, L->comb, L->p2p_flags};
  int64_t mine[moe_layer::P2P_NBUF];
  for (int b = 0; b < moe_layer::P2P_NBUF; ++b) mine[b] = bufs[b] ? (int64_t)((const char*)bufs[b] - L->ws_base) : -1;
  constexpr int W = 2 * moe_layer::P2P_NBUF;
  int32_t* dev = nullptr;
  CUDA_TRY(cudaMalloc(&dev, sizeof(int32_t) * W * (D + 1)));
  CUDA_TRY(cudaMemcpy(dev, mine, sizeof(mine), cudaMemcpyHostToDevice));
  int ge = L->tr->allgather_i32(dev, dev + W, W, st);
  L->peer_off.assign((size_t)D * moe_layer::P2P_NBUF, -1);
  if (!ge) {
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaMemcpy(L->peer_off.data(), dev + W, sizeof(int64_t) * D * moe_layer::P2P_NBUF,
                        cudaMemcpyDeviceToHost));
  }
  cudaFree(dev);
  return (moe_status_t)ge;
}

// Calibration (moe_layer_calibrate): one all2all in which every rank sends
// `per` bytes of its send buffer to every peer, on this layer's data plane
// with a comm budget of `ctas` (NCCL maxCTAs / put CTAs per direction / 2);
// *ms = this rank's time from issue to all of its rows received.  Collective.
moe_status_t time_all2all(moe_layer* L, int ctas, int64_t per, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1,
                          float* ms) {
  const moe_config_t& c = L->cfg;
  const int D = c.ep, me = c.rank;
  if (c.a2a_p2p) CUDA_TRY_STATUS(p2p_map_peers(L, st));
  TR_TRY(L->tr->allgather_i32(L->hist, L->ghist, 1, st));  // ranks start together
  CUDA_TRY(cudaStreamSynchronize(st));
  if (c.a2a_p2p == 0) {
    TR_TRY(L->tr->set_comm_ctas(ctas));
    CUDA_TRY(cudaEventRecord(e0, L->s_disp));
    TR_TRY(L->tr->group_start(0));
    for (int peer = 0; peer < D; ++peer) {
      TR_TRY(L->tr->send((char*)L->send + peer * per, per, peer, 0, L->s_disp));
      TR_TRY(L->tr->recv((char*)L->recv + peer * per, per, peer, 0, L->s_disp));
    }
    TR_TRY(L->tr->group_end(0, L->s_disp));
  } else {
    // slot 0 (dispatch, chunk 0) of the peer-memory tables: rows of peer d go to
    // d's receive buffer at my offset
    const uint32_t epoch = ++L->p2p_epoch;
    auto* hsegs = reinterpret_cast<P2PSeg*>(L->p2p_host);
    auto* hpre = reinterpret_cast<int64_t*>(L->p2p_host + P2P_SEGS_BYTES);
    auto* hfp = reinterpret_cast<uint32_t**>(L->p2p_host + P2P_SEGS_BYTES + P2P_PRE_BYTES);
    hpre[0] = 0;
    for (int d = 0; d < D; ++d) {
      char* base = L->peer_ws[d];
      hsegs[d].src = reinterpret_cast<const uint4*>((char*)L->send + d * per);
      hsegs[d].dst = reinterpret_cast<uint4*>(base + L->peer_off[(size_t)d * moe_layer::P2P_NBUF + moe_layer::P2P_RECV] +
                                              me * per);
      hpre[d + 1] = hpre[d] + per / 16;
      hfp[d] = reinterpret_cast<uint32_t*>(base + L->peer_off[(size_t)d * moe_layer::P2P_NBUF + moe_layer::P2P_FLAGS] +
                                           (int64_t)me * 4);
    }
    CUDA_TRY(cudaMemcpyAsync(L->p2p_tab, L->p2p_host, p2p_table_bytes(D), cudaMemcpyHostToDevice, L->s_disp));
    CUDA_TRY(cudaEventRecord(e0, L->s_disp));
    auto* dsegs = reinterpret_cast<P2PSeg*>(L->p2p_tab);
    auto* dpre = reinterpret_cast<int64_t*>(L->p2p_tab + P2P_SEGS_BYTES);
    auto* dfp = reinterpret_cast<uint32_t**>(L->p2p_tab + P2P_SEGS_BYTES + P2P_PRE_BYTES);
    if (c.a2a_p2p == 2) {
      for (int d = 0; d < D; ++d)
        CUDA_TRY(cudaMemcpyAsync(hsegs[d].dst, hsegs[d].src, per, cudaMemcpyDeviceToDevice, L->s_disp));
      KERNEL_TRY(launch_p2p_signal(dfp, D, epoch, L->s_disp));
    } else {
      KERNEL_TRY(launch_p2p_put(dsegs, dpre, D, hpre[D], 2 * ctas, L->p2p_done, dfp, D, epoch, L->s_disp));
    }
    TR_TRY(L->tr->p2p_after_put(0, L->s_disp));
    TR_TRY(L->tr->p2p_before_wait(0, 1, L->s_disp));
    KERNEL_TRY(launch_p2p_wait(L->p2p_flags, D, epoch, L->s_disp));
  }
  CUDA_TRY(cudaEventRecord(e1, L->s_disp));
  CUDA_TRY(cudaEventSynchronize(e1));
  CUDA_TRY(cudaEventElapsedTime(ms, e0, e1));
  return MOE_OK;
}

namespace {

// a2a_p2p: this forward's segments (rows of each chunk, per peer, at the peer's
// own offsets), the consumer flag addresses, and the fused-combine row table.
moe_status_t ep_p2p_tables(Ep& X) {
  moe_layer* L = X.L;
  const int E = X.E, D = X.D, E_loc = X.E_loc, me = X.me, S = X.S, G = X.G;
  const moe_plan_t& plan = X.plan;
  if (moe_status_t r = p2p_map_peers(L, X.st)) return r;
  X.epoch = ++L->p2p_epoch;
  // address, in peer d's workspace, of byte `off` of its buffer b
  auto peer_buf = [&](int d, int b, int64_t off) -> char* {
    return L->peer_ws[d] + L->peer_off[(size_t)d * moe_layer::P2P_NBUF + b] + off;
  };
  // every rank's layout, from the same global counts
  const size_t RP = (size_t)E_loc * S * D;
  std::vector<int64_t> rpos_all((size_t)D * RP), spos_all((size_t)D * E * S);
  for (int d = 0; d < D; ++d) {
    int64_t row = 0;
    for (int el = 0; el < E_loc; ++el)
      for (int sl = 0; sl < S; ++sl)
        for (int src = 0; src < D; ++src) {
          rpos_all[d * RP + ((size_t)el * S + sl) * D + src] = row;
          row += X.cnt(src, d * E_loc + el, sl);
        }
    row = 0;
    for (int ex = 0; ex < E; ++ex)
      for (int sl = 0; sl < S; ++sl) {
        spos_all[(size_t)d * E * S + (size_t)ex * S + sl] = row;
        row += X.cnt(d, ex, sl);
      }
  }
  const int32_t* ug = X.ug;
  std::vector<int64_t> urecv_all, usend_all;
  if (X.lr) {
    urecv_all.assign((size_t)D * (G + 1), 0);
    usend_all.assign((size_t)D * (G + 1), 0);
    for (int d = 0; d < D; ++d) {
      int64_t row = 0;
      for (int ch = 0; ch < plan.num_chunks; ++ch)
        for (int src = 0; src < D; ++src) {
          urecv_all[(size_t)d * (G + 1) + ch * D + src] = row;
          row += ug[(size_t)src * G + ch * D + d];
        }
      for (int g = 0; g < G; ++g)
        usend_all[(size_t)d * (G + 1) + g + 1] = usend_all[(size_t)d * (G + 1) + g] + ug[(size_t)d * G + g];
    }
  }
  auto* hsegs = reinterpret_cast<P2PSeg*>(L->p2p_host);
  auto* hpre = reinterpret_cast<int64_t*>(L->p2p_host + P2P_SEGS_BYTES);
  auto* hfp = reinterpret_cast<uint32_t**>(L->p2p_host + P2P_SEGS_BYTES + P2P_PRE_BYTES);
  const size_t rowb = X.row_bytes(), drowb = X.drow();
  const size_t metab = (size_t)lr_meta_pitch(X.k) * sizeof(int32_t);
  char* ds = X.dsend();
  const int dr_id = X.fp8 ? moe_layer::P2P_RECVQ : (X.lr ? moe_layer::P2P_RECVU : moe_layer::P2P_RECV);
  bool overflow = false;
  for (int dir = 0; dir < 2; ++dir)
    for (int ch = 0; ch < plan.num_chunks; ++ch) {
      const size_t slot = (size_t)dir * MOE_MAX_CHUNKS + ch;
      P2PSeg* sg = hsegs + slot * moe_layer::P2P_MAXS;
      int64_t* pr = hpre + slot * (moe_layer::P2P_MAXS + 1);
      int n = 0;
      pr[0] = 0;
      auto add = [&](const char* src, char* dst, int64_t bytes) {
        if (bytes <= 0) return;
        if (n >= moe_layer::P2P_MAXS) { overflow = true; return; }
        sg[n].src = reinterpret_cast<const uint4*>(src);
        sg[n].dst = reinterpret_cast<uint4*>(dst);
        pr[n + 1] = pr[n] + bytes / 16;
        ++n;
      };
      for (int d = 0; d < D; ++d)
        hfp[slot * D + d] = reinterpret_cast<uint32_t*>(peer_buf(d, moe_layer::P2P_FLAGS, (int64_t)(slot * D + me) * 4));
      const int sl = X.slice(ch), g0 = X.g0(ch), g1 = X.g1(ch);
      for (int peer = 0; peer < D; ++peer) {
        if (X.lr && dir == 0) {
          const int64_t s0 = X.usend_off[ch * D + peer], ns = ug[(size_t)me * G + ch * D + peer];
          const int64_t r0 = urecv_all[(size_t)peer * (G + 1) + ch * D + me];
          add(ds + s0 * drowb, peer_buf(peer, dr_id, r0 * drowb), ns * (int64_t)drowb);
          add((char*)L->meta_send + s0 * metab, peer_buf(peer, moe_layer::P2P_META, r0 * metab), ns * (int64_t)metab);
        } else if (X.lr) {
          const int64_t r0 = X.urecv[(size_t)ch * D + peer], nb = ug[(size_t)peer * G + ch * D + me];
          const int64_t s0 = usend_all[(size_t)peer * (G + 1) + ch * D + me];
          add((char*)L->recvu + r0 * rowb, peer_buf(peer, moe_layer::P2P_COMB, s0 * rowb), nb * (int64_t)rowb);
        } else {
          for (int el = g0; el < g1; ++el) {
            if (dir == 0) {
              const int ex = peer * E_loc + el;
              add(ds + X.send_pos[(size_t)ex * S + sl] * drowb,
                  peer_buf(peer, dr_id, rpos_all[peer * RP + ((size_t)el * S + sl) * D + me] * drowb),
                  X.cnt(me, ex, sl) * (int64_t)drowb);
            } else {
              const int ex = me * E_loc + el;
              add((char*)L->o + X.rpos(el, sl, peer) * rowb,
                  peer_buf(peer, moe_layer::P2P_COMB, spos_all[(size_t)peer * E * S + (size_t)ex * S + sl] * rowb),
                  X.cnt(peer, ex, sl) * (int64_t)rowb);
            }
          }
        }
      }
      X.nseg[dir][ch] = n;
      X.total[dir][ch] = pr[n];
      // Fused combine: the chunk's DownGemm stores every output row straight
      // into its home rank's combine buffer.  Not on the copy-engine plane
      // (there the combine rows move on the copy engines too, so no SM stores
      // a row of either direction) and not with LocalReduce (its partials need
      // all of a row's experts first).  A chunk of several DENSE experts runs
      // as several launches; only the last raises the flags (compute_moe).
      if (dir == 1 && L->p2p_fuse && !X.copy_engine && !X.lr && !L->split_rem && !L->comm_only) {
        bool one_kind = true;
        for (int el = g0 + 1; el < g1; ++el) one_kind &= plan.expert_kind[el] == plan.expert_kind[g0];
        if (one_kind) {
          auto* rs = reinterpret_cast<GemmRowSeg*>(L->p2p_host + P2P_SEGS_BYTES + P2P_PRE_BYTES + p2p_fptr_bytes(D)) +
                     (size_t)ch * moe_layer::P2P_MAXS;
          int nr = 0;
          for (int el = g0; el < g1; ++el)  // GEMM rows (e_l, slice, src) ascending
            for (int src = 0; src < D; ++src) {
              const int ex = me * E_loc + el;
              const int64_t rows = X.cnt(src, ex, sl);
              if (!rows) continue;
              if (nr >= moe_layer::P2P_MAXS) { overflow = true; continue; }
              rs[nr].r0 = X.rpos(el, sl, src);
              rs[nr].n = rows;
              rs[nr].dst = peer_buf(src, moe_layer::P2P_COMB, spos_all[(size_t)src * E * S + (size_t)ex * S + sl] * rowb);
              ++nr;
            }
          X.fuse_comb[ch] = true;
          X.fuse_nrseg[ch] = nr;
        }
      }
    }
  if (overflow) {  // cannot happen for E <= 256 (segments per chunk <= D * E_loc <= E)
    set_error("a2a_p2p: more segments per chunk than the table holds");
    return MOE_ERR_UNSUPPORTED;
  }
  CUDA_TRY(cudaMemcpyAsync(L->p2p_tab, L->p2p_host, p2p_table_bytes(D), cudaMemcpyHostToDevice, X.st));
  return MOE_OK;
}

// One direction of one chunk on the peer-memory planes: the put kernel's
// stores (2 * comm_ctas CTAs), or the copy engines' peer copies followed by a
// one-thread flag kernel.
moe_status_t ep_put(Ep& X, int dir, int ch, cudaStream_t ps) {
  moe_layer* L = X.L;
  const int D = X.D;
  const size_t slot = (size_t)dir * MOE_MAX_CHUNKS + ch;
  auto* dsegs = reinterpret_cast<P2PSeg*>(L->p2p_tab) + slot * moe_layer::P2P_MAXS;
  auto* dpre = reinterpret_cast<int64_t*>(L->p2p_tab + P2P_SEGS_BYTES) + slot * (moe_layer::P2P_MAXS + 1);
  auto* dfp = reinterpret_cast<uint32_t**>(L->p2p_tab + P2P_SEGS_BYTES + P2P_PRE_BYTES) + slot * D;
  if (X.copy_engine) {
    const auto* hs = reinterpret_cast<const P2PSeg*>(L->p2p_host) + slot * moe_layer::P2P_MAXS;
    const auto* hp = reinterpret_cast<const int64_t*>(L->p2p_host + P2P_SEGS_BYTES) + slot * (moe_layer::P2P_MAXS + 1);
    const int n = X.nseg[dir][ch];
    if (n > 0) {
      // one cudaMemcpyAsync per run of segments that are contiguous on both
      // sides (the batched copy API is closed on this pool: it raised GPU
      // faults); each copy is a peer copy on the copy engines
      int i = 0;
      while (i < n) {
        char* dst = reinterpret_cast<char*>(hs[i].dst);
        const char* src = reinterpret_cast<const char*>(hs[i].src);
        size_t bytes = (size_t)(hp[i + 1] - hp[i]) * 16;
        int j = i + 1;
        while (j < n && reinterpret_cast<char*>(hs[j].dst) == dst + bytes &&
               reinterpret_cast<const char*>(hs[j].src) == src + bytes) {
          bytes += (size_t)(hp[j + 1] - hp[j]) * 16;
          ++j;
        }
        if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ps));
        i = j;
      }
    }
    KERNEL_TRY(launch_p2p_signal(dfp, D, X.epoch, ps));
  } else {
    KERNEL_TRY(launch_p2p_put(dsegs, dpre, X.nseg[dir][ch], X.total[dir][ch], 2 * X.comm_ctas, L->p2p_done + slot,
                              dfp, D, X.epoch, ps));
  }
  TR_TRY(L->tr->p2p_after_put((int)slot, ps));
  return MOE_OK;
}

// All2All dispatch of chunk ch on s_disp.
moe_status_t ep_dispatch(Ep& X, int ch) {
  moe_layer* L = X.L;
  const int D = X.D, E_loc = X.E_loc, me = X.me, G = X.G, S = X.S;
  Nvtx nv("epsmoe dispatch");
  int d0 = prof_rec(L, L->s_disp);
  if (X.p2p) {
    if (moe_status_t r = ep_put(X, 0, ch, L->s_disp)) return r;
  } else {
    const size_t drow = X.drow();
    const size_t meta_bytes = (size_t)lr_meta_pitch(X.k) * sizeof(int32_t);
    TR_TRY(L->tr->group_start(0));
    if (X.lr) {  // one unique-row message + its meta per peer (R16)
      char* urows = X.fp8 ? (char*)L->recvq : (char*)L->recvu;
      for (int peer = 0; peer < D; ++peer) {
        const int64_t s0 = X.usend_off[ch * D + peer], ns = X.ug[(size_t)me * G + ch * D + peer];
        if (ns) {
          TR_TRY(L->tr->send(X.dsend() + s0 * drow, ns * drow, peer, 0, L->s_disp));
          TR_TRY(L->tr->send((char*)L->meta_send + s0 * meta_bytes, ns * meta_bytes, peer, 0, L->s_disp));
        }
        const int64_t r0 = X.urecv[(size_t)ch * D + peer], nr = X.ug[(size_t)peer * G + ch * D + me];
        if (nr) {
          TR_TRY(L->tr->recv(urows + r0 * drow, nr * drow, peer, 0, L->s_disp));
          TR_TRY(L->tr->recv((char*)L->meta_recv + r0 * meta_bytes, nr * meta_bytes, peer, 0, L->s_disp));
        }
      }
    } else {
      const int sl = X.slice(ch);
      for (int peer = 0; peer < D; ++peer)
        for (int el = X.g0(ch); el < X.g1(ch); ++el) {
          const int ex = peer * E_loc + el;
          const int64_t n_send = X.cnt(me, ex, sl);
          if (n_send)
            TR_TRY(L->tr->send(X.dsend() + X.send_pos[(size_t)ex * S + sl] * drow, n_send * drow, peer, 0, L->s_disp));
          const int64_t n_recv = X.cnt(peer, me * E_loc + el, sl);
          if (n_recv) TR_TRY(L->tr->recv(X.drecv() + X.rpos(el, sl, peer) * drow, n_recv * drow, peer, 0, L->s_disp));
        }
    }
    TR_TRY(L->tr->group_end(0, L->s_disp));
  }
  prof_mark(L, MOE_STAGE_DISPATCH, d0, prof_rec(L, L->s_disp));
  CUDA_TRY(cudaEventRecord(L->ev_disp[ch], L->s_disp));
  return MOE_OK;
}

// All2All combine of chunk ch on s_comb, after the chunk's GEMMs.
moe_status_t ep_combine(Ep& X, int ch) {
  moe_layer* L = X.L;
  const int D = X.D, E_loc = X.E_loc, me = X.me, G = X.G, S = X.S;
  Nvtx nv("epsmoe combine");
  CUDA_TRY(cudaStreamWaitEvent(L->s_comb, L->ev_gemm[ch], 0));
  int b0 = prof_rec(L, L->s_comb);
  if (X.p2p) {
    if (!X.fuse_comb[ch])
      if (moe_status_t r = ep_put(X, 1, ch, L->s_comb)) return r;
  } else {
    const size_t row_bytes = X.row_bytes();
    TR_TRY(L->tr->group_start(1));
    if (X.lr) {  // each unique row returns as its LocalReduce partial (R16)
      for (int peer = 0; peer < D; ++peer) {
        const int64_t r0 = X.urecv[(size_t)ch * D + peer], nb = X.ug[(size_t)peer * G + ch * D + me];
        if (nb) TR_TRY(L->tr->send((char*)L->recvu + r0 * row_bytes, nb * row_bytes, peer, 1, L->s_comb));
        const int64_t s0 = X.usend_off[ch * D + peer], nh = X.ug[(size_t)me * G + ch * D + peer];
        if (nh) TR_TRY(L->tr->recv((char*)L->comb + s0 * row_bytes, nh * row_bytes, peer, 1, L->s_comb));
      }
    } else {
      const int sl = X.slice(ch);
      for (int peer = 0; peer < D; ++peer)
        for (int el = X.g0(ch); el < X.g1(ch); ++el) {
          const int64_t n_back = X.cnt(peer, me * E_loc + el, sl);
          if (n_back)
            TR_TRY(L->tr->send((char*)L->o + X.rpos(el, sl, peer) * row_bytes, n_back * row_bytes, peer, 1,
                               L->s_comb));
          const int ex = peer * E_loc + el;
          const int64_t n_home = X.cnt(me, ex, sl);
          if (n_home)
            TR_TRY(L->tr->recv((char*)L->comb + X.send_pos[(size_t)ex * S + sl] * row_bytes, n_home * row_bytes, peer,
                               1, L->s_comb));
        }
    }
    TR_TRY(L->tr->group_end(1, L->s_comb));
  }
  prof_mark(L, MOE_STAGE_COMB_A2A, b0, prof_rec(L, L->s_comb));
  return MOE_OK;
}

// ComputeMoE of chunk ch once its dispatch arrived.
moe_status_t ep_compute(Ep& X, int ch) {
  moe_layer* L = X.L;
  const int D = X.D, E_loc = X.E_loc, me = X.me, H = X.H, k = X.k;
  const moe_plan_t& plan = X.plan;
  Nvtx nv("epsmoe compute");
  const int sl = X.slice(ch), g0 = X.g0(ch), g1 = X.g1(ch);
  cudaStream_t cs = X.comp_stream(ch);
  CUDA_TRY(cudaStreamWaitEvent(cs, L->ev_disp[ch], 0));  // (p2p: my puts read `send`)
  if (X.p2p) {  // every source's rows
    TR_TRY(L->tr->p2p_before_wait(ch, 1, cs));
    KERNEL_TRY(launch_p2p_wait(L->p2p_flags + (size_t)ch * D, D, X.epoch, cs));
  }
  if (L->comm_only) {  // measurement: the chunk's all2all without its ComputeMoE
    CUDA_TRY(cudaEventRecord(L->ev_gemm[ch], cs));
    return MOE_OK;
  }
  const int64_t u0 = X.urecv[(size_t)ch * D], u1 = X.urecv[(size_t)(ch + 1) * D];
  const size_t row_bytes = X.row_bytes(), drow = X.drow();
  if (X.lr) {  // unique rows -> expert-major GEMM rows (R6 order, so the GEMMs are unchanged)
    KERNEL_TRY(launch_lr_expand(L->recvu, X.fp8 ? L->recvq : nullptr, L->qpitch, u0, u1, H, k, D, ch, L->lr_usrc_d,
                                L->lr_recv_off_d, L->meta_recv, L->recv, cs));
  } else if (X.fp8) {  // the chunk's rows: one range per expert, merged where contiguous (all, if S == 1)
    int el = g0;
    while (el < g1) {
      const int64_t r0 = X.rpos(el, sl, 0);
      int64_t r1 = X.rpos(el, sl, D - 1) + X.cnt(D - 1, me * E_loc + el, sl);
      while (++el < g1 && X.rpos(el, sl, 0) == r1) r1 = X.rpos(el, sl, D - 1) + X.cnt(D - 1, me * E_loc + el, sl);
      KERNEL_TRY(launch_dequant_rows(X.drecv() + r0 * drow, r1 - r0, H, L->qpitch, (char*)L->recv + r0 * row_bytes, cs));
    }
  }
  int a = g0;
  while (a < g1) {
    int b = a + 1;
    while (b < g1 && plan.expert_kind[b] == plan.expert_kind[a]) ++b;
    double rows = 0;
    for (int el = a; el < b; ++el) rows += X.tcount[ch * E_loc + el];
    const bool fz = X.p2p && X.fuse_comb[ch];
    const size_t cslot = (size_t)MOE_MAX_CHUNKS + ch;
    int err = compute_moe(
        L, L->recv, L->recv_cap, L->recv_start_d + ch * E_loc, L->recv_count_d + ch * E_loc, a, b,
        plan.expert_kind[a], X.F.num_ctas, pick_cta_pair(plan, rows / (b - a)), plan.tile_m != 0, rows / (b - a), cs,
        nullptr,
        fz ? reinterpret_cast<const GemmRowSeg*>(L->p2p_tab + P2P_SEGS_BYTES + P2P_PRE_BYTES + p2p_fptr_bytes(D)) +
                 (size_t)ch * moe_layer::P2P_MAXS
           : nullptr,
        fz ? X.fuse_nrseg[ch] : 0,
        fz ? reinterpret_cast<uint32_t**>(L->p2p_tab + P2P_SEGS_BYTES + P2P_PRE_BYTES) + cslot * D : nullptr,
        fz ? D : 0, X.epoch);
    if (err) { set_error(std::string("ComputeMoE: ") + cudaGetErrorString((cudaError_t)err)); return MOE_ERR_CUDA; }
    a = b;
  }
  // LocalReduce: the chunk's partial per unique row, in place of its x row
  if (X.lr) KERNEL_TRY(launch_lr_reduce(L->o, L->meta_recv, u0, u1, H, k, L->recvu, cs));
  if (X.p2p && X.fuse_comb[ch]) TR_TRY(L->tr->p2p_after_put(MOE_MAX_CHUNKS + ch, cs));  // combine rows are out
  CUDA_TRY(cudaEventRecord(L->ev_gemm[ch], cs));
  return MOE_OK;
}

// Debug: rows per (chunk, peer) in both directions.
void ep_debug_rows(Ep& X, moe_debug_t* dbg) {
  const int D = X.D, E_loc = X.E_loc, me = X.me, G = X.G;
  for (int ch = 0; ch < X.plan.num_chunks; ++ch) {
    const int sl = X.slice(ch);
    for (int peer = 0; peer < D; ++peer) {
      int64_t sent = 0, got = 0;
      if (X.lr) {
        sent = X.ug[(size_t)me * G + ch * D + peer];
        got = X.ug[(size_t)peer * G + ch * D + me];
      } else {
        for (int el = X.g0(ch); el < X.g1(ch); ++el) {
          sent += X.cnt(me, peer * E_loc + el, sl);
          got += X.cnt(peer, me * E_loc + el, sl);
        }
      }
      dbg->chunk_rows_host[(size_t)ch * D + peer] = sent;
      dbg->chunk_rows_host[((size_t)MOE_MAX_CHUNKS + ch) * D + peer] = got;
    }
  }
}

}  // namespace

// EP > 1: count exchange (C3), plan, layouts, and Algorithm 1's chunked
// dispatch / ComputeMoE / combine over the transport or the peer-memory planes.
moe_status_t fwd_ep(Fwd& F) {
  moe_layer* L = F.L;
  Ep X(F);
  const int64_t T = F.T;
  cudaStream_t st = F.st;
  Nvtx nv("epsmoe fwd_ep");
  if (moe_status_t r = ep_counts(X)) return r;
  if (int e = L->tr->set_comm_ctas(X.plan.comm_ctas)) return (moe_status_t)e;  // NCCL maxCTAs (NEXT-1)
  if (moe_status_t r = ep_lr_layout(X)) return r;
  X.p2p = X.c.a2a_p2p != 0;
  X.copy_engine = X.c.a2a_p2p == 2;
  if (X.p2p)
    if (moe_status_t r = ep_p2p_tables(X)) return r;
  // SM partition (NEXT-1): below the SM count, the expert
  // GEMMs run one grid at a time on the caller's stream after the shared
  // experts, so no more than sm_gemm GEMM CTAs are ever resident and the
  // reserved SMs stay free for the all2all.  With every SM theirs, odd
  // chunks compute on s_comp2 so that chunk c+1 fills the SMs chunk c's last
  // tile wave leaves idle (ordering from the dispatch events; the final
  // combine waits for every chunk through the combine stream).
  X.capped = F.num_ctas < L->num_sms;
  X.two_streams = !X.capped && L->chunk_streams > 1 && X.plan.num_chunks > 1;
  CUDA_TRY(cudaEventRecord(L->ev_ready, st));
  CUDA_TRY(cudaStreamWaitEvent(L->s_disp, L->ev_ready, 0));
  CUDA_TRY(cudaStreamWaitEvent(L->s_comb, L->ev_ready, 0));
  // Algorithm 1 issue order
  const int PN = X.plan.num_chunks;
  if (moe_status_t r = ep_dispatch(X, 0)) return r;
  if (X.capped && F.side) CUDA_TRY(cudaStreamWaitEvent(st, L->ev_shared, 0));  // shared GEMMs first
  for (int p = 1; p <= PN; ++p) {
    if (p <= PN - 1)
      if (moe_status_t r = ep_dispatch(X, p)) return r;
    if (moe_status_t r = ep_compute(X, p - 1)) return r;
    if (p - 2 >= 0)
      if (moe_status_t r = ep_combine(X, p - 2)) return r;
  }
  if (moe_status_t r = ep_combine(X, PN - 1)) return r;
  CUDA_TRY(cudaEventRecord(L->ev_comb_done, L->s_comb));
  CUDA_TRY(cudaStreamWaitEvent(st, L->ev_comb_done, 0));
  if (F.side && !X.capped) CUDA_TRY(cudaStreamWaitEvent(st, L->ev_shared, 0));
  if (X.p2p) {  // every chunk's combine rows from every expert rank
    TR_TRY(L->tr->p2p_before_wait(MOE_MAX_CHUNKS, PN, st));
    KERNEL_TRY(launch_p2p_wait(L->p2p_flags + (size_t)MOE_MAX_CHUNKS * X.D, PN * X.D, X.epoch, st));
  }
  // weighted unpermute / home-side LocalReduce
  int c0 = prof_rec(L, st);
  if (X.lr)
    KERNEL_TRY(launch_lr_combine(L->comb, L->SF ? L->s : nullptr, (int)T, X.H, X.k, L->posg, F.y, st));
  else
    KERNEL_TRY(launch_combine(L->comb, L->SF ? L->s : nullptr, (int)T, X.H, X.k, L->pos, F.topk_w, F.y, st));
  prof_mark(L, MOE_STAGE_COMBINE, c0, prof_rec(L, st));
  moe_debug_t* dbg = F.dbg;
  if (dbg && dbg->chunk_rows_host) ep_debug_rows(X, dbg);
  if (dbg && X.lr) {
    if (dbg->lr_pos) CUDA_TRY(cudaMemcpyAsync(dbg->lr_pos, L->posg, sizeof(int32_t) * T * X.k, cudaMemcpyDeviceToDevice, st));
    if (dbg->lr_hist)
      CUDA_TRY(cudaMemcpyAsync(dbg->lr_hist, L->u_hist, sizeof(int32_t) * X.G, cudaMemcpyDeviceToDevice, st));
  }
  return MOE_OK;
}

}  // namespace epsmoe
