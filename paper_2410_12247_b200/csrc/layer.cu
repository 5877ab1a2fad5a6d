// The MoE layer: create / forward / destroy, workspace carve-up, the stream &
// event DAG of Algorithm 1 and the NCCL all2all over NVLink.
//
// Streams (ep > 1): the caller's stream carries routing, permute, shared
// experts and the expert GEMMs (ComputeMoE); s_disp carries the dispatch
// All2All of every chunk on communicator A; s_comb the combine All2All on
// communicator B.  Per chunk c:  D_c (dispatch done) -> GEMMs -> G_c -> combine.
// Issue order = Algorithm 1: dispatch(0); for p: dispatch(p), compute(p-1),
// combine(p-2); combine(PN-1).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/epsmoe.h"
#include "gemm.h"
#include "internal.h"
#include "lr.h"
#include "p2p.h"
#include "route.h"
#include "transport.h"

struct moe_layer {
  moe_config_t cfg;
  moe_weights_t w;
  int E_loc = 0, SF = 0, num_sms = 148, device = 0;
  int64_t send_cap = 0, recv_cap = 0, gemm_rows_cap = 0;
  // workspace carve-up (device)
  void* wr_pad = nullptr;
  float* logits = nullptr;
  int32_t *topk_idx = nullptr, *pos = nullptr, *range_hist = nullptr, *range_off = nullptr;
  int32_t* row_token = nullptr;   // [T*k]: token of each send row (gathered GateUp A, ep == 1)
  int32_t* tickets = nullptr;     // [4]: GEMM tile-ticket counters (caller stream, side stream)
  float* topk_w = nullptr;
  int32_t *hist = nullptr, *seg_start = nullptr, *ghist = nullptr;
  int32_t *recv_start_d = nullptr, *recv_count_d = nullptr;
  void *send = nullptr, *recv = nullptr, *h = nullptr, *o = nullptr, *comb = nullptr;
  void *hs = nullptr, *s = nullptr;
  void *sendq = nullptr, *recvq = nullptr;  // ep > 1 && dispatch_fp8: packed FP8 rows (pitch qpitch)
  int qpitch = 0;
  // local_reduce (NEXT-3, R16): dedup send rows / meta, unique receive rows
  int32_t *posg = nullptr, *u_hist = nullptr, *u_start = nullptr, *ughist = nullptr;
  int32_t *meta_send = nullptr, *meta_recv = nullptr, *lr_recv_off_d = nullptr, *lr_usrc_d = nullptr;
  void* recvu = nullptr;  // bf16 [recv_cap, H]: received unique rows, then their LocalReduce partials
  // a2a_p2p: own put kernels over peer-mapped workspaces.  flags [2][64][ep]:
  // per (direction, chunk, source) completion epochs written by the sources;
  // done [2][64]: put-kernel CTA counters; segment tables per launch.
  static constexpr int P2P_MAXS = 2 * MOE_MAX_EXPERTS;  // segments per put launch
  char* ws_base = nullptr;
  std::vector<char*> peer_ws;  // [ep] every rank's workspace base, mapped here
  // [ep][P2P_NBUF] byte offsets of the buffers peers write into, per rank (a
  // rank's max_tokens, hence its workspace layout, may differ from its peers')
  enum { P2P_RECV, P2P_RECVQ, P2P_RECVU, P2P_META, P2P_COMB, P2P_FLAGS, P2P_NBUF };
  std::vector<int64_t> peer_off;
  uint32_t p2p_epoch = 0;
  uint32_t *p2p_flags = nullptr, *p2p_done = nullptr;
  // device tables [segs [2][64][P2P_MAXS] | pre [2][64][P2P_MAXS+1] | consumer flag
  // addresses [2][64][ep] | fused-combine row segments [64][P2P_MAXS]], pinned mirror
  char* p2p_tab = nullptr;
  char* p2p_host = nullptr;
  bool p2p_fuse = true;  // EPSMOE_P2P_FUSE=0: combine by put kernel instead of the DownGemm's scatter
  int32_t* ughist_host = nullptr;  // pinned [ep*256]
  void *x_dev[2] = {}, *y_dev[2] = {};  // forward_host staging, double-buffered across calls
  int hb = 0;                            // staging buffer of the next host call
  cudaEvent_t ev_xfree[2] = {}, ev_yfree[2] = {};  // staging buffer b consumed / drained
  // host
  int32_t* ghist_host = nullptr;    // pinned [ep*E]
  // pinned: per-chunk GEMM row tables [2][TBL] (start, count; chunk c at c*E_loc), then the
  // local_reduce receive tables [2][256+4]
  static constexpr int TBL = MOE_MAX_CHUNKS * MOE_MAX_EXPERTS;
  int32_t* tables_host = nullptr;
  // token-sliced chunks (R8 extension): per-(expert, slice) counts, local and all ranks
  int32_t *slice_hist = nullptr, *gslice = nullptr;
  int32_t* gslice_host = nullptr;  // pinned [ep * E * 64]
  cudaStream_t s_disp = nullptr, s_comb = nullptr;
  cudaStream_t s_side = nullptr;  // shared experts, concurrent with routing / dispatch
  // odd chunks' ComputeMoE runs here: chunk c+1's persistent GEMMs fill the SMs
  // chunk c's last tile wave leaves idle (EPSMOE_CHUNK_STREAMS=1: all on the caller's stream)
  cudaStream_t s_comp2 = nullptr;
  cudaEvent_t ev_routed = nullptr, ev_comp2 = nullptr;
  int chunk_streams = 2;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;  // forward_host copy streams
  static constexpr int MAX_HOST_SLICES = 8;
  cudaEvent_t ev_in[MAX_HOST_SLICES] = {}, ev_out[MAX_HOST_SLICES] = {};
  cudaEvent_t ev_router = nullptr, ev_shared = nullptr;
  // ep == 1 with shared experts, how the shared DownGemm meets the combine
  // (EPSMOE_FUSE_COMBINE): 0 in order (default); 1 one kernel (EPI_COMBINE
  // epilogue); 2 token pieces, piece p's combine on s_side concurrent with piece
  // p+1's DownGemm.  All three are bit-identical.  Measured on dsv2 (B200,
  // power-capped): 1 is 0.6 ms slower (the epilogue's random 64-B o-row reads
  // outlast the MMA of the next tile), 2 is a wash (the co-running HBM stream
  // lowers the GEMM's clock by as much as it hides).
  int fuse_combine = 0;
  static constexpr int COMB_PIECES = 4;
  cudaEvent_t ev_piece[COMB_PIECES] = {};
  bool ce_batch = true;           // copy-engine plane: cudaMemcpyBatchAsync per chunk (cleared if unsupported)
  bool overlap_shared = true;     // shared experts on s_side, concurrent with routing (EPSMOE_OVERLAP_SHARED=0: in order)
  bool split_rem = false;         // EPSMOE_SPLIT_REM=1: expert GEMMs as bulk on CTA pairs + remainder rows on
                                  // single CTAs; measured 1-3% slower than padding (DSv2, Mixtral), so off
  int comm_ctas = 0;              // ep > 1: NCCL maxCTAs per communicator (EPSMOE_COMM_CTAS, default 8);
                                  // the persistent GEMM grid leaves 2*comm_ctas SMs free for them
  bool gather_a = false;          // EPSMOE_GATHER=1: GateUp gathers x rows itself at ep == 1 (16-B cp.async
                                  // into the swizzled stage) instead of reading a materialised send buffer;
                                  // measured 1.9x slower GateUp on B200 (request-bound), so off by default
  cudaEvent_t ev_hist = nullptr, ev_ready = nullptr, ev_comb_done = nullptr;
  std::vector<cudaEvent_t> ev_disp, ev_gemm;
  epsmoe::Transport* tr = nullptr;  // all2all transport (NCCL, or in-process for tests), ep > 1
  moe_cost_model_t cost;
  int last_launches = 0;
  // ep > 1 measurement hook (moe_layer_set_comm_only): forwards skip ComputeMoE
  // and the shared experts, so the same chunked all2all runs alone
  bool comm_only = false;
  // per-stage device timing (moe_layer_set_profiling)
  bool prof = false;
  std::vector<cudaEvent_t> pev;
  int pev_used = 0;
  struct Mark { int stage, e0, e1; };
  std::vector<Mark> marks;
};

namespace epsmoe {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

}  // namespace epsmoe

using namespace epsmoe;

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                      \
      return MOE_ERR_CUDA;                                                                \
    }                                                                                     \
  } while (0)
#define KERNEL_TRY(expr)                                                                  \
  do {                                                                                    \
    int _e = (expr);                                                                      \
    if (_e != 0) {                                                                        \
      set_error(std::string(#expr) + ": " + cudaGetErrorString((cudaError_t)_e));         \
      return MOE_ERR_CUDA;                                                                \
    }                                                                                     \
    ++L->last_launches;                                                                   \
  } while (0)
#define TR_TRY(expr)                                                                      \
  do {                                                                                    \
    int _r = (expr);                                                                      \
    if (_r != 0) return (moe_status_t)_r;                                                 \
  } while (0)
#define NCCL_TRY(expr)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess) {                                                              \
      set_error(std::string(#expr) + ": " + ncclGetErrorString(_r));                      \
      return MOE_ERR_NCCL;                                                                \
    }                                                                                     \
  } while (0)

namespace {

constexpr size_t ALIGN = 256;
inline size_t align_up(size_t v) { return (v + ALIGN - 1) & ~(ALIGN - 1); }

struct Carve {
  size_t off = 0;
  char* base = nullptr;
  template <typename T>
  T* take(size_t count) {
    size_t o = off;
    off = align_up(off + count * sizeof(T));
    return base ? reinterpret_cast<T*>(base + o) : nullptr;
  }
};

// a2a_p2p segment tables (host mirror == device layout): segs | pre | flag pointers
constexpr size_t P2P_SEGS_BYTES = sizeof(epsmoe::P2PSeg) * 2 * MOE_MAX_CHUNKS * moe_layer::P2P_MAXS;
constexpr size_t P2P_PRE_BYTES = sizeof(int64_t) * 2 * MOE_MAX_CHUNKS * (moe_layer::P2P_MAXS + 1);
constexpr size_t P2P_RSEG_BYTES = sizeof(epsmoe::GemmRowSeg) * MOE_MAX_CHUNKS * moe_layer::P2P_MAXS;
size_t p2p_fptr_bytes(int ep) { return sizeof(uint32_t*) * 2 * MOE_MAX_CHUNKS * ep; }
size_t p2p_table_bytes(int ep) { return P2P_SEGS_BYTES + P2P_PRE_BYTES + p2p_fptr_bytes(ep) + P2P_RSEG_BYTES; }

int validate(const moe_config_t* c) {
  if (!c) return MOE_ERR_INVALID;
  std::string why;
  if (c->num_experts < 1 || c->num_experts > MOE_MAX_EXPERTS) why = "num_experts out of [1, 256]";
  else if (c->ep < 1 || c->num_experts % c->ep) why = "num_experts % ep != 0 (R12)";
  else if (c->rank < 0 || c->rank >= c->ep) why = "rank out of range";
  else if (c->top_k < 1 || c->top_k > MOE_MAX_TOPK || c->top_k > c->num_experts) why = "top_k out of range";
  else if (c->hidden < 64 || c->hidden % 64 || c->hidden > MOE_MAX_HIDDEN) why = "hidden must be a multiple of 64 in [64, 8192]";
  else if (c->ffn < 128 || c->ffn % 128) why = "ffn must be a positive multiple of 128";
  else if (c->num_shared < 0 || (c->num_shared > 0 && ((int64_t)c->num_shared * c->shared_ffn) % 128))
    why = "num_shared * shared_ffn must be a multiple of 128";
  else if (c->dispatch_fp8 && c->hidden % 128) why = "dispatch_fp8 needs hidden % 128 == 0";
  else if (c->max_tokens < 1) why = "max_tokens must be >= 1";
  else if (c->local_reduce != 0 && c->local_reduce != 1) why = "local_reduce must be 0 or 1";
  else if (c->a2a_p2p < 0 || c->a2a_p2p > 2) why = "a2a_p2p must be 0, 1 or 2";
  else if (c->route_groups > 1 &&
           (c->route_groups > 32 || c->num_experts % c->route_groups || c->route_topk_groups < 1 ||
            c->route_topk_groups > c->route_groups ||
            c->top_k > c->route_topk_groups * (c->num_experts / c->route_groups)))
    why = "route_groups must divide e (<= 32) with 1 <= route_topk_groups <= route_groups and topk <= M*e/groups";
  if (!why.empty()) { set_error("invalid config: " + why); return MOE_ERR_INVALID; }
  return MOE_OK;
}

// Carve the workspace (base == nullptr: only measure).
size_t carve(moe_layer* L, char* base) {
  const moe_config_t& c = L->cfg;
  const int64_t T = c.max_tokens, E = c.num_experts, k = c.top_k, H = c.hidden, F = c.ffn;
  const int64_t D = c.ep, E_loc = E / D, SF = (int64_t)c.num_shared * c.shared_ffn;
  const int64_t R = max_ranges(T);
  L->send_cap = T * k;
  L->recv_cap = (D == 1) ? 0 : D * T * std::min<int64_t>(k, E_loc);
  L->gemm_rows_cap = (D == 1) ? L->send_cap : L->recv_cap;
  Carve cv;
  cv.base = base;
  L->wr_pad = cv.take<uint16_t>(256 * H);
  L->logits = cv.take<float>(T * E);
  L->topk_idx = cv.take<int32_t>(T * k);
  L->topk_w = cv.take<float>(T * k);
  L->pos = cv.take<int32_t>(T * k);
  L->row_token = cv.take<int32_t>(T * k);
  L->tickets = cv.take<int32_t>(6);  // tile-ticket pairs: caller stream, s_side, s_comp2
  L->range_hist = cv.take<int32_t>(E * R);
  L->range_off = cv.take<int32_t>(E * R);
  L->hist = cv.take<int32_t>(MOE_MAX_EXPERTS + 1);
  L->seg_start = cv.take<int32_t>(MOE_MAX_EXPERTS + 1);
  L->ghist = cv.take<int32_t>(D * E);
  L->recv_start_d = cv.take<int32_t>(moe_layer::TBL);
  L->recv_count_d = cv.take<int32_t>(moe_layer::TBL);
  if (D > 1) {
    L->slice_hist = cv.take<int32_t>(E * MOE_MAX_CHUNKS);
    L->gslice = cv.take<int32_t>(D * E * MOE_MAX_CHUNKS);
  }
  L->send = cv.take<uint16_t>(L->send_cap * H);
  L->recv = (D == 1) ? nullptr : cv.take<uint16_t>(L->recv_cap * H);
  L->h = cv.take<uint16_t>(L->gemm_rows_cap * F);
  L->o = cv.take<uint16_t>(L->gemm_rows_cap * H);
  L->comb = (D == 1) ? nullptr : cv.take<uint16_t>(L->send_cap * H);
  L->qpitch = fp8_row_pitch((int)H);
  if (D > 1 && c.dispatch_fp8) {
    L->sendq = cv.take<uint8_t>(L->send_cap * L->qpitch);
    L->recvq = cv.take<uint8_t>(L->recv_cap * L->qpitch);
  }
  if (c.local_reduce) {
    L->posg = cv.take<int32_t>(T * k);
    L->u_hist = cv.take<int32_t>(MOE_MAX_EXPERTS + 1);
    L->u_start = cv.take<int32_t>(MOE_MAX_EXPERTS + 1);
    if (D > 1) {
      L->ughist = cv.take<int32_t>(D * MOE_MAX_EXPERTS);
      L->meta_send = cv.take<int32_t>(L->send_cap * lr_meta_pitch((int)k));
      L->meta_recv = cv.take<int32_t>(L->recv_cap * lr_meta_pitch((int)k));
      L->recvu = cv.take<uint16_t>(L->recv_cap * H);
      L->lr_recv_off_d = cv.take<int32_t>(MOE_MAX_EXPERTS + 1);
      L->lr_usrc_d = cv.take<int32_t>(MOE_MAX_EXPERTS + 1);
    }
  }
  if (D > 1 && c.a2a_p2p) {
    L->p2p_flags = cv.take<uint32_t>(2 * MOE_MAX_CHUNKS * D);
    L->p2p_done = cv.take<uint32_t>(2 * MOE_MAX_CHUNKS);
    L->p2p_tab = cv.take<char>(p2p_table_bytes((int)D));
  }
  L->hs = SF ? cv.take<uint16_t>(T * SF) : nullptr;
  L->s = SF ? cv.take<uint16_t>(T * H) : nullptr;
  for (int b = 0; b < 2; ++b) {
    L->x_dev[b] = cv.take<uint16_t>(T * H);
    L->y_dev[b] = cv.take<uint16_t>(T * H);
  }
  return cv.off + ALIGN;
}

// Record a profiling event on `st` (no-op unless profiling is on).
int prof_rec(moe_layer* L, cudaStream_t st) {
  if (!L->prof || L->pev_used >= (int)L->pev.size()) return -1;
  cudaEventRecord(L->pev[L->pev_used], st);
  return L->pev_used++;
}
void prof_mark(moe_layer* L, int stage, int e0, int e1) {
  if (e0 >= 0 && e1 >= 0) L->marks.push_back({stage, e0, e1});
}

GemmArgs base_args(int epi, int num_ctas) {
  GemmArgs a;
  std::memset(&a, 0, sizeof(a));
  a.epi = epi;
  a.G = 1;
  a.num_ctas = num_ctas;
  a.cta_pair = 1;  // dense single-group GEMMs (router, shared experts): large M
  return a;
}

// All2all layout of one forward on rank c.rank from the global histogram gh
// [ep, E] (R6): send_off[e] = first send row of expert e (expert-major, local
// tokens); recv_off[e_l * ep + src] = first recv row of (local expert, source).
void exchange_layout(const moe_config_t& c, const int32_t* gh, int64_t* send_off, int64_t* recv_off) {
  const int E = c.num_experts, D = c.ep, E_loc = E / D, me = c.rank;
  send_off[0] = 0;
  for (int ex = 0; ex < E; ++ex) send_off[ex + 1] = send_off[ex] + gh[(int64_t)me * E + ex];
  recv_off[0] = 0;
  for (int el = 0; el < E_loc; ++el)
    for (int src = 0; src < D; ++src) {
      size_t i = (size_t)el * D + src;
      recv_off[i + 1] = recv_off[i] + gh[(int64_t)src * E + me * E_loc + el];
    }
}

// Tile rows for a chunk's expert GEMMs: 256 (CTA pair) unless the plan says
// otherwise or the chunk's mean rows per expert is small (decode-like load).
int pick_cta_pair(const moe_plan_t& plan, double mean_rows) {
  if (plan.tile_m == 256) return 1;
  if (plan.tile_m == 128) return 0;
  return mean_rows >= 512.0 ? 1 : 0;
}

// ComputeMoE for local experts [g0, g1): GateUpGemm+SiluAct fused,
// then DownGemm.  Rows of expert g are [row_start[g], +row_count[g]) of A.
int compute_moe(moe_layer* L, const void* A, int64_t a_rows, const int32_t* row_start, const int32_t* row_count,
                int g0, int g1, int kind, int num_ctas, int cta_pair, bool tile_forced, double rows_per_group,
                cudaStream_t st, const int32_t* a_row_index = nullptr, const GemmRowSeg* down_rseg = nullptr, int down_nrseg = 0,
                uint32_t* const* down_sig = nullptr, int down_nsig = 0, uint32_t down_epoch = 0) {
  const moe_config_t& c = L->cfg;
  GemmArgs g1a = base_args(EPI_SWIGLU, num_ctas);
  g1a.rows_hint = rows_per_group;
  g1a.cta_pair = cta_pair;
  g1a.A = A;
  g1a.a_row_index = a_row_index;
  g1a.tile_counter = (st == L->s_comp2) ? L->tickets + 4 : L->tickets;
  g1a.a_rows = a_rows;
  g1a.B0 = L->w.w_gate;
  g1a.B1 = L->w.w_up;
  g1a.b_rows = (int64_t)L->E_loc * c.ffn;
  g1a.b_group_rows = c.ffn;
  g1a.K = c.hidden;
  g1a.N = c.ffn;
  g1a.out = L->h;
  g1a.ldo = c.ffn;
  g1a.out_rows = L->gemm_rows_cap;
  GemmArgs g2a = base_args(EPI_BF16, num_ctas);
  g2a.rows_hint = rows_per_group;
  g2a.rseg = down_rseg;  // DownGemm fused with the combine all2all (a2a_p2p)
  g2a.nrseg = down_nrseg;
  g2a.sig_flags = down_sig;
  g2a.nsig = down_nsig;
  g2a.sig_epoch = down_epoch;
  g2a.cta_pair = cta_pair;
  g2a.tile_counter = g1a.tile_counter;
  g2a.A = L->h;
  g2a.a_rows = L->gemm_rows_cap;
  g2a.B0 = L->w.w_down;
  g2a.b_rows = (int64_t)L->E_loc * c.hidden;
  g2a.b_group_rows = c.hidden;
  g2a.K = c.ffn;
  g2a.N = c.hidden;
  g2a.out = L->o;
  g2a.ldo = c.hidden;
  g2a.out_rows = L->gemm_rows_cap;
  // CTA-pair tiles cover each expert's first floor(M/256)*256 rows; with
  // split_rem the remaining < 256 rows go to a second launch on 128-row
  // single-CTA tiles (halves the M padding: ~64 instead of ~128 rows/expert).
  const bool split = cta_pair && L->split_rem;
  auto run = [&](int a, int b) -> int {
    int stage = MOE_STAGE_GATEUP;
    for (GemmArgs* ga : {&g1a, &g2a}) {
      ga->G = b - a;
      ga->b_base = a;
      ga->row_start = row_start + a;
      ga->row_count = row_count + a;
      int p0 = prof_rec(L, st);
      // DownGemm of a light launch: 128-row tiles would leave SMs idle (fewer
      // (expert, n-tile) tiles than CTAs, e.g. Mixtral decode: 8 x 16 = 128 on
      // 148 SMs), so it takes CTA pairs, which halve the weight rows each CTA
      // streams (measured Mixtral decode Down 0.221 -> 0.184 ms).  Bit-neutral.
      int pair = cta_pair;
      if (ga == &g2a && !pair && !tile_forced && (b - a) * ((c.hidden + 255) / 256) < num_ctas) pair = 1;
      for (int part = 0; part < (split ? 2 : 1); ++part) {
        ga->row_mode = split ? 1 + part : 0;
        ga->cta_pair = (split && part == 1) ? 0 : pair;
        int e = gemm_launch(*ga, st);
        if (e) return e;
        ++L->last_launches;
      }
      prof_mark(L, stage, p0, prof_rec(L, st));
      stage = MOE_STAGE_DOWN;
    }
    return 0;
  };
  if (kind == MOE_GEMM_GROUPED) return run(g0, g1);
  for (int e = g0; e < g1; ++e) {
    int e2 = run(e, e + 1);
    if (e2) return e2;
  }
  return 0;
}

}  // namespace

extern "C" {

const char* moe_last_error(void) { return g_err.c_str(); }

size_t moe_layer_workspace_bytes(const moe_config_t* cfg) {
  if (validate(cfg) != MOE_OK) return 0;
  moe_layer tmp;
  tmp.cfg = *cfg;
  return carve(&tmp, nullptr);
}

moe_status_t moe_get_unique_id(void* out128) {
  if (!out128) return MOE_ERR_INVALID;
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return MOE_OK;
}

moe_status_t moe_plan_compute(const moe_config_t* cfg, const moe_cost_model_t* cost, int64_t global_tokens,
                              const int32_t* global_hist, moe_plan_t* out) {
  if (!out) return MOE_ERR_INVALID;
  int v = validate(cfg);
  if (v) return (moe_status_t)v;
  moe_cost_model_t def;
  if (!cost) {
    default_cost_model(*cfg, &def);
    cost = &def;
  }
  return (moe_status_t)plan_compute(*cfg, *cost, global_tokens, global_hist, out);
}

moe_status_t moe_local_group_create(int32_t ep, void** out) {
  if (!out || ep < 1) { set_error("bad argument"); return MOE_ERR_INVALID; }
  *out = new epsmoe::LocalGroup(ep);
  return MOE_OK;
}

moe_status_t moe_local_group_destroy(void* group) {
  delete static_cast<epsmoe::LocalGroup*>(group);
  return MOE_OK;
}

static moe_status_t create_impl(const moe_config_t* cfg, const moe_weights_t* w, const void* uid_d,
                                const void* uid_c, epsmoe::LocalGroup* group, void* workspace,
                                size_t workspace_bytes, moe_layer_t** out) {
  if (!out || !w) { set_error("null argument"); return MOE_ERR_INVALID; }
  *out = nullptr;
  int v = validate(cfg);
  if (v) return (moe_status_t)v;
  if (!w->w_router || !w->w_gate || !w->w_up || !w->w_down) { set_error("missing weights"); return MOE_ERR_INVALID; }
  if (cfg->num_shared > 0 && (!w->ws_gate || !w->ws_up || !w->ws_down)) {
    set_error("missing shared-expert weights");
    return MOE_ERR_INVALID;
  }
  if (cfg->ep > 1 && !group && (!uid_d || !uid_c)) {
    set_error("ep > 1 needs two NCCL unique ids");
    return MOE_ERR_INVALID;
  }
  if (group && group->ep != cfg->ep) { set_error("local group size != ep"); return MOE_ERR_INVALID; }
  moe_layer* L = new moe_layer();
  L->cfg = *cfg;
  L->w = *w;
  L->E_loc = cfg->num_experts / cfg->ep;
  L->SF = cfg->num_shared * cfg->shared_ffn;
  size_t need = carve(L, nullptr);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace too small: need " + std::to_string(need) + " bytes");
    delete L;
    return MOE_ERR_CAPACITY;
  }
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + ALIGN - 1) & ~(uintptr_t)(ALIGN - 1));
  carve(L, base);
  L->ws_base = base;
  if (cudaMemset(L->tickets, 0, 6 * sizeof(int32_t)) != cudaSuccess ||
      (L->p2p_flags && (cudaMemset(L->p2p_flags, 0, sizeof(uint32_t) * 2 * MOE_MAX_CHUNKS * cfg->ep) != cudaSuccess ||
                        cudaMemset(L->p2p_done, 0, sizeof(uint32_t) * 2 * MOE_MAX_CHUNKS) != cudaSuccess))) {
    set_error("workspace memset failed");
    delete L;
    return MOE_ERR_CUDA;
  }
  auto fail = [&](moe_status_t st) { moe_layer_destroy(L); return st; };
  if (cudaGetDevice(&L->device) != cudaSuccess) return fail(MOE_ERR_CUDA);
  cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, L->device);
  int cc_major = 0, cc_minor = 0;
  cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, L->device);
  cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, L->device);
  if (cc_major != 10 || cc_minor != 0) {
    set_error("this build targets sm_100a (B200); device is sm_" + std::to_string(cc_major * 10 + cc_minor));
    return fail(MOE_ERR_UNSUPPORTED);
  }
  if (launch_pad_rows(w->w_router, cfg->num_experts, cfg->hidden, L->wr_pad, 256, 0)) {
    set_error("router pad failed");
    return fail(MOE_ERR_CUDA);
  }
  if (cudaHostAlloc(&L->ghist_host, sizeof(int32_t) * cfg->ep * cfg->num_experts, cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(&L->tables_host, sizeof(int32_t) * (2 * moe_layer::TBL + 2 * (MOE_MAX_EXPERTS + 4)),
                    cudaHostAllocDefault) != cudaSuccess ||
      (cfg->ep > 1 && cudaHostAlloc(&L->gslice_host, sizeof(int32_t) * cfg->ep * cfg->num_experts * MOE_MAX_CHUNKS,
                                    cudaHostAllocDefault) != cudaSuccess) ||
      (L->p2p_tab && cudaHostAlloc(&L->p2p_host, p2p_table_bytes(cfg->ep), cudaHostAllocDefault) != cudaSuccess) ||
      cudaHostAlloc(&L->ughist_host, sizeof(int32_t) * cfg->ep * MOE_MAX_EXPERTS, cudaHostAllocDefault) != cudaSuccess) {
    set_error("cudaHostAlloc failed");
    return fail(MOE_ERR_CUDA);
  }
  default_cost_model(L->cfg, &L->cost);
  if (const char* ov = std::getenv("EPSMOE_OVERLAP_SHARED")) L->overlap_shared = std::atoi(ov) != 0;
  if (const char* fc = std::getenv("EPSMOE_FUSE_COMBINE")) L->fuse_combine = std::atoi(fc);
  if (const char* gv = std::getenv("EPSMOE_GATHER")) L->gather_a = std::atoi(gv) != 0;
  if (const char* pf = std::getenv("EPSMOE_P2P_FUSE")) L->p2p_fuse = std::atoi(pf) != 0;
  if (const char* sv = std::getenv("EPSMOE_SPLIT_REM")) L->split_rem = std::atoi(sv) != 0;
  if (cfg->ep > 1) {
    const char* cv = std::getenv("EPSMOE_COMM_CTAS");
    L->comm_ctas = std::max(1, std::min(32, cv ? std::atoi(cv) : 8));
  }
  if (cudaStreamCreateWithFlags(&L->s_h2d, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&L->s_d2h, cudaStreamNonBlocking) != cudaSuccess) {
    set_error("copy stream creation failed");
    return fail(MOE_ERR_CUDA);
  }
  for (int b = 0; b < 2; ++b)
    if (cudaEventCreateWithFlags(&L->ev_xfree[b], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&L->ev_yfree[b], cudaEventDisableTiming) != cudaSuccess) {
      set_error("event creation failed");
      return fail(MOE_ERR_CUDA);
    }
  for (int i = 0; i < moe_layer::MAX_HOST_SLICES; ++i)
    if (cudaEventCreateWithFlags(&L->ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&L->ev_out[i], cudaEventDisableTiming) != cudaSuccess) {
      set_error("event creation failed");
      return fail(MOE_ERR_CUDA);
    }
  if (const char* cs = std::getenv("EPSMOE_CHUNK_STREAMS")) L->chunk_streams = std::max(1, std::min(2, std::atoi(cs)));
  if (cudaStreamCreateWithFlags(&L->s_comp2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_routed, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_comp2, cudaEventDisableTiming) != cudaSuccess) {
    set_error("stream creation failed");
    return fail(MOE_ERR_CUDA);
  }
  if (cudaStreamCreateWithFlags(&L->s_side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_router, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->ev_shared, cudaEventDisableTiming) != cudaSuccess) {
    set_error("side stream creation failed");
    return fail(MOE_ERR_CUDA);
  }
  for (auto& e : L->ev_piece)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      set_error("event creation failed");
      return fail(MOE_ERR_CUDA);
    }
  if (cfg->ep > 1) {
    if (cudaStreamCreateWithFlags(&L->s_disp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&L->s_comb, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&L->ev_hist, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&L->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&L->ev_comb_done, cudaEventDisableTiming) != cudaSuccess) {
      set_error("stream/event creation failed");
      return fail(MOE_ERR_CUDA);
    }
    L->ev_disp.resize(MOE_MAX_CHUNKS);
    L->ev_gemm.resize(MOE_MAX_CHUNKS);
    for (int i = 0; i < MOE_MAX_CHUNKS; ++i) {
      cudaEventCreateWithFlags(&L->ev_disp[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&L->ev_gemm[i], cudaEventDisableTiming);
    }
    if (group) {
      L->tr = new epsmoe::LocalTransport(group, cfg->rank);
    } else {
      ncclUniqueId id_d, id_c;
      std::memcpy(&id_d, uid_d, sizeof(id_d));
      std::memcpy(&id_c, uid_c, sizeof(id_c));
      ncclConfig_t ncfg = NCCL_CONFIG_INITIALIZER;
      ncfg.blocking = 1;
      ncfg.maxCTAs = L->comm_ctas;  // the paper's comm-SM control
      ncfg.minCTAs = std::min(L->comm_ctas, 2);
      ncclComm_t cd = nullptr, cc = nullptr;
      ncclResult_t r1 = ncclCommInitRankConfig(&cd, cfg->ep, id_d, cfg->rank, &ncfg);
      ncclResult_t r2 = r1 == ncclSuccess ? ncclCommInitRankConfig(&cc, cfg->ep, id_c, cfg->rank, &ncfg) : r1;
      L->tr = new epsmoe::NcclTransport(cd, cc);
      if (r1 != ncclSuccess || r2 != ncclSuccess) {
        set_error(std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r1 != ncclSuccess ? r1 : r2));
        return fail(MOE_ERR_NCCL);
      }
      // every rank must agree on the shape (MOE_ERR_MISMATCH)
      int32_t sig[9] = {cfg->num_experts, cfg->top_k, cfg->hidden, cfg->ffn, cfg->num_shared, cfg->shared_ffn,
                        cfg->norm_topk | (cfg->dispatch_fp8 << 1) | (cfg->local_reduce << 2) |
                            (cfg->route_groups << 3) | (cfg->route_topk_groups << 9) | (cfg->a2a_p2p << 15),
                        (int32_t)(cfg->routed_scale * 1e6f), (int32_t)cfg->max_tokens};
      int32_t* d_sig = nullptr;
      if (cudaMalloc(&d_sig, sizeof(sig) * (cfg->ep + 1)) != cudaSuccess) return fail(MOE_ERR_CUDA);
      cudaMemcpy(d_sig, sig, sizeof(sig), cudaMemcpyHostToDevice);
      int r3 = L->tr->allgather_i32(d_sig, d_sig + 9, 9, 0);
      std::vector<int32_t> all(9 * cfg->ep);
      cudaMemcpy(all.data(), d_sig + 9, sizeof(int32_t) * 9 * cfg->ep, cudaMemcpyDeviceToHost);
      cudaFree(d_sig);
      if (r3) return fail((moe_status_t)r3);
      for (int r = 0; r < cfg->ep; ++r)
        if (std::memcmp(all.data() + 9 * r, sig, sizeof(sig)) != 0) {
          set_error("config mismatch across ranks");
          return fail(MOE_ERR_MISMATCH);
        }
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error(std::string("create: ") + cudaGetErrorString(cudaGetLastError()));
    return fail(MOE_ERR_CUDA);
  }
  *out = L;
  return MOE_OK;
}

moe_status_t moe_layer_create(const moe_config_t* cfg, const moe_weights_t* w, const void* uid_d,
                              const void* uid_c, void* workspace, size_t workspace_bytes, moe_layer_t** out) {
  return create_impl(cfg, w, uid_d, uid_c, nullptr, workspace, workspace_bytes, out);
}

moe_status_t moe_layer_create_local(const moe_config_t* cfg, const moe_weights_t* w, void* group, void* workspace,
                                    size_t workspace_bytes, moe_layer_t** out) {
  if (!group) { set_error("null group"); return MOE_ERR_INVALID; }
  return create_impl(cfg, w, nullptr, nullptr, static_cast<epsmoe::LocalGroup*>(group), workspace,
                     workspace_bytes, out);
}

moe_status_t moe_layer_destroy(moe_layer_t* L) {
  if (!L) return MOE_OK;
  delete L->tr;
  if (L->s_disp) cudaStreamDestroy(L->s_disp);
  if (L->s_side) cudaStreamDestroy(L->s_side);
  if (L->s_comp2) cudaStreamDestroy(L->s_comp2);
  for (cudaEvent_t e : {L->ev_routed, L->ev_comp2})
    if (e) cudaEventDestroy(e);
  if (L->s_h2d) cudaStreamDestroy(L->s_h2d);
  if (L->s_d2h) cudaStreamDestroy(L->s_d2h);
  for (int i = 0; i < moe_layer::MAX_HOST_SLICES; ++i) {
    if (L->ev_in[i]) cudaEventDestroy(L->ev_in[i]);
    if (L->ev_out[i]) cudaEventDestroy(L->ev_out[i]);
  }
  for (cudaEvent_t e : {L->ev_router, L->ev_shared, L->ev_xfree[0], L->ev_xfree[1], L->ev_yfree[0], L->ev_yfree[1]})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : L->ev_piece)
    if (e) cudaEventDestroy(e);
  if (L->s_comb) cudaStreamDestroy(L->s_comb);
  for (cudaEvent_t e : {L->ev_hist, L->ev_ready, L->ev_comb_done})
    if (e) cudaEventDestroy(e);
  for (auto e : L->ev_disp) if (e) cudaEventDestroy(e);
  for (auto e : L->ev_gemm) if (e) cudaEventDestroy(e);
  for (auto e : L->pev) if (e) cudaEventDestroy(e);
  if (L->ghist_host) cudaFreeHost(L->ghist_host);
  if (L->tables_host) cudaFreeHost(L->tables_host);
  if (L->ughist_host) cudaFreeHost(L->ughist_host);
  if (L->gslice_host) cudaFreeHost(L->gslice_host);
  if (L->p2p_host) cudaFreeHost(L->p2p_host);
  delete L;
  return MOE_OK;
}

moe_status_t moe_exchange_layout(const moe_config_t* cfg, const moe_plan_t* plan_in, const int32_t* ghist,
                                 int64_t* send_off, int64_t* recv_off, int64_t* chunk_send, int64_t* chunk_recv) {
  int v = validate(cfg);
  if (v) return (moe_status_t)v;
  if (!plan_in || !ghist || !send_off || !recv_off) { set_error("null argument"); return MOE_ERR_INVALID; }
  moe_plan_t plan = *plan_in;
  int pv = plan_normalise(*cfg, &plan);
  if (pv) { set_error("invalid plan"); return (moe_status_t)pv; }
  if (plan.token_slices > 1) {  // per-slice counts are not derivable from ghist
    set_error("moe_exchange_layout: token_slices > 1 needs the per-slice histogram (see moe_layer_forward)");
    return MOE_ERR_UNSUPPORTED;
  }
  exchange_layout(*cfg, ghist, send_off, recv_off);
  const int E = cfg->num_experts, D = cfg->ep, E_loc = E / D, me = cfg->rank;
  for (int ch = 0; ch < plan.num_chunks; ++ch)
    for (int peer = 0; peer < D; ++peer) {
      int64_t s = 0, r = 0;
      for (int el = plan.group_begin[ch]; el < plan.group_begin[ch + 1]; ++el) {
        s += ghist[(int64_t)me * E + peer * E_loc + el];   // my pairs for peer's expert el
        r += ghist[(int64_t)peer * E + me * E_loc + el];   // peer's pairs for my expert el
      }
      if (chunk_send) chunk_send[(size_t)ch * D + peer] = s;
      if (chunk_recv) chunk_recv[(size_t)ch * D + peer] = r;
    }
  return MOE_OK;
}

// Persistent GEMM grid of a forward (the SM partition, NEXT-1): all SMs
// at ep == 1 and on the copy-engine plane; else 2 * comm_ctas SMs are left to
// the all2all's kernels (NCCL's two communicators, or the put kernels).
static int gemm_sm_budget(const moe_layer* L) {
  if (L->cfg.ep == 1 || L->cfg.a2a_p2p == 2) return L->num_sms;
  return L->num_sms - 2 * L->comm_ctas;
}

moe_status_t moe_plan_pipeline(const moe_layer_t* L, int64_t global_tokens, const int32_t* global_hist,
                               moe_plan_t* out) {
  if (!L || !out) return MOE_ERR_INVALID;
  int r = plan_compute(L->cfg, L->cost, global_tokens, global_hist, out);
  if (r == MOE_OK && L->cfg.ep > 1) {  // SM partition of this layer (NEXT-1)
    out->comm_ctas = L->comm_ctas;
    out->sm_gemm = gemm_sm_budget(L);
  }
  return (moe_status_t)r;
}

moe_status_t moe_layer_set_cost_model(moe_layer_t* L, const moe_cost_model_t* cost) {
  if (!L || !cost || cost->n_points < 1 || cost->n_points > MOE_COST_POINTS) return MOE_ERR_INVALID;
  L->cost = *cost;
  return MOE_OK;
}

int32_t moe_layer_last_launches(const moe_layer_t* L) { return L ? L->last_launches : 0; }

moe_status_t moe_layer_set_profiling(moe_layer_t* L, int32_t enable) {
  if (!L) return MOE_ERR_INVALID;
  if (enable && L->pev.empty()) {
    L->pev.resize(4096);
    for (auto& e : L->pev) CUDA_TRY(cudaEventCreate(&e));
  }
  L->prof = enable != 0;
  return MOE_OK;
}

moe_status_t moe_layer_set_comm_only(moe_layer_t* L, int32_t enable) {
  if (!L) return MOE_ERR_INVALID;
  L->comm_only = enable != 0 && L->cfg.ep > 1;
  return MOE_OK;
}

moe_status_t moe_layer_stage_ms(const moe_layer_t* L, float* ms, int32_t* counts) {
  if (!L || !ms) return MOE_ERR_INVALID;
  for (int i = 0; i < MOE_NUM_STAGES; ++i) {
    ms[i] = 0.f;
    if (counts) counts[i] = 0;
  }
  if (L->pev_used > 0) CUDA_TRY(cudaEventSynchronize(L->pev[L->pev_used - 1]));
  // exposed all2all: comm intervals not covered by any compute interval
  std::vector<std::pair<float, float>> comp, comm;
  int t0 = -1;
  for (auto& m : L->marks)
    if (m.stage == MOE_STAGE_TOTAL) t0 = m.e0;
  for (auto& m : L->marks) {
    float v = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&v, L->pev[m.e0], L->pev[m.e1]));
    ms[m.stage] += v;
    if (counts) counts[m.stage] += 1;
    if (t0 >= 0 && m.stage != MOE_STAGE_TOTAL) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, L->pev[t0], L->pev[m.e0]);
      cudaEventElapsedTime(&b, L->pev[t0], L->pev[m.e1]);
      (m.stage == MOE_STAGE_DISPATCH || m.stage == MOE_STAGE_COMB_A2A ? comm : comp).push_back({a, b});
    }
  }
  std::sort(comp.begin(), comp.end());
  float exposed = 0.f;
  for (auto& c : comm) {
    // subtract the union of compute intervals from [c.first, c.second]
    float cur = c.first, cov = 0.f;
    for (auto& k : comp) {
      if (k.second <= cur) continue;
      if (k.first >= c.second) break;
      float lo = std::max(cur, k.first), hi = std::min(c.second, k.second);
      if (hi > lo) { cov += hi - lo; cur = hi; }
    }
    exposed += std::max(0.f, (c.second - c.first) - cov);
  }
  ms[MOE_STAGE_EXPOSED_A2A] = exposed;
  return MOE_OK;
}

namespace {

// One forward's context, shared by its phases (routing, EP = 1 compute + combine,
// the EP > 1 pipeline, debug outputs).
struct Fwd {
  moe_layer* L;
  const void* x;
  int64_t T;
  void* y;
  const moe_plan_t* plan_in;
  cudaStream_t st;
  moe_debug_t* dbg;
  moe_plan_t plan;
  int num_ctas = 0;
  int32_t* topk_idx = nullptr;
  float* topk_w = nullptr;
  bool override_routing = false;
  // set by the routing phase
  bool side = false, fp8 = false, gather = false, lr_ep = false;
  int fuse = 0;
};

// Router (K1) + topKGating (K2) + histogram + split (K3), with the shared
// experts launched alongside.
moe_status_t fwd_routing(Fwd& F) {
  moe_layer* L = F.L;
  const moe_config_t& c = L->cfg;
  const void* x = F.x;
  const int64_t T = F.T;
  void* y = F.y;
  cudaStream_t st = F.st;
  moe_debug_t* dbg = F.dbg;
  moe_plan_t& plan = F.plan;
  const moe_plan_t* plan_in = F.plan_in;
  const int E = c.num_experts, k = c.top_k, H = c.hidden, D = c.ep, E_loc = L->E_loc;
  const int num_ctas = F.num_ctas;
  int32_t* topk_idx = F.topk_idx;
  float* topk_w = F.topk_w;
  const bool override_routing = F.override_routing;
  (void)x; (void)y; (void)dbg; (void)plan_in; (void)E_loc; (void)override_routing; (void)topk_idx;
  // ---- Router (K1) + topKGating (K2) + histogram
  int p0 = prof_rec(L, st);
  if (T > 0 && !override_routing) {
    GemmArgs ra = base_args(EPI_F32, num_ctas);
    ra.A = x;
    ra.a_rows = T;
    ra.B0 = L->wr_pad;
    ra.b_rows = 256;
    ra.K = H;
    ra.N = E;
    ra.out = L->logits;
    ra.ldo = E;
    ra.bias = L->w.router_bias;
    ra.m_single = (int)T;
    ra.tile_counter = L->tickets;
    KERNEL_TRY(gemm_launch(ra, st));
  }
  int p1 = prof_rec(L, st);
  prof_mark(L, MOE_STAGE_ROUTER, p0, p1);

  // Shared experts depend only on x: they run on s_side, concurrently
  // with topKGating / split (HBM-bound kernels that co-reside with the GEMM's
  // CTAs) and, for ep > 1, with the count exchange, host wait and dispatch(0).
  // ep == 1 with EPSMOE_FUSE_COMBINE=1/2 (off by default, measured no faster):
  // the shared DownGemm is deferred and meets the combine (EPI_COMBINE epilogue,
  // or token pieces), so only GateUp runs here.  (A debug request for s
  // materialises it: unfused path.)
  const int fuse =
      ((D == 1) && L->SF && T > 0 && !c.local_reduce && !(dbg && dbg->shared_out)) ? L->fuse_combine : 0;
  auto shared_experts = [&](cudaStream_t ss) -> int {
    if (!L->SF || T == 0) return 0;
    int q0 = prof_rec(L, ss);
    GemmArgs a = base_args(EPI_SWIGLU, num_ctas);
    a.A = x;
    a.a_rows = T;
    a.B0 = L->w.ws_gate;
    a.B1 = L->w.ws_up;
    a.b_rows = L->SF;
    a.K = H;
    a.N = L->SF;
    a.out = L->hs;
    a.ldo = L->SF;
    a.m_single = (int)T;
    a.rows_hint = (double)T;
    a.tile_counter = (ss == L->s_side) ? L->tickets + 2 : L->tickets;
    int e = gemm_launch(a, ss);
    if (e) return e;
    ++L->last_launches;
    if (fuse) {
      prof_mark(L, MOE_STAGE_SHARED, q0, prof_rec(L, ss));
      return 0;
    }
    GemmArgs b = base_args(EPI_BF16, num_ctas);
    b.A = L->hs;
    b.a_rows = T;
    b.B0 = L->w.ws_down;
    b.b_rows = H;
    b.K = L->SF;
    b.N = H;
    b.out = L->s;
    b.ldo = H;
    b.m_single = (int)T;
    b.rows_hint = (double)T;
    b.tile_counter = a.tile_counter;
    e = gemm_launch(b, ss);
    if (!e) ++L->last_launches;
    prof_mark(L, MOE_STAGE_SHARED, q0, prof_rec(L, ss));
    return e;
  };
  // ep == 1: the routing kernels stream with L2 evict-first hints, so they
  // co-run with the shared GEMMs (measured ~1% faster per layer than in order).
  const bool has_shared = L->SF && T > 0 && !(L->comm_only && D > 1);
  // (small decode batches: the routing kernels are latency-bound and a concurrent
  // persistent GEMM only delays them, so they stay in order below 8K tokens)
  const bool side = has_shared && (D > 1 || (L->overlap_shared && T >= 8192));
  if (side) {
    CUDA_TRY(cudaEventRecord(L->ev_router, st));
    CUDA_TRY(cudaStreamWaitEvent(L->s_side, L->ev_router, 0));
    int e = shared_experts(L->s_side);
    if (e) { set_error(std::string("shared experts: ") + cudaGetErrorString((cudaError_t)e)); return MOE_ERR_CUDA; }
    CUDA_TRY(cudaEventRecord(L->ev_shared, L->s_side));
  }

  KERNEL_TRY(launch_gate_topk(L->logits, (int)T, E, k, c.norm_topk, c.routed_scale, override_routing ? 1 : 0,
                              c.route_groups > 1 ? c.route_groups : 0, c.route_topk_groups, topk_idx, topk_w,
                              L->range_hist, st));
  KERNEL_TRY(launch_range_scan(L->range_hist, (int)T, E, L->range_off, L->hist, L->seg_start, st));
  ++L->last_launches;  // range scan + expert scan
  // ---- split (K3): x -> send rows, expert-major (R6).  At ep == 1 the send
  // buffer is only the GateUp GEMM's A operand; with EPSMOE_GATHER=1 the split
  // is index-only and the GEMM gathers x's rows itself (measured slower, off).
  const bool fp8 = c.dispatch_fp8 != 0;
  const bool gather = (D == 1) && L->gather_a && T > 0 && !fp8;
  // ep > 1 with local_reduce: index-only here (pos feeds the dedup rows' codes);
  // the dedup permute runs once the plan fixes the chunks
  const bool lr_ep = (D > 1) && c.local_reduce;
  KERNEL_TRY(launch_permute(x, (int)T, H, E, k, topk_idx, L->range_off, L->seg_start,
                            (gather || lr_ep) ? nullptr : L->send, L->pos, gather ? L->row_token : nullptr,
                            lr_ep ? 0 : (fp8 ? (D == 1 ? 1 : 2) : 0), L->sendq, L->qpitch, st));
  prof_mark(L, MOE_STAGE_ROUTE, p1, prof_rec(L, st));
  if (has_shared && !side) {
    int e = shared_experts(st);
    if (e) { set_error(std::string("shared experts: ") + cudaGetErrorString((cudaError_t)e)); return MOE_ERR_CUDA; }
  }

  F.side = side;
  F.fp8 = fp8;
  F.gather = gather;
  F.lr_ep = lr_ep;
  F.fuse = fuse;
  return MOE_OK;
}

// EP = 1: ComputeMoE over the plan's chunks on local rows, then the combine.
moe_status_t fwd_local(Fwd& F) {
  moe_layer* L = F.L;
  const moe_config_t& c = L->cfg;
  const void* x = F.x;
  const int64_t T = F.T;
  void* y = F.y;
  cudaStream_t st = F.st;
  moe_debug_t* dbg = F.dbg;
  moe_plan_t& plan = F.plan;
  const moe_plan_t* plan_in = F.plan_in;
  const int E = c.num_experts, k = c.top_k, H = c.hidden, D = c.ep, E_loc = L->E_loc;
  const int num_ctas = F.num_ctas;
  int32_t* topk_idx = F.topk_idx;
  float* topk_w = F.topk_w;
  const bool override_routing = F.override_routing;
  (void)x; (void)y; (void)dbg; (void)plan_in; (void)E_loc; (void)override_routing; (void)topk_idx;
  const bool side = F.side, fp8 = F.fp8, gather = F.gather, lr_ep = F.lr_ep;
  const int fuse = F.fuse;
  (void)side; (void)fp8; (void)gather; (void)lr_ep; (void)fuse;
  // ---- EP = 1: no all2all; every chunk is local (C = 0 => PN = 1 is optimal)
  if (!plan_in) plan_compute(c, L->cost, T, nullptr, &plan);
  if (side) CUDA_TRY(cudaStreamWaitEvent(st, L->ev_shared, 0));
  const bool two = L->chunk_streams > 1 && plan.num_chunks > 1 && T > 0;
  if (two) {  // odd chunks on s_comp2 (after the routing on st)
    CUDA_TRY(cudaEventRecord(L->ev_routed, st));
    CUDA_TRY(cudaStreamWaitEvent(L->s_comp2, L->ev_routed, 0));
  }
  for (int ch = 0; T > 0 && ch < plan.num_chunks; ++ch) {
    int g0 = plan.group_begin[ch], g1 = plan.group_begin[ch + 1];
    cudaStream_t cs = (two && (ch & 1)) ? L->s_comp2 : st;
    // maximal runs of equal kind inside the chunk
    int a = g0;
    while (a < g1) {
      int b = a + 1;
      while (b < g1 && plan.expert_kind[b] == plan.expert_kind[a]) ++b;
      int err = compute_moe(L, gather ? x : L->send, gather ? T : L->send_cap, L->seg_start, L->hist, a, b,
                            plan.expert_kind[a], num_ctas, pick_cta_pair(plan, (double)T * k / E), plan.tile_m != 0,
                            (double)T * k / E, cs, gather ? L->row_token : nullptr);
      if (err) { set_error(std::string("ComputeMoE: ") + cudaGetErrorString((cudaError_t)err)); return MOE_ERR_CUDA; }
      a = b;
    }
  }
  if (two) {
    CUDA_TRY(cudaEventRecord(L->ev_comp2, L->s_comp2));
    CUDA_TRY(cudaStreamWaitEvent(st, L->ev_comp2, 0));
  }
  int c0 = prof_rec(L, st);
  if (fuse == 2) {
    // shared DownGemm in token pieces; piece p's combine (HBM-bound) runs on
    // s_side next to piece p+1's DownGemm (compute-bound) on the other SMs' slack
    const int P = (T >= 8192) ? moe_layer::COMB_PIECES : 1;
    for (int pc = 0; pc < P; ++pc) {
      const int64_t t0 = T * pc / P, t1 = T * (pc + 1) / P;
      if (t1 == t0) continue;
      GemmArgs b = base_args(EPI_BF16, num_ctas);
      b.A = static_cast<const uint16_t*>(L->hs) + t0 * L->SF;
      b.a_rows = t1 - t0;
      b.B0 = L->w.ws_down;
      b.b_rows = H;
      b.K = L->SF;
      b.N = H;
      b.out = static_cast<uint16_t*>(L->s) + t0 * H;
      b.ldo = H;
      b.m_single = (int)(t1 - t0);
      b.tile_counter = L->tickets;
      int e = gemm_launch(b, st);
      if (e) { set_error(std::string("shared DownGemm: ") + cudaGetErrorString((cudaError_t)e)); return MOE_ERR_CUDA; }
      ++L->last_launches;
      CUDA_TRY(cudaEventRecord(L->ev_piece[pc], st));
      CUDA_TRY(cudaStreamWaitEvent(L->s_side, L->ev_piece[pc], 0));
      KERNEL_TRY(launch_combine(L->o, static_cast<const uint16_t*>(L->s) + t0 * H, (int)(t1 - t0), H, k, L->pos + t0 * k, topk_w + t0 * k,
                                reinterpret_cast<uint16_t*>(y) + t0 * H, L->s_side));
    }
    CUDA_TRY(cudaEventRecord(L->ev_shared, L->s_side));
    CUDA_TRY(cudaStreamWaitEvent(st, L->ev_shared, 0));
  } else if (fuse == 1) {
    // shared DownGemm + K7 in one kernel: y = bf16(fmaf_j(w_j, o[pos[t][j]], fp32(bf16(hs W_sdown^T))))
    GemmArgs b = base_args(EPI_COMBINE, num_ctas);
    b.A = L->hs;
    b.a_rows = T;
    b.B0 = L->w.ws_down;
    b.b_rows = H;
    b.K = L->SF;
    b.N = H;
    b.out = y;
    b.ldo = H;
    b.m_single = (int)T;
    b.tile_counter = L->tickets;
    b.comb_o = L->o;
    b.comb_pos = L->pos;
    b.comb_w = topk_w;
    b.comb_k = k;
    int e = gemm_launch(b, st);
    if (e) { set_error(std::string("shared DownGemm + combine: ") + cudaGetErrorString((cudaError_t)e)); return MOE_ERR_CUDA; }
    ++L->last_launches;
  } else if (c.local_reduce) {
    // R16 at ep == 1: groups = chunks; LocalReduce partials + home sum in one pass
    LrChunks chs;
    chs.n = plan.num_chunks;
    for (int i = 0; i <= plan.num_chunks; ++i) chs.begin[i] = plan.group_begin[i];
    KERNEL_TRY(launch_lr_combine_local(L->o, L->SF ? L->s : nullptr, (int)T, H, k, topk_idx, L->pos, topk_w, E,
                                       chs, y, st));
  } else {
    KERNEL_TRY(launch_combine(L->o, L->SF ? L->s : nullptr, (int)T, H, k, L->pos, topk_w, y, st));
  }
  prof_mark(L, MOE_STAGE_COMBINE, c0, prof_rec(L, st));
  return MOE_OK;
}

// EP > 1: count exchange (C3), plan, layouts, and Algorithm 1's chunked
// dispatch / ComputeMoE / combine over the transport or the put kernels.
moe_status_t fwd_ep(Fwd& F) {
  moe_layer* L = F.L;
  const moe_config_t& c = L->cfg;
  const void* x = F.x;
  const int64_t T = F.T;
  void* y = F.y;
  cudaStream_t st = F.st;
  moe_debug_t* dbg = F.dbg;
  moe_plan_t& plan = F.plan;
  const moe_plan_t* plan_in = F.plan_in;
  const int E = c.num_experts, k = c.top_k, H = c.hidden, D = c.ep, E_loc = L->E_loc;
  const int num_ctas = F.num_ctas;
  int32_t* topk_idx = F.topk_idx;
  float* topk_w = F.topk_w;
  const bool override_routing = F.override_routing;
  (void)x; (void)y; (void)dbg; (void)plan_in; (void)E_loc; (void)override_routing; (void)topk_idx;
  const bool side = F.side, fp8 = F.fp8, gather = F.gather, lr_ep = F.lr_ep;
  const int fuse = F.fuse;
  (void)side; (void)fp8; (void)gather; (void)lr_ep; (void)fuse;
  // ---- EP > 1: count exchange (C3), plan, chunked dispatch / compute / combine
  TR_TRY(L->tr->allgather_i32(L->hist, L->ghist, E, st));
  CUDA_TRY(cudaMemcpyAsync(L->ghist_host, L->ghist, sizeof(int32_t) * D * E, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaEventRecord(L->ev_hist, st));
  CUDA_TRY(cudaEventSynchronize(L->ev_hist));
  const int32_t* gh = L->ghist_host;
  if (!plan_in) {
    int64_t m = 0;
    for (int i = 0; i < D * E; ++i) m += gh[i];
    plan_compute(c, L->cost, m / k, gh, &plan);
  }
  const int me = c.rank;
  // send offsets (local, expert-major) and recv layout [e_l][src] (R6)
  std::vector<int64_t> send_off(E + 1, 0);
  std::vector<int64_t> recv_off((size_t)E_loc * D + 1, 0);
  exchange_layout(c, gh, send_off.data(), recv_off.data());
  if (recv_off.back() > L->recv_cap) { set_error("recv rows exceed capacity"); return MOE_ERR_CAPACITY; }
  // Token-sliced chunks (R8 extension, S > 1): chunk c = (expert group c / S,
  // source-token slice c % S); the (expert, slice) counts of every rank take
  // one more exchange.  Send rows stay (e, t), so (e, s) is contiguous; recv
  // rows become (e_l, s, src, t), so each expert's rows of a chunk are.  Every
  // row still meets the same weights and returns to the same send row, so
  // slicing changes no bit of y.
  const int S = plan.token_slices;
  const int NG = plan.num_chunks / S;
  const int32_t* hsl = gh;  // [D][E * S]
  if (S > 1) {
    KERNEL_TRY(launch_slice_hist(topk_idx, (int)T, k, E, S, L->slice_hist, st));
    TR_TRY(L->tr->allgather_i32(L->slice_hist, L->gslice, E * S, st));
    CUDA_TRY(cudaMemcpyAsync(L->gslice_host, L->gslice, sizeof(int32_t) * D * E * S, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(L->ev_hist, st));
    CUDA_TRY(cudaEventSynchronize(L->ev_hist));
    hsl = L->gslice_host;
  }
  auto cnt = [&](int src, int ex, int sl) -> int64_t { return hsl[((int64_t)src * E + ex) * S + sl]; };
  std::vector<int64_t> send_pos((size_t)E * S);
  for (int ex = 0; ex < E; ++ex) {
    int64_t p0 = send_off[ex];
    for (int sl = 0; sl < S; ++sl) {
      send_pos[(size_t)ex * S + sl] = p0;
      p0 += cnt(me, ex, sl);
    }
  }
  std::vector<int64_t> recv_pos((size_t)E_loc * S * D + 1, 0);  // (e_l, s, src)
  for (int el = 0, i = 0; el < E_loc; ++el)
    for (int sl = 0; sl < S; ++sl)
      for (int src = 0; src < D; ++src, ++i) recv_pos[i + 1] = recv_pos[i] + cnt(src, me * E_loc + el, sl);
  auto rpos = [&](int el, int sl, int src) -> int64_t { return recv_pos[((size_t)el * S + sl) * D + src]; };
  // per-chunk GEMM row tables: chunk c's experts at [c * E_loc + e_l]
  int32_t* tstart = L->tables_host;
  int32_t* tcount = L->tables_host + moe_layer::TBL;
  for (int ch = 0; ch < plan.num_chunks; ++ch) {
    const int grp = ch / S, sl = ch % S;
    for (int el = plan.group_begin[grp]; el < plan.group_begin[grp + 1]; ++el) {
      tstart[ch * E_loc + el] = (int32_t)rpos(el, sl, 0);
      tcount[ch * E_loc + el] = (int32_t)(rpos(el, sl, D - 1) + cnt(D - 1, me * E_loc + el, sl) - rpos(el, sl, 0));
    }
  }
  const size_t tbytes = sizeof(int32_t) * (size_t)plan.num_chunks * E_loc;
  CUDA_TRY(cudaMemcpyAsync(L->recv_start_d, tstart, tbytes, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(L->recv_count_d, tcount, tbytes, cudaMemcpyHostToDevice, st));
  (void)NG;
  // ---- local_reduce (R16): the dedup layout needs the plan's chunks, and the
  // unique-row counts per (chunk, peer) need a second (G-int) exchange
  const int G = plan.num_chunks * D;
  std::vector<int64_t> usend_off(G + 1, 0);                     // my send rows of group g = c*D + peer
  std::vector<int64_t> urecv((size_t)plan.num_chunks * D + 1, 0);  // first unique recv row of (c, src)
  const int32_t* ug = L->ughist_host;                           // [D][G]
  if (lr_ep) {
    int q0 = prof_rec(L, st);
    LrChunks chs;
    chs.n = plan.num_chunks;
    for (int i = 0; i <= plan.num_chunks; ++i) chs.begin[i] = plan.group_begin[i];
    KERNEL_TRY(launch_lr_count(topk_idx, (int)T, k, E_loc, D, chs, L->range_hist, st));
    KERNEL_TRY(launch_range_scan(L->range_hist, (int)T, G, L->range_off, L->u_hist, L->u_start, st));
    KERNEL_TRY(launch_lr_permute(x, (int)T, H, k, topk_idx, topk_w, L->pos, L->seg_start, E_loc, D, chs,
                                 L->range_off, L->u_start, fp8 ? nullptr : L->send, fp8 ? L->sendq : nullptr,
                                 L->qpitch, L->posg, L->meta_send, st));
    prof_mark(L, MOE_STAGE_ROUTE, q0, prof_rec(L, st));
    TR_TRY(L->tr->allgather_i32(L->u_hist, L->ughist, G, st));
    CUDA_TRY(cudaMemcpyAsync(L->ughist_host, L->ughist, sizeof(int32_t) * D * G, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(L->ev_hist, st));
    CUDA_TRY(cudaEventSynchronize(L->ev_hist));
    for (int g = 0; g < G; ++g) usend_off[g + 1] = usend_off[g] + ug[(size_t)me * G + g];
    int64_t row = 0;
    for (int ch = 0; ch < plan.num_chunks; ++ch)
      for (int src = 0; src < D; ++src) {
        urecv[(size_t)ch * D + src] = row;
        row += ug[(size_t)src * G + ch * D + me];
      }
    urecv[G] = row;
    if (row > L->recv_cap) { set_error("unique recv rows exceed capacity"); return MOE_ERR_CAPACITY; }
    int32_t* tb = L->tables_host + 2 * moe_layer::TBL;  // [E_loc*D+1] recv_off, then [G+1] urecv
    for (int i = 0; i <= E_loc * D; ++i) tb[i] = (int32_t)recv_off[i];
    for (int i = 0; i <= G; ++i) tb[MOE_MAX_EXPERTS + 4 + i] = (int32_t)urecv[i];
    CUDA_TRY(cudaMemcpyAsync(L->lr_recv_off_d, tb, sizeof(int32_t) * (E_loc * D + 1), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(L->lr_usrc_d, tb + MOE_MAX_EXPERTS + 4, sizeof(int32_t) * (G + 1),
                             cudaMemcpyHostToDevice, st));
  }
  // ---- a2a_p2p: this forward's put-kernel segments (rows of each chunk, per
  // peer, at the peer's own offsets) and consumer flag addresses
  const bool p2p = c.a2a_p2p != 0;
  uint32_t epoch = 0;
  int p2p_nseg[2][MOE_MAX_CHUNKS] = {};
  int64_t p2p_total[2][MOE_MAX_CHUNKS] = {};
  // fused combine: the chunk's DownGemm scatters its rows into the home ranks'
  // combine buffers (one GEMM launch per chunk: its experts share one kind)
  bool fuse_comb[MOE_MAX_CHUNKS] = {};
  int fuse_nrseg[MOE_MAX_CHUNKS] = {};
  if (p2p) {
    if (L->peer_ws.empty()) {  // first forward (collective): map the peers, learn their layouts
      TR_TRY(L->tr->map_peers(L->ws_base, L->peer_ws));
      const void* bufs[moe_layer::P2P_NBUF] = {L->recv, L->recvq, L->recvu, L->meta_recv, L->comb, L->p2p_flags};
      int64_t mine[moe_layer::P2P_NBUF];
      for (int b = 0; b < moe_layer::P2P_NBUF; ++b)
        mine[b] = bufs[b] ? (int64_t)((const char*)bufs[b] - L->ws_base) : -1;
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
      if (ge) return (moe_status_t)ge;
    }
    epoch = ++L->p2p_epoch;
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
            row += cnt(src, d * E_loc + el, sl);
          }
      row = 0;
      for (int ex = 0; ex < E; ++ex)
        for (int sl = 0; sl < S; ++sl) {
          spos_all[(size_t)d * E * S + (size_t)ex * S + sl] = row;
          row += cnt(d, ex, sl);
        }
    }
    std::vector<int64_t> urecv_all, usend_all;
    if (lr_ep) {
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
    auto* hsegs = reinterpret_cast<epsmoe::P2PSeg*>(L->p2p_host);
    auto* hpre = reinterpret_cast<int64_t*>(L->p2p_host + P2P_SEGS_BYTES);
    auto* hfp = reinterpret_cast<uint32_t**>(L->p2p_host + P2P_SEGS_BYTES + P2P_PRE_BYTES);
    const size_t rowb = (size_t)H * 2;
    const size_t drowb = fp8 ? (size_t)L->qpitch : rowb;
    const size_t metab = (size_t)lr_meta_pitch(k) * sizeof(int32_t);
    char* ds = fp8 ? (char*)L->sendq : (char*)L->send;
    const int dr_id = fp8 ? moe_layer::P2P_RECVQ : (lr_ep ? moe_layer::P2P_RECVU : moe_layer::P2P_RECV);
    for (int dir = 0; dir < 2; ++dir)
      for (int ch = 0; ch < plan.num_chunks; ++ch) {
        const size_t slot = (size_t)dir * MOE_MAX_CHUNKS + ch;
        epsmoe::P2PSeg* sg = hsegs + slot * moe_layer::P2P_MAXS;
        int64_t* pr = hpre + slot * (moe_layer::P2P_MAXS + 1);
        int n = 0;
        pr[0] = 0;
        auto add = [&](const char* src, char* dst, int64_t bytes) {
          if (bytes <= 0 || n >= moe_layer::P2P_MAXS) return;
          sg[n].src = reinterpret_cast<const uint4*>(src);
          sg[n].dst = reinterpret_cast<uint4*>(dst);
          pr[n + 1] = pr[n] + bytes / 16;
          ++n;
        };
        for (int d = 0; d < D; ++d)
          hfp[slot * D + d] =
              reinterpret_cast<uint32_t*>(peer_buf(d, moe_layer::P2P_FLAGS, (int64_t)(slot * D + me) * 4));
        const int sl = ch % S, g0 = plan.group_begin[ch / S], g1 = plan.group_begin[ch / S + 1];
        for (int peer = 0; peer < D; ++peer) {
          if (lr_ep && dir == 0) {
            const int64_t s0 = usend_off[ch * D + peer], ns = ug[(size_t)me * G + ch * D + peer];
            const int64_t r0 = urecv_all[(size_t)peer * (G + 1) + ch * D + me];
            add(ds + s0 * drowb, peer_buf(peer, dr_id, r0 * drowb), ns * (int64_t)drowb);
            add((char*)L->meta_send + s0 * metab, peer_buf(peer, moe_layer::P2P_META, r0 * metab), ns * (int64_t)metab);
          } else if (lr_ep) {
            const int64_t r0 = urecv[(size_t)ch * D + peer], nb = ug[(size_t)peer * G + ch * D + me];
            const int64_t s0 = usend_all[(size_t)peer * (G + 1) + ch * D + me];
            add((char*)L->recvu + r0 * rowb, peer_buf(peer, moe_layer::P2P_COMB, s0 * rowb), nb * (int64_t)rowb);
          } else {
            for (int el = g0; el < g1; ++el) {
              if (dir == 0) {
                const int ex = peer * E_loc + el;
                add(ds + send_pos[(size_t)ex * S + sl] * drowb,
                    peer_buf(peer, dr_id, rpos_all[peer * RP + ((size_t)el * S + sl) * D + me] * drowb),
                    cnt(me, ex, sl) * (int64_t)drowb);
              } else {
                const int ex = me * E_loc + el;
                add((char*)L->o + rpos(el, sl, peer) * rowb,
                    peer_buf(peer, moe_layer::P2P_COMB, spos_all[(size_t)peer * E * S + (size_t)ex * S + sl] * rowb),
                    cnt(peer, ex, sl) * (int64_t)rowb);
              }
            }
          }
        }
        p2p_nseg[dir][ch] = n;
        p2p_total[dir][ch] = pr[n];
        if (dir == 1 && L->p2p_fuse && !lr_ep && !L->split_rem && !L->comm_only) {
          bool one_kind = true;
          for (int el = g0 + 1; el < g1; ++el) one_kind &= plan.expert_kind[el] == plan.expert_kind[g0];
          if (one_kind) {
            auto* rs = reinterpret_cast<epsmoe::GemmRowSeg*>(L->p2p_host + P2P_SEGS_BYTES + P2P_PRE_BYTES +
                                                               p2p_fptr_bytes(D)) +
                       (size_t)ch * moe_layer::P2P_MAXS;
            int nr = 0;
            for (int el = g0; el < g1; ++el)  // GEMM rows (e_l, slice, src) ascending
              for (int src = 0; src < D; ++src) {
                const int ex = me * E_loc + el;
                const int64_t rows = cnt(src, ex, sl);
                if (!rows || nr >= moe_layer::P2P_MAXS) continue;
                rs[nr].r0 = rpos(el, sl, src);
                rs[nr].n = rows;
                rs[nr].dst = peer_buf(src, moe_layer::P2P_COMB, spos_all[(size_t)src * E * S + (size_t)ex * S + sl] * rowb);
                ++nr;
              }
            fuse_comb[ch] = true;
            fuse_nrseg[ch] = nr;
          }
        }
      }
    CUDA_TRY(cudaMemcpyAsync(L->p2p_tab, L->p2p_host, p2p_table_bytes(D), cudaMemcpyHostToDevice, st));
  }
  const bool copy_engine = c.a2a_p2p == 2;
  auto p2p_put = [&](int dir, int ch, cudaStream_t ps) -> moe_status_t {
    const size_t slot = (size_t)dir * MOE_MAX_CHUNKS + ch;
    auto* dsegs = reinterpret_cast<epsmoe::P2PSeg*>(L->p2p_tab) + slot * moe_layer::P2P_MAXS;
    auto* dpre = reinterpret_cast<int64_t*>(L->p2p_tab + P2P_SEGS_BYTES) + slot * (moe_layer::P2P_MAXS + 1);
    auto* dfp = reinterpret_cast<uint32_t**>(L->p2p_tab + P2P_SEGS_BYTES + P2P_PRE_BYTES) + slot * D;
    if (copy_engine) {
      // the same segments as cudaMemcpyAsync peer copies (copy engines: no SM
      // moves a row), then one thread raises the chunk's flags after them
      const auto* hs = reinterpret_cast<const epsmoe::P2PSeg*>(L->p2p_host) + slot * moe_layer::P2P_MAXS;
      const auto* hp = reinterpret_cast<const int64_t*>(L->p2p_host + P2P_SEGS_BYTES) + slot * (moe_layer::P2P_MAXS + 1);
      // one batched call for the chunk's segments (cudaMemcpyBatchAsync, CUDA 12.8+),
      // else one cudaMemcpyAsync per segment
      const int n = p2p_nseg[dir][ch];
      if (n > 0) {
        std::vector<void*> dsts(n), srcs(n);
        std::vector<size_t> sizes(n);
        for (int i = 0; i < n; ++i) {
          dsts[i] = hs[i].dst;
          srcs[i] = const_cast<uint4*>(hs[i].src);
          sizes[i] = (size_t)(hp[i + 1] - hp[i]) * 16;
        }
        cudaMemcpyAttributes attr;
        std::memset(&attr, 0, sizeof(attr));
        attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        size_t attr_idx = 0, fail_idx = 0;
        if (L->ce_batch && cudaMemcpyBatchAsync(dsts.data(), srcs.data(), sizes.data(), (size_t)n, &attr, &attr_idx, 1,
                                                &fail_idx, ps) != cudaSuccess) {
          (void)cudaGetLastError();
          L->ce_batch = false;  // not supported here: per-segment copies from now on
          for (int i = 0; i < n; ++i) CUDA_TRY(cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDeviceToDevice, ps));
        } else if (!L->ce_batch) {
          for (int i = 0; i < n; ++i) CUDA_TRY(cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDeviceToDevice, ps));
        }
      }
      KERNEL_TRY(launch_p2p_signal(dfp, D, epoch, ps));
      TR_TRY(L->tr->p2p_after_put((int)slot, ps));
      return MOE_OK;
    }
    KERNEL_TRY(launch_p2p_put(dsegs, dpre, p2p_nseg[dir][ch], p2p_total[dir][ch], 2 * L->comm_ctas,
                              L->p2p_done + slot, dfp, D, epoch, ps));
    TR_TRY(L->tr->p2p_after_put((int)slot, ps));
    return MOE_OK;
  };
  CUDA_TRY(cudaEventRecord(L->ev_ready, st));
  CUDA_TRY(cudaStreamWaitEvent(L->s_disp, L->ev_ready, 0));
  CUDA_TRY(cudaStreamWaitEvent(L->s_comb, L->ev_ready, 0));
  const size_t row_bytes = (size_t)H * 2;
  // dispatch payload: bf16 rows, or packed FP8 rows (NEXT-2) dequantised per chunk on arrival
  char* dsend = fp8 ? (char*)L->sendq : (char*)L->send;
  char* drecv = fp8 ? (char*)L->recvq : (char*)L->recv;
  const size_t drow = fp8 ? (size_t)L->qpitch : row_bytes;
  const size_t meta_bytes = (size_t)lr_meta_pitch(k) * sizeof(int32_t);
  auto dispatch = [&](int ch) -> moe_status_t {
    const int sl = ch % S, g0 = plan.group_begin[ch / S], g1 = plan.group_begin[ch / S + 1];
    int d0 = prof_rec(L, L->s_disp);
    if (p2p) {
      moe_status_t r = p2p_put(0, ch, L->s_disp);
      if (r) return r;
      prof_mark(L, MOE_STAGE_DISPATCH, d0, prof_rec(L, L->s_disp));
      CUDA_TRY(cudaEventRecord(L->ev_disp[ch], L->s_disp));
      return MOE_OK;
    }
    TR_TRY(L->tr->group_start(0));
    if (lr_ep) {  // one unique-row message + its meta per peer (R16)
      char* urows = fp8 ? (char*)L->recvq : (char*)L->recvu;
      for (int peer = 0; peer < D; ++peer) {
        const int64_t s0 = usend_off[ch * D + peer], ns = ug[(size_t)me * G + ch * D + peer];
        if (ns) {
          TR_TRY(L->tr->send(dsend + s0 * drow, ns * drow, peer, 0, L->s_disp));
          TR_TRY(L->tr->send((char*)L->meta_send + s0 * meta_bytes, ns * meta_bytes, peer, 0, L->s_disp));
        }
        const int64_t r0 = urecv[(size_t)ch * D + peer], nr = ug[(size_t)peer * G + ch * D + me];
        if (nr) {
          TR_TRY(L->tr->recv(urows + r0 * drow, nr * drow, peer, 0, L->s_disp));
          TR_TRY(L->tr->recv((char*)L->meta_recv + r0 * meta_bytes, nr * meta_bytes, peer, 0, L->s_disp));
        }
      }
    }
    for (int peer = 0; peer < D && !lr_ep; ++peer)
      for (int el = g0; el < g1; ++el) {
        const int ex = peer * E_loc + el;
        const int64_t n_send = cnt(me, ex, sl);
        if (n_send)
          TR_TRY(L->tr->send(dsend + send_pos[(size_t)ex * S + sl] * drow, n_send * drow, peer, 0, L->s_disp));
        const int64_t n_recv = cnt(peer, me * E_loc + el, sl);
        if (n_recv) TR_TRY(L->tr->recv(drecv + rpos(el, sl, peer) * drow, n_recv * drow, peer, 0, L->s_disp));
      }
    TR_TRY(L->tr->group_end(0, L->s_disp));
    prof_mark(L, MOE_STAGE_DISPATCH, d0, prof_rec(L, L->s_disp));
    CUDA_TRY(cudaEventRecord(L->ev_disp[ch], L->s_disp));
    return MOE_OK;
  };
  auto combine_send = [&](int ch) -> moe_status_t {
    const int sl = ch % S, g0 = plan.group_begin[ch / S], g1 = plan.group_begin[ch / S + 1];
    CUDA_TRY(cudaStreamWaitEvent(L->s_comb, L->ev_gemm[ch], 0));
    int b0 = prof_rec(L, L->s_comb);
    if (p2p) {
      if (!fuse_comb[ch]) {
        moe_status_t r = p2p_put(1, ch, L->s_comb);
        if (r) return r;
      }
      prof_mark(L, MOE_STAGE_COMB_A2A, b0, prof_rec(L, L->s_comb));
      return MOE_OK;
    }
    TR_TRY(L->tr->group_start(1));
    if (lr_ep) {  // each unique row returns as its LocalReduce partial (R16)
      for (int peer = 0; peer < D; ++peer) {
        const int64_t r0 = urecv[(size_t)ch * D + peer], nb = ug[(size_t)peer * G + ch * D + me];
        if (nb) TR_TRY(L->tr->send((char*)L->recvu + r0 * row_bytes, nb * row_bytes, peer, 1, L->s_comb));
        const int64_t s0 = usend_off[ch * D + peer], nh = ug[(size_t)me * G + ch * D + peer];
        if (nh) TR_TRY(L->tr->recv((char*)L->comb + s0 * row_bytes, nh * row_bytes, peer, 1, L->s_comb));
      }
    }
    for (int peer = 0; peer < D && !lr_ep; ++peer)
      for (int el = g0; el < g1; ++el) {
        const int64_t n_back = cnt(peer, me * E_loc + el, sl);
        if (n_back)
          TR_TRY(L->tr->send((char*)L->o + rpos(el, sl, peer) * row_bytes, n_back * row_bytes, peer, 1, L->s_comb));
        const int ex = peer * E_loc + el;
        const int64_t n_home = cnt(me, ex, sl);
        if (n_home)
          TR_TRY(L->tr->recv((char*)L->comb + send_pos[(size_t)ex * S + sl] * row_bytes, n_home * row_bytes, peer, 1,
                             L->s_comb));
      }
    TR_TRY(L->tr->group_end(1, L->s_comb));
    prof_mark(L, MOE_STAGE_COMB_A2A, b0, prof_rec(L, L->s_comb));
    return MOE_OK;
  };
  // odd chunks compute on s_comp2, so a chunk's GEMMs fill the SMs the previous
  // chunk's last tile wave leaves idle (ordering comes from the dispatch event;
  // the final combine waits for every chunk through the combine stream)
  const bool two = L->chunk_streams > 1 && plan.num_chunks > 1;
  auto compute = [&](int ch) -> moe_status_t {
    const int sl = ch % S, g0 = plan.group_begin[ch / S], g1 = plan.group_begin[ch / S + 1];
    cudaStream_t cs = (two && (ch & 1)) ? L->s_comp2 : st;
    CUDA_TRY(cudaStreamWaitEvent(cs, L->ev_disp[ch], 0));  // (p2p: my puts read `send`)
    if (p2p) {  // every source's rows
      TR_TRY(L->tr->p2p_before_wait(ch, 1, cs));
      KERNEL_TRY(launch_p2p_wait(L->p2p_flags + (size_t)ch * D, D, epoch, cs));
    }
    if (L->comm_only) {  // measurement: the chunk's all2all without its ComputeMoE
      CUDA_TRY(cudaEventRecord(L->ev_gemm[ch], cs));
      return MOE_OK;
    }
    const int64_t u0 = urecv[(size_t)ch * D], u1 = urecv[(size_t)(ch + 1) * D];
    if (lr_ep) {  // unique rows -> expert-major GEMM rows (R6 order, so the GEMMs are unchanged)
      KERNEL_TRY(launch_lr_expand(L->recvu, fp8 ? L->recvq : nullptr, L->qpitch, u0, u1, H, k, D, ch, L->lr_usrc_d,
                                  L->lr_recv_off_d, L->meta_recv, L->recv, cs));
    } else if (fp8) {  // the chunk's rows: one range per expert, merged where contiguous (all, if S == 1)
      int el = g0;
      while (el < g1) {
        const int64_t r0 = rpos(el, sl, 0);
        int64_t r1 = rpos(el, sl, D - 1) + cnt(D - 1, me * E_loc + el, sl);
        while (++el < g1 && rpos(el, sl, 0) == r1) r1 = rpos(el, sl, D - 1) + cnt(D - 1, me * E_loc + el, sl);
        KERNEL_TRY(launch_dequant_rows(drecv + r0 * drow, r1 - r0, H, L->qpitch, (char*)L->recv + r0 * row_bytes,
                                       cs));
      }
    }
    int a = g0;
    while (a < g1) {
      int b = a + 1;
      while (b < g1 && plan.expert_kind[b] == plan.expert_kind[a]) ++b;
      double rows = 0;
      for (int el = a; el < b; ++el) rows += tcount[ch * E_loc + el];
      const bool fz = p2p && fuse_comb[ch];
      const size_t cslot = (size_t)MOE_MAX_CHUNKS + ch;
      int err = compute_moe(
          L, L->recv, L->recv_cap, L->recv_start_d + ch * E_loc, L->recv_count_d + ch * E_loc, a, b,
          plan.expert_kind[a], num_ctas, pick_cta_pair(plan, rows / (b - a)), plan.tile_m != 0, rows / (b - a), cs,
          nullptr,
          fz ? reinterpret_cast<const GemmRowSeg*>(L->p2p_tab + P2P_SEGS_BYTES + P2P_PRE_BYTES + p2p_fptr_bytes(D)) +
                   (size_t)ch * moe_layer::P2P_MAXS
             : nullptr,
          fz ? fuse_nrseg[ch] : 0,
          fz ? reinterpret_cast<uint32_t**>(L->p2p_tab + P2P_SEGS_BYTES + P2P_PRE_BYTES) + cslot * D : nullptr,
          fz ? D : 0, epoch);
      if (err) { set_error(std::string("ComputeMoE: ") + cudaGetErrorString((cudaError_t)err)); return MOE_ERR_CUDA; }
      a = b;
    }
    // LocalReduce: the chunk's partial per unique row, in place of its x row
    if (lr_ep) KERNEL_TRY(launch_lr_reduce(L->o, L->meta_recv, u0, u1, H, k, L->recvu, cs));
    if (p2p && fuse_comb[ch]) TR_TRY(L->tr->p2p_after_put(MOE_MAX_CHUNKS + ch, cs));  // combine rows are out
    CUDA_TRY(cudaEventRecord(L->ev_gemm[ch], cs));
    return MOE_OK;
  };
  // Algorithm 1 issue order
  const int PN = plan.num_chunks;
  moe_status_t s_ = dispatch(0);
  if (s_) return s_;
  for (int p = 1; p <= PN; ++p) {
    if (p <= PN - 1 && (s_ = dispatch(p))) return s_;
    if ((s_ = compute(p - 1))) return s_;
    if (p - 2 >= 0 && (s_ = combine_send(p - 2))) return s_;
  }
  if ((s_ = combine_send(PN - 1))) return s_;
  CUDA_TRY(cudaEventRecord(L->ev_comb_done, L->s_comb));
  CUDA_TRY(cudaStreamWaitEvent(st, L->ev_comb_done, 0));
  if (side) CUDA_TRY(cudaStreamWaitEvent(st, L->ev_shared, 0));
  if (p2p) {  // every chunk's combine rows from every expert rank
    TR_TRY(L->tr->p2p_before_wait(MOE_MAX_CHUNKS, plan.num_chunks, st));
    KERNEL_TRY(launch_p2p_wait(L->p2p_flags + (size_t)MOE_MAX_CHUNKS * D, plan.num_chunks * D, epoch, st));
  }
  int c0 = prof_rec(L, st);
  if (lr_ep)
    KERNEL_TRY(launch_lr_combine(L->comb, L->SF ? L->s : nullptr, (int)T, H, k, L->posg, y, st));
  else
    KERNEL_TRY(launch_combine(L->comb, L->SF ? L->s : nullptr, (int)T, H, k, L->pos, topk_w, y, st));
  prof_mark(L, MOE_STAGE_COMBINE, c0, prof_rec(L, st));
  if (dbg && dbg->chunk_rows_host) {
    for (int ch = 0; ch < plan.num_chunks; ++ch) {
      const int sl = ch % S, g0 = plan.group_begin[ch / S], g1 = plan.group_begin[ch / S + 1];
      for (int peer = 0; peer < D; ++peer) {
        int64_t sent = 0, got = 0;
        if (lr_ep) {
          sent = ug[(size_t)me * G + ch * D + peer];
          got = ug[(size_t)peer * G + ch * D + me];
        } else {
          for (int el = g0; el < g1; ++el) {
            sent += cnt(me, peer * E_loc + el, sl);
            got += cnt(peer, me * E_loc + el, sl);
          }
        }
        dbg->chunk_rows_host[(size_t)ch * D + peer] = sent;
        dbg->chunk_rows_host[((size_t)MOE_MAX_CHUNKS + ch) * D + peer] = got;
      }
    }
  }
  if (dbg && lr_ep) {
    if (dbg->lr_pos) CUDA_TRY(cudaMemcpyAsync(dbg->lr_pos, L->posg, sizeof(int32_t) * T * k, cudaMemcpyDeviceToDevice, st));
    if (dbg->lr_hist) CUDA_TRY(cudaMemcpyAsync(dbg->lr_hist, L->u_hist, sizeof(int32_t) * G, cudaMemcpyDeviceToDevice, st));
  }
  return MOE_OK;
}

// Debug outputs (moe_debug_t).
moe_status_t fwd_debug(Fwd& F) {
  moe_layer* L = F.L;
  const moe_config_t& c = L->cfg;
  const void* x = F.x;
  const int64_t T = F.T;
  void* y = F.y;
  cudaStream_t st = F.st;
  moe_debug_t* dbg = F.dbg;
  moe_plan_t& plan = F.plan;
  const moe_plan_t* plan_in = F.plan_in;
  const int E = c.num_experts, k = c.top_k, H = c.hidden, D = c.ep, E_loc = L->E_loc;
  const int num_ctas = F.num_ctas;
  int32_t* topk_idx = F.topk_idx;
  float* topk_w = F.topk_w;
  const bool override_routing = F.override_routing;
  (void)x; (void)y; (void)dbg; (void)plan_in; (void)E_loc; (void)override_routing; (void)topk_idx;
  if (dbg) {
    if (dbg->logits && !override_routing)
      CUDA_TRY(cudaMemcpyAsync(dbg->logits, L->logits, sizeof(float) * T * E, cudaMemcpyDeviceToDevice, st));
    if (dbg->topk_idx && !override_routing)
      CUDA_TRY(cudaMemcpyAsync(dbg->topk_idx, L->topk_idx, sizeof(int32_t) * T * k, cudaMemcpyDeviceToDevice, st));
    if (dbg->topk_w && !override_routing)
      CUDA_TRY(cudaMemcpyAsync(dbg->topk_w, L->topk_w, sizeof(float) * T * k, cudaMemcpyDeviceToDevice, st));
    if (dbg->pos) CUDA_TRY(cudaMemcpyAsync(dbg->pos, L->pos, sizeof(int32_t) * T * k, cudaMemcpyDeviceToDevice, st));
    if (dbg->hist) CUDA_TRY(cudaMemcpyAsync(dbg->hist, L->hist, sizeof(int32_t) * E, cudaMemcpyDeviceToDevice, st));
    if (dbg->seg_start)
      CUDA_TRY(cudaMemcpyAsync(dbg->seg_start, L->seg_start, sizeof(int32_t) * (E + 1), cudaMemcpyDeviceToDevice, st));
    if (dbg->shared_out && L->SF)
      CUDA_TRY(cudaMemcpyAsync(dbg->shared_out, L->s, (size_t)T * H * 2, cudaMemcpyDeviceToDevice, st));
    if (dbg->global_hist_host) {
      if (D == 1) {
        CUDA_TRY(cudaMemcpyAsync(dbg->global_hist_host, L->hist, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
      } else {
        std::memcpy(dbg->global_hist_host, L->ghist_host, sizeof(int32_t) * D * E);
      }
    }
    if (dbg->plan_used) {
      *dbg->plan_used = plan;
      dbg->plan_used->sm_gemm = num_ctas;
      if (D > 1) dbg->plan_used->comm_ctas = L->comm_ctas;
    }
  }
  return MOE_OK;
}

}  // namespace

moe_status_t moe_layer_forward(moe_layer_t* L, const void* x, int64_t T, void* y, const moe_plan_t* plan_in,
                               void* stream_v, moe_debug_t* dbg) {
  if (!L || (!x && T > 0) || (!y && T > 0) || T < 0) { set_error("null argument"); return MOE_ERR_INVALID; }
  const moe_config_t& c = L->cfg;
  if (T > c.max_tokens) { set_error("T_loc > max_tokens"); return MOE_ERR_CAPACITY; }
  cudaStream_t st = (cudaStream_t)stream_v;
  const int D = c.ep;
  L->last_launches = 0;
  L->pev_used = 0;
  L->marks.clear();
  const int p_total = prof_rec(L, st);
  const bool override_routing = dbg && dbg->override_routing;
  if (override_routing && (!dbg->topk_idx || !dbg->topk_w)) { set_error("override needs topk_idx/topk_w"); return MOE_ERR_INVALID; }
  int32_t* topk_idx = override_routing ? dbg->topk_idx : L->topk_idx;
  float* topk_w = override_routing ? dbg->topk_w : L->topk_w;

  moe_plan_t plan;
  if (plan_in) {
    plan = *plan_in;
    int pv = plan_normalise(c, &plan);
    if (pv) { set_error("invalid plan"); return (moe_status_t)pv; }
  }
  // GEMM SM budget (A15, Table IV): a persistent GEMM owns every SM
  // it runs on (~220 KB smem), so at ep > 1 it must leave SMs for the two
  // communicators' kernels or the all2all could not overlap it at all.  The
  // copy-engine plane moves rows without SMs (its flag / wait kernels are one
  // warp and co-reside), so there the GEMMs keep every SM.
  const int default_ctas = gemm_sm_budget(L);
  int num_ctas = (plan_in && plan.sm_gemm > 0) ? std::min(plan.sm_gemm, L->num_sms) : default_ctas;

  Fwd F{L, x, T, y, plan_in, st, dbg, plan};
  F.num_ctas = num_ctas;
  F.topk_idx = topk_idx;
  F.topk_w = topk_w;
  F.override_routing = override_routing;
  if (moe_status_t r = fwd_routing(F)) return r;
  if (moe_status_t r = (D == 1) ? fwd_local(F) : fwd_ep(F)) return r;
  prof_mark(L, MOE_STAGE_TOTAL, p_total, prof_rec(L, st));
  return dbg ? fwd_debug(F) : MOE_OK;
}

// Token-slice schedule of moe_layer_forward_host: relative slice sizes chosen
// from a small family by simulating the three-stream pipeline (H2D copy ->
// layer -> D2H copy, each stream in order) with a model of this config:
// PCIe ~50 GB/s each way; layer time per token from its FLOPs at ~1.25 PF/s,
// inflated by the 256-row tile padding of a slice's rows per expert, plus a
// fixed ~0.3 ms per forward.  A function of the config only, so every rank
// (each slice is a collective when ep > 1) derives the same schedule.
std::vector<double> host_slice_schedule(const moe_config_t& c, bool overlapped) {
  // Overlapped calls (async) run the copy streams ahead across calls: a call
  // then costs its busiest stream and slicing only shortens the one-off fill and
  // drain while inflating the GEMMs' tile padding, so one slice (measured: DSv2
  // e2e 23.6 ms per call over 8 calls unsliced vs 24.9-26.8 sliced; Mixtral 8.7
  // vs 9.1-11.1).
  if (overlapped) return {1.0};
  const double T = (double)c.max_tokens, H = c.hidden, F = c.ffn, k = c.top_k, E = c.num_experts;
  const double SF = (double)c.num_shared * c.shared_ffn;
  const double copy_tok = 2.0 * H / 50e9;
  const double flop_tok = 6.0 * H * F * k + 6.0 * H * SF + 2.0 * H * E;
  auto layer_time = [&](double n) {
    const double rows = n * k * c.ep / E;  // rows per local expert (uniform routing)
    const double eff = rows > 0 ? rows / (std::ceil(rows / 256.0) * 256.0) : 1.0;
    return n * flop_tok / 1.25e15 / eff + 3e-4;
  };
  static const std::vector<std::vector<double>> family = {
      {1}, {1, 1}, {1, 1, 1, 1}, {1, 2, 2, 1}, {1, 2, 3, 2}, {1, 3, 3, 1}, {1, 2, 3, 2, 1}, {1, 2, 4, 4, 2, 1},
      {1, 2, 3, 3, 3, 2, 1}, {1, 1, 1, 1, 1, 1, 1, 1}};
  std::vector<double> best = family[0];
  double best_t = 1e30;
  for (const auto& w : family) {
    double wsum = 0;
    for (double v : w) wsum += v;
    double h_end = 0, c_end = 0, d_end = 0;
    for (double v : w) {
      const double n = T * v / wsum;
      h_end += n * copy_tok;
      c_end = std::max(c_end, h_end) + layer_time(n);
      d_end = std::max(d_end, c_end) + n * copy_tok;
    }
    if (d_end < best_t * 0.99) { best_t = d_end; best = w; }  // a larger family member must win by > 1%
  }
  return best;
}

namespace {
// One host-buffer call: token slices of x_host -> staging buffer b (s_h2d) ->
// layer (st) -> y_host (s_d2h), each stream in order, event-chained per slice.
// The staging pair alternates between calls, so a call's copies overlap the
// previous call's compute; buffer b is reused only after the call two back
// consumed (x) and drained (y) it.
moe_status_t host_call(moe_layer* L, const void* x_host, int64_t T, void* y_host, const moe_plan_t* plan,
                       void* stream_v, bool overlapped) {
  if (!L || T < 0 || T > L->cfg.max_tokens) { set_error("bad argument"); return MOE_ERR_INVALID; }
  cudaStream_t st = (cudaStream_t)stream_v;
  const int64_t row = (int64_t)L->cfg.hidden * 2;
  // y_t depends only on x_t: slices of the batch pipeline the
  // copies against the layer.  The schedule is a function of the config only
  // (identical on every rank: each slice's forward is a collective when ep > 1).
  // EPSMOE_HOST_SLICES="w0,w1,..." (<= 8 relative weights) overrides it.
  std::vector<double> wts;
  if (const char* hs = std::getenv("EPSMOE_HOST_SLICES")) {
    for (const char* p = hs; *p && (int)wts.size() < moe_layer::MAX_HOST_SLICES;) {
      char* end = nullptr;
      double v = std::strtod(p, &end);
      if (end == p) break;
      if (v > 0) wts.push_back(v);
      p = (*end == ',') ? end + 1 : end;
    }
  }
  if (wts.empty()) wts = host_slice_schedule(L->cfg, overlapped);
  const int S = (int)wts.size();
  std::vector<int64_t> bound(S + 1, 0);
  double wsum = 0, acc = 0;
  for (double v : wts) wsum += v;
  for (int s = 0; s < S; ++s) {
    acc += wts[s];
    bound[s + 1] = (s + 1 == S) ? T : std::min<int64_t>(T, (int64_t)std::llround(T * acc / wsum));
  }
  const int b = L->hb;
  L->hb ^= 1;
  CUDA_TRY(cudaStreamWaitEvent(L->s_h2d, L->ev_xfree[b], 0));  // x staging b read by the call two back
  CUDA_TRY(cudaStreamWaitEvent(st, L->ev_yfree[b], 0));        // y staging b copied out by the call two back
  for (int s = 0; s < S; ++s) {
    const int64_t t0 = bound[s], n = bound[s + 1] - t0;
    char* xd = (char*)L->x_dev[b] + t0 * row;
    char* yd = (char*)L->y_dev[b] + t0 * row;
    if (n) CUDA_TRY(cudaMemcpyAsync(xd, (const char*)x_host + t0 * row, n * row, cudaMemcpyHostToDevice, L->s_h2d));
    CUDA_TRY(cudaEventRecord(L->ev_in[s], L->s_h2d));
    CUDA_TRY(cudaStreamWaitEvent(st, L->ev_in[s], 0));
    moe_status_t rs = moe_layer_forward(L, xd, n, yd, plan, stream_v, nullptr);
    if (rs) return rs;
    CUDA_TRY(cudaEventRecord(L->ev_out[s], st));
    CUDA_TRY(cudaStreamWaitEvent(L->s_d2h, L->ev_out[s], 0));
    if (n) CUDA_TRY(cudaMemcpyAsync((char*)y_host + t0 * row, yd, n * row, cudaMemcpyDeviceToHost, L->s_d2h));
  }
  CUDA_TRY(cudaEventRecord(L->ev_xfree[b], st));
  CUDA_TRY(cudaEventRecord(L->ev_yfree[b], L->s_d2h));
  if (!overlapped) {
    CUDA_TRY(cudaStreamSynchronize(L->s_d2h));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  return MOE_OK;
}
}  // namespace

moe_status_t moe_layer_forward_host(moe_layer_t* L, const void* x_host, int64_t T, void* y_host,
                                    const moe_plan_t* plan, void* stream_v) {
  return host_call(L, x_host, T, y_host, plan, stream_v, false);
}

moe_status_t moe_layer_forward_host_async(moe_layer_t* L, const void* x_host, int64_t T, void* y_host,
                                          const moe_plan_t* plan, void* stream_v) {
  return host_call(L, x_host, T, y_host, plan, stream_v, true);
}

moe_status_t moe_layer_host_sync(moe_layer_t* L, void* stream_v) {
  if (!L) { set_error("null layer"); return MOE_ERR_INVALID; }
  CUDA_TRY(cudaStreamSynchronize(L->s_d2h));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream_v));
  return MOE_OK;
}

moe_status_t moe_gemm_grouped(int32_t epi, const void* A, int64_t a_rows, const void* B0, const void* B1,
                              int64_t b_rows, int32_t b_group_rows, int32_t kdim, int32_t n, void* out, int64_t ldo,
                              const float* bias, int32_t groups, const int32_t* row_start, const int32_t* row_count,
                              int32_t num_ctas, int32_t tile_m, void* stream) {
  if (epi < 0 || epi > 2 || !A || !B0 || (epi == 0 && !B1) || !out || groups < 1 || !row_start || !row_count) {
    set_error("moe_gemm_grouped: bad argument");
    return MOE_ERR_INVALID;
  }
  GemmArgs a = base_args(epi, num_ctas > 0 ? num_ctas : 148);
  if (tile_m != 128 && tile_m != 256) { set_error("moe_gemm_grouped: tile_m must be 128 or 256"); return MOE_ERR_INVALID; }
  a.cta_pair = tile_m == 256;
  a.A = A;
  a.a_rows = a_rows;
  a.B0 = B0;
  a.B1 = B1;
  a.b_rows = b_rows;
  a.b_group_rows = b_group_rows;
  a.K = kdim;
  a.N = n;
  a.out = out;
  a.ldo = ldo;
  a.bias = bias;
  a.G = groups;
  a.row_start = row_start;
  a.row_count = row_count;
  a.rows_hint = (double)a_rows / groups;  // raster choice (the counts are on the device)
  int e = gemm_launch(a, (cudaStream_t)stream);
  if (e) { set_error(std::string("gemm: ") + cudaGetErrorString((cudaError_t)e)); return MOE_ERR_CUDA; }
  return MOE_OK;
}

moe_status_t moe_layer_calibrate(moe_layer_t* L, void* stream, moe_cost_model_t* out) {
  if (!L) return MOE_ERR_INVALID;
  // Measured GEMM time per expert vs rows, both kinds (X2/X3 analog on B200).
  const moe_config_t& c = L->cfg;
  cudaStream_t st = (cudaStream_t)stream;
  moe_cost_model_t m = L->cost;
  const int G = std::min(L->E_loc, 8);
  const float pts[MOE_COST_POINTS] = {16, 64, 128, 256, 512, 1024, 2048, 3072, 4096, 6144, 8192, 16384};
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  std::vector<int32_t> hs(2 * MOE_MAX_EXPERTS);
  int np = 0;
  for (int i = 0; i < MOE_COST_POINTS; ++i) {
    int64_t rows = (int64_t)pts[i];
    if (rows * G > L->gemm_rows_cap) break;
    for (int g = 0; g < G; ++g) { hs[g] = (int32_t)(g * rows); hs[MOE_MAX_EXPERTS + g] = (int32_t)rows; }
    CUDA_TRY(cudaMemcpy(L->recv_start_d, hs.data(), sizeof(int32_t) * G, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(L->recv_count_d, hs.data() + MOE_MAX_EXPERTS, sizeof(int32_t) * G, cudaMemcpyHostToDevice));
    const void* A = L->recv ? L->recv : L->send;
    int64_t arows = L->recv ? L->recv_cap : L->send_cap;
    for (int kind = 1; kind <= 2; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        CUDA_TRY(cudaEventRecord(e0, st));
        int err = compute_moe(L, A, arows, L->recv_start_d, L->recv_count_d, 0, G, kind, L->num_sms,
                              rows >= 512 ? 1 : 0, false, rows, st);
        if (err) { set_error("calibrate gemm failed"); return MOE_ERR_CUDA; }
        CUDA_TRY(cudaEventRecord(e1, st));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      m.gemm_ms[kind - 1][i] = best / G;
    }
    m.m_points[i] = pts[i];
    np = i + 1;
  }
  m.n_points = np;
  if (c.ep > 1) {
    // All2all cost (dispatch channel): every rank sends `per` bytes to every
    // peer; time vs the bytes crossing one rank gives a2a_fixed_ms + 1/a2a_gbps.
    const int D = c.ep;
    const int64_t cap = std::min<int64_t>(L->send_cap, L->recv_cap) * c.hidden * 2 / D;
    std::vector<double> xs, ys;
    for (int64_t per : {int64_t(1) << 18, int64_t(1) << 21, int64_t(1) << 23, int64_t(1) << 25}) {
      if (per > cap) break;
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        TR_TRY(L->tr->allgather_i32(L->hist, L->ghist, 1, st));  // ranks start together
        CUDA_TRY(cudaStreamSynchronize(st));
        CUDA_TRY(cudaEventRecord(e0, L->s_disp));
        TR_TRY(L->tr->group_start(0));
        for (int peer = 0; peer < D; ++peer) {
          TR_TRY(L->tr->send((char*)L->send + peer * per, per, peer, 0, L->s_disp));
          TR_TRY(L->tr->recv((char*)L->recv + peer * per, per, peer, 0, L->s_disp));
        }
        TR_TRY(L->tr->group_end(0, L->s_disp));
        CUDA_TRY(cudaEventRecord(e1, L->s_disp));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      xs.push_back((double)per * (D - 1));
      ys.push_back(best);
    }
    if (xs.size() >= 2) {  // least squares: ms = a + x / (gbps * 1e6)
      double sx = 0, sy = 0, sxx = 0, sxy = 0;
      const double n = (double)xs.size();
      for (size_t i = 0; i < xs.size(); ++i) {
        sx += xs[i]; sy += ys[i]; sxx += xs[i] * xs[i]; sxy += xs[i] * ys[i];
      }
      const double slope = (n * sxy - sx * sy) / std::max(1e-30, n * sxx - sx * sx);
      const double icpt = (sy - slope * sx) / n;
      if (slope > 0) m.a2a_gbps = (float)(1.0 / (slope * 1e6));
      m.a2a_fixed_ms = (float)std::max(0.002, icpt);
      m.k_ms = 2.0f * m.a2a_fixed_ms;  // a chunk adds one dispatch and one combine group
    }
    // every rank must plan identically: adopt rank 0's model
    constexpr int W = (int)(sizeof(moe_cost_model_t) / sizeof(int32_t));
    int32_t* dev = nullptr;
    CUDA_TRY(cudaMalloc(&dev, sizeof(int32_t) * W * (D + 1)));
    CUDA_TRY(cudaMemcpy(dev, &m, sizeof(m), cudaMemcpyHostToDevice));
    int ge = L->tr->allgather_i32(dev, dev + W, W, st);
    if (!ge) {
      CUDA_TRY(cudaStreamSynchronize(st));
      CUDA_TRY(cudaMemcpy(&m, dev + W, sizeof(m), cudaMemcpyDeviceToHost));  // rank 0's record
    }
    cudaFree(dev);
    if (ge) return (moe_status_t)ge;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  L->cost = m;
  if (out) *out = m;
  return MOE_OK;
}

}  // extern "C"
