// The MoE layer: create / forward / destroy, workspace carve-up, the stream &
// event DAG of Algorithm 1 and the NCCL all2all over NVLink.
//
// Streams (ep > 1): the caller's stream carries routing, permute, shared
// experts and the expert GEMMs (ComputeMoE); s_disp carries the dispatch
// All2All of every chunk on communicator A; s_comb the combine All2All on
// communicator B.  Per chunk c:  D_c (dispatch done) -> GEMMs -> G_c -> combine.
// Issue order = Algorithm 1: dispatch(0); for p: dispatch(p), compute(p-1),
// combine(p-2); combine(PN-1).
#include "layer_impl.h"

namespace epsmoe {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

}  // namespace epsmoe

using namespace epsmoe;

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
  // (the host-buffer calls' staging is allocated on their first use, outside
  // the workspace: device-pointer callers never pay for it)
  return cv.off + ALIGN;
}

}  // namespace

namespace epsmoe {

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

GemmArgs layer_args(moe_layer* L, int epi, int num_ctas) {
  GemmArgs a = base_args(epi, num_ctas);
  a.resident = L->probe;
  return a;
}

// ComputeMoE for local experts [g0, g1): GateUpGemm+SiluAct fused,
// then DownGemm.  Rows of expert g are [row_start[g], +row_count[g]) of A.
int compute_moe(moe_layer* L, const void* A, int64_t a_rows, const int32_t* row_start, const int32_t* row_count,
                int g0, int g1, int kind, int num_ctas, int cta_pair, bool tile_forced, double rows_per_group,
                cudaStream_t st, const int32_t* a_row_index, const GemmRowSeg* down_rseg, int down_nrseg,
                uint32_t* const* down_sig, int down_nsig, uint32_t down_epoch) {
  const moe_config_t& c = L->cfg;
  GemmArgs g1a = layer_args(L, EPI_SWIGLU, num_ctas);
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
  GemmArgs g2a = layer_args(L, EPI_BF16, num_ctas);
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
  // DENSE: one launch per expert.  A fused-combine chunk's completion flags may
  // only rise after its LAST expert's rows are out, so only the last launch
  // carries them (every launch fences its peer stores system-wide before it
  // ends, and the launches are stream-ordered).
  for (int e = g0; e < g1; ++e) {
    g2a.nsig = (e == g1 - 1) ? down_nsig : 0;
    g2a.sig_flags = (e == g1 - 1) ? down_sig : nullptr;
    int e2 = run(e, e + 1);
    if (e2) return e2;
  }
  return 0;
}

// Grid of the GEMMs issued before the plan exists (router, shared experts) at
// ep > 1 on the SM-reserving planes: the smallest grid any comm budget of the
// installed cost model can give, so that they never hold more SMs than the
// plan later leaves to the GEMMs (the shared experts run beside dispatch(0)).
int pre_plan_sm_budget(const moe_layer* L) {
  if (L->cfg.ep == 1 || L->cfg.a2a_p2p == 2) return L->num_sms;
  int cc = L->comm_ctas;
  const int n = std::min(L->cost.n_comm, (int)MOE_COMM_POINTS);
  for (int i = 0; i < n; ++i) cc = std::max(cc, (int)L->cost.comm_ctas[i]);
  return std::max(2, L->num_sms - 2 * cc);
}

}  // namespace epsmoe

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

// How an ep > 1 layer reaches its peers: two NCCL ids, the in-process test
// group, or the caller's host allgather.
struct TransportSpec {
  const void* uid_d = nullptr;
  const void* uid_c = nullptr;
  epsmoe::LocalGroup* group = nullptr;
  moe_host_allgather_fn gather = nullptr;
  void* gather_ctx = nullptr;
};

static moe_status_t create_impl(const moe_config_t* cfg, const moe_weights_t* w, const TransportSpec& ts,
                                void* workspace, size_t workspace_bytes, moe_layer_t** out) {
  const void* uid_d = ts.uid_d;
  const void* uid_c = ts.uid_c;
  epsmoe::LocalGroup* group = ts.group;
  if (!out || !w) { set_error("null argument"); return MOE_ERR_INVALID; }
  *out = nullptr;
  int v = validate(cfg);
  if (v) return (moe_status_t)v;
  if (!w->w_router || !w->w_gate || !w->w_up || !w->w_down) { set_error("missing weights"); return MOE_ERR_INVALID; }
  if (cfg->num_shared > 0 && (!w->ws_gate || !w->ws_up || !w->ws_down)) {
    set_error("missing shared-expert weights");
    return MOE_ERR_INVALID;
  }
  if (cfg->ep > 1 && !group && !ts.gather && (!uid_d || !uid_c)) {
    set_error("ep > 1 needs two NCCL unique ids");
    return MOE_ERR_INVALID;
  }
  if (ts.gather && cfg->ep > 1 && cfg->a2a_p2p == 0) {
    set_error("the host-collective transport moves rows only on a2a_p2p = 1 or 2");
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
  if (const char* ds = std::getenv("EPSMOE_DECODE_SIDE")) L->decode_side = std::atoi(ds) != 0;
  if (const char* fc = std::getenv("EPSMOE_FUSE_COMBINE")) L->fuse_combine = std::atoi(fc);
  if (const char* gv = std::getenv("EPSMOE_GATHER")) L->gather_a = std::atoi(gv) != 0;
  if (const char* pf = std::getenv("EPSMOE_P2P_FUSE")) L->p2p_fuse = std::atoi(pf) != 0;
  if (const char* sv = std::getenv("EPSMOE_SPLIT_REM")) L->split_rem = std::atoi(sv) != 0;
  if (cfg->ep > 1) L->comm_ctas = default_comm_ctas();
  L->cost.num_sms = L->num_sms;
  L->cost.gemm_scale_at[0] = (float)L->num_sms / (float)std::max(1, L->num_sms - 2 * L->cost.comm_ctas[0]);
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
      if (ts.gather) {
        L->tr = new epsmoe::HostCollTransport(ts.gather, ts.gather_ctx, cfg->ep, cfg->rank);
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
      L->tr = new epsmoe::NcclTransport(cd, cc, L->comm_ctas);
      if (r1 != ncclSuccess || r2 != ncclSuccess) {
        set_error(std::string("ncclCommInitRankConfig: ") + ncclGetErrorString(r1 != ncclSuccess ? r1 : r2));
        return fail(MOE_ERR_NCCL);
      }
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
  TransportSpec ts;
  ts.uid_d = uid_d;
  ts.uid_c = uid_c;
  return create_impl(cfg, w, ts, workspace, workspace_bytes, out);
}

moe_status_t moe_layer_create_hostcoll(const moe_config_t* cfg, const moe_weights_t* w,
                                       moe_host_allgather_fn allgather, void* ctx, void* workspace,
                                       size_t workspace_bytes, moe_layer_t** out) {
  if (!allgather) { set_error("null allgather"); return MOE_ERR_INVALID; }
  TransportSpec ts;
  ts.gather = allgather;
  ts.gather_ctx = ctx;
  return create_impl(cfg, w, ts, workspace, workspace_bytes, out);
}

moe_status_t moe_layer_create_local(const moe_config_t* cfg, const moe_weights_t* w, void* group, void* workspace,
                                    size_t workspace_bytes, moe_layer_t** out) {
  if (!group) { set_error("null group"); return MOE_ERR_INVALID; }
  TransportSpec ts;
  ts.group = static_cast<epsmoe::LocalGroup*>(group);
  return create_impl(cfg, w, ts, workspace, workspace_bytes, out);
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
  if (L->staging) cudaFree(L->staging);
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

moe_status_t moe_plan_pipeline(const moe_layer_t* L, int64_t global_tokens, const int32_t* global_hist,
                               moe_plan_t* out) {
  if (!L || !out) return MOE_ERR_INVALID;
  // (at ep > 1 the plan carries the SM partition the cost model picked, NEXT-1)
  return (moe_status_t)plan_compute(L->cfg, L->cost, global_tokens, global_hist, out);
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

}  // extern "C"

namespace epsmoe {

// Router (K1) + topKGating (K2) + histogram + split (K3), with the shared
// experts launched alongside.
moe_status_t fwd_routing(Fwd& F) {
  moe_layer* L = F.L;
  const moe_config_t& c = L->cfg;
  const void* x = F.x;
  const int64_t T = F.T;
  cudaStream_t st = F.st;
  moe_debug_t* dbg = F.dbg;
  const int E = c.num_experts, k = c.top_k, H = c.hidden, D = c.ep;
  const int num_ctas = F.num_ctas;
  int32_t* topk_idx = F.topk_idx;
  float* topk_w = F.topk_w;
  const bool override_routing = F.override_routing;
  // ---- Router (K1) + topKGating (K2) + histogram
  auto router = [&]() -> int {
    if (T == 0 || override_routing) return 0;
    GemmArgs ra = layer_args(L, EPI_F32, num_ctas);
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
    return gemm_launch(ra, st);
  };

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
    GemmArgs a = layer_args(L, EPI_SWIGLU, num_ctas);
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
    GemmArgs b = layer_args(L, EPI_BF16, num_ctas);
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
  // Small ep == 1 batches (decode): the router and shared GEMMs each fill only a
  // few SMs (their grids stop at the tile count) and both need only x, so the
  // shared experts start with the router instead of after it and the whole
  // latency-bound routing chain runs beside them.
  const bool side_early = has_shared && D == 1 && L->overlap_shared && T < 8192 && !fuse && L->decode_side;
  if (side_early) {
    CUDA_TRY(cudaEventRecord(L->ev_router, st));
    CUDA_TRY(cudaStreamWaitEvent(L->s_side, L->ev_router, 0));
    int e = shared_experts(L->s_side);
    if (e) { set_error(std::string("shared experts: ") + cudaGetErrorString((cudaError_t)e)); return MOE_ERR_CUDA; }
    CUDA_TRY(cudaEventRecord(L->ev_shared, L->s_side));
  }
  int p0 = prof_rec(L, st);
  if (T > 0 && !override_routing) KERNEL_TRY(router());
  int p1 = prof_rec(L, st);
  prof_mark(L, MOE_STAGE_ROUTER, p0, p1);
  // (at larger batches the persistent router grid covers every SM: the shared
  // experts follow it on s_side, concurrent with topKGating / split)
  const bool side = has_shared && (side_early || D > 1 || (L->overlap_shared && T >= 8192));
  if (side && !side_early) {
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
  moe_plan_t& plan = F.plan;
  const int E = c.num_experts, k = c.top_k, H = c.hidden;
  const int num_ctas = F.num_ctas;
  int32_t* topk_idx = F.topk_idx;
  float* topk_w = F.topk_w;
  const bool side = F.side, gather = F.gather;
  const int fuse = F.fuse;
  // ---- EP = 1: no all2all; every chunk is local (C = 0 => PN = 1 is optimal)
  if (!F.plan_in) plan_compute(c, L->cost, T, nullptr, &plan);
  if (side) CUDA_TRY(cudaStreamWaitEvent(st, L->ev_shared, 0));
  // (a GEMM grid below the SM count is a partition to keep: one grid at a time)
  const bool two = L->chunk_streams > 1 && plan.num_chunks > 1 && T > 0 && num_ctas >= L->num_sms;
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
      GemmArgs b = layer_args(L, EPI_BF16, num_ctas);
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
    GemmArgs b = layer_args(L, EPI_COMBINE, num_ctas);
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

// Debug outputs (moe_debug_t).
moe_status_t fwd_debug(Fwd& F) {
  moe_layer* L = F.L;
  const moe_config_t& c = L->cfg;
  const int64_t T = F.T;
  cudaStream_t st = F.st;
  moe_debug_t* dbg = F.dbg;
  const int E = c.num_experts, k = c.top_k, H = c.hidden, D = c.ep;
  const bool own_routing = !F.override_routing;
  if (dbg->logits && own_routing)
    CUDA_TRY(cudaMemcpyAsync(dbg->logits, L->logits, sizeof(float) * T * E, cudaMemcpyDeviceToDevice, st));
  if (dbg->topk_idx && own_routing)
    CUDA_TRY(cudaMemcpyAsync(dbg->topk_idx, L->topk_idx, sizeof(int32_t) * T * k, cudaMemcpyDeviceToDevice, st));
  if (dbg->topk_w && own_routing)
    CUDA_TRY(cudaMemcpyAsync(dbg->topk_w, L->topk_w, sizeof(float) * T * k, cudaMemcpyDeviceToDevice, st));
  if (dbg->pos) CUDA_TRY(cudaMemcpyAsync(dbg->pos, L->pos, sizeof(int32_t) * T * k, cudaMemcpyDeviceToDevice, st));
  if (dbg->hist) CUDA_TRY(cudaMemcpyAsync(dbg->hist, L->hist, sizeof(int32_t) * E, cudaMemcpyDeviceToDevice, st));
  if (dbg->seg_start)
    CUDA_TRY(cudaMemcpyAsync(dbg->seg_start, L->seg_start, sizeof(int32_t) * (E + 1), cudaMemcpyDeviceToDevice, st));
  if (dbg->shared_out && L->SF)
    CUDA_TRY(cudaMemcpyAsync(dbg->shared_out, L->s, (size_t)T * H * 2, cudaMemcpyDeviceToDevice, st));
  // the weighted unpermute's input rows: o at the send rows (ep == 1: the GEMM
  // output itself; ep > 1: the combine buffer the all2all filled)
  if (dbg->combine_in && !c.local_reduce && T > 0)
    CUDA_TRY(cudaMemcpyAsync(dbg->combine_in, D == 1 ? L->o : L->comb, (size_t)T * k * H * 2,
                             cudaMemcpyDeviceToDevice, st));
  if (dbg->global_hist_host) {
    if (D == 1) {
      CUDA_TRY(cudaMemcpyAsync(dbg->global_hist_host, L->hist, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
    } else {
      std::memcpy(dbg->global_hist_host, L->ghist_host, sizeof(int32_t) * D * E);
    }
  }
  if (dbg->plan_used) {
    *dbg->plan_used = F.plan;
    dbg->plan_used->sm_gemm = F.num_ctas;
    if (D > 1) dbg->plan_used->comm_ctas = F.plan.comm_ctas > 0 ? F.plan.comm_ctas : L->comm_ctas;
  }
  return MOE_OK;
}

}  // namespace epsmoe

extern "C" {

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

  moe_plan_t plan{};
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
  const int default_ctas = pre_plan_sm_budget(L);
  int num_ctas = (plan_in && plan.sm_gemm > 0) ? std::min(plan.sm_gemm, L->num_sms) : default_ctas;

  Fwd F{L, x, T, y, plan_in, st, dbg, plan};
  F.num_ctas = num_ctas;
  F.topk_idx = topk_idx;
  F.topk_w = topk_w;
  F.override_routing = override_routing;
  L->probe = dbg ? dbg->gemm_resident : nullptr;  // SM-partition probe of this forward's GEMMs
  moe_status_t r = fwd_routing(F);
  if (r == MOE_OK) r = (D == 1) ? fwd_local(F) : fwd_ep(F);
  L->probe = nullptr;
  if (r != MOE_OK) return r;
  prof_mark(L, MOE_STAGE_TOTAL, p_total, prof_rec(L, st));
  return dbg ? fwd_debug(F) : MOE_OK;
}

}  // extern "C"
