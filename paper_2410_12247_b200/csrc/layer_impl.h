// Internal state of one MoE layer handle and the helpers its translation units
// share (layer.cu: lifecycle, routing, EP = 1 path; layer_ep.cu: the EP > 1
// pipeline of Algorithm 1; layer_host.cu: host-buffer calls; calibrate.cu: the
// measured cost model).
#pragma once
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
  void* staging = nullptr;               // their one cudaMalloc (first host-buffer call), freed by destroy
  int hb = 0;                            // staging buffer of the next host call
  bool host_inflight = false;            // an async host call is queued (cleared by moe_layer_host_sync)
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
  bool overlap_shared = true;     // shared experts on s_side, concurrent with routing (EPSMOE_OVERLAP_SHARED=0: in order)
  bool decode_side = true;        // ep == 1, T < 8192: shared experts concurrent with the router too (EPSMOE_DECODE_SIDE)
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
  int32_t* probe = nullptr;  // this forward's moe_debug_t.gemm_resident (or nullptr)
  // per-stage device timing (moe_layer_set_profiling)
  bool prof = false;
  std::vector<cudaEvent_t> pev;
  int pev_used = 0;
  struct Mark { int stage, e0, e1; };
  std::vector<Mark> marks;
};

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
#define CUDA_TRY_STATUS(expr)                                                             \
  do {                                                                                    \
    moe_status_t _s = (expr);                                                             \
    if (_s != MOE_OK) return _s;                                                          \
  } while (0)
#define NCCL_TRY(expr)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess) {                                                              \
      set_error(std::string(#expr) + ": " + ncclGetErrorString(_r));                      \
      return MOE_ERR_NCCL;                                                                \
    }                                                                                     \
  } while (0)

namespace epsmoe {

// a2a_p2p segment tables (host mirror == device layout): segs | pre | flag pointers | fused-combine rows
constexpr size_t P2P_SEGS_BYTES = sizeof(P2PSeg) * 2 * MOE_MAX_CHUNKS * moe_layer::P2P_MAXS;
constexpr size_t P2P_PRE_BYTES = sizeof(int64_t) * 2 * MOE_MAX_CHUNKS * (moe_layer::P2P_MAXS + 1);
constexpr size_t P2P_RSEG_BYTES = sizeof(GemmRowSeg) * MOE_MAX_CHUNKS * moe_layer::P2P_MAXS;
inline size_t p2p_fptr_bytes(int ep) { return sizeof(uint32_t*) * 2 * MOE_MAX_CHUNKS * ep; }
inline size_t p2p_table_bytes(int ep) { return P2P_SEGS_BYTES + P2P_PRE_BYTES + p2p_fptr_bytes(ep) + P2P_RSEG_BYTES; }

// Per-stage profiling events (no-op unless moe_layer_set_profiling is on).
int prof_rec(moe_layer* L, cudaStream_t st);
void prof_mark(moe_layer* L, int stage, int e0, int e1);
// GemmArgs of a dense single-group launch of kind `epi` (layer_args: with the
// forward's SM-partition probe, moe_debug_t.gemm_resident).
GemmArgs base_args(int epi, int num_ctas);
GemmArgs layer_args(moe_layer* L, int epi, int num_ctas);
// All2all layout (R6) of rank c.rank from the global histogram gh [ep, E].
void exchange_layout(const moe_config_t& c, const int32_t* gh, int64_t* send_off, int64_t* recv_off);
// Tile rows for a chunk's expert GEMMs (1: 256-row CTA pairs, 0: 128-row tiles).
int pick_cta_pair(const moe_plan_t& plan, double mean_rows);
// ComputeMoE of local experts [g0, g1): GateUpGemm + SiluAct, DownGemm.
int compute_moe(moe_layer* L, const void* A, int64_t a_rows, const int32_t* row_start, const int32_t* row_count,
                int g0, int g1, int kind, int num_ctas, int cta_pair, bool tile_forced, double rows_per_group,
                cudaStream_t st, const int32_t* a_row_index = nullptr, const GemmRowSeg* down_rseg = nullptr,
                int down_nrseg = 0, uint32_t* const* down_sig = nullptr, int down_nsig = 0, uint32_t down_epoch = 0);
// Persistent GEMM grid of a forward when the plan does not fix it (the SM partition, NEXT-1).
int pre_plan_sm_budget(const moe_layer* L);

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

// Router (K1) + topKGating (K2) + histogram + split (K3), shared experts alongside.
moe_status_t fwd_routing(Fwd& F);
// EP = 1: ComputeMoE over the plan's chunks, then the weighted unpermute.
moe_status_t fwd_local(Fwd& F);
// EP > 1: count exchange, plan, layouts, Algorithm 1's chunked dispatch / ComputeMoE / combine.
moe_status_t fwd_ep(Fwd& F);
// Debug outputs (moe_debug_t).
moe_status_t fwd_debug(Fwd& F);
// a2a_p2p: map every rank's workspace once (collective).
moe_status_t p2p_map_peers(moe_layer* L, cudaStream_t st);
// Calibration: one all2all of `per` bytes per peer on the layer's data plane
// with comm budget `ctas`; *ms = this rank's completion time.  Collective.
moe_status_t time_all2all(moe_layer* L, int ctas, int64_t per, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1,
                          float* ms);

}  // namespace epsmoe
