/*
 * epsmoe.h — C ABI of the B200 (sm_100a) EPS-MoE layer: the expert-parallel
 * MoE FFN layer in prefill with the paper's expert pipeline scheduler.
 *
 * Paper: "EPS-MoE: Expert Pipeline Scheduler for Cost-Efficient MoE
 * Inference", arXiv 2410.12247.  P:n = line n of its LaTeX.
 *
 * The arguments follow Algorithm 1's problem statement:
 *   m (tokens), k / n (MoE input / output dim = hidden / ffn), ep, topk,
 *   e (experts), PN (pipeline number); plus shared experts.
 * What one call computes (the plain MoE layer):
 *   y_t = FFN_shared(x_t) + sum_{j<topk} w_{t,j} FFN_{e_{t,j}}(x_t),
 *   FFN_e(x) = (silu(x W_gate,e^T) * (x W_up,e^T)) W_down,e^T,
 * with (e_{t,.}, w_{t,.}) = topKGating(Router(x_t)), executed as
 * Algorithm 1: split -> per chunk {All2All dispatch, ComputeMoE,
 * All2All combine} -> weighted LocalReduce on the token's home rank.
 *
 * Conventions
 *  - Every call returns moe_status_t (0 = MOE_OK).  No C++ exception crosses
 *    the ABI.  On error, moe_last_error() returns a thread-local message.
 *  - Device pointers are CUDA device addresses; "host" pointers are plain CPU
 *    memory (pinned for the *_host entry points' best throughput).
 *  - Matrices are row-major bf16 unless stated otherwise, with the reduction
 *    (K) dimension contiguous ("K-major").
 *  - cudaStream_t / ncclUniqueId are passed as void* / 128-byte buffers so the
 *    header needs neither cuda_runtime.h nor nccl.h.
 */
#ifndef EPSMOE_H_
#define EPSMOE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MOE_OK = 0,
  MOE_ERR_INVALID = 1,     /* bad argument / unsupported shape                 */
  MOE_ERR_UNSUPPORTED = 2, /* valid but not implemented on this build          */
  MOE_ERR_CAPACITY = 3,    /* T_loc > max_tokens, or workspace too small       */
  MOE_ERR_CUDA = 4,        /* a CUDA runtime / driver call failed              */
  MOE_ERR_NCCL = 5,        /* an NCCL call failed; the handle must be destroyed */
  MOE_ERR_MISMATCH = 6     /* ranks disagree on the configuration              */
} moe_status_t;

#define MOE_MAX_EXPERTS 256     /* e  <= 256 (router tile width)                 */
#define MOE_MAX_TOPK 8          /* topk <= 8                                     */
#define MOE_MAX_CHUNKS 64       /* PN <= 64                                      */
#define MOE_MAX_HIDDEN 8192     /* k (hidden) <= 8192                            */

typedef struct moe_layer moe_layer_t; /* opaque, library-owned */

/* Layer shape (Algorithm 1 "Data").  Identical on every rank
 * except `rank`.  Constraints: num_experts % ep == 0 (R12), hidden and ffn
 * multiples of 64 (hidden a multiple of 32 bf16 per output chunk), ffn and
 * num_shared*shared_ffn multiples of 128, 1 <= top_k <= min(8, num_experts). */
typedef struct {
  int32_t num_experts;  /* e: routed experts (global) */
  int32_t top_k;        /* topk */
  int32_t hidden;       /* k: MoE input dim = output dim of DownGemm */
  int32_t ffn;          /* n: output dim of Gate/Up GEMMs per expert */
  int32_t num_shared;   /* shared experts, fused into one MLP (R10) */
  int32_t shared_ffn;   /* width of each shared expert                        */
  int32_t ep;           /* ep: expert-parallel degree = ranks */
  int32_t rank;         /* this rank, 0 <= rank < ep                          */
  int64_t max_tokens;   /* capacity: the largest T_loc of ANY rank in any forward
                           (identical on every rank; sizes the workspace: a
                           rank receives up to ep * max_tokens * min(topk,
                           E_loc) rows)                                      */
  int32_t norm_topk;    /* 1: renormalise the top-k weights (Mixtral); 0: raw
                           softmax probabilities (DeepSeek)             (R1)  */
  float routed_scale;   /* multiplies routed weights (1.0)                    */
  int32_t dispatch_fp8; /* 1: routed rows travel as FP8 e4m3 with one power-of-
                           two scale per 128 columns (Table II "FP8", P:312,
                           P:331; NEXT-2, R15); experts see the exact dequant;
                           needs hidden % 128 == 0.  0: bf16 payload.        */
  int32_t local_reduce; /* 1: expert-side LocalReduce (NEXT-3, R16): a
                           token travels once per (destination rank, chunk)
                           and returns as that group's partial sum
                           p = bf16(sum of w_j o_j in slot order); home side
                           y = bf16(s + p_g ... in (chunk, rank) order).
                           0: per-pair transfer, home-side weighted sum (R7). */
  int32_t route_groups; /* device-limited routing (DeepSeek-V2; NEXT-4,
                           R17): experts form route_groups contiguous groups
                           (<= 32, dividing e); only experts of the
                           route_topk_groups groups with the largest best
                           logit may be selected.  0 or 1: off.             */
  int32_t route_topk_groups; /* M, 1 <= M <= route_groups, topk <= M*e/groups */
  int32_t a2a_p2p;      /* ep > 1 all2all data plane.  0: NCCL grouped send/recv
                           (two communicators).  1: the layer's own put
                           kernels store rows straight into the peers'
                           workspaces (cudaIpc-mapped over NVLink; the
                           workspace must be a cudaMalloc allocation) and
                           raise per-(chunk, source) flags there; NCCL only
                           allgathers counts (and, once, the buffer offsets
                           of every rank's workspace).  2: as 1, but the
                           rows move as cudaMemcpyAsync peer copies on the
                           copy engines (no SM moves a row; NEXT-1's
                           zero-CTA transfer) and one thread raises the
                           flags after them.  Other values: MOE_ERR_INVALID. */
} moe_config_t;

/* Caller-owned device weights (bf16, K-major), valid for the layer's life.
 * Routed experts: only this rank's E_loc = e/ep experts, global ids
 * [rank*E_loc, (rank+1)*E_loc) (EP).  Router + shared experts are
 * replicated on every rank (DP). */
typedef struct {
  const void* w_router;     /* [e, k]                                       */
  const void* w_gate;       /* [E_loc, n, k]                                */
  const void* w_up;         /* [E_loc, n, k]                                */
  const void* w_down;       /* [E_loc, k, n]                                */
  const void* ws_gate;      /* [S*F_s, k] or NULL if num_shared == 0        */
  const void* ws_up;        /* [S*F_s, k]                                   */
  const void* ws_down;      /* [k, S*F_s]                                   */
  const float* router_bias; /* [e] fp32 device or NULL: added to the fp32
                               logits (synthetic skew hook)  */
} moe_weights_t;

/* GEMM kind per expert: GroupGemm vs DenseGemm. */
typedef enum {
  MOE_GEMM_AUTO = 0,    /* per-expert choice from the measured cost model (A8) */
  MOE_GEMM_GROUPED = 1, /* one persistent launch over every tile of a chunk    */
  MOE_GEMM_DENSE = 2    /* one persistent launch per expert, experts in turn   */
} moe_gemm_kind_t;

/* Output of the expert pipeline scheduler (Algorithm 1's PN). */
typedef struct {
  int32_t num_chunks;   /* PN = groups * token_slices <= 64 */
  int32_t token_slices; /* S: 1 = paper (chunks are expert groups, R8); S > 1 (ep
                           > 1, not with local_reduce): every expert group is
                           split into S source-token slices (balanced ranges
                           of each rank's tokens), chunk c = (group c / S,
                           slice c % S); the forward then exchanges the
                           (expert, slice) counts once more                    */
  int32_t gemm_kind;    /* moe_gemm_kind_t applied to all experts (AUTO: see below) */
  int32_t sm_gemm;      /* persistent GEMM grid (0 = all SMs); at ep > 1 every
                           persistent GEMM grid of the forward together stays
                           within it (one grid resident at a time when it is
                           below the SM count)              P:492, A15, NEXT-1 */
  int32_t comm_ctas;    /* NCCL maxCTAs per communicator / put-kernel CTAs per
                           direction / 2 (0 = the layer's default) */
  int32_t group_begin[MOE_MAX_CHUNKS + 1]; /* local-expert group bounds (R8),
                                              [0 .. PN / token_slices]        */
  uint8_t expert_kind[MOE_MAX_EXPERTS];    /* resolved kind per local expert      */
  float pred_comm_ms;   /* T_comm before splitting    */
  float pred_comp_ms;   /* T_comp before splitting    */
  float pred_k_ms;      /* R(N) = kN + b: slope    */
  float pred_b_ms;      /*                 intercept                              */
  float pred_gain_ms;   /* G = C - b - (C/N + kN)    */
  int32_t tile_m;       /* expert-GEMM tile rows: 256 (CTA pair, cta_group::2),
                           128 (single CTA), 0 = by load (256 if the chunk's mean
                           rows per expert >= 512)                               */
} moe_plan_t;

/* Measured cost model behind moe_plan_pipeline (calibrated on B200 by
 * moe_layer_calibrate, or supplied by the caller).  GEMM time of one expert
 * with m rows is linear-interpolated in m from `m_points` (all SMs); all2all
 * time is a2a_fixed_ms + wire bytes / GB/s; per-chunk overhead R(N) = k*N + b.
 * The SM partition (Table IV; NEXT-1): candidate
 * comm budgets comm_ctas[i] (CTAs per communicator / put direction), each with
 * its measured all2all rate a2a_gbps_at[i] and the factor gemm_scale_at[i] by
 * which the expert GEMMs slow down on the num_sms - 2 * comm_ctas[i] SMs left
 * to them.  n_comm = 0: one candidate, the layer's default budget, at a2a_gbps
 * with proportional GEMM scaling. */
#define MOE_COST_POINTS 12
#define MOE_COMM_POINTS 4
typedef struct {
  int32_t n_points;
  float m_points[MOE_COST_POINTS];          /* rows per expert, ascending       */
  float gemm_ms[2][MOE_COST_POINTS];        /* [0] GROUPED, [1] DENSE: ms per
                                               expert (GateUp+Down) at m       */
  float a2a_fixed_ms;                       /* latency term of one all2all     */
  float a2a_gbps;                           /* effective per-rank GB/s         */
  float k_ms;                               /* R(N) slope         */
  float b_ms;                               /* R(N) intercept         */
  int32_t num_sms;                          /* SMs of the measured device (0 = 148) */
  int32_t n_comm;                           /* comm-budget candidates (<= 4)   */
  int32_t comm_ctas[MOE_COMM_POINTS];       /* CTAs per communicator           */
  float a2a_gbps_at[MOE_COMM_POINTS];       /* all2all GB/s at that budget     */
  float gemm_scale_at[MOE_COMM_POINTS];     /* GEMM time factor on the SMs left */
} moe_cost_model_t;

/* Debug / test hooks (NULL in benchmarks).  All array pointers are DEVICE
 * pointers sized for T_loc; any may be NULL. */
typedef struct {
  int32_t override_routing; /* 1: topk_idx / topk_w below are INPUTS (explicit
                               routing, e.g. the fig:eps_overview fixture)   */
  float* logits;            /* out [T_loc, e] fp32                            */
  int32_t* topk_idx;        /* out/in [T_loc, topk]                           */
  float* topk_w;            /* out/in [T_loc, topk]                           */
  int32_t* pos;             /* out [T_loc, topk]: send row of pair (t, j)     */
  int32_t* hist;            /* out [e]: this rank's pairs per expert          */
  int32_t* seg_start;       /* out [e+1]: send-layout expert offsets (R6)     */
  void* shared_out;         /* out [T_loc, H] bf16: shared-expert output s
                               (requesting it disables the ep = 1 fused
                               shared-DownGemm + combine kernel)             */
  int32_t* global_hist_host;/* out HOST [ep, e]                               */
  moe_plan_t* plan_used;    /* out HOST: the plan the forward executed        */
  int32_t* lr_pos;          /* out [T_loc, topk] (local_reduce, ep > 1): send
                               row of the token's i-th group (ascending
                               g = chunk*ep + rank), -1 past its group count */
  int32_t* lr_hist;         /* out [PN*ep] (local_reduce, ep > 1): send rows
                               per group g                                   */
  int64_t* chunk_rows_host; /* out HOST [2][64][ep] (ep > 1): rows this rank
                               sends to [0][c] / receives from [1][c] each
                               peer in chunk c < PN (dedup rows under
                               local_reduce)                                 */
  void* combine_in;         /* out [T_loc * topk, H] bf16 (local_reduce = 0):
                               the expert outputs o the weighted unpermute
                               reads, at the send rows (row pos[t][j] holds
                               o_{t,j}), for the stage-wise combine check     */
  int32_t* gemm_resident;   /* out [2] int32 (zeroed by the caller): the
                               persistent GEMM CTAs of this forward count
                               themselves in [0] while resident and record
                               the maximum in [1] (SM-partition probe)       */
} moe_debug_t;

/* ---------------------------------------------------------------- lifecycle */

/* Bytes of device workspace moe_layer_create needs for `cfg` (worst case:
 * every routed row of every rank lands on this rank, so no reallocation is
 * ever needed). */
size_t moe_layer_workspace_bytes(const moe_config_t* cfg);

/* Write a fresh ncclUniqueId (128 bytes) to `out` (host).  Rank 0 calls it
 * twice (dispatch and combine communicators) and broadcasts the bytes. */
moe_status_t moe_get_unique_id(void* out128);

/* Create the layer.  Collective over the `ep` ranks when ep > 1 (builds two
 * NCCL communicators from the two 128-byte ids; NULL allowed when ep == 1).
 * `workspace` (device, >= moe_layer_workspace_bytes) is caller-owned and
 * must outlive the layer.  The layer keeps the weight pointers, not copies
 * (except a zero-padded copy of the router).  Must be called with the target
 * device current.  On success *out is the new handle. */
moe_status_t moe_layer_create(const moe_config_t* cfg, const moe_weights_t* w,
                              const void* nccl_uid_dispatch, const void* nccl_uid_combine,
                              void* workspace, size_t workspace_bytes, moe_layer_t** out);

moe_status_t moe_layer_destroy(moe_layer_t* layer);

/* Create the layer with the caller's blocking HOST allgather in place of
 * NCCL: allgather(ctx, send, recv, bytes) must write rank r's `bytes` bytes at
 * recv + r * bytes on every rank (collective, same call order; 0 = success).
 * It carries the count exchange and the one-time cudaIpc mapping of the
 * workspaces; routed rows move only on the layer's peer-memory planes, so
 * cfg->a2a_p2p must be 1 or 2 (else MOE_ERR_INVALID).  One process per rank
 * (ranks may share a GPU: separate contexts, real mappings and device flags).
 * `workspace` must be a cudaMalloc allocation (or inside one). */
typedef int (*moe_host_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes);
moe_status_t moe_layer_create_hostcoll(const moe_config_t* cfg, const moe_weights_t* w,
                                       moe_host_allgather_fn allgather, void* ctx, void* workspace,
                                       size_t workspace_bytes, moe_layer_t** out);

/* In-process EP group for tests on ONE GPU: the ep ranks are ep layer objects
 * of one process, each driven by its own host thread; the all2all becomes
 * host-rendezvous + device-to-device copies (same forward code as NCCL).
 * moe_layer_create_local replaces moe_layer_create's NCCL ids with `group`. */
moe_status_t moe_local_group_create(int32_t ep, void** group);
moe_status_t moe_local_group_destroy(void* group);
moe_status_t moe_layer_create_local(const moe_config_t* cfg, const moe_weights_t* w, void* group,
                                    void* workspace, size_t workspace_bytes, moe_layer_t** out);

/* ------------------------------------------------------------------ planner */

/* Pure, host-only, deterministic: the expert pipeline scheduler.
 *   N = argmax_{1<=N<=E_loc} min(T_comm, T_comp)(N-1)/N - (kN + b)  (P:408-415,
 *       ties -> smaller N), T_comm / T_comp from the cost model for the
 *       max-loaded rank; T_comm prices the wire bytes: FP8 dispatch rows
 *       (H + H/128, padded to 16 B, R15), bf16 combine rows, and under
 *       local_reduce the expected dedup rows of N chunks (R16);
 *   ep > 1: (sm_gemm, comm_ctas) = the comm-budget candidate minimising the
 *       modelled pipelined layer time T_comp + T_comm - G(N) (NEXT-1; the
 *       copy-engine plane reserves no SMs);
 *   kind_e = argmin over {GROUPED, DENSE} of the modelled expert time (A8);
 *   group_begin = balanced contiguous expert groups (R8).
 * `global_hist` is HOST [ep, e] (pairs per rank and expert) or NULL for
 * uniform routing (mm = m*topk/e, CalcPN P:540-552).  `global_tokens` = m.
 * No GPU needed: usable from CPU-only tests. */
moe_status_t moe_plan_compute(const moe_config_t* cfg, const moe_cost_model_t* cost,
                              int64_t global_tokens, const int32_t* global_hist, moe_plan_t* out);

/* Pure, host-only: the all2all layout one forward uses on rank cfg->rank
 * (R6: send rows expert-major in token order; recv rows ordered by (local
 * expert, source rank, token)).  ghist: HOST [ep, e] pairs per (rank, expert).
 * Outputs (HOST, caller-allocated; chunk_* may be NULL):
 *   send_off  [e + 1]            first send row of expert e on this rank
 *   recv_off  [E_loc * ep + 1]   first recv row of (local expert, source rank)
 *   chunk_send[PN * ep]          rows this rank sends peer p in chunk c
 *   chunk_recv[PN * ep]          rows this rank receives from peer p in chunk c
 * chunk_send on rank r for peer d equals chunk_recv on rank d for peer r. */
moe_status_t moe_exchange_layout(const moe_config_t* cfg, const moe_plan_t* plan, const int32_t* ghist,
                                 int64_t* send_off, int64_t* recv_off, int64_t* chunk_send, int64_t* chunk_recv);

/* moe_plan_compute with the layer's calibrated cost model. */
moe_status_t moe_plan_pipeline(const moe_layer_t* layer, int64_t global_tokens,
                               const int32_t* global_hist, moe_plan_t* out);

/* Measure the B200 cost model (GEMM time vs rows per expert for both kinds;
 * all2all fixed cost and bandwidth from a time-vs-bytes fit when ep > 1, the
 * per-chunk overhead k from the fixed cost) and install it in the layer.
 * Collective when ep > 1: every rank ends with rank 0's model.  Optional; without it a built-in model
 * is used.  `out` (host, may be NULL) receives the model. */
moe_status_t moe_layer_calibrate(moe_layer_t* layer, void* stream, moe_cost_model_t* out);
/* Install a caller's model.  ep > 1: must be the same on every rank (each
 * rank plans from its own copy; calibrate() guarantees it by adopting rank 0's). */
moe_status_t moe_layer_set_cost_model(moe_layer_t* layer, const moe_cost_model_t* cost);

/* ------------------------------------------------------------------ forward */

/* One MoE layer forward (Algorithm 1).  Collective when ep > 1
 * (same call order on every rank; T_loc may differ per rank).
 *   x: DEVICE [T_loc, k] bf16, must stay valid until `stream` reaches the
 *      end of this call; y: DEVICE [T_loc, k] bf16, written stream-ordered.
 *   plan: NULL = moe_plan_pipeline on the realised global histogram.
 *   stream: cudaStream_t (NULL = legacy default stream).
 * ep == 1: no host synchronisation (CUDA-graph capturable when plan != NULL
 * and dbg == NULL).  ep > 1: one device->host wait for the histogram
 * allgather per call (hidden behind the shared-expert GEMMs). */
moe_status_t moe_layer_forward(moe_layer_t* layer, const void* x, int64_t T_loc, void* y,
                               const moe_plan_t* plan, void* stream, moe_debug_t* dbg);

/* moe_layer_forward on HOST buffers: copies x host->device, runs the layer,
 * copies y device->host, all on `stream`, and returns when y_host is ready.
 * x_host / y_host: [T_loc, k] bf16 (pinned memory recommended). */
moe_status_t moe_layer_forward_host(moe_layer_t* layer, const void* x_host, int64_t T_loc, void* y_host,
                                    const moe_plan_t* plan, void* stream);

/* moe_layer_forward_host without the final wait: enqueues the copies and the
 * layer and returns.  Consecutive calls overlap: the layer double-buffers its
 * device staging, so call i+1's host->device copy runs while call i computes
 * and call i's device->host copy drains while call i+1 computes.  x_host and
 * y_host belong to the layer until moe_layer_host_sync returns; y_host is not
 * valid before that.  ep > 1: collective like moe_layer_forward. */
moe_status_t moe_layer_forward_host_async(moe_layer_t* layer, const void* x_host, int64_t T_loc, void* y_host,
                                          const moe_plan_t* plan, void* stream);
/* Wait for every host-buffer call issued so far (`stream` = the calls' stream). */
moe_status_t moe_layer_host_sync(moe_layer_t* layer, void* stream);

/* Per-stage device timing of the last forward (CUDA events recorded on the
 * stream each stage is launched on).  enable = 1 turns recording on. */
enum {
  MOE_STAGE_ROUTER = 0,  /* K1 router GEMM                                  */
  MOE_STAGE_ROUTE = 1,   /* K2 gating + histogram + scan + K3 permute        */
  MOE_STAGE_SHARED = 2,  /* shared-expert GEMMs                              */
  MOE_STAGE_GATEUP = 3,  /* GateUpGemm + SiluAct, summed over launches       */
  MOE_STAGE_DOWN = 4,    /* DownGemm, summed over launches                   */
  MOE_STAGE_COMBINE = 5, /* weighted unpermute (LocalReduce)                 */
  MOE_STAGE_DISPATCH = 6,/* all2all dispatch, summed over chunks (ep > 1)    */
  MOE_STAGE_COMB_A2A = 7,/* all2all combine, summed over chunks (ep > 1)     */
  MOE_STAGE_TOTAL = 8,   /* whole forward on the caller's stream             */
  MOE_STAGE_EXPOSED_A2A = 9, /* all2all time not covered by compute (ep > 1) */
  MOE_NUM_STAGES = 10
};
moe_status_t moe_layer_set_profiling(moe_layer_t* layer, int32_t enable);
/* Measurement hook for the exposed-all2all figure ("the same
 * chunked dispatch/combine with the GEMMs replaced by no-ops"; the paper's
 * overlap claim).  enable != 0: later forwards run routing, the
 * count exchange, the plan, every chunk's dispatch and combine all2all (same
 * plan, streams, events and data plane; the fused DownGemm combine becomes the
 * put kernel) and the weighted unpermute, but skip ComputeMoE (expert GEMMs,
 * SwiGLU, LocalReduce partials, FP8 dequantisation) and the shared experts, so
 * y is UNDEFINED while it is set.  Collective: every rank of the EP group sets
 * the same value between forwards.  Ignored at ep == 1 (no all2all).  Errors:
 * MOE_ERR_INVALID for a NULL layer. */
moe_status_t moe_layer_set_comm_only(moe_layer_t* layer, int32_t enable);

/* Waits for the last forward's events; ms[MOE_NUM_STAGES] (host) in ms;
 * counts[MOE_NUM_STAGES] (host, may be NULL) = launches timed per stage. */
moe_status_t moe_layer_stage_ms(const moe_layer_t* layer, float* ms, int32_t* counts);

/* Number of kernels the last forward launched (for the bench's gpu_launches). */
int32_t moe_layer_last_launches(const moe_layer_t* layer);

/* Thread-local message of the last error ("" if none). */
const char* moe_last_error(void);

/* --------------------------------------------------------- test / calibration */

/* One grouped GEMM of the layer's kernel family on caller buffers (device):
 *   epi 0 (GateUp+Silu): out[r, 0:n] = bf16(silu(A_r B0_g^T) * (A_r B1_g^T))
 *   epi 1 (Down):        out[r, 0:n] = bf16(A_r B0_g^T)
 *   epi 2 (fp32):        out[r, 0:n] = fp32(A_r B0_g^T) (+ bias)
 * for rows r of group g in [row_start[g], row_start[g] + row_count[g]),
 * B*_g = rows [g*b_group_rows, g*b_group_rows + n) (epi 0/1) of B0/B1 [.., kdim].
 * row_start/row_count: DEVICE int32 [groups].  num_ctas: persistent grid.
 * tile_m: 128 (single-CTA tiles) or 256 (CTA-pair tiles, cta_group::2). */
moe_status_t moe_gemm_grouped(int32_t epi, const void* A, int64_t a_rows, const void* B0, const void* B1,
                              int64_t b_rows, int32_t b_group_rows, int32_t kdim, int32_t n, void* out,
                              int64_t ldo, const float* bias, int32_t groups, const int32_t* row_start,
                              const int32_t* row_count, int32_t num_ctas, int32_t tile_m, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EPSMOE_H_ */
