// Internal interface of local_reduce.cu: expert-side LocalReduce with
// per-(token, destination, chunk) dedup (NEXT-3, R16).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace epsmoe {

// Words per dedup-row meta record: k slot codes, k weights, padded to 16 B so
// records move as whole vectors.
__host__ __device__ inline int lr_meta_pitch(int k) { return (2 * k + 3) & ~3; }

// The plan's chunks as local-expert groups (R8), passed by value.
struct LrChunks {
  int n;               // PN
  int32_t begin[65];   // group_begin[0..n]
};

// Per-range counts of distinct (token, group g = chunk * D + owner) into
// range_hist[g][range] (G = ch.n * D <= 256); scan with launch_range_scan.
int launch_lr_count(const int32_t* topk_idx, int T, int k, int E_loc, int D, const LrChunks& ch,
                    int32_t* range_hist, cudaStream_t st);
// One send row per distinct (t, g), rows (g asc, t asc) from u_start + range_off;
// posg [T, k]: row of t's i-th group (ascending g), -1 padded; meta [rows, 2k]:
// k slot codes ((local expert << 24) | pos - seg_start[e]) then k weights (pitch lr_meta_pitch(k)).
// sendq != nullptr: packed FP8 rows (R15) instead of bf16 rows into send.
int launch_lr_permute(const void* x, int T, int H, int k, const int32_t* topk_idx, const float* topk_w,
                      const int32_t* pos, const int32_t* seg_start, int E_loc, int D, const LrChunks& ch,
                      const int32_t* range_off, const int32_t* u_start, void* send, void* sendq, int qpitch,
                      int32_t* posg, int32_t* meta, cudaStream_t st);
// Receiver: unique rows [r0, r1) of chunk c -> expert-major GEMM rows of A;
// usrc_start [N*D+1]: first unique row of (chunk, src); recv_off [E_loc*D+1]:
// first GEMM row of (local expert, src).  meta codes become GEMM rows.
int launch_lr_expand(const void* rows, const void* rowsq, int qpitch, int64_t r0, int64_t r1, int H, int k, int D,
                     int c, const int32_t* usrc_start, const int32_t* recv_off, int32_t* meta, void* A,
                     cudaStream_t st);
// LocalReduce: p[u] = bf16(fmaf chain over the row's slots from 0), rows [r0, r1).
int launch_lr_reduce(const void* o, const int32_t* meta, int64_t r0, int64_t r1, int H, int k, void* p,
                     cudaStream_t st);
// Home: y = bf16(fp32(s) + comb[posg[t][0]] + ...), groups ascending.
int launch_lr_combine(const void* comb, const void* s, int T, int H, int k, const int32_t* posg, void* y,
                      cudaStream_t st);
// ep == 1: both sides from o / pos in one pass (groups = chunks of e).
int launch_lr_combine_local(const void* o, const void* s, int T, int H, int k, const int32_t* topk_idx,
                            const int32_t* pos, const float* topk_w, int E, const LrChunks& ch, void* y,
                            cudaStream_t st);

}  // namespace epsmoe
