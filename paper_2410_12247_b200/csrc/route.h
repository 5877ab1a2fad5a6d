// Internal interface of route.cu (HBM-bound kernels of the layer).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace epsmoe {

// Tokens are counted in ranges of range_len(T) consecutive tokens, one warp
// per range, so every row offset is a deterministic prefix sum.  Long batches
// use 32-token ranges; short ones (decode) shorter ranges, so that up to ~2048
// warps share the work instead of T/32.
int range_len(int64_t T);
int num_ranges(int64_t T);
int max_ranges(int64_t T_max);  // over every T <= T_max (workspace sizing)
// route_groups > 1 (and route_topk_groups < route_groups): device-limited routing (R17).
int launch_gate_topk(const float* logits, int T, int E, int k, int norm_topk, float scale, int override_routing,
                     int route_groups, int route_topk_groups, int32_t* topk_idx, float* topk_w,
                     int32_t* range_hist, cudaStream_t st);
// per-range offsets, per-expert totals (hist) and expert segment starts (seg_start[E+1])
int launch_range_scan(const int32_t* range_hist, int T, int E, int32_t* range_off, int32_t* hist,
                      int32_t* seg_start, cudaStream_t st);
// send == nullptr (and fp8 != 2): index-only (pos, row_token).  fp8: 0 bf16 rows, 1 bf16 rows of the FP8
// round trip, 2 packed FP8 rows (pitch qpitch = H + H/128 rounded up to 16) into sendq.
int launch_permute(const void* x, int T, int H, int E, int k, const int32_t* topk_idx, const int32_t* range_off,
                   const int32_t* seg_start, void* send, int32_t* pos, int32_t* row_token, int fp8, void* sendq,
                   int qpitch, cudaStream_t st);
// packed FP8 rows -> bf16 rows (exact), rows [0, rows)
int launch_dequant_rows(const void* q, int64_t rows, int H, int qpitch, void* out, cudaStream_t st);
inline int fp8_row_pitch(int H) { return ((H + H / 128) + 15) & ~15; }
int launch_combine(const void* o, const void* s, int T, int H, int k, const int32_t* pos, const float* topk_w,
                   void* y, cudaStream_t st);
// hs[e * S + s] = pairs of expert e among the tokens of slice s (token-sliced chunks, R8)
int launch_slice_hist(const int32_t* topk_idx, int T, int k, int E, int S, int32_t* hs, cudaStream_t st);
int launch_pad_rows(const void* src, int rows, int H, void* dst, int rows_pad, cudaStream_t st);

}  // namespace epsmoe
