// Expert-side LocalReduce with per-(token, destination, chunk) dedup (NEXT-3,
// R16).  ComputeMoE ends with LocalReduce on the expert side, which
// overlaps the combine all2all (P:295 fig:comp_overlap_comm): a token
// travels once to each (destination rank, chunk) holding any of its experts and
// returns from there as one partial sum.
//
// Group of pair (t, j): g = c * D + d, d = owner rank of e = topk_idx[t][j]
// (e / E_loc), c = chunk of e's local id (balanced contiguous groups, R8).
//
// Sender (rank r):   lr_count -> range scan over g -> lr_permute: one send row
//                    per distinct (t, g), rows ordered (g asc, t asc); per row a
//                    meta record of the group's slots in slot order:
//                    code = (local expert << 24) | index of t among r's rows
//                    for that expert (pos - seg_start), and w.
// Receiver (rank d): lr_expand: each unique row -> the expert-major GEMM rows
//                    (local expert, src, t) (R6) it feeds; code -> that row.
//                    lr_reduce after DownGemm: p = bf16(fmaf chain, slot
//                    order, from 0) per unique row = the combine payload.
// Home (rank r):     lr_combine: y = bf16(fp32(s) + p_g ... in g order).
// ep == 1:           lr_combine_local does both sides in one pass.
//
// Every row index is a deterministic prefix sum (ranges of range_len(T)
// tokens, one warp each), as in route.cu: no atomics decide a row.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lr.h"
#include "route.h"
#include "rowops.cuh"

namespace epsmoe {
namespace {
using namespace rowops;

constexpr int WARPS_R = 4;  // range kernels: small blocks that co-reside with GEMM CTAs
constexpr int MAX_K = 8;
constexpr uint32_t FULL = 0xffffffffu;

__device__ __forceinline__ int chunk_of_local(const LrChunks& ch, int el) {
  int c = 0;
  for (int i = 1; i < ch.n; ++i)
    if (ch.begin[i] <= el) c = i;
  return c;
}

// Per token: this lane's group (lanes < k), whether it is the first lane of
// its group (leader), and the leader mask of the token.
struct TokGroups {
  int g;
  bool lead;
  uint32_t lmask;
};
__device__ __forceinline__ TokGroups token_groups(const int32_t* __restrict__ topk_idx, int64_t t, int k, int lane,
                                                  const int32_t* chunk_s, int E_loc, int D) {
  TokGroups r;
  r.g = 0x7fffffff;
  if (lane < k) {
    const int e = topk_idx[t * k + lane];
    r.g = chunk_s[e % E_loc] * D + e / E_loc;
  }
  r.lead = lane < k;
#pragma unroll
  for (int j = 0; j < MAX_K; ++j) {
    const int gj = __shfl_sync(FULL, r.g, j);
    if (j < k && j < lane && gj == r.g) r.lead = false;
  }
  r.lmask = __ballot_sync(FULL, r.lead);
  return r;
}

__device__ __forceinline__ void load_chunks(const LrChunks& ch, int E_loc, int32_t* chunk_s) {
  for (int el = threadIdx.x; el < E_loc; el += blockDim.x) chunk_s[el] = chunk_of_local(ch, el);
  __syncthreads();
}

__global__ void __launch_bounds__(WARPS_R * 32)
lr_count_kernel(const int32_t* __restrict__ topk_idx, int T, int k, int E_loc, int D, LrChunks ch, int G,
                int32_t* __restrict__ range_hist, int R, int rt) {
  __shared__ int32_t hist_s[WARPS_R][256];
  __shared__ int32_t chunk_s[256];
  load_chunks(ch, E_loc, chunk_s);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * WARPS_R + warp;
  for (int g = lane; g < G; g += 32) hist_s[warp][g] = 0;
  __syncwarp();
  if (r < R) {
    const int t_end = min(T, (r + 1) * rt);
    for (int t = r * rt; t < t_end; ++t) {
      const TokGroups tg = token_groups(topk_idx, t, k, lane, chunk_s, E_loc, D);
      if (tg.lead) atomicAdd(&hist_s[warp][tg.g], 1);  // order-free count
      __syncwarp();
    }
  }
  __syncwarp();
  if (r < R)
    for (int g = lane; g < G; g += 32) range_hist[(int64_t)g * R + r] = hist_s[warp][g];
}

// fp8: 0 = bf16 rows into `send`; 2 = packed FP8 rows (R15) into `sendq`.
template <int fp8>
__global__ void __launch_bounds__(WARPS_R * 32, 4)
lr_permute_kernel(const __nv_bfloat16* __restrict__ x, int T, int H, int k, const int32_t* __restrict__ topk_idx,
                  const float* __restrict__ topk_w, const int32_t* __restrict__ pos,
                  const int32_t* __restrict__ seg_start, int E_loc, int D, LrChunks ch, int G,
                  const int32_t* __restrict__ range_off, const int32_t* __restrict__ u_start, int R, int rt,
                  __nv_bfloat16* __restrict__ send, uint8_t* __restrict__ sendq, int qpitch,
                  int32_t* __restrict__ posg, int32_t* __restrict__ meta) {
  __shared__ int32_t off_s[WARPS_R][256];
  __shared__ int32_t chunk_s[256];
  load_chunks(ch, E_loc, chunk_s);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * WARPS_R + warp;
  if (r >= R) return;
  for (int g = lane; g < G; g += 32) off_s[warp][g] = u_start[g] + range_off[(int64_t)g * R + r];
  __syncwarp();
  const int nvec = H >> 3;
  const int t_end = min(T, (r + 1) * rt);
  const uint64_t pol = evict_first_policy();
  for (int t = r * rt; t < t_end; ++t) {
    const TokGroups tg = token_groups(topk_idx, t, k, lane, chunk_s, E_loc, D);
    int code = -1;
    float w = 0.f;
    if (lane < k) {
      const int e = topk_idx[(int64_t)t * k + lane];
      code = ((e % E_loc) << 24) | (pos[(int64_t)t * k + lane] - seg_start[e]);
      w = topk_w[(int64_t)t * k + lane];
    }
    // rank of this leader's group among the token's groups (ascending g)
    int rank = 0;
#pragma unroll
    for (int j = 0; j < MAX_K; ++j) {
      const int gj = __shfl_sync(FULL, tg.g, j);
      if (((tg.lmask >> j) & 1u) && gj < tg.g) ++rank;
    }
    const int dest = tg.lead ? off_s[warp][tg.g] : 0;
    __syncwarp();
    if (tg.lead) off_s[warp][tg.g] = dest + 1;
    const int nd = __popc(tg.lmask);
    if (lane < k && lane >= nd) posg[(int64_t)t * k + lane] = -1;
    if (tg.lead) posg[(int64_t)t * k + rank] = dest;
    // meta of row dest: the group's (code, w) in slot order, then -1 / 0 padding
    int n = 0;
    int32_t* m = meta + (int64_t)dest * lr_meta_pitch(k);
#pragma unroll
    for (int j = 0; j < MAX_K; ++j) {
      const int gj = __shfl_sync(FULL, tg.g, j);
      const int cj = __shfl_sync(FULL, code, j);
      const float wj = __shfl_sync(FULL, w, j);
      if (tg.lead && j < k && gj == tg.g) {
        m[n] = cj;
        m[k + n] = __float_as_int(wj);
        ++n;
      }
    }
    if (tg.lead)
      for (; n < k; ++n) {
        m[n] = -1;
        m[k + n] = 0;
      }
    // the token's row, read once, to each of its group rows
    int dj[MAX_K];
#pragma unroll
    for (int j = 0; j < MAX_K; ++j) dj[j] = __shfl_sync(FULL, dest, j);
    const uint4* src = reinterpret_cast<const uint4*>(x + (int64_t)t * H);
    constexpr int MAXV = 16;
    for (int base = 0; base < nvec; base += 32 * MAXV) {
      uint4 buf[MAXV];
#pragma unroll
      for (int i = 0; i < MAXV; ++i) {
        const int c = base + lane + 32 * i;
        if (c < nvec) buf[i] = ld_stream(src + c, pol);
      }
      if constexpr (fp8 == 2) {
        int sexp[MAXV];
        uint2 q[MAXV];
#pragma unroll
        for (int i = 0; i < MAXV; ++i) {
          float mx = (base + lane + 32 * i < nvec) ? amax8(buf[i]) : 0.f;
#pragma unroll
          for (int off = 8; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, off));
          sexp[i] = fp8_block_exp(mx);
          if (base + lane + 32 * i < nvec) q[i] = quant8(buf[i], pow2f(-sexp[i]));
        }
#pragma unroll
        for (int j = 0; j < MAX_K; ++j) {
          if (!((tg.lmask >> j) & 1u)) continue;
          uint8_t* row = sendq + (int64_t)dj[j] * qpitch;
#pragma unroll
          for (int i = 0; i < MAXV; ++i) {
            const int c = base + lane + 32 * i;
            if (c < nvec) {
              reinterpret_cast<uint2*>(row)[c] = q[i];
              if ((lane & 15) == 0) row[H + (c >> 4)] = (uint8_t)(int8_t)sexp[i];
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < MAX_K; ++j) {
          if (!((tg.lmask >> j) & 1u)) continue;
          uint4* dst = reinterpret_cast<uint4*>(send + (int64_t)dj[j] * H);
#pragma unroll
          for (int i = 0; i < MAXV; ++i) {
            const int c = base + lane + 32 * i;
            if (c < nvec) st_stream(dst + c, buf[i], pol);
          }
        }
      }
    }
  }
}

// Receiver: unique rows [r0, r1) of chunk c (ordered (src, t)) -> expert-major
// GEMM rows.  fp8: 0 bf16 rows `rows`; 1 packed FP8 rows `rowsq` (exact dequant).
// meta codes are rewritten in place to the GEMM row each slot reads back.
template <int fp8>
__global__ void __launch_bounds__(256)
lr_expand_kernel(const __nv_bfloat16* __restrict__ rows, const uint8_t* __restrict__ rowsq, int qpitch, int64_t r0,
                 int64_t r1, int H, int k, int D, int c, const int32_t* __restrict__ usrc_start,
                 const int32_t* __restrict__ recv_off, int32_t* __restrict__ meta, __nv_bfloat16* __restrict__ A) {
  const int64_t u = r0 + (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= r1) return;
  const int lane = threadIdx.x & 31;
  int src = 0;
  for (int s = 1; s < D; ++s)
    if (usrc_start[c * D + s] <= u) src = s;
  int R = -1;
  if (lane < k) {
    const int code = meta[u * lr_meta_pitch(k) + lane];
    if (code >= 0) R = recv_off[(code >> 24) * D + src] + (code & 0xFFFFFF);
    meta[u * lr_meta_pitch(k) + lane] = R;
  }
  int Rs[MAX_K];
#pragma unroll
  for (int j = 0; j < MAX_K; ++j) Rs[j] = __shfl_sync(FULL, R, j);
  const int nvec = H >> 3;
  const uint64_t pol = evict_first_policy();
  for (int cc = lane; cc < nvec; cc += 32) {
    uint4 v;
    if constexpr (fp8 == 1) {
      const uint8_t* q = rowsq + u * qpitch;
      v = dequant8(reinterpret_cast<const uint2*>(q)[cc], pow2f((int)(int8_t)q[H + (cc >> 4)]));
    } else {
      v = ld_stream(reinterpret_cast<const uint4*>(rows + u * H) + cc, pol);
    }
#pragma unroll
    for (int j = 0; j < MAX_K; ++j)
      if (j < k && Rs[j] >= 0) reinterpret_cast<uint4*>(A + (int64_t)Rs[j] * H)[cc] = v;
  }
}

// LocalReduce: p[u] = bf16(acc), acc = 0; acc = fmaf(w_s, o[R_s], acc)
// over the row's slots in slot order.
__global__ void __launch_bounds__(256)
lr_reduce_kernel(const __nv_bfloat16* __restrict__ o, const int32_t* __restrict__ meta, int64_t r0, int64_t r1,
                 int H, int k, __nv_bfloat16* __restrict__ p) {
  const int64_t u = r0 + (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= r1) return;
  const int lane = threadIdx.x & 31;
  int R = -1;
  float w = 0.f;
  if (lane < k) {
    R = meta[u * lr_meta_pitch(k) + lane];
    w = __int_as_float(meta[u * lr_meta_pitch(k) + k + lane]);
  }
  int Rs[MAX_K];
  float ws[MAX_K];
#pragma unroll
  for (int j = 0; j < MAX_K; ++j) {
    Rs[j] = __shfl_sync(FULL, R, j);
    ws[j] = __shfl_sync(FULL, w, j);
  }
  const int nvec = H >> 3;
  const uint64_t pol = evict_first_policy();
  for (int cc = lane; cc < nvec; cc += 32) {
    uint4 ov[MAX_K];
#pragma unroll
    for (int j = 0; j < MAX_K; ++j)
      if (j < k && Rs[j] >= 0) ov[j] = ld_stream(reinterpret_cast<const uint4*>(o + (int64_t)Rs[j] * H) + cc, pol);
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
#pragma unroll
    for (int j = 0; j < MAX_K; ++j) {
      if (j < k && Rs[j] >= 0) {
        const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(&ov[j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(ws[j], __bfloat162float(ob[i]), acc[i]);
      }
    }
    uint4 out;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
    for (int i = 0; i < 4; ++i) o2[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    st_stream(reinterpret_cast<uint4*>(p + u * H) + cc, out, pol);
  }
}

// Home side: y[t] = bf16(acc), acc = fp32(s[t]) (0 without shared experts);
// acc = acc + comb[posg[t][i]] for the token's groups in ascending g.
__global__ void __launch_bounds__(256)
lr_combine_kernel(const __nv_bfloat16* __restrict__ comb, const __nv_bfloat16* __restrict__ s, int T, int H, int k,
                  const int32_t* __restrict__ posg, __nv_bfloat16* __restrict__ y) {
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const int pr = (lane < k) ? posg[(int64_t)t * k + lane] : -1;
  int ps[MAX_K];
#pragma unroll
  for (int j = 0; j < MAX_K; ++j) ps[j] = __shfl_sync(FULL, pr, j);
  const int nvec = H >> 3;
  const uint64_t pol = evict_first_policy();
  for (int cc = lane; cc < nvec; cc += 32) {
    uint4 pv[MAX_K];
#pragma unroll
    for (int j = 0; j < MAX_K; ++j)
      if (j < k && ps[j] >= 0) pv[j] = ld_stream(reinterpret_cast<const uint4*>(comb + (int64_t)ps[j] * H) + cc, pol);
    float acc[8];
    if (s) {
      const uint4 sv = ld_stream(reinterpret_cast<const uint4*>(s + (int64_t)t * H) + cc, pol);
      const __nv_bfloat16* sb = reinterpret_cast<const __nv_bfloat16*>(&sv);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __bfloat162float(sb[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < MAX_K; ++j) {
      if (j < k && ps[j] >= 0) {
        const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&pv[j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], __bfloat162float(pb[i]));
      }
    }
    uint4 out;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
    for (int i = 0; i < 4; ++i) o2[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    st_stream(reinterpret_cast<uint4*>(y + (int64_t)t * H) + cc, out, pol);
  }
}

// ep == 1 (D = 1, g = chunk): both sides in one pass over o rows (pos).
__global__ void __launch_bounds__(256)
lr_combine_local_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ s, int T, int H, int k,
                        const int32_t* __restrict__ topk_idx, const int32_t* __restrict__ pos,
                        const float* __restrict__ topk_w, int E, LrChunks ch, __nv_bfloat16* __restrict__ y) {
  __shared__ int32_t chunk_s[256];
  load_chunks(ch, E, chunk_s);
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const TokGroups tg = token_groups(topk_idx, t, k, lane, chunk_s, E, 1);
  // group rank of each slot (its group's position in ascending g)
  int grank = 0;
#pragma unroll
  for (int j = 0; j < MAX_K; ++j) {
    const int gj = __shfl_sync(FULL, tg.g, j);
    if (((tg.lmask >> j) & 1u) && gj < tg.g) ++grank;
  }
  const int pr = (lane < k) ? pos[(int64_t)t * k + lane] : 0;
  const float pw = (lane < k) ? topk_w[(int64_t)t * k + lane] : 0.f;
  int rows[MAX_K], gr[MAX_K];
  float ws[MAX_K];
#pragma unroll
  for (int j = 0; j < MAX_K; ++j) {
    rows[j] = __shfl_sync(FULL, pr, j);
    ws[j] = __shfl_sync(FULL, pw, j);
    gr[j] = __shfl_sync(FULL, grank, j);
  }
  const int nd = __popc(tg.lmask);
  const int nvec = H >> 3;
  const uint64_t pol = evict_first_policy();
  for (int cc = lane; cc < nvec; cc += 32) {
    uint4 ov[MAX_K];
#pragma unroll
    for (int j = 0; j < MAX_K; ++j)
      if (j < k) ov[j] = ld_stream(reinterpret_cast<const uint4*>(o + (int64_t)rows[j] * H) + cc, pol);
    float acc[8];
    if (s) {
      const uint4 sv = ld_stream(reinterpret_cast<const uint4*>(s + (int64_t)t * H) + cc, pol);
      const __nv_bfloat16* sb = reinterpret_cast<const __nv_bfloat16*>(&sv);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __bfloat162float(sb[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    }
    for (int gi = 0; gi < nd; ++gi) {
      float part[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) part[i] = 0.f;
#pragma unroll
      for (int j = 0; j < MAX_K; ++j) {
        if (j < k && gr[j] == gi) {
          const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(&ov[j]);
#pragma unroll
          for (int i = 0; i < 8; ++i) part[i] = __fmaf_rn(ws[j], __bfloat162float(ob[i]), part[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __fadd_rn(acc[i], __bfloat162float(__float2bfloat16_rn(part[i])));
    }
    uint4 out;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&out);
#pragma unroll
    for (int i = 0; i < 4; ++i) o2[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    st_stream(reinterpret_cast<uint4*>(y + (int64_t)t * H) + cc, out, pol);
  }
}

}  // namespace

int launch_lr_count(const int32_t* topk_idx, int T, int k, int E_loc, int D, const LrChunks& ch,
                    int32_t* range_hist, cudaStream_t st) {
  const int R = num_ranges(T);
  if (R == 0) return 0;
  lr_count_kernel<<<(R + WARPS_R - 1) / WARPS_R, WARPS_R * 32, 0, st>>>(topk_idx, T, k, E_loc, D, ch, ch.n * D,
                                                                         range_hist, R, range_len(T));
  return (int)cudaGetLastError();
}

int launch_lr_permute(const void* x, int T, int H, int k, const int32_t* topk_idx, const float* topk_w,
                      const int32_t* pos, const int32_t* seg_start, int E_loc, int D, const LrChunks& ch,
                      const int32_t* range_off, const int32_t* u_start, void* send, void* sendq, int qpitch,
                      int32_t* posg, int32_t* meta, cudaStream_t st) {
  const int R = num_ranges(T);
  if (R == 0) return 0;
  const dim3 grid((R + WARPS_R - 1) / WARPS_R), block(WARPS_R * 32);
  const int G = ch.n * D;
  auto xb = (const __nv_bfloat16*)x;
  if (sendq)
    lr_permute_kernel<2><<<grid, block, 0, st>>>(xb, T, H, k, topk_idx, topk_w, pos, seg_start, E_loc, D, ch, G,
                                                 range_off, u_start, R, range_len(T), nullptr, (uint8_t*)sendq, qpitch,
                                                 posg, meta);
  else
    lr_permute_kernel<0><<<grid, block, 0, st>>>(xb, T, H, k, topk_idx, topk_w, pos, seg_start, E_loc, D, ch, G,
                                                 range_off, u_start, R, range_len(T), (__nv_bfloat16*)send, nullptr, qpitch,
                                                 posg, meta);
  return (int)cudaGetLastError();
}

int launch_lr_expand(const void* rows, const void* rowsq, int qpitch, int64_t r0, int64_t r1, int H, int k, int D,
                     int c, const int32_t* usrc_start, const int32_t* recv_off, int32_t* meta, void* A,
                     cudaStream_t st) {
  if (r1 <= r0) return 0;
  const unsigned grid = (unsigned)((r1 - r0 + 7) / 8);
  if (rowsq)
    lr_expand_kernel<1><<<grid, 256, 0, st>>>(nullptr, (const uint8_t*)rowsq, qpitch, r0, r1, H, k, D, c, usrc_start,
                                              recv_off, meta, (__nv_bfloat16*)A);
  else
    lr_expand_kernel<0><<<grid, 256, 0, st>>>((const __nv_bfloat16*)rows, nullptr, qpitch, r0, r1, H, k, D, c,
                                              usrc_start, recv_off, meta, (__nv_bfloat16*)A);
  return (int)cudaGetLastError();
}

int launch_lr_reduce(const void* o, const int32_t* meta, int64_t r0, int64_t r1, int H, int k, void* p,
                     cudaStream_t st) {
  if (r1 <= r0) return 0;
  lr_reduce_kernel<<<(unsigned)((r1 - r0 + 7) / 8), 256, 0, st>>>((const __nv_bfloat16*)o, meta, r0, r1, H, k,
                                                                  (__nv_bfloat16*)p);
  return (int)cudaGetLastError();
}

int launch_lr_combine(const void* comb, const void* s, int T, int H, int k, const int32_t* posg, void* y,
                      cudaStream_t st) {
  if (T == 0) return 0;
  lr_combine_kernel<<<(T + 7) / 8, 256, 0, st>>>((const __nv_bfloat16*)comb, (const __nv_bfloat16*)s, T, H, k, posg,
                                                 (__nv_bfloat16*)y);
  return (int)cudaGetLastError();
}

int launch_lr_combine_local(const void* o, const void* s, int T, int H, int k, const int32_t* topk_idx,
                            const int32_t* pos, const float* topk_w, int E, const LrChunks& ch, void* y,
                            cudaStream_t st) {
  if (T == 0) return 0;
  lr_combine_local_kernel<<<(T + 7) / 8, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)s, T, H, k,
                                                       topk_idx, pos, topk_w, E, ch, (__nv_bfloat16*)y);
  return (int)cudaGetLastError();
}

}  // namespace epsmoe
