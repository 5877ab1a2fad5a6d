// HBM-bound kernels of the layer: topKGating (K2), histogram/scan/permute
// (`split`, K3) and the gate-weighted unpermute fused into combine (K7).
//
// Layout readings: send buffer rows are ordered by (expert asc,
// token asc) (R6); tokens are processed in ranges of range_len(T) consecutive
// tokens, one warp per range, so every per-expert offset is a deterministic
// prefix sum: no atomics decide any row index.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "route.h"
#include "rowops.cuh"

namespace epsmoe {
namespace {
using namespace rowops;

constexpr int WARPS = 8;    // combine
constexpr int WARPS_R = 4;  // gate / permute: small blocks (4 KB smem) that co-reside with GEMM CTAs
constexpr int MAX_EPL = 8;  // E <= 256: logits per lane
constexpr int MAX_K = 8;    // top_k <= 8

__device__ __forceinline__ bool better(float av, int ae, float bv, int be) {
  return av > bv || (av == bv && ae < be);
}
// A NaN logit (only NaN / Inf inputs make one) ranks as -inf (R18): never ahead of
// a number, 0 in the softmax sum.  An all-NaN row then still selects k valid
// experts (the lowest ids: -inf ties) and its weights are NaN (max = -inf), so
// the token's y is NaN instead of an out-of-range expert index.
__device__ __forceinline__ float logit_or_neg_inf(float v) { return v != v ? -INFINITY : v; }

// U consecutive tokens of a routing range, unrestricted routing (see the
// kernel below for the per-token definition; this is the same arithmetic).
constexpr int GATE_U = 4;
template <int U, int EPL>
__device__ __forceinline__ void gate_tokens(const float* __restrict__ logits, int t0, int E, int k, int norm_topk,
                                            float scale, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                                            int32_t* hist, int lane) {
  float v[U][EPL];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const float* row = logits + (int64_t)(t0 + u) * E;
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const int e = lane + 32 * i;
      v[u][i] = (e < E) ? logit_or_neg_inf(row[e]) : -INFINITY;
    }
  }
  uint32_t taken[U];
  float top_v[U][MAX_K];
  int top_e[U][MAX_K];
#pragma unroll
  for (int u = 0; u < U; ++u) taken[u] = 0;
#pragma unroll
  for (int j = 0; j < MAX_K; ++j) {
    if (j < k) {
      float bv[U];
      int be[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bv[u] = -INFINITY;
        be[u] = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int e = lane + 32 * i;
          if (e < E && !((taken[u] >> i) & 1u) && better(v[u][i], e, bv[u], be[u])) { bv[u] = v[u][i]; be[u] = e; }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv[u], off);
          const int oe = __shfl_xor_sync(0xffffffffu, be[u], off);
          if (better(ov, oe, bv[u], be[u])) { bv[u] = ov; be[u] = oe; }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        top_v[u][j] = bv[u];
        top_e[u][j] = be[u];
        if ((be[u] & 31) == lane) taken[u] |= 1u << (be[u] >> 5);
      }
    }
  }
  float sm[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const float m = top_v[u][0];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < EPL; ++i) s += expf(v[u][i] - m);
    sm[u] = s;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int u = 0; u < U; ++u) sm[u] += __shfl_xor_sync(0xffffffffu, sm[u], off);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const float m = top_v[u][0];
    float psel = 0.f, pj = 0.f;
    int ej = 0;
#pragma unroll
    for (int j = 0; j < MAX_K; ++j) {
      if (j < k) {
        const float pv = expf(top_v[u][j] - m) / sm[u];
        psel += pv;
        if (j == lane) { pj = pv; ej = top_e[u][j]; }
      }
    }
    const int64_t t = t0 + u;
    if (lane < k) {
      const float w = norm_topk ? pj / psel : pj;
      topk_idx[t * k + lane] = ej;
      topk_w[t * k + lane] = w * scale;
    }
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < MAX_K; ++j)
        if (j < k) hist[top_e[u][j]] += 1;
  }
  __syncwarp();
}

// K2 topKGating.  One warp per range of range_len(T) tokens, tokens
// in order.  idx = k largest logits (ties -> lower expert id, R2); p = softmax
// over all E in fp32; w_j = p_{idx_j} (/ sum_j p_{idx_j} if norm_topk) * scale.
// Also writes the range's expert histogram range_hist[e * R + r].
// EPL = ceil(E / 32) logits per lane (a loop over MAX_EPL with the e < E guard
// would add only -inf candidates and +0 softmax terms: the same bits, more work).
template <int EPL>
__global__ void __launch_bounds__(WARPS_R * 32)
gate_topk_kernel(const float* __restrict__ logits, int T, int E, int k, int norm_topk, float scale,
                 int override_routing, int route_groups, int route_topk_groups, int32_t* __restrict__ topk_idx,
                 float* __restrict__ topk_w, int32_t* __restrict__ range_hist, int R, int rt, int interleave) {
  __shared__ int32_t hist_s[WARPS_R][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * WARPS_R + warp;
  for (int e = lane; e < E; e += 32) hist_s[warp][e] = 0;
  __syncwarp();
  if (r < R) {
    const int t_end = min(T, (r + 1) * rt);
    int t = r * rt;
    if (interleave && !override_routing && !route_groups) {
      // GATE_U tokens at a time: the same per-token operations (lane-strided
      // logits, local argmax in i order, the same xor-shuffle trees, the same
      // softmax sum order), interleaved so their shuffle / expf latencies overlap:
      // bit-identical to the one-token loop below, which takes the remainder
      for (; t + GATE_U <= t_end; t += GATE_U) gate_tokens<GATE_U, EPL>(logits, t, E, k, norm_topk, scale, topk_idx, topk_w,
                                                                  hist_s[warp], lane);
    }
    for (; t < t_end; ++t) {
      if (override_routing) {
        if (lane < k) {
          int e = topk_idx[(int64_t)t * k + lane];
          atomicAdd(&hist_s[warp][e], 1);  // order-free count
        }
        continue;
      }
      float v[EPL];
      const float* row = logits + (int64_t)t * E;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        int e = lane + 32 * i;
        v[i] = (e < E) ? logit_or_neg_inf(row[e]) : -INFINITY;
      }
      uint32_t taken = 0;
      if (route_groups) {
        // device-limited routing (R17): lane q < route_groups holds group q's
        // best logit; the route_topk_groups best groups (score desc, id asc)
        // stay eligible, the other groups' experts are marked taken
        const int gsz = E / route_groups;
        float gscore = -INFINITY;
        for (int q = 0; q < route_groups; ++q) {
          float m = -INFINITY;
#pragma unroll
          for (int i = 0; i < EPL; ++i) {
            const int e = lane + 32 * i;
            if (e < E && e / gsz == q) m = fmaxf(m, v[i]);
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
          if (lane == q) gscore = m;
        }
        uint32_t keep = 0;
        bool used = lane >= route_groups;
        for (int j = 0; j < route_topk_groups; ++j) {
          float bv = used ? -INFINITY : gscore;
          int bg = used ? 0x7fffffff : lane;
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const int og = __shfl_xor_sync(0xffffffffu, bg, off);
            if (better(ov, og, bv, bg)) { bv = ov; bg = og; }
          }
          keep |= 1u << bg;
          if (lane == bg) used = true;
        }
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          const int e = lane + 32 * i;
          if (e < E && !((keep >> (e / gsz)) & 1u)) taken |= 1u << i;
        }
      }
      float top_v[8];
      int top_e[8];
      for (int j = 0; j < k; ++j) {
        float bv = -INFINITY;
        int be = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < EPL; ++i) {
          int e = lane + 32 * i;
          if (e < E && !((taken >> i) & 1u) && better(v[i], e, bv, be)) { bv = v[i]; be = e; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          float ov = __shfl_xor_sync(0xffffffffu, bv, off);
          int oe = __shfl_xor_sync(0xffffffffu, be, off);
          if (better(ov, oe, bv, be)) { bv = ov; be = oe; }
        }
        top_v[j] = bv;
        top_e[j] = be;
        if ((be & 31) == lane) taken |= 1u << (be >> 5);
      }
      // softmax denominator over all E (max = top-1 logit)
      const float m = top_v[0];
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < EPL; ++i) s += expf(v[i] - m);   // -inf lanes add 0
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      float psel = 0.f;
      float pj = 0.f;
      for (int j = 0; j < k; ++j) {
        float pv = expf(top_v[j] - m) / s;
        psel += pv;
        if (j == lane) pj = pv;
      }
      if (lane < k) {
        float w = norm_topk ? pj / psel : pj;
        topk_idx[(int64_t)t * k + lane] = top_e[lane];
        topk_w[(int64_t)t * k + lane] = w * scale;
      }
      if (lane == 0)
        for (int j = 0; j < k; ++j) hist_s[warp][top_e[j]] += 1;
      __syncwarp();
    }
  }
  __syncwarp();
  if (r < R)
    for (int e = lane; e < E; e += 32) range_hist[(int64_t)e * R + r] = hist_s[warp][e];
}

// Exclusive scan of range_hist[e][0..R) per expert (one block per expert);
// range_off[e][r] = sum_{r' < r}, hist[e] = total.
__global__ void __launch_bounds__(1024)
range_scan_kernel(const int32_t* __restrict__ range_hist, int R, int32_t* __restrict__ range_off,
                  int32_t* __restrict__ hist) {
  __shared__ int32_t warp_sum[32];
  const int e = blockIdx.x;
  const int per = (R + blockDim.x - 1) / blockDim.x;
  const int r0 = threadIdx.x * per;
  const int32_t* src = range_hist + (int64_t)e * R;
  int local = 0;
  for (int i = 0; i < per; ++i)
    if (r0 + i < R) local += src[r0 + i];
  // block exclusive scan of `local`
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) warp_sum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int ws = (lane < (int)(blockDim.x >> 5)) ? warp_sum[lane] : 0;
    int wi = ws;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, wi, off);
      if (lane >= off) wi += v;
    }
    warp_sum[lane] = wi - ws;  // exclusive per-warp base
    if (lane == 31) hist[e] = wi;
  }
  __syncthreads();
  int run = warp_sum[warp] + incl - local;
  int32_t* dst = range_off + (int64_t)e * R;
  for (int i = 0; i < per; ++i)
    if (r0 + i < R) {
      dst[r0 + i] = run;
      run += src[r0 + i];
    }
}

__device__ __forceinline__ int block_exclusive_scan_256(int v, int* sh) {
  // blockDim.x == 256
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += sh[w];
  __syncthreads();
  return base + incl - v;
}

// seg_start[e] = sum_{e' < e} hist[e'] (send layout expert-major, R6), [E] = total.
__global__ void __launch_bounds__(256) seg_scan_kernel(const int32_t* __restrict__ hist, int E,
                                                       int32_t* __restrict__ seg_start) {
  __shared__ int32_t scan_tmp[8];
  int hv = (threadIdx.x < E) ? hist[threadIdx.x] : 0;
  int ex = block_exclusive_scan_256(hv, scan_tmp);
  if (threadIdx.x < E) seg_start[threadIdx.x] = ex;
  if (threadIdx.x == 255) seg_start[E] = ex + hv;
}

// K3 permute (`split`).  One warp per token range; each token's row is
// read once and written to its k destination rows with 16-byte stores.
// fp8: 0 = bf16 rows; 1 = bf16 rows of the FP8 round trip (ep == 1: the
// values experts see when the payload is FP8); 2 = packed FP8 rows of `qpitch`
// bytes (H e4m3 bytes, then H/128 int8 block exponents) into `sendq`.
template <int fp8, bool SPLIT>
__global__ void __launch_bounds__(WARPS_R * 32, 4)
permute_kernel(const __nv_bfloat16* __restrict__ x, int T, int H, int E, int k,
               const int32_t* __restrict__ topk_idx, const int32_t* __restrict__ range_off,
               const int32_t* __restrict__ seg_start, int R, int rt, __nv_bfloat16* __restrict__ send,
               int32_t* __restrict__ pos, int32_t* __restrict__ row_token, uint8_t* __restrict__ sendq,
               int qpitch) {
  __shared__ int32_t off_s[WARPS_R][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * WARPS_R + warp;
  if (r >= R) return;
  for (int e = lane; e < E; e += 32) off_s[warp][e] = seg_start[e] + range_off[(int64_t)e * R + r];
  __syncwarp();
  const int nvec = H >> 3;  // uint4 = 8 bf16
  const int t_end = min(T, (r + 1) * rt);
  const uint64_t pol = evict_first_policy();
  for (int t = r * rt; t < t_end; ++t) {
    int dest = 0;
    if (lane < k) {
      int e = topk_idx[(int64_t)t * k + lane];
      dest = off_s[warp][e];
      if (!SPLIT || blockIdx.y == 0) {  // column splits (small batches): the first writes the indices
        pos[(int64_t)t * k + lane] = dest;
        if (row_token) row_token[dest] = t;
      }
    }
    __syncwarp();
    if (lane < k) {
      int e = topk_idx[(int64_t)t * k + lane];
      off_s[warp][e] = dest + 1;  // experts of one token are distinct
    }
    __syncwarp();
    if (send == nullptr && fp8 != 2) continue;  // index-only split: the GEMM gathers rows of x itself
    const uint4* src = reinterpret_cast<const uint4*>(x + (int64_t)t * H);
    // 16 x 16 B per lane in flight per pass (H <= 4096 per pass, <= 2 passes):
    // keeps the kernel under 128 registers so it co-resides with a GEMM CTA.
    // Small batches split a row's 32-vector blocks over gridDim.y warps
    // (blocks y, y + Y, ...); every value is copied / quantised exactly as unsplit.
    constexpr int MAXV = 16;
    const int stride = SPLIT ? 32 * (int)gridDim.y : 32;  // vectors between a warp's consecutive blocks
    for (int base = (SPLIT ? 32 * (int)blockIdx.y : 0) + lane; base - lane < nvec; base += MAXV * stride) {
      // this lane's vector of pass slot i: base + i * stride (>= nvec: none)
      uint4 buf[MAXV];
#pragma unroll
      for (int i = 0; i < MAXV; ++i) {
        int c = base + i * stride;
        if (c < nvec) buf[i] = ld_stream(src + c, pol);
      }
      if constexpr (fp8 != 0) {
        // per-block exponent: amax over the half warp holding the block's 16 uint4
        int sexp[MAXV];
#pragma unroll
        for (int i = 0; i < MAXV; ++i) {
          float m = (base + i * stride < nvec) ? amax8(buf[i]) : 0.f;
#pragma unroll
          for (int off = 8; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
          sexp[i] = fp8_block_exp(m);
        }
        if (fp8 == 1) {
#pragma unroll
          for (int i = 0; i < MAXV; ++i)
            if (base + i * stride < nvec) buf[i] = dequant8(quant8(buf[i], pow2f(-sexp[i])), pow2f(sexp[i]));
        } else {
          uint2 q[MAXV];
#pragma unroll
          for (int i = 0; i < MAXV; ++i)
            if (base + i * stride < nvec) q[i] = quant8(buf[i], pow2f(-sexp[i]));
          for (int j = 0; j < k; ++j) {
            int d = __shfl_sync(0xffffffffu, dest, j);
            uint8_t* row = sendq + (int64_t)d * qpitch;
#pragma unroll
            for (int i = 0; i < MAXV; ++i) {
              const int c = base + i * stride;
              if (c < nvec) {
                reinterpret_cast<uint2*>(row)[c] = q[i];
                if ((lane & 15) == 0) row[H + (c >> 4)] = (uint8_t)(int8_t)sexp[i];
              }
            }
          }
          continue;
        }
      }
      for (int j = 0; j < k; ++j) {
        int d = __shfl_sync(0xffffffffu, dest, j);
        uint4* dst = reinterpret_cast<uint4*>(send + (int64_t)d * H);
#pragma unroll
        for (int i = 0; i < MAXV; ++i) {
          int c = base + i * stride;
          if (c < nvec) st_stream(dst + c, buf[i], pol);
        }
      }
    }
  }
}

// Receiver side of the FP8 dispatch: rows [0, rows) of packed FP8 rows (pitch
// qpitch) -> bf16 rows (pitch H), x' = q 2^s exactly.  One warp per row.
__global__ void __launch_bounds__(256) dequant_rows_kernel(const uint8_t* __restrict__ q, int64_t rows, int H,
                                                           int qpitch, __nv_bfloat16* __restrict__ out) {
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const uint8_t* src = q + row * qpitch;
  uint4* dst = reinterpret_cast<uint4*>(out + row * H);
  const int nvec = H >> 3;
  for (int c = lane; c < nvec; c += 32) {
    const uint2 v = reinterpret_cast<const uint2*>(src)[c];
    const int s = (int)(int8_t)src[H + (c >> 4)];
    dst[c] = dequant8(v, pow2f(s));
  }
}

// K7 LocalReduce fused into combine (R7): one warp per token,
// acc = fp32(s) (0 without shared experts); acc = fmaf(w_j, o[pos[t][j]], acc)
// in slot order; y = bf16(acc).
template <bool SPLIT>
__global__ void __launch_bounds__(WARPS * 32)
combine_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ s, int T, int H,
               int k, const int32_t* __restrict__ pos, const float* __restrict__ topk_w,
               __nv_bfloat16* __restrict__ y) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * WARPS + warp;
  if (t >= T) return;
  int prow = 0;
  float pw = 0.f;
  if (lane < k) {
    prow = pos[(int64_t)t * k + lane];
    pw = topk_w[(int64_t)t * k + lane];
  }
  const int nvec = H >> 3;
  const uint64_t pol = evict_first_policy();
  const uint4* orow[MAX_K];
  float wj[MAX_K];
#pragma unroll
  for (int j = 0; j < MAX_K; ++j) {
    const int row = __shfl_sync(0xffffffffu, prow, j < k ? j : 0);
    orow[j] = reinterpret_cast<const uint4*>(o + (int64_t)row * H);
    wj[j] = __shfl_sync(0xffffffffu, pw, j < k ? j : 0);
  }
  // small batches: gridDim.y warps share a token's columns (interleaved 32-vector
  // blocks); each element's arithmetic is unchanged
  const int stride = SPLIT ? 32 * (int)gridDim.y : 32;
  for (int c = (SPLIT ? 32 * (int)blockIdx.y : 0) + lane; c < nvec; c += stride) {
    // all k rows in flight first, then the fmaf chain in slot order (R4)
    uint4 ov[MAX_K];
#pragma unroll
    for (int j = 0; j < MAX_K; ++j)
      if (j < k) ov[j] = ld_stream(orow[j] + c, pol);
    float acc[8];
    if (s) {
      uint4 sv = ld_stream(reinterpret_cast<const uint4*>(s + (int64_t)t * H) + c, pol);
      const __nv_bfloat16* sb = reinterpret_cast<const __nv_bfloat16*>(&sv);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __bfloat162float(sb[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < MAX_K; ++j) {
      if (j < k) {
        const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(&ov[j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = __fmaf_rn(wj[j], __bfloat162float(ob[i]), acc[i]);
      }
    }
    uint4 outv;
    __nv_bfloat162* ob2 = reinterpret_cast<__nv_bfloat162*>(&outv);
#pragma unroll
    for (int i = 0; i < 4; ++i) ob2[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
    st_stream(reinterpret_cast<uint4*>(y + (int64_t)t * H) + c, outv, pol);
  }
}

// Pairs per (expert, token slice) for token-sliced chunks (R8 extension):
// slice s of T tokens = balanced contiguous ranges, the first T mod S one
// token longer.  Order-free counts (atomics on a zeroed array).
__global__ void __launch_bounds__(256) slice_hist_kernel(const int32_t* __restrict__ topk_idx, int T, int k, int S,
                                                         int32_t* __restrict__ hs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)T * k) return;
  const int t = (int)(i / k);
  const int base = T / S, rem = T % S;
  const int s = (t < rem * (base + 1)) ? t / (base + 1) : rem + (t - rem * (base + 1)) / base;
  atomicAdd(&hs[topk_idx[i] * S + s], 1);
}

// Zero-pad copy of the router weight into a [256, H] buffer (create time).
__global__ void pad_rows_kernel(const __nv_bfloat16* __restrict__ src, int rows, int H,
                                __nv_bfloat16* __restrict__ dst, int rows_pad) {
  int64_t n = (int64_t)rows_pad * H;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t rr = i / H;
    dst[i] = rr < rows ? src[i] : __float2bfloat16(0.f);
  }
}

}  // namespace

static int ranges_target() {
  static const int v = [] {
    const char* e = std::getenv("EPSMOE_RANGES");
    return e ? std::max(64, std::atoi(e)) : 2048;
  }();
  return v;
}
int range_len(int64_t T) {
  int p = 1;
  while (p < 32 && (T + p - 1) / p > ranges_target()) p <<= 1;
  return p;
}
int num_ranges(int64_t T) {
  const int p = range_len(T);
  return (int)((T + p - 1) / p);
}
int max_ranges(int64_t T_max) {
  return (int)std::max<int64_t>(std::min<int64_t>(T_max, ranges_target()), num_ranges(T_max));
}

static int gate_interleave() {  // EPSMOE_GATE_U=0: one token at a time (bit-identical, slower)
  static const int v = [] {
    const char* e = std::getenv("EPSMOE_GATE_U");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

int launch_gate_topk(const float* logits, int T, int E, int k, int norm_topk, float scale, int override_routing,
                     int route_groups, int route_topk_groups, int32_t* topk_idx, float* topk_w,
                     int32_t* range_hist, cudaStream_t st) {
  int R = num_ranges(T);
  if (R == 0) return 0;
  if (route_groups <= 1 || route_topk_groups >= route_groups) route_groups = 0;  // unrestricted
  const dim3 grid((R + WARPS_R - 1) / WARPS_R), block(WARPS_R * 32);
  const int rt = range_len(T), il = gate_interleave();
#define EPSMOE_GATE_CASE(n)                                                                                \
  case n:                                                                                                  \
    gate_topk_kernel<n><<<grid, block, 0, st>>>(logits, T, E, k, norm_topk, scale, override_routing,        \
                                                route_groups, route_topk_groups, topk_idx, topk_w,         \
                                                range_hist, R, rt, il);                                    \
    break;
  switch ((E + 31) / 32) {
    EPSMOE_GATE_CASE(1) EPSMOE_GATE_CASE(2) EPSMOE_GATE_CASE(3) EPSMOE_GATE_CASE(4)
    EPSMOE_GATE_CASE(5) EPSMOE_GATE_CASE(6) EPSMOE_GATE_CASE(7) EPSMOE_GATE_CASE(8)
    default: return (int)cudaErrorInvalidValue;
  }
#undef EPSMOE_GATE_CASE
  return (int)cudaGetLastError();
}

int launch_range_scan(const int32_t* range_hist, int T, int E, int32_t* range_off, int32_t* hist,
                      int32_t* seg_start, cudaStream_t st) {
  int R = num_ranges(T);
  if (R == 0) {
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(int32_t) * E, st);
    if (e != cudaSuccess) return (int)e;
  } else {
    range_scan_kernel<<<E, 1024, 0, st>>>(range_hist, R, range_off, hist);
  }
  seg_scan_kernel<<<1, 256, 0, st>>>(hist, E, seg_start);
  return (int)cudaGetLastError();
}

// Column splits for small batches: enough warps to cover the SMs (a warp per
// token alone leaves decode batches latency-bound).
static int column_splits(int64_t rows, int H) {
  const int64_t target = 148 * 16;  // warps
  const int max_split = std::max(1, (H / 8) / 32);
  return (int)std::max<int64_t>(1, std::min<int64_t>(max_split, (target + rows - 1) / std::max<int64_t>(rows, 1)));
}

int launch_permute(const void* x, int T, int H, int E, int k, const int32_t* topk_idx, const int32_t* range_off,
                   const int32_t* seg_start, void* send, int32_t* pos, int32_t* row_token, int fp8, void* sendq,
                   int qpitch, cudaStream_t st) {
  int R = num_ranges(T);
  const int rt = range_len(T);
  if (R == 0) return 0;
  const int splits = column_splits(R, H);
  const dim3 grid((R + WARPS_R - 1) / WARPS_R, splits), block(WARPS_R * 32);
  auto xb = (const __nv_bfloat16*)x;
  auto sb = (__nv_bfloat16*)send;
  auto qb = (uint8_t*)sendq;
  if (fp8 == 0)
    (splits > 1 ? permute_kernel<0, true> : permute_kernel<0, false>)<<<grid, block, 0, st>>>(
        xb, T, H, E, k, topk_idx, range_off, seg_start, R, rt, sb, pos, row_token, qb, qpitch);
  else if (fp8 == 1)
    (splits > 1 ? permute_kernel<1, true> : permute_kernel<1, false>)<<<grid, block, 0, st>>>(
        xb, T, H, E, k, topk_idx, range_off, seg_start, R, rt, sb, pos, row_token, qb, qpitch);
  else
    (splits > 1 ? permute_kernel<2, true> : permute_kernel<2, false>)<<<grid, block, 0, st>>>(
        xb, T, H, E, k, topk_idx, range_off, seg_start, R, rt, sb, pos, row_token, qb, qpitch);
  return (int)cudaGetLastError();
}

int launch_dequant_rows(const void* q, int64_t rows, int H, int qpitch, void* out, cudaStream_t st) {
  if (rows <= 0) return 0;
  dequant_rows_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>((const uint8_t*)q, rows, H, qpitch,
                                                                   (__nv_bfloat16*)out);
  return (int)cudaGetLastError();
}

int launch_combine(const void* o, const void* s, int T, int H, int k, const int32_t* pos, const float* topk_w,
                   void* y, cudaStream_t st) {
  if (T == 0) return 0;
  const int splits = column_splits(T, H);
  const dim3 grid((T + WARPS - 1) / WARPS, splits);
  (splits > 1 ? combine_kernel<true> : combine_kernel<false>)<<<grid, WARPS * 32, 0, st>>>((const __nv_bfloat16*)o,
                                                                 (const __nv_bfloat16*)s, T, H, k, pos, topk_w,
                                                                 (__nv_bfloat16*)y);
  return (int)cudaGetLastError();
}

int launch_slice_hist(const int32_t* topk_idx, int T, int k, int E, int S, int32_t* hs, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(hs, 0, sizeof(int32_t) * E * S, st);
  if (e != cudaSuccess) return (int)e;
  if (T == 0) return 0;
  const int64_t n = (int64_t)T * k;
  slice_hist_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(topk_idx, T, k, S, hs);
  return (int)cudaGetLastError();
}

int launch_pad_rows(const void* src, int rows, int H, void* dst, int rows_pad, cudaStream_t st) {
  pad_rows_kernel<<<296, 256, 0, st>>>((const __nv_bfloat16*)src, rows, H, (__nv_bfloat16*)dst, rows_pad);
  return (int)cudaGetLastError();
}

}  // namespace epsmoe
