// Device helpers shared by the HBM-bound row kernels (route.cu,
// local_reduce.cu): streaming 16-B accesses and the FP8 dispatch codec (R15).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>

#include <cstdint>

namespace epsmoe {
namespace rowops {

// Streaming 16-byte accesses for the HBM-bound kernels: L1 no-allocate, L2
// evict-first, so the activations they stream (GBs per layer) do not evict
// the concurrently running GEMMs' operand tiles from L2.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld_stream(const uint4* ptr, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_stream(uint4* ptr, const uint4& v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
// ---- FP8 dispatch payload (NEXT-2, R15): per 128-column block a power-of-two
// scale 2^s with s the smallest integer such that max|x| / 2^s <= 448; values
// x 2^-s are rounded to e4m3 (RNE, never saturating); the receiver's x' = q 2^s
// is exact in bf16.  One uint4 = 8 bf16 = 1/16 of a block; the 16 uint4 of a
// block sit in 16 consecutive lanes (a half warp) of the permute's copy loop.
__device__ __forceinline__ int fp8_block_exp(float amax) {
  const uint32_t b = __float_as_uint(amax);
  if (amax == 0.f || (b >> 23) == 0) return -126;  // zero / subnormal block
  const int e = (int)(b >> 23) - 127;
  const int s = ((b & 0x7FFFFFu) <= 0x600000u) ? e - 8 : e - 7;  // mantissa <= 1.75 ?
  return max(-126, s);
}
__device__ __forceinline__ float pow2f(int s) { return __uint_as_float((uint32_t)(127 + s) << 23); }

// 8 bf16 -> 8 e4m3 bytes of x * inv (inv = 2^-s, exact)
__device__ __forceinline__ uint2 quant8(const uint4& v, float inv) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
  uint32_t w[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float2 a = __bfloat1622float2(p[2 * h]), b = __bfloat1622float2(p[2 * h + 1]);
    __nv_fp8x2_storage_t qa = __nv_cvt_float2_to_fp8x2(make_float2(a.x * inv, a.y * inv), __NV_SATFINITE, __NV_E4M3);
    __nv_fp8x2_storage_t qb = __nv_cvt_float2_to_fp8x2(make_float2(b.x * inv, b.y * inv), __NV_SATFINITE, __NV_E4M3);
    w[h] = (uint32_t)qa | ((uint32_t)qb << 16);
  }
  return make_uint2(w[0], w[1]);
}
// 8 e4m3 bytes -> 8 bf16 of q * scale (exact)
__device__ __forceinline__ uint4 dequant8(const uint2& q, float scale) {
  uint4 out;
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(&out);
  const uint32_t w[2] = {q.x, q.y};
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(w[h] >> (16 * part)), __NV_E4M3);
      float2 f = __half22float2(*reinterpret_cast<__half2*>(&hr));
      o[2 * h + part] = __floats2bfloat162_rn(f.x * scale, f.y * scale);
    }
  return out;
}
__device__ __forceinline__ float amax8(const uint4& v) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
  float m = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(p[i]);
    m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
  }
  return m;
}

}  // namespace rowops
}  // namespace epsmoe
