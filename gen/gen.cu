// Device twin of gen/synth.py (seeded synthetic inputs; NO method arithmetic).
// Bit-identical to the numpy generator (tests/test_gen.py).  Built into
// gen/libepsgen.so; used by bench.py and tests to fill large device buffers.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr uint64_t TID_MUL = 0xD1B54A32D192ED03ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float v) {
  uint32_t b = __float_as_uint(v);
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

__global__ void fill_kernel(uint16_t* __restrict__ dst, int64_t n, uint64_t key,
                            int64_t index_base, int mode, float param) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint64_t h = mix64(key + (uint64_t)(index_base + i + 1) * GOLDEN);
    float v;
    if (mode == 0) {
      float f = __fsub_rn(__fmul_rn((float)(uint32_t)(h >> 40), 1.1920928955078125e-07f), 1.0f);
      v = __fmul_rn(f, param);
    } else {
      int nn = (int)((h >> 32) % 17ull) - 8;
      v = __fdiv_rn((float)nn, param);
    }
    dst[i] = f32_to_bf16_rne(v);
  }
}

}  // namespace

extern "C" {

// Fill dst[0..n) (device, bf16 bits) with elements index_base..index_base+n-1
// of stream (seed, tid).  mode 0 = "unif" (param = fp32 scale), 1 = "grid"
// (param = denominator).  Returns a cudaError_t.
int epsgen_fill_bf16(void* dst, int64_t n, uint64_t seed, int32_t tid, int64_t index_base,
                     int32_t mode, float param, void* stream) {
  if (n <= 0) return 0;
  uint64_t key = mix64(seed ^ ((uint64_t)(tid + 1) * TID_MUL));
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>((uint16_t*)dst, n, key,
                                                                  index_base, mode, param);
  return (int)cudaGetLastError();
}

}
