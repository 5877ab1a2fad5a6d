// The layer's own all2all data plane over NVLink peer memory (a2a_p2p = 1, or
// 2 with the copies on the copy engines):
// every rank's workspace is mapped into every other rank (cudaIpc, or plain
// pointers for the in-process test group), so a chunk's dispatch / combine is
// one put kernel per rank that stores its rows straight into the peers'
// receive buffers with 16-B vector stores, then raises a per-(chunk, source)
// completion flag in each peer's memory; the consumer's stream waits on its
// flags before the chunk's GEMMs (dispatch) or the final combine.  No NCCL
// call moves routed rows in this mode; NCCL (or the test transport) only
// allgathers the counts.
//
// Ordering: the put kernel's stores, then __threadfence_system() in every CTA
// before it counts itself done; the last CTA raises the flags with st.release
// at system scope.  The waiter spins with ld.acquire at system scope, so the
// rows are visible to every kernel that follows it on that stream.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "p2p.h"

namespace epsmoe {
namespace {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int PUT_THREADS = 256;
constexpr int VEC_PER_THREAD = 8;  // a warp moves 32 x 8 consecutive 16-B vectors per step

// segs[0..nseg): contiguous copies; pre[i] = first 16-B vector of segment i
// (pre[nseg] = total).  Warp w of the grid takes vectors [w*256, (w+1)*256),
// lane l the vectors base + i*32 + l (coalesced 512-B accesses per step).
__global__ void __launch_bounds__(PUT_THREADS)
p2p_put_kernel(const P2PSeg* __restrict__ segs, const int64_t* __restrict__ pre, int nseg,
               uint32_t* __restrict__ done_ctas, uint32_t* const* __restrict__ flags, int nflags, uint32_t epoch) {
  const int64_t total = pre[nseg];
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (PUT_THREADS / 32);
  constexpr int64_t STEP = 32 * VEC_PER_THREAD;
  for (int64_t base = ((int64_t)blockIdx.x * (PUT_THREADS / 32) + (threadIdx.x >> 5)) * STEP; base < total;
       base += warps * STEP) {
    // segment of this lane's first vector (binary search), then advance in order
    int64_t v = base + lane;
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= v) lo = mid; else hi = mid - 1;
    }
    int s = lo;
#pragma unroll
    for (int i = 0; i < VEC_PER_THREAD; ++i, v += 32) {
      if (v >= total) break;
      while (v >= pre[s + 1]) ++s;
      const int64_t off = v - pre[s];
      segs[s].dst[off] = segs[s].src[off];
    }
  }
  // completion: every CTA publishes its stores system-wide, the last one raises the flags
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(done_ctas, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      for (int i = 0; i < nflags; ++i) st_release_sys(flags[i], epoch);
      atomicExch(done_ctas, 0u);  // reusable by the next forward's launch
    }
  }
}

// One warp: lane i waits until flags[i] reached `epoch` (i < n).  A wait that
// outlives ~10 s (a lost peer) traps, so the stream reports an error instead of
// hanging the device.
__global__ void p2p_wait_kernel(const uint32_t* __restrict__ flags, int n, uint32_t epoch) {
  const uint64_t t0 = globaltimer();
  for (int i = threadIdx.x; i < n; i += 32)
    while ((int32_t)(ld_acquire_sys(flags + i) - epoch) < 0) {
      __nanosleep(256);
      if (globaltimer() - t0 > 10000000000ull) {
        printf("epsmoe p2p wait timeout: flag %d of %d = %u, epoch %u\n", i, n, ld_acquire_sys(flags + i), epoch);
        asm volatile("trap;");
      }
    }
  __syncwarp();
}

// Copy-engine plane (a2a_p2p = 2): the chunk's rows were moved by
// cudaMemcpyAsync peer copies earlier on this stream (no SM involved); this
// one-thread kernel runs after they completed and raises the flags.
__global__ void p2p_signal_kernel(uint32_t* const* __restrict__ flags, int nflags, uint32_t epoch) {
  __threadfence_system();
  for (int i = 0; i < nflags; ++i) st_release_sys(flags[i], epoch);
}

}  // namespace

int launch_p2p_signal(uint32_t* const* flags, int nflags, uint32_t epoch, cudaStream_t st) {
  p2p_signal_kernel<<<1, 1, 0, st>>>(flags, nflags, epoch);
  return (int)cudaGetLastError();
}

int launch_p2p_put(const P2PSeg* segs, const int64_t* pre, int nseg, int64_t total_vec, int ctas,
                   uint32_t* done_ctas, uint32_t* const* flags, int nflags, uint32_t epoch, cudaStream_t st) {
  constexpr int64_t per_cta = (PUT_THREADS / 32) * 32 * VEC_PER_THREAD;
  int grid = (int)std::min<int64_t>(ctas, (total_vec + per_cta - 1) / per_cta);
  if (grid < 1) grid = 1;  // the flags are raised even when nothing moves
  p2p_put_kernel<<<grid, PUT_THREADS, 0, st>>>(segs, pre, nseg, done_ctas, flags, nflags, epoch);
  return (int)cudaGetLastError();
}

int launch_p2p_wait(const uint32_t* flags, int n, uint32_t epoch, cudaStream_t st) {
  p2p_wait_kernel<<<1, 32, 0, st>>>(flags, n, epoch);
  return (int)cudaGetLastError();
}

}  // namespace epsmoe
