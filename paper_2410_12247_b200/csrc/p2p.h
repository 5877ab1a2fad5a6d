// Internal interface of p2p.cu: put / wait kernels of the NVLink peer-memory
// all2all data plane (a2a_p2p = 1).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

namespace epsmoe {

// One contiguous copy of n 16-B vectors (src local, dst in a peer's mapped
// workspace or local).
struct P2PSeg {
  const uint4* src;
  uint4* dst;
};

// pre[0..nseg]: exclusive prefix of the segments' vector counts (device).
// ctas: grid cap (the SM share of the all2all).  done_ctas: device counter,
// zero between launches.  flags: device array of nflags flag addresses (one per
// consumer rank), each set to `epoch` once every vector has been stored.
int launch_p2p_put(const P2PSeg* segs, const int64_t* pre, int nseg, int64_t total_vec, int ctas,
                   uint32_t* done_ctas, uint32_t* const* flags, int nflags, uint32_t epoch, cudaStream_t st);
// a2a_p2p = 2: raise flags[0..nflags) to `epoch` (system-scope release) once the
// copy-engine copies issued before it on `st` have completed.
int launch_p2p_signal(uint32_t* const* flags, int nflags, uint32_t epoch, cudaStream_t st);
// Stream-ordered wait until flags[0..n) all reached `epoch`.
int launch_p2p_wait(const uint32_t* flags, int n, uint32_t epoch, cudaStream_t st);

}  // namespace epsmoe
