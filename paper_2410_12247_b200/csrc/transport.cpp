// Transports for the EP all2all (see transport.h).  Return codes: 0 = ok,
// MOE_ERR_NCCL / MOE_ERR_CUDA on failure (message via set_error).
#include "transport.h"

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>

#include "../../include/epsmoe.h"
#include "internal.h"

namespace epsmoe {

// ------------------------------------------------------------------ NCCL
static int nccl_err(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return 0;
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return MOE_ERR_NCCL;
}

NcclTransport::~NcclTransport() {
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  for (const Split& s : splits_)
    for (ncclComm_t c : s.c)
      if (c) ncclCommDestroy(c);
  for (auto c : base_)
    if (c) ncclCommDestroy(c);
}

// cudaIpc mapping of every rank's `mine` (+ its offset inside its cudaMalloc
// allocation); `gather(send, recv, bytes)` is a blocking host allgather of
// `bytes` per rank.  opened: handles to close on teardown.
static int ipc_map_peers(void* mine, int nranks, int me,
                         const std::function<int(const void*, void*, size_t)>& gather,
                         std::vector<void*>& opened, std::vector<char*>& out) {
  // handle of the whole allocation + this pointer's offset inside it
  CUdeviceptr base = 0;
  size_t size = 0;
  using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || reinterpret_cast<RangeFn>(fp)(&base, &size, (CUdeviceptr)mine) != CUDA_SUCCESS) {
    set_error("map_peers: cuMemGetAddressRange failed");
    return MOE_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void*)base) != cudaSuccess) {
    set_error("map_peers: cudaIpcGetMemHandle failed (workspace must come from cudaMalloc)");
    return MOE_ERR_CUDA;
  }
  constexpr int W = (int)(sizeof(cudaIpcMemHandle_t) / 4) + 2;  // handle words + 64-bit offset
  int32_t rec[W];
  std::memcpy(rec, &h, sizeof(h));
  const int64_t off = (int64_t)((CUdeviceptr)mine - base);
  std::memcpy(rec + W - 2, &off, sizeof(off));
  std::vector<int32_t> all((size_t)W * nranks);
  if (int e = gather(rec, all.data(), sizeof(rec))) return e;
  out.assign(nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    if (r == me) { out[r] = (char*)mine; continue; }
    cudaIpcMemHandle_t hr;
    int64_t offr = 0;
    std::memcpy(&hr, all.data() + (size_t)r * W, sizeof(hr));
    std::memcpy(&offr, all.data() + (size_t)r * W + W - 2, sizeof(offr));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hr, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      set_error("map_peers: cudaIpcOpenMemHandle failed for rank " + std::to_string(r));
      return MOE_ERR_CUDA;
    }
    opened.push_back(p);
    out[r] = (char*)p + offr;
  }
  return 0;
}

int NcclTransport::map_peers(void* mine, std::vector<char*>& out) {
  int nranks = 0, me = 0;
  if (int e = nccl_err(ncclCommCount(comm_[0], &nranks), "ncclCommCount")) return e;
  if (int e = nccl_err(ncclCommUserRank(comm_[0], &me), "ncclCommUserRank")) return e;
  // the handles travel through a device buffer and one allgather on communicator 0
  auto gather = [&](const void* send, void* recv, size_t bytes) -> int {
    char* dev = nullptr;
    if (cudaMalloc(&dev, bytes * (nranks + 1)) != cudaSuccess) return MOE_ERR_CUDA;
    cudaMemcpy(dev, send, bytes, cudaMemcpyHostToDevice);
    int e = nccl_err(ncclAllGather(dev, dev + bytes, bytes, ncclUint8, comm_[0], 0), "ncclAllGather");
    if (!e) e = cudaMemcpy(recv, dev + bytes, bytes * nranks, cudaMemcpyDeviceToHost) ? MOE_ERR_CUDA : 0;
    cudaFree(dev);
    return e;
  };
  return ipc_map_peers(mine, nranks, me, gather, opened_, out);
}

// NEXT-1: the communicators' CTA budget.  ncclCommSplit (color 0, key = rank:
// same ranks, same order) with maxCTAs = ctas gives communicators with the new
// SM budget without a new bootstrap; they are kept for reuse.
int NcclTransport::set_comm_ctas(int ctas) {
  if (ctas <= 0 || ctas == ctas_) return 0;
  for (const Split& s : splits_)
    if (s.ctas == ctas) {
      comm_[0] = s.c[0];
      comm_[1] = s.c[1];
      ctas_ = ctas;
      return 0;
    }
  Split s{ctas, {nullptr, nullptr}};
  int me = 0;
  if (int e = nccl_err(ncclCommUserRank(base_[0], &me), "ncclCommUserRank")) return e;
  for (int i = 0; i < 2; ++i) {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 1;
    cfg.maxCTAs = ctas;
    cfg.minCTAs = std::min(ctas, 2);
    if (int e = nccl_err(ncclCommSplit(base_[i], 0, me, &s.c[i], &cfg), "ncclCommSplit")) return e;
  }
  splits_.push_back(s);
  comm_[0] = s.c[0];
  comm_[1] = s.c[1];
  ctas_ = ctas;
  return 0;
}

int NcclTransport::poll_async() {
  for (ncclComm_t c : base_) {
    ncclResult_t r = ncclSuccess;
    if (c && ncclCommGetAsyncError(c, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress)
      return nccl_err(r, "ncclCommGetAsyncError");
  }
  for (const Split& s : splits_)
    for (ncclComm_t c : s.c) {
      ncclResult_t r = ncclSuccess;
      if (c && ncclCommGetAsyncError(c, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress)
        return nccl_err(r, "ncclCommGetAsyncError");
    }
  return 0;
}

// ------------------------------------------------------------------ host collective
HostCollTransport::~HostCollTransport() {
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
}

int HostCollTransport::unsupported() {
  set_error("host-collective transport: routed rows move only on a2a_p2p = 1 or 2 (no send / recv)");
  return MOE_ERR_UNSUPPORTED;
}

int HostCollTransport::gather_host(const void* send, void* recv, size_t bytes) {
  if (fn_(ctx_, send, recv, bytes) != 0) {
    set_error("host allgather callback failed");
    return MOE_ERR_MISMATCH;
  }
  return 0;
}

int HostCollTransport::allgather_i32(const int32_t* send, int32_t* recv, size_t count, cudaStream_t st) {
  std::vector<int32_t> mine(count), all(count * ep_);
  if (cudaMemcpyAsync(mine.data(), send, count * sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("host-collective allgather: device->host copy failed");
    return MOE_ERR_CUDA;
  }
  if (int e = gather_host(mine.data(), all.data(), count * sizeof(int32_t))) return e;
  if (cudaMemcpyAsync(recv, all.data(), all.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("host-collective allgather: host->device copy failed");
    return MOE_ERR_CUDA;
  }
  return 0;
}

int HostCollTransport::map_peers(void* mine, std::vector<char*>& out) {
  auto gather = [&](const void* send, void* recv, size_t bytes) { return gather_host(send, recv, bytes); };
  return ipc_map_peers(mine, ep_, rank_, gather, opened_, out);
}


int NcclTransport::allgather_i32(const int32_t* send, int32_t* recv, size_t count, cudaStream_t st) {
  return nccl_err(ncclAllGather(send, recv, count, ncclInt32, comm_[0], st), "ncclAllGather");
}
int NcclTransport::group_start(int) { return nccl_err(ncclGroupStart(), "ncclGroupStart"); }
int NcclTransport::send(const void* buf, size_t bytes, int peer, int channel, cudaStream_t st) {
  return nccl_err(ncclSend(buf, bytes, ncclUint8, peer, comm_[channel], st), "ncclSend");
}
int NcclTransport::recv(void* buf, size_t bytes, int peer, int channel, cudaStream_t st) {
  return nccl_err(ncclRecv(buf, bytes, ncclUint8, peer, comm_[channel], st), "ncclRecv");
}
int NcclTransport::group_end(int, cudaStream_t) { return nccl_err(ncclGroupEnd(), "ncclGroupEnd"); }

// ------------------------------------------------------------------ local
LocalGroup::LocalGroup(int n)
    : ep(n), sends(n), recvs(n), gather_src(n), peer_ptr(n), ev_put(n), ev_ready(n), ev_done(n) {
  for (int r = 0; r < n; ++r) {
    cudaEventCreateWithFlags(&ev_ready[r], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_done[r], cudaEventDisableTiming);
    ev_put[r].resize(2 * 64);
    for (auto& e : ev_put[r]) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
}
LocalGroup::~LocalGroup() {
  for (int r = 0; r < ep; ++r) {
    cudaEventDestroy(ev_ready[r]);
    cudaEventDestroy(ev_done[r]);
    for (auto e : ev_put[r]) cudaEventDestroy(e);
  }
}
void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  uint64_t gen = generation;
  if (++arrived == ep) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return generation != gen; });
  }
}

static int cuda_err(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return MOE_ERR_CUDA;
}

int LocalTransport::allgather_i32(const int32_t* send, int32_t* recv, size_t count, cudaStream_t st) {
  LocalGroup& g = *g_;
  g.gather_src[rank_] = send;
  if (int e = cuda_err(cudaEventRecord(g.ev_ready[rank_], st), "cudaEventRecord")) return e;
  g.barrier();
  for (int p = 0; p < g.ep; ++p) {
    if (int e = cuda_err(cudaStreamWaitEvent(st, g.ev_ready[p], 0), "cudaStreamWaitEvent")) return e;
    if (int e = cuda_err(cudaMemcpyAsync(recv + (size_t)p * count, g.gather_src[p], count * sizeof(int32_t),
                                         cudaMemcpyDeviceToDevice, st),
                         "cudaMemcpyAsync"))
      return e;
  }
  if (int e = cuda_err(cudaEventRecord(g.ev_done[rank_], st), "cudaEventRecord")) return e;
  g.barrier();
  for (int p = 0; p < g.ep; ++p)  // sources stay untouched until every reader copied them
    if (int e = cuda_err(cudaStreamWaitEvent(st, g.ev_done[p], 0), "cudaStreamWaitEvent")) return e;
  g.barrier();
  return 0;
}

int LocalTransport::map_peers(void* mine, std::vector<char*>& out) {
  LocalGroup& g = *g_;
  g.peer_ptr[rank_] = (char*)mine;
  g.barrier();
  out = g.peer_ptr;
  g.barrier();
  return 0;
}

LocalTransport::LocalTransport(LocalGroup* g, int rank) : g_(g), rank_(rank) {
  const char* ev = std::getenv("EPSMOE_LOCAL_P2P_EVENTS");
  order_puts_ = ev ? std::atoi(ev) != 0 : true;
}

int LocalTransport::p2p_after_put(int slot, cudaStream_t ps) {
  if (!order_puts_) return 0;
  return cuda_err(cudaEventRecord(g_->ev_put[rank_][slot], ps), "cudaEventRecord");
}
int LocalTransport::p2p_before_wait(int slot0, int nslots, cudaStream_t st) {
  if (!order_puts_) return 0;  // the device flags alone order the rows
  LocalGroup& g = *g_;
  g.barrier();  // every rank has issued (recorded) these puts
  for (int p = 0; p < g.ep; ++p)
    for (int s = slot0; s < slot0 + nslots; ++s)
      if (int e = cuda_err(cudaStreamWaitEvent(st, g.ev_put[p][s], 0), "cudaStreamWaitEvent")) return e;
  g.barrier();  // nobody re-records before every rank waited
  return 0;
}

int LocalTransport::group_start(int) {
  g_->sends[rank_].clear();
  g_->recvs[rank_].clear();
  return 0;
}
int LocalTransport::send(const void* buf, size_t bytes, int peer, int channel, cudaStream_t) {
  g_->sends[rank_].push_back({buf, nullptr, bytes, peer, channel});
  return 0;
}
int LocalTransport::recv(void* buf, size_t bytes, int peer, int channel, cudaStream_t) {
  g_->recvs[rank_].push_back({nullptr, buf, bytes, peer, channel});
  return 0;
}

int LocalTransport::group_end(int channel, cudaStream_t st) {
  LocalGroup& g = *g_;
  if (int e = cuda_err(cudaEventRecord(g.ev_ready[rank_], st), "cudaEventRecord")) return e;
  g.barrier();  // every rank has posted its ops and recorded its ready event
  // What NCCL would need to complete this group instead of hanging: every op
  // on the group's communicator, and per peer as many sends to this rank as
  // this rank posts receives from it, matched in order with equal sizes.
  std::string bad;
  std::vector<size_t> sends_in(g.ep, 0), recvs_from(g.ep, 0);
  for (int p = 0; p < g.ep; ++p)
    for (const auto& op : g.sends[p]) {
      if (op.channel != channel) bad = "send on another communicator in this group";
      if (op.peer == rank_) ++sends_in[p];
    }
  for (const auto& rv : g.recvs[rank_]) {
    if (rv.channel != channel) bad = "recv on another communicator in this group";
    ++recvs_from[rv.peer];
  }
  for (int p = 0; p < g.ep && bad.empty(); ++p)
    if (sends_in[p] != recvs_from[p])
      bad = std::to_string(sends_in[p]) + " sends from rank " + std::to_string(p) + " but " +
            std::to_string(recvs_from[p]) + " recvs";
  std::vector<size_t> next(g.ep, 0);
  for (const auto& rv : g.recvs[rank_]) {
    if (!bad.empty()) break;
    // k-th recv from peer p matches p's k-th send to this rank (NCCL p2p order)
    const auto& ps = g.sends[rv.peer];
    size_t& i = next[rv.peer];
    while (i < ps.size() && ps[i].peer != rank_) ++i;
    if (i >= ps.size() || ps[i].bytes != rv.bytes) {
      bad = "unmatched recv from rank " + std::to_string(rv.peer);
      break;
    }
    ++i;
  }
  if (!bad.empty()) {
    set_error("local transport (NCCL p2p contract): " + bad);
    g.barrier();
    g.barrier();
    return MOE_ERR_MISMATCH;
  }
  std::fill(next.begin(), next.end(), 0);
  for (const auto& rv : g.recvs[rank_]) {
    const auto& ps = g.sends[rv.peer];
    size_t& i = next[rv.peer];
    while (ps[i].peer != rank_) ++i;
    if (int e = cuda_err(cudaStreamWaitEvent(st, g.ev_ready[rv.peer], 0), "cudaStreamWaitEvent")) return e;
    if (int e = cuda_err(cudaMemcpyAsync(rv.dst, ps[i].src, rv.bytes, cudaMemcpyDeviceToDevice, st),
                         "cudaMemcpyAsync"))
      return e;
    ++i;
  }
  if (int e = cuda_err(cudaEventRecord(g.ev_done[rank_], st), "cudaEventRecord")) return e;
  g.barrier();  // all copies enqueued
  for (int p = 0; p < g.ep; ++p)  // a sender's buffer is reusable once its readers copied it
    if (int e = cuda_err(cudaStreamWaitEvent(st, g.ev_done[p], 0), "cudaStreamWaitEvent")) return e;
  g.barrier();  // nobody re-records ev_done before every rank waited on it
  return 0;
}

}  // namespace epsmoe
