// All2all transport behind the EP layer.
//
//   HostCollTransport — counts over a caller-supplied host allgather, rows
//                    over the layer's own peer-memory planes only.
//   NcclTransport  — production: two NCCL communicators over NVLink (channel 0 =
//                    dispatch, channel 1 = combine) so both phases can be in
//                    flight; grouped ncclSend/ncclRecv; ncclAllGather of counts.
//   LocalTransport — test transport: the ep ranks are ep layer objects in ONE
//                    process on ONE GPU, each driven by its own host thread.
//                    Every group end is a host rendezvous; each posted recv is
//                    matched to the peer's send (same order) and executed as a
//                    device-to-device cudaMemcpyAsync on the receiver's stream,
//                    event-chained to the sender.  It lets the very same EP
//                    forward code (tables, chunk DAG, events) run on one B200.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

#include "../../include/epsmoe.h"

namespace epsmoe {

class Transport {
 public:
  virtual ~Transport() = default;
  // recv[r * count + i] = send_of_rank_r[i]; stream-ordered on `st`.
  virtual int allgather_i32(const int32_t* send, int32_t* recv, size_t count, cudaStream_t st) = 0;
  virtual int group_start(int channel) = 0;
  virtual int send(const void* buf, size_t bytes, int peer, int channel, cudaStream_t st) = 0;
  virtual int recv(void* buf, size_t bytes, int peer, int channel, cudaStream_t st) = 0;
  virtual int group_end(int channel, cudaStream_t st) = 0;
  virtual const char* name() const = 0;
  // Collective: every rank's `mine` (a device allocation of identical layout on
  // every rank) mapped into this process; out[rank] = mine.  For the put-kernel
  // all2all (a2a_p2p).
  virtual int map_peers(void* mine, std::vector<char*>& out) = 0;
  // a2a_p2p hooks around the device flags (no-ops across processes).  The
  // in-process test group shares one GPU's hardware queues between ranks, so a
  // rank's spinning flag-wait kernel could sit in front of the put kernel it
  // waits for; there the put is also ordered by a CUDA event.
  virtual int p2p_after_put(int slot, cudaStream_t) { (void)slot; return 0; }
  virtual int p2p_before_wait(int slot0, int nslots, cudaStream_t) { (void)slot0; (void)nslots; return 0; }
  // SM budget of the send/recv kernels (NCCL maxCTAs per communicator, the
  // paper's comm-SM control P:202-209, NEXT-1).  Collective: every rank passes
  // the same value in the same forward (plans agree).  0 = keep.
  virtual int set_comm_ctas(int ctas) { (void)ctas; return 0; }
  // Asynchronous errors of the collectives (ncclCommGetAsyncError); polled
  // while the host waits for the count exchange.  0 = none.
  virtual int poll_async() { return 0; }
};


class NcclTransport : public Transport {
 public:
  NcclTransport(ncclComm_t d, ncclComm_t c, int ctas) : comm_{d, c}, base_{d, c}, ctas_(ctas) {}
  ~NcclTransport() override;
  int set_comm_ctas(int ctas) override;
  int poll_async() override;
  int allgather_i32(const int32_t* send, int32_t* recv, size_t count, cudaStream_t st) override;
  int group_start(int channel) override;
  int send(const void* buf, size_t bytes, int peer, int channel, cudaStream_t st) override;
  int recv(void* buf, size_t bytes, int peer, int channel, cudaStream_t st) override;
  int group_end(int channel, cudaStream_t st) override;
  const char* name() const override { return "nccl"; }
  // cudaIpc handles of the allocations holding `mine` (+ offset), allgathered
  // over communicator 0 and opened with peer access.
  int map_peers(void* mine, std::vector<char*>& out) override;

 private:
  ncclComm_t comm_[2];         // in use
  ncclComm_t base_[2];         // created with the layer's initial maxCTAs
  int ctas_;                   // maxCTAs of comm_
  struct Split { int ctas; ncclComm_t c[2]; };
  std::vector<Split> splits_;  // ncclCommSplit copies with other maxCTAs (NEXT-1), kept for reuse
  std::vector<void*> opened_;  // cudaIpcOpenMemHandle results, closed on destruction
};

// Host-collective transport (moe_layer_create_hostcoll): the caller's blocking
// host allgather (e.g. torch.distributed over gloo) carries the count
// exchange and the one-time peer mapping; routed rows move only on the
// layer's own peer-memory planes (a2a_p2p = 1 or 2), so send / recv are
// unsupported.  One process per rank; the ranks may share one GPU (tests:
// separate contexts, real cudaIpc mappings and device flags, no host
// ordering of the puts) or be one GPU each.
class HostCollTransport : public Transport {
 public:
  HostCollTransport(moe_host_allgather_fn fn, void* ctx, int ep, int rank) : fn_(fn), ctx_(ctx), ep_(ep), rank_(rank) {}
  ~HostCollTransport() override;
  int allgather_i32(const int32_t* send, int32_t* recv, size_t count, cudaStream_t st) override;
  int group_start(int) override { return unsupported(); }
  int send(const void*, size_t, int, int, cudaStream_t) override { return unsupported(); }
  int recv(void*, size_t, int, int, cudaStream_t) override { return unsupported(); }
  int group_end(int, cudaStream_t) override { return unsupported(); }
  const char* name() const override { return "hostcoll"; }
  int map_peers(void* mine, std::vector<char*>& out) override;

 private:
  int unsupported();
  int gather_host(const void* send, void* recv, size_t bytes);
  moe_host_allgather_fn fn_;
  void* ctx_;
  int ep_, rank_;
  std::vector<void*> opened_;
};

// Shared rendezvous state of the ep local ranks (moe_local_group_create).
struct LocalGroup {
  explicit LocalGroup(int ep);
  ~LocalGroup();
  void barrier();
  struct Op {
    const void* src;
    void* dst;
    size_t bytes;
    int peer;
    int channel;  // communicator (0 dispatch, 1 combine): NCCL matches p2p per communicator
  };
  int ep;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<std::vector<Op>> sends, recvs;  // [rank] ops posted in the current group
  std::vector<const void*> gather_src;        // [rank] allgather source pointers
  std::vector<char*> peer_ptr;                // [rank] map_peers slots
  std::vector<std::vector<cudaEvent_t>> ev_put;  // [rank][slot] a2a_p2p put completions
  std::vector<cudaEvent_t> ev_ready, ev_done; // [rank]
};

class LocalTransport : public Transport {
 public:
  // order_puts: p2p_before_wait also orders the peers' puts before the wait by
  // CUDA events (default; EPSMOE_LOCAL_P2P_EVENTS=0 turns it off).  The ranks'
  // streams share one context's hardware queues, and with more streams than
  // queues (CUDA_DEVICE_MAX_CONNECTIONS, default 8) a spinning flag wait can
  // sit in front of the put it waits for: measured, a 2-rank copy-engine
  // forward hung until the wait kernel's 10 s trap.  Off (with <= 32 streams
  // and CUDA_DEVICE_MAX_CONNECTIONS=32), the device flags alone order the data,
  // as across processes (moe_layer_create_hostcoll), where contexts never share
  // a queue.
  LocalTransport(LocalGroup* g, int rank);
  int allgather_i32(const int32_t* send, int32_t* recv, size_t count, cudaStream_t st) override;
  int group_start(int channel) override;
  int send(const void* buf, size_t bytes, int peer, int channel, cudaStream_t st) override;
  int recv(void* buf, size_t bytes, int peer, int channel, cudaStream_t st) override;
  int group_end(int channel, cudaStream_t st) override;
  const char* name() const override { return "local"; }
  int map_peers(void* mine, std::vector<char*>& out) override;  // same device: the pointers themselves
  int p2p_after_put(int slot, cudaStream_t ps) override;
  int p2p_before_wait(int slot0, int nslots, cudaStream_t st) override;

 private:
  LocalGroup* g_;
  int rank_;
  bool order_puts_ = true;
};

}  // namespace epsmoe
