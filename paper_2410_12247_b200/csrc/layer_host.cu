// Host-buffer entry points: moe_layer_forward_host / _async / moe_layer_host_sync
// (H2D copy -> layer -> D2H copy on three streams, double-buffered staging).
#include "layer_impl.h"

using namespace epsmoe;

// Token-slice schedule of moe_layer_forward_host: relative slice sizes chosen
// from a small family by simulating the three-stream pipeline (H2D copy ->
// layer -> D2H copy, each stream in order) with a model of this config:
// PCIe ~50 GB/s each way; layer time per token from its FLOPs at ~1.25 PF/s,
// inflated by the 256-row tile padding of a slice's rows per expert, plus a
// fixed ~0.3 ms per forward.  A function of the config only, so every rank
// (each slice is a collective when ep > 1) derives the same schedule.
static std::vector<double> host_slice_schedule(const moe_config_t& c, bool overlapped) {
  // Overlapped calls (async) run the copy streams ahead across calls: a call
  // then costs its busiest stream and slicing only shortens the one-off fill and
  // drain while inflating the GEMMs' tile padding, so one slice (measured: DSv2
  // e2e 23.6 ms per call over 8 calls unsliced vs 24.9-26.8 sliced; Mixtral 8.7
  // vs 9.1-11.1).
  if (overlapped) return {1.0};
  const double T = (double)c.max_tokens, H = c.hidden, F = c.ffn, k = c.top_k, E = c.num_experts;
  const double SF = (double)c.num_shared * c.shared_ffn;
  const double copy_tok = 2.0 * H / 50e9;
  const double flop_tok = 6.0 * H * F * k + 6.0 * H * SF + 2.0 * H * E;
  auto layer_time = [&](double n) {
    const double rows = n * k * c.ep / E;  // rows per local expert (uniform routing)
    const double eff = rows > 0 ? rows / (std::ceil(rows / 256.0) * 256.0) : 1.0;
    return n * flop_tok / 1.25e15 / eff + 3e-4;
  };
  static const std::vector<std::vector<double>> family = {
      {1}, {1, 1}, {1, 1, 1, 1}, {1, 2, 2, 1}, {1, 2, 3, 2}, {1, 3, 3, 1}, {1, 2, 3, 2, 1}, {1, 2, 4, 4, 2, 1},
      {1, 2, 3, 3, 3, 2, 1}, {1, 1, 1, 1, 1, 1, 1, 1}};
  std::vector<double> best = family[0];
  double best_t = 1e30;
  for (const auto& w : family) {
    double wsum = 0;
    for (double v : w) wsum += v;
    double h_end = 0, c_end = 0, d_end = 0;
    for (double v : w) {
      const double n = T * v / wsum;
      h_end += n * copy_tok;
      c_end = std::max(c_end, h_end) + layer_time(n);
      d_end = std::max(d_end, c_end) + n * copy_tok;
    }
    if (d_end < best_t * 0.99) { best_t = d_end; best = w; }  // a larger family member must win by > 1%
  }
  return best;
}

namespace {
// One host-buffer call: token slices of x_host -> staging buffer b (s_h2d) ->
// layer (st) -> y_host (s_d2h), each stream in order, event-chained per slice.
// The staging pair alternates between calls, so a call's copies overlap the
// previous call's compute; buffer b is reused only after the call two back
// consumed (x) and drained (y) it.
moe_status_t host_call(moe_layer* L, const void* x_host, int64_t T, void* y_host, const moe_plan_t* plan,
                       void* stream_v, bool overlapped) {
  if (!L || T < 0 || T > L->cfg.max_tokens) { set_error("bad argument"); return MOE_ERR_INVALID; }
  cudaStream_t st = (cudaStream_t)stream_v;
  const int64_t row = (int64_t)L->cfg.hidden * 2;
  // y_t depends only on x_t: slices of the batch pipeline the
  // copies against the layer.  The schedule is a function of the config only
  // (identical on every rank: each slice's forward is a collective when ep > 1).
  // EPSMOE_HOST_SLICES="w0,w1,..." (<= 8 relative weights) overrides it.
  std::vector<double> wts;
  if (const char* hs = std::getenv("EPSMOE_HOST_SLICES")) {
    for (const char* p = hs; *p && (int)wts.size() < moe_layer::MAX_HOST_SLICES;) {
      char* end = nullptr;
      double v = std::strtod(p, &end);
      if (end == p) break;
      if (v > 0) wts.push_back(v);
      p = (*end == ',') ? end + 1 : end;
    }
  }
  // The first async call after a sync has no earlier compute to hide its H2D
  // behind: it takes the standalone call's slicing (ep == 1 only, where no
  // other rank must agree on the number of forwards); y_t depends only on x_t,
  // so the slices give the same bits (test_forward_host_async_overlapped_calls).
  if (wts.empty())
    wts = host_slice_schedule(L->cfg, overlapped && (L->host_inflight || L->cfg.ep > 1));
  const int S = (int)wts.size();
  std::vector<int64_t> bound(S + 1, 0);
  double wsum = 0, acc = 0;
  for (double v : wts) wsum += v;
  for (int s = 0; s < S; ++s) {
    acc += wts[s];
    bound[s + 1] = (s + 1 == S) ? T : std::min<int64_t>(T, (int64_t)std::llround(T * acc / wsum));
  }
  if (!L->staging) {  // first host-buffer call: the double-buffered x / y staging
    const size_t one = (size_t)L->cfg.max_tokens * row;
    CUDA_TRY(cudaMalloc(&L->staging, 4 * one));
    for (int i = 0; i < 2; ++i) {
      L->x_dev[i] = static_cast<char*>(L->staging) + (2 * i) * one;
      L->y_dev[i] = static_cast<char*>(L->staging) + (2 * i + 1) * one;
    }
  }
  const int b = L->hb;
  L->hb ^= 1;
  CUDA_TRY(cudaStreamWaitEvent(L->s_h2d, L->ev_xfree[b], 0));  // x staging b read by the call two back
  CUDA_TRY(cudaStreamWaitEvent(st, L->ev_yfree[b], 0));        // y staging b copied out by the call two back
  for (int s = 0; s < S; ++s) {
    const int64_t t0 = bound[s], n = bound[s + 1] - t0;
    char* xd = (char*)L->x_dev[b] + t0 * row;
    char* yd = (char*)L->y_dev[b] + t0 * row;
    if (n) CUDA_TRY(cudaMemcpyAsync(xd, (const char*)x_host + t0 * row, n * row, cudaMemcpyHostToDevice, L->s_h2d));
    CUDA_TRY(cudaEventRecord(L->ev_in[s], L->s_h2d));
    CUDA_TRY(cudaStreamWaitEvent(st, L->ev_in[s], 0));
    moe_status_t rs = moe_layer_forward(L, xd, n, yd, plan, stream_v, nullptr);
    if (rs) return rs;
    CUDA_TRY(cudaEventRecord(L->ev_out[s], st));
    CUDA_TRY(cudaStreamWaitEvent(L->s_d2h, L->ev_out[s], 0));
    if (n) CUDA_TRY(cudaMemcpyAsync((char*)y_host + t0 * row, yd, n * row, cudaMemcpyDeviceToHost, L->s_d2h));
  }
  CUDA_TRY(cudaEventRecord(L->ev_xfree[b], st));
  CUDA_TRY(cudaEventRecord(L->ev_yfree[b], L->s_d2h));
  if (overlapped) L->host_inflight = true;
  if (!overlapped) {
    CUDA_TRY(cudaStreamSynchronize(L->s_d2h));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  return MOE_OK;
}
}  // namespace

extern "C" {

moe_status_t moe_layer_forward_host(moe_layer_t* L, const void* x_host, int64_t T, void* y_host,
                                    const moe_plan_t* plan, void* stream_v) {
  return host_call(L, x_host, T, y_host, plan, stream_v, false);
}

moe_status_t moe_layer_forward_host_async(moe_layer_t* L, const void* x_host, int64_t T, void* y_host,
                                          const moe_plan_t* plan, void* stream_v) {
  return host_call(L, x_host, T, y_host, plan, stream_v, true);
}

moe_status_t moe_layer_host_sync(moe_layer_t* L, void* stream_v) {
  if (!L) { set_error("null layer"); return MOE_ERR_INVALID; }
  CUDA_TRY(cudaStreamSynchronize(L->s_d2h));
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream_v));
  L->host_inflight = false;
  return MOE_OK;
}

}  // extern "C"
