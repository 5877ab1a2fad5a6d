// The measured B200 cost model behind the expert pipeline scheduler
// (moe_layer_calibrate) and the GEMM test hook (moe_gemm_grouped).
#include "layer_impl.h"

using namespace epsmoe;

extern "C" {

moe_status_t moe_gemm_grouped(int32_t epi, const void* A, int64_t a_rows, const void* B0, const void* B1,
                              int64_t b_rows, int32_t b_group_rows, int32_t kdim, int32_t n, void* out, int64_t ldo,
                              const float* bias, int32_t groups, const int32_t* row_start, const int32_t* row_count,
                              int32_t num_ctas, int32_t tile_m, void* stream) {
  if (epi < 0 || epi > 2 || !A || !B0 || (epi == 0 && !B1) || !out || groups < 1 || !row_start || !row_count) {
    set_error("moe_gemm_grouped: bad argument");
    return MOE_ERR_INVALID;
  }
  GemmArgs a = base_args(epi, num_ctas > 0 ? num_ctas : 148);
  if (tile_m != 128 && tile_m != 256) { set_error("moe_gemm_grouped: tile_m must be 128 or 256"); return MOE_ERR_INVALID; }
  a.cta_pair = tile_m == 256;
  a.A = A;
  a.a_rows = a_rows;
  a.B0 = B0;
  a.B1 = B1;
  a.b_rows = b_rows;
  a.b_group_rows = b_group_rows;
  a.K = kdim;
  a.N = n;
  a.out = out;
  a.ldo = ldo;
  a.bias = bias;
  a.G = groups;
  a.row_start = row_start;
  a.row_count = row_count;
  a.rows_hint = (double)a_rows / groups;  // raster choice (the counts are on the device)
  int e = gemm_launch(a, (cudaStream_t)stream);
  if (e) { set_error(std::string("gemm: ") + cudaGetErrorString((cudaError_t)e)); return MOE_ERR_CUDA; }
  return MOE_OK;
}

moe_status_t moe_layer_calibrate(moe_layer_t* L, void* stream, moe_cost_model_t* out) {
  if (!L) return MOE_ERR_INVALID;
  // Measured GEMM time per expert vs rows, both kinds (X2/X3 analog on B200).
  const moe_config_t& c = L->cfg;
  cudaStream_t st = (cudaStream_t)stream;
  moe_cost_model_t m = L->cost;
  const int G = std::min(L->E_loc, 8);
  const float pts[MOE_COST_POINTS] = {16, 64, 128, 256, 512, 1024, 2048, 3072, 4096, 6144, 8192, 16384};
  struct Ev {  // destroyed on every exit path
    cudaEvent_t e = nullptr;
    ~Ev() { if (e) cudaEventDestroy(e); }
  } ev0, ev1;
  CUDA_TRY(cudaEventCreate(&ev0.e));
  CUDA_TRY(cudaEventCreate(&ev1.e));
  cudaEvent_t e0 = ev0.e, e1 = ev1.e;
  std::vector<int32_t> hs(2 * MOE_MAX_EXPERTS);
  int np = 0;
  for (int i = 0; i < MOE_COST_POINTS; ++i) {
    int64_t rows = (int64_t)pts[i];
    if (rows * G > L->gemm_rows_cap) break;
    for (int g = 0; g < G; ++g) { hs[g] = (int32_t)(g * rows); hs[MOE_MAX_EXPERTS + g] = (int32_t)rows; }
    CUDA_TRY(cudaMemcpy(L->recv_start_d, hs.data(), sizeof(int32_t) * G, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(L->recv_count_d, hs.data() + MOE_MAX_EXPERTS, sizeof(int32_t) * G, cudaMemcpyHostToDevice));
    const void* A = L->recv ? L->recv : L->send;
    int64_t arows = L->recv ? L->recv_cap : L->send_cap;
    for (int kind = 1; kind <= 2; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        CUDA_TRY(cudaEventRecord(e0, st));
        int err = compute_moe(L, A, arows, L->recv_start_d, L->recv_count_d, 0, G, kind, L->num_sms,
                              rows >= 512 ? 1 : 0, false, rows, st);
        if (err) { set_error("calibrate gemm failed"); return MOE_ERR_CUDA; }
        CUDA_TRY(cudaEventRecord(e1, st));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      m.gemm_ms[kind - 1][i] = best / G;
    }
    m.m_points[i] = pts[i];
    np = i + 1;
  }
  // too little capacity for even the smallest point: keep the previous GEMM table
  // (a model without points would price every GEMM at zero)
  if (np == 0) {
    std::memcpy(m.m_points, L->cost.m_points, sizeof(m.m_points));
    std::memcpy(m.gemm_ms, L->cost.gemm_ms, sizeof(m.gemm_ms));
    np = L->cost.n_points;
  }
  m.n_points = np;
  // SM partition (NEXT-1, Table IV analog P:467-490): the expert GEMMs of G
  // experts x `rows` rows on num_sms - 2 * cc SMs vs all SMs, for the comm
  // budgets cc the planner may choose
  const int cands[MOE_COMM_POINTS] = {4, 8, 12, 16};
  m.num_sms = L->num_sms;
  {
    int64_t rows = 2048;
    while (rows > 16 && rows * G > L->gemm_rows_cap) rows /= 2;
    for (int g = 0; g < G; ++g) { hs[g] = (int32_t)(g * rows); hs[MOE_MAX_EXPERTS + g] = (int32_t)rows; }
    CUDA_TRY(cudaMemcpy(L->recv_start_d, hs.data(), sizeof(int32_t) * G, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(L->recv_count_d, hs.data() + MOE_MAX_EXPERTS, sizeof(int32_t) * G, cudaMemcpyHostToDevice));
    const void* A = L->recv ? L->recv : L->send;
    const int64_t arows = L->recv ? L->recv_cap : L->send_cap;
    auto time_grid = [&](int grid, float* best) -> moe_status_t {
      *best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        CUDA_TRY(cudaEventRecord(e0, st));
        int err = compute_moe(L, A, arows, L->recv_start_d, L->recv_count_d, 0, G, MOE_GEMM_GROUPED, grid,
                              rows >= 512 ? 1 : 0, false, (double)rows, st);
        if (err) { set_error("calibrate gemm failed"); return MOE_ERR_CUDA; }
        CUDA_TRY(cudaEventRecord(e1, st));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        *best = std::min(*best, ms);
      }
      return MOE_OK;
    };
    float t_all = 0.f;
    CUDA_TRY_STATUS(time_grid(L->num_sms, &t_all));
    m.n_comm = MOE_COMM_POINTS;
    for (int i = 0; i < MOE_COMM_POINTS; ++i) {
      float t = 0.f;
      CUDA_TRY_STATUS(time_grid(L->num_sms - 2 * cands[i], &t));
      m.comm_ctas[i] = cands[i];
      m.gemm_scale_at[i] = t_all > 0.f ? std::max(1.0f, t / t_all) : 1.0f;
      m.a2a_gbps_at[i] = m.a2a_gbps;
    }
  }
  if (c.ep > 1) {
    // All2all cost per comm budget: every rank sends `per` bytes to every
    // peer on the layer's own data plane; time vs the bytes crossing one rank
    // gives a2a_fixed_ms + 1 / GB/s (least squares over the sizes).
    const int D = c.ep;
    const int64_t cap = std::min<int64_t>(L->send_cap, L->recv_cap) * c.hidden * 2 / D;
    const int nb = (c.a2a_p2p == 2) ? 1 : MOE_COMM_POINTS;  // copy engines: no SM budget to choose
    double fixed_sum = 0.0;
    int fixed_n = 0;
    for (int i = 0; i < nb; ++i) {
      std::vector<double> xs, ys;
      for (int64_t per : {int64_t(1) << 21, int64_t(1) << 23, int64_t(1) << 25}) {
        if (per > cap) break;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
          float ms = 0.f;
          CUDA_TRY_STATUS(time_all2all(L, cands[i], per, st, e0, e1, &ms));
          best = std::min(best, ms);
        }
        xs.push_back((double)per * (D - 1));
        ys.push_back(best);
      }
      if (xs.size() >= 2) {  // least squares: ms = a + x / (gbps * 1e6)
        double sx = 0, sy = 0, sxx = 0, sxy = 0;
        const double n = (double)xs.size();
        for (size_t q = 0; q < xs.size(); ++q) {
          sx += xs[q]; sy += ys[q]; sxx += xs[q] * xs[q]; sxy += xs[q] * ys[q];
        }
        const double slope = (n * sxy - sx * sy) / std::max(1e-30, n * sxx - sx * sx);
        const double icpt = (sy - slope * sx) / n;
        if (slope > 0) m.a2a_gbps_at[i] = (float)(1.0 / (slope * 1e6));
        fixed_sum += std::max(0.002, icpt);
        ++fixed_n;
      } else if (xs.size() == 1 && ys[0] > 0) {
        m.a2a_gbps_at[i] = (float)(xs[0] / (ys[0] * 1e6));
      }
    }
    if (c.a2a_p2p == 2) {
      m.n_comm = 1;
      m.comm_ctas[0] = 0;
      m.gemm_scale_at[0] = 1.0f;
    }
    m.a2a_gbps = m.a2a_gbps_at[0];
    for (int i = 1; i < nb; ++i) m.a2a_gbps = std::max(m.a2a_gbps, m.a2a_gbps_at[i]);
    if (fixed_n) {
      m.a2a_fixed_ms = (float)(fixed_sum / fixed_n);
      m.k_ms = 2.0f * m.a2a_fixed_ms;  // a chunk adds one dispatch and one combine group
    }
    // back to the layer's own budget on the NCCL plane
    TR_TRY(L->tr->set_comm_ctas(L->comm_ctas));
    // every rank must plan identically: adopt rank 0's model
    constexpr int W = (int)(sizeof(moe_cost_model_t) / sizeof(int32_t));
    int32_t* dev = nullptr;
    CUDA_TRY(cudaMalloc(&dev, sizeof(int32_t) * W * (D + 1)));
    CUDA_TRY(cudaMemcpy(dev, &m, sizeof(m), cudaMemcpyHostToDevice));
    int ge = L->tr->allgather_i32(dev, dev + W, W, st);
    if (!ge) {
      CUDA_TRY(cudaStreamSynchronize(st));
      CUDA_TRY(cudaMemcpy(&m, dev + W, sizeof(m), cudaMemcpyDeviceToHost));  // rank 0's record
    }
    cudaFree(dev);
    if (ge) return (moe_status_t)ge;
  }
  L->cost = m;
  if (out) *out = m;
  return MOE_OK;
}

}  // extern "C"
