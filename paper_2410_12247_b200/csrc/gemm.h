// Internal interface of the tcgen05 grouped / dense GEMM (gemm_sm100.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace epsmoe {

enum EpiKind : int {
  EPI_SWIGLU = 0,  // acc = [gate(128) | up(128)] -> h = bf16(silu(g) * u)   (GateUpGemm+SiluAct)
  EPI_BF16 = 1,    // acc -> bf16                                             (DownGemm)
  EPI_F32 = 2,     // acc (+ bias[col]) -> fp32                               (Router)
  EPI_COMBINE = 3, // shared DownGemm fused with K7: s = bf16(acc);
                   // y = bf16(fmaf chain over slots j of w_j * o[pos[t][j]] on fp32(s))
};

// Output scatter of a DownGemm fused with the combine all2all (a2a_p2p): GEMM
// rows [r0, r0 + n) go to consecutive rows starting at dst (bf16, row pitch
// ldo), typically another rank's combine buffer in mapped peer memory.
struct GemmRowSeg {
  int64_t r0, n;
  char* dst;
};

// One grouped GEMM launch: for each group g (an expert), rows
// [row_start[g], row_start[g] + row_count[g]) of A (K-major, [rows, K] bf16)
// times B_g^T where B_g = rows [(b_base + g) * b_group_rows, ...) of B
// ([*, K] bf16, K-major).  Output rows are the same rows of `out`.
struct GemmArgs {
  int epi;                 // EpiKind
  const void* A;           // [a_rows, K] bf16
  int64_t a_rows;          // allocated rows of A (TMA bound)
  const void* B0;          // [b_rows, K] bf16 (gate for SWIGLU)
  const void* B1;          // [b_rows, K] bf16 (up for SWIGLU) or nullptr
  int64_t b_rows;          // allocated rows of B0/B1
  int b_group_rows;        // rows of B per group (F for gate/up, H for down, 0 = shared)
  int b_base;              // first group's index into B
  int K;                   // reduction length (multiple of 64)
  int N;                   // logical output columns (F for SWIGLU)
  void* out;               // bf16 or fp32
  int64_t ldo;             // output row pitch in elements
  int64_t out_rows;        // allocated rows of `out` (TMA store bound; 0 = a_rows)
  const float* bias;       // EPI_F32 only, [N] or nullptr
  int G;                   // groups (<= 256)
  const int32_t* row_start;  // device [G] (nullptr -> single group at row 0)
  const int32_t* row_count;  // device [G] (nullptr -> single group of m_single rows)
  int m_single;
  int num_ctas;            // persistent grid size (SM budget)
  int cta_pair;            // 1: 256-row tiles on CTA pairs (cta_group::2); 0: 128-row tiles
  const int32_t* a_row_index;  // optional gather: logical A row r is physical row a_row_index[r] of A
                               // (16-B cp.async into the swizzled stage; EPI_SWIGLU only).  nullptr = contiguous A.
  int32_t* tile_counter;       // device int32[2], zero-initialised, for dynamic tile tickets; launches
                               // that may run concurrently need distinct counters (nullptr = shared)
  int row_mode;                // 0: all rows of each group; 1: only the first floor(n/256)*256 rows
                               // (bulk); 2: only the rows after them (remainder, < 256)
  // EPI_COMBINE only (single dense group, row = token t): routed expert outputs
  // o [*, N] bf16, pos [rows, comb_k] int32 rows of o, w [rows, comb_k] fp32.
  const void* comb_o;
  const int32_t* comb_pos;
  const float* comb_w;
  int comb_k;                  // 1..8
  double rows_hint;            // expected rows per group (0 = unknown): picks the tile raster
  // EPI_BF16 only: scatter the output rows (device table sorted by r0; rows in
  // no segment are dropped) and, once every CTA's stores are system-visible,
  // set *sig_flags[i] = sig_epoch (i < nsig) from the last CTA.
  const GemmRowSeg* rseg;
  int nrseg;
  uint32_t* const* sig_flags;
  int nsig;
  uint32_t sig_epoch;
  // optional SM-partition probe (device int32[2]): each CTA adds itself to [0]
  // while resident and records the running maximum in [1]
  int32_t* resident;
};

// Launch on `stream`.  Returns a cudaError_t-compatible code (0 = success).
int gemm_launch(const GemmArgs& a, cudaStream_t stream);

}  // namespace epsmoe
