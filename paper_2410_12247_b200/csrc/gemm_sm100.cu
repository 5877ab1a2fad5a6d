// Expert FFN GEMMs on 5th-gen tensor cores (sm_100a): persistent, warp-
// specialised, TMA -> smem ring -> tcgen05.mma (bf16 in / fp32 accumulate in
// TMEM) -> double-buffered TMEM accumulators -> fused epilogue.
//
// Two tile shapes (template CG):
//   CG = 1: one CTA per 128x256 tile, cta_group::1, 4 x 48 KB stages.
//   CG = 2: a CTA pair (cluster of 2) per 256x256 tile, cta_group::2: each CTA
//           TMA-loads its 128 rows of A and half (128 rows) of B, the leader
//           CTA issues M=256 MMAs that read both CTAs' smem and write each
//           CTA's own TMEM; 6 x 32 KB stages per CTA.  Per MAC this halves B's
//           smem/L2 traffic.
//
// One kernel family serves every GEMM of the layer:
//   GateUpGemm + SiluAct  EPI_SWIGLU: the 256 accumulator columns
//        are 128 rows of W_gate and 128 rows of W_up of one expert (two TMA
//        boxes; no weight repacking); epilogue h = bf16(silu(g) * u).
//   DownGemm                  EPI_BF16:  o = bf16(acc).
//   Router                    EPI_F32:   logits = fp32(acc) + beta.
//   shared DownGemm + K7 combine      EPI_COMBINE: s = bf16(acc), then the
//        weighted unpermute y = bf16(fmaf_j(w_j, o[pos[t][j]], fp32(s))) in slot
//        order (R4) while the tensor core computes the next tile: the combine's
//        HBM stream hides under a compute-bound GEMM instead of running alone.
//
// Tile scheduling: tiles are numbered group-major (expert), then in blocks of
// RASTER m-tiles (n-major across a block) so that tiles in flight together
// share A rows and B columns in L2.  By default tiles are handed out
// dynamically: the leader CTA's producer takes the next ticket from a global
// atomic counter and broadcasts it (smem queue + mbarriers; DSMEM to the peer
// CTA), so the tiles processed at any moment stay contiguous in the order
// even when units drift — which keeps their shared operands L2-resident.
// Group row counts are read from device memory: no host round trip sizes the
// launch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm.h"
#include "ptx.cuh"

namespace epsmoe {
namespace {

constexpr int BM = 128;         // rows per CTA
constexpr int BN = 256;         // accumulator columns per tile
constexpr int BK = 64;          // K per stage (one 128 B swizzle atom of bf16)
constexpr int MAX_G = 256;
constexpr int NUM_THREADS = 192;  // w0 TMA, w1 MMA + TMEM owner, w2..5 epilogue
constexpr int TMEM_COLS = 512;    // 2 x 256-column fp32 accumulators
#ifndef EPSMOE_TQ
#define EPSMOE_TQ 4
#endif
constexpr int TQ = EPSMOE_TQ;     // tile-ticket queue depth

template <int CG>
struct Cfg {
  static constexpr int TILE_M = BM * CG;
  static constexpr int B_ROWS = BN / CG;              // B rows each CTA loads per stage
  static constexpr int A_BYTES = BM * BK * 2;         // 16 KB
  static constexpr int B_BYTES = B_ROWS * BK * 2;     // 32 KB (CG=1) / 16 KB (CG=2)
  static constexpr int STAGES = (CG == 1) ? 4 : 6;
  // consumers of a ticket that must release it before the slot is refilled:
  // MMA (1) + own epilogue warps (4) [+ peer producer (1) + peer epilogue (4)]
  static constexpr int TQ_CONSUMERS = (CG == 1) ? 5 : 10;
};

struct KParams {
  int K, N, G, m_single, b_group_rows, b_base;
  int raster_gm;  // tile order inside a group: blocks of raster_gm m-tiles, m fastest inside a block
  int dynamic;    // 1: dynamic tile tickets (tile_counter), 0: static round robin
  int ticket_ahead;  // dynamic: the leader publishes the next tile before loading the current one
  int row_mode;   // 0 all rows, 1 bulk (multiple of 256), 2 remainder (see GemmArgs)
  int diag;       // diagnostics only (EPSMOE_GEMM_DIAG): 1 skip output stores, 2 skip TMEM loads + stores,
                  // 3 bulk stores into a 256-row window (L2-resident: same store traffic, no DRAM writes)
  int tma_store;  // bf16 outputs: full 32-row warp slices leave through TMA bulk-tensor stores (tmO)
  int half_tiles;
  int n_mma;       // MMA N: BN, or for EPI_F32 (the router, N = E) E rounded up to 16 - no 256-column padding  // CTA pairs: a group's last m-tile with <= 128 rows runs as an M = 128 2-CTA MMA (see kernel)
  int64_t ldo;
  void* out;
  const float* bias;
  const int32_t* row_start;
  const int32_t* row_count;
  const int32_t* a_row_index;
  const uint8_t* a_ptr;   // GATHER: A base (row pitch K * 2 bytes)
  int32_t* tile_counter;  // [2]: next ticket, CTAs finished (reset by the last CTA)
  const GemmRowSeg* rseg;       // EPI_BF16 output scatter (see GemmArgs)
  int nrseg;
  uint32_t* const* sig_flags;
  int nsig;
  uint32_t sig_epoch;
  const __nv_bfloat16* comb_o;  // EPI_COMBINE (see GemmArgs)
  const int32_t* comb_pos;
  const float* comb_w;
  int comb_k;
  int32_t* resident;  // SM-partition probe (GemmArgs::resident) or nullptr
};

constexpr int COMB_MAX_K = 8;

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// o rows are read once: L2 evict-first, L1-allocating (a lane's four 16-B
// pieces share two 32-B sectors)
__device__ __forceinline__ uint4 ld_once(const void* ptr, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr), "l"(pol));
  return r;
}
__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

template <int CG>
struct __align__(8) SmemTail {
  uint64_t full[Cfg<CG>::STAGES];
  uint64_t empty[Cfg<CG>::STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t gfull[Cfg<CG>::STAGES];  // GATHER, peer CTA: its A copies landed (forwarded to the leader)
  uint64_t qfull[TQ];
  uint64_t qempty[TQ];
  int4 tq[TQ];  // published tiles: {t, g, mt, nt | HALF_BIT}
  uint32_t tmem_holder;
  int32_t tile_prefix[MAX_G + 1];
  int32_t gstart[MAX_G];
  int32_t gcount[MAX_G];
  alignas(1024) uint8_t stage_out[4][32 * 64];  // per epilogue warp: 32 rows x 32 bf16, 64-B swizzle
  int32_t comb_pos[4][32 * 8];                   // EPI_COMBINE: per epilogue warp, its rows' pos / w
  float comb_w[4][32 * 8];
};

template <int CG>
constexpr size_t smem_bytes() {
  return 1024 + Cfg<CG>::STAGES * (Cfg<CG>::A_BYTES + Cfg<CG>::B_BYTES) + sizeof(SmemTail<CG>);
}

__device__ __forceinline__ float silu_f32(float g) { return g / (1.0f + expf(-g)); }

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Coalesced epilogue store of one warp's 32 rows x 32 bf16 columns: each lane
// holds its row's 64 B (pk), the warp transposes through a 16-B-chunk XOR-
// swizzled smem tile (conflict-free both ways), then 4 lanes write each row's
// 64 B as two full 32-B sectors (8 rows per instruction) instead of 32
// scattered 16-B pieces.  Rows >= vr (past the group's end) are not written.
// The staging layout is exactly TMA's 64-byte swizzle (16-B chunk c of row r at
// c ^ ((r >> 1) & 3)), so a fully valid 32-row slice leaves as one async
// bulk-tensor store (tmo: 32 x 32 box, SWIZZLE_64B) instead of 128 STGs.
__device__ __forceinline__ void stage_write(const uint32_t (&pk)[16], uint8_t* stg, int lane, bool tma) {
  if (tma) {  // the previous bulk store from this buffer must have read it
    if (lane == 0) ptx::bulk_wait_read0();
    __syncwarp();
  }
  uint4* srow = reinterpret_cast<uint4*>(stg + lane * 64);
  const int sw = (lane >> 1) & 3;
#pragma unroll
  for (int j = 0; j < 4; ++j) srow[j ^ sw] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
}
// 16-B piece jq of staged row r (row-major view: 4 lanes per row, 8 rows per pass)
__device__ __forceinline__ uint4* stage_piece(uint8_t* stg, int r, int jq) {
  return reinterpret_cast<uint4*>(stg + r * 64) + (jq ^ ((r >> 1) & 3));
}
__device__ __forceinline__ void stage_flush(uint8_t* stg, __nv_bfloat16* out_row0, int64_t ldo, int vr, int lane,
                                            const CUtensorMap* tmo, int col, int row0) {
  if (tmo && vr == 32) {
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_2d(tmo, ptx::smem_u32(stg), col, row0);
      ptx::bulk_commit();
    }
    return;
  }
  __syncwarp();
  const int j = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i * 8 + (lane >> 2);
    const uint4 v = *stage_piece(stg, r, j);
    if (r < vr) reinterpret_cast<uint4*>(out_row0 + (int64_t)r * ldo)[j] = v;
  }
  __syncwarp();
}
__device__ __forceinline__ void store_chunk(const uint32_t (&pk)[16], uint8_t* stg, __nv_bfloat16* out_row0,
                                            int64_t ldo, int vr, int lane, const CUtensorMap* tmo, int col,
                                            int row0) {
  stage_write(pk, stg, lane, tmo != nullptr);
  stage_flush(stg, out_row0, ldo, vr, lane, tmo, col, row0);
}

// floor(a / b) for 0 <= a < 2^23, b >= 1: float reciprocal estimate (off by at
// most one) and an exact integer correction - a few instructions instead of
// the ~20-instruction integer division sequence.
__device__ __forceinline__ int fdiv(int a, int b) {
  int q = __float2int_rz(__int2float_rn(a) * __frcp_rn(__int2float_rn(b)));
  if (q * b > a) --q;
  else if ((q + 1) * b <= a) ++q;
  return q;
}

constexpr int HALF_BIT = 1 << 30;  // Tile.nt tag: a group's last m-tile with <= BM rows

struct Tile {
  int t, g, mt, nt;  // t < 0: no more tiles
  bool half;         // valid rows of the m-tile <= BM (half-tile MMA candidate)
};
__device__ __forceinline__ Tile unpack_tile(int4 v) { return Tile{v.x, v.y, v.z, v.w & ~HALF_BIT, (v.w & HALF_BIT) != 0}; }

// Tile-ticket stream shared by every role of a CTA (pair).  The fetcher (the
// leader's producer lane) takes tickets, decodes each ticket ONCE into
// (group, m-tile, n-tile, half) and publishes the decoded tile; every other
// role (MMA issuer, epilogue warps, the peer CTA's producer) consumes it in
// the same order, so no consumer decodes on its critical path (K = 1536 Down
// GEMMs change tile every 24 k-blocks).  Static mode needs no communication.
template <int CG>
struct Tickets {
  SmemTail<CG>* st;
  const KParams* p;
  int total, unit, num_units;
  uint32_t rank;
  int G, n_tiles, gm_cfg;
  uint32_t slot = 0, phase = 0;
  int static_next;
  int prefetched = -2;  // fetcher: ticket taken one tile ahead (hides the atomic's latency)
  int gc = 0;           // fetcher: group cursor (a fetcher's tickets only increase)

  __device__ Tickets(SmemTail<CG>* s, const KParams* pp, int tot, int u, int nu, uint32_t r, int g, int nt, int gm)
      : st(s), p(pp), total(tot), unit(u), num_units(nu), rank(r), G(g), n_tiles(nt), gm_cfg(gm), static_next(u) {}

  __device__ __forceinline__ void advance() {
    if (++slot == TQ) { slot = 0; phase ^= 1; }
  }
  // Linear tile index -> (group, m-tile, n-tile).  Inside a group, tiles are
  // visited in blocks of `gm` m-tiles: n-tile major across the block, m fastest
  // inside it (gm = 1: plain n-fastest order).  The group comes from a monotone
  // cursor (the fetcher's tickets, and each role's static tiles, only increase),
  // the raster from fdiv.
  __device__ __forceinline__ Tile decode_fast(int t) {
    while (st->tile_prefix[gc + 1] <= t) ++gc;
    const int p0 = st->tile_prefix[gc];
    const int local = t - p0;
    const int m_tiles = fdiv(st->tile_prefix[gc + 1] - p0, n_tiles);
    const int bsz = gm_cfg >= m_tiles ? m_tiles * n_tiles : gm_cfg * n_tiles;
    const int blk = fdiv(local, bsz);
    const int within = local - blk * bsz;
    const int gm = min(gm_cfg, m_tiles - blk * gm_cfg);
    const int q = fdiv(within, gm);
    Tile d{t, gc, blk * gm_cfg + (within - q * gm), q, false};
    d.half = st->gcount[gc] - d.mt * Cfg<CG>::TILE_M <= BM;
    return d;
  }
  // Fetcher side (one thread): the next tile (t = -1 when done).
  __device__ __forceinline__ Tile fetch() {
    if (!p->dynamic) {
      const int t = static_next;
      static_next += num_units;
      return t < total ? decode_fast(t) : Tile{-1, 0, 0, 0, false};
    }
    int t = (prefetched == -2) ? atomicAdd(p->tile_counter, 1) : prefetched;
    if (t >= total) t = -1;
    // next ticket in flight while this tile's loads are issued (-1 stays -1)
    prefetched = (t < 0) ? -1 : atomicAdd(p->tile_counter, 1);
    const Tile d = (t < 0) ? Tile{-1, 0, 0, 0, false} : decode_fast(t);
    const int4 v = make_int4(d.t, d.g, d.mt, d.nt | (d.half ? HALF_BIT : 0));
    ptx::mbar_wait(ptx::smem_u32(&st->qempty[slot]), phase ^ 1);  // releases are relaxed: no acquire needed
    st->tq[slot] = v;
    ptx::mbar_arrive(ptx::smem_u32(&st->qfull[slot]));
    if constexpr (CG == 2) {
      ptx::st_cluster_v4(ptx::mapa(ptx::smem_u32(&st->tq[slot]), 1), v);
      ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&st->qfull[slot]), 1));
    }
    advance();
    return d;
  }
  // Consumer side: `arrive` = this thread releases the ticket for its role.
  __device__ __forceinline__ Tile consume(bool arrive) {
    if (!p->dynamic) {  // static: this role's tiles u, u + U, ... (increasing: the cursor decode holds)
      const int t = static_next;
      static_next += num_units;
      return t < total ? decode_fast(t) : Tile{-1, 0, 0, 0, false};
    }
    if (CG == 2 && rank != 0)
      ptx::mbar_wait_cluster(ptx::smem_u32(&st->qfull[slot]), phase);  // ticket written by the leader (DSMEM)
    else
      ptx::mbar_wait(ptx::smem_u32(&st->qfull[slot]), phase);
    const Tile d = unpack_tile(st->tq[slot]);
    if (arrive) release(slot);
    advance();
    return d;
  }
  // Release a consumed ticket slot on the fetcher's qempty barrier.
  __device__ __forceinline__ void release(uint32_t s) {
    if constexpr (CG == 2)
      ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&st->qempty[s]), 0));
    else
      ptx::mbar_arrive(ptx::smem_u32(&st->qempty[s]));
  }
};

template <int EPI, int CG, bool GATHER>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
            const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmO,
            const __grid_constant__ CUtensorMap tmB0h, const __grid_constant__ CUtensorMap tmB1h,
            const __grid_constant__ CUtensorMap tmAh, const KParams p) {
  using C = Cfg<CG>;
  // Half tiles (CTA pairs, GateUp / Down): a group's last m-tile holding <= 128
  // valid rows is issued as one M = 128 cta_group::2 MMA (64 rows per CTA)
  // instead of M = 256, halving its tensor work (the M padding is ~128 rows per
  // expert on average).  Accumulator layout of that shape (per CTA, 64 rows):
  // TMEM lanes 0-63 hold columns [0, 128) of the pair's 256, lanes 64-127
  // columns [128, 256), both at TMEM columns 0-127.  So epilogue warps 0/1 own
  // rows 0-63 x the low column half and warps 2/3 the same rows x the high
  // half.  For SwiGLU each CTA then loads 64 gate + 64 up rows (64-row boxes
  // tmB0h / tmB1h) so that a warp sees matching gate and up columns; A comes
  // as 64-row boxes (tmAh), so a half tile also moves 25% fewer bytes.
  constexpr bool HALF_OK = (CG == 2) && !GATHER && (EPI == EPI_SWIGLU || EPI == EPI_BF16);
  // SM-partition probe: this CTA is resident from here to the end of the kernel
  if (p.resident && threadIdx.x == 0) atomicMax(p.resident + 1, atomicAdd(p.resident, 1) + 1);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  SmemTail<CG>& st = *reinterpret_cast<SmemTail<CG>*>(smem + C::STAGES * (C::A_BYTES + C::B_BYTES));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? ptx::cluster_ctarank() : 0;  // CTA rank inside the pair
  const int unit = blockIdx.x / CG;                               // pair (or CTA) id
  const int num_units = gridDim.x / CG;
  const int G = p.row_count ? p.G : 1;
  const int n_out_tile = (EPI == EPI_SWIGLU) ? 128 : BN;  // output columns per tile
  const int n_tiles = (p.N + n_out_tile - 1) / n_out_tile;
  const int num_kb = p.K / BK;

  // ---- group table: start rows, counts, tile prefix (warp-parallel scan)
  for (int g = threadIdx.x; g < G; g += NUM_THREADS) {
    int cnt = p.row_count ? p.row_count[g] : p.m_single;
    int start = p.row_start ? p.row_start[g] : 0;
    const int bulk = cnt & ~255;
    if (p.row_mode == 1) cnt = bulk;
    else if (p.row_mode == 2) { start += bulk; cnt -= bulk; }
    st.gcount[g] = cnt;
    st.gstart[g] = start;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::STAGES; ++i) {
      // GATHER: + the 32 producer lanes' cp.async completions (+ the peer's forwarder)
      ptx::mbar_init(ptx::smem_u32(&st.full[i]), GATHER ? 1 + 32 + (CG - 1) : 1);
      ptx::mbar_init(ptx::smem_u32(&st.gfull[i]), 32);
      ptx::mbar_init(ptx::smem_u32(&st.empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&st.tfull[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&st.tempty[i]), 4 * CG);  // one arrive per epilogue warp (both CTAs)
    }
    for (int i = 0; i < TQ; ++i) {
      ptx::mbar_init(ptx::smem_u32(&st.qfull[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&st.qempty[i]), C::TQ_CONSUMERS + ((GATHER && CG == 2) ? 1 : 0));
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<TMEM_COLS, CG>(ptx::smem_u32(&st.tmem_holder));
  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch_desc(&tmA);
    ptx::tma_prefetch_desc(&tmB0);
    if (EPI == EPI_SWIGLU) ptx::tma_prefetch_desc(&tmB1);
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int PER = (MAX_G + 31) / 32;
    int local[PER];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int g = lane * PER + i;
      int tiles = (g < G) ? ((st.gcount[g] + C::TILE_M - 1) / C::TILE_M) * n_tiles : 0;
      local[i] = sum;
      sum += tiles;
    }
    int incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    int excl = incl - sum;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      int g = lane * PER + i;
      if (g < G) st.tile_prefix[g] = excl + local[i];
    }
    if (lane == 31) st.tile_prefix[G] = incl;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) ptx::cluster_sync();  // peer barriers initialised before any remote signal
  ptx::tc_fence_after();
  const uint32_t tmem_base = st.tmem_holder;
  const int total = st.tile_prefix[G];
  Tickets<CG> tk(&st, &p, total, unit, num_units, rank, G, n_tiles, p.raster_gm);

  if (warp == 0) {
    // ===================== TMA producer (each CTA loads its own halves) =====================
    // The leader's lane 0 fetches tickets; the peer's lane 0 consumes them.
    // GATHER (A rows picked by a_row_index, i.e. GateUp reading x directly):
    // the whole warp copies A with 16-B cp.async into the swizzled stage; lane 0
    // still TMA-loads B.
    uint32_t stage = 0, phase = 0;
    // GATHER: this lane's A row indices of the tile, A row pitch
    int32_t gidx[GATHER ? BM / 4 : 1];
    const size_t a_pitch = (size_t)p.K * 2;
    // Dynamic tickets: the leader publishes tile i+1 before it loads tile i, so
    // the peer's producer and the MMA issuer find the next tile already decoded
    // at every tile boundary (EPSMOE_TICKET_AHEAD=0: publish when loading it).
    Tile ahead{-2, 0, 0, 0, false};
    while (true) {
      int4 tv = make_int4(0, 0, 0, 0);
      if (lane == 0) {
        Tile d;
        if (rank != 0) {
          d = tk.consume(true);
        } else if (p.dynamic && p.ticket_ahead) {
          d = (ahead.t == -2) ? tk.fetch() : ahead;
          if (d.t >= 0) ahead = tk.fetch();
        } else {
          d = tk.fetch();
        }
        tv = make_int4(d.t, d.g, d.mt, d.nt | (d.half ? HALF_BIT : 0));
      }
      if constexpr (GATHER) {
        tv.x = __shfl_sync(0xffffffffu, tv.x, 0);
        tv.y = __shfl_sync(0xffffffffu, tv.y, 0);
        tv.z = __shfl_sync(0xffffffffu, tv.z, 0);
        tv.w = __shfl_sync(0xffffffffu, tv.w, 0);
      } else if (lane != 0) {
        break;  // TMA: lane 0 alone
      }
      const Tile d = unpack_tile(tv);
      if (d.t < 0) break;
      const int g = d.g, mt = d.mt, nt = d.nt;
      const bool half = HALF_OK && p.half_tiles && d.half;
      const int a_row = st.gstart[g] + mt * C::TILE_M + (int)rank * (half ? BM / 2 : BM);
      const int b_row0 = (p.b_base + g) * p.b_group_rows + nt * n_out_tile;
      if constexpr (GATHER) {
        // this lane's rows of the tile: chunk (lane & 7) of rows (lane >> 3) + 4 i;
        // rows past the group's end read the group's first row (not stored)
        const int local0 = mt * C::TILE_M + (int)rank * BM;
#pragma unroll
        for (int i = 0; i < BM / 4; ++i) {
          const int r = (lane >> 3) + 4 * i;
          const int src = (local0 + r < st.gcount[g]) ? a_row + r : st.gstart[g];
          gidx[i] = p.a_row_index[src];
        }
      }
      if (GATHER || lane == 0) {
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(ptx::smem_u32(&st.empty[stage]), phase ^ 1);
          const uint32_t fb = ptx::smem_u32(&st.full[stage]);
          const uint32_t a_dst = ptx::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_dst = ptx::smem_u32(sB + stage * C::B_BYTES);
          if ((CG == 1 || rank == 0) && lane == 0)
            ptx::mbar_arrive_expect_tx(fb, CG * ((GATHER ? 0 : (half ? C::A_BYTES / 2 : C::A_BYTES)) +
                                                 (EPI == EPI_F32 ? (p.n_mma / CG) * BK * 2 : C::B_BYTES)));
          if constexpr (GATHER) {
            // A by 16-B cp.async straight into the 128-B swizzle (chunk c of row r at
            // c ^ (r & 7)): 4 rows x 128 B per warp instruction, no TMA descriptor per row
            const int c = lane & 7;
            const uint8_t* src0 = p.a_ptr + (size_t)kb * (BK * 2) + c * 16;
#pragma unroll
            for (int i = 0; i < BM / 4; ++i) {
              const int r = (lane >> 3) + 4 * i;
              ptx::cp_async16(a_dst + r * 128 + ((c ^ (r & 7)) << 4), src0 + (size_t)gidx[i] * a_pitch);
            }
            // each lane's completion arrives asynchronously (no wait, no fence in this
            // warp): on the full barrier, or in the peer on gfull for its forwarder
            ptx::cp_async_mbar_arrive_noinc((CG == 1 || rank == 0) ? fb : ptx::smem_u32(&st.gfull[stage]));
            if (lane != 0) {
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
              continue;
            }
          } else if constexpr (CG == 1) {
            ptx::tma_load_2d(a_dst, &tmA, fb, kb * BK, a_row);
          } else {
            ptx::tma_load_2d_pair(a_dst, half ? &tmAh : &tmA, fb, kb * BK, a_row);
          }
          if constexpr (CG == 1) {
            if (EPI == EPI_SWIGLU) {
              ptx::tma_load_2d(b_dst, &tmB0, fb, kb * BK, b_row0);
              ptx::tma_load_2d(b_dst + C::B_BYTES / 2, &tmB1, fb, kb * BK, b_row0);
            } else {
              ptx::tma_load_2d(b_dst, &tmB0, fb, kb * BK, b_row0);
            }
          } else if (HALF_OK && EPI == EPI_SWIGLU && half) {
            // half tile: this CTA's B = gate rows [64r, 64r+64) then up rows [64r, 64r+64)
            ptx::tma_load_2d_pair(b_dst, &tmB0h, fb, kb * BK, b_row0 + (int)rank * 64);
            ptx::tma_load_2d_pair(b_dst + C::B_BYTES / 2, &tmB1h, fb, kb * BK, b_row0 + (int)rank * 64);
          } else {
            // SwiGLU: CTA0 gate rows -> acc cols [0,128); CTA1 up rows -> [128,256)
            const void* tb = (EPI == EPI_SWIGLU && rank == 1) ? (const void*)&tmB1 : (const void*)&tmB0;
            const int brow = (EPI == EPI_SWIGLU) ? b_row0
                             : b_row0 + (int)rank * (EPI == EPI_F32 ? p.n_mma / 2 : C::B_ROWS);
            ptx::tma_load_2d_pair(b_dst, tb, fb, kb * BK, brow);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread of the leader CTA) =====================
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc_full = ptx::idesc_bf16_f32(C::TILE_M, BN);
      constexpr uint32_t idesc_half = ptx::idesc_bf16_f32(C::TILE_M / 2, BN);
      uint32_t stage = 0, phase = 0, iter = 0;
      while (true) {
        const Tile d = tk.consume(true);
        if (d.t < 0) break;
        uint32_t idesc = (EPI == EPI_F32) ? ptx::idesc_bf16_f32(C::TILE_M, p.n_mma) : idesc_full;
        if (HALF_OK && p.half_tiles && d.half) idesc = idesc_half;
        const uint32_t acc = iter & 1, accph = (iter >> 1) & 1;
        ptx::mbar_wait(ptx::smem_u32(&st.tempty[acc]), accph ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          // GATHER pair: the peer's A arrives by a cluster-scope release (not a TMA
          // complete_tx), so the wait needs cluster-scope acquire
          if constexpr (GATHER && CG == 2) ptx::mbar_wait_cluster(ptx::smem_u32(&st.full[stage]), phase);
          else ptx::mbar_wait(ptx::smem_u32(&st.full[stage]), phase);
          if constexpr (GATHER) ptx::fence_proxy_async_smem();  // cp.async (generic) writes -> MMA reads
          ptx::tc_fence_after();
          const uint64_t adesc = ptx::sdesc_k_sw128(ptx::smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bdesc = ptx::sdesc_k_sw128(ptx::smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance 16 bf16 = 32 B along K inside the 128 B swizzle atom
            if constexpr (CG == 1)
              ptx::mma_bf16_ss(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            else
              ptx::mma_bf16_ss_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          if constexpr (CG == 1) ptx::mma_commit(ptx::smem_u32(&st.empty[stage]));
          else ptx::mma_commit_pair(ptx::smem_u32(&st.empty[stage]), 0x3);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (CG == 1) ptx::mma_commit(ptx::smem_u32(&st.tfull[acc]));
        else ptx::mma_commit_pair(ptx::smem_u32(&st.tfull[acc]), 0x3);
        ++iter;
      }
    }
    if constexpr (GATHER && CG == 2) {
      // the peer's forwarder: its A copies of a stage landed (gfull) -> proxy fence ->
      // cluster-release arrive on the leader's full barrier
      if (lane == 0 && rank == 1) {
        uint32_t stage = 0, phase = 0;
        while (tk.consume(true).t >= 0) {
          for (int kb = 0; kb < num_kb; ++kb) {
            ptx::mbar_wait(ptx::smem_u32(&st.gfull[stage]), phase);
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&st.full[stage]), 0));
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else {
    // ===================== epilogue (4 warps, TMEM lane quadrant = warp % 4) =====
    const int q = warp & 3;
    const uint32_t tempty_leader0 = (CG == 2) ? ptx::mapa(ptx::smem_u32(&st.tempty[0]), 0) : 0;
    const uint32_t tempty_leader1 = (CG == 2) ? ptx::mapa(ptx::smem_u32(&st.tempty[1]), 0) : 0;
    uint32_t iter = 0;
    while (true) {
      const Tile d = tk.consume(false);
      __syncwarp();
      if (lane == 0 && p.dynamic) tk.release((tk.slot + TQ - 1) % TQ);  // once per warp
      if (d.t < 0) break;
      const int g = d.g, mt = d.mt, nt = d.nt;
      const uint32_t acc = iter & 1, accph = (iter >> 1) & 1;
      ptx::mbar_wait(ptx::smem_u32(&st.tfull[acc]), accph);
      ptx::tc_fence_after();
      const bool half = HALF_OK && p.half_tiles && d.half;
      const int hq = half ? (q >> 1) : 0;  // half tile: which 128 (Down) / 64 (SwiGLU) column half
      const int local_row = half ? mt * C::TILE_M + (int)rank * (BM / 2) + (q & 1) * 32 + lane
                                 : mt * C::TILE_M + (int)rank * BM + q * 32 + lane;
      const bool valid = local_row < st.gcount[g];
      const int64_t grow = (int64_t)st.gstart[g] + local_row;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      // rows of this warp's 32-row slice that belong to the group
      const int vr = (p.diag == 1) ? 0 : max(0, min(32, st.gcount[g] - (local_row - lane)));
      if (p.diag == 2) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 1) ptx::mbar_arrive(ptx::smem_u32(&st.tempty[acc]));
          else ptx::mbar_arrive_cluster_relaxed(acc ? tempty_leader1 : tempty_leader0);
        }
        ++iter;
        continue;
      }
      uint8_t* stg = st.stage_out[q];
      if (EPI == EPI_SWIGLU) {
        // full tile: 4 x 32 output columns, gate at TMEM column c*32, up at 128 + c*32;
        // half tile: this warp's 64 output columns nt*128 + 64*hq + [0, 64), gate at c*32, up at 64 + c*32
        const int ocol = nt * 128 + hq * 64;
        const int nchunk = half ? 2 : 4, up_off = half ? 64 : 128;
        __nv_bfloat16* out0 = reinterpret_cast<__nv_bfloat16*>(p.out) + (grow - lane) * p.ldo + ocol;
#pragma unroll 1
        for (int c = 0; c < nchunk; ++c) {
          uint32_t gr[32], ur[32], pk[16];
          ptx::tmem_ld32(taddr + c * 32, gr);
          ptx::tmem_ld32(taddr + up_off + c * 32, ur);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float g0 = __uint_as_float(gr[2 * i]), g1 = __uint_as_float(gr[2 * i + 1]);
            float u0 = __uint_as_float(ur[2 * i]), u1 = __uint_as_float(ur[2 * i + 1]);
            pk[i] = pack_bf16(silu_f32(g0) * u0, silu_f32(g1) * u1);
          }
          store_chunk(pk, stg, out0 + c * 32, p.ldo, vr, lane, p.tma_store ? &tmO : nullptr, ocol + c * 32,
                      (p.diag == 3 ? (int)((grow - lane) & 255) : (int)(grow - lane)));
        }
      } else if (EPI == EPI_BF16 && p.rseg) {
        // DownGemm fused with the combine all2all: each row is stored straight
        // into its destination (a peer's combine buffer) while later tiles compute
        char* rowp = nullptr;
        if (valid) {
          int lo = 0, hi = p.nrseg - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.rseg[mid].r0 <= grow) lo = mid; else hi = mid - 1;
          }
          const GemmRowSeg sg = p.rseg[lo];
          if (grow >= sg.r0 && grow < sg.r0 + sg.n) rowp = sg.dst + (grow - sg.r0) * p.ldo * 2;
        }
        const int jq = lane & 3;
#pragma unroll 1
        for (int c = 0; c < (half ? BN / 64 : BN / 32); ++c) {  // half tile: this warp's 128 columns
          const int col0 = nt * BN + hq * 128 + c * 32;
          if (col0 >= p.N) break;
          uint32_t r[32], pk[16];
          ptx::tmem_ld32(taddr + c * 32, r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
          stage_write(pk, stg, lane, false);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = i * 8 + (lane >> 2);
            char* dp = reinterpret_cast<char*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rowp), rr));
            const uint4 v = *stage_piece(stg, rr, jq);
            if (rr < vr && dp) reinterpret_cast<uint4*>(dp + (size_t)col0 * 2)[jq] = v;
          }
          __syncwarp();
        }
      } else if (EPI == EPI_BF16) {
        const int ocol = nt * BN + hq * 128;  // half tile: this warp's 128 of the 256 columns
        __nv_bfloat16* out0 = reinterpret_cast<__nv_bfloat16*>(p.out) + (grow - lane) * p.ldo + ocol;
#pragma unroll 1
        for (int c = 0; c < (half ? BN / 64 : BN / 32); ++c) {
          if (ocol + c * 32 >= p.N) break;  // N is a multiple of 32 (warp-uniform)
          uint32_t r[32], pk[16];
          ptx::tmem_ld32(taddr + c * 32, r);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
          store_chunk(pk, stg, out0 + c * 32, p.ldo, vr, lane, p.tma_store ? &tmO : nullptr, ocol + c * 32,
                      (p.diag == 3 ? (int)((grow - lane) & 255) : (int)(grow - lane)));
        }
      } else if (EPI == EPI_COMBINE) {
        // s = bf16(acc) is staged row-major in smem; the weighted unpermute then
        // runs with 4 lanes per row so each o row piece is one contiguous 64-B
        // read (8 rows per instruction) instead of 32 scattered 16-B pieces.
        __nv_bfloat16* out0 = reinterpret_cast<__nv_bfloat16*>(p.out) + (grow - lane) * p.ldo + nt * BN;
        const int kk = p.comb_k;
        const uint64_t pol = evict_first_policy();
        int32_t* cpos = st.comb_pos[q];
        float* cw = st.comb_w[q];
        __syncwarp();  // previous tile's readers are done
#pragma unroll
        for (int j = 0; j < COMB_MAX_K; ++j) {
          if (j < kk) {
            cpos[lane * COMB_MAX_K + j] = valid ? p.comb_pos[grow * kk + j] : 0;
            cw[lane * COMB_MAX_K + j] = valid ? p.comb_w[grow * kk + j] : 0.f;
          }
        }
        __syncwarp();
        const int jq = lane & 3;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int col0 = nt * BN + c * 32;
          if (col0 >= p.N) break;  // N is a multiple of 32 (warp-uniform)
          // the k expert-output pieces of this lane's 4 rows in flight before the TMEM read
          uint4 ov[4][COMB_MAX_K];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = i * 8 + (lane >> 2);
#pragma unroll
            for (int j = 0; j < COMB_MAX_K; ++j)
              ov[i][j] = (r < vr && j < kk)
                             ? ld_once(p.comb_o + (int64_t)cpos[r * COMB_MAX_K + j] * p.N + col0 + 8 * jq, pol)
                             : make_uint4(0, 0, 0, 0);
          }
          uint32_t rr[32], pk[16];
          ptx::tmem_ld32(taddr + c * 32, rr);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1]));
          stage_write(pk, stg, lane, p.tma_store != 0);  // s = bf16(acc)
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = i * 8 + (lane >> 2);
            uint4* sp = stage_piece(stg, r, jq);
            const uint4 sv = *sp;
            const uint32_t s4[4] = {sv.x, sv.y, sv.z, sv.w};
            float a[8];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              a[2 * h] = bf16_lo(s4[h]);
              a[2 * h + 1] = bf16_hi(s4[h]);
            }
#pragma unroll
            for (int j = 0; j < COMB_MAX_K; ++j) {
              if (j < kk) {
                const float w = cw[r * COMB_MAX_K + j];
                const uint32_t o4[4] = {ov[i][j].x, ov[i][j].y, ov[i][j].z, ov[i][j].w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  a[2 * h] = __fmaf_rn(w, bf16_lo(o4[h]), a[2 * h]);
                  a[2 * h + 1] = __fmaf_rn(w, bf16_hi(o4[h]), a[2 * h + 1]);
                }
              }
            }
            *sp = make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]),
                             pack_bf16(a[6], a[7]));
          }
          stage_flush(stg, out0 + c * 32, p.ldo, vr, lane, p.tma_store ? &tmO : nullptr, col0, (p.diag == 3 ? (int)((grow - lane) & 255) : (int)(grow - lane)));
        }
      } else {
        float* out = reinterpret_cast<float*>(p.out) + grow * p.ldo;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          const int col0 = nt * BN + c * 32;
          if (col0 >= p.N) break;  // warp-uniform; columns past n_mma were never computed
          uint32_t r[32];
          ptx::tmem_ld32(taddr + c * 32, r);
          ptx::tmem_wait_ld();
          if (valid) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int col = col0 + i;
              if (col < p.N) {
                float v = __uint_as_float(r[i]);
                if (p.bias) v = __fadd_rn(v, p.bias[col]);
                out[col] = v;
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 1) ptx::mbar_arrive(ptx::smem_u32(&st.tempty[acc]));
        // relaxed: the TMEM reads are ordered by tcgen05.wait::ld + fence::before_thread_sync;
        // the tile's global stores need not complete before the accumulator is reused
        else ptx::mbar_arrive_cluster_relaxed(acc ? tempty_leader1 : tempty_leader0);
      }
      ++iter;
    }
  }

  // scattered rows visible to the peers before this launch ends (flags raised by
  // this launch's last CTA, or by a later stream-ordered launch: DENSE chunks)
  if (p.nsig || p.rseg) __threadfence_system();
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) ptx::cluster_sync();  // no CTA leaves while its peer may still signal it
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc<TMEM_COLS, CG>(tmem_base);
  if (warp >= 2 && lane == 0 && p.tma_store) ptx::bulk_wait0();  // output stores complete
  if ((p.dynamic || p.nsig) && threadIdx.x == 0) {
    // the last CTA to finish resets the ticket counter for the next launch and
    // raises the completion flags of a fused scatter
    __threadfence();
    if (atomicAdd(p.tile_counter + 1, 1) == (int)gridDim.x - 1) {
      if (p.nsig) {
        __threadfence_system();
        for (int i = 0; i < p.nsig; ++i)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.sig_flags[i]), "r"(p.sig_epoch) : "memory");
      }
      p.tile_counter[0] = 0;
      p.tile_counter[1] = 0;
      __threadfence();
    }
  }
  if (p.resident && threadIdx.x == 0) atomicSub(p.resident, 1);
}

// ------------------------------------------------------------------ host side

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// Tile rasterisation block (m-tiles).  Blocks of 4 m-tiles (n-major across
// the block) keep a group's A and B tiles in flight together; when a group's
// weights dwarf its rows (B > 4 A, A <= 48 MB: Mixtral's GateUp) all m-tiles
// of an n-tile go first instead, so A stays L2-resident and B streams once
// (measured: Mixtral GateUp DRAM reads ~4x lower, layer -4.5%; DSv2 shapes and
// the dense shared GEMMs are faster with blocks of 4).  EPSMOE_RASTER_GM
// overrides.
int raster_gm(int epi, int N, int K, double rows_hint, int tile_m) {
  static int v = env_int("EPSMOE_RASTER_GM", 0);
  if (v > 0) return v;
  if (rows_hint > 0) {
    const double a_bytes = rows_hint * K * 2.0;
    const double b_bytes = (epi == EPI_SWIGLU ? 2.0 : 1.0) * N * K * 2.0;
    if (b_bytes > 4.0 * a_bytes && a_bytes <= 48e6) return 1 << 20;
    // a group's rows overflow L2: blocks holding ~64 MB of A, B streamed once per block
    if (a_bytes > 48e6) return std::max(4, std::min(64, (int)(64e6 / ((double)tile_m * K * 2.0))));
  }
  return 4;
}
// Tile scheduling per epilogue kind: 1 = dynamic tickets, 0 = static round
// robin.  EPSMOE_DYN_SCHED: 0 all static, 1 all dynamic, 2 dynamic except the
// DownGemm (EPI_BF16).
int dynamic_sched(int epi) {
  static int v = env_int("EPSMOE_DYN_SCHED", 1);
  if (v == 2) return epi == EPI_BF16 ? 0 : 1;
  return v;
}

// Fallback ticket counter for launches without a caller-owned one (the
// moe_gemm_grouped test hook; stream-serialised use only).
int32_t* ticket_counter(int) {
  static int32_t* base = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (cudaMalloc(&base, 2 * sizeof(int32_t)) == cudaSuccess) cudaMemset(base, 0, 2 * sizeof(int32_t));
  });
  return base;
}

// 2D bf16 K-major tensor [rows, K] with a {64, box_rows} box and 128 B swizzle.
bool make_tmap(CUtensorMap* m, const void* base, int64_t rows, int K, int box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// bf16 output tensor [rows, ld] for the epilogue's bulk stores: 32 x 32 box
// (one warp's 32 rows x 32 columns), 64-byte swizzle (the staging layout).
bool make_tmap_out(CUtensorMap* m, void* base, int64_t rows, int64_t ld) {
  auto enc = get_encode_fn();
  if (!enc || rows <= 0) return false;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int EPI, int CG, bool GATHER>
int launch_epi(const GemmArgs& a, cudaStream_t stream) {
  static bool attr_set = false;
  auto kern = gemm_kernel<EPI, CG, GATHER>;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<CG>());
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  CUtensorMap tA, tB0, tB1, tB0h, tB1h, tAh;
  // router (EPI_F32, N = E in one n-tile): the MMA covers E rounded up to 16 columns
  const int n_mma = (EPI == EPI_F32 && a.N <= BN && !env_int("EPSMOE_ROUTER_NFULL", 0)) ? ((a.N + 15) & ~15) : BN;
  const int b_box = (EPI == EPI_F32) ? n_mma / CG : (EPI == EPI_SWIGLU || CG == 2) ? 128 : 256;
  if (!make_tmap(&tA, a.A, a.a_rows, a.K, GATHER ? 1 : BM)) return (int)cudaErrorInvalidValue;
  if (!make_tmap(&tB0, a.B0, a.b_rows, a.K, b_box)) return (int)cudaErrorInvalidValue;
  if (EPI == EPI_SWIGLU) {
    if (!make_tmap(&tB1, a.B1, a.b_rows, a.K, b_box)) return (int)cudaErrorInvalidValue;
  } else {
    tB1 = tB0;
  }
  // half tiles (CTA pairs): 64-row boxes of W_gate / W_up for SwiGLU
  const int half_env = env_int("EPSMOE_HALF_TILES", 1);
  tB0h = tB0;
  tB1h = tB1;
  tAh = tA;
  if (CG == 2 && !GATHER && (EPI == EPI_SWIGLU || EPI == EPI_BF16) && half_env &&
      !make_tmap(&tAh, a.A, a.a_rows, a.K, BM / 2))
    return (int)cudaErrorInvalidValue;
  if (EPI == EPI_SWIGLU && CG == 2 && !GATHER && half_env) {
    if (!make_tmap(&tB0h, a.B0, a.b_rows, a.K, 64) || !make_tmap(&tB1h, a.B1, a.b_rows, a.K, 64))
      return (int)cudaErrorInvalidValue;
  }
  KParams p;
  p.K = a.K;
  p.N = a.N;
  p.G = a.G;
  p.m_single = a.m_single;
  p.b_group_rows = a.b_group_rows;
  p.b_base = a.b_base;
  p.raster_gm = raster_gm(EPI, a.N, a.K, a.rows_hint, BM * CG);
  p.ldo = a.ldo;
  p.out = a.out;
  p.bias = a.bias;
  p.row_start = a.row_start;
  p.row_count = a.row_count;
  p.a_row_index = a.a_row_index;
  p.a_ptr = reinterpret_cast<const uint8_t*>(a.A);
  p.row_mode = a.row_mode;
  p.rseg = (EPI == EPI_BF16) ? a.rseg : nullptr;
  p.nrseg = a.nrseg;
  p.sig_flags = a.sig_flags;
  p.nsig = a.sig_flags ? a.nsig : 0;
  p.sig_epoch = a.sig_epoch;
  p.comb_o = reinterpret_cast<const __nv_bfloat16*>(a.comb_o);
  p.comb_pos = a.comb_pos;
  p.comb_w = a.comb_w;
  p.comb_k = a.comb_k;
  p.resident = a.resident;
  p.diag = env_int("EPSMOE_GEMM_DIAG", 0);
  p.n_mma = n_mma;
  p.half_tiles = (CG == 2 && !GATHER && (EPI == EPI_SWIGLU || EPI == EPI_BF16) && a.row_mode == 0) ? half_env : 0;
  CUtensorMap tO;
  std::memset(&tO, 0, sizeof(tO));
  p.tma_store = 0;
  if (EPI != EPI_F32 && !p.rseg && env_int("EPSMOE_TMA_STORE", 1) &&
      make_tmap_out(&tO, a.out, a.out_rows > 0 ? a.out_rows : a.a_rows, a.ldo))
    p.tma_store = 1;
  // Launches that may run concurrently must use different counters (caller's).
  p.tile_counter = a.tile_counter ? a.tile_counter : ticket_counter(0);
  p.dynamic = (dynamic_sched(EPI) && p.tile_counter) ? 1 : 0;
  static const int ticket_ahead = env_int("EPSMOE_TICKET_AHEAD", 1);
  p.ticket_ahead = ticket_ahead;
  int grid = a.num_ctas;
  if (!a.row_count) {
    // one dense group (router, shared experts): no more CTAs than tiles - idle
    // persistent CTAs would only hold SMs a concurrent kernel could use (decode)
    const int n_out = (EPI == EPI_SWIGLU) ? 128 : BN;
    const int64_t tiles =
        ((int64_t)a.m_single + BM * CG - 1) / (BM * CG) * (int64_t)((a.N + n_out - 1) / n_out);
    if (tiles * CG < grid) grid = (int)(tiles * CG);
  }
  if (CG == 2) grid &= ~1;
  if (grid < CG) grid = CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = smem_bytes<CG>();
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tA, tB0, tB1, tO, tB0h, tB1h, tAh, p);
  return (int)e;
}

template <int CG>
int launch_cg(const GemmArgs& a, cudaStream_t stream) {
  switch (a.epi) {
    case EPI_SWIGLU:
      return a.a_row_index ? launch_epi<EPI_SWIGLU, CG, true>(a, stream) : launch_epi<EPI_SWIGLU, CG, false>(a, stream);
    case EPI_BF16: return launch_epi<EPI_BF16, CG, false>(a, stream);
    case EPI_F32: return launch_epi<EPI_F32, CG, false>(a, stream);
    case EPI_COMBINE: return launch_epi<EPI_COMBINE, CG, false>(a, stream);
  }
  return (int)cudaErrorInvalidValue;
}

}  // namespace

int gemm_launch(const GemmArgs& a, cudaStream_t stream) {
  if (a.K % BK != 0 || a.K <= 0 || a.G < 1 || a.G > MAX_G || a.num_ctas < 1) return (int)cudaErrorInvalidValue;
  if (a.epi == EPI_COMBINE && (!a.comb_o || !a.comb_pos || !a.comb_w || a.comb_k < 1 || a.comb_k > COMB_MAX_K ||
                               a.G != 1 || a.row_start || a.N % 32))
    return (int)cudaErrorInvalidValue;
  if (a.row_count == nullptr && a.m_single <= 0) return 0;
  return a.cta_pair ? launch_cg<2>(a, stream) : launch_cg<1>(a, stream);
}

}  // namespace epsmoe
