// a7 building block: out-projection partial GEMM  Y[T][N] = X[T][K] . W[K][N]  (tcgen05).
//
// PAPER: MuxWise serves Llama-70B with tensor parallelism of degree 8 over NVLink
// (P:686); under KV-head sharding each GPU holds Hq/G q heads, so its attention
// output X = O_local [T][Hq/G * d] times its row shard of W_o gives a partial sum of the layer
// output that an all-reduce completes.  This kernel is that per-GPU GEMM (bf16 in, fp32
// accumulate in TMEM, bf16 or fp32 out); the all-reduce runs on the side's NCCL communicator.
//
// W is a weight, so it is stored PACKED (mux_outproj_pack_w): 128 n x 64 k tiles of 16 KiB in
// exactly the SWIZZLE_128B MN-major image tcgen05 reads (two 8 KiB halves of 64 n, row = k,
// 16-byte chunk c of row k stored at chunk c ^ (k & 7)), tile (nt, kb) at (nt*KB + kb)*16 KiB.
// Each pipeline stage's W operand is then one contiguous 16 KiB cp.async.bulk: the tensor-map
// load of the row-major W fetched 128-byte rows 8 KiB apart and capped the skinny kernel at
// ~40 GB/s per SM (ncu, profiles/r01_summary.md).
//
// Tile kernel (T > 128), default: CTA pairs (cta_group::2, below: 256 x 256 tiles, 1446 TF/s at
// 8192x4096x4096 vs 1357 for the single-CTA kernel and 1515 for cuBLAS).  Single-CTA fallback:
// persistent, one CTA per SM of the side's partition walking 128 x 256
// output tiles, 6 warps: warp 4 = producer (TMA for X, bulk copies for W), warp 5 = TMEM owner
// + single-thread tcgen05.mma issuer, warps 0-3 = epilogue (thread = output row).  4-stage ring
// of {A: X 128 rows x 64 k (K-major, TMA SWIZZLE_128B), B: 2 packed W tiles = 64 k x 256 n
// (MN-major)}, 48 KiB per stage; two 256-column TMEM accumulators so a tile's epilogue
// overlaps the next tile's mainloop.
//
// Skinny kernel (T <= 128, the decode side: one token per sequence): the 128-row M tile would
// be mostly zero fill, so it computes the transpose Y^T = W^T . X^T: M = 128 columns of W (A =
// one packed tile, MN-major), N = T rounded up to 32 (B = X, K-major via TMA), one CTA per 128
// columns of W, a ~200 KiB ring of 2-4 stages of ks k-blocks each (one ks x 16 KiB bulk copy of
// W per stage), stored straight from TMEM (no split-K: bitwise deterministic).  Measured limit:
// ~100 GB/s of smem fill per SM (bytes in flight / DRAM latency), so on a decode partition its
// time is W + X-re-read bytes / (SMs x ~100 GB/s).
// Rows / columns past T / N come from TMA zero fill or packing pads and are not stored.
#include <algorithm>

#include "pool.h"

namespace mux {
namespace {

constexpr int kGBM = 128, kGBN = 256, kGBK = 64, kGStages = 4;
constexpr int kGThreads = 192;
constexpr int kPackTile = 128 * kGBK * 2;  // 16 KiB

struct GemmSmem {
  static constexpr int kA = kGBM * kGBK * 2;          // 16 KiB
  static constexpr int kB = kGBK * kGBN * 2;          // 32 KiB
  static constexpr int kStage = kA + kB;
  static constexpr int kBar = kGStages * kStage;
  // full[4] empty[4] acc_full[2] acc_empty[2]
  static constexpr int kTmemSlot = kBar + (2 * kGStages + 4) * 8;
  static constexpr int kBytes = kTmemSlot + 16;
};

struct GemmParams {
  void* y;
  const uint8_t* w_pk;
  int T, N, K, y_f32;
  int m_tiles, n_tiles;
};

__device__ __forceinline__ void store_row32(const GemmParams& p, int row, int col, const uint32_t* v) {
  if (row >= p.T) return;
  if (p.y_f32) {
    float* dst = static_cast<float*>(p.y) + static_cast<size_t>(row) * p.N + col;
    if (col + 32 <= p.N && (p.N & 3) == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        reinterpret_cast<float4*>(dst)[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                                        __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
    } else {
      for (int i = 0; i < 32 && col + i < p.N; ++i) dst[i] = __uint_as_float(v[i]);
    }
  } else {
    uint16_t* dst = static_cast<uint16_t*>(p.y) + static_cast<size_t>(row) * p.N + col;
    if (col + 32 <= p.N && (p.N & 7) == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        reinterpret_cast<uint4*>(dst)[i] =
            make_uint4(dev::pack_bf16(__uint_as_float(v[8 * i]), __uint_as_float(v[8 * i + 1])),
                       dev::pack_bf16(__uint_as_float(v[8 * i + 2]), __uint_as_float(v[8 * i + 3])),
                       dev::pack_bf16(__uint_as_float(v[8 * i + 4]), __uint_as_float(v[8 * i + 5])),
                       dev::pack_bf16(__uint_as_float(v[8 * i + 6]), __uint_as_float(v[8 * i + 7])));
    } else {
      for (int i = 0; i < 32 && col + i < p.N; ++i)
        dst[i] = static_cast<uint16_t>(dev::pack_bf16(__uint_as_float(v[i]), 0.f) & 0xFFFFu);
    }
  }
}

// Persistent: CTA c walks tiles c, c + gridDim.x, ... (n fastest: co-running CTAs share a few
// X row panels while all of the packed W stays in L2).  The smem ring runs continuously across tiles, and the accumulator
// is double-buffered in TMEM (2 x 256 columns): tile i+1's mainloop overlaps tile i's epilogue.
__global__ void __launch_bounds__(kGThreads, 1)
    outproj_kernel(const __grid_constant__ CUtensorMap tmap_x, const GemmParams p) {
  using L = GemmSmem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + kGStages;
  uint64_t* acc_full = empty + kGStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  const int warp = dev::warp_idx_uniform(), lane = threadIdx.x & 31;
  const int nk = (p.K + kGBK - 1) / kGBK;
  const int ntiles = (p.N + 127) / 128;                       // 128-column packed W tiles
  const int tiles = p.m_tiles * p.n_tiles;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kGStages + 2; ++i) dev::mbar_init(&full[i], 1);
    dev::mbar_init(&acc_empty[0], 4);
    dev::mbar_init(&acc_empty[1], 4);
    dev::fence_mbar_init();
  }
  if (warp == 5) dev::tmem_alloc(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      dev::tma_prefetch(&tmap_x);
      int it = 0;  // global k-block counter (ring position)
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m0 = (t / p.n_tiles) * kGBM, nt0 = (t % p.n_tiles) * 2;
        const bool second = nt0 + 1 < ntiles;
        const uint8_t* w0 = p.w_pk + static_cast<size_t>(nt0) * nk * kPackTile;
        const uint8_t* w1 = w0 + static_cast<size_t>(nk) * kPackTile;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kGStages;
          if (it >= kGStages) dev::mbar_wait_sleep(&empty[s], ((it / kGStages) - 1) & 1);
          dev::mbar_expect_tx(&full[s], L::kA + (second ? 2 : 1) * kPackTile);
          uint8_t* a = smem + s * L::kStage;
          uint8_t* bt = a + L::kA;
          dev::tma_load_3d(a, &tmap_x, &full[s], kb * kGBK, m0, 0);
          dev::bulk_load(bt, w0 + static_cast<size_t>(kb) * kPackTile, kPackTile, &full[s]);
          if (second) dev::bulk_load(bt + kPackTile, w1 + static_cast<size_t>(kb) * kPackTile, kPackTile, &full[s]);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idesc = dev::umma_idesc_bf16(kGBM, kGBN, 0, 1);
      const uint64_t d0 = dev::umma_desc_sw128(dev::smem_u32(smem), 16, 1024);                      // A K-major
      const uint64_t e0 = dev::umma_desc_sw128(dev::smem_u32(smem + L::kA), kGBK * 128, 1024);     // B MN-major
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int b = i & 1;
        if (i >= 2) dev::mbar_wait_sleep(&acc_empty[b], ((i >> 1) - 1) & 1);   // epilogue drained buffer b
        dev::tc_fence_after();
        const uint32_t acc = tmem + b * kGBN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kGStages;
          dev::mbar_wait_sleep(&full[s], (it / kGStages) & 1);
          dev::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kGBK / 16; ++kk)
            dev::umma_ss(acc, d0 + ((s * L::kStage + kk * 32) >> 4), e0 + ((s * L::kStage + kk * 16 * 128) >> 4),
                         idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          dev::umma_commit(&empty[s]);
        }
        dev::umma_commit(&acc_full[b]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: thread = output row m0 + 32*warp + lane; 256 fp32 columns from TMEM buffer b
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int b = i & 1;
      const int m0 = (t / p.n_tiles) * kGBM, nt0 = (t % p.n_tiles) * 2;
      const int ncols = nt0 + 1 < ntiles ? kGBN : 128;
      dev::mbar_wait_sleep(&acc_full[b], (i >> 1) & 1);
      dev::tc_fence_after();
      const int row = m0 + warp * 32 + lane;
      const uint32_t taddr = tmem + b * kGBN + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < ncols / 32; ++c) {
        uint32_t v[32];
        dev::tmem_ld32(taddr + c * 32, v);
        dev::tmem_wait_ld();
        if (c == ncols / 32 - 1) {  // every TMEM read of buffer b is done: release it
          dev::tc_fence_before();
          __syncwarp();
          if (lane == 0) dev::mbar_arrive(&acc_empty[b]);
        }
        store_row32(p, row, nt0 * 128 + c * 32, v);
      }
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- CTA-pair tile kernel (T > 128)
// A cluster of 2 CTAs (cta_group::2) computes one 256 x 256 output tile: each CTA loads its own
// 128 rows of X and ONE packed 128-column W tile per k-block (32 KiB per stage instead of 48),
// the leader CTA issues M=256 N=256 MMAs reading both CTAs' smem, and each CTA's TMEM holds its
// 128 rows x 256 columns.  Per-SM smem fill per FLOP drops by a third.  Persistent over pairs;
// both CTAs' loads complete on the leader's full barrier; the leader's commits multicast to
// both CTAs' empty / accumulator barriers; the peer's epilogue releases an accumulator with a
// remote arrive on the leader's barrier.
// f4 (QKV projection + RoPE + append, fused): the pair kernel's epilogue, per output row (token)
// and 128-column head of Y = X . W_qkv: q heads get RoPE and go to q_out (bf16); k heads get RoPE
// and go to the token's pool slot (bf16); v heads go to the pool slot as fp16 (R25).
struct QkvParams {
  const int32_t* qo_indptr;
  const int32_t* kv_len;
  const int32_t* page_indptr;
  const int32_t* page_ids;
  int num_seqs;
  uint16_t* kpool;          // this layer's K pages [num_pages][Hkv][16][128]
  uint16_t* vpool;
  uint16_t* q_out;          // [T][Hq][128]
  const float2* rope;       // [max_pos][64] (cos, sin), mux_rope_table
  int rope_max_pos;
  int hq, hkv;
  int* err;                 // pool error word (V range, position past the table)
};

constexpr int kHeadD = 128;

// y (128 fp32 of one head, one row) -> bf16 row at dst (16-byte stores)
__device__ __forceinline__ void store_head_bf16(uint16_t* dst, const float* y) {
#pragma unroll
  for (int i = 0; i < kHeadD / 8; ++i)
    reinterpret_cast<uint4*>(dst)[i] = make_uint4(dev::pack_bf16(y[8 * i], y[8 * i + 1]), dev::pack_bf16(y[8 * i + 2], y[8 * i + 3]),
                                                  dev::pack_bf16(y[8 * i + 4], y[8 * i + 5]), dev::pack_bf16(y[8 * i + 6], y[8 * i + 7]));
}

// RoPE (R26, Llama rotate-half): (y_c, y_{c+64}) rotated by angle pos * theta^(-2c/128)
__device__ __forceinline__ void rope_head(float* y, const float2* __restrict__ cs) {
#pragma unroll
  for (int c = 0; c < kHeadD / 2; ++c) {
    const float2 t = __ldg(cs + c);
    const float a = y[c], b = y[c + kHeadD / 2];
    y[c] = a * t.x - b * t.y;
    y[c + kHeadD / 2] = b * t.x + a * t.y;
  }
}

constexpr int kP2Stages = 6;
struct Gemm2Smem {
  static constexpr int kA = kGBM * kGBK * 2;          // 16 KiB: my 128 rows x 64 k
  static constexpr int kB = kPackTile;                // 16 KiB: my 128 columns x 64 k
  static constexpr int kStage = kA + kB;
  static constexpr int kBar = kP2Stages * kStage;
  static constexpr int kTmemSlot = kBar + (2 * kP2Stages + 4) * 8;
  static constexpr int kBytes = kTmemSlot + 16;
};

// EPI: 0 = plain Y store, 1 = fused QKV + RoPE + append (f4), 2 = SwiGLU gate/up (f4 FFN)
template <int EPI>
__global__ void __launch_bounds__(kGThreads, 1)
    outproj2_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                    const GemmParams p, const QkvParams qp) {
  using L = Gemm2Smem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + kP2Stages;
  uint64_t* acc_full = empty + kP2Stages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  const int warp = dev::warp_idx_uniform(), lane = threadIdx.x & 31;
  const uint32_t rank = dev::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nk = (p.K + kGBK - 1) / kGBK;
  const int KB = nk;
  const int ntiles128 = (p.N + 127) / 128;
  const int tiles = p.m_tiles * p.n_tiles;        // m_tiles counts 256-row tiles here

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kP2Stages + 2; ++i) dev::mbar_init(&full[i], 1);
    dev::mbar_init(&acc_empty[0], 8);             // 4 epilogue warps x 2 CTAs (leader's copy is used)
    dev::mbar_init(&acc_empty[1], 8);
    dev::fence_mbar_init();
  }
  if (warp == 5) dev::tmem_alloc_pair(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::cluster_sync();                            // both CTAs' barriers exist before any remote use
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t full_leader = dev::mapa(dev::smem_u32(full), 0);
  const uint32_t acc_empty_leader = dev::mapa(dev::smem_u32(acc_empty), 0);

  if (warp == 4) {
    if (lane == 0) {
      dev::tma_prefetch(&tmap_x);
      dev::tma_prefetch(&tmap_w);
      int it = 0;
      for (int t = pair; t < tiles; t += npairs) {
        const int m0 = (t / p.n_tiles) * 2 * kGBM + static_cast<int>(rank) * kGBM;
        const int wt = (t % p.n_tiles) * 2 + static_cast<int>(rank);   // my packed 128-column tile
        const int wtile = wt < ntiles128 ? wt : ntiles128 - 1;          // N tail: any valid tile (not stored)
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kP2Stages;
          if (it >= kP2Stages) dev::mbar_wait_sleep(&empty[s], ((it / kP2Stages) - 1) & 1);
          if (leader) dev::mbar_expect_tx(&full[s], 2 * L::kStage);      // both CTAs' bytes
          uint8_t* a = smem + s * L::kStage;
          const uint32_t fb = full_leader + s * 8;
          dev::tma_load_3d_pair(a, &tmap_x, fb, kb * kGBK, m0, 0);
          dev::tma_load_3d_pair(a + L::kA, &tmap_w, fb, 0, 0, wtile * KB + kb);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = dev::umma_idesc_bf16(2 * kGBM, kGBN, 0, 1);
      const uint64_t d0 = dev::umma_desc_sw128(dev::smem_u32(smem), 16, 1024);                   // A K-major
      const uint64_t e0 = dev::umma_desc_sw128(dev::smem_u32(smem + L::kA), kGBK * 128, 1024);  // B MN-major
      int it = 0, i = 0;
      for (int t = pair; t < tiles; t += npairs, ++i) {
        const int b = i & 1;
        if (i >= 2) dev::mbar_wait_sleep(&acc_empty[b], ((i >> 1) - 1) & 1);
        dev::tc_fence_after();
        const uint32_t acc = tmem + b * kGBN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kP2Stages;
          dev::mbar_wait_sleep(&full[s], (it / kP2Stages) & 1);
          dev::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kGBK / 16; ++kk)
            dev::umma_ss_pair(acc, d0 + ((s * L::kStage + kk * 32) >> 4), e0 + ((s * L::kStage + kk * 16 * 128) >> 4),
                              idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          dev::umma_commit_pair(&empty[s]);
        }
        dev::umma_commit_pair(&acc_full[b]);
      }
    }
    __syncwarp();
  } else if (EPI == 2) {
    // SwiGLU epilogue (both CTAs): W13 is packed with 128-column blocks of W1 and W3 interleaved,
    // so output tile n0 holds gate columns [n0/2, n0/2 + 128) then the matching up columns;
    // h = silu(gate) * up -> H[row][n0/2 + c] (bf16, row stride p.N / 2 = inter)
    int i = 0;
    for (int t = pair; t < tiles; t += npairs, ++i) {
      const int b = i & 1;
      const int m0 = (t / p.n_tiles) * 2 * kGBM + static_cast<int>(rank) * kGBM;
      const int n0 = (t % p.n_tiles) * kGBN;
      dev::mbar_wait_sleep(&acc_full[b], (i >> 1) & 1);
      dev::tc_fence_after();
      const int row = m0 + warp * 32 + lane;
      const uint32_t taddr = tmem + b * kGBN + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t g[32], u[32];
        dev::tmem_ld32(taddr + c * 32, g);
        dev::tmem_ld32(taddr + 128 + c * 32, u);
        dev::tmem_wait_ld();
        if (c == 3) {
          dev::tc_fence_before();
          __syncwarp();
          if (lane == 0) dev::mbar_arrive_cluster(acc_empty_leader + b * 8);
        }
        if (row >= p.T) continue;
        float hv[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float gv = __uint_as_float(g[k]);
          // silu(g) = g / (1 + e^-g)
          hv[k] = gv / (1.f + dev::ex2(-gv * 1.4426950408889634f)) * __uint_as_float(u[k]);
        }
        uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p.y) + static_cast<size_t>(row) * (p.N / 2) +
                                              n0 / 2 + c * 32);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          dst[k] = make_uint4(dev::pack_bf16(hv[8 * k], hv[8 * k + 1]), dev::pack_bf16(hv[8 * k + 2], hv[8 * k + 3]),
                              dev::pack_bf16(hv[8 * k + 4], hv[8 * k + 5]), dev::pack_bf16(hv[8 * k + 6], hv[8 * k + 7]));
      }
    }
  } else if (EPI == 1) {
    // fused QKV epilogue (both CTAs): my 128 rows (tokens) x 2 heads of TMEM buffer b
    int i = 0;
    for (int t = pair; t < tiles; t += npairs, ++i) {
      const int b = i & 1;
      const int m0 = (t / p.n_tiles) * 2 * kGBM + static_cast<int>(rank) * kGBM;
      const int n0 = (t % p.n_tiles) * kGBN;
      dev::mbar_wait_sleep(&acc_full[b], (i >> 1) & 1);
      dev::tc_fence_after();
      const int row = m0 + warp * 32 + lane;
      // the token's sequence, position and pool slot (as mux_append_kv)
      int pos = 0, page = 0;
      if (row < p.T) {
        int lo = 0, hi = qp.num_seqs - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (__ldg(qp.qo_indptr + mid) <= row) lo = mid; else hi = mid - 1;
        }
        const int q0 = __ldg(qp.qo_indptr + lo), n = __ldg(qp.qo_indptr + lo + 1) - q0;
        pos = __ldg(qp.kv_len + lo) - n + (row - q0);
        page = __ldg(qp.page_ids + __ldg(qp.page_indptr + lo) + (pos >> 4));
      }
      const bool pos_ok = pos < qp.rope_max_pos;
      if (row < p.T && !pos_ok && qp.err) atomicOr(qp.err, 2);
      const uint32_t taddr = tmem + b * kGBN + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int hh = 0; hh < kGBN / kHeadD; ++hh) {
        float y[kHeadD];
#pragma unroll
        for (int c = 0; c < kHeadD / 32; ++c) {
          dev::tmem_ld32(taddr + hh * kHeadD + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&y[32 * c]));
        }
        dev::tmem_wait_ld();
        if (hh == kGBN / kHeadD - 1) {
          dev::tc_fence_before();
          __syncwarp();
          if (lane == 0) dev::mbar_arrive_cluster(acc_empty_leader + b * 8);
        }
        const int gh = n0 / kHeadD + hh;             // global head column: q heads, k heads, v heads
        if (row >= p.T || gh >= qp.hq + 2 * qp.hkv) continue;
        if (gh < qp.hq + qp.hkv && pos_ok) rope_head(y, qp.rope + static_cast<size_t>(pos) * (kHeadD / 2));
        if (gh < qp.hq) {
          store_head_bf16(qp.q_out + (static_cast<size_t>(row) * qp.hq + gh) * kHeadD, y);
        } else if (gh < qp.hq + qp.hkv) {
          store_head_bf16(qp.kpool + ((static_cast<size_t>(page) * qp.hkv + (gh - qp.hq)) * kPage + (pos & 15)) * kHeadD, y);
        } else {
          uint16_t* dst = qp.vpool + ((static_cast<size_t>(page) * qp.hkv + (gh - qp.hq - qp.hkv)) * kPage + (pos & 15)) * kHeadD;
          bool big = false;
#pragma unroll
          for (int c = 0; c < kHeadD; ++c) big |= fabsf(y[c]) > 65504.f;
          if (big && qp.err) atomicOr(qp.err, MUX_POOL_ERR_V_RANGE);
#pragma unroll
          for (int k = 0; k < kHeadD / 8; ++k)
            reinterpret_cast<uint4*>(dst)[k] =
                make_uint4(dev::pack_f16_satfinite(y[8 * k], y[8 * k + 1]), dev::pack_f16_satfinite(y[8 * k + 2], y[8 * k + 3]),
                           dev::pack_f16_satfinite(y[8 * k + 4], y[8 * k + 5]), dev::pack_f16_satfinite(y[8 * k + 6], y[8 * k + 7]));
        }
      }
    }
  } else {
    // epilogue (both CTAs): my 128 rows x 256 columns of TMEM buffer b
    int i = 0;
    for (int t = pair; t < tiles; t += npairs, ++i) {
      const int b = i & 1;
      const int m0 = (t / p.n_tiles) * 2 * kGBM + static_cast<int>(rank) * kGBM;
      const int n0 = (t % p.n_tiles) * kGBN;
      const int ncols = n0 + 128 < p.N ? kGBN : 128;
      dev::mbar_wait_sleep(&acc_full[b], (i >> 1) & 1);
      dev::tc_fence_after();
      const int row = m0 + warp * 32 + lane;
      const uint32_t taddr = tmem + b * kGBN + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < kGBN / 32; ++c) {
        uint32_t v[32];
        dev::tmem_ld32(taddr + c * 32, v);
        dev::tmem_wait_ld();
        if (c == kGBN / 32 - 1) {
          dev::tc_fence_before();
          __syncwarp();
          if (lane == 0) dev::mbar_arrive_cluster(acc_empty_leader + b * 8);
        }
        if (c * 32 < ncols) store_row32(p, row, n0 + c * 32, v);
      }
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  dev::cluster_sync();
  if (warp == 5) {
    dev::tc_fence_after();
    dev::tmem_dealloc_pair(tmem, 512);
  }
}

// ---------------------------------------------------------------- skinny (T <= 128)
// stage = KS consecutive k-blocks: KS packed W tiles (ONE contiguous KS x 16 KiB bulk copy) +
// KS X boxes of TN x 128 B; as many stages as fit ~200 KiB
constexpr int kSMaxStages = 12;
constexpr int kSkinnyRing = 200 * 1024;

__host__ __device__ inline int skinny_stage_bytes(int TN, int ks) { return ks * (kPackTile + TN * kGBK * 2); }
__host__ __device__ inline int skinny_stages(int TN, int ks) {
  const int s = kSkinnyRing / skinny_stage_bytes(TN, ks);
  return s < kSMaxStages ? s : kSMaxStages;
}
constexpr int kSkinnySmemMax = kSkinnyRing + (2 * kSMaxStages + 1) * 8 + 16 + 1024;

struct SkinnyParams {
  void* y;
  const uint8_t* w_pk;
  int T, N, K, TN, ks, y_f32;
};

__global__ void __launch_bounds__(kGThreads, 1)
    outproj_skinny_kernel(const __grid_constant__ CUtensorMap tmap_x, const SkinnyParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int ks = p.ks;
  const int stage_bytes = skinny_stage_bytes(p.TN, ks), nst = skinny_stages(p.TN, ks);
  const int x_off = ks * kPackTile;                      // X boxes follow the W tiles in a stage
  const uint32_t x_box = static_cast<uint32_t>(p.TN) * kGBK * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * stage_bytes);
  uint64_t* empty = full + kSMaxStages;
  uint64_t* acc_full = empty + kSMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = dev::warp_idx_uniform(), lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128;
  const int nk = (p.K + kGBK - 1) / kGBK;
  const int nstage = (nk + ks - 1) / ks;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kSMaxStages + 1; ++i) dev::mbar_init(&full[i], 1);
    dev::fence_mbar_init();
  }
  if (warp == 5) dev::tmem_alloc(tmem_slot, 128);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      dev::tma_prefetch(&tmap_x);
      const uint8_t* wt = p.w_pk + static_cast<size_t>(blockIdx.x) * nk * kPackTile;
      for (int i = 0; i < nstage; ++i) {
        const int s = i % nst, kb = i * ks, cnt = min(ks, nk - kb);
        if (i >= nst) dev::mbar_wait_sleep(&empty[s], ((i / nst) - 1) & 1);
        dev::mbar_expect_tx(&full[s], cnt * (kPackTile + x_box));
        uint8_t* a = smem + s * stage_bytes;
        dev::bulk_load(a, wt + static_cast<size_t>(kb) * kPackTile, cnt * kPackTile, &full[s]);
        for (int j = 0; j < cnt; ++j) dev::tma_load_3d(a + x_off + j * x_box, &tmap_x, &full[s], (kb + j) * kGBK, 0, 0);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      const uint32_t idesc = dev::umma_idesc_bf16(128, p.TN, 1, 0);
      const uint64_t d0 = dev::umma_desc_sw128(dev::smem_u32(smem), kGBK * 128, 1024);       // A = W^T, MN-major
      const uint64_t e0 = dev::umma_desc_sw128(dev::smem_u32(smem + x_off), 16, 1024);       // B = X^T, K-major
      for (int i = 0; i < nstage; ++i) {
        const int s = i % nst, cnt = min(ks, nk - i * ks);
        dev::mbar_wait_sleep(&full[s], (i / nst) & 1);
        dev::tc_fence_after();
        for (int j = 0; j < cnt; ++j)
#pragma unroll
          for (int kk = 0; kk < kGBK / 16; ++kk)
            dev::umma_ss(tmem, d0 + ((s * stage_bytes + j * kPackTile + kk * 16 * 128) >> 4),
                         e0 + ((s * stage_bytes + j * x_box + kk * 32) >> 4), idesc, (i > 0 || j > 0 || kk > 0) ? 1u : 0u);
        dev::umma_commit(&empty[s]);
      }
      dev::umma_commit(acc_full);
    }
    __syncwarp();
  } else {
    // epilogue: TMEM lane = output column n0 + 32*warp + lane, TMEM column = token t; a warp
    // stores 32 consecutive columns of one token row per instruction
    dev::mbar_wait_sleep(acc_full, 0);
    dev::tc_fence_after();
    const int col = n0 + warp * 32 + lane;
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
    for (int c = 0; c * 32 < p.TN; ++c) {
      uint32_t v[32];
      dev::tmem_ld32(taddr + c * 32, v);
      dev::tmem_wait_ld();
      if (col < p.N) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int t = c * 32 + j;
          if (t < p.T) {
            const size_t off = static_cast<size_t>(t) * p.N + col;
            const float f = __uint_as_float(v[j]);
            if (p.y_f32)
              static_cast<float*>(p.y)[off] = f;
            else
              static_cast<uint16_t*>(p.y)[off] = static_cast<uint16_t>(dev::pack_bf16(f, 0.f) & 0xFFFFu);
          }
        }
      }
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 128);
  }
}

// ---------------------------------------------------------------- weight packing
// one thread per 16-byte chunk of the packed image: (tile, half, row k, stored chunk position)
__global__ void pack_w_kernel(const uint16_t* __restrict__ w, uint4* __restrict__ out, int K, int N, int KB,
                              size_t nchunks) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nchunks;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int pos = static_cast<int>(i & 7);           // stored chunk position within the 128 B row
    const int k = static_cast<int>((i >> 3) & 63);      // row = k within the tile
    const int half = static_cast<int>((i >> 9) & 1);    // n 0-63 / 64-127 of the tile
    const size_t tile = i >> 10;                        // nt * KB + kb
    const int kb = static_cast<int>(tile % KB), nt = static_cast<int>(tile / KB);
    const int c = pos ^ (k & 7);                        // logical chunk (8 columns)
    const int n = nt * 128 + half * 64 + c * 8, kk = kb * kGBK + k;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (kk < K && n < N) v = *reinterpret_cast<const uint4*>(w + static_cast<size_t>(kk) * N + n);
    out[i] = v;
  }
}

}  // namespace
}  // namespace mux

using namespace mux;

extern "C" size_t mux_outproj_packed_bytes(int32_t K, int32_t N) {
  if (K < 1 || N < 1) return 0;
  return static_cast<size_t>((N + 127) / 128) * ((K + kGBK - 1) / kGBK) * kPackTile;
}

extern "C" int mux_outproj_pack_w(const void* w, void* w_packed, int32_t K, int32_t N, mux_stream_t stream) {
  if (!w || !w_packed) return fail(MUX_ERR_INVALID_ARG, "mux_outproj_pack_w: NULL pointer");
  if (K < 1 || N < 1) return fail(MUX_ERR_INVALID_ARG, "mux_outproj_pack_w: K, N must be >= 1");
  if (N % 8) return fail(MUX_ERR_UNSUPPORTED, "mux_outproj_pack_w: N must be a multiple of 8");
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(w_packed)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "mux_outproj_pack_w: pointers must be 16-byte aligned");
  const size_t nchunks = mux_outproj_packed_bytes(K, N) / 16;
  const int blocks = static_cast<int>(std::min<size_t>((nchunks + 255) / 256, 148 * 16));
  pack_w_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(w), static_cast<uint4*>(w_packed), K, N, (K + kGBK - 1) / kGBK, nchunks);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

namespace mux {
// num_sms: SMs the launch may occupy (the side's partition); <= 0 = the whole device
int outproj_launch(const void* x, const void* w, void* y, int32_t y_dtype, int32_t T, int32_t K, int32_t N,
                   mux_stream_t stream, int num_sms) {
  if (!x || !w || !y) return fail(MUX_ERR_INVALID_ARG, "mux_outproj: NULL pointer");
  if (T < 1 || K < 1 || N < 1) return fail(MUX_ERR_INVALID_ARG, "mux_outproj: T, K, N must be >= 1");
  if (y_dtype != MUX_DTYPE_BF16 && y_dtype != MUX_DTYPE_F32) return fail(MUX_ERR_INVALID_ARG, "bad y_dtype");
  if ((K % 8) || (N % 8)) return fail(MUX_ERR_UNSUPPORTED, "mux_outproj: K and N must be multiples of 8");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(y)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "mux_outproj: pointers must be 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint8_t* wp = static_cast<const uint8_t*>(w);
  // X [T][K] -> K-major boxes {64 k, rows}
  CUtensorMap tx;
  uint64_t dx[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(T), 1};
  uint64_t sx[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K) * T * 2};
  if (T <= 128) {
    const int TN = T <= 32 ? 32 : (T <= 64 ? 64 : 128);
    uint32_t bx[3] = {kGBK, static_cast<uint32_t>(TN), 1};
    int rc = make_tmap_bf16(&tx, x, 3, dx, sx, bx);
    if (rc) return rc;
    static bool attr_done = false;
    if (!attr_done) {
      MUX_CUDA(cudaFuncSetAttribute(outproj_skinny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kSkinnySmemMax));
      attr_done = true;
    }
    // k-blocks per stage: the largest that still leaves >= 2 stages in the ring (fewer, bigger
    // copies and barrier round trips: 17.6 us at ks 4 vs 22.3 at ks 2 and 31.5 at ks 1 for
    // T=64, K=N=4096 on 32 CTAs, scripts/skinny_dbg.py)
    const int ks = TN <= 64 ? 4 : 2;
    SkinnyParams sp{y, wp, T, N, K, TN, ks, y_dtype == MUX_DTYPE_F32};
    outproj_skinny_kernel<<<(N + 127) / 128, kGThreads, kSkinnySmemMax, st>>>(tx, sp);
    MUX_CUDA(cudaGetLastError());
    return MUX_OK;
  }
  uint32_t bx[3] = {kGBK, kGBM, 1};
  int rc = make_tmap_bf16(&tx, x, 3, dx, sx, bx);
  if (rc) return rc;
  static const bool single_only = getenv("MUX_OUTPROJ_SINGLE") != nullptr;  // developer A/B switch
  const int sms_avail = num_sms > 0 ? num_sms : device_sm_count();
  if (!single_only && sms_avail >= 2) {
    // packed W as {64 elements, 128 rows, tiles}: one box = one 16 KiB tile image (no swizzle:
    // the image is already in the SWIZZLE_128B layout)
    const int KB = (K + kGBK - 1) / kGBK, NT = (N + 127) / 128;
    CUtensorMap tw;
    uint64_t dw[3] = {64, 128, static_cast<uint64_t>(KB) * NT};
    uint64_t sw[2] = {128, 16384};
    uint32_t bw[3] = {64, 128, 1};
    if ((rc = make_tmap_bf16(&tw, w, 3, dw, sw, bw, false))) return rc;
    static bool attr2 = false;
    const int smem2 = Gemm2Smem::kBytes + 1024;
    if (!attr2) {
      MUX_CUDA(cudaFuncSetAttribute(outproj2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
      attr2 = true;
    }
    GemmParams prm{y, wp, T, N, K, y_dtype == MUX_DTYPE_F32, (T + 2 * kGBM - 1) / (2 * kGBM), (N + kGBN - 1) / kGBN};
    const int tiles = prm.m_tiles * prm.n_tiles;
    const int sms = num_sms > 0 ? num_sms : device_sm_count();
    const int pairs = std::max(1, std::min(tiles, sms / 2));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = smem2;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, outproj2_kernel<0>, tx, tw, prm, QkvParams{});
    if (e == cudaSuccess) return MUX_OK;
    (void)cudaGetLastError();  // no CTA pairs on this partition: fall back to the single-CTA kernel
  }
  static bool attr_done = false;
  const int smem = GemmSmem::kBytes + 1024;
  if (!attr_done) {
    MUX_CUDA(cudaFuncSetAttribute(outproj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_done = true;
  }
  GemmParams prm{y, wp, T, N, K, y_dtype == MUX_DTYPE_F32, (T + kGBM - 1) / kGBM, (N + kGBN - 1) / kGBN};
  const int tiles = prm.m_tiles * prm.n_tiles;
  const int sms = num_sms > 0 ? num_sms : device_sm_count();
  outproj_kernel<<<std::min(tiles, std::max(sms, 1)), kGThreads, smem, st>>>(tx, prm);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
}  // namespace mux

// ---------------------------------------------------------------- f4: RoPE table + fused QKV launch
namespace mux {
namespace {
// (cos, sin) of pos * theta^(-2c/d) for c < d/2, computed in double and rounded to fp32 once
__global__ void rope_table_kernel(float2* t, int max_pos, int half, double theta) {
  const size_t n = static_cast<size_t>(max_pos) * half;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int pos = static_cast<int>(i / half), c = static_cast<int>(i % half);
    const double a = pos * pow(theta, -2.0 * c / (2.0 * half));
    double sn, cs;
    sincos(a, &sn, &cs);
    t[i] = make_float2(static_cast<float>(cs), static_cast<float>(sn));
  }
}
}  // namespace
}  // namespace mux

extern "C" size_t mux_rope_table_bytes(int32_t max_pos, int32_t head_dim) {
  if (max_pos < 1 || head_dim < 2) return 0;
  return static_cast<size_t>(max_pos) * (head_dim / 2) * sizeof(float2);
}

extern "C" int mux_rope_table(void* table, int32_t max_pos, int32_t head_dim, double theta, mux_stream_t stream) {
  if (!table || max_pos < 1 || head_dim != 128 || !(theta > 1.0))
    return mux::fail(MUX_ERR_INVALID_ARG, "mux_rope_table: table, max_pos >= 1, head_dim 128, theta > 1 required");
  const size_t n = static_cast<size_t>(max_pos) * (head_dim / 2);
  const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 4096));
  mux::rope_table_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(static_cast<float2*>(table),
                                                                                    max_pos, head_dim / 2, theta);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

namespace mux {
int qkv_launch(mux_pool_t pool, int32_t layer, const mux_batch* b, int32_t hq, const void* x, int32_t hidden,
               const void* w_qkv, const void* rope, int32_t rope_max_pos, void* q_out, mux_stream_t stream,
               int num_sms) {
  int rc = check_pool_layer(pool, layer);
  if (rc) return rc;
  if ((rc = validate_batch(b, false))) return rc;
  const int d = pool->desc.head_dim, hkv = pool->desc.num_kv_heads;
  if (d != kHeadD) return fail(MUX_ERR_UNSUPPORTED, "mux_qkv_rope_append: head_dim must be 128");
  if (hq < 2 || hq % hkv || (hq & 1) || (hkv & 1))
    return fail(MUX_ERR_UNSUPPORTED, "mux_qkv_rope_append: Hq, Hkv even and Hq a multiple of Hkv");
  if (!x || !w_qkv || !rope || !q_out) return fail(MUX_ERR_INVALID_ARG, "mux_qkv_rope_append: NULL pointer");
  if (hidden < 8 || hidden % 8) return fail(MUX_ERR_UNSUPPORTED, "mux_qkv_rope_append: hidden must be a multiple of 8");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w_qkv) | reinterpret_cast<uintptr_t>(q_out)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "mux_qkv_rope_append: pointers must be 16-byte aligned");
  if (b->h_kv_len)
    for (int s2 = 0; s2 < b->num_seqs; ++s2)
      if (b->h_kv_len[s2] > rope_max_pos) return fail(MUX_ERR_INVALID_ARG, "position past the RoPE table");
  if ((rc = append_checks(pool, b))) return rc;
  if ((rc = pool_tmaps(pool))) return rc;
  const int T = b->total_q, K = hidden, N = (hq + 2 * hkv) * d;
  CUtensorMap tx, tw;
  uint64_t dx[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(T), 1};
  uint64_t sx[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K) * T * 2};
  uint32_t bx[3] = {kGBK, kGBM, 1};
  if ((rc = make_tmap_bf16(&tx, x, 3, dx, sx, bx))) return rc;
  const int KB = (K + kGBK - 1) / kGBK, NT = (N + 127) / 128;
  uint64_t dw[3] = {64, 128, static_cast<uint64_t>(KB) * NT};
  uint64_t sw[2] = {128, 16384};
  uint32_t bw[3] = {64, 128, 1};
  if ((rc = make_tmap_bf16(&tw, w_qkv, 3, dw, sw, bw, false))) return rc;
  static bool attr = false;
  const int smem2 = Gemm2Smem::kBytes + 1024;
  if (!attr) {
    MUX_CUDA(cudaFuncSetAttribute(outproj2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    attr = true;
  }
  GemmParams prm{nullptr, static_cast<const uint8_t*>(w_qkv), T, N, K, 0, (T + 2 * kGBM - 1) / (2 * kGBM),
                 (N + kGBN - 1) / kGBN};
  const size_t off = static_cast<size_t>(layer) * pool->layer_elems();
  QkvParams qp{b->qo_indptr, b->kv_len, b->page_indptr, b->page_ids, b->num_seqs,
               static_cast<uint16_t*>(pool->desc.k_storage) + off, static_cast<uint16_t*>(pool->desc.v_storage) + off,
               static_cast<uint16_t*>(q_out), static_cast<const float2*>(rope), rope_max_pos, hq, hkv, pool->d_err};
  const int tiles = prm.m_tiles * prm.n_tiles;
  const int pairs = std::max(1, std::min(tiles, (num_sms > 0 ? num_sms : device_sm_count()) / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = smem2;
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MUX_CUDA(cudaLaunchKernelEx(&cfg, outproj2_kernel<1>, tx, tw, prm, qp));
  return MUX_OK;
}
}  // namespace mux

extern "C" int mux_qkv_rope_append(mux_pool_t pool, int32_t layer, const mux_batch* b, int32_t hq, const void* x,
                                   int32_t hidden, const void* w_qkv, const void* rope, int32_t rope_max_pos,
                                   void* q_out, mux_stream_t stream) {
  return mux::qkv_launch(pool, layer, b, hq, x, hidden, w_qkv, rope, rope_max_pos, q_out, stream, 0);
}

// ---------------------------------------------------------------- f4: SwiGLU FFN (gate/up fused)
namespace mux {
namespace {
// W13 [K][2 inter] with 128-column blocks of W1 and W3 interleaved, written in the packed tile image
__global__ void pack_w13_kernel(const uint16_t* __restrict__ w1, const uint16_t* __restrict__ w3,
                                uint4* __restrict__ out, int K, int inter, int KB, size_t nchunks) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < nchunks;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int pos = static_cast<int>(i & 7);
    const int k = static_cast<int>((i >> 3) & 63);
    const int half = static_cast<int>((i >> 9) & 1);
    const size_t tile = i >> 10;
    const int kb = static_cast<int>(tile % KB), nt = static_cast<int>(tile / KB);
    const int c = pos ^ (k & 7);
    const int n = nt * 128 + half * 64 + c * 8, kk = kb * kGBK + k;   // column of W13
    const uint16_t* src = (n / 128) & 1 ? w3 : w1;                     // odd 128-blocks: W3
    const int col = (n / 256) * 128 + (n % 128);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (kk < K && col < inter) v = *reinterpret_cast<const uint4*>(src + static_cast<size_t>(kk) * inter + col);
    out[i] = v;
  }
}
}  // namespace
}  // namespace mux

extern "C" size_t mux_ffn_w13_packed_bytes(int32_t hidden, int32_t inter) {
  return mux_outproj_packed_bytes(hidden, 2 * inter);
}

extern "C" int mux_ffn_pack_w13(const void* w1, const void* w3, void* w13_packed, int32_t hidden, int32_t inter,
                                mux_stream_t stream) {
  using namespace mux;
  if (!w1 || !w3 || !w13_packed) return fail(MUX_ERR_INVALID_ARG, "mux_ffn_pack_w13: NULL pointer");
  if (hidden < 1 || inter < 128 || inter % 128) return fail(MUX_ERR_UNSUPPORTED, "mux_ffn_pack_w13: inter % 128 == 0");
  if ((reinterpret_cast<uintptr_t>(w1) | reinterpret_cast<uintptr_t>(w3) | reinterpret_cast<uintptr_t>(w13_packed)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "mux_ffn_pack_w13: pointers must be 16-byte aligned");
  const size_t nchunks = mux_ffn_w13_packed_bytes(hidden, inter) / 16;
  const int blocks = static_cast<int>(std::min<size_t>((nchunks + 255) / 256, 148 * 16));
  pack_w13_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(w1), static_cast<const uint16_t*>(w3), static_cast<uint4*>(w13_packed), hidden,
      inter, (hidden + kGBK - 1) / kGBK, nchunks);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

namespace mux {
int ffn_launch(const void* x, const void* w13_packed, const void* w2_packed, void* h, void* y, int32_t T,
               int32_t hidden, int32_t inter, mux_stream_t stream, int num_sms) {
  if (!x || !w13_packed || !w2_packed || !h || !y) return fail(MUX_ERR_INVALID_ARG, "mux_ffn_swiglu: NULL pointer");
  if (T < 1 || hidden < 8 || hidden % 8 || inter < 128 || inter % 128)
    return fail(MUX_ERR_UNSUPPORTED, "mux_ffn_swiglu: T >= 1, hidden % 8 == 0, inter % 128 == 0");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(y)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "mux_ffn_swiglu: pointers must be 16-byte aligned");
  const int K = hidden, N = 2 * inter;
  CUtensorMap tx, tw;
  uint64_t dx[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(T), 1};
  uint64_t sx[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K) * T * 2};
  uint32_t bx[3] = {kGBK, kGBM, 1};
  int rc;
  if ((rc = make_tmap_bf16(&tx, x, 3, dx, sx, bx))) return rc;
  const int KB = (K + kGBK - 1) / kGBK, NT = N / 128;
  uint64_t dw[3] = {64, 128, static_cast<uint64_t>(KB) * NT};
  uint64_t sw[2] = {128, 16384};
  uint32_t bw[3] = {64, 128, 1};
  if ((rc = make_tmap_bf16(&tw, w13_packed, 3, dw, sw, bw, false))) return rc;
  static bool attr = false;
  const int smem2 = Gemm2Smem::kBytes + 1024;
  if (!attr) {
    MUX_CUDA(cudaFuncSetAttribute(outproj2_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
    attr = true;
  }
  // N = 2 inter columns of W13; the epilogue writes H [T][inter] (bf16)
  GemmParams prm{h, static_cast<const uint8_t*>(w13_packed), T, N, K, 0, (T + 2 * kGBM - 1) / (2 * kGBM), N / kGBN};
  const int tiles = prm.m_tiles * prm.n_tiles;
  const int pairs = std::max(1, std::min(tiles, (num_sms > 0 ? num_sms : device_sm_count()) / 2));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = smem2;
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MUX_CUDA(cudaLaunchKernelEx(&cfg, outproj2_kernel<2>, tx, tw, prm, QkvParams{}));
  // down projection: Y = H . W2 (the plain GEMM)
  return outproj_launch(h, w2_packed, y, MUX_DTYPE_BF16, T, inter, hidden, stream, num_sms);
}
}  // namespace mux

extern "C" int mux_ffn_swiglu(const void* x, const void* w13_packed, const void* w2_packed, void* h, void* y,
                              int32_t T, int32_t hidden, int32_t inter, mux_stream_t stream) {
  return mux::ffn_launch(x, w13_packed, w2_packed, h, y, T, hidden, inter, stream, 0);
}

extern "C" int mux_outproj(const void* x, const void* w, void* y, int32_t y_dtype, int32_t T, int32_t K, int32_t N,
                           mux_stream_t stream) {
  return mux::outproj_launch(x, w, y, y_dtype, T, K, N, stream, 0);
}

extern "C" int mux_outproj_sms(const void* x, const void* w, void* y, int32_t y_dtype, int32_t T, int32_t K,
                               int32_t N, mux_stream_t stream, int32_t num_sms) {
  return mux::outproj_launch(x, w, y, y_dtype, T, K, N, stream, num_sms);
}
