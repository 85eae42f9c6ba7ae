// a7 building block: out-projection partial GEMM  Y[T][N] = X[T][K] . W[K][N]  (tcgen05).
//
// PAPER: MuxWise serves Llama-70B with tensor parallelism of degree 8 over NVLink
// (P:686); under KV-head sharding each GPU holds Hq/G q heads, so its attention
// output X = O_local [T][Hq/G * d] times its row shard of W_o gives a partial sum of the layer
// output that an all-reduce completes.  This kernel is that per-GPU GEMM (bf16 in, fp32
// accumulate in TMEM, bf16 or fp32 out); the all-reduce runs on the side's NCCL communicator.
//
// B200 design: one CTA per 128 x 256 output tile, 6 warps: warp 4 = TMA producer, warp 5 =
// TMEM owner + single-thread tcgen05.mma issuer, warps 0-3 = epilogue (thread = output row).
// 4-stage ring of {A: 128 rows x 64 k (K-major, SWIZZLE_128B), B: 64 k x 256 n (MN-major,
// 4 boxes of 64 n)}, 48 KiB per stage; 4 MMAs (M=128, N=256, K=16) per stage; rows / columns
// past T / N come from out-of-bounds TMA zero fill and are not stored.
//
// Skinny variant (T <= 128, the decode side: one token per sequence): the 128-row M tile would
// be mostly zero fill and N/256 CTAs too few to stream W_o at the partition's bandwidth, so the
// kernel computes the transpose  Y^T = W^T . X^T  instead: M = 128 columns of W (A operand
// MN-major, straight from W's row-major layout), N = T rounded up to 32 (B = X, K-major), one
// CTA per 128 columns of W, 6-stage ring, stored directly from TMEM (no split-K: the
// result stays bitwise deterministic).
#include "pool.h"

namespace mux {
namespace {

constexpr int kGBM = 128, kGBN = 256, kGBK = 64, kGStages = 4;
constexpr int kGThreads = 192;

struct GemmSmem {
  static constexpr int kA = kGBM * kGBK * 2;          // 16 KiB
  static constexpr int kB = kGBK * kGBN * 2;          // 32 KiB
  static constexpr int kStage = kA + kB;
  static constexpr int kBar = kGStages * kStage;
  static constexpr int kTmemSlot = kBar + (2 * kGStages + 1) * 8;
  static constexpr int kBytes = kTmemSlot + 16;
};

struct GemmParams {
  void* y;
  int T, N, K, y_f32;
};

__global__ void __launch_bounds__(kGThreads, 1)
    outproj_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                   const GemmParams p) {
  using L = GemmSmem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + kGStages;
  uint64_t* acc_full = empty + kGStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  const int warp = dev::warp_idx_uniform(), lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kGBM, n0 = blockIdx.x * kGBN;
  const int nk = (p.K + kGBK - 1) / kGBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kGStages + 1; ++i) dev::mbar_init(&full[i], 1);
    dev::fence_mbar_init();
  }
  if (warp == 5) dev::tmem_alloc(tmem_slot, 256);
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (lane == 0) {
      dev::tma_prefetch(&tmap_x);
      dev::tma_prefetch(&tmap_w);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kGStages;
        if (kb >= kGStages) dev::mbar_wait_sleep(&empty[s], ((kb / kGStages) - 1) & 1);
        dev::mbar_expect_tx(&full[s], L::kStage);
        uint8_t* a = smem + s * L::kStage;
        uint8_t* bt = a + L::kA;
        dev::tma_load_3d(a, &tmap_x, &full[s], kb * kGBK, m0, 0);
#pragma unroll
        for (int nb = 0; nb < kGBN / 64; ++nb)
          dev::tma_load_3d(bt + nb * (kGBK * 128), &tmap_w, &full[s], n0 + nb * 64, kb * kGBK, 0);
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {
      constexpr uint32_t idesc = dev::umma_idesc_bf16(kGBM, kGBN, 0, 1);
      const uint64_t d0 = dev::umma_desc_sw128(dev::smem_u32(smem), 16, 1024);                      // A K-major
      const uint64_t e0 = dev::umma_desc_sw128(dev::smem_u32(smem + L::kA), kGBK * 128, 1024);     // B MN-major
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kGStages;
        dev::mbar_wait_sleep(&full[s], (kb / kGStages) & 1);
        dev::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kGBK / 16; ++kk)
          dev::umma_ss(tmem, d0 + ((s * L::kStage + kk * 32) >> 4), e0 + ((s * L::kStage + kk * 16 * 128) >> 4), idesc,
                       (kb > 0 || kk > 0) ? 1u : 0u);
        dev::umma_commit(&empty[s]);
      }
      dev::umma_commit(acc_full);
    }
    __syncwarp();
  } else {
    // epilogue: thread = output row m0 + 32*warp + lane; 256 fp32 columns from TMEM
    dev::mbar_wait_sleep(acc_full, 0);
    dev::tc_fence_after();
    const int row = m0 + warp * 32 + lane;
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < kGBN / 32; ++c) {
      uint32_t v[32];
      dev::tmem_ld32(taddr + c * 32, v);
      dev::tmem_wait_ld();
      const int col = n0 + c * 32;
      if (row < p.T) {
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
            for (int i = 0; i < 32 && col + i < p.N; ++i) {
              const uint32_t pk = dev::pack_bf16(__uint_as_float(v[i]), 0.f);
              dst[i] = static_cast<uint16_t>(pk & 0xFFFFu);
            }
          }
        }
      }
    }
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    dev::tc_fence_after();
    dev::tmem_dealloc(tmem, 256);
  }
}

constexpr int kSStages = 6;

struct SkinnySmem {
  static constexpr int kA = 128 * kGBK * 2;           // 16 KiB: 64 k x 128 n of W (2 boxes of 64 n)
  static constexpr int kB = 128 * kGBK * 2;           // up to 128 t x 64 k of X
  static constexpr int kStage = kA + kB;
  static constexpr int kBar = kSStages * kStage;
  static constexpr int kTmemSlot = kBar + (2 * kSStages + 1) * 8;
  static constexpr int kBytes = kTmemSlot + 16;
};

struct SkinnyParams {
  void* y;
  int T, N, K, TN, kb_per_split, y_f32, atomic;
};

__global__ void __launch_bounds__(kGThreads, 1)
    outproj_skinny_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                          const SkinnyParams p) {
  using L = SkinnySmem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + kSStages;
  uint64_t* acc_full = empty + kSStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  const int warp = dev::warp_idx_uniform(), lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 128;
  const int nk_total = (p.K + kGBK - 1) / kGBK;
  const int kb0 = blockIdx.y * p.kb_per_split;
  const int kb1 = min(nk_total, kb0 + p.kb_per_split);
  const int nk = kb1 - kb0;
  const uint32_t b_bytes = static_cast<uint32_t>(p.TN) * kGBK * 2;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kSStages + 1; ++i) dev::mbar_init(&full[i], 1);
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
      dev::tma_prefetch(&tmap_w);
      for (int i = 0; i < nk; ++i) {
        const int s = i % kSStages, kb = kb0 + i;
        if (i >= kSStages) dev::mbar_wait_sleep(&empty[s], ((i / kSStages) - 1) & 1);
        dev::mbar_expect_tx(&full[s], L::kA + b_bytes);
        uint8_t* a = smem + s * L::kStage;
        dev::tma_load_3d(a, &tmap_w, &full[s], n0, kb * kGBK, 0);
        dev::tma_load_3d(a + kGBK * 128, &tmap_w, &full[s], n0 + 64, kb * kGBK, 0);
        dev::tma_load_3d(a + L::kA, &tmap_x, &full[s], kb * kGBK, 0, 0);
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && nk > 0) {
      const uint32_t idesc = dev::umma_idesc_bf16(128, p.TN, 1, 0);
      const uint64_t d0 = dev::umma_desc_sw128(dev::smem_u32(smem), kGBK * 128, 1024);      // A = W^T, MN-major
      const uint64_t e0 = dev::umma_desc_sw128(dev::smem_u32(smem + L::kA), 16, 1024);      // B = X^T, K-major
      for (int i = 0; i < nk; ++i) {
        const int s = i % kSStages;
        dev::mbar_wait_sleep(&full[s], (i / kSStages) & 1);
        dev::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kGBK / 16; ++kk)
          dev::umma_ss(tmem, d0 + ((s * L::kStage + kk * 16 * 128) >> 4), e0 + ((s * L::kStage + kk * 32) >> 4), idesc,
                       (i > 0 || kk > 0) ? 1u : 0u);
        dev::umma_commit(&empty[s]);
      }
      dev::umma_commit(acc_full);
    }
    __syncwarp();
  } else if (nk > 0) {
    // epilogue: TMEM lane = output column n0 + 32*warp + lane, TMEM column = token t
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
            if (p.atomic)
              atomicAdd(static_cast<float*>(p.y) + off, f);
            else if (p.y_f32)
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

}  // namespace
}  // namespace mux

using namespace mux;


extern "C" int mux_outproj(const void* x, const void* w, void* y, int32_t y_dtype, int32_t T, int32_t K, int32_t N,
                           mux_stream_t stream) {
  if (!x || !w || !y) return fail(MUX_ERR_INVALID_ARG, "mux_outproj: NULL pointer");
  if (T < 1 || K < 1 || N < 1) return fail(MUX_ERR_INVALID_ARG, "mux_outproj: T, K, N must be >= 1");
  if (y_dtype != MUX_DTYPE_BF16 && y_dtype != MUX_DTYPE_F32) return fail(MUX_ERR_INVALID_ARG, "bad y_dtype");
  if ((K % 8) || (N % 8)) return fail(MUX_ERR_UNSUPPORTED, "mux_outproj: K and N must be multiples of 8");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(y)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "mux_outproj: pointers must be 16-byte aligned");
  // X [T][K] -> K-major A boxes {64 k, 128 rows}; W [K][N] -> MN-major B boxes {64 n, 64 k}
  CUtensorMap tx, tw;
  uint64_t dx[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(T), 1};
  uint64_t sx[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K) * T * 2};
  uint32_t bx[3] = {kGBK, kGBM, 1};
  int rc = make_tmap_bf16(&tx, x, 3, dx, sx, bx);
  if (rc) return rc;
  uint64_t dw[3] = {static_cast<uint64_t>(N), static_cast<uint64_t>(K), 1};
  uint64_t sw[2] = {static_cast<uint64_t>(N) * 2, static_cast<uint64_t>(N) * K * 2};
  uint32_t bw[3] = {64, kGBK, 1};
  if ((rc = make_tmap_bf16(&tw, w, 3, dw, sw, bw))) return rc;
  static bool attr_done = false;
  const int smem = GemmSmem::kBytes + 1024;
  if (!attr_done) {
    MUX_CUDA(cudaFuncSetAttribute(outproj_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_done = true;
  }
  if (T <= 128) {
    const int TN = T <= 32 ? 32 : (T <= 64 ? 64 : 128);
    uint32_t bxs[3] = {kGBK, static_cast<uint32_t>(TN), 1};
    if ((rc = make_tmap_bf16(&tx, x, 3, dx, sx, bxs))) return rc;
    static bool sk_attr_done = false;
    const int ssm = SkinnySmem::kBytes + 1024;
    if (!sk_attr_done) {
      MUX_CUDA(cudaFuncSetAttribute(outproj_skinny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ssm));
      sk_attr_done = true;
    }
    const int nk = (K + kGBK - 1) / kGBK;
    const int ntiles = (N + 127) / 128;
    // split = 1: deterministic (atomic split-K would break the mux == isolated bitwise identity)
    const int split = 1, per = nk;
    SkinnyParams sp{y, T, N, K, TN, per, y_dtype == MUX_DTYPE_F32, 0};
    outproj_skinny_kernel<<<dim3(ntiles, split), kGThreads, ssm, reinterpret_cast<cudaStream_t>(stream)>>>(tx, tw, sp);
    MUX_CUDA(cudaGetLastError());
    return MUX_OK;
  }
  GemmParams prm{y, T, N, K, y_dtype == MUX_DTYPE_F32};
  dim3 grid((N + kGBN - 1) / kGBN, (T + kGBM - 1) / kGBM);
  outproj_kernel<<<grid, kGThreads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(tx, tw, prm);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
