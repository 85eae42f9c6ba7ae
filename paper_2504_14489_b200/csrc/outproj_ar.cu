// f4 (fused communication): out-projection GEMM + all-reduce of the partial
// sums in ONE kernel over peer memory.
//
// PAPER: Llama-70B is served with tensor parallelism of degree 8 over NVLink;
// under KV-head sharding each GPU's attention output O_g times its row shard of W_o is a partial
// sum of the layer output, and the G partials are summed (R23; Table 2's n d^2 term of the
// projection).  a7 computes that with mux_outproj and then an NCCL all-reduce on the
// side's stream; here the collective leaves the GPU tile by tile from the GEMM's epilogue.
//
// B200 design: the CTA-pair tcgen05 GEMM of outproj.cu (256 x 256 output tiles, M = 256 MMAs across
// a cluster of two, packed W by bulk tensor copies, double-buffered TMEM accumulators).  Tile t is
// OWNED by rank t mod G.
//   phase 1 (epilogue warps, per tile): the fp32 accumulator rows -> bf16 (the NCCL wire type of
//     R23) -> stored straight into the owner's staging slot [t / G][my rank] (st.global on the
//     owner's memory, mapped by CUDA IPC / VMM; local when the owner is this rank), then one
//     fence.acq_rel.sys + red.add.sys on the owner's per-slot counter.
//   phase 2 (epilogue warps, the tiles this rank owns, split in 128-row halves over its CTAs):
//     wait (ld.acquire.sys) until the slot counter reached 2 G per launch (two CTAs per rank), sum
//     the G partials in rank order 0..G-1 in fp32 (deterministic: the same bits on every rank and
//     every run), round to bf16 and store the half tile into EVERY rank's Y (all-gather by peer
//     stores), then count the half tile on every rank's done counter.
//   phase 3: the first CTA of each rank waits until its done counter shows all 2 x tiles half
//     tiles of the launch: the kernel ends with this rank's Y complete.
// Counters are never reset: launch number `epoch` (1, 2, ...) waits for epoch x count; epoch 0 in
// the call = take it from the rank's own launch counter in the workspace (CUDA-graph friendly).
// Deadlock freedom: phase 1 waits on nothing remote, phase 2 only on phase 1 of other ranks,
// phase 3 only on phase 2; every rank's grid fits its SMs (one CTA per SM, all co-resident).
// With fewer GPUs than ranks the same kernel runs ALL ranks' CTAs in one launch on one device
// (mux_outproj_allreduce_emulated), which is how the G-rank protocol is tested here.
#include <algorithm>

#include "pool.h"

namespace mux {
namespace {

constexpr int kArBM = 128, kArBN = 256, kArBK = 64;
constexpr int kArThreads = 192;                 // warps 0-3 epilogue, 4 producer, 5 MMA issuer
constexpr int kArStages = 6;
constexpr int kArPack = 128 * kArBK * 2;         // one packed 128-column W tile per k-block: 16 KiB
constexpr int kArTileElems = 2 * kArBM * kArBN;  // 256 x 256 output tile

struct ArSmem {
  static constexpr int kA = kArBM * kArBK * 2;  // 16 KiB: my 128 rows x 64 k
  static constexpr int kB = kArPack;            // 16 KiB: my 128 columns x 64 k
  static constexpr int kStage = kA + kB;
  static constexpr int kBar = kArStages * kStage;
  static constexpr int kTmemSlot = kBar + (2 * kArStages + 4) * 8;
  static constexpr int kBytes = kTmemSlot + 16;
};

struct ArMaps {
  CUtensorMap x[MUX_AR_MAX_WORLD];
  CUtensorMap w[MUX_AR_MAX_WORLD];
};

struct ArParams {
  int T, N, K, m_tiles, n_tiles, tiles, nslots;
  int G, rank0, pairs;  // ranks rank0 .. rank0 + (grid / 2 / pairs) - 1 run in this launch
  uint32_t epoch;
  uint16_t* stage[MUX_AR_MAX_WORLD];
  uint16_t* y[MUX_AR_MAX_WORLD];
};

// staging of one rank: [nslots][G][256][256] bf16, then uint32 counters [nslots], done, launches
__host__ __device__ inline size_t ar_stage_elems(int nslots, int G) {
  return static_cast<size_t>(nslots) * G * kArTileElems;
}
__device__ __forceinline__ uint32_t* ar_flags(const ArParams& p, int r) {
  return reinterpret_cast<uint32_t*>(p.stage[r] + ar_stage_elems(p.nslots, p.G));
}
__device__ __forceinline__ void red_add_sys(uint32_t* a, uint32_t v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// A rank that never arrives (a peer that crashed, or ranks that called with different arguments)
// must not hang the GPU: after kArWaitLimitNs the kernel traps (the launch fails with an error).
#ifndef MUX_AR_WAIT_LIMIT_NS
#define MUX_AR_WAIT_LIMIT_NS 20000000000ull
#endif
__device__ __forceinline__ void wait_count(const uint32_t* a, uint32_t target) {
  if (static_cast<int32_t>(ld_acquire_sys(a) - target) >= 0) return;
  const uint64_t t0 = dev::globaltimer();
  while (static_cast<int32_t>(ld_acquire_sys(a) - target) < 0) {
    __nanosleep(64);
    if (dev::globaltimer() - t0 > MUX_AR_WAIT_LIMIT_NS) __trap();
  }
}

__global__ void __launch_bounds__(kArThreads, 1)
    outproj_ar_kernel(const __grid_constant__ ArMaps maps, const ArParams p) {
  using L = ArSmem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBar);
  uint64_t* empty = full + kArStages;
  uint64_t* acc_full = empty + kArStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kTmemSlot);
  const int warp = dev::warp_idx_uniform(), lane = threadIdx.x & 31;
  const uint32_t crank = dev::cluster_ctarank();
  const bool leader = crank == 0;
  const int gpair = blockIdx.x >> 1;
  const int rl = gpair / p.pairs, pair = gpair % p.pairs;   // rank within the launch, pair within the rank
  const int rank = p.rank0 + rl;
  const int nk = (p.K + kArBK - 1) / kArBK;
  const int ntiles128 = (p.N + 127) / 128;
  const CUtensorMap* tmx = &maps.x[rl];
  const CUtensorMap* tmw = &maps.w[rl];
  // epoch 0 = automatic: this rank's launch counter (the word after `done`, bumped by CTA 0 at the
  // end of every launch; the next launch on the stream reads it after this kernel completed)
  uint32_t* my_words = ar_flags(p, rank);
  const uint32_t epoch = p.epoch ? p.epoch : *reinterpret_cast<volatile uint32_t*>(my_words + p.nslots + 1) + 1;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kArStages + 2; ++i) dev::mbar_init(&full[i], 1);
    dev::mbar_init(&acc_empty[0], 8);  // 4 epilogue warps x 2 CTAs (the leader's copy is used)
    dev::mbar_init(&acc_empty[1], 8);
    dev::fence_mbar_init();
  }
  if (warp == 5) dev::tmem_alloc_pair(tmem_slot, 512);
  dev::tc_fence_before();
  __syncthreads();
  dev::cluster_sync();
  dev::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t full_leader = dev::mapa(dev::smem_u32(full), 0);
  const uint32_t acc_empty_leader = dev::mapa(dev::smem_u32(acc_empty), 0);

  if (warp == 4) {
    // ---------------------------------------------------------------- producer (as outproj2)
    if (lane == 0) {
      dev::tma_prefetch(tmx);
      dev::tma_prefetch(tmw);
      int it = 0;
      for (int t = pair; t < p.tiles; t += p.pairs) {
        const int m0 = (t / p.n_tiles) * 2 * kArBM + static_cast<int>(crank) * kArBM;
        const int wt = (t % p.n_tiles) * 2 + static_cast<int>(crank);
        const int wtile = wt < ntiles128 ? wt : ntiles128 - 1;   // N tail: any valid tile (never stored)
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kArStages;
          if (it >= kArStages) dev::mbar_wait_sleep(&empty[s], ((it / kArStages) - 1) & 1);
          if (leader) dev::mbar_expect_tx(&full[s], 2 * L::kStage);
          uint8_t* a = smem + s * L::kStage;
          const uint32_t fb = full_leader + s * 8;
          dev::tma_load_3d_pair(a, tmx, fb, kb * kArBK, m0, 0);
          dev::tma_load_3d_pair(a + L::kA, tmw, fb, 0, 0, wtile * nk + kb);
        }
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = dev::umma_idesc_bf16(2 * kArBM, kArBN, 0, 1);
      const uint64_t d0 = dev::umma_desc_sw128(dev::smem_u32(smem), 16, 1024);
      const uint64_t e0 = dev::umma_desc_sw128(dev::smem_u32(smem + L::kA), kArBK * 128, 1024);
      int it = 0, i = 0;
      for (int t = pair; t < p.tiles; t += p.pairs, ++i) {
        const int b = i & 1;
        if (i >= 2) dev::mbar_wait_sleep(&acc_empty[b], ((i >> 1) - 1) & 1);
        dev::tc_fence_after();
        const uint32_t acc = tmem + b * kArBN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kArStages;
          dev::mbar_wait_sleep(&full[s], (it / kArStages) & 1);
          dev::tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kArBK / 16; ++kk)
            dev::umma_ss_pair(acc, d0 + ((s * L::kStage + kk * 32) >> 4), e0 + ((s * L::kStage + kk * 16 * 128) >> 4),
                              idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          dev::umma_commit_pair(&empty[s]);
        }
        dev::umma_commit_pair(&acc_full[b]);
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue warps 0-3
    const int G = p.G;
    // the half tiles (units) this rank owns, spread over its CTAs: unit u = (slot u / 2, half u % 2)
    const int cid = pair * 2 + static_cast<int>(crank), ncta = 2 * p.pairs;
    const int nown = rank < p.tiles ? (p.tiles - rank + G - 1) / G : 0;
    uint32_t* my_flags = my_words;
    const uint32_t need = epoch * static_cast<uint32_t>(2 * G);
    int next_u = cid;
    // sum the G partials of one unit in rank order (fp32), round to bf16, store into every rank's Y,
    // count it on every rank.  Each warp takes 32 rows in batches of 8 (8 independent 16-byte loads
    // per rank in flight per lane); lane = 8 columns.
    auto reduce_unit = [&](int u) {
      const int s = u >> 1, half = u & 1;
      const int t = s * G + rank;
      const int m0 = (t / p.n_tiles) * 2 * kArBM, n0 = (t % p.n_tiles) * kArBN;
      const uint16_t* src = p.stage[rank] + static_cast<size_t>(s) * G * kArTileElems;
      const int col = n0 + 8 * lane;
#pragma unroll 1
      for (int rb = 0; rb < 32; rb += 8) {
        float acc[8][8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[k][e] = 0.f;
        for (int r = 0; r < G; ++r) {             // rank order: the same sum on every rank
          uint4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            v[k] = __ldcg(reinterpret_cast<const uint4*>(src + static_cast<size_t>(r) * kArTileElems +
                                                           static_cast<size_t>(half * kArBM + warp * 32 + rb + k) * kArBN +
                                                           8 * lane));
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            acc[k][0] += dev::bf16lo(v[k].x); acc[k][1] += dev::bf16hi(v[k].x);
            acc[k][2] += dev::bf16lo(v[k].y); acc[k][3] += dev::bf16hi(v[k].y);
            acc[k][4] += dev::bf16lo(v[k].z); acc[k][5] += dev::bf16hi(v[k].z);
            acc[k][6] += dev::bf16lo(v[k].w); acc[k][7] += dev::bf16hi(v[k].w);
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int row = m0 + half * kArBM + warp * 32 + rb + k;
          if (row < p.T && col < p.N) {
            const uint4 o = make_uint4(dev::pack_bf16(acc[k][0], acc[k][1]), dev::pack_bf16(acc[k][2], acc[k][3]),
                                       dev::pack_bf16(acc[k][4], acc[k][5]), dev::pack_bf16(acc[k][6], acc[k][7]));
            for (int r = 0; r < G; ++r) *reinterpret_cast<uint4*>(p.y[r] + static_cast<size_t>(row) * p.N + col) = o;
          }
        }
      }
      dev::named_bar_sync(1, 128);
      if (threadIdx.x == 0) {
        fence_sys();
        for (int r = 0; r < G; ++r) red_add_sys(ar_flags(p, r) + p.nslots, 1u);
      }
    };
    // phase 1: my 128 rows of each tile -> bf16 -> the owner's staging slot, then count it there;
    // between tiles (while the MMA fills the other accumulator) reduce owned units that are ready
    int i = 0;
    for (int t = pair; t < p.tiles; t += p.pairs, ++i) {
      const int b = i & 1;
      const int owner = t % G, slot = t / G;
      dev::mbar_wait_sleep(&acc_full[b], (i >> 1) & 1);
      dev::tc_fence_after();
      const int rloc = static_cast<int>(crank) * kArBM + warp * 32 + lane;   // row within the 256-row tile
      uint16_t* dst = p.stage[owner] + (static_cast<size_t>(slot) * G + rank) * kArTileElems +
                      static_cast<size_t>(rloc) * kArBN;
      const uint32_t taddr = tmem + b * kArBN + (static_cast<uint32_t>(warp * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < kArBN / 32; ++c) {
        uint32_t v[32];
        dev::tmem_ld32(taddr + c * 32, v);
        dev::tmem_wait_ld();
        if (c == kArBN / 32 - 1) {
          dev::tc_fence_before();
          __syncwarp();
          if (lane == 0) dev::mbar_arrive_cluster(acc_empty_leader + b * 8);
        }
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          d4[k] = make_uint4(dev::pack_bf16(__uint_as_float(v[8 * k]), __uint_as_float(v[8 * k + 1])),
                             dev::pack_bf16(__uint_as_float(v[8 * k + 2]), __uint_as_float(v[8 * k + 3])),
                             dev::pack_bf16(__uint_as_float(v[8 * k + 4]), __uint_as_float(v[8 * k + 5])),
                             dev::pack_bf16(__uint_as_float(v[8 * k + 6]), __uint_as_float(v[8 * k + 7])));
      }
      dev::named_bar_sync(1, 128);                 // all 128 rows of this CTA's half stored
      if (threadIdx.x == 0) {
        fence_sys();
        red_add_sys(ar_flags(p, owner) + slot, 1u);
      }
      // overlap: at most two ready units per tile (the next accumulator must not wait long)
      for (int k = 0; k < 2 && next_u < 2 * nown; ++k) {
        const bool ready = dev::bar_red_or(1, 128, threadIdx.x == 0 &&
                                                       static_cast<int32_t>(ld_acquire_sys(my_flags + (next_u >> 1)) - need) >= 0);
        if (!ready) break;
        reduce_unit(next_u);
        next_u += ncta;
      }
    }
    // phase 2 (the remaining half tiles this rank owns; blocking waits)
    while (next_u < 2 * nown) {
      const int s = next_u >> 1;
      if (threadIdx.x == 0) wait_count(my_flags + s, need);
      dev::named_bar_sync(1, 128);
      reduce_unit(next_u);
      next_u += ncta;
    }
    // phase 3: this rank's Y is complete once every half tile of the launch was counted here
    // (every CTA of this rank read the launch counter before its phase-1 arrivals, which the
    // waits below imply, so CTA 0 may bump it afterwards)
    if (cid == 0 && threadIdx.x == 0) {
      wait_count(my_flags + p.nslots, epoch * static_cast<uint32_t>(2 * p.tiles));
      if (!p.epoch) my_flags[p.nslots + 1] = epoch;
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

int ar_check(int32_t T, int32_t K, int32_t N, const mux_ar_peers* peers) {
  if (!peers) return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce: peers NULL");
  if (peers->world < 1 || peers->world > MUX_AR_MAX_WORLD)
    return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce: world must be 1..8");
  if (T < 1 || K < 1 || N < 1) return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce: T, K, N must be >= 1");
  if ((K % 8) || (N % 8)) return fail(MUX_ERR_UNSUPPORTED, "mux_outproj_allreduce: K and N must be multiples of 8");
  for (int r = 0; r < peers->world; ++r) {
    if (!peers->stage[r] || !peers->y[r]) return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce: NULL peer buffer");
    if ((reinterpret_cast<uintptr_t>(peers->stage[r]) | reinterpret_cast<uintptr_t>(peers->y[r])) & 15)
      return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce: peer buffers must be 16-byte aligned");
  }
  return MUX_OK;
}

int ar_maps(ArMaps* m, int idx, const void* x, const void* w, int32_t T, int32_t K, int32_t N) {
  if (!x || !w) return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce: x / w_packed NULL");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce: x / w_packed must be 16-byte aligned");
  uint64_t dx[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(T), 1};
  uint64_t sx[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K) * T * 2};
  uint32_t bx[3] = {kArBK, kArBM, 1};
  int rc = make_tmap_bf16(&m->x[idx], x, 3, dx, sx, bx);
  if (rc) return rc;
  const int KB = (K + kArBK - 1) / kArBK, NT = (N + 127) / 128;
  uint64_t dw[3] = {64, 128, static_cast<uint64_t>(KB) * NT};
  uint64_t sw[2] = {128, 16384};
  uint32_t bw[3] = {64, 128, 1};
  return make_tmap_bf16(&m->w[idx], w, 3, dw, sw, bw, false);
}

int ar_launch(const ArMaps& maps, ArParams prm, int nranks, int sms, bool cooperative, cudaStream_t st) {
  static bool attr = false;
  const int smem = ArSmem::kBytes + 1024;
  if (!attr) {
    MUX_CUDA(cudaFuncSetAttribute(outproj_ar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  prm.pairs = std::max(1, std::min(prm.tiles, sms / (2 * nranks)));
  if (sms < 2 * nranks) return fail(MUX_ERR_NO_CONFIG, "mux_outproj_allreduce: fewer than 2 SMs per rank");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * prm.pairs * nranks);
  cfg.blockDim = dim3(kArThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = cooperative ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, outproj_ar_kernel, maps, prm);
  if (e != cudaSuccess && cooperative) {
    // cooperative + cluster launch refused: the grid is still at most one CTA per SM
    (void)cudaGetLastError();
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, outproj_ar_kernel, maps, prm);
  }
  MUX_CUDA(e);
  return MUX_OK;
}

ArParams ar_params(int32_t T, int32_t K, int32_t N, const mux_ar_peers* peers) {
  ArParams prm{};
  prm.T = T;
  prm.N = N;
  prm.K = K;
  prm.m_tiles = (T + 2 * kArBM - 1) / (2 * kArBM);
  prm.n_tiles = (N + kArBN - 1) / kArBN;
  prm.tiles = prm.m_tiles * prm.n_tiles;
  prm.G = peers->world;
  prm.nslots = (prm.tiles + prm.G - 1) / prm.G;
  prm.epoch = peers->epoch;
  for (int r = 0; r < peers->world; ++r) {
    prm.stage[r] = static_cast<uint16_t*>(peers->stage[r]);
    prm.y[r] = static_cast<uint16_t*>(peers->y[r]);
  }
  return prm;
}

}  // namespace
}  // namespace mux

using namespace mux;

extern "C" size_t mux_outproj_ar_ws_bytes(int32_t T, int32_t N, int32_t world) {
  if (T < 1 || N < 1 || world < 1 || world > MUX_AR_MAX_WORLD) return 0;
  const int tiles = ((T + 2 * kArBM - 1) / (2 * kArBM)) * ((N + kArBN - 1) / kArBN);
  const int nslots = (tiles + world - 1) / world;
  return ar_stage_elems(nslots, world) * 2 + (static_cast<size_t>(nslots) + 2) * 4;
}

extern "C" int mux_outproj_allreduce(const void* x, const void* w_packed, int32_t T, int32_t K, int32_t N,
                                     const mux_ar_peers* peers, int32_t num_sms, mux_stream_t stream) {
  int rc = ar_check(T, K, N, peers);
  if (rc) return rc;
  if (peers->rank < 0 || peers->rank >= peers->world)
    return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce: rank out of range");
  ArMaps maps{};
  if ((rc = ar_maps(&maps, 0, x, w_packed, T, K, N))) return rc;
  ArParams prm = ar_params(T, K, N, peers);
  prm.rank0 = peers->rank;
  const int sms = num_sms > 0 ? num_sms : device_sm_count();
  return ar_launch(maps, prm, 1, sms, false, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int mux_outproj_allreduce_emulated(const void* const* x, const void* const* w_packed, int32_t T, int32_t K,
                                              int32_t N, const mux_ar_peers* peers, mux_stream_t stream) {
  int rc = ar_check(T, K, N, peers);
  if (rc) return rc;
  if (!x || !w_packed) return fail(MUX_ERR_INVALID_ARG, "mux_outproj_allreduce_emulated: x / w_packed NULL");
  ArMaps maps{};
  for (int r = 0; r < peers->world; ++r)
    if ((rc = ar_maps(&maps, r, x[r], w_packed[r], T, K, N))) return rc;
  ArParams prm = ar_params(T, K, N, peers);
  prm.rank0 = 0;
  return ar_launch(maps, prm, peers->world, device_sm_count(), true, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int mux_ipc_alloc(size_t bytes, void** ptr, void* handle) {
  if (!ptr || !handle || bytes == 0) return fail(MUX_ERR_INVALID_ARG, "mux_ipc_alloc: bad argument");
  *ptr = nullptr;
  void* p = nullptr;
  MUX_CUDA(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(e, "mux_ipc_alloc");
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == MUX_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return MUX_OK;
}

extern "C" int mux_ipc_open(const void* handle, void** ptr) {
  if (!ptr || !handle) return fail(MUX_ERR_INVALID_ARG, "mux_ipc_open: bad argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  *ptr = nullptr;
  MUX_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return MUX_OK;
}

extern "C" int mux_ipc_close(void* ptr) {
  if (!ptr) return MUX_OK;
  MUX_CUDA(cudaIpcCloseMemHandle(ptr));
  return MUX_OK;
}

extern "C" int mux_ipc_free(void* ptr) {
  if (!ptr) return MUX_OK;
  MUX_CUDA(cudaFree(ptr));
  return MUX_OK;
}
