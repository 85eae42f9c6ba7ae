// Per-SM read-streaming ceilings on B200 (developer microbenchmark, not part of libmux).
// One CTA per SM (large smem forces 1/SM), grid = nsm CTAs; each CTA streams its own
// contiguous slice.  Mechanisms: (a) TMA 4D boxes 64x16 (the decode kernel's pattern),
// (b) 1D cp.async.bulk of CHUNK bytes, (c) LDG.128 with many loads in flight.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}

template <int CHUNK, int STAGES, int NC>
__global__ void __launch_bounds__(288, 1) k_bulk(const uint8_t* src, size_t per_cta, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + STAGES * CHUNK);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) { for (int i = 0; i < STAGES; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const uint8_t* base = src + blockIdx.x * per_cta;
  const int n = per_cta / CHUNK;
  unsigned long long acc = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      int s = i % STAGES;
      if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
      expect(&full[s], CHUNK);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32(sm + s * CHUNK)), "l"(base + (size_t)i * CHUNK), "r"(CHUNK), "r"(su32(&full[s])) : "memory");
    }
  } else if ((threadIdx.x & 31) == 0 && threadIdx.x / 32 <= NC) {
    const int w = threadIdx.x / 32 - 1;
    for (int i = w; i < n; i += NC) {
      int s = i % STAGES;
      wait(&full[s], (i / STAGES) & 1);
      acc += sm[s * CHUNK + (i & 127)];
      arrive(&empty[s]);
    }
    sink[blockIdx.x * 16 + w] = acc;
  }
}

template <int STAGES, int NC, int BOXES>
__global__ void __launch_bounds__(288, 1) k_tma(const __grid_constant__ CUtensorMap map, int pages_per_cta, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int STAGE = 8192;  // K+V page, d=128: 4 boxes of 64x16 bf16
  uint64_t* full = (uint64_t*)(sm + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) { for (int i = 0; i < STAGES; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  unsigned long long acc = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < pages_per_cta; ++i) {
      int s = i % STAGES;
      if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
      expect(&full[s], STAGE);
      int page = blockIdx.x * pages_per_cta + i;
      if (BOXES == 4) {
      for (int bx = 0; bx < 4; ++bx) {
        int c0 = (bx & 1) * 64, hd = bx >> 1;  // two "heads" stand in for K and V
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     :: "r"(su32(sm + s * STAGE + bx * 2048)), "l"((uint64_t)&map), "r"(c0), "r"(0), "r"(hd), "r"(page), "r"(su32(&full[s])) : "memory");
      }
      } else {  // 5D map {64, 16, 2, 2, pages}: one box = both 64-dim halves of one head
        for (int hd = 0; hd < 2; ++hd)
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     :: "r"(su32(sm + s * STAGE + hd * 4096)), "l"((uint64_t)&map), "r"(0), "r"(0), "r"(0), "r"(hd), "r"(page), "r"(su32(&full[s])) : "memory");
      }
    }
  } else if ((threadIdx.x & 31) == 0 && threadIdx.x / 32 <= NC) {
    const int w = threadIdx.x / 32 - 1;
    for (int i = w; i < pages_per_cta; i += NC) {
      int s = i % STAGES;
      wait(&full[s], (i / STAGES) & 1);
      acc += sm[s * STAGE + (i & 127)];
      arrive(&empty[s]);
    }
    sink[blockIdx.x * 16 + w] = acc;
  }
}

// decode's pattern: one 5-D box = one page of 8 kv heads (8 x 4 KiB = 32 KiB), SWIZZLE_128B
template <int STAGES, int NC>
__global__ void __launch_bounds__(288, 1) k_tma32(const __grid_constant__ CUtensorMap map, int pages_per_cta,
                                                  unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);   // SWIZZLE_128B needs 1 KiB alignment
  constexpr int STAGE = 32768;
  uint64_t* full = (uint64_t*)(sm + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) { for (int i = 0; i < STAGES; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], 1); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  unsigned long long acc = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < pages_per_cta; ++i) {
      int s = i % STAGES;
      if (i >= STAGES) wait(&empty[s], ((i / STAGES) - 1) & 1);
      expect(&full[s], STAGE);
      int page = blockIdx.x * pages_per_cta + i;
      asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                   :: "r"(su32(sm + s * STAGE)), "l"((uint64_t)&map), "r"(0), "r"(0), "r"(0), "r"(0), "r"(page), "r"(su32(&full[s])) : "memory");
    }
  } else if ((threadIdx.x & 31) == 0 && threadIdx.x / 32 <= NC) {
    const int w = threadIdx.x / 32 - 1;
    for (int i = w; i < pages_per_cta; i += NC) {
      int s = i % STAGES;
      wait(&full[s], (i / STAGES) & 1);
      acc += sm[s * STAGE + (i & 127)];
      arrive(&empty[s]);
    }
    sink[blockIdx.x * 16 + w] = acc;
  }
}

template <int UNROLL>
__global__ void __launch_bounds__(512, 1) k_ldg(const uint4* src, size_t per_cta16, unsigned long long* sink) {
  const uint4* base = src + blockIdx.x * per_cta16;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i + (UNROLL - 1) * 512 < per_cta16; i += UNROLL * 512) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(base + i + u * 512));
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678) sink[blockIdx.x] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  int vid = -1;
  const size_t bytes = (size_t)4 << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  unsigned long long* sink; CK(cudaMalloc(&sink, 4096 * 16 * 8));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int nsm_list[] = {8, 16, 32, 64, 148};
  EncodeFn enc; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  const int total_pages = bytes / 8192;
  CUtensorMap map;
  cuuint64_t dims[4] = {128, 16, 2, (cuuint64_t)total_pages};
  cuuint64_t strides[3] = {256, 4096, 8192};
  cuuint32_t box[4] = {64, 16, 1, 1}, es[4] = {1, 1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode failed\n"); return 1; }
  CUtensorMap map5;
  cuuint64_t dims5[5] = {64, 16, 2, 2, (cuuint64_t)total_pages};
  cuuint64_t strides5[4] = {256, 128, 4096, 8192};
  cuuint32_t box5[5] = {64, 16, 2, 1, 1}, es5[5] = {1, 1, 1, 1, 1};
  if (enc(&map5, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, buf, dims5, strides5, box5, es5, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode5 failed\n"); return 1; }
  CUtensorMap mapg;
  const int total_pages32 = bytes / 32768;
  cuuint64_t dimsg[5] = {64, 16, 2, 8, (cuuint64_t)total_pages32};
  cuuint64_t stridesg[4] = {256, 128, 4096, 32768};
  cuuint32_t boxg[5] = {64, 16, 2, 8, 1}, esg[5] = {1, 1, 1, 1, 1};
  if (enc(&mapg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, buf, dimsg, stridesg, boxg, esg, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encodeg failed\n"); return 1; }
  auto run = [&](const char* name, auto launch, int nsm, size_t moved) {
    launch(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); for (int r = 0; r < 3; ++r) launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 3;
    printf("%-22s nsm=%3d  %7.1f GB/s total  %6.1f GB/s/SM\n", name, nsm, moved / ms / 1e6, moved / ms / 1e6 / nsm);
  };
  for (int nsm : {16, 32, 148}) {
    vid = -1;
    size_t per = (bytes / 148) & ~size_t(65535);
    int ppc = per / 8192;
#define TMA(NC, BX) if (++vid == only || only < 0) { auto k = k_tma<24, NC, BX>; int smem = 24 * 8192 + 1024; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      run("tma " #BX "box/8K nc=" #NC, [&] { k<<<nsm, 288, smem>>>(BX == 4 ? map : map5, ppc, sink); }, nsm, (size_t)nsm * ppc * 8192); }
    TMA(1, 4) TMA(4, 4) TMA(8, 4) TMA(1, 2) TMA(4, 2) TMA(8, 2)
#define BULK(CH, ST, NC) if (++vid == only || only < 0) { auto k = k_bulk<CH, ST, NC>; int smem = ST * CH + 1024; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      run("bulk " #CH " st" #ST " nc=" #NC, [&] { k<<<nsm, 288, smem>>>(buf, per, sink); }, nsm, (size_t)nsm * per); }
    BULK(4096, 48, 1) BULK(4096, 48, 8) BULK(8192, 24, 8) BULK(16384, 12, 8) BULK(32768, 6, 6) BULK(65536, 3, 3)
#define TMA32(ST) if (++vid == only || only < 0) { auto k = k_tma32<ST, 6>; int smem = ST * 32768 + 2048; cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
      int pp32 = per / 32768; run("tma5d 32K-box st" #ST, [&] { k<<<nsm, 288, smem>>>(mapg, pp32, sink); }, nsm, (size_t)nsm * pp32 * 32768); }
    TMA32(6) TMA32(3)
    if (++vid == only || only < 0) { auto k = k_ldg<8>;
      run("ldg.128 x8 512thr", [&] { k<<<nsm, 512>>>((const uint4*)buf, per / 16, sink); }, nsm, (size_t)nsm * per); }
  }
  return 0;
}
