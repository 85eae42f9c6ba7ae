// tcgen05.mma issue/throughput microbenchmark for the prefill kernel's exact MMA shapes
// (developer tool).  One CTA per SM, one thread issues R repetitions of a pattern, commits
// once and waits; cycles / repetition vs the nominal rate max(M,128)*N/256 cycles per K=16 MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2504_14489_b200/csrc scripts/ubench_umma.cu -o scripts/ubench_umma -lcuda
#include <cstdio>
#include "../paper_2504_14489_b200/csrc/mux_internal.h"
using namespace mux;

template <int PAT>
__global__ void __launch_bounds__(128, 1) kern(long long* out, int reps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { dev::mbar_init(&bar, 1); dev::fence_mbar_init(); }
  if (warp == 0) dev::tmem_alloc(&slot, 512);
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(s)[i] = make_uint4(0, 0, 0, 0);
  dev::fence_proxy_async_smem();
  dev::tc_fence_before();
  __syncthreads();
  dev::tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint64_t da = dev::umma_desc_sw128(dev::smem_u32(s), 16, 1024);           // A K-major (Q)
    const uint64_t db = dev::umma_desc_sw128(dev::smem_u32(s + 32768), 16, 1024);   // B K-major (K)
    const uint64_t dv = dev::umma_desc_sw128(dev::smem_u32(s + 65536), 2048, 1024); // B MN-major (V)
    constexpr uint32_t i64 = dev::umma_idesc_bf16(128, 64, 0, 0);
    constexpr uint32_t i128 = dev::umma_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t ipv = dev::umma_idesc_f16(128, 128, 0, 1);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (PAT == 0 || PAT == 4)   // QK, N=64, SS, 8 k-steps (x2 heads for PAT 4)
        for (int h = 0; h < (PAT == 4 ? 2 : 1); ++h)
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            dev::umma_ss(tm + h * 64, da + ((kk * 32) >> 4), db + ((kk * 32) >> 4), i64, kk > 0);
      if (PAT == 1)               // QK, N=128, SS
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dev::umma_ss(tm, da + ((kk * 32) >> 4), db + ((kk * 32) >> 4), i128, kk > 0);
      if (PAT == 2 || PAT == 4)   // PV: A = P in TMEM, B = V MN-major smem, N=128, 4 k-steps (x2 heads for PAT 4)
        for (int h = 0; h < (PAT == 4 ? 2 : 1); ++h)
#pragma unroll
          for (int pp = 0; pp < 4; ++pp)
            dev::umma_ts(tm + 256 + h * 128, tm + 128 + h * 64 + pp * 8, dv + ((pp * 4096) >> 4), ipv, 1u);
      if (PAT == 3)               // PV with A from smem (SS), N=128, 4 k-steps
#pragma unroll
        for (int pp = 0; pp < 4; ++pp)
          dev::umma_ss(tm + 256, da + ((pp * 32) >> 4), dv + ((pp * 4096) >> 4), i128, 1u);
    }
    dev::umma_commit(&bar);
    dev::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  dev::tc_fence_before();
  __syncthreads();
  if (warp == 0) { dev::tc_fence_after(); dev::tmem_dealloc(tm, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  const char* names[] = {"QK SS M128 N64 x8", "QK SS M128 N128 x8", "PV TS M128 N128 x4", "PV SS M128 N128 x4",
                         "period: 2x(QK N64 x8) + 2x(PV TS x4)"};
  const double nominal[] = {8 * 32.0, 8 * 64.0, 4 * 64.0, 4 * 64.0, 2 * 8 * 32.0 + 2 * 4 * 64.0};
  const int smem = 96 * 1024 + 1024;
  auto go = [&](auto kfn, int p) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kfn<<<148, 128, smem>>>(d, 10);
    cudaDeviceSynchronize();
    const int reps = 2000;
    kfn<<<148, 128, smem>>>(d, reps);
    long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %8.1f cycles/rep  nominal %6.0f  (%.2fx)  %s\n", names[p], double(c) / reps, nominal[p],
           double(c) / reps / nominal[p], cudaGetErrorString(cudaGetLastError()));
  };
  go(kern<0>, 0); go(kern<1>, 1); go(kern<2>, 2); go(kern<3>, 3); go(kern<4>, 4);
  return 0;
}
