// Per-SM throughput of MUFU.EX2 and friends on B200 (developer microbenchmark).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void __launch_bounds__(512) k(float* out, int iters, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * 1e-6f - 1.0f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(r) : "f"(a[i])); a[i] = __uint_as_float(r) * 0.5f; }
      if (OP == 2) asm volatile("cvt.rmi.f32.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      // ex2 of a packed f16 pair: counts 2 results per op
      if (OP == 4) { uint32_t r = __float_as_uint(a[i]); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r)); a[i] = __uint_as_float(r); }
      if (OP == 5) { uint32_t r = __float_as_uint(a[i]); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r)); a[i] = __uint_as_float(r); }
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 4 * 512 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"ex2.approx", "cvt.rn.bf16x2 (+fmul)", "cvt.rmi (floor)", "ffma", "ex2.approx.f16x2 (x2)",
                         "ex2.approx.ftz.bf16x2 (x2)"};
  int sm_clk; cudaDeviceGetAttribute(&sm_clk, cudaDevAttrClockRate, 0);
  for (int op = 0; op < 6; ++op) {
    auto run = [&](int iters) {
      if (op == 0) k<0><<<148 * 4, 512>>>(out, iters, 1.f);
      if (op == 1) k<1><<<148 * 4, 512>>>(out, iters, 1.f);
      if (op == 2) k<2><<<148 * 4, 512>>>(out, iters, 1.f);
      if (op == 3) k<3><<<148 * 4, 512>>>(out, iters, 1.f);
      if (op == 4) k<4><<<148 * 4, 512>>>(out, iters, 1.f);
      if (op == 5) k<5><<<148 * 4, 512>>>(out, iters, 1.f);
    };
    run(10); cudaDeviceSynchronize();
    int iters = 4096;
    cudaEventRecord(a); run(iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = 148.0 * 4 * 512 * 8 * iters * (op >= 4 ? 2 : 1);
    printf("%-24s %.1f Gop/s  = %.2f per SM per ns  (%.1f per SM-clk at %.0f MHz max)\n", names[op], ops / ms / 1e6,
           ops / ms / 1e6 / 148, ops / ms / 1e6 / 148 / (sm_clk / 1e6), sm_clk / 1e3);
  }
  return 0;
}
