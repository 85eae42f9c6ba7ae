// Developer microbenchmark: does cvt.rn.f16x2.f32 (F2FP) share the MUFU/XU pipe with ex2?
// Times per-SM throughput of ex2 alone, the f16x2 pack alone, and the softmax mix (2 ex2 : 1 pack)
// plus integer / FMA alternatives for the pack.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void __launch_bounds__(512) k(uint32_t* out, int iters, float seed) {
  float a[8];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * 1e-6f - 1.0f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (OP == 0) {  // 2 ex2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
      }
      if (OP == 1) {  // 1 pack
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
        acc ^= r;
      }
      if (OP == 2) {  // 2 ex2 + 1 pack (the softmax mix)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
        acc ^= r;
      }
      if (OP == 3) {  // 2 ex2 + bf16 truncating pack (PRMT)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        uint32_t r;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(a[i])), "r"(__float_as_uint(a[i + 1])));
        acc ^= r;
      }
      if (OP == 4) {  // 2 ex2 + 1 fmax (FMNMX)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        float m;
        asm volatile("max.f32 %0, %1, %2;" : "=f"(m) : "f"(a[i]), "f"(a[i + 1]));
        acc ^= __float_as_uint(m);
      }
      if (OP == 5) {  // 1 fmax only
        float m;
        asm volatile("max.f32 %0, %1, %2;" : "=f"(m) : "f"(a[i]), "f"(a[i + 1]));
        acc ^= __float_as_uint(m);
        a[i] = m;
      }
      if (OP == 6) {  // 2 ex2 + pack via f16 integer trick on the ALU (normals only): (bits >> 13) - (112 << 10)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        uint32_t lo = (__float_as_uint(a[i]) >> 13) - (112u << 10);
        uint32_t hi = (__float_as_uint(a[i + 1]) >> 13) - (112u << 10);
        uint32_t r;
        asm volatile("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(lo), "r"(hi));
        acc ^= r;
      }
      if (OP == 7) {  // 2 ex2 + add.f32x2 (row sum) + pack: the full exp step minus the ffma2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i + 1]));
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
        acc ^= r;
        uint64_t s, x;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a[i]), "f"(a[i + 1]));
        asm volatile("add.rn.f32x2 %0, %1, %1;" : "=l"(s) : "l"(x));
        acc ^= static_cast<uint32_t>(s);
      }
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(s) ^ acc;
}
int main() {
  uint32_t* out;
  cudaMalloc(&out, 148 * 4 * 512 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"2 ex2", "1 cvt f16x2 pack", "2 ex2 + 1 pack", "2 ex2 + prmt bf16",
                         "2 ex2 + 1 fmax", "1 fmax", "2 ex2 + int f16 pack", "2 ex2 + pack + add2"};
  for (int op = 0; op < 8; ++op) {
    auto run = [&](int iters) {
      switch (op) {
        case 0: k<0><<<148 * 4, 512>>>(out, iters, 1.f); break;
        case 1: k<1><<<148 * 4, 512>>>(out, iters, 1.f); break;
        case 2: k<2><<<148 * 4, 512>>>(out, iters, 1.f); break;
        case 3: k<3><<<148 * 4, 512>>>(out, iters, 1.f); break;
        case 4: k<4><<<148 * 4, 512>>>(out, iters, 1.f); break;
        case 5: k<5><<<148 * 4, 512>>>(out, iters, 1.f); break;
        case 6: k<6><<<148 * 4, 512>>>(out, iters, 1.f); break;
        case 7: k<7><<<148 * 4, 512>>>(out, iters, 1.f); break;
      }
    };
    run(10);
    cudaDeviceSynchronize();
    int iters = 4096;
    cudaEventRecord(a);
    run(iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // per SM: pairs processed per ns (each iteration of the i-loop = one pair; 4 pairs per iteration)
    double pairs = 148.0 * 4 * 512 * 4 * iters;
    printf("%-24s %.2f pairs per SM per ns (%.3f ms)\n", names[op], pairs / ms / 1e6 / 148, ms);
  }
  return 0;
}
