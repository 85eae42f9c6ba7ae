// Cycles per 128-element row of the prefill softmax exp/pack math (no TMEM), 1..2 warps/SMSP.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t f2pack(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void f2unpack(uint64_t r, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) { uint32_t r; asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
template <int MODE>
__global__ void k(const float* in, uint32_t* out, long long* cyc, int rows, float sl2, float m) {
  float s[128];
  for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x * 131 + i) & 4095];
  uint32_t sink = 0;
  const uint64_t S2 = f2pack(sl2, sl2), NM = f2pack(-m, -m), M1 = f2pack(-1.f, -1.f);
  long long t0 = clock64();
  for (int r = 0; r < rows; ++r) {
    uint64_t acc = f2pack(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      float a, b;
      f2unpack(ffma2(f2pack(s[2 * i], s[2 * i + 1]), S2, NM), a, b);
      float e0, e1;
      if (MODE == 1) { e0 = a; e1 = b; }   // no MUFU
      else { e0 = ex2(a); e1 = ex2(b); }
      const uint64_t e = f2pack(e0, e1);
      acc = fadd2(acc, e);
      if (MODE == 3) sink ^= pack_f16(e0, e1);        // the prefill v6 mix: FFMA2, 2 ex2, FADD2, F2FP.F16
      if (MODE == 4) sink ^= pack_bf16(e0, e1);       // same with a bf16 pack
      if (MODE < 2) {                      // MODE 2: exp + sum only
        const uint32_t u0 = __float_as_uint(e0) & 0xFFFF0000u, u1 = __float_as_uint(e1) & 0xFFFF0000u;
        uint32_t hi = __byte_perm(__float_as_uint(e0), __float_as_uint(e1), 0x7632);
        float r0, r1;
        f2unpack(ffma2(f2pack(__uint_as_float(u0), __uint_as_float(u1)), M1, e), r0, r1);
        sink ^= hi ^ pack_bf16(r0, r1);
      }
    }
    float x, y; f2unpack(acc, x, y);
    sink ^= __float_as_uint(x + y);
    s[r & 127] += 1e-7f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* in; uint32_t* out; long long* cyc;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* mn[] = {"full (exp+sum+hi/lo)", "no MUFU", "exp+sum only", "v6 mix (f16 pack)", "v6 mix (bf16 pack)"};
  for (int mode = 0; mode < 5; ++mode)
    for (int warps : {4, 8, 16}) {
      auto run = [&] {
        if (mode == 0) k<0><<<148, warps * 32>>>(in, out, cyc, 200, 0.1f, 1.f);
        if (mode == 1) k<1><<<148, warps * 32>>>(in, out, cyc, 200, 0.1f, 1.f);
        if (mode == 2) k<2><<<148, warps * 32>>>(in, out, cyc, 200, 0.1f, 1.f);
        if (mode == 3) k<3><<<148, warps * 32>>>(in, out, cyc, 200, 0.1f, 1.f);
        if (mode == 4) k<4><<<148, warps * 32>>>(in, out, cyc, 200, 0.1f, 1.f);
      };
      run(); cudaDeviceSynchronize(); run(); cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-22s warps/SM=%d: %.0f cycles per row per warp (%d warps/SMSP)\n", mn[mode], warps, c / 200.0, warps / 4);
    }
  return 0;
}
