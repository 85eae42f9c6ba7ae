// Issue cost (cycles per warp-instruction per SMSP) of the softmax's instruction types on B200.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
  uint32_t r[8]; uint64_t q[8];
  for (int i = 0; i < 8; ++i) { r[i] = threadIdx.x * 7 + i * 13 + 0x3f800000u; q[i] = ((uint64_t)r[i] << 32) | r[i]; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+r"(r[i]));
      if (OP == 1) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(q[i]));
      if (OP == 2) asm volatile("add.rn.f32x2 %0, %0, %0;" : "+l"(q[i]));
      if (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[i]));
      if (OP == 4) asm volatile("cvt.rn.f16x2.f32 %0, %0, %0;" : "+r"(r[i]));
      if (OP == 5) asm volatile("prmt.b32 %0, %0, %0, 0x7632;" : "+r"(r[i]));
      if (OP == 6) asm volatile("lop3.b32 %0, %0, %0, 0x5555, 0xc0;" : "+r"(r[i]));
      if (OP == 7) asm volatile("max.f32 %0, %0, %0;" : "+r"(r[i]));
      if (OP == 8) asm volatile("mad.lo.u32 %0, %0, 8388608, %0;" : "+r"(r[i]));
      if (OP == 9) asm volatile("add.rn.f32 %0, %0, %0;" : "+r"(r[i]));
      if (OP == 10) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[i]));
      if (OP == 11) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[i]));
      if (OP == 12) { asm volatile("{.reg .f16 lo, hi; .reg .f32 a, b; mov.b32 {lo, hi}, %0; cvt.f32.f16 a, lo; cvt.f32.f16 b, hi; add.f32 a, a, b; mov.b32 %0, a;}" : "+r"(r[i])); }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0; for (int i = 0; i < 8; ++i) s ^= r[i] ^ (uint32_t)q[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name, uint32_t* out, long long* cyc) {
  for (int warps : {4, 8, 16}) {
    const int iters = 256;
    k<OP><<<148, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    k<OP><<<148, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double per_warp_instr = (double)c / (iters * 8);           // cycles between instructions of one warp
    printf("%-14s warps/SMSP=%d  %.2f cycles/instr per warp  -> SMSP issue %.2f cycles/instr\n", name, warps / 4,
           per_warp_instr, per_warp_instr / (warps / 4));
  }
}
int main() {
  uint32_t* out; long long* cyc; cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
  run<0>("FFMA", out, cyc); run<1>("FFMA2", out, cyc); run<2>("FADD2", out, cyc); run<3>("MUFU.EX2", out, cyc);
  run<4>("F2FP.F16", out, cyc); run<5>("PRMT", out, cyc); run<6>("LOP3", out, cyc); run<7>("FMNMX", out, cyc);
  run<8>("IMAD", out, cyc); run<9>("FADD", out, cyc); run<10>("EX2.F16x2", out, cyc); run<11>("EX2.BF16x2", out, cyc);
  run<12>("HCVT2+FADD", out, cyc);
  return 0;
}
