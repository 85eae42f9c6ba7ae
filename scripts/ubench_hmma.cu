// Legacy tensor-pipe (mma.sync m16n8k16 bf16) rate and latency on B200, plus SHFL / MOVM / LDSM
// issue costs: what bounds the decode consumer's per-page instruction chain (developer tool).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
template <int OP, int CHAINS>
__global__ void k(float* out, long long* cyc, int iters) {
  __shared__ __align__(16) uint16_t sm[16 * 1024];
  for (int i = threadIdx.x; i < 16 * 1024; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float c[CHAINS][4];
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  uint32_t x[CHAINS];
  for (int j = 0; j < CHAINS; ++j) { c[j][0] = c[j][1] = c[j][2] = c[j][3] = 0.f; x[j] = threadIdx.x + j; }
  const uint32_t saddr = (uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x & 31) * 16;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) {
      if (OP == 0)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      if (OP == 1) asm volatile("shfl.sync.bfly.b32 %0, %0, 4, 0x1f, 0xffffffff;" : "+r"(x[j]));
      if (OP == 2) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(x[j]));
      if (OP == 4) {   // LDS.128, 16 consecutive bytes per lane, conflict-free
        uint32_t r0, r1, r2, r3;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(saddr + ((((it << 3) + j) << 9) & 0x7FFF)));
        x[j] += r0 ^ r1 ^ r2 ^ r3;
      }
      if (OP == 5) {   // LDSM.x4.trans
        uint32_t r0, r1, r2, r3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(saddr + ((((it << 3) + j) << 9) & 0x7FFF)));
        x[j] += r0 ^ r1 ^ r2 ^ r3;
      }
      if (OP == 6) {   // LDS.32
        uint32_t r0;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r0) : "r"((uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x & 31) * 4 + ((((it << 3) + j) << 7) & 0x7FFF)));
        x[j] += r0;
      }
      if (OP == 7) {   // LDSM.x2
        uint32_t r0, r1;
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                     : "=r"(r0), "=r"(r1) : "r"(saddr + ((((it << 3) + j) << 9) & 0x7FFF)));
        x[j] += r0 ^ r1;
      }
      if (OP == 3) {
        uint32_t r0, r1, r2, r3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(saddr + ((((it << 3) + j) << 9) & 0x7FFF)));
        x[j] += r0 ^ r1 ^ r2 ^ r3;
      }
    }
  }
  float s = 0; for (int j = 0; j < CHAINS; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3] + x[j];
  asm volatile("" : "+f"(s));
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP, int CHAINS> void run(const char* name, float* out, long long* cyc) {
  for (int warps : {4, 8, 16}) {
    const int iters = 256;
    k<OP, CHAINS><<<148, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    k<OP, CHAINS><<<148, warps * 32>>>(out, cyc, iters); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double per = (double)c / (iters * CHAINS);
    printf("%-8s chains=%d warps/SMSP=%d  %.2f cycles/instr per warp -> SMSP %.2f cycles/instr\n", name, CHAINS,
           warps / 4, per, per / (warps / 4));
  }
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
  run<0, 1>("HMMA", out, cyc); run<0, 2>("HMMA", out, cyc); run<0, 8>("HMMA", out, cyc);
  run<1, 1>("SHFL", out, cyc); run<1, 8>("SHFL", out, cyc);
  run<2, 1>("MOVM", out, cyc); run<2, 8>("MOVM", out, cyc);
  run<3, 1>("LDSM.x4", out, cyc); run<3, 8>("LDSM.x4", out, cyc);
  run<4, 8>("LDS.128", out, cyc); run<5, 8>("LDSM.x4.T", out, cyc); run<6, 8>("LDS.32", out, cyc);
  run<7, 8>("LDSM.x2", out, cyc);
  return 0;
}
