// Read-bandwidth probe (include/mux.h mux_stream_read): the decode roofline's partition-level
// denominator BW_read(k_d).  Same op size (32 KiB bulk copies) and ring depth class
// as the decode kernel's page stream, no math: what the TMA engines of k_d SMs can pull from HBM.
#include "mux_internal.h"

namespace mux {
namespace {

constexpr uint32_t kChunk = 32 * 1024;
constexpr int kProbeStages = 6;

__global__ void __launch_bounds__(64, 1) stream_read_kernel(const uint8_t* __restrict__ src, size_t chunks) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kProbeStages * kChunk);
  uint64_t* empty = full + kProbeStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kProbeStages; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], 1);
    }
    dev::fence_mbar_init();
  }
  __syncthreads();
  size_t n = 0;   // chunks of this CTA
  if (blockIdx.x < chunks) n = (chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (lane == 0 && warp == 0) {          // producer
    for (size_t i = 0; i < n; ++i) {
      const int s = static_cast<int>(i % kProbeStages);
      if (i >= kProbeStages) dev::mbar_wait(&empty[s], static_cast<uint32_t>((i / kProbeStages) - 1) & 1);
      dev::mbar_expect_tx(&full[s], kChunk);
      dev::bulk_load(ring + s * kChunk, src + (blockIdx.x + i * gridDim.x) * static_cast<size_t>(kChunk), kChunk,
                     &full[s]);
    }
  } else if (lane == 0 && warp == 1) {   // consumer: hand the stage back as soon as it landed
    for (size_t i = 0; i < n; ++i) {
      const int s = static_cast<int>(i % kProbeStages);
      dev::mbar_wait(&full[s], static_cast<uint32_t>(i / kProbeStages) & 1);
      dev::mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
}

}  // namespace
}  // namespace mux

using namespace mux;

extern "C" int mux_stream_read(const void* src, size_t bytes, int32_t num_ctas, mux_stream_t stream) {
  const size_t chunks = bytes / kChunk;
  if (!src || chunks < 1 || num_ctas < 1 || (reinterpret_cast<uintptr_t>(src) & 15))
    return fail(MUX_ERR_INVALID_ARG, "mux_stream_read: need a 16-byte aligned src, >= 32 KiB and num_ctas >= 1");
  const int smem = kProbeStages * kChunk + 2 * kProbeStages * 8 + 1024;
  static bool attr_done = false;
  if (!attr_done) {
    MUX_CUDA(cudaFuncSetAttribute(stream_read_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_done = true;
  }
  stream_read_kernel<<<num_ctas, 64, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), chunks);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
