// Host plumbing of libmux: thread-local errors, driver entry points, tensor-map encoding,
// batch validation and the host-only helpers of the ABI (partition-config rule, N_PL).
#include <math.h>
#include <stdio.h>

#include <mutex>
#include <string>

#include "mux_internal.h"

namespace mux {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s failed: %s (%d)", what, cudaGetErrorString(e), static_cast<int>(e));
  return fail(MUX_ERR_CUDA, buf);
}

int cu_fail(CUresult r, const char* what) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s failed: CUresult %d", what, static_cast<int>(r));
  return fail(MUX_ERR_CUDA, buf);
}

template <typename F>
static bool entry(const char* name, F* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return false;
  *out = reinterpret_cast<F>(fn);
  return true;
}

int driver(const Driver** out) {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    bool ok = true;
    ok &= entry("cuTensorMapEncodeTiled", &d.tensorMapEncodeTiled);
    ok &= entry("cuDeviceGet", &d.deviceGet);
    ok &= entry("cuDeviceGetDevResource", &d.deviceGetDevResource);
    ok &= entry("cuDevSmResourceSplitByCount", &d.devSmResourceSplitByCount);
    ok &= entry("cuDevResourceGenerateDesc", &d.devResourceGenerateDesc);
    ok &= entry("cuGreenCtxCreate", &d.greenCtxCreate);
    ok &= entry("cuGreenCtxDestroy", &d.greenCtxDestroy);
    ok &= entry("cuGreenCtxStreamCreate", &d.greenCtxStreamCreate);
    ok &= entry("cuGreenCtxGetDevResource", &d.greenCtxGetDevResource);
    ok &= entry("cuStreamDestroy", &d.streamDestroy);
    entry("cuStreamGetGreenCtx", &d.streamGetGreenCtx);
    d.ok = ok;
  });
  if (!d.ok) return fail(MUX_ERR_CUDA, "CUDA driver entry points unavailable (no driver / GPU?)");
  *out = &d;
  return MUX_OK;
}

int make_tmap_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                   const uint64_t* strides_bytes, const uint32_t* box, bool swizzle) {
  const Driver* d;
  int rc = driver(&d);
  if (rc) return rc;
  cuuint32_t elem_strides[5] = {1, 1, 1, 1, 1};
  CUresult r = d->tensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base),
                                       reinterpret_cast<const cuuint64_t*>(dims),
                                       reinterpret_cast<const cuuint64_t*>(strides_bytes),
                                       reinterpret_cast<const cuuint32_t*>(box), elem_strides,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuTensorMapEncodeTiled");
  return MUX_OK;
}

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  return dev;
}

int device_sm_count() {
  int dev = current_device(), n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

int stream_sm_count(cudaStream_t stream) {
  const Driver* d;
  if (stream && driver(&d) == MUX_OK && d->streamGetGreenCtx) {
    CUgreenCtx g = nullptr;
    CUdevResource res{};
    if (d->streamGetGreenCtx(reinterpret_cast<CUstream>(stream), &g) == CUDA_SUCCESS && g &&
        d->greenCtxGetDevResource(g, &res, CU_DEV_RESOURCE_TYPE_SM) == CUDA_SUCCESS && res.sm.smCount > 0)
      return static_cast<int>(res.sm.smCount);
  }
  return device_sm_count();
}

int validate_batch(const mux_batch* b, bool decode_shape) {
  if (!b) return fail(MUX_ERR_INVALID_ARG, "batch is NULL");
  if (b->num_seqs < 1) return fail(MUX_ERR_INVALID_ARG, "batch.num_seqs < 1");
  if (!b->qo_indptr || !b->kv_len || !b->page_indptr || !b->page_ids)
    return fail(MUX_ERR_INVALID_ARG, "batch device arrays must be non-NULL");
  if (b->total_q < b->num_seqs || b->max_q < 1 || b->max_kv < b->max_q)
    return fail(MUX_ERR_INVALID_ARG, "batch totals inconsistent (total_q/max_q/max_kv)");
  if (decode_shape && (b->max_q != 1 || b->total_q != b->num_seqs))
    return fail(MUX_ERR_INVALID_ARG, "decode batch must have exactly one new token per sequence");
  if (b->h_qo_indptr && b->h_kv_len) {
    if (b->h_qo_indptr[0] != 0) return fail(MUX_ERR_INVALID_ARG, "qo_indptr[0] != 0");
    int max_q = 0, max_kv = 0;
    for (int s = 0; s < b->num_seqs; ++s) {
      int n = b->h_qo_indptr[s + 1] - b->h_qo_indptr[s];
      int L = b->h_kv_len[s];
      if (n < 1) return fail(MUX_ERR_INVALID_ARG, "sequence with n_b < 1 new tokens (S:85)");
      if (L < n) return fail(MUX_ERR_INVALID_ARG, "kv_len < number of new tokens");
      if (n > max_q) max_q = n;
      if (L > max_kv) max_kv = L;
      if (b->h_page_indptr) {
        int np = b->h_page_indptr[s + 1] - b->h_page_indptr[s];
        if (np != (L + kPage - 1) / kPage)
          return fail(MUX_ERR_INVALID_ARG, "page table length != ceil(kv_len/16)");
      }
    }
    if (b->h_qo_indptr[b->num_seqs] != b->total_q) return fail(MUX_ERR_INVALID_ARG, "total_q != qo_indptr[B]");
    if (max_q != b->max_q || max_kv != b->max_kv)
      return fail(MUX_ERR_INVALID_ARG, "max_q / max_kv do not match the host arrays");
  }
  return MUX_OK;
}

}  // namespace mux

extern "C" {

const char* mux_last_error(void) { return mux::g_last_error.c_str(); }

#ifndef MUX_EXTRA_FLAGS
#define MUX_EXTRA_FLAGS ""
#endif
// the developer A/B defines this build was compiled with (build.py passes MUX_NVCC_EXTRA here), so a
// bench line or test log can tell a production build ("extra=") from an A/B build
const char* mux_version(void) { return "mux-b200 0.2 sm_100a extra=" MUX_EXTRA_FLAGS; }

int32_t mux_partition_configs(int32_t total_sms, int32_t granularity, int32_t min_side, int32_t* out,
                              int32_t cap) {
  if (total_sms <= 0 || granularity <= 0 || min_side < 0) {
    mux::set_error("mux_partition_configs: bad arguments");
    return -MUX_ERR_INVALID_ARG;
  }
  int32_t n = 0;
  for (int32_t k = 1; total_sms - k * granularity >= min_side; ++k) {
    if (out && n < cap) out[n] = k * granularity;
    ++n;
  }
  if (n == 0) {
    mux::set_error("mux_partition_configs: no split leaves min_side SMs for prefill");
    return -MUX_ERR_NO_CONFIG;
  }
  return n;
}

int32_t mux_num_prefill_layers(double t_decode, double t_prefill, int32_t n_layers_model, int32_t remaining) {
  if (remaining <= 0) return 0;
  if (!(t_decode > 0.0) || !(t_prefill > 0.0) || n_layers_model <= 0) return 1;
  double x = ceil(t_decode * static_cast<double>(n_layers_model) / t_prefill);
  if (x < 1.0) x = 1.0;
  if (x > static_cast<double>(remaining)) return remaining;
  return static_cast<int32_t>(x);
}

int32_t mux_device_sm_count(int32_t device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
  return n;
}

}  // extern "C"
