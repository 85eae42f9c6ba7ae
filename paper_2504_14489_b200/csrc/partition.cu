// a6 SM-partitioned co-execution: green-context SM splits + mux_run_layer.
//
// PAPER: "the intra-process approach GreenContext enables low-overhead resource
// adjustment by binding CUDA streams to specific SMs, with reconfiguration costing only a
// stream synchronization ... both phases reside in the same process ... share the same
// memory space for maintaining a single KV cache pool";  P:498 decode launched first when
// both are pending;  P:529-530 prefill executed layer by layer ("PLs");  P:626-631 16-SM
// partition granularity.
//
// B200 design: every requested split is created ONCE, disjointly (one
// cuDevSmResourceSplitByCount per split -> {k decode SMs, remainder}), each side gets its
// own green context and stream.  Switching split = choosing another pre-created stream
// pair (the paper's "stream synchronisation" reconfiguration).  mux_run_layer enqueues
// the decode side first, then the prefill layers; 1-thread %globaltimer stamp kernels
// bracket each side (per-side start/end without a profiler).
#include <vector>

#include "pool.h"

namespace mux {
namespace {

struct SplitCtx {
  int dec_sms = 0, pf_sms = 0;
  CUgreenCtx gdec = nullptr, gpf = nullptr;
  CUstream sdec = nullptr, spf = nullptr;
};

__global__ void stamp_kernel(unsigned long long* dst) { *dst = dev::globaltimer(); }

}  // namespace
}  // namespace mux

struct mux_part {
  int device = 0;
  int total_sms = 0;
  std::vector<mux::SplitCtx> splits;
  cudaStream_t full_dec = nullptr, full_pf = nullptr;  // split -1: whole GPU, plain streams
  cudaEvent_t ev_in = nullptr, ev_dec = nullptr, ev_pf = nullptr;
  int64_t mem_bytes = 0;                               // device memory taken by the green contexts
};

using namespace mux;

static void destroy_part(mux_part* p) {
  const Driver* d = nullptr;
  driver(&d);
  for (auto& s : p->splits) {
    if (d) {
      if (s.sdec) d->streamDestroy(s.sdec);
      if (s.spf) d->streamDestroy(s.spf);
      if (s.gdec) d->greenCtxDestroy(s.gdec);
      if (s.gpf) d->greenCtxDestroy(s.gpf);
    }
  }
  if (p->full_dec) cudaStreamDestroy(p->full_dec);
  if (p->full_pf) cudaStreamDestroy(p->full_pf);
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->ev_dec) cudaEventDestroy(p->ev_dec);
  if (p->ev_pf) cudaEventDestroy(p->ev_pf);
  delete p;
}

extern "C" {

int mux_partition_create(mux_part_t* out, int32_t device, const int32_t* decode_sms, int32_t n_splits) {
  if (!out || n_splits < 0 || (n_splits > 0 && !decode_sms)) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  *out = nullptr;
  const Driver* d;
  int rc = driver(&d);
  if (rc) return rc;
  MUX_CUDA(cudaSetDevice(device));
  MUX_CUDA(cudaFree(nullptr));  // make sure the primary context exists
  auto* p = new mux_part();
  p->device = device;
  cudaDeviceGetAttribute(&p->total_sms, cudaDevAttrMultiProcessorCount, device);
  size_t free0 = 0, total = 0, free1 = 0;
  cudaMemGetInfo(&free0, &total);
  auto bail = [&](int code) {
    destroy_part(p);
    return code;
  };
  CUdevice cudev;
  CUresult r = d->deviceGet(&cudev, device);
  if (r != CUDA_SUCCESS) return bail(cu_fail(r, "cuDeviceGet"));
  for (int i = 0; i < n_splits; ++i) {
    const int k = decode_sms[i];
    if (k < 8 || k >= p->total_sms) return bail(fail(MUX_ERR_INVALID_ARG, "decode SM count out of range"));
    CUdevResource all{}, grp{}, rem{};
    if ((r = d->deviceGetDevResource(cudev, &all, CU_DEV_RESOURCE_TYPE_SM)) != CUDA_SUCCESS)
      return bail(cu_fail(r, "cuDeviceGetDevResource"));
    unsigned int nb = 1;
    if ((r = d->devSmResourceSplitByCount(&grp, &nb, &all, &rem, 0, static_cast<unsigned>(k))) != CUDA_SUCCESS ||
        nb != 1)
      return bail(r != CUDA_SUCCESS ? cu_fail(r, "cuDevSmResourceSplitByCount")
                                    : fail(MUX_ERR_NO_CONFIG, "SM split produced no group"));
    SplitCtx s;
    s.dec_sms = static_cast<int>(grp.sm.smCount);
    s.pf_sms = static_cast<int>(rem.sm.smCount);
    if (s.pf_sms < 8) return bail(fail(MUX_ERR_NO_CONFIG, "split leaves fewer than 8 SMs for prefill"));
    CUdevResourceDesc ddec, dpf;
    if ((r = d->devResourceGenerateDesc(&ddec, &grp, 1)) != CUDA_SUCCESS)
      return bail(cu_fail(r, "cuDevResourceGenerateDesc(decode)"));
    if ((r = d->devResourceGenerateDesc(&dpf, &rem, 1)) != CUDA_SUCCESS)
      return bail(cu_fail(r, "cuDevResourceGenerateDesc(prefill)"));
    if ((r = d->greenCtxCreate(&s.gdec, ddec, cudev, CU_GREEN_CTX_DEFAULT_STREAM)) != CUDA_SUCCESS)
      return bail(cu_fail(r, "cuGreenCtxCreate(decode)"));
    p->splits.push_back(s);  // owned from here on (cleanup on failure)
    SplitCtx& sp = p->splits.back();
    if ((r = d->greenCtxCreate(&sp.gpf, dpf, cudev, CU_GREEN_CTX_DEFAULT_STREAM)) != CUDA_SUCCESS)
      return bail(cu_fail(r, "cuGreenCtxCreate(prefill)"));
    if ((r = d->greenCtxStreamCreate(&sp.sdec, sp.gdec, CU_STREAM_NON_BLOCKING, 0)) != CUDA_SUCCESS)
      return bail(cu_fail(r, "cuGreenCtxStreamCreate(decode)"));
    if ((r = d->greenCtxStreamCreate(&sp.spf, sp.gpf, CU_STREAM_NON_BLOCKING, 0)) != CUDA_SUCCESS)
      return bail(cu_fail(r, "cuGreenCtxStreamCreate(prefill)"));
  }
  cudaError_t e = cudaStreamCreateWithFlags(&p->full_dec, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->full_pf, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_dec, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_pf, cudaEventDisableTiming);
  if (e != cudaSuccess) return bail(cuda_fail(e, "stream/event create"));
  cudaMemGetInfo(&free1, &total);
  p->mem_bytes = static_cast<int64_t>(free0) - static_cast<int64_t>(free1);
  *out = p;
  return MUX_OK;
}

int mux_partition_destroy(mux_part_t p) {
  if (!p) return MUX_OK;
  cudaDeviceSynchronize();
  destroy_part(p);
  return MUX_OK;
}

int32_t mux_partition_count(mux_part_t p) { return p ? static_cast<int32_t>(p->splits.size()) : 0; }

int mux_partition_query(mux_part_t p, int32_t idx, int32_t* dec_sms, int32_t* pf_sms, mux_stream_t* dec_stream,
                        mux_stream_t* pf_stream) {
  if (!p || idx < -1 || idx >= static_cast<int32_t>(p->splits.size()))
    return fail(MUX_ERR_INVALID_ARG, "split index out of range");
  if (idx == -1) {
    if (dec_sms) *dec_sms = p->total_sms;
    if (pf_sms) *pf_sms = p->total_sms;
    if (dec_stream) *dec_stream = reinterpret_cast<mux_stream_t>(p->full_dec);
    if (pf_stream) *pf_stream = reinterpret_cast<mux_stream_t>(p->full_pf);
    return MUX_OK;
  }
  const auto& s = p->splits[idx];
  if (dec_sms) *dec_sms = s.dec_sms;
  if (pf_sms) *pf_sms = s.pf_sms;
  if (dec_stream) *dec_stream = reinterpret_cast<mux_stream_t>(s.sdec);
  if (pf_stream) *pf_stream = reinterpret_cast<mux_stream_t>(s.spf);
  return MUX_OK;
}

int mux_partition_memory(mux_part_t p, int64_t* bytes) {
  if (!p || !bytes) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  *bytes = p->mem_bytes;
  return MUX_OK;
}

}  // extern "C"

namespace mux {
// elements of the all-reduce run_side enqueues after each layer's out-projection (0 = none)
int64_t side_allreduce_count(const mux_side* s) {
  return ((s->ar_fn || s->ar_peers) && s->w_o) ? static_cast<int64_t>(s->batch->total_q) * s->hidden : 0;
}

void launch_stamp(unsigned long long* dst, cudaStream_t st) { stamp_kernel<<<1, 1, 0, st>>>(dst); }

int run_side(mux_pool_t pool, const mux_side* s, bool decode, int sms, cudaStream_t st, unsigned long long* t0,
             unsigned long long* t1) {
  if (s->w_o && (s->o_dtype != MUX_DTYPE_BF16 || !s->y || s->hidden < 1))
    return fail(MUX_ERR_INVALID_ARG, "out-projection needs bf16 o, y and hidden >= 1");
  if (s->ar_fn && (!s->w_o || !s->ar_comm || s->y_dtype != MUX_DTYPE_BF16))
    return fail(MUX_ERR_INVALID_ARG, "all-reduce needs w_o, a bf16 y and ar_comm");
  if (s->ar_peers && (!s->w_o || s->ar_fn || s->y_dtype != MUX_DTYPE_BF16 || s->ar_peers->rank < 0 ||
                      s->ar_peers->rank >= s->ar_peers->world || s->ar_peers->y[s->ar_peers->rank] != s->y))
    return fail(MUX_ERR_INVALID_ARG, "fused all-reduce needs w_o, a bf16 y == ar_peers->y[rank] and no ar_fn");
  if (s->w_qkv && (s->append || !s->x_in || !s->rope || s->hidden_in < 8))
    return fail(MUX_ERR_INVALID_ARG, "fused QKV needs x_in, hidden_in, rope and append == 0");
  if (s->w13 && (!s->w_o || !s->w2 || !s->ffn_h || !s->ffn_y || s->ffn_inter < 128 || s->y_dtype != MUX_DTYPE_BF16))
    return fail(MUX_ERR_INVALID_ARG, "FFN needs w_o (bf16 y), w2, ffn_h, ffn_y and ffn_inter");
  using nccl_allreduce_t = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  auto ar = reinterpret_cast<nccl_allreduce_t>(s->ar_fn);
  auto ev = [&](int i, int which) -> int {
    if (s->attn_events) MUX_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(s->attn_events[2 * i + which]), st));
    return MUX_OK;
  };
  if (t0) stamp_kernel<<<1, 1, 0, st>>>(t0);
  const int nl = pool->desc.num_layers;
  int splits = 1;
  if (decode) {
    splits = s->num_splits > 0 ? s->num_splits
                               : mux_decode_num_splits(s->batch->num_seqs, pool->desc.num_kv_heads,
                                                       pool->desc.head_dim, s->batch->h_kv_len, s->batch->max_kv, sms);
  }
  for (int i = 0; i < s->num_layers; ++i) {
    const int layer = (s->layer0 + i) % nl;
    auto at = [&](const void* base, int64_t stride) {
      return base ? static_cast<const void*>(static_cast<const uint8_t*>(base) + stride * i) : nullptr;
    };
    int rc;
    if (s->w_qkv) {   // f4: projection + RoPE + append in one kernel; q is its output
      rc = qkv_launch(pool, layer, s->batch, s->num_q_heads, s->x_in, s->hidden_in, s->w_qkv, s->rope,
                      s->rope_max_pos, const_cast<void*>(at(s->q, s->q_stride)), reinterpret_cast<mux_stream_t>(st), sms);
      if (rc) return rc;
    }
    if (s->append) {
      rc = mux_append_kv(pool, layer, s->batch, at(s->k_new, s->kv_stride), at(s->v_new, s->kv_stride),
                         reinterpret_cast<mux_stream_t>(st));
      if (rc) return rc;
    }
    void* o = const_cast<void*>(at(s->o, s->o_stride));
    float* lse = static_cast<float*>(const_cast<void*>(at(s->lse, s->lse_stride)));
    if ((rc = ev(i, 0))) return rc;
    if (decode)
      rc = decode_launch_sms(pool, layer, s->batch, s->num_q_heads, at(s->q, s->q_stride), o, s->o_dtype, lse,
                             s->scale, splits, s->ws, s->ws_bytes, reinterpret_cast<mux_stream_t>(st), sms);
    else
      rc = prefill_launch_sms(pool, layer, s->batch, s->num_q_heads, at(s->q, s->q_stride), o, s->o_dtype, lse,
                              s->scale, reinterpret_cast<mux_stream_t>(st), sms);
    if (rc) return rc;
    if ((rc = ev(i, 1))) return rc;
    if (s->w_o) {
      void* y = const_cast<void*>(at(s->y, s->y_stride));
      if (s->ar_peers) {   // f4: out-projection + all-reduce in one kernel
        mux_ar_peers pr = *s->ar_peers;
        if (pr.epoch) pr.epoch += static_cast<uint32_t>(i);   // explicit epochs; 0 = the kernel's counter
        for (int r = 0; r < pr.world; ++r) pr.y[r] = static_cast<uint8_t*>(pr.y[r]) + s->y_stride * i;
        rc = mux_outproj_allreduce(o, at(s->w_o, s->w_stride), s->batch->total_q,
                                   s->num_q_heads * pool->desc.head_dim, s->hidden, &pr, sms,
                                   reinterpret_cast<mux_stream_t>(st));
        if (rc) return rc;
      } else {
        rc = outproj_launch(o, at(s->w_o, s->w_stride), y, s->y_dtype, s->batch->total_q,
                            s->num_q_heads * pool->desc.head_dim, s->hidden, reinterpret_cast<mux_stream_t>(st), sms);
        if (rc) return rc;
        if (ar) {
          const int nrc = ar(y, y, static_cast<size_t>(side_allreduce_count(s)), 9 /* ncclBfloat16 */,
                             0 /* ncclSum */, s->ar_comm, st);
          if (nrc) return fail(MUX_ERR_CUDA, "ncclAllReduce of the out-projection failed (NCCL error " + std::to_string(nrc) + ")");
        }
      }
      if (s->w13) {   // f4: the layer's FFN on the attention block's output
        rc = ffn_launch(y, s->w13, s->w2, s->ffn_h, s->ffn_y, s->batch->total_q, s->hidden, s->ffn_inter,
                        reinterpret_cast<mux_stream_t>(st), sms);
        if (rc) return rc;
      }
    }
    if (s->hook) s->hook(s->hook_user, decode ? 0 : 1, i, reinterpret_cast<mux_stream_t>(st));
  }
  if (t1) stamp_kernel<<<1, 1, 0, st>>>(t1);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}
}  // namespace mux

extern "C" {

int mux_side_plan(const mux_side* s, int32_t pool_layers, int64_t* out, int32_t cap, int32_t* n) {
  if (!s || !s->batch || !n || pool_layers < 1 || s->num_layers < 0 || s->layer0 < 0)
    return fail(MUX_ERR_INVALID_ARG, "mux_side_plan: bad argument");
  for (int i = 0; i < s->num_layers && out && i < cap; ++i) {
    out[2 * i] = (s->layer0 + i) % pool_layers;
    out[2 * i + 1] = mux::side_allreduce_count(s);
  }
  *n = s->num_layers;
  return MUX_OK;
}

int mux_run_layer(mux_part_t part, int32_t split_idx, mux_pool_t pool, const mux_side* prefill,
                  const mux_side* decode, mux_side_times* times, mux_stream_t join_stream) {
  if (!part || !pool) return fail(MUX_ERR_INVALID_ARG, "part/pool NULL");
  if (split_idx < -1 || split_idx >= static_cast<int32_t>(part->splits.size()))
    return fail(MUX_ERR_INVALID_ARG, "split index out of range");
  for (const mux_side* s : {prefill, decode}) {
    if (!s) continue;
    if (!s->batch || s->num_layers < 0 || s->layer0 < 0) return fail(MUX_ERR_INVALID_ARG, "bad mux_side");
  }
  int dec_sms, pf_sms;
  mux_stream_t ds, ps;
  int rc = mux_partition_query(part, split_idx, &dec_sms, &pf_sms, &ds, &ps);
  if (rc) return rc;
  cudaStream_t dst = reinterpret_cast<cudaStream_t>(ds), pst = reinterpret_cast<cudaStream_t>(ps);
  cudaStream_t js = reinterpret_cast<cudaStream_t>(join_stream);
  MUX_CUDA(cudaEventRecord(part->ev_in, js));
  auto* tt = reinterpret_cast<unsigned long long*>(times);
  // decode first: its whole iteration is enqueued before any prefill layer
  if (decode) {
    MUX_CUDA(cudaStreamWaitEvent(dst, part->ev_in, 0));
    if ((rc = run_side(pool, decode, true, dec_sms, dst, tt ? tt + 0 : nullptr, tt ? tt + 1 : nullptr))) return rc;
    MUX_CUDA(cudaEventRecord(part->ev_dec, dst));
  }
  if (prefill) {
    MUX_CUDA(cudaStreamWaitEvent(pst, part->ev_in, 0));
    if ((rc = run_side(pool, prefill, false, pf_sms, pst, tt ? tt + 2 : nullptr, tt ? tt + 3 : nullptr))) return rc;
    MUX_CUDA(cudaEventRecord(part->ev_pf, pst));
  }
  if (decode) MUX_CUDA(cudaStreamWaitEvent(js, part->ev_dec, 0));
  if (prefill) MUX_CUDA(cudaStreamWaitEvent(js, part->ev_pf, 0));
  return MUX_OK;
}

}  // extern "C"
