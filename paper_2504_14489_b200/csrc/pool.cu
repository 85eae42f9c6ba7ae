// a1 paged KV pool + host page allocator, and a2 mux_append_kv (slot-mapped bf16 scatter).
//
// P:159 / P:426 / P:473: one KV pool shared by prefill and decode and by all requests;
// paged (PagedAttention).  P:251-252: the KV cache is filled as prefill and
// decode process tokens.  Allocation policy: DESIGN.md R18 (paper silent).
#include <string.h>

#include <algorithm>

#include "pool.h"

namespace mux {

// splitmix64 counter generator + Fisher-Yates: the seeded initial free list (R18)
static uint64_t splitmix64(uint64_t& s) {
  s += 0x9E3779B97F4A7C15ull;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int pool_tmaps(mux_pool* p) {
  if (p->tmaps_ready) return MUX_OK;
  const auto& d = p->desc;
  const uint64_t D = static_cast<uint64_t>(d.head_dim);
  uint64_t dims[5] = {64, static_cast<uint64_t>(kPage), D / 64, static_cast<uint64_t>(d.num_kv_heads),
                      static_cast<uint64_t>(d.num_layers) * static_cast<uint64_t>(d.num_pages)};
  uint64_t strides[4] = {D * 2, 128, kPage * D * 2, static_cast<uint64_t>(d.num_kv_heads) * kPage * D * 2};
  // kv heads per decode CTA (csrc/decode.cu): the largest power of two <= 8 (4 under the 2-CTA
  // switch) dividing Hkv, the instantiations launch_decode has (Hkv = 3, 6, 12 ... -> 1 or 2)
  int hg = 1;
  for (int c = 2; c <= 8; c *= 2)
    if (d.num_kv_heads % c == 0) hg = c;
  p->hg = hg;
  uint32_t box1[5] = {64, static_cast<uint32_t>(kPage), static_cast<uint32_t>(D / 64), 1, 1};
  uint32_t boxg[5] = {64, static_cast<uint32_t>(kPage), static_cast<uint32_t>(D / 64), static_cast<uint32_t>(hg), 1};
  int rc;
  if ((rc = make_tmap_bf16(&p->tmap_k1, d.k_storage, 5, dims, strides, box1))) return rc;
  if ((rc = make_tmap_bf16(&p->tmap_v1, d.v_storage, 5, dims, strides, box1))) return rc;
  if ((rc = make_tmap_bf16(&p->tmap_kg, d.k_storage, 5, dims, strides, boxg))) return rc;
  if ((rc = make_tmap_bf16(&p->tmap_vg, d.v_storage, 5, dims, strides, boxg))) return rc;
  if (d.num_kv_heads % 4 == 0) {   // two-CTA decode on small partitions: pages of 4 kv heads
    uint32_t box4[5] = {64, static_cast<uint32_t>(kPage), static_cast<uint32_t>(D / 64), 4, 1};
    if ((rc = make_tmap_bf16(&p->tmap_kg4, d.k_storage, 5, dims, strides, box4))) return rc;
    if ((rc = make_tmap_bf16(&p->tmap_vg4, d.v_storage, 5, dims, strides, box4))) return rc;
  }
  uint32_t boxh[5] = {64, static_cast<uint32_t>(kPage), 1, 1, 1};
  if ((rc = make_tmap_bf16(&p->tmap_kh, d.k_storage, 5, dims, strides, boxh))) return rc;
  if (!p->d_err) {
    MUX_CUDA(cudaMalloc(&p->d_err, sizeof(int)));
    MUX_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
  }
  p->tmaps_ready = true;
  return MUX_OK;
}

// host checks of a write of the batch's new rows (when the host copies of the tables are given):
// page ids in range; no write into a page shared by another sequence (R13)
int append_checks(mux_pool* p, const mux_batch* b) {
  if (!(b->h_qo_indptr && b->h_kv_len && b->h_page_indptr && b->h_page_ids)) return MUX_OK;
  for (int s = 0; s < b->num_seqs; ++s) {
    int n = b->h_qo_indptr[s + 1] - b->h_qo_indptr[s];
    int L = b->h_kv_len[s];
    for (int pg = (L - n) / kPage; pg <= (L - 1) / kPage; ++pg) {
      int id = b->h_page_ids[b->h_page_indptr[s] + pg];
      if (id < 0 || id >= p->desc.num_pages) return fail(MUX_ERR_INVALID_ARG, "page id out of range");
      if (p->ref[id] > 1) return fail(MUX_ERR_SHARED_PAGE_WRITE, "append would write a shared page");
    }
  }
  return MUX_OK;
}

int check_pool_layer(mux_pool* p, int32_t layer) {
  if (!p) return fail(MUX_ERR_INVALID_ARG, "pool is NULL");
  if (layer < 0 || layer >= p->desc.num_layers) return fail(MUX_ERR_INVALID_ARG, "layer out of range");
  return MUX_OK;
}

// ------------------------------------------------------------------ append kernel (a2)
// One CTA per new row; thread i moves 16-byte chunk i of the row's Hkv*d bf16 for K and V.
// slot(b, t) = page_ids[page_indptr[b] + t/16] * 16 + t%16.
__global__ void __launch_bounds__(256) append_kv_kernel(uint4* __restrict__ kpool, uint4* __restrict__ vpool,
                                                        const uint4* __restrict__ k_new,
                                                        const uint4* __restrict__ v_new,
                                                        const int32_t* __restrict__ qo_indptr,
                                                        const int32_t* __restrict__ kv_len,
                                                        const int32_t* __restrict__ page_indptr,
                                                        const int32_t* __restrict__ page_ids, int num_seqs,
                                                        int chunks_per_head, int hkv, int* __restrict__ err) {
  const int row = blockIdx.x;
  int lo = 0, hi = num_seqs - 1;  // last b with qo_indptr[b] <= row
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (__ldg(qo_indptr + mid) <= row) lo = mid; else hi = mid - 1;
  }
  const int b = lo;
  const int q0 = __ldg(qo_indptr + b);
  const int n = __ldg(qo_indptr + b + 1) - q0;
  const int t = __ldg(kv_len + b) - n + (row - q0);
  const int page = __ldg(page_ids + __ldg(page_indptr + b) + (t >> 4));
  const int slot = t & 15;
  const int row_chunks = chunks_per_head * hkv;
  for (int i = threadIdx.x; i < row_chunks; i += blockDim.x) {
    const int h = i / chunks_per_head, c = i - h * chunks_per_head;
    const size_t dst = ((static_cast<size_t>(page) * hkv + h) * kPage + slot) * chunks_per_head + c;
    const size_t src = static_cast<size_t>(row) * row_chunks + i;
    kpool[dst] = __ldg(k_new + src);
    // the V cache holds fp16 (R25): bf16 -> fp16 round-to-nearest-even, exact for every
    // bf16 value in [2^-14, 65504]; larger magnitudes (bf16 >= 65536) clamp to +-65504 and flag the pool
    uint4 w = __ldg(v_new + src);
    const uint32_t mx = __vmaxu2(__vmaxu2(w.x & 0x7FFF7FFFu, w.y & 0x7FFF7FFFu), __vmaxu2(w.z & 0x7FFF7FFFu, w.w & 0x7FFF7FFFu));
    if (__vmaxu2(mx, 0x477F477Fu) != 0x477F477Fu && err) atomicOr(err, MUX_POOL_ERR_V_RANGE);
    w.x = dev::pack_f16_satfinite(dev::bf16lo(w.x), dev::bf16hi(w.x));
    w.y = dev::pack_f16_satfinite(dev::bf16lo(w.y), dev::bf16hi(w.y));
    w.z = dev::pack_f16_satfinite(dev::bf16lo(w.z), dev::bf16hi(w.z));
    w.w = dev::pack_f16_satfinite(dev::bf16lo(w.w), dev::bf16hi(w.w));
    vpool[dst] = w;
  }
}

}  // namespace mux

using namespace mux;

extern "C" {

int mux_pool_create(mux_pool_t* out, const mux_pool_desc* desc) {
  if (!out || !desc) return fail(MUX_ERR_INVALID_ARG, "mux_pool_create: NULL argument");
  *out = nullptr;
  const auto& d = *desc;
  if (d.page_size != kPage) return fail(MUX_ERR_UNSUPPORTED, "page_size must be 16");
  if (d.head_dim != 64 && d.head_dim != 128) return fail(MUX_ERR_UNSUPPORTED, "head_dim must be 64 or 128");
  if (d.num_layers < 1 || d.num_pages < 1 || d.num_kv_heads < 1)
    return fail(MUX_ERR_INVALID_ARG, "num_layers/num_pages/num_kv_heads must be >= 1");
  if ((d.k_storage == nullptr) != (d.v_storage == nullptr))
    return fail(MUX_ERR_INVALID_ARG, "k_storage and v_storage must be both NULL or both set");
  if ((reinterpret_cast<uintptr_t>(d.k_storage) | reinterpret_cast<uintptr_t>(d.v_storage)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "pool storage must be 16-byte aligned");
  auto* p = new mux_pool();
  p->desc = d;
  if (!d.k_storage) {
    size_t bytes = static_cast<size_t>(p->layer_elems()) * d.num_layers * 2;
    void *k = nullptr, *v = nullptr;
    cudaError_t e = cudaMalloc(&k, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&v, bytes);
    if (e != cudaSuccess) {
      if (k) cudaFree(k);
      delete p;
      return cuda_fail(e, "cudaMalloc(pool storage)");
    }
    p->desc.k_storage = k;
    p->desc.v_storage = v;
    p->owns_storage = true;
  }
  std::vector<int32_t> perm(d.num_pages);
  for (int32_t i = 0; i < d.num_pages; ++i) perm[i] = i;
  uint64_t s = d.free_list_seed;
  for (int64_t i = d.num_pages - 1; i > 0; --i) {
    uint64_t j = splitmix64(s) % static_cast<uint64_t>(i + 1);
    std::swap(perm[i], perm[j]);
  }
  p->free_list.assign(perm.begin(), perm.end());
  p->ref.assign(d.num_pages, 0);
  *out = p;
  return MUX_OK;
}

int mux_pool_destroy(mux_pool_t p) {
  if (!p) return MUX_OK;
  if (p->d_err) cudaFree(p->d_err);
  if (p->owns_storage) {
    cudaFree(p->desc.k_storage);
    cudaFree(p->desc.v_storage);
  }
  delete p;
  return MUX_OK;
}

int mux_pool_alloc_pages(mux_pool_t p, int32_t n, int32_t* out_ids) {
  if (!p || n < 0 || (n > 0 && !out_ids)) return fail(MUX_ERR_INVALID_ARG, "mux_pool_alloc_pages: bad argument");
  if (static_cast<size_t>(n) > p->free_list.size())
    return fail(MUX_ERR_POOL_EXHAUSTED, "pool exhausted: requested more pages than free");
  for (int32_t i = 0; i < n; ++i) {
    int32_t id = p->free_list.front();
    p->free_list.pop_front();
    p->ref[id] = 1;
    out_ids[i] = id;
  }
  return MUX_OK;
}

static int check_live(mux_pool_t p, int32_t n, const int32_t* ids) {
  if (!p || n < 0 || (n > 0 && !ids)) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  for (int32_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= p->desc.num_pages || p->ref[ids[i]] < 1)
      return fail(MUX_ERR_INVALID_ARG, "page id out of range or not allocated");
  return MUX_OK;
}

int mux_pool_share_pages(mux_pool_t p, int32_t n, const int32_t* ids) {
  int rc = check_live(p, n, ids);
  if (rc) return rc;
  for (int32_t i = 0; i < n; ++i) p->ref[ids[i]] += 1;
  return MUX_OK;
}

int mux_pool_free_pages(mux_pool_t p, int32_t n, const int32_t* ids) {
  int rc = check_live(p, n, ids);
  if (rc) return rc;
  for (int32_t i = 0; i < n; ++i) {
    if (--p->ref[ids[i]] == 0) p->free_list.push_back(ids[i]);
  }
  return MUX_OK;
}

int mux_pool_num_free(mux_pool_t p, int32_t* out) {
  if (!p || !out) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  *out = static_cast<int32_t>(p->free_list.size());
  return MUX_OK;
}

int mux_pool_refcount(mux_pool_t p, int32_t page, int32_t* out) {
  if (!p || !out || page < 0 || page >= p->desc.num_pages) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  *out = p->ref[page];
  return MUX_OK;
}

int mux_pool_free_list(mux_pool_t p, int32_t* out, int32_t cap, int32_t* n_out) {
  if (!p || !n_out) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  int32_t n = 0;
  for (int32_t id : p->free_list) {
    if (out && n < cap) out[n] = id;
    ++n;
  }
  *n_out = n;
  return MUX_OK;
}

int mux_pool_error_flags(mux_pool_t p, uint32_t* flags, int32_t clear) {
  if (!p || !flags) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  *flags = 0;
  if (!p->d_err) return MUX_OK;
  int v = 0;
  MUX_CUDA(cudaMemcpy(&v, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  *flags = static_cast<uint32_t>(v);
  if (clear) MUX_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
  return MUX_OK;
}

int mux_pool_storage(mux_pool_t p, void** k, void** v) {
  if (!p) return fail(MUX_ERR_INVALID_ARG, "pool is NULL");
  if (k) *k = p->desc.k_storage;
  if (v) *v = p->desc.v_storage;
  return MUX_OK;
}

int mux_append_kv(mux_pool_t p, int32_t layer, const mux_batch* b, const void* k_new, const void* v_new,
                  mux_stream_t stream) {
  int rc = check_pool_layer(p, layer);
  if (rc) return rc;
  if ((rc = validate_batch(b, false))) return rc;
  if (!k_new || !v_new) return fail(MUX_ERR_INVALID_ARG, "k_new/v_new NULL");
  if ((reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new)) & 15)
    return fail(MUX_ERR_INVALID_ARG, "k_new/v_new must be 16-byte aligned");
  if ((rc = append_checks(p, b))) return rc;
  if ((rc = pool_tmaps(p))) return rc;   // also allocates the pool's device error word
  const int d = p->desc.head_dim, hkv = p->desc.num_kv_heads;
  const int chunks_per_head = d / 8;
  const size_t off = static_cast<size_t>(layer) * p->layer_elems();
  auto* kp = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p->desc.k_storage) + off);
  auto* vp = reinterpret_cast<uint4*>(static_cast<uint16_t*>(p->desc.v_storage) + off);
  int threads = std::min(256, std::max(32, ((chunks_per_head * hkv + 31) / 32) * 32));
  append_kv_kernel<<<b->total_q, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      kp, vp, static_cast<const uint4*>(k_new), static_cast<const uint4*>(v_new), b->qo_indptr, b->kv_len,
      b->page_indptr, b->page_ids, b->num_seqs, chunks_per_head, hkv, p->d_err);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

}  // extern "C"
