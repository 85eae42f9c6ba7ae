// Paged KV pool object (a1) — internal definition shared by the kernels' host launchers.
#pragma once
#include <deque>
#include <vector>

#include "mux_internal.h"

struct mux_pool {
  mux_pool_desc desc;
  bool owns_storage = false;
  std::deque<int32_t> free_list;     // front = next to allocate
  std::vector<int32_t> ref;          // refcount per page
  bool tmaps_ready = false;
  // 5-D views of K and V: {64 dims, 16 slots, d/64 halves, Hkv, layers*pages}, SWIZZLE_128B.
  // tmap_*1: box = one (page, kv head) block (both 64-dim halves, 4 KiB at d=128)   -> prefill
  // tmap_*g: box = one page of a whole kv-head group of hg heads (hg x 4 KiB)        -> decode
  // tmap_kh: box = one 64-dim half of one (page, kv head) block (2 KiB)            -> prefill K
  // tmap_*g4: box = one page of 4 kv heads (the two-CTA decode of small partitions)
  CUtensorMap tmap_k1, tmap_v1, tmap_kg, tmap_vg, tmap_kh, tmap_kg4, tmap_vg4;
  int hg = 1;                        // kv heads per decode CTA (largest power of two <= 8 dividing Hkv)
  int* d_err = nullptr;              // device error word (bit 0: append clamped a V value to fp16 range)
  int64_t layer_elems() const {      // elements per layer of K (or V)
    return static_cast<int64_t>(desc.num_pages) * desc.num_kv_heads * mux::kPage * desc.head_dim;
  }
};

namespace mux {
int pool_tmaps(mux_pool* p);  // build the K/V tensor maps on first use
int check_pool_layer(mux_pool* p, int32_t layer);
int append_checks(mux_pool* p, const mux_batch* b);  // host checks of a write of the new rows
}  // namespace mux
