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
  CUtensorMap tmap_k, tmap_v;        // dims {d, 16, Hkv, layers*pages}, box {64, 16, 1, 1}, SW128
  int64_t layer_elems() const {      // elements per layer of K (or V)
    return static_cast<int64_t>(desc.num_pages) * desc.num_kv_heads * mux::kPage * desc.head_dim;
  }
};

namespace mux {
int pool_tmaps(mux_pool* p);  // build the K/V tensor maps on first use
int check_pool_layer(mux_pool* p, int32_t layer);
}  // namespace mux
