"""paper_2504_14489_b200 — B200-native hot path of MuxWise (arXiv 2504.14489).

Thin ctypes binding over the C-ABI library libmux.so (include/mux.h).  Every step of the
path runs in libmux's CUDA kernels; this module only marshals arguments.  PyTorch is used
for device memory and streams.  There is NO CPU fallback: if libmux.so is missing or
cannot be loaded, importing the binding raises.
"""
from .binding import (  # noqa: F401
    MuxError, Batch, Pool, Partition, lib, last_error,
    mux_pool_create, mux_append_kv, mux_prefill_attn, mux_decode_attn, mux_decode_workspace_bytes,
    mux_decode_num_splits, mux_partition_configs, mux_num_prefill_layers, mux_partition_create,
    mux_run_layer, mux_device_sm_count, mux_stream_read, mux_outproj, mux_outproj_pack_w, mux_outproj_packed_bytes, PackedW, Engine, MUX_DTYPE_BF16, MUX_DTYPE_F32, SideTimes, make_side, EventSet, mux_side_plan,
    mux_rope_table, mux_qkv_rope_append, mux_ffn_pack_w13, mux_ffn_swiglu,
    mux_outproj_ar_ws_bytes, mux_outproj_allreduce, mux_outproj_allreduce_emulated,
)
