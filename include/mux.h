/*
 * mux.h — C ABI of the B200-native MuxWise hot path (arXiv 2504.14489, "Towards
 * High-Goodput LLM Serving with Prefill-decode Multiplexing").
 *
 * What sits behind this boundary (PAPER.md line numbers "P:n"):
 *   - ONE paged KV-cache pool shared by prefill and decode ("they share the memory
 *     space on each GPU, enabling efficient KV cache reuse"; "a single KV cache
 *     pool"; P:1111 PagedAttention) ............................ mux_pool_*
 *   - KV generated as tokens are processed ........... mux_append_kv
 *   - prefill attention with a cached prefix, Table 2 row "Prefill w/ cache"
 *     O(nd^2 + Lnd), Eq.1 .................... mux_prefill_attn
 *   - decode attention over r+1 keys, Table 2 row "Decode", Eq.2,
 *     split-KV + log-sum-exp combine (BASELINE.json north_star) .. mux_decode_attn
 *   - intra-process SM partitioning with streams bound to SM sets, reconfiguration =
 *     a stream synchronization (GreenContext); 16-SM granularity;
 *     layer-wise prefill execution; decode launched first
 *                                          ..................... mux_partition_*, mux_run_layer
 *
 * Conventions (all functions):
 *   - Return an int status (enum mux_status). Errors are returned, never thrown or
 *     printed; mux_last_error() gives a thread-local message for the last failure.
 *   - Arguments are validated on the host BEFORE any launch; a failed call enqueues
 *     nothing.
 *   - "device" pointers are CUDA device memory (the Python binding passes torch
 *     storage); "host" pointers are ordinary CPU memory.  The caller owns every buffer
 *     it passes (Q/O/LSE, page tables, workspaces, streams).  The library owns pool
 *     metadata, the host page allocator and (only when k_storage/v_storage are NULL)
 *     the pool storage, plus partition objects' green contexts and streams.
 *   - All device work is asynchronous on the given stream; nothing synchronises the
 *     device implicitly except create/destroy calls.
 *   - Host-side calls on one pool / partition object are NOT thread-safe.
 *   - Layout: K and V are separate bf16 tensors
 *     [num_layers][num_pages][Hkv][16][d] ("HND" per page), page size 16, one page table
 *     per sequence shared by all layers; token t of sequence b lives at
 *     (page_ids[page_indptr[b] + t/16], slot t%16).
 */
#ifndef MUX_H_
#define MUX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the ABI is the only exported surface of libmux.so */
#endif

/* A CUDA stream (identical to cudaStream_t / CUstream). NULL = legacy default stream. */
typedef struct CUstream_st* mux_stream_t;

enum mux_status {
  MUX_OK = 0,
  MUX_ERR_INVALID_ARG = 1,       /* bad pointer/shape/length (e.g. n_b < 1, kv_len < n_b) */
  MUX_ERR_UNSUPPORTED = 2,       /* head_dim not in {64,128}, page_size != 16, Hq % Hkv != 0, group > 16 */
  MUX_ERR_POOL_EXHAUSTED = 3,    /* fewer free pages than requested (no partial effect) */
  MUX_ERR_SHARED_PAGE_WRITE = 4, /* append would write a page whose refcount > 1 */
  MUX_ERR_NO_CONFIG = 5,         /* no SM split satisfies the rule */
  MUX_ERR_CUDA = 6,              /* a CUDA runtime/driver call failed (message has the code) */
  MUX_ERR_WORKSPACE = 7          /* workspace NULL or smaller than mux_decode_workspace_bytes() */
};

enum mux_dtype { MUX_DTYPE_BF16 = 0, MUX_DTYPE_F32 = 1 };

typedef struct mux_pool* mux_pool_t;
typedef struct mux_part* mux_part_t;

/* ------------------------------------------------------------------------------------
 * Paged KV pool (a1).  P:159/P:426/P:473 one pool shared across phases and requests;
 * P:1111 paged.  The allocation policy is this library's (paper silent, R18):
 *   free list = permutation of [0, num_pages) by Fisher-Yates with a splitmix64
 *   generator seeded by free_list_seed (i = n-1..1: j = next() % (i+1); swap a[i], a[j]);
 *   alloc pops from the front (all-or-nothing), free appends to the tail (FIFO) when the
 *   refcount reaches 0, share increments refcounts (read-only prefix sharing).
 * ---------------------------------------------------------------------------------- */
typedef struct {
  int32_t num_layers;    /* >= 1 */
  int32_t num_pages;     /* >= 1 */
  int32_t page_size;     /* must be 16 */
  int32_t num_kv_heads;  /* Hkv held by THIS pool (the local shard under KV-head sharding) */
  int32_t head_dim;      /* 64 or 128 */
  void* k_storage;       /* device, 16-B aligned, num_layers*num_pages*Hkv*16*d bf16; NULL => library cudaMalloc */
  void* v_storage;       /* device, same shape, IEEE fp16 (binary16): mux_append_kv stores V rows as fp16
                            (R25, exact for bf16 values in [2^-14, 65504]); K stays bf16;
                            must be both NULL or both non-NULL */
  uint64_t free_list_seed;
} mux_pool_desc;

int mux_pool_create(mux_pool_t* out, const mux_pool_desc* desc);
int mux_pool_destroy(mux_pool_t pool);
/* host; writes n page ids to out_ids (host) in allocation order; all-or-nothing */
int mux_pool_alloc_pages(mux_pool_t pool, int32_t n, int32_t* out_ids);
/* host; refcount += 1 for each id (ids must be live) */
int mux_pool_share_pages(mux_pool_t pool, int32_t n, const int32_t* ids);
/* host; refcount -= 1 for each id, pages reaching 0 go to the free-list tail (FIFO) */
int mux_pool_free_pages(mux_pool_t pool, int32_t n, const int32_t* ids);
int mux_pool_num_free(mux_pool_t pool, int32_t* out);
int mux_pool_refcount(mux_pool_t pool, int32_t page, int32_t* out);
/* copy the current free list (front first) to out (host, capacity cap); *n_out = length */
int mux_pool_free_list(mux_pool_t pool, int32_t* out, int32_t cap, int32_t* n_out);
int mux_pool_storage(mux_pool_t pool, void** k_storage, void** v_storage);
/* Sticky device-side error bits of kernels that used this pool (synchronises the device).
 * bit 0 (MUX_POOL_ERR_V_RANGE): mux_append_kv met a V value with |v| >= 65536, outside the fp16
 * range the V cache is stored in (R25, "P precision"); the value was clamped to
 * +-65504 and attention over it is not within tolerance.  clear != 0 resets the bits. */
#define MUX_POOL_ERR_V_RANGE 1u
int mux_pool_error_flags(mux_pool_t pool, uint32_t* flags, int32_t clear);

/* ------------------------------------------------------------------------------------
 * Batch descriptor shared by append / prefill / decode.
 * Sequence b has n_b = qo_indptr[b+1]-qo_indptr[b] >= 1 new tokens (rows of Q/O and of
 * the new K/V) and kv_len[b] = L_b >= n_b keys after the append (L total,
 * r = L - n reused, n new).  Prefill: r_b = cached prefix.  Decode: n_b = 1 and
 * kv_len = c_b, the context INCLUDING the current token (R4).  New row i of
 * sequence b sits at position r_b + i and attends keys 0..r_b+i (R3).
 * The page table of b is page_ids[page_indptr[b] .. page_indptr[b+1]) and must hold
 * exactly ceil(L_b/16) pages.
 * Host copies (h_*) are optional; when given, the library validates lengths, page
 * counts, id ranges and (for append) shared-page writes on the host before launching.
 * ---------------------------------------------------------------------------------- */
typedef struct {
  int32_t num_seqs;
  const int32_t* qo_indptr;    /* device [num_seqs+1], qo_indptr[0] = 0 */
  const int32_t* kv_len;       /* device [num_seqs] */
  const int32_t* page_indptr;  /* device [num_seqs+1] */
  const int32_t* page_ids;     /* device [page_indptr[num_seqs]] */
  int32_t total_q;             /* qo_indptr[num_seqs] */
  int32_t max_q;               /* max_b n_b  (decode: 1) */
  int32_t max_kv;              /* max_b L_b */
  const int32_t* h_qo_indptr;  /* host copies, optional (NULL = skip host validation) */
  const int32_t* h_kv_len;
  const int32_t* h_page_indptr;
  const int32_t* h_page_ids;
} mux_batch;

/* a2: write the new tokens' K/V rows into their pool slots of `layer`: K as a bit-exact copy, V
 * converted to the pool's fp16 (R25; exact for bf16 values in [2^-14, 65504], larger magnitudes
 * clamp to +-65504 and set MUX_POOL_ERR_V_RANGE).
 * k_new, v_new: device bf16 [total_q][Hkv][d]; row qo_indptr[b]+i -> position L_b-n_b+i. */
int mux_append_kv(mux_pool_t pool, int32_t layer, const mux_batch* batch,
                  const void* k_new, const void* v_new, mux_stream_t stream);

/* a3: prefill causal attention with cached-prefix pages (tcgen05 + TMEM + TMA kernel).
 * q: device bf16 [total_q][Hq][d]; o: device [total_q][Hq][d] of o_dtype;
 * lse: device f32 [total_q][Hq] natural-log LSE, or NULL.  scale: softmax scale (1/sqrt(d)
 * in the paper's models; passed explicitly, R1).  GQA: q head h uses kv head
 * h / (Hq/Hkv) (R2).  Hq = num_q_heads. */
int mux_prefill_attn(mux_pool_t pool, int32_t layer, const mux_batch* batch, int32_t num_q_heads,
                     const void* q, void* o, int32_t o_dtype, float* lse, float scale,
                     mux_stream_t stream);

/* a4 + a5: decode split-KV paged attention followed (num_splits > 1) by the
 * log-sum-exp split combine.  q: device bf16 [num_seqs][Hq][d]; o, lse as prefill.
 * num_splits: 0 = auto (mux_decode_num_splits for this device's SM count).  Splits are
 * BALANCED: every split covers C = ceil(ceil(max_kv/16) / num_splits) pages of its sequence,
 * so a sequence of p pages uses ceil(p/C) splits (the longest uses num_splits) and every CTA
 * carries the same work; a ragged batch does not leave SMs idle behind its longest sequence.
 * ws: device workspace of >= mux_decode_workspace_bytes(num_seqs, Hq, d, num_splits)
 * bytes (may be NULL when the resolved num_splits is 1). */
int mux_decode_attn(mux_pool_t pool, int32_t layer, const mux_batch* batch, int32_t num_q_heads,
                    const void* q, void* o, int32_t o_dtype, float* lse, float scale,
                    int32_t num_splits, void* ws, size_t ws_bytes, mux_stream_t stream);
/* the same, with the launch sized for the num_sms SMs `stream` runs on (a partition; <= 0 = the
 * device): on partitions of <= 16 SMs (Hkv % 4 == 0, g <= 8) two CTAs of 4 kv heads share each SM
 * so one CTA's ring fill / drain overlaps the other's streaming; the split model (num_splits <= 0)
 * uses the same count.  mux_run_layer calls this with its sides' partition sizes. */
int mux_decode_attn_sms(mux_pool_t pool, int32_t layer, const mux_batch* batch, int32_t num_q_heads,
                        const void* q, void* o, int32_t o_dtype, float* lse, float scale, int32_t num_splits,
                        void* ws, size_t ws_bytes, mux_stream_t stream, int32_t num_sms);
size_t mux_decode_workspace_bytes(int32_t num_seqs, int32_t num_q_heads, int32_t head_dim,
                                  int32_t num_splits);
/* host split-count choice for the balanced split-KV: simulates the launch (every split covers
 * C = ceil(ceil(max_kv/16)/S) pages; CTAs of ~4 us start-up + ~100 GB/s streaming dispatched in
 * launch order onto `num_sms` SMs; + the combine pass when S > 1) for S in {1,2,3,4,6,...,64}
 * and returns the S of smallest predicted time.  kv_len: host array of the batch's contexts
 * (NULL = every sequence at max_kv).  Pure host function. */
int32_t mux_decode_num_splits(int32_t num_seqs, int32_t num_kv_heads, int32_t head_dim, const int32_t* kv_len,
                              int32_t max_kv, int32_t num_sms);

/* ------------------------------------------------------------------------------------
 * SM partitions (a6).  P:473: GreenContext binds streams to SM sets, reconfiguration
 * costs a stream synchronisation; 16-SM granularity.  For every requested
 * decode SM count k the library splits the device's SMs ONCE, disjointly, into
 * {k decode SMs, remainder prefill SMs} (cuDevSmResourceSplitByCount) and creates one
 * green context + one stream per side.  Split index -1 means "no partition": two plain
 * streams on the whole GPU.
 * ---------------------------------------------------------------------------------- */
/* rule of SPEC S:303-310 extended to any SM count: decode = k*granularity (k >= 1) while
 * total - decode >= min_side, ascending.  Writes up to cap values, returns the count
 * (108 SMs -> 6 configs, 132 -> 7; 148 -> 8) or -MUX_ERR_NO_CONFIG. */
int32_t mux_partition_configs(int32_t total_sms, int32_t granularity, int32_t min_side,
                              int32_t* out, int32_t cap);
/* N_PL = ceil(T_d * N_T / T_P), clamped to [1, remaining] (0 if remaining == 0). */
int32_t mux_num_prefill_layers(double t_decode, double t_prefill, int32_t n_layers_model,
                               int32_t remaining);

int mux_partition_create(mux_part_t* out, int32_t device, const int32_t* decode_sms, int32_t n_splits);
int mux_partition_destroy(mux_part_t part);
/* granted SM counts (exact, from the driver) and the two streams of split `idx` */
int mux_partition_query(mux_part_t part, int32_t idx, int32_t* dec_sms, int32_t* pf_sms,
                        mux_stream_t* dec_stream, mux_stream_t* pf_stream);
int32_t mux_partition_count(mux_part_t part);
/* device memory (bytes) taken by creating the partition's green contexts/streams */
int mux_partition_memory(mux_part_t part, int64_t* bytes);
int32_t mux_device_sm_count(int32_t device);

/* Per-layer host hook of a mux_run_layer side, called while the side's work is ENQUEUED
 * (host side, in layer order, after that layer's attention (+ out-projection) was enqueued on
 * `stream`).  Multi-GPU callers enqueue the layer's all-reduce of the out-projection partial
 * sums here on the side's own communicator, so the collective runs on the side's SMs
 * (SURVEY §8e).  side: 0 = decode, 1 = prefill. */
typedef void (*mux_layer_hook)(void* user, int32_t side, int32_t layer_index, mux_stream_t stream);

/* One side of a mux_run_layer call.  For layer i in [0, num_layers) the side processes
 * pool layer (layer0 + i) % pool_layers with inputs at base + i*stride (bytes; stride 0
 * = the same buffer every layer). */
typedef struct mux_ar_peers mux_ar_peers;   /* f4 fused all-reduce peers, defined below */
typedef struct {
  const mux_batch* batch;
  int32_t num_q_heads;
  const void* q;           /* bf16 [total_q][Hq][d] */
  const void* k_new;       /* bf16 [total_q][Hkv][d]; ignored when append == 0 */
  const void* v_new;
  void* o;                 /* [total_q][Hq][d] of o_dtype */
  float* lse;              /* [total_q][Hq] or NULL */
  int64_t q_stride, kv_stride, o_stride, lse_stride;
  int32_t o_dtype;
  float scale;
  int32_t layer0, num_layers;
  int32_t append;          /* 1: mux_append_kv before the attention of every layer */
  int32_t num_splits;      /* decode only; 0 = auto for the decode partition's SM count */
  void* ws;                /* decode only */
  size_t ws_bytes;
  /* a7 (optional, w_o == NULL: off): after each layer's attention, y = o . w_o with
   * o [total_q][Hq*d] bf16 (o_dtype must be bf16), w_o = [Hq*d][hidden] bf16 PACKED by
   * mux_outproj_pack_w (w_stride = packed bytes per layer, 0 = shared), y [total_q][hidden] */
  const void* w_o;
  void* y;
  int64_t w_stride, y_stride;
  int32_t hidden;
  int32_t y_dtype;
  mux_layer_hook hook;     /* optional */
  void* hook_user;
  /* Multi-GPU: after each layer's out-projection, y is all-reduced
   * in place (sum, bf16, count total_q * hidden) on the side's own stream by calling ar_fn, the
   * ncclAllReduce entry point of the NCCL library that created ar_comm (the caller dlsym's it:
   * ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
   * cudaStream_t)).  Enqueued from C inside the layer loop (no host callback); a non-zero NCCL
   * result returns MUX_ERR_CUDA.  NULL = no collective (single GPU).  Needs w_o. */
  void* ar_fn;
  void* ar_comm;
  /* optional timing of the dominant kernels: 2 * num_layers cudaEvent_t handles (created by the
   * caller with timing enabled), recorded on the side's stream right before and right after each
   * layer's attention launch(es) (decode: attention + split combine).  NULL = none. */
  void* const* attn_events;
  /* f4 full transformer layer (optional, single GPU; the paper's layer = attention + FFN):
   * w_qkv != NULL: each layer starts with mux_qkv_rope_append(x_in [total_q][hidden_in] bf16,
   * w_qkv packed, rope table) writing q (the side's q buffer) and the new K/V into the pool,
   * instead of mux_append_kv (k_new / v_new unused; append must be 0).
   * w13 != NULL: each layer ends with mux_ffn_swiglu(y -> ffn_y, scratch ffn_h, ffn_inter) on the
   * out-projection output (needs w_o; norms and residual adds are elementwise and not modelled).
   * Weights are shared by all layers. */
  const void* x_in;
  int32_t hidden_in;
  const void* w_qkv;
  const void* rope;
  int32_t rope_max_pos;
  const void* w13;
  const void* w2;
  void* ffn_h;
  void* ffn_y;
  int32_t ffn_inter;
  /* f4 fused communication (optional, instead of ar_fn): each layer's out-projection AND its
   * all-reduce run as ONE mux_outproj_allreduce kernel (declared below) with these peers; layer i
   * of the call uses every rank's y shifted by i * y_stride (the same buffer layout on every rank)
   * and epoch 0 (automatic) or, when ar_peers->epoch != 0, ar_peers->epoch + i (the caller then
   * advances its epoch by num_layers per call).  Needs
   * w_o, a bf16 y equal to ar_peers->y[ar_peers->rank] (layer 0), and ar_fn == NULL. */
  const mux_ar_peers* ar_peers;
} mux_side;

/* Host-only dry run of a side's collective schedule (no GPU needed): for each layer i the side
 * would process, in enqueue order, out[2*i] = pool layer (layer0 + i) % pool_layers and
 * out[2*i+1] = element count of the all-reduce run_side enqueues after it (total_q * hidden when
 * ar_fn is set, else 0).  NCCL needs every rank to issue the same collectives in the same order
 * on a communicator; multi-rank callers compare these plans across ranks (tests/test_dist_gloo.py).
 * *n = num_layers; at most cap entries written. */
int mux_side_plan(const mux_side* side, int32_t pool_layers, int64_t* out, int32_t cap, int32_t* n);

/* device timestamps (%globaltimer, ns) written by 1-thread stamp kernels on each side */
typedef struct {
  uint64_t dec_start_ns, dec_end_ns, pf_start_ns, pf_end_ns;
} mux_side_times;

/* a6: co-execute decode (a2+a4+a5 per layer, enqueued FIRST) on the decode SM set
 * and prefill (a2+a3 per layer, layer-wise P:529) on the prefill SM set of split
 * `split_idx`.  Either side may be NULL (that side does not run: isolated mode, so iso and
 * mux timings come from the same call).  Ordering: both side streams wait for the work
 * already enqueued on join_stream; join_stream then waits for both sides.  times: device
 * buffer (or NULL) filled asynchronously; read it after synchronising join_stream. */
int mux_run_layer(mux_part_t part, int32_t split_idx, mux_pool_t pool,
                  const mux_side* prefill, const mux_side* decode,
                  mux_side_times* times, mux_stream_t join_stream);

/* a7 building block (multi-GPU out-projection partial sums, P:702 TP): Y[T][N] (bf16 or
 * f32) = X[T][K] (bf16, row-major) . W[K][N], fp32 accumulation.
 *
 * W is a weight: it is passed PACKED, once re-laid out by mux_outproj_pack_w into tiles of
 * 128 columns x 64 rows (16 KiB each, in the 128-byte-swizzled image the tensor cores read),
 * tile (nt, kb) at byte offset (nt * ceil(K/64) + kb) * 16384, zero-padded past K and N, so
 * every stage of the GEMM is one contiguous 16 KiB bulk copy.
 * Requirements: K and N multiples of 8; x, w_packed, y 16-byte aligned.  Deterministic
 * (no atomics).  Errors: MUX_ERR_INVALID_ARG / MUX_ERR_UNSUPPORTED / MUX_ERR_CUDA. */
int mux_outproj(const void* x, const void* w_packed, void* y, int32_t y_dtype, int32_t T, int32_t K,
                int32_t N, mux_stream_t stream);
/* the same GEMM sized for num_sms SMs (the partition `stream` runs on; <= 0 = the whole
 * device): also the TC(k_p) dense-GEMM denominator of SURVEY §8(d) on a green context */
int mux_outproj_sms(const void* x, const void* w_packed, void* y, int32_t y_dtype, int32_t T, int32_t K,
                    int32_t N, mux_stream_t stream, int32_t num_sms);

/* ------------------------------------------------------------------------------------
 * f4 (fused communication): the out-projection GEMM and the all-reduce of
 * its partial sums in ONE kernel over peer memory.  PAPER: Llama-70B runs with tensor
 * parallelism of degree 8 over NVLink; per layer the G KV-head shards'
 * partials O_g . W_o,g are summed (R23).  Replaces a7's mux_outproj + NCCL all-reduce.
 *
 * Rank r computes Y_r = X_r . W_r (X [T][K] bf16 row-major, W PACKED by mux_outproj_pack_w,
 * fp32 accumulation; 256 x 256 tiles on CTA pairs).  Tile t is owned by rank t mod G: the
 * epilogue stores each partial tile as bf16 (the wire type of R23) into the OWNER's staging
 * slot and raises a counter there (release, system scope); each rank sums the G partials of its
 * tiles in rank order 0..G-1 in fp32 (identical bits on every rank, run to run), rounds to bf16
 * and stores the tile into EVERY rank's Y [T][N] bf16 (all-gather), counting completions on each
 * rank; the kernel returns once this rank's Y is complete.  Traffic per rank equals a ring
 * all-reduce's (2 (G-1)/G of Y), but it leaves the GPU tile by tile during the GEMM.
 *
 * peers: world G (1..MUX_AR_MAX_WORLD), this rank, epoch (0 = automatic: the kernel keeps a launch
 * counter in the rank's own workspace, so repeated calls and CUDA-graph replays need nothing from
 * the host; else an explicit counter shared by all ranks, 1 on the first call with a workspace, +1
 * per call; the two modes must not be mixed on one workspace; counters are never reset) and, per rank r,
 * its staging workspace (mux_outproj_ar_ws_bytes(T, N, G) bytes, zero-filled ONCE before the
 * first call; a workspace serves one (T, N, G): its counters sit behind T x N-sized slots) and its Y,
 * as addresses valid in THIS process (peers' allocations mapped by CUDA
 * IPC or VMM; rank == r: local).  Every rank calls with the same T, K, N, world and epoch.
 * num_sms: SMs the launch may use (<= 0: the device); one CTA per SM, so all of a rank's CTAs are
 * resident and the cross-rank waits cannot deadlock; a rank that never arrives (crashed peer,
 * mismatched calls) makes the waiting kernels trap after 20 s instead of hanging the GPU (the
 * launch then fails with a CUDA error).  Any T >= 1 (a decode side's few rows run in
 * one 256-row tile; rows past T are zero-filled and never stored).  Requirements: K and N multiples
 * of 8, 16-byte aligned buffers.  Errors: MUX_ERR_INVALID_ARG / MUX_ERR_UNSUPPORTED / MUX_ERR_CUDA. */
#define MUX_AR_MAX_WORLD 8
#define MUX_IPC_HANDLE_BYTES 64
/* peer buffers for it: device memory another process can map through CUDA IPC.  mux_ipc_alloc:
 * cudaMalloc'd, zero-filled, its 64-byte handle written to `handle` (exchange it with the other
 * ranks, e.g. torch.distributed.all_gather_object); mux_ipc_open maps another process's handle
 * (not this process's own: use the local pointer for your rank); mux_ipc_close / mux_ipc_free undo them. */
int mux_ipc_alloc(size_t bytes, void** ptr, void* handle);
int mux_ipc_open(const void* handle, void** ptr);
int mux_ipc_close(void* ptr);
int mux_ipc_free(void* ptr);
struct mux_ar_peers {
  int32_t world;
  int32_t rank;
  uint32_t epoch;
  void* stage[MUX_AR_MAX_WORLD];
  void* y[MUX_AR_MAX_WORLD];
};
size_t mux_outproj_ar_ws_bytes(int32_t T, int32_t N, int32_t world);
int mux_outproj_allreduce(const void* x, const void* w_packed, int32_t T, int32_t K, int32_t N,
                          const mux_ar_peers* peers, int32_t num_sms, mux_stream_t stream);
/* the same kernel with ALL `world` ranks' CTAs in ONE launch on this device (x[r], w_packed[r]
 * per rank; every peers->stage / y local; peers->rank ignored): the G-rank protocol with fewer
 * GPUs than ranks (the ranks' CTAs wait on one another, so they must share one launch, at most
 * one CTA per SM; cooperative when the driver accepts it with clusters). */
int mux_outproj_allreduce_emulated(const void* const* x, const void* const* w_packed, int32_t T, int32_t K,
                                   int32_t N, const mux_ar_peers* peers, mux_stream_t stream);

/* ------------------------------------------------------------------------------------
 * f4 (first part): QKV projection + RoPE + KV append, ONE kernel.
 * PAPER: each transformer layer = attention + FFN; the attention layer's projections
 * are Table 2's n d^2 terms; "attention ... generates the keys and values of new
 * tokens ... stored in a KV cache".  Llama-3 models (P:245 cites Llama 3; the
 * evaluation serves Llama-3-8B / 70B) rotate q and k with RoPE (R26).
 *
 * Y = X . W_qkv, X [total_q][hidden] bf16 row-major (row = new token, in batch order),
 * W_qkv = [hidden][(Hq + 2 Hkv) * 128] bf16 PACKED by mux_outproj_pack_w, columns = Hq query
 * heads, then Hkv key heads, then Hkv value heads (128 each), fp32 accumulation (tcgen05, CTA
 * pairs).  For the token at position p = L_b - n_b + i of sequence b (as mux_append_kv):
 *   query heads: RoPE(p), stored bf16 to q_out [total_q][Hq][128];
 *   key heads:   RoPE(p), stored bf16 into the token's slot of `layer` in the pool;
 *   value heads: stored fp16 (R25) into the slot (|v| > 65504 clamps, MUX_POOL_ERR_V_RANGE).
 * RoPE (R26, rotate-half): (y_c, y_{c+64}) -> (y_c cos a - y_{c+64} sin a, y_{c+64} cos a + y_c sin a),
 * a = p * theta^(-2c/128), c < 64, with (cos a, sin a) read from `rope`, a device table
 * [rope_max_pos][64] float2 made by mux_rope_table (double precision, rounded to fp32 once).
 * Requirements: head_dim 128, Hq and Hkv even, Hq % Hkv == 0, hidden % 8 == 0, 16-byte aligned
 * pointers, every position < rope_max_pos (checked on the host when the batch has host copies;
 * on the device a position past the table skips the rotation and sets error bit 2).
 * Replaces mux_append_kv for the batch's rows (same page-sharing checks). */
size_t mux_rope_table_bytes(int32_t max_pos, int32_t head_dim);
int mux_rope_table(void* table, int32_t max_pos, int32_t head_dim, double theta, mux_stream_t stream);
int mux_qkv_rope_append(mux_pool_t pool, int32_t layer, const mux_batch* batch, int32_t num_q_heads,
                        const void* x, int32_t hidden, const void* w_qkv_packed, const void* rope,
                        int32_t rope_max_pos, void* q_out, mux_stream_t stream);

/* f4 (second part): the layer's FFN, Llama SwiGLU ("each transformer layer contains an
 * attention layer and a feed-forward network (FFN) layer"; Table 2's FFN column, O(n d^2), P:588-590;
 * DESIGN.md R27):  H = silu(X . W1) * (X . W3),  Y = H . W2,  silu(g) = g / (1 + e^-g).
 * X [T][hidden] bf16, W1 / W3 [hidden][inter] bf16, W2 [inter][hidden] bf16 (packed by
 * mux_outproj_pack_w), H [T][inter] bf16 (caller's scratch: the activation between the two GEMMs),
 * Y [T][hidden] bf16.  The gate and up projections are ONE CTA-pair GEMM over W13 = W1 and W3
 * interleaved in 128-column blocks (mux_ffn_pack_w13, weight prep) whose epilogue forms
 * silu(gate) * up; the down projection is mux_outproj.  fp32 accumulation; inter % 128 == 0,
 * hidden % 8 == 0, 16-byte aligned pointers. */
size_t mux_ffn_w13_packed_bytes(int32_t hidden, int32_t inter);
int mux_ffn_pack_w13(const void* w1, const void* w3, void* w13_packed, int32_t hidden, int32_t inter,
                     mux_stream_t stream);
int mux_ffn_swiglu(const void* x, const void* w13_packed, const void* w2_packed, void* h, void* y, int32_t T,
                   int32_t hidden, int32_t inter, mux_stream_t stream);

/* bytes of the packed layout of a [K][N] weight: ceil(N/128) * ceil(K/64) * 16384 */
size_t mux_outproj_packed_bytes(int32_t K, int32_t N);

/* pack W [K][N] bf16 row-major (device) into w_packed (device, mux_outproj_packed_bytes),
 * asynchronously on `stream`; bit-exact re-layout (plus zero padding). */
int mux_outproj_pack_w(const void* w, void* w_packed, int32_t K, int32_t N, mux_stream_t stream);

/* ------------------------------------------------------------------------------------
 * f1: bubble-less multiplex ENGINE above mux_run_layer.
 * PAPER: layer-wise prefill ("splits the prefill phase into layers (PLs) ... can
 * launch enough PBs to occupy compute resources for prefill, and return in time before the
 * decode phase finishes"), decode-first launching, query-based synchronisation
 * ("periodically polls CUDA events ... the corresponding prefill request is
 * immediately merged into the current decode batch"), decode-termination hand-off of the
 * later prefill layers to the freed SMs, best-fit decode SMs from worst-case
 * estimates and N_PL = ceil(T_d * N_T / T_P).
 *
 * One host thread drives both sides.  A decode ITERATION = all N_T layers of the current
 * decode batch (append of the new token + attention + out-projection per layer); it is
 * launched when the previous one has completed (its tokens must return to the host before
 * the next iteration), after retiring finished requests and merging completed
 * prefills.  A prefill GROUP = N_PL consecutive layers of the active prefill batch; the engine
 * keeps up to two groups queued on the prefill stream so the prefill SMs never drain.  When
 * the decode batch is empty the remaining prefill layers go to the whole GPU.
 * Activations are synthetic: token t of request j uses row (src_base_j + t) % src_rows of
 * src_q / src_k / src_v (the QKV projections are outside this hot path).
 * ---------------------------------------------------------------------------------- */
typedef struct mux_engine* mux_engine_t;

typedef struct {
  int32_t num_q_heads;          /* Hq; Hkv, d and N_T (= pool num_layers) come from the pool */
  float scale;
  const void* src_q;            /* device bf16 [src_rows][Hq][d] */
  const void* src_k;            /* device bf16 [src_rows][Hkv][d] */
  const void* src_v;
  int32_t src_rows;
  const void* w_o;              /* packed W_o (mux_outproj_pack_w), NULL = no out-projection */
  int32_t hidden;
  int32_t max_decode_seqs;      /* decode batch capacity */
  int32_t max_prefill_tokens;   /* cap on sum n of one prefill batch (>= the longest prompt) */
  int32_t fixed_split;          /* >= -1: always this split (-1 = whole GPU, time-sliced sides);
                                   -2: best-fit by the cost model below */
  int32_t n_cost;               /* entries of the cost arrays (= partition split count) */
  const double* dec_theta;      /* [n_cost][3] Eq.2 per split, us per layer (NULL: no model) */
  const double* pf_theta;       /* [n_cost][4] Eq.1 per split, us per layer */
  const double* dec_slowdown;   /* [n_cost] contention guard max slowdown, NULL = 1 */
  double tbt_slo_us;            /* decode iteration target for the best-fit rule */
  int32_t fixed_pl;             /* > 0: layers per prefill group instead of N_PL */
  int32_t handoff;              /* 1: decode termination hands the prefill to the whole GPU */
  int32_t keep_pages;           /* 1: finished requests keep their pages (for inspection) */
  int32_t serialize;            /* 1: temporal multiplexing baseline: both sides on ONE whole-GPU
                                   stream (no overlap); fixed_split must be -1 */
  /* f2 launch-gap removal ("each decode iteration as a CUDA graph"): 1 = every decode
   * iteration (gathers + N_T x (append, attention, combine, out-projection)) is ONE graph launch,
   * captured lazily per (split, batch size, split-KV count, pages per split) and replayed; the
   * iteration's batch arrays are copied into a fixed device buffer right before the launch. */
  int32_t use_graphs;
  /* Output log (optional, for checking the engine's results): after every decode iteration and
   * after the last layer group of every prefill batch, the LAST layer's attention output rows
   * (o_f32 ? f32 : bf16, [rows][Hq][d]) are appended to o_log and, with w_o, the out-projection
   * rows (bf16 [rows][hidden]) to y_log, until log_rows rows are used (device buffers, owned by
   * the caller).  mux_engine_out_rows() says which (request, position) each row holds. */
  void* o_log;
  void* y_log;
  int32_t log_rows;
  int32_t o_f32;                /* 1: attention outputs in f32 (needs w_o == NULL); 0: bf16 */
  /* f2 run-ahead: 1 = the next decode iteration is enqueued while the current one runs (two in
   * flight; its batch = the current one's minus requests whose last token is already enqueued,
   * plus merged prefills), so the decode SMs see no host turn-around gap between iterations.
   * Valid when the next iteration's inputs are produced on the device (on-device sampling; here
   * synthetic rows).  0 = launch after completion (the token returns to the host first). */
  int32_t overlap;
} mux_engine_desc;

typedef struct {
  int32_t id;
  int32_t cached;               /* r: prefix tokens already in the pool (preloaded at admission) */
  int32_t prompt;               /* n >= 1: new prompt tokens (prefill) */
  int32_t gen;                  /* decode iterations after the prefill (>= 0) */
  int32_t src_base;
  /* arrival (online serving): the request joins the FCFS queue once the engine has COMPLETED
   * arrival_iter decode iterations AND arrival_us microseconds (host clock) have passed since
   * mux_engine_run started; 0 / 0 = at the start.  A request whose arrival_iter cannot be reached
   * (no decode work left) is admitted when the engine would otherwise idle. */
  int32_t arrival_iter;
  double arrival_us;
} mux_request;

typedef struct {
  double makespan_us;           /* first to last engine kernel, device clock */
  int64_t prefill_tokens, decode_tokens;
  int32_t decode_iters, prefill_groups, split_changes, handoffs;
  double busy_dec_us, busy_pf_us;
  double bubble_ratio;          /* R21: idle share of each side's [first, last] window, averaged */
  double bubble_ratio_dec, bubble_ratio_pf;
  double tbt_mean_us, tbt_max_us; /* decode iteration end-to-end intervals */
  double ttft_mean_us, ttft_max_us;   /* prefill completion - arrival, device clock */
  /* launch gap (f2): device idle time of the decode side between consecutive decode iterations
   * (start of iteration i+1 - end of iteration i, %globaltimer), i.e. the host's turn-around */
  double gap_mean_us, gap_max_us;
  int32_t graphs;               /* CUDA graphs captured (use_graphs) */
  int64_t graph_bytes;          /* device memory taken by instantiating them (cudaMemGetInfo delta) */
  int32_t logged_rows;          /* rows written to o_log / y_log */
} mux_engine_stats;

int mux_engine_create(mux_engine_t* out, mux_part_t part, mux_pool_t pool, const mux_engine_desc* desc);
/* queue requests (FCFS in arrival order, submission order among equal arrivals) */
int mux_engine_submit(mux_engine_t eng, const mux_request* reqs, int32_t n);
/* run until every submitted request has finished its decode; blocks the calling thread */
int mux_engine_run(mux_engine_t eng, mux_engine_stats* stats);
/* a finished request's final context length and page table (needs keep_pages) */
int mux_engine_request_pages(mux_engine_t eng, int32_t id, int32_t* kv_len, int32_t* page_ids, int32_t cap,
                             int32_t* n_pages);
/* per-iteration trace: for decode iteration i, out[i] = {split, batch size, start, end (ns)} */
int mux_engine_trace(mux_engine_t eng, int64_t* out, int32_t cap, int32_t* n);
/* the output log's rows (after mux_engine_run): out[3*i] = request id, out[3*i+1] = absolute
 * position p of the query token (it attended keys 0..p of the request), out[3*i+2] = 0 for a
 * prefill row, 1 for a decode row; row i of o_log / y_log.  *n = rows logged. */
int mux_engine_out_rows(mux_engine_t eng, int32_t* out, int32_t cap, int32_t* n);
int mux_engine_destroy(mux_engine_t eng);

/* ------------------------------------------------------------------------------------
 * Read-bandwidth probe: the partition-level denominator of the decode roofline (SURVEY
 * §8(d) "BW_read(k_d): a read-only streaming kernel measured in the same green context";
 * decode is memory-intensive).  Streams floor(bytes / 32 KiB) chunks of `src`
 * (device, 16-byte aligned, read only) into shared memory with 32 KiB bulk copies through a
 * 6-stage ring per CTA, the access pattern and op size of the decode kernel's page stream,
 * and does nothing else with the data.  Grid: `num_ctas` CTAs (one per SM of the partition
 * the stream belongs to), chunk c read by CTA c mod num_ctas.  Asynchronous on `stream`;
 * time it with events on that stream.  Errors: MUX_ERR_INVALID_ARG (null src, < 1 chunk,
 * num_ctas < 1), MUX_ERR_CUDA. */
int mux_stream_read(const void* src, size_t bytes, int32_t num_ctas, mux_stream_t stream);

const char* mux_last_error(void);
/* library version string, e.g. "mux-b200 0.1 sm_100a" */
const char* mux_version(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* MUX_H_ */
