// f1: bubble-less multiplex engine above mux_run_layer's building blocks (include/mux.h).
//
// PAPER: P:529-531 layer-wise prefill ("PLs": launch enough prefill layers to keep the
// prefill SMs busy and return before the decode iteration finishes; switch the later
// prefill layers to the freed SMs when the decode batch terminates), P:535-537 query-based
// synchronisation (poll CUDA events; merge a finished prefill into the decode batch at once),
// P:498 decode launched first, P:657 best-fit decode SMs from worst-case estimates
// (solo prediction x the contention guard's max slowdown)
// N_PL = ceil(T_d N_T / T_P).
//
// B200 design: one host thread, no locks.  The device work of a decode iteration / prefill
// group is exactly what mux_run_layer enqueues for one side (mux::run_side: append + attention
// (+ combine) + out-projection per layer), on the green-context streams of the current split.
// Batches are rebuilt on the host (page tables grow by one page every 16 decode tokens),
// staged in pinned memory and copied with the iteration on its own stream; activations are
// gathered from the caller's synthetic source rows by a copy kernel.  Every iteration and
// group is bracketed by %globaltimer stamps in a device log, from which the run's bubble
// ratio, TBT, TTFT and the decode side's inter-iteration launch gap are computed after the run
// (no profiler).  f2 launch-gap removal: with use_graphs every decode iteration is
// ONE CUDA graph launch (captured lazily per (split, batch size, split-KV count, pages per split),
// replayed with the batch arrays copied into a fixed device buffer first).  Requests arrive over
// time (arrival_iter / arrival_us): prefills then merge into a RUNNING decode batch.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <deque>
#include <map>
#include <thread>
#include <tuple>
#include <vector>

#include "pool.h"

namespace mux {
namespace {

__global__ void gather_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                   const int32_t* __restrict__ idx, int rows, int vec_per_row) {
  const size_t n = static_cast<size_t>(rows) * vec_per_row;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t r = i / vec_per_row, c = i % vec_per_row;
    dst[i] = src[static_cast<size_t>(__ldg(idx + r)) * vec_per_row + c];
  }
}

// %globaltimer into log[*idx + off]: a captured decode iteration writes its stamps to the log
// slot the host stored in device memory before the replay (a graph's parameters are fixed)
__global__ void stamp_at_kernel(unsigned long long* log, const int32_t* idx, int off) {
  log[*idx + off] = dev::globaltimer();
}

int gather(const void* src, void* dst, const int32_t* idx, int rows, int row_bytes, cudaStream_t st) {
  if (rows <= 0) return MUX_OK;
  const int vec = row_bytes / 16;
  const int blocks = static_cast<int>(std::min<size_t>((static_cast<size_t>(rows) * vec + 255) / 256, 1184));
  gather_rows_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), idx, rows,
                                            vec);
  MUX_CUDA(cudaGetLastError());
  return MUX_OK;
}

struct Req {
  mux_request r{};
  std::vector<int32_t> pages;
  int ctx = 0;          // tokens in the pool (kv_len after the last append)
  int gen_launched = 0;  // decode iterations enqueued for it
  int gen_done = 0;      // ... and completed
  int ttft_log = -1;    // log slot of the end stamp of its last prefill group
  int arrive_log = -1;  // log slot of the end stamp of the decode iteration that met arrival_iter
  bool arrived = false;
  bool finished = false;
};

// one staging slot of a side: pinned host arrays + their device copy
struct Slot {
  int32_t* h = nullptr;
  int32_t* d = nullptr;
  size_t cap = 0;       // int32 entries
  cudaEvent_t done = nullptr;
  bool used = false;
};

struct Group {
  cudaEvent_t ev;
  bool last;
  std::vector<int> reqs;
};

struct Interval {
  int side;             // 0 decode, 1 prefill
  int log;              // index of the start stamp; end = log + 1
  int split, batch;
};

double eq2(const double* th, double sum_r, int bs) { return th[0] * sum_r + th[1] * bs + th[2]; }
double eq1(const double* th, double sum_n2, double sum_nr, double sum_n) {
  return th[0] * sum_n2 + th[1] * sum_nr + th[2] * sum_n + th[3];
}

}  // namespace
}  // namespace mux

struct mux_engine {
  mux_part_t part = nullptr;
  mux_pool_t pool = nullptr;
  mux_engine_desc desc{};
  std::vector<double> dec_theta, pf_theta, slowdown;
  std::vector<mux::Req> reqs;
  int Hkv = 0, d = 0, NT = 0;
  size_t osz = 2;                      // bytes per attention output element (bf16 / f32)
  // device buffers
  void *dq = nullptr, *dk = nullptr, *dv = nullptr, *do_ = nullptr, *dy = nullptr, *ws = nullptr;
  // f2 graphs: the iteration's batch arrays at a FIXED address, [0] = the log slot of its start
  // stamp (the end stamp goes to the next slot), then the build_batch layout
  int32_t* dfix = nullptr;
  size_t ws_bytes = 0;
  // f2: decode-iteration graphs keyed by (split, batch size, split-KV count, pages per split)
  std::map<std::tuple<int, int, int, int>, cudaGraphExec_t> graphs;
  int64_t graph_bytes = 0;
  std::vector<int32_t> out_rows;       // [row][3] = request id, position, decode?
  int log_rows_used = 0;
  void *pq[2] = {}, *pk[2] = {}, *pv[2] = {}, *po[2] = {}, *py[2] = {};
  void *prek = nullptr, *prev = nullptr;
  int cap_dec = 0, cap_pf = 0, cap_pre = 0;
  mux::Slot dslot[2], pslot[2], preslot[2];
  unsigned long long* log = nullptr;
  int log_cap = 0, log_n = 0;
  std::vector<mux::Interval> iv;
  std::vector<cudaEvent_t> events;
  bool ran = false;
};

using namespace mux;

namespace {

int slot_reserve(Slot& s, size_t n) {
  if (s.cap >= n) return MUX_OK;
  if (s.h) cudaFreeHost(s.h);
  if (s.d) cudaFree(s.d);
  s.h = nullptr;
  s.d = nullptr;
  MUX_CUDA(cudaMallocHost(&s.h, n * 4));
  MUX_CUDA(cudaMalloc(&s.d, n * 4));
  if (!s.done) MUX_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
  s.cap = n;
  return MUX_OK;
}

// the staging buffer may be rewritten only after the copy that read it has run
int slot_acquire(Slot& s) {
  if (s.used) MUX_CUDA(cudaEventSynchronize(s.done));
  s.used = false;
  return MUX_OK;
}

int new_event(mux_engine* e, cudaEvent_t* ev) {
  MUX_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
  e->events.push_back(*ev);
  return MUX_OK;
}

int event_done(cudaEvent_t ev, bool* done) {
  const cudaError_t q = cudaEventQuery(ev);
  *done = q == cudaSuccess;
  if (q == cudaSuccess || q == cudaErrorNotReady) {
    if (q == cudaErrorNotReady) cudaGetLastError();   // not an error: clear it
    return MUX_OK;
  }
  return cuda_fail(q, "engine: cudaEventQuery (a kernel of the run failed)");
}

int log_pair(mux_engine* e, int* idx) {
  if (e->log_n + 2 > e->log_cap) return fail(MUX_ERR_INVALID_ARG, "engine log full");
  *idx = e->log_n;
  e->log_n += 2;
  return MUX_OK;
}

}  // namespace

extern "C" {

int mux_engine_create(mux_engine_t* out, mux_part_t part, mux_pool_t pool, const mux_engine_desc* desc) {
  if (!out || !part || !pool || !desc) return fail(MUX_ERR_INVALID_ARG, "mux_engine_create: NULL argument");
  *out = nullptr;
  const int Hkv = pool->desc.num_kv_heads, d = pool->desc.head_dim;
  if (desc->num_q_heads < Hkv || desc->num_q_heads % Hkv) return fail(MUX_ERR_UNSUPPORTED, "Hq must be a multiple of Hkv");
  if (!desc->src_q || !desc->src_k || !desc->src_v || desc->src_rows < 1)
    return fail(MUX_ERR_INVALID_ARG, "engine needs src_q/src_k/src_v rows");
  if (desc->max_decode_seqs < 1 || desc->max_prefill_tokens < 1) return fail(MUX_ERR_INVALID_ARG, "engine capacities");
  if (desc->w_o && desc->hidden < 8) return fail(MUX_ERR_INVALID_ARG, "hidden < 8 with w_o");
  const int nsplit = mux_partition_count(part);
  if (desc->fixed_split < -2 || desc->fixed_split >= nsplit) return fail(MUX_ERR_INVALID_ARG, "fixed_split out of range");
  const bool model = desc->dec_theta && desc->pf_theta;
  if (desc->serialize && desc->fixed_split != -1) return fail(MUX_ERR_INVALID_ARG, "serialize needs fixed_split = -1");
  if (desc->fixed_split == -2 && (!model || desc->n_cost != nsplit))
    return fail(MUX_ERR_INVALID_ARG, "best-fit split needs a cost model with one entry per split");
  if (desc->o_f32 && desc->w_o) return fail(MUX_ERR_INVALID_ARG, "o_f32 needs w_o == NULL (the out-projection reads bf16 O)");
  if (desc->log_rows < 0 || (desc->log_rows > 0 && !desc->o_log) || (desc->log_rows > 0 && desc->w_o && !desc->y_log))
    return fail(MUX_ERR_INVALID_ARG, "output log: o_log (and y_log with w_o) needed for log_rows > 0");
  auto* e = new mux_engine();
  e->part = part;
  e->pool = pool;
  e->desc = *desc;
  e->Hkv = Hkv;
  e->d = d;
  e->NT = pool->desc.num_layers;
  e->osz = desc->o_f32 ? 4 : 2;
  if (model) {
    e->dec_theta.assign(desc->dec_theta, desc->dec_theta + 3 * desc->n_cost);
    e->pf_theta.assign(desc->pf_theta, desc->pf_theta + 4 * desc->n_cost);
    e->slowdown.assign(desc->n_cost, 1.0);
    if (desc->dec_slowdown) e->slowdown.assign(desc->dec_slowdown, desc->dec_slowdown + desc->n_cost);
  }
  e->desc.dec_theta = e->desc.pf_theta = e->desc.dec_slowdown = nullptr;
  *out = e;
  return MUX_OK;
}

int mux_engine_submit(mux_engine_t e, const mux_request* rq, int32_t n) {
  if (!e || n < 0 || (n > 0 && !rq)) return fail(MUX_ERR_INVALID_ARG, "mux_engine_submit: bad argument");
  for (int i = 0; i < n; ++i) {
    if (rq[i].prompt < 1 || rq[i].cached < 0 || rq[i].gen < 0)
      return fail(MUX_ERR_INVALID_ARG, "request needs prompt >= 1, cached >= 0, gen >= 0");
    if (rq[i].prompt > e->desc.max_prefill_tokens) return fail(MUX_ERR_INVALID_ARG, "prompt > max_prefill_tokens");
    if (rq[i].arrival_iter < 0 || !(rq[i].arrival_us >= 0.0)) return fail(MUX_ERR_INVALID_ARG, "arrival must be >= 0");
    Req r;
    r.r = rq[i];
    e->reqs.push_back(r);
  }
  return MUX_OK;
}

static int engine_alloc(mux_engine* e) {
  const int Hq = e->desc.num_q_heads, d = e->d, Hkv = e->Hkv;
  int64_t tot_pages = 0, max_pre = 0, iters = 0;
  for (auto& r : e->reqs) {
    tot_pages += (r.r.cached + r.r.prompt + r.r.gen + kPage - 1) / kPage;
    max_pre += r.r.cached;
    iters += r.r.gen;
  }
  e->cap_dec = e->desc.max_decode_seqs;
  e->cap_pf = e->desc.max_prefill_tokens;
  e->cap_pre = static_cast<int>(std::max<int64_t>(1, max_pre));
  const size_t qrow = static_cast<size_t>(Hq) * d * 2, kvrow = static_cast<size_t>(Hkv) * d * 2;
  MUX_CUDA(cudaMalloc(&e->dq, e->cap_dec * qrow));
  MUX_CUDA(cudaMalloc(&e->dk, e->cap_dec * kvrow));
  MUX_CUDA(cudaMalloc(&e->dv, e->cap_dec * kvrow));
  const size_t orow = static_cast<size_t>(Hq) * d * e->osz;
  MUX_CUDA(cudaMalloc(&e->do_, e->cap_dec * orow));
  if (e->desc.w_o) MUX_CUDA(cudaMalloc(&e->dy, static_cast<size_t>(e->cap_dec) * e->desc.hidden * 2));
  e->ws_bytes = mux_decode_workspace_bytes(e->cap_dec, Hq, d, 64);
  MUX_CUDA(cudaMalloc(&e->ws, std::max<size_t>(e->ws_bytes, 256)));
  for (int i = 0; i < 2; ++i) {
    MUX_CUDA(cudaMalloc(&e->pq[i], e->cap_pf * qrow));
    MUX_CUDA(cudaMalloc(&e->pk[i], e->cap_pf * kvrow));
    MUX_CUDA(cudaMalloc(&e->pv[i], e->cap_pf * kvrow));
    MUX_CUDA(cudaMalloc(&e->po[i], e->cap_pf * orow));
    if (e->desc.w_o) MUX_CUDA(cudaMalloc(&e->py[i], static_cast<size_t>(e->cap_pf) * e->desc.hidden * 2));
  }
  MUX_CUDA(cudaMalloc(&e->prek, e->cap_pre * kvrow));
  MUX_CUDA(cudaMalloc(&e->prev, e->cap_pre * kvrow));
  const size_t nreq = e->reqs.size();
  for (int i = 0; i < 2; ++i) {
    int rc = slot_reserve(e->dslot[i], 4 * static_cast<size_t>(e->cap_dec) + 9 + tot_pages);
    if (!rc) rc = slot_reserve(e->pslot[i], 4 * nreq + 8 + tot_pages + e->cap_pf);
    if (!rc) rc = slot_reserve(e->preslot[i], 4 * nreq + 8 + tot_pages + e->cap_pre);
    if (rc) return rc;
  }
  if (e->desc.use_graphs) MUX_CUDA(cudaMalloc(&e->dfix, (4 * static_cast<size_t>(e->cap_dec) + 9 + tot_pages) * 4));
  e->log_cap = static_cast<int>(2 * (iters + static_cast<int64_t>(e->NT) * nreq + 64));
  MUX_CUDA(cudaMalloc(&e->log, static_cast<size_t>(e->log_cap) * 8));
  return pool_tmaps(e->pool);   // device-side pool state exists before any graph capture
}

// host arrays of a batch in a slot: [qo (B+1)][kv (B)][pind (B+1)][idx rows][page ids]
struct Built {
  mux_batch b{};
  int32_t* d_idx = nullptr;
  int rows = 0;
  size_t n = 0;
};

static Built build_batch(Slot& s, const std::vector<Req*>& rs, const std::vector<int>& n_new,
                         const std::vector<int>& kv, const std::vector<int>& pos0, int src_rows,
                         int32_t* dev = nullptr /* device copy of the arrays: default the slot's */) {
  if (!dev) dev = s.d;
  Built out;
  const int B = static_cast<int>(rs.size());
  int32_t* qo = s.h;
  int32_t* kl = qo + B + 1;
  int32_t* pi = kl + B;
  int32_t* idx = pi + B + 1;
  int rows = 0;
  for (int i = 0; i < B; ++i) rows += n_new[i];
  int32_t* pids = idx + rows;
  qo[0] = 0;
  pi[0] = 0;
  int max_q = 0, max_kv = 0, r = 0, pg = 0;
  for (int i = 0; i < B; ++i) {
    qo[i + 1] = qo[i] + n_new[i];
    kl[i] = kv[i];
    const int np = (kv[i] + kPage - 1) / kPage;
    for (int p = 0; p < np; ++p) pids[pg++] = rs[i]->pages[p];
    pi[i + 1] = pg;
    for (int t = 0; t < n_new[i]; ++t) idx[r++] = static_cast<int32_t>((static_cast<int64_t>(rs[i]->r.src_base) + pos0[i] + t) % src_rows);
    max_q = std::max(max_q, n_new[i]);
    max_kv = std::max(max_kv, kv[i]);
  }
  out.n = static_cast<size_t>(pids + pg - s.h);
  mux_batch& b = out.b;
  b.num_seqs = B;
  b.qo_indptr = dev;
  b.kv_len = dev + B + 1;
  b.page_indptr = dev + 2 * B + 1;
  b.page_ids = dev + 3 * B + 2 + rows;
  b.total_q = rows;
  b.max_q = max_q;
  b.max_kv = max_kv;
  b.h_qo_indptr = qo;
  b.h_kv_len = kl;
  b.h_page_indptr = pi;
  b.h_page_ids = pids;
  out.d_idx = dev + 3 * B + 2;
  out.rows = rows;
  return out;
}

int mux_engine_run(mux_engine_t e, mux_engine_stats* st) {
  if (!e) return fail(MUX_ERR_INVALID_ARG, "engine NULL");
  if (e->ran) return fail(MUX_ERR_INVALID_ARG, "mux_engine_run may be called once per engine");
  e->ran = true;
  int rc = engine_alloc(e);
  if (rc) return rc;
  const mux_engine_desc& D = e->desc;
  const int Hq = D.num_q_heads, d = e->d, NT = e->NT, Hkv = e->Hkv;
  const size_t qrow = static_cast<size_t>(Hq) * d * 2, kvrow = static_cast<size_t>(Hkv) * d * 2;
  const int nsplit = mux_partition_count(e->part);
  // FCFS in arrival order (arrival_iter, then arrival_us), submission order among equals
  std::vector<int> order(e->reqs.size());
  for (int i = 0; i < static_cast<int>(e->reqs.size()); ++i) {
    e->reqs[i].gen_launched = e->reqs[i].gen_done = 0;
    order[i] = i;
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const mux_request &x = e->reqs[a].r, &y = e->reqs[b].r;
    return x.arrival_iter != y.arrival_iter ? x.arrival_iter < y.arrival_iter : x.arrival_us < y.arrival_us;
  });
  std::deque<int> queue(order.begin(), order.end());
  const auto t_run0 = std::chrono::steady_clock::now();
  auto elapsed_us = [&]() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_run0).count();
  };
  int dec_done = 0;                    // decode iterations completed (arrival_iter clock)
  std::vector<int> iter_end_log;       // log slot of each completed iteration's end stamp
  const size_t orow = static_cast<size_t>(Hq) * d * e->osz;
  // output log: rows [row0, row0 + rows) of `o` (and `y`) appended if they fit
  auto log_out = [&](const void* o, const void* y, int rows, cudaStream_t st) -> int {
    if (!D.log_rows || e->log_rows_used + rows > D.log_rows) return MUX_OK;
    const size_t r0 = static_cast<size_t>(e->log_rows_used);
    MUX_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(D.o_log) + r0 * orow, o, rows * orow, cudaMemcpyDeviceToDevice, st));
    if (D.w_o) {
      const size_t yrow = static_cast<size_t>(D.hidden) * 2;
      MUX_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(D.y_log) + r0 * yrow, y, rows * yrow, cudaMemcpyDeviceToDevice, st));
    }
    e->log_rows_used += rows;
    return MUX_OK;
  };
  std::vector<int> decode, ready;
  std::deque<Group> pf_out;
  struct Job {
    bool active = false;
    std::vector<int> reqs;
    int layers_done = 0, buf = 0;
    Built batch;
    double sum_n2 = 0, sum_nr = 0, sum_n = 0;
  } job;
  int job_buf = 0, dslot_i = 0, pslot_i = 0, preslot_i = 0;
  // decode iterations in flight, oldest first: 1 (launch after completion) or, with
  // desc.overlap, 2 (the next iteration is enqueued behind the running one: no device gap)
  struct Iter {
    cudaEvent_t ev;
    std::vector<int> members;
    int li;
  };
  std::deque<Iter> dec_q;
  const size_t depth = D.overlap ? 2 : 1;
  cudaEvent_t last_dec_ev = nullptr;
  int cur_split = D.fixed_split >= -1 ? D.fixed_split : -1;
  int last_dec_split = -3, last_pf_split = -3;
  cudaEvent_t last_pf_ev = nullptr;
  bool decode_seen = false;
  int split_changes = 0, handoffs = 0, iters = 0, groups = 0;
  int64_t pf_tokens = 0, dc_tokens = 0;

  auto streams = [&](int sp, cudaStream_t* ds, cudaStream_t* ps, int* dsms, int* psms) {
    mux_stream_t a, b;
    int r2 = mux_partition_query(e->part, sp, dsms, psms, &a, &b);
    *ds = reinterpret_cast<cudaStream_t>(a);
    *ps = D.serialize ? *ds : reinterpret_cast<cudaStream_t>(b);  // one stream: no overlap
    return r2;
  };
  auto release = [&](Req& r) {
    r.finished = true;
    if (!D.keep_pages && !r.pages.empty()) mux_pool_free_pages(e->pool, static_cast<int32_t>(r.pages.size()), r.pages.data());
  };
  auto choose_split = [&]() -> int {
    if (D.fixed_split >= -1) return D.fixed_split;
    double sum_r = 0;
    for (int i : decode) sum_r += e->reqs[i].ctx;
    int best = -1, best_sms = 1 << 30, big = -1, big_sms = -1;
    for (int i = 0; i < nsplit; ++i) {
      int ds, ps;
      mux_partition_query(e->part, i, &ds, &ps, nullptr, nullptr);
      const double worst = eq2(&e->dec_theta[3 * i], sum_r, static_cast<int>(decode.size())) * e->slowdown[i] * NT;
      if (worst <= D.tbt_slo_us && ds < best_sms) {
        best = i;
        best_sms = ds;
      }
      if (ds > big_sms) {
        big = i;
        big_sms = ds;
      }
    }
    return best >= 0 ? best : big;  // infeasible SLO: the largest decode share
  };

  bool done = false;
  while (true) {
    bool did = false;
    // ---- 1. decode iteration completed: tokens "returned", finished requests retire
    // event_done: cudaSuccess -> true, cudaErrorNotReady -> false, anything else (a sticky fault of
    // a kernel, e.g. cudaErrorIllegalAddress) ends the run with MUX_ERR_CUDA instead of polling forever
    while (!dec_q.empty()) {
      if ((rc = event_done(dec_q.front().ev, &done)) != MUX_OK) return rc;
      if (!done) break;
      did = true;
      ++dec_done;
      iter_end_log.push_back(dec_q.front().li + 1);
      for (int i : dec_q.front().members) {
        Req& r = e->reqs[i];
        if (++r.gen_done == r.r.gen) release(r);
      }
      dec_q.pop_front();
    }
    // ---- 2. prefill groups completed (in order); a finished prefill is ready to merge
    while (!pf_out.empty()) {
      if ((rc = event_done(pf_out.front().ev, &done)) != MUX_OK) return rc;
      if (!done) break;
      Group g = pf_out.front();
      pf_out.pop_front();
      did = true;
      if (g.last)
        for (int i : g.reqs) {
          Req& r = e->reqs[i];
          if (r.r.gen > 0) ready.push_back(i);
          else release(r);
        }
    }
    // ---- 3. next decode iteration (launched first)
    if (dec_q.size() < depth) {
      // requests whose last iteration is already enqueued leave the batch
      decode.erase(std::remove_if(decode.begin(), decode.end(),
                                  [&](int i) { return e->reqs[i].gen_launched >= e->reqs[i].r.gen; }),
                   decode.end());
      while (!ready.empty() && static_cast<int>(decode.size()) < D.max_decode_seqs) {
        decode.push_back(ready.front());
        ready.erase(ready.begin());
      }
      if (!decode.empty()) {
        decode_seen = true;
        // no prefill work left anywhere: the decode iterations get the whole GPU (R24)
        const bool pf_idle = !job.active && queue.empty() && pf_out.empty();
        const int sp = pf_idle ? -1 : choose_split();
        if (last_dec_split != -3 && sp != last_dec_split) ++split_changes;
        cur_split = sp;
        cudaStream_t ds, ps;
        int dsms, psms;
        if ((rc = streams(sp, &ds, &ps, &dsms, &psms))) return rc;
        // the iteration reuses the previous one's buffers: order it after it across a split change
        if (last_dec_ev && sp != last_dec_split) MUX_CUDA(cudaStreamWaitEvent(ds, last_dec_ev, 0));
        std::vector<Req*> rs;
        std::vector<int> nn, kv, p0;
        for (int i : decode) {
          Req& r = e->reqs[i];
          ++r.gen_launched;
          if (r.ctx % kPage == 0) {  // the new token opens a page
            int32_t id;
            if ((rc = mux_pool_alloc_pages(e->pool, 1, &id))) return rc;
            r.pages.push_back(id);
          }
          p0.push_back(r.ctx);
          r.ctx += 1;
          rs.push_back(&r);
          nn.push_back(1);
          kv.push_back(r.ctx);
        }
        int li;
        if ((rc = log_pair(e, &li))) return rc;
        // batch arrays: the slot's own device copy, or (graphs) the fixed buffer every captured
        // iteration reads, with [0] = the log slot of its end stamp (stream order keeps a running
        // iteration's reads ahead of the next upload)
        Slot& s = e->dslot[dslot_i];
        dslot_i ^= 1;
        if ((rc = slot_acquire(s))) return rc;
        const int off = D.use_graphs ? 1 : 0;
        int32_t* dev = D.use_graphs ? e->dfix : s.d;
        Slot view = s;
        view.h = s.h + off;
        Built bt = build_batch(view, rs, nn, kv, p0, D.src_rows, dev + off);
        s.h[0] = D.use_graphs ? li : s.h[0];
        launch_stamp(e->log + li, ds);   // the iteration starts with its batch upload
        MUX_CUDA(cudaMemcpyAsync(dev, s.h, (bt.n + off) * 4, cudaMemcpyHostToDevice, ds));
        MUX_CUDA(cudaEventRecord(s.done, ds));
        s.used = true;
        const int B = bt.rows;
        auto gathers = [&]() -> int {
          int r2;
          if ((r2 = gather(D.src_q, e->dq, bt.d_idx, B, static_cast<int>(qrow), ds))) return r2;
          if ((r2 = gather(D.src_k, e->dk, bt.d_idx, B, static_cast<int>(kvrow), ds))) return r2;
          return gather(D.src_v, e->dv, bt.d_idx, B, static_cast<int>(kvrow), ds);
        };
        mux_side side{};
        side.batch = &bt.b;
        side.num_q_heads = Hq;
        side.q = e->dq;
        side.k_new = e->dk;
        side.v_new = e->dv;
        side.o = e->do_;
        side.o_dtype = e->osz == 4 ? MUX_DTYPE_F32 : MUX_DTYPE_BF16;
        side.scale = D.scale;
        side.layer0 = 0;
        side.num_layers = NT;
        side.append = 1;
        side.num_splits = 0;
        side.ws = e->ws;
        side.ws_bytes = e->ws_bytes;
        if (D.w_o) {
          side.w_o = D.w_o;
          side.y = e->dy;
          side.hidden = D.hidden;
          side.y_dtype = MUX_DTYPE_BF16;
        }
        if (!D.use_graphs) {
          if ((rc = gathers())) return rc;
          if ((rc = run_side(e->pool, &side, true, dsms, ds, nullptr, e->log + li + 1))) return rc;
        } else {
          // f2: the whole iteration is one graph launch.  Its launch shapes are fixed by
          // (split, B, split-KV count, pages per split); everything else it reads from device memory.
          const int S = mux_decode_num_splits(B, Hkv, d, bt.b.h_kv_len, bt.b.max_kv, dsms);
          const int maxp = (bt.b.max_kv + kPage - 1) / kPage;
          const int pps = std::max(1, (maxp + S - 1) / S);
          side.num_splits = S;
          const auto key = std::make_tuple(sp, B, S, pps);
          auto it = e->graphs.find(key);
          if (it == e->graphs.end()) {
            MUX_CUDA(cudaStreamBeginCapture(ds, cudaStreamCaptureModeThreadLocal));
            int r2 = gathers();
            if (!r2) r2 = run_side(e->pool, &side, true, dsms, ds, nullptr, nullptr);
            if (!r2) stamp_at_kernel<<<1, 1, 0, ds>>>(e->log, e->dfix, 1);   // end stamp: log[li + 1]
            cudaGraph_t g = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(ds, &g);
            if (r2) {
              if (g) cudaGraphDestroy(g);
              return r2;
            }
            MUX_CUDA(ce);
            size_t f0 = 0, f1 = 0, tot = 0;
            MUX_CUDA(cudaMemGetInfo(&f0, &tot));
            cudaGraphExec_t x = nullptr;
            const cudaError_t ie = cudaGraphInstantiate(&x, g, 0);
            cudaGraphDestroy(g);
            MUX_CUDA(ie);
            MUX_CUDA(cudaGraphUpload(x, ds));
            MUX_CUDA(cudaMemGetInfo(&f1, &tot));
            e->graph_bytes += static_cast<int64_t>(f0) - static_cast<int64_t>(f1);
            it = e->graphs.emplace(key, x).first;
          }
          MUX_CUDA(cudaGraphLaunch(it->second, ds));
        }
        if (D.log_rows && e->log_rows_used + B <= D.log_rows) {
          for (int k = 0; k < B; ++k) {
            const Req& r = *rs[k];
            e->out_rows.insert(e->out_rows.end(), {r.r.id, p0[k], 1});
          }
          if ((rc = log_out(e->do_, e->dy, B, ds))) return rc;
        }
        e->iv.push_back({0, li, sp, B});
        Iter it{};
        if ((rc = new_event(e, &it.ev))) return rc;
        MUX_CUDA(cudaEventRecord(it.ev, ds));
        it.members = decode;
        it.li = li;
        dec_q.push_back(it);
        last_dec_ev = it.ev;
        last_dec_split = sp;
        dc_tokens += B;
        ++iters;
        did = true;
      }
    }
    // ---- 4. admit the next prefill batch (FCFS, up to max_prefill_tokens new tokens)
    // arrival gate: decode iterations completed and host time since the start; a request waiting
    // for an iteration count no decode work can reach is admitted when the engine would idle
    const bool no_decode_work = decode.empty() && ready.empty() && dec_q.empty();
    auto admissible = [&](int i) {
      const mux_request& r = e->reqs[i].r;
      if (elapsed_us() < r.arrival_us) return false;
      return dec_done >= r.arrival_iter || (no_decode_work && pf_out.empty() && !job.active);
    };
    if (!job.active && !queue.empty() && admissible(queue.front())) {
      job = Job();
      int tok = 0;
      while (!queue.empty() && admissible(queue.front()) &&
             (job.reqs.empty() || tok + e->reqs[queue.front()].r.prompt <= D.max_prefill_tokens)) {
        Req& r = e->reqs[queue.front()];
        const int k = std::min(r.r.arrival_iter, dec_done);
        r.arrive_log = k > 0 ? iter_end_log[k - 1] : -1;
        r.arrived = true;
        tok += r.r.prompt;
        job.reqs.push_back(queue.front());
        queue.pop_front();
      }
      job.active = true;
      job.buf = job_buf;
      job_buf ^= 1;
      // target stream of the prep work: that of the first group
      const int sp = (decode.empty() && ready.empty() && dec_q.empty()) ? -1 : cur_split;
      cudaStream_t ds, ps;
      int dsms, psms;
      if ((rc = streams(sp, &ds, &ps, &dsms, &psms))) return rc;
      if (last_pf_ev && sp != last_pf_split) MUX_CUDA(cudaStreamWaitEvent(ps, last_pf_ev, 0));
      std::vector<Req*> rs, pre_rs;
      std::vector<int> nn, kv, p0, pre_n, pre_kv, pre_p0;
      for (int i : job.reqs) {
        Req& r = e->reqs[i];
        const int L = r.r.cached + r.r.prompt;
        const int np = (L + kPage - 1) / kPage;
        r.pages.resize(np);
        if ((rc = mux_pool_alloc_pages(e->pool, np, r.pages.data()))) return rc;
        rs.push_back(&r);
        nn.push_back(r.r.prompt);
        kv.push_back(L);
        p0.push_back(r.r.cached);
        if (r.r.cached > 0) {
          pre_rs.push_back(&r);
          pre_n.push_back(r.r.cached);
          pre_kv.push_back(r.r.cached);
          pre_p0.push_back(0);
        }
        r.ctx = L;
        const double n = r.r.prompt, rr = r.r.cached;
        job.sum_n2 += n * n;
        job.sum_nr += n * rr;
        job.sum_n += n;
        pf_tokens += r.r.prompt;
      }
      // cached prefix: already "in the pool" when the request arrives -> preload every layer
      if (!pre_rs.empty()) {
        Slot& s = e->preslot[preslot_i];
        preslot_i ^= 1;
        if ((rc = slot_acquire(s))) return rc;
        Built pb = build_batch(s, pre_rs, pre_n, pre_kv, pre_p0, D.src_rows);
        MUX_CUDA(cudaMemcpyAsync(s.d, s.h, pb.n * 4, cudaMemcpyHostToDevice, ps));
        MUX_CUDA(cudaEventRecord(s.done, ps));
        s.used = true;
        if ((rc = gather(D.src_k, e->prek, pb.d_idx, pb.rows, static_cast<int>(kvrow), ps))) return rc;
        if ((rc = gather(D.src_v, e->prev, pb.d_idx, pb.rows, static_cast<int>(kvrow), ps))) return rc;
        for (int l = 0; l < NT; ++l)
          if ((rc = mux_append_kv(e->pool, l, &pb.b, e->prek, e->prev, reinterpret_cast<mux_stream_t>(ps)))) return rc;
      }
      Slot& s = e->pslot[pslot_i];
      pslot_i ^= 1;
      if ((rc = slot_acquire(s))) return rc;
      job.batch = build_batch(s, rs, nn, kv, p0, D.src_rows);
      MUX_CUDA(cudaMemcpyAsync(s.d, s.h, job.batch.n * 4, cudaMemcpyHostToDevice, ps));
      MUX_CUDA(cudaEventRecord(s.done, ps));
      s.used = true;
      const int T = job.batch.rows;
      if ((rc = gather(D.src_q, e->pq[job.buf], job.batch.d_idx, T, static_cast<int>(qrow), ps))) return rc;
      if ((rc = gather(D.src_k, e->pk[job.buf], job.batch.d_idx, T, static_cast<int>(kvrow), ps))) return rc;
      if ((rc = gather(D.src_v, e->pv[job.buf], job.batch.d_idx, T, static_cast<int>(kvrow), ps))) return rc;
      cudaEvent_t prep;
      if ((rc = new_event(e, &prep))) return rc;
      MUX_CUDA(cudaEventRecord(prep, ps));
      last_pf_ev = prep;
      last_pf_split = sp;
      did = true;
    }
    // ---- 5. keep up to two prefill groups of N_PL layers queued (layer-wise prefill)
    if (job.active && job.layers_done < NT && pf_out.size() < 2) {
      const bool dec_idle = decode.empty() && ready.empty() && dec_q.empty();
      int sp = cur_split;
      if (dec_idle && (D.handoff || !decode_seen)) {
        if (sp != -1 && decode_seen && last_pf_split != -1) ++handoffs;
        sp = -1;  // no decode work: every SM to the prefill (P:531 hand-off)
      }
      cudaStream_t ds, ps;
      int dsms, psms;
      if ((rc = streams(sp, &ds, &ps, &dsms, &psms))) return rc;
      if (last_pf_ev && sp != last_pf_split) MUX_CUDA(cudaStreamWaitEvent(ps, last_pf_ev, 0));
      int npl = NT;
      if (D.fixed_pl > 0) {
        npl = D.fixed_pl;
      } else if (!e->dec_theta.empty() && !dec_idle && sp >= 0) {
        double sum_r = 0;
        for (int i : decode) sum_r += e->reqs[i].ctx;
        const double td = eq2(&e->dec_theta[3 * sp], sum_r, static_cast<int>(decode.size()));
        const double tp = eq1(&e->pf_theta[4 * sp], job.sum_n2, job.sum_nr, job.sum_n);
        // N_PL = ceil(T_d N_T / T_P) with T_d = N_T td, T_P = N_T tp (per-layer predictions)
        npl = mux_num_prefill_layers(td * NT, tp * NT, NT, NT - job.layers_done);
      }
      npl = std::max(1, std::min(npl, NT - job.layers_done));
      mux_side side{};
      side.batch = &job.batch.b;
      side.num_q_heads = Hq;
      side.q = e->pq[job.buf];
      side.k_new = e->pk[job.buf];
      side.v_new = e->pv[job.buf];
      side.o = e->po[job.buf];
      side.o_dtype = e->osz == 4 ? MUX_DTYPE_F32 : MUX_DTYPE_BF16;
      side.scale = D.scale;
      side.layer0 = job.layers_done;
      side.num_layers = npl;
      side.append = 1;
      if (D.w_o) {
        side.w_o = D.w_o;
        side.y = e->py[job.buf];
        side.hidden = D.hidden;
        side.y_dtype = MUX_DTYPE_BF16;
      }
      int li;
      if ((rc = log_pair(e, &li))) return rc;
      if ((rc = run_side(e->pool, &side, false, psms, ps, e->log + li, e->log + li + 1))) return rc;
      e->iv.push_back({1, li, sp, job.batch.rows});
      Group g;
      if ((rc = new_event(e, &g.ev))) return rc;
      MUX_CUDA(cudaEventRecord(g.ev, ps));
      job.layers_done += npl;
      g.last = job.layers_done == NT;
      if (g.last) {
        g.reqs = job.reqs;
        for (int i : job.reqs) e->reqs[i].ttft_log = li + 1;
        job.active = false;
        const int T = job.batch.rows;
        if (D.log_rows && e->log_rows_used + T <= D.log_rows) {
          for (int i : job.reqs) {
            const Req& r = e->reqs[i];
            for (int t = 0; t < r.r.prompt; ++t) e->out_rows.insert(e->out_rows.end(), {r.r.id, r.r.cached + t, 0});
          }
          if ((rc = log_out(e->po[job.buf], e->py[job.buf], T, ps))) return rc;
        }
      }
      pf_out.push_back(g);
      last_pf_ev = g.ev;
      last_pf_split = sp;
      ++groups;
      did = true;
    }
    // ---- 6. done?
    if (dec_q.empty() && pf_out.empty() && !job.active && queue.empty() && ready.empty() && decode.empty()) break;
    if (!did) std::this_thread::yield();
  }
  MUX_CUDA(cudaDeviceSynchronize());

  // ---- statistics from the device log
  std::vector<unsigned long long> lg(e->log_n);
  if (e->log_n) MUX_CUDA(cudaMemcpy(lg.data(), e->log, e->log_n * 8, cudaMemcpyDeviceToHost));
  mux_engine_stats S{};
  unsigned long long t_first = ~0ull, t_last = 0;
  for (auto& v : e->iv) {
    t_first = std::min(t_first, lg[v.log]);
    t_last = std::max(t_last, lg[v.log + 1]);
  }
  double bub[2] = {0, 0}, busy[2] = {0, 0};
  int have[2] = {0, 0};
  for (int side = 0; side < 2; ++side) {
    std::vector<std::pair<unsigned long long, unsigned long long>> xs;
    for (auto& v : e->iv)
      if (v.side == side) xs.push_back({lg[v.log], lg[v.log + 1]});
    if (xs.empty()) continue;
    std::sort(xs.begin(), xs.end());
    unsigned long long w0 = xs.front().first, w1 = 0, cs = xs.front().first, ce = xs.front().second;
    double b = 0;
    for (auto& x : xs) {
      w1 = std::max(w1, x.second);
      if (x.first > ce) {
        b += static_cast<double>(ce - cs);
        cs = x.first;
        ce = x.second;
      } else {
        ce = std::max(ce, x.second);
      }
    }
    b += static_cast<double>(ce - cs);
    busy[side] = b * 1e-3;
    bub[side] = w1 > w0 ? 1.0 - b / static_cast<double>(w1 - w0) : 0.0;
    have[side] = 1;
  }
  S.makespan_us = t_last > t_first ? (t_last - t_first) * 1e-3 : 0.0;
  S.prefill_tokens = pf_tokens;
  S.decode_tokens = dc_tokens;
  S.decode_iters = iters;
  S.prefill_groups = groups;
  S.split_changes = split_changes;
  S.handoffs = handoffs;
  S.busy_dec_us = busy[0];
  S.busy_pf_us = busy[1];
  S.bubble_ratio_dec = bub[0];
  S.bubble_ratio_pf = bub[1];
  S.bubble_ratio = (have[0] + have[1]) ? (bub[0] * have[0] + bub[1] * have[1]) / (have[0] + have[1]) : 0.0;
  unsigned long long prev_end = 0;
  double tsum = 0;
  int tn = 0;
  for (auto& v : e->iv) {
    if (v.side != 0) continue;
    if (prev_end) {
      const double t = (lg[v.log + 1] - prev_end) * 1e-3;
      tsum += t;
      ++tn;
      S.tbt_max_us = std::max(S.tbt_max_us, t);
    }
    prev_end = lg[v.log + 1];
  }
  S.tbt_mean_us = tn ? tsum / tn : 0.0;
  // decode-side launch gap: idle device time between consecutive iterations
  prev_end = 0;
  double gsum = 0;
  int gn = 0;
  for (auto& v : e->iv) {
    if (v.side != 0) continue;
    if (prev_end) {
      const double t = lg[v.log] > prev_end ? (lg[v.log] - prev_end) * 1e-3 : 0.0;
      gsum += t;
      ++gn;
      S.gap_max_us = std::max(S.gap_max_us, t);
    }
    prev_end = lg[v.log + 1];
  }
  S.gap_mean_us = gn ? gsum / gn : 0.0;
  S.graphs = static_cast<int32_t>(e->graphs.size());
  S.graph_bytes = e->graph_bytes;
  S.logged_rows = e->log_rows_used;
  double fsum = 0;
  int fn = 0;
  for (auto& r : e->reqs)
    if (r.ttft_log >= 0) {
      const unsigned long long a = r.arrive_log >= 0 ? lg[r.arrive_log] : t_first;
      const double t = lg[r.ttft_log] > a ? (lg[r.ttft_log] - a) * 1e-3 : 0.0;
      fsum += t;
      ++fn;
      S.ttft_max_us = std::max(S.ttft_max_us, t);
    }
  S.ttft_mean_us = fn ? fsum / fn : 0.0;
  if (st) *st = S;
  return MUX_OK;
}

int mux_engine_request_pages(mux_engine_t e, int32_t id, int32_t* kv_len, int32_t* page_ids, int32_t cap,
                             int32_t* n_pages) {
  if (!e) return fail(MUX_ERR_INVALID_ARG, "engine NULL");
  for (auto& r : e->reqs)
    if (r.r.id == id) {
      if (kv_len) *kv_len = r.ctx;
      const int n = static_cast<int>(r.pages.size());
      if (n_pages) *n_pages = n;
      if (page_ids)
        for (int i = 0; i < n && i < cap; ++i) page_ids[i] = r.pages[i];
      return MUX_OK;
    }
  return fail(MUX_ERR_INVALID_ARG, "no request with this id");
}

int mux_engine_trace(mux_engine_t e, int64_t* out, int32_t cap, int32_t* n) {
  if (!e || !n) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  std::vector<unsigned long long> lg(e->log_n);
  if (e->log_n) MUX_CUDA(cudaMemcpy(lg.data(), e->log, e->log_n * 8, cudaMemcpyDeviceToHost));
  int k = 0;
  for (auto& v : e->iv) {
    if (out && k < cap) {
      out[6 * k + 0] = v.side;
      out[6 * k + 1] = v.split;
      out[6 * k + 2] = v.batch;
      out[6 * k + 3] = static_cast<int64_t>(lg[v.log]);
      out[6 * k + 4] = static_cast<int64_t>(lg[v.log + 1]);
      out[6 * k + 5] = 0;
    }
    ++k;
  }
  *n = k;
  return MUX_OK;
}

int mux_engine_out_rows(mux_engine_t e, int32_t* out, int32_t cap, int32_t* n) {
  if (!e || !n) return fail(MUX_ERR_INVALID_ARG, "bad argument");
  const int rows = static_cast<int>(e->out_rows.size() / 3);
  if (out)
    for (int i = 0; i < rows && i < cap; ++i)
      for (int j = 0; j < 3; ++j) out[3 * i + j] = e->out_rows[3 * i + j];
  *n = rows;
  return MUX_OK;
}

int mux_engine_destroy(mux_engine_t e) {
  if (!e) return MUX_OK;
  cudaDeviceSynchronize();
  for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second);
  if (e->dfix) cudaFree(e->dfix);
  for (void* p : {e->dq, e->dk, e->dv, e->do_, e->dy, e->ws, e->prek, e->prev})
    if (p) cudaFree(p);
  for (int i = 0; i < 2; ++i) {
    for (void* p : {e->pq[i], e->pk[i], e->pv[i], e->po[i], e->py[i]})
      if (p) cudaFree(p);
    for (Slot* s : {&e->dslot[i], &e->pslot[i], &e->preslot[i]}) {
      if (s->h) cudaFreeHost(s->h);
      if (s->d) cudaFree(s->d);
      if (s->done) cudaEventDestroy(s->done);
    }
  }
  if (e->log) cudaFree(e->log);
  for (auto ev : e->events) cudaEventDestroy(ev);
  delete e;
  return MUX_OK;
}

}  // extern "C"
