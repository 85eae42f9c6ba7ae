// a4 decode split-KV paged attention + a5 log-sum-exp split combine.
//
// PAPER: decode attends one new token over r+1 cached keys, O(d^2 + (r+1)d) (Table 2,
// P:590), memory-intensive, latency linear in sum r (Eq.2).  The split-KV
// (flash-decoding) organisation + combine pass is BASELINE.json's north_star; it is an
// exact reorganisation of the softmax.
//
// B200 design: HBM-bound, so the kernel is a page-streaming engine.
//   grid (num_splits, Hkv/HG, B); one CTA per SM; 10 warps: 0-7 consumers, 8 K producer, 9 V producer.
//   Producers: one lane each issues one TMA op per page (cp.async.bulk.tensor.5d, SWIZZLE_128B):
//   the K and the V block of the page for all HG (<= 8) kv heads of the CTA's group — 32 KiB
//   each at d=128, HG=8.  The per-SM TMA engine is op-rate bound (measured: 2 KiB boxes cap
//   an SM at ~49 GB/s, 32 KiB ops at ~200 GB/s), so big boxes are what lets a 16-48 SM
//   decode partition pull near-full HBM bandwidth.  ~192 KiB ring in flight per SM.
//   Consumers: warp w owns kv head w%HG and every (8/HG)-th page; legacy tensor pipe (the
//   group of g <= 8 q heads is the N=8 side, so FP32 ALU is left for the softmax):
//     S^T[16 tok x 8 heads] = K_page[16 x d] . Q^T      (mma.m16n8k16, A = K via ldmatrix)
//     online softmax per head column with a lazy reference max (moves only when a score exceeds it
//     by > 8); the exact page max (warp shuffles over the 8 token lanes) only when a warp vote
//     says some column grew
//     P^T -> B fragments with movmatrix.trans (no smem round trip), P in fp16 (11-bit, DESIGN.md
//     "P precision"), which the fp16 V cache (R25) allows in ONE mma per tile (r01: bf16 V needed
//     P = P_hi + P_lo, two bf16 MMAs)
//     O^T[d x 8] += V_page^T . P^T (A = V^T via ldmatrix.trans, fp16)
//   Warps merge their (m, l, O) states in smem at the end; with one split the CTA writes
//   the normalised output, otherwise fp32 partials (o, m, l) for the combine kernel.
//   Per SM the kernel is bound by the shared-memory port (TMA writes + ldmatrix reads of every KV
//   byte, 128 B/clk) and the per-page dependency chain; the A/B switches below (MUX_DEC_*) record the
//   variants measured against it (profiles/r01_summary.md).
#include <math.h>

#include <algorithm>
#include <queue>
#include <vector>

#include "pool.h"

#ifndef MUX_DEC_EVICT_FIRST
#define MUX_DEC_EVICT_FIRST 1
#endif
// A/B switch: mbarrier waits of the producers (bit 0) / consumers (bit 1) as sleeping try_waits
// (suspend-time hint) instead of spins
#ifndef MUX_DEC_SLEEP
#define MUX_DEC_SLEEP 0
#endif
#if MUX_DEC_SLEEP & 1
#define DEC_WAIT_P(b, ph) dev::mbar_wait_sleep(b, ph, 2000)
#else
#define DEC_WAIT_P(b, ph) dev::mbar_wait(b, ph)
#endif
#if MUX_DEC_SLEEP & 2
#define DEC_WAIT_C(b, ph) dev::mbar_wait_sleep(b, ph, 2000)
#else
#define DEC_WAIT_C(b, ph) dev::mbar_wait(b, ph)
#endif

namespace mux {
namespace {

// Consumer warps per CTA and head_dim split.  Default: 8 warps, one per (kv head, page lane).
// MUX_DEC_SPLITD=2 (A/B build switch, g <= 8 only): 16 warps, two per kv head, each owning half of
// head_dim (its half of the QK reduction and of the O rows), the two partial score tiles exchanged
// through shared memory behind a 64-thread named barrier.  Measured slower on B200 (cfg2 layer on
// 16 SMs: 704 us vs 560; profiles/r01_summary.md), kept for the record and for later tuning.
#ifndef MUX_DEC_SPLITD
#define MUX_DEC_SPLITD 1
#endif
// C2: two CTAs per SM (4 kv heads, 4 consumer warps, 96 KiB ring each): on small decode partitions
// one CTA's ring fill / drain overlaps the other's streaming (8 SMs: 1188 -> 1146-1179 us per cfg2
// layer in the multiplexed step, 16 SMs: 616 -> 601 us; slower in the mux layer at 32-96 SMs, r01), so
// it is chosen at launch for partitions of <= kDec2CtaMaxSms SMs (decode_launch_sms, the split model)
constexpr int kDec2CtaMaxSms = 16;
template <int NT, bool C2 = false> struct DecodeCfg {
  static constexpr int kSplitD = (NT == 1 && MUX_DEC_SPLITD == 2 && !C2) ? 2 : 1;   // warps per (head, page)
  static constexpr int kConsumerWarps = C2 ? 4 : 8 * kSplitD;
  static constexpr int kCtasPerSm = C2 ? 2 : 1;
  static constexpr int kThreads = (kConsumerWarps + 2) * 32;   // + K producer + V producer
};
#ifndef MUX_DEC_RING_KB
#define MUX_DEC_RING_KB 192   // A/B switch: KiB of K + V stages per SM
#endif
template <bool C2> constexpr int ring_bytes() { return (C2 ? MUX_DEC_RING_KB / 2 : MUX_DEC_RING_KB) * 1024; }

struct DecodeParams {
  const uint16_t* q;         // [B][Hq][D]
  void* o;                   // [B][Hq][D]
  float* lse;                // [B][Hq] or null
  float* part_o;             // [B][Hq][S][D]
  float* part_m;             // [B][Hq][S]  (log2 domain)
  float* part_l;             // [B][Hq][S]
  const int32_t* kv_len;
  const int32_t* page_indptr;
  const int32_t* page_ids;
  int num_splits, hq, hkv, g;
  int pages_per_split;       // C: every split of every sequence covers <= C pages (balanced units)
  int page_row0;             // layer * num_pages (TMA page coordinate offset)
  int o_f32;
  float scale_log2;
};

// Two rings of stages, K and V: a stage = one page (16 tokens) of K (or V) for the HG kv heads
// of this CTA's group, as TMA lands it: [HG][d/64][16 rows][128 B] (SWIZZLE_128B).  A K stage
// is released right after QK (before the page's PV), so K refills run ahead of V.
template <int D, int NT, int HG, bool C2 = false>
struct DecodeSmem {
  using C = DecodeCfg<NT, C2>;
  static constexpr int kRingBytes = ring_bytes<C2>();
  static constexpr int kHeadBytes = D * kPage * 2;             // one (page, head) block of K (or V)
  static constexpr int kStageBytes = HG * kHeadBytes;          // K (or V) of HG heads
  static constexpr int kQStride = D + 8;                       // padded bf16 row -> conflict-free ldmatrix
  static constexpr int kQRowsPerHead = 8 * NT;                 // g <= 8*NT
  static constexpr int kQBytes = HG * kQRowsPerHead * kQStride * 2;
  // partial-score exchange of the head_dim halves: [pair][2 buffers][2 halves][32 lanes][4 f32]
  static constexpr int kPairs = C::kConsumerWarps / C::kSplitD;
  static constexpr int kXBytes = C::kSplitD > 1 ? kPairs * 2 * 2 * 32 * 16 : 0;
  static constexpr int kSmemCap = (C2 ? 112 : 224) * 1024;
  static constexpr int kRing = (kRingBytes < kSmemCap - kQBytes - kXBytes) ? kRingBytes : kSmemCap - kQBytes - kXBytes;
  // stages per ring; a multiple of the page lanes of a head (W): a warp takes every W-th page, and
  // its successive waits on one stage's mbarrier must be successive phases (parity)
  static constexpr int kW = kPairs / HG > 0 ? kPairs / HG : 1;
  static constexpr int kStagesFit = (kRing / 2 / kStageBytes) > 16 ? 16 : (kRing / 2 / kStageBytes);
  static constexpr int kStages = kStagesFit / kW * kW;
  static constexpr int kVOff = kStages * kStageBytes;
  static constexpr int kQOff = 2 * kStages * kStageBytes;
  static constexpr int kXOff = kQOff + kQBytes;
  // merge area (aliases the ring, Q and the exchange after the main loop): per pair 16 heads x D f32 + m, l
  static constexpr int kMergeM = kPairs * 16 * D * 4;
  static constexpr int kMergeL = kMergeM + kPairs * 16 * 4;
  static constexpr int kMergeEnd = kMergeL + kPairs * 16 * 4;
  static constexpr int kBarOff = (kXOff + kXBytes) > kMergeEnd ? (kXOff + kXBytes) : kMergeEnd;
  static constexpr int kBytes = kBarOff + 4 * kStages * 8;
  static_assert(kStages >= 2 && kStages % kW == 0, "ring too small");
  static_assert(kBytes + 1024 <= kSmemCap + 3 * 1024, "shared memory");
};

template <int D, int NT, int HG, bool C2>
__global__ void __launch_bounds__(DecodeCfg<NT, C2>::kThreads, DecodeCfg<NT, C2>::kCtasPerSm)
    decode_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                  const DecodeParams p) {
  using L = DecodeSmem<D, NT, HG, C2>;
  using C = DecodeCfg<NT, C2>;
  constexpr int kConsumerWarps = C::kConsumerWarps;
  constexpr int kThreads = C::kThreads;
  constexpr int SD = C::kSplitD;
  constexpr int DH = D / SD;                       // head_dim columns owned by one warp
  constexpr int STAGES = L::kStages;
  constexpr int kWarpsPerHead = L::kW;             // page lanes: warps (pairs) sharing one head split its pages
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* kfull = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* kempty = kfull + STAGES;
  uint64_t* vfull = kempty + STAGES;
  uint64_t* vempty = vfull + STAGES;
  uint16_t* qs = reinterpret_cast<uint16_t*>(smem + L::kQOff);

  const int split = blockIdx.x, grp = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kv_len = __ldg(p.kv_len + b);
  const int npages = (kv_len + kPage - 1) / kPage;
  // balanced split-KV: a fixed chunk of C pages per split for EVERY sequence, so all CTAs carry
  // (at most) the same work; a sequence shorter than the longest uses fewer splits and its
  // surplus CTAs exit at once (the combine recomputes the split count from kv_len).
  const int pps = p.pages_per_split;
  const int pg0 = min(npages, split * pps);
  const int pg1 = split == p.num_splits - 1 ? npages : min(npages, pg0 + pps);  // last split: the rest
  const int n_my = pg1 - pg0;
  if (split > 0 && n_my <= 0) return;
  const int* ptab = p.page_ids + __ldg(p.page_indptr + b);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      dev::mbar_init(&kfull[s], 1);
      dev::mbar_init(&kempty[s], HG * SD);  // every consuming warp of every head releases the stage
      dev::mbar_init(&vfull[s], 1);
      dev::mbar_init(&vempty[s], HG * SD);
    }
    dev::fence_mbar_init();
  }
  // Q rows of the HG*g q heads of this group -> [HG][8*NT][D+8] padded smem; rows >= g are zero
  {
    const uint16_t* qsrc = p.q + (static_cast<size_t>(b) * p.hq + static_cast<size_t>(grp) * HG * p.g) * D;
    for (int i = threadIdx.x; i < HG * L::kQRowsPerHead * (D / 8); i += kThreads) {
      const int row = i / (D / 8), c = i % (D / 8);
      const int hh = row / L::kQRowsPerHead, r = row % L::kQRowsPerHead;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < p.g) v = __ldg(reinterpret_cast<const uint4*>(qsrc + static_cast<size_t>(hh * p.g + r) * D) + c);
      *reinterpret_cast<uint4*>(qs + row * L::kQStride + c * 8) = v;
    }
  }
  __syncthreads();

  const int pair = warp / SD;             // (head, page lane) slot of this consumer warp
  const int half = warp % SD;             // which head_dim half it owns
  const int hw = pair % HG;               // kv head (within the group)
  const int pl = pair / HG;               // its page lane among the pairs of that head
  float m_run[NT][2], l_run[NT][2];
  float oacc[DH / 16][NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    m_run[nt][0] = m_run[nt][1] = -INFINITY;
    l_run[nt][0] = l_run[nt][1] = 0.f;
#pragma unroll
    for (int mt = 0; mt < DH / 16; ++mt) oacc[mt][nt][0] = oacc[mt][nt][1] = oacc[mt][nt][2] = oacc[mt][nt][3] = 0.f;
  }

  if (warp >= kConsumerWarps) {
    // ------------------------------------------------------------ producers: K and V warps,
    // one TMA op per page each, independent rings
    const bool is_v = warp == kConsumerWarps + 1;
    const CUtensorMap* map = is_v ? &tmap_v : &tmap_k;
    uint64_t* full = is_v ? vfull : kfull;
    uint64_t* empty = is_v ? vempty : kempty;
    uint8_t* ring = smem + (is_v ? L::kVOff : 0);
    if (lane == 0) dev::tma_prefetch(map);
#if MUX_DEC_EVICT_FIRST
    // K/V pages are read once per layer: evict-first keeps them from displacing the co-running
    // prefill's re-read K/V tiles in L2 (SM-partitioned sides still share the 126 MB L2)
    const uint64_t pol = dev::l2_evict_first();
#endif
    int ids = 0;
    for (int i = 0; i < n_my; ++i) {
      if ((i & 31) == 0) ids = (pg0 + i + lane < pg1) ? __ldg(ptab + pg0 + i + lane) : 0;
      const int page = __shfl_sync(0xffffffffu, ids, i & 31);
      const int s = i % STAGES;
      if (lane == 0) {
        if (i >= STAGES) DEC_WAIT_P(&empty[s], ((i / STAGES) - 1) & 1);
        dev::mbar_expect_tx(&full[s], L::kStageBytes);
#if MUX_DEC_EVICT_FIRST
        dev::tma_load_5d_hint(ring + s * L::kStageBytes, map, &full[s], 0, 0, 0, grp * HG, p.page_row0 + page, pol);
#else
        dev::tma_load_5d(ring + s * L::kStageBytes, map, &full[s], 0, 0, 0, grp * HG, p.page_row0 + page);
#endif
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    // Q^T fragments of this warp's head_dim half (k-chunks [half*DH/16, (half+1)*DH/16))
    uint32_t qf[NT][DH / 16][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int kc = 0; kc < DH / 16; kc += 2) {
        const int mi = lane >> 3;
        const int row = hw * L::kQRowsPerHead + nt * 8 + (lane & 7);
        const int chunk = 2 * (half * DH / 16 + kc) + mi;
        dev::ldsm_x4(dev::smem_u32(qs + row * L::kQStride + chunk * 8), qf[nt][kc][0], qf[nt][kc][1],
                     qf[nt][kc + 1][0], qf[nt][kc + 1][1]);
      }
    }
    float4* xb = reinterpret_cast<float4*>(smem + L::kXOff) + pair * 2 * 2 * 32;   // [2 buf][2 half][32]
    const int g4 = lane >> 2;
    int it = 0;
    for (int i = pl; i < n_my; i += kWarpsPerHead, ++it) {
      const int s = i % STAGES;
      DEC_WAIT_C(&kfull[s], (i / STAGES) & 1);
      uint8_t* kbuf = smem + s * L::kStageBytes + hw * L::kHeadBytes;
      uint8_t* vbuf = smem + L::kVOff + s * L::kStageBytes + hw * L::kHeadBytes;
      const int pos0 = (pg0 + i) * kPage;
      const int valid = min(kPage, kv_len - pos0);
      // ---- partial S^T[16 tok x 8 heads] = K[:, half] . Q[:, half]^T, even / odd k-chunks apart
      float sacc[NT][4], sacc2[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) sacc[nt][e] = sacc2[nt][e] = 0.f;
      const uint32_t kbase = dev::smem_u32(kbuf);
#pragma unroll
      for (int kc = 0; kc < DH / 16; ++kc) {
        const int mi = lane >> 3;
        const int tok = (lane & 7) + ((mi & 1) << 3);
        const int chunk = 2 * (half * DH / 16 + kc) + (mi >> 1);
        uint32_t a0, a1, a2, a3;
        dev::ldsm_x4(kbase + (chunk >> 3) * 2048 + dev::sw128(tok, chunk & 7), a0, a1, a2, a3);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          dev::mma_bf16_16816((kc & 1) ? sacc2[nt] : sacc[nt], a0, a1, a2, a3, qf[nt][kc][0], qf[nt][kc][1]);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) sacc[nt][e] += sacc2[nt][e];
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&kempty[s]);     // K page consumed: its stage may refill
      if constexpr (SD > 1) {
        // full S = own half + partner's half, added in the same order by both warps (identical S)
        float4* mine = xb + ((it & 1) * 2 + half) * 32 + lane;
        float4* other = xb + ((it & 1) * 2 + (half ^ 1)) * 32 + lane;
        *mine = make_float4(sacc[0][0], sacc[0][1], sacc[0][2], sacc[0][3]);
        dev::named_bar_sync(1 + pair, 64);
        const float4 o4 = *other;
        const float lo[4] = {half ? o4.x : sacc[0][0], half ? o4.y : sacc[0][1], half ? o4.z : sacc[0][2],
                             half ? o4.w : sacc[0][3]};
        const float hi[4] = {half ? sacc[0][0] : o4.x, half ? sacc[0][1] : o4.y, half ? sacc[0][2] : o4.z,
                             half ? sacc[0][3] : o4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) sacc[0][e] = lo[e] + hi[e];
      }
      // ---- online softmax (log2 domain); thread holds tokens g4, g4+8 x heads 2q, 2q+1
      const bool v0 = g4 < valid, v1 = (g4 + 8) < valid;
      uint32_t ph[NT][2];
      float alpha[NT][2];
      float x[NT][4];
      bool grow = false;   // does any score exceed its column's reference max by more than 8?
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        x[nt][0] = v0 ? sacc[nt][0] * p.scale_log2 : -INFINITY;
        x[nt][1] = v0 ? sacc[nt][1] * p.scale_log2 : -INFINITY;
        x[nt][2] = v1 ? sacc[nt][2] * p.scale_log2 : -INFINITY;
        x[nt][3] = v1 ? sacc[nt][3] * p.scale_log2 : -INFINITY;
        grow |= (fmaxf(x[nt][0], x[nt][2]) > m_run[nt][0] + 8.f) | (fmaxf(x[nt][1], x[nt][3]) > m_run[nt][1] + 8.f);
      }
      // lazy rescale (FA4-style): a column's reference max moves only when the page max exceeds it by
      // more than 8 (P <= 2^8 stays far inside fp16's range); otherwise alpha = 1 and the O
      // rescale below is skipped.  The exact page max (3 shuffle rounds per column on the page's
      // critical path) is only needed when some column grows, which one warp vote tells (after the
      // first page: rarely); the result is the same as always taking the max.
      grow = __any_sync(0xffffffffu, grow);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        float mn0 = m_run[nt][0], mn1 = m_run[nt][1];
        if (grow) {
          float mx0 = fmaxf(x[nt][0], x[nt][2]), mx1 = fmaxf(x[nt][1], x[nt][3]);
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) {
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
          }
          mn0 = (mx0 > m_run[nt][0] + 8.f) ? mx0 : m_run[nt][0];   // finite after page 0: valid >= 1
          mn1 = (mx1 > m_run[nt][1] + 8.f) ? mx1 : m_run[nt][1];
        }
        alpha[nt][0] = (mn0 != m_run[nt][0]) ? dev::ex2(m_run[nt][0] - mn0) : 1.f;
        alpha[nt][1] = (mn1 != m_run[nt][1]) ? dev::ex2(m_run[nt][1] - mn1) : 1.f;
        m_run[nt][0] = mn0;
        m_run[nt][1] = mn1;
        const float p0 = dev::ex2(x[nt][0] - mn0), p1 = dev::ex2(x[nt][1] - mn1);
        const float p2 = dev::ex2(x[nt][2] - mn0), p3 = dev::ex2(x[nt][3] - mn1);
        l_run[nt][0] = l_run[nt][0] * alpha[nt][0] + p0 + p2;
        l_run[nt][1] = l_run[nt][1] * alpha[nt][1] + p1 + p3;
        // P in fp16: 11 significant bits, against the fp16 V cache
        ph[nt][0] = dev::movmatrix_t(dev::pack_f16(p0, p1));    // tokens 0-7  -> b0
        ph[nt][1] = dev::movmatrix_t(dev::pack_f16(p2, p3));    // tokens 8-15 -> b1
      }
      DEC_WAIT_C(&vfull[s], (i / STAGES) & 1);
      if (valid < kPage) {
        // slots past the sequence end may hold anything (NaN-poisoned in tests): zero this warp's
        // V columns there so P = 0 never meets NaN in the PV MMA; K rows are masked by select.
        for (int r = valid; r < kPage; ++r)
          for (int c = lane; c < DH / 8; c += 32) {
            const int cc = half * (DH / 8) + c;   // logical 16-byte column chunk of the head row
            *reinterpret_cast<uint4*>(vbuf + (cc >> 3) * 2048 + dev::sw128(r, cc & 7)) = make_uint4(0, 0, 0, 0);
          }
        __syncwarp();
      }
      // ---- O^T[half] = alpha * O^T[half] + V^T[half] . P^T  (fp16 x fp16, fp32 accumulate)
      bool rescale = false;   // alpha != 1 only where a column grew (so never without `grow`)
      if (grow) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) rescale |= (alpha[nt][0] != 1.f) | (alpha[nt][1] != 1.f);
        rescale = __any_sync(0xffffffffu, rescale);
      }
      const uint32_t vbase = dev::smem_u32(vbuf);
#pragma unroll
      for (int mt = 0; mt < DH / 16; ++mt) {
        const int mi = lane >> 3;
        const int tok = (lane & 7) + ((mi >> 1) << 3);
        const int chunk = 2 * (half * DH / 16 + mt) + (mi & 1);
        uint32_t a0, a1, a2, a3;
        dev::ldsm_x4_t(vbase + (chunk >> 3) * 2048 + dev::sw128(tok, chunk & 7), a0, a1, a2, a3);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (rescale) {
            oacc[mt][nt][0] *= alpha[nt][0];
            oacc[mt][nt][1] *= alpha[nt][1];
            oacc[mt][nt][2] *= alpha[nt][0];
            oacc[mt][nt][3] *= alpha[nt][1];
          }
          dev::mma_f16_16816(oacc[mt][nt], a0, a1, a2, a3, ph[nt][0], ph[nt][1]);
        }
      }
      __syncwarp();
      if (lane == 0) dev::mbar_arrive(&vempty[s]);
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        l_run[nt][0] += __shfl_xor_sync(0xffffffffu, l_run[nt][0], off);
        l_run[nt][1] += __shfl_xor_sync(0xffffffffu, l_run[nt][1], off);
      }
  }
  __syncthreads();  // all TMA traffic consumed: the stage ring becomes the merge area

  float* mo = reinterpret_cast<float*>(smem);
  float* mm = reinterpret_cast<float*>(smem + L::kMergeM);
  float* ml = reinterpret_cast<float*>(smem + L::kMergeL);
  if (warp < kConsumerWarps) {
    const int g4 = lane >> 2, q4 = lane & 3;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int h0 = nt * 8 + 2 * q4;
      if (g4 == 0 && half == 0) {   // both halves hold the same m, l
        mm[pair * 16 + h0] = m_run[nt][0];
        mm[pair * 16 + h0 + 1] = m_run[nt][1];
        ml[pair * 16 + h0] = l_run[nt][0];
        ml[pair * 16 + h0 + 1] = l_run[nt][1];
      }
      float* base = mo + (pair * 16) * D + half * DH;
#pragma unroll
      for (int mt = 0; mt < DH / 16; ++mt) {
        base[h0 * D + mt * 16 + g4] = oacc[mt][nt][0];
        base[(h0 + 1) * D + mt * 16 + g4] = oacc[mt][nt][1];
        base[h0 * D + mt * 16 + g4 + 8] = oacc[mt][nt][2];
        base[(h0 + 1) * D + mt * 16 + g4 + 8] = oacc[mt][nt][3];
      }
    }
  }
  __syncthreads();
  // merge the page lanes of each head: element (head-in-group, q head, dim) per thread
  for (int e = threadIdx.x; e < HG * p.g * D; e += kThreads) {
    const int c = e % D, hq_in = (e / D) % p.g, hh = e / (D * p.g);
    float M = -INFINITY;
#pragma unroll
    for (int k = 0; k < kWarpsPerHead; ++k) M = fmaxf(M, mm[(hh + k * HG) * 16 + hq_in]);
    float Ls = 0.f, acc = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int k = 0; k < kWarpsPerHead; ++k) {
        const int w = hh + k * HG;
        const float mw = mm[w * 16 + hq_in];
        if (mw == -INFINITY) continue;
        const float sc = dev::ex2(mw - M);
        Ls += sc * ml[w * 16 + hq_in];
        acc += sc * mo[(w * 16 + hq_in) * D + c];
      }
    }
    const int qh = (grp * HG + hh) * p.g + hq_in;
    const size_t row = static_cast<size_t>(b) * p.hq + qh;
    if (p.num_splits == 1) {
      const float out = acc / Ls;
      if (p.o_f32) static_cast<float*>(p.o)[row * D + c] = out;
      else static_cast<__nv_bfloat16*>(p.o)[row * D + c] = __float2bfloat16_rn(out);
      if (c == 0 && p.lse) p.lse[row] = (M + __log2f(Ls)) * 0.69314718055994531f;
    } else {
      const size_t pr = row * p.num_splits + split;
      p.part_o[pr * D + c] = (Ls > 0.f) ? acc / Ls : 0.f;
      if (c == 0) {
        p.part_m[pr] = M;
        p.part_l[pr] = Ls;
      }
    }
  }
}

// a5: O = sum_s w_s o_s / sum_s w_s with w_s = l_s 2^(m_s - M); LSE = ln2 (M + log2 sum w_s)
template <int D>
__global__ void __launch_bounds__(D) combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_m,
                                                    const float* __restrict__ part_l, void* o, float* lse,
                                                    const int32_t* __restrict__ kv_len, int hq, int pages_per_split,
                                                    int num_splits, int o_f32) {
  const size_t row = blockIdx.x;  // b*Hq + h
  const int c = threadIdx.x;
  // splits this sequence actually used (the others exited without writing partials)
  const int npages = (__ldg(kv_len + row / hq) + kPage - 1) / kPage;
  const int used = max(1, min(num_splits, (npages + pages_per_split - 1) / pages_per_split));
  float M = -INFINITY;
  for (int s = 0; s < used; ++s) {
    const float l = part_l[row * num_splits + s];
    if (l > 0.f) M = fmaxf(M, part_m[row * num_splits + s]);
  }
  float W = 0.f, acc = 0.f;
  for (int s = 0; s < used; ++s) {
    const float l = part_l[row * num_splits + s];
    if (!(l > 0.f)) continue;
    const float w = l * dev::ex2(part_m[row * num_splits + s] - M);
    W += w;
    acc += w * part_o[(row * num_splits + s) * D + c];
  }
  const float out = acc / W;
  if (o_f32) static_cast<float*>(o)[row * D + c] = out;
  else static_cast<__nv_bfloat16*>(o)[row * D + c] = __float2bfloat16_rn(out);
  if (c == 0 && lse) lse[row] = (M + __log2f(W)) * 0.69314718055994531f;
}

template <int D, int NT, int HG, bool C2 = false>
int launch_decode_hg(mux_pool* pool, const DecodeParams& prm, int B, cudaStream_t st) {
  using L = DecodeSmem<D, NT, HG, C2>;
  auto kern = decode_kernel<D, NT, HG, C2>;
  const int smem = L::kBytes + 1024;
  static bool attr_done = false;
  if (!attr_done) {
    MUX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_done = true;
  }
  dim3 grid(prm.num_splits, prm.hkv / HG, B);
  kern<<<grid, DecodeCfg<NT, C2>::kThreads, smem, st>>>(C2 ? pool->tmap_kg4 : pool->tmap_kg,
                                                        C2 ? pool->tmap_vg4 : pool->tmap_vg, prm);
  MUX_CUDA(cudaGetLastError());
  if (prm.num_splits > 1) {
    combine_kernel<D><<<B * prm.hq, D, 0, st>>>(prm.part_o, prm.part_m, prm.part_l, prm.o, prm.lse, prm.kv_len,
                                                prm.hq, prm.pages_per_split, prm.num_splits, prm.o_f32);
    MUX_CUDA(cudaGetLastError());
  }
  return MUX_OK;
}

// two CTAs per SM on small partitions (g <= 8, Hkv % 4 == 0: 4 kv heads per CTA)
bool use_dec_2cta(int hkv, int g, int num_sms) {
  return num_sms > 0 && num_sms <= kDec2CtaMaxSms && hkv % 4 == 0 && g <= 8;
}

template <int D, int NT>
int launch_decode(mux_pool* pool, const DecodeParams& prm, int B, cudaStream_t st, int num_sms) {
  if constexpr (NT == 1) {
    if (use_dec_2cta(prm.hkv, prm.g, num_sms)) return launch_decode_hg<D, NT, 4, true>(pool, prm, B, st);
  }
  switch (pool->hg) {
    case 8: return launch_decode_hg<D, NT, 8>(pool, prm, B, st);
    case 4: return launch_decode_hg<D, NT, 4>(pool, prm, B, st);
    case 2: return launch_decode_hg<D, NT, 2>(pool, prm, B, st);
    case 1: return launch_decode_hg<D, NT, 1>(pool, prm, B, st);
    default: return fail(MUX_ERR_UNSUPPORTED, "internal: kv heads per decode CTA not in {1, 2, 4, 8}");
  }
}

}  // namespace
}  // namespace mux

using namespace mux;

extern "C" {

size_t mux_decode_workspace_bytes(int32_t num_seqs, int32_t hq, int32_t d, int32_t num_splits) {
  if (num_splits <= 1) return 0;
  const size_t rows = static_cast<size_t>(num_seqs) * hq * num_splits;
  return rows * d * 4 + rows * 8 + 256;
}

int32_t mux_decode_num_splits(int32_t num_seqs, int32_t hkv, int32_t head_dim, const int32_t* kv_len,
                              int32_t max_kv, int32_t num_sms) {
  if (num_seqs < 1 || hkv < 1 || max_kv < 1) return 1;
  if (num_sms < 1) num_sms = 148;
  if (head_dim < 1) head_dim = 128;
  // the launch's CTA shape (decode_launch_sms): two CTAs of 4 kv heads per SM on small partitions,
  // else the largest power of two <= 8 dividing Hkv (as pool_tmaps)
  const bool c2 = num_sms <= kDec2CtaMaxSms && hkv % 4 == 0;
  int hg = 1;
  for (int c = 2; c <= (c2 ? 4 : 8); c *= 2)
    if (hkv % c == 0) hg = c;
  const int groups = hkv / hg;
  const int max_pages = (max_kv + kPage - 1) / kPage;
  // Host model of one launch (constants from B200 measurements, profiles/r01_summary.md): a CTA
  // streams ~100 GB/s of K+V pages, costs ~4 us to start and drain, an empty CTA ~0.3 us; the
  // combine pass ~6 us + its partial traffic.  The grid's CTAs are dispatched in launch order
  // (split fastest) onto the first free SM; the split count with the smallest predicted
  // makespan wins.  Balanced splits: C = ceil(max_pages / S) pages per split for every sequence.
  // two CTAs share an SM on small partitions: twice the slots, each streaming about half as fast
  const int slots = num_sms * (c2 ? 2 : 1);
  const double cta_bytes_per_us = c2 ? 6.5e4 : 1.0e5;
  const double page_us = static_cast<double>(hg) * kPage * head_dim * 2 * 2 / cta_bytes_per_us;
  const double cta_us = 4.0, empty_us = 0.3;
  std::vector<int> pages(num_seqs);
  for (int i = 0; i < num_seqs; ++i) {
    const int L = kv_len ? kv_len[i] : max_kv;
    pages[i] = (std::max(L, 1) + kPage - 1) / kPage;
  }
  int64_t total_pages = 0;
  for (int p : pages) total_pages += p;
  // ~6.5 TB/s measured copy bandwidth (MEASURED_PEAKS hbm_gbs), in bytes per us
  const double hbm_floor_us = static_cast<double>(total_pages) * groups * page_us * cta_bytes_per_us / 6.5e6;
  static const int cands[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64};
  int best_s = 1;
  double best_t = 1e300;
  std::vector<double> sm;
  for (int S : cands) {
    if (S > 1 && S > max_pages) break;
    const int64_t ctas = static_cast<int64_t>(num_seqs) * groups * S;
    if (S > 1 && ctas > 16LL * slots) break;       // finer units cannot pay for themselves
    const int C = (max_pages + S - 1) / S;
    sm.assign(std::min<int64_t>(slots, ctas), 0.0);
    std::priority_queue<double, std::vector<double>, std::greater<double>> q(sm.begin(), sm.end());
    double span = 0.0;
    for (int b = 0; b < num_seqs; ++b)
      for (int gi = 0; gi < groups; ++gi)
        for (int sp = 0; sp < S; ++sp) {
          const int p0 = sp * C;
          const int np = sp == S - 1 ? std::max(0, pages[b] - p0) : std::max(0, std::min(C, pages[b] - p0));
          const double t = (np > 0 || sp == 0) ? cta_us + np * page_us : empty_us;
          const double st = q.top();
          q.pop();
          q.push(st + t);
          span = std::max(span, st + t);
        }
    // the chip's HBM bandwidth caps any SM count; near the cap the SMs' streams interfere, so
    // the smaller of the two terms still counts a quarter (fitted to the cfg2 decode on 148 SMs:
    // 2 splits 168 us vs 1 split 178 us measured)
    span = std::max(span, hbm_floor_us) + 0.25 * std::min(span, hbm_floor_us);
    if (S > 1) span += 6.0 + static_cast<double>(num_seqs) * hkv * 8 * S * (head_dim + 2) * 4 / (num_sms * 1.0e5);
    if (span < best_t * 0.98) {  // a finer split must win by > 2% (model noise)
      best_t = span;
      best_s = S;
    }
  }
  return best_s;
}

int mux_decode_attn(mux_pool_t pool, int32_t layer, const mux_batch* b, int32_t hq, const void* q, void* o,
                    int32_t o_dtype, float* lse, float scale, int32_t num_splits, void* ws, size_t ws_bytes,
                    mux_stream_t stream) {
  // the public call sizes its launch for the whole device; mux_run_layer passes the partition's SMs
  return mux::decode_launch_sms(pool, layer, b, hq, q, o, o_dtype, lse, scale, num_splits, ws, ws_bytes, stream,
                                device_sm_count());
}

int mux_decode_attn_sms(mux_pool_t pool, int32_t layer, const mux_batch* b, int32_t hq, const void* q, void* o,
                        int32_t o_dtype, float* lse, float scale, int32_t num_splits, void* ws, size_t ws_bytes,
                        mux_stream_t stream, int32_t num_sms) {
  return mux::decode_launch_sms(pool, layer, b, hq, q, o, o_dtype, lse, scale, num_splits, ws, ws_bytes, stream,
                                num_sms);
}

}  // extern "C"

namespace mux {
int decode_launch_sms(mux_pool_t pool, int32_t layer, const mux_batch* b, int32_t hq, const void* q, void* o,
                      int32_t o_dtype, float* lse, float scale, int32_t num_splits, void* ws, size_t ws_bytes,
                      mux_stream_t stream, int num_sms) {
  int rc = check_pool_layer(pool, layer);
  if (rc) return rc;
  if ((rc = validate_batch(b, true))) return rc;
  const int d = pool->desc.head_dim, hkv = pool->desc.num_kv_heads;
  if (hq < 1 || hq % hkv) return fail(MUX_ERR_UNSUPPORTED, "num_q_heads must be a positive multiple of Hkv");
  const int g = hq / hkv;
  if (g > 16) return fail(MUX_ERR_UNSUPPORTED, "GQA group size > 16 not supported");
  if (!q || !o) return fail(MUX_ERR_INVALID_ARG, "q/o NULL");
  if (o_dtype != MUX_DTYPE_BF16 && o_dtype != MUX_DTYPE_F32) return fail(MUX_ERR_INVALID_ARG, "bad o_dtype");
  if (reinterpret_cast<uintptr_t>(q) & 15) return fail(MUX_ERR_INVALID_ARG, "q must be 16-byte aligned");
  if (num_sms <= 0) num_sms = device_sm_count();
  if (num_splits <= 0) num_splits = mux_decode_num_splits(b->num_seqs, hkv, d, b->h_kv_len, b->max_kv, num_sms);
  if (num_splits > 1) {
    if (!ws || ws_bytes < mux_decode_workspace_bytes(b->num_seqs, hq, d, num_splits))
      return fail(MUX_ERR_WORKSPACE, "decode workspace missing or too small");
  }
  if ((rc = pool_tmaps(pool))) return rc;
  DecodeParams prm{};
  prm.q = static_cast<const uint16_t*>(q);
  prm.o = o;
  prm.lse = lse;
  const size_t rows = static_cast<size_t>(b->num_seqs) * hq * num_splits;
  prm.part_o = static_cast<float*>(ws);
  prm.part_m = num_splits > 1 ? prm.part_o + rows * d : nullptr;
  prm.part_l = num_splits > 1 ? prm.part_m + rows : nullptr;
  prm.kv_len = b->kv_len;
  prm.page_indptr = b->page_indptr;
  prm.page_ids = b->page_ids;
  prm.num_splits = num_splits;
  {
    const int max_pages = (b->max_kv + kPage - 1) / kPage;
    prm.pages_per_split = std::max(1, (max_pages + num_splits - 1) / num_splits);
  }
  prm.hq = hq;
  prm.hkv = hkv;
  prm.g = g;
  prm.page_row0 = layer * pool->desc.num_pages;
  prm.o_f32 = o_dtype == MUX_DTYPE_F32;
  prm.scale_log2 = scale * 1.4426950408889634f;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (d == 128) return g <= 8 ? launch_decode<128, 1>(pool, prm, b->num_seqs, st, num_sms)
                              : launch_decode<128, 2>(pool, prm, b->num_seqs, st, num_sms);
  return g <= 8 ? launch_decode<64, 1>(pool, prm, b->num_seqs, st, num_sms)
                : launch_decode<64, 2>(pool, prm, b->num_seqs, st, num_sms);
}
}  // namespace mux
