#include <algorithm>
#include <cstdlib>
// Stage (3) streaming: the persistent, warp-specialised residual / bonus sampler (sm_100a, fp32 rows, V % 8 == 0).
//
// persist_stream_kernel, one CTA per SM, programmatic dependent of the selector:
//   warp 16     producer: takes work items (request b, chunk c) from a global counter and issues 1-D bulk copies on
//               the TMA engine (cp.async.bulk + mbarrier complete_tx) of the chunk of the row to resample from —
//               p[b][a_b] and q[b][a_b] after a rejection, p[b][w_b] for the bonus — into a 3-stage ring;
//   warps 0..15 consumers: fold the staged chunk into the sampling-contract segment sums (lane: 8 elements left to
//               right; segment: xor butterfly), 2 segments each;
//   warp 17     publisher: folds warp and chunk sums, stores them, counts chunks on per-request counters;
//   then every warp: the descent T = u*mass -> chunk -> warp -> segment -> lane -> element for the requests it owns,
//               once their chunks are counted, re-reading only the one 1024-element warp run that holds the sample.
// Speculative variant (SPEC, tetris_resample_spec_f32): the rows of requests whose FIRST drafted token is rejected —
// p[b][0] and q[b][0], whatever the selection decides as long as w_b >= 1 — do not depend on the selection, so the
// kernel computes that set itself (verify_token at position 0, the accept test's arithmetic: each CTA evaluates its
// share and appends the rejected requests to a global list, except the first, which it streams itself at once) and
// streams it while the selector is still running (phase A, before griddepcontrol.wait; producers take list items as
// entries appear); a planner warp (18) then lists every other request from the selector's row info (phase B).  A
// phase-A request whose window turns out to be 0 is streamed again in phase B (its phase-A sums live in a separate
// region and are discarded).  Both phases take items one at a time with two of look-ahead (claims of 4 streamed 5 %
// slower here).
// HBM is touched once per streamed element; the descent's re-read is 4-8 KB per request.
#include "common.cuh"
#include "fused_select.cuh"
#include "launch.h"

namespace tetris {

// Element form of the streamed rows: fp32 probabilities (3 stages of 64 KB), or bf16 logits + per-row lse (the logits
// contract, tetris_b200.h; 6 stages of 32 KB: the same bytes in flight per SM)
template <bool BF>
#ifndef TETRIS_F32_STAGES  // A/B experiments only
#define TETRIS_F32_STAGES 3
#endif
struct Elem {
  using T = float;
  static constexpr int kBytes = 4;
  static constexpr int kStages = TETRIS_F32_STAGES;
};
template <>
struct Elem<true> {
  using T = uint16_t;
  static constexpr int kBytes = 2;
  static constexpr int kStages = 6;
};
constexpr int kMaxStages = 6;
constexpr int kConsumerWarps = 16;                         // 2 segments of the staged chunk each
constexpr int kSegsPerChunk = kChunkElems / kSegElems;     // 32
constexpr int kSegsPerConsumer = kSegsPerChunk / kConsumerWarps;
constexpr int kProducerWarp = kConsumerWarps;
constexpr int kPublisherWarp = kConsumerWarps + 1;
constexpr int kPersistThreads = (kConsumerWarps + 2) * 32;
constexpr int kRing = 64;
constexpr size_t kPersistSmem = 192 * 1024;  // dynamic: the stage ring (p + q chunk per stage)
template <bool BF>
__host__ __device__ constexpr size_t stage_row_bytes() { return (size_t)kChunkElems * Elem<BF>::kBytes; }
template <bool BF>
__host__ __device__ constexpr size_t stage_bytes() { return 2 * stage_row_bytes<BF>(); }
static_assert(Elem<false>::kStages * stage_bytes<false>() <= kPersistSmem, "fp32 ring");
static_assert(Elem<true>::kStages * stage_bytes<true>() == kPersistSmem, "bf16 ring");



// diagnostics (tools/dbg_stream.py): per-CTA %globaltimer stamps, a no-op unless a debug buffer is registered
__device__ __forceinline__ void gstamp(const StreamArgs& a, int slot) {
  if (a.dbg) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[64 + 16 * blockIdx.x + slot] = t;
    a.dbg[64 + 16 * gridDim.x + 16 * blockIdx.x + slot] = clock64();  // SM cycles, for in-CTA phase lengths
  }
}

struct StageMeta {
  int b, c, res, phase;  // phase 1: speculative (phase A) item
  float lp, lq;          // logits form: the lse of the p / q row
};

constexpr int kSpecMaxR = 4096;  // speculative variant: requests per call (lists in shared memory)

struct SpecShared {
  uint32_t inA[kSpecMaxR / 32];  // phase-A set (first drafted token rejected), copied by the planner
  uint16_t listB[kSpecMaxR];
  uint64_t listB_ready;          // mbarrier: the planner warp has written listB
  int countA, countB;
  int own;                       // the phase-A request this CTA streams itself (-1: none)
};

struct PersistShared {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  uint64_t ring_full[kRing];
  uint64_t ring_free[kRing];
  StageMeta meta[kMaxStages];
  StageMeta ring_meta[kRing];
  double ring_g[kRing][kSegsPerChunk];  // segment sums of each published chunk
};

// A lane's 8 staged elements as fp32 probabilities: an fp32 stage (two 16-byte halves, swizzled), or 8 bf16 logits
// (one 16-byte word; consecutive lanes read consecutive words, conflict-free) through the logits contract.
template <bool BF>
__device__ __forceinline__ void stage_lane(const uint8_t* row, int off, int lane, const ExpRow& er, float (&v)[8]) {
  if (BF) {
#ifdef TETRIS_EXP_FAKE  // A/B experiment only: the staged bf16 values as probabilities (no exp)
    const uint4 raw = *reinterpret_cast<const uint4*>(row + (size_t)off * 2);
    const uint32_t wv[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float((wv[i] << 16) & 0x7fffffffu);
      v[2 * i + 1] = __uint_as_float(wv[i] & 0x7fff0000u);
    }
#else
    prob8_from_bf16(*reinterpret_cast<const uint4*>(row + (size_t)off * 2), er, v);
#endif
  } else {
    lds8_swz(reinterpret_cast<const float*>(row) + off, lane, v);
  }
}

// Segment sum (lane fold + xor butterfly) of the staged segment at chunk offset `off0` (element e0 of the row).
template <bool BF>
__device__ __forceinline__ double consume_segment(const uint8_t* __restrict__ sp, const uint8_t* __restrict__ sq,
                                                  bool res, int64_t e0, int off0, int V, int lane, float lp, float lq) {
#ifdef TETRIS_CONSUME_NOP  // A/B experiment only: the pipeline without the consumers' arithmetic
  return 0.0;
#endif
  const int off = off0 + lane * kLaneElems;
  double w[8];
  if (e0 + lane * kLaneElems < V) {
    float pv[8];
    stage_lane<BF>(sp, off, lane, BF ? exp_row(lp) : ExpRow{}, pv);
    if (res) {
      float qv[8];
      stage_lane<BF>(sq, off, lane, BF ? exp_row(lq) : ExpRow{}, qv);
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = BF ? w_res_pos(pv[i], qv[i]) : w_res32(pv[i], qv[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = BF ? widen_pos_normal(pv[i]) : w_plain32(pv[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = 0.0;
  }
  return fold8(w);  // the lane's sum; the caller runs the segment butterflies (interleaved over its segments)
}

// A lane's 8 row elements from global memory as fp32 probabilities (zeros past the row end)
template <bool BF>
__device__ __forceinline__ void row_lane(const void* row, int64_t e, int V, float lse, float (&v)[8]) {
  if (BF) {
    if (e < V) {
      uint4 raw;
      asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
          : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w)
          : "l"(reinterpret_cast<const uint16_t*>(row) + e));
      prob8_from_bf16(raw, exp_row(lse), v);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
    }
  } else {
    load_lane<float, true>(reinterpret_cast<const float*>(row), e, V, v);
  }
}

// Diagnostics for tools/micro/descent.cu only (-DTETRIS_DESCENT_PROBE): clock64 at points of the descent, lane 0.
#ifdef TETRIS_DESCENT_PROBE
__device__ long long g_probe[4096][8];
#define DESCENT_PROBE(i)                                                                                          \
  do {                                                                                                             \
    if ((threadIdx.x & 31) == 0)                                                                                   \
      g_probe[(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) & 4095][i] = clock64();                         \
  } while (0)
#else
#define DESCENT_PROBE(i) \
  do {                   \
  } while (0)
#endif

// descent below the warp level, reading the warp run from global memory (all 32 lanes, T uniform)
template <bool RES, bool BF>
__device__ int descend_global(const void* __restrict__ P, const void* __restrict__ Q, int64_t e0, int V, int lane,
                              double T, float lp, float lq) {
  double G[kWarpSegs];
  float pv[kWarpSegs][8], qv[kWarpSegs][8];
#pragma unroll
  for (int s = 0; s < kWarpSegs; ++s) {
    row_lane<BF>(P, e0 + s * kSegElems + lane * kLaneElems, V, lp, pv[s]);
    if (RES) row_lane<BF>(Q, e0 + s * kSegElems + lane * kLaneElems, V, lq, qv[s]);
  }
#ifdef TETRIS_DESCENT_PROBE
  if (pv[0][0] == -1.f) G[0] = 0.0;  // the loads are in
#endif
  DESCENT_PROBE(4);
#pragma unroll
  for (int s = 0; s < kWarpSegs; ++s) {
    double wl[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) wl[i] = RES ? w_res((double)pv[s][i], (double)qv[s][i]) : w_plain((double)pv[s][i]);
    G[s] = fold8(wl);
  }
  // the four segments' butterflies level by level (seg_sum's arithmetic; the shuffle latencies overlap)
#pragma unroll
  for (int mm = 1; mm < 32; mm <<= 1) {
    double o[kWarpSegs];
#pragma unroll
    for (int s = 0; s < kWarpSegs; ++s) o[s] = __shfl_xor_sync(kFull, G[s], mm);
#pragma unroll
    for (int s = 0; s < kWarpSegs; ++s) G[s] = G[s] + o[s];
  }
  DESCENT_PROBE(5);
  const int s = seq_find(G, kWarpSegs, T);
  if (s < 0) return -1;
  double w[8];  // the chosen segment's weights, recomputed from the loaded lanes (identical arithmetic)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float pp = pv[0][i], qq = RES ? qv[0][i] : 0.f;
#pragma unroll
    for (int ss = 1; ss < kWarpSegs; ++ss) {
      pp = (s == ss) ? pv[ss][i] : pp;
      if (RES) qq = (s == ss) ? qv[ss][i] : qq;
    }
    w[i] = RES ? w_res((double)pp, (double)qq) : w_plain((double)pp);
  }
  double lv[5];
  lv[0] = fold8(w);
  double x = lv[0];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    x = x + __shfl_xor_sync(kFull, x, 1 << t);
    lv[t + 1] = x;
  }
  int g = 0;
#pragma unroll
  for (int t = 4; t >= 0; --t) {
    const double L = __shfl_sync(kFull, lv[t], g);
    const double Rr = __shfl_sync(kFull, lv[t], g + (1 << t));
    if (!(L > T || Rr == 0.0)) {
      T = T - L;
      g += 1 << t;
    }
  }
  DESCENT_PROBE(6);
  double Tl = T;
  const int li_own = seq_find(w, 8, Tl);
  const int li = __shfl_sync(kFull, li_own, g);
  if (li < 0) return -1;
  return (int)(e0 + s * kSegElems + g * kLaneElems + li);
}

// Rows of at most kSegSumMaxChunks chunks publish the 32 segment sums of every chunk in place of the 8 warp sums (the
// consumers' values, folded by the publisher in the same order): the descent then knows the segment before it reads the
// row and re-reads that one segment (8 elements per lane) instead of the warp run's four.
constexpr int kSegSumMaxChunks = 4;
constexpr int kChunkSegs = kChunkWarps * kWarpSegs;  // 32
static_assert(kChunkSegs == 32, "one segment sum per lane");

// descent below the segment level: G = the chosen warp run's four segment sums (as published)
template <bool RES, bool BF>
__device__ int descend_seg(const void* __restrict__ P, const void* __restrict__ Q, int64_t e0, int V, int lane,
                           double T, float lp, float lq, const double (&G)[kWarpSegs]) {
  const int s = seq_find(G, kWarpSegs, T);
  if (s < 0) return -1;
  float pv[8], qv[8];
  row_lane<BF>(P, e0 + s * kSegElems + lane * kLaneElems, V, lp, pv);
  if (RES) row_lane<BF>(Q, e0 + s * kSegElems + lane * kLaneElems, V, lq, qv);
#ifdef TETRIS_DESCENT_PROBE
  if (pv[0] == -1.f) T = 0.0;  // the loads are in
#endif
  DESCENT_PROBE(4);
  DESCENT_PROBE(5);
  double w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = RES ? w_res((double)pv[i], (double)qv[i]) : w_plain((double)pv[i]);
  double lv[5];
  lv[0] = fold8(w);
  double x = lv[0];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    x = x + __shfl_xor_sync(kFull, x, 1 << t);
    lv[t + 1] = x;
  }
  int g = 0;
#pragma unroll
  for (int t = 4; t >= 0; --t) {
    const double L = __shfl_sync(kFull, lv[t], g);
    const double Rr = __shfl_sync(kFull, lv[t], g + (1 << t));
    if (!(L > T || Rr == 0.0)) {
      T = T - L;
      g += 1 << t;
    }
  }
  DESCENT_PROBE(6);
  double Tl = T;
  const int li_own = seq_find(w, 8, Tl);
  const int li = __shfl_sync(kFull, li_own, g);
  if (li < 0) return -1;
  return (int)(e0 + s * kSegElems + g * kLaneElems + li);
}

// Descent for request b after every chunk sum is published (one warp): the chunk and warp sums of all chunks are
// fetched in one round trip (lane l holds sums l, l+32, ...), then the one warp run holding the sample is re-read.
template <bool BF>
__device__ void finalize_request(const StreamArgs& a, int b, bool res, int lane, const double* chunk_sums,
                                 const double* warp_sums) {
  DESCENT_PROBE(0);
  const int nch = a.nch;
  const long long prow = __ldcg(a.prow + (int64_t)b * a.row_stride);
  const long long qrow = a.qrow ? __ldcg(a.qrow + (int64_t)b * a.row_stride) : -1;
  const float lp = BF ? a.lse_p[prow] : 0.f;
  const float lq = (BF && qrow >= 0) ? a.lse_q[qrow] : 0.f;
  const double* cs = chunk_sums + (int64_t)b * nch;
  const bool segm = nch <= kSegSumMaxChunks;  // warp_sums holds segment sums (32 per chunk)
  const double* ws = warp_sums + (int64_t)b * nch * (segm ? kChunkSegs : kChunkWarps);
  // nch <= 16: every sum the descent needs in ONE round trip — the chunk sums (lane c holds chunk c) and the
  // nch * 8 warp sums (lane l holds sums l, l + 32, l + 64, l + 96: chunk c's eight are register c / 4, lanes
  // 8 (c % 4) .. + 7).  Larger rows: chunk sums (two per lane) first, the chosen chunk's warp sums second.
  const bool one_trip = nch <= 16;
  double wv[4];
  double s_lo = lane < nch ? __ldcg(cs + lane) : 0.0;
  double s_hi = lane + 32 < nch ? __ldcg(cs + lane + 32) : 0.0;
  if (one_trip) {  // (segment sums: lane l holds segment l of chunk x in wv[x])
#pragma unroll
    for (int x = 0; x < 4; ++x)
      wv[x] = lane + 32 * x < nch * (segm ? kChunkSegs : kChunkWarps) ? __ldcg(ws + lane + 32 * x) : 0.0;
  }
  // accepted-prefix tokens of the compacted stream: every load of the descent's first round trip goes out together
  // (the sums above, the request's counts and uniform, its first 32 drafted tokens)
  int acc = 0, off = 0, end = 0, d0 = 0;
  if (a.accepted) {
    acc = __ldcg(a.accepted + b);
    off = __ldcg(a.offsets + b);
    end = __ldcg(a.offsets + b + 1);
    d0 = lane < a.k ? __ldg(a.d + (int64_t)b * a.k + lane) : 0;
  }
  const double u = __ldg(a.u + b);
  if (a.accepted)
    for (int j = lane; j < acc && off + j < end; j += 32) a.tokens[off + j] = j < 32 ? d0 : a.d[(int64_t)b * a.k + j];
  uint32_t bad = 0;
  if (!(u >= 0.0 && u < 1.0)) bad |= TETRIS_ST_BAD_UNIFORM;
  DESCENT_PROBE(1);
  // mass = chunk sums folded left to right (every lane holds the same value)
  double mass = 0.0;
  for (int c = 0; c < nch; ++c) mass = mass + __shfl_sync(kFull, c < 32 ? s_lo : s_hi, c & 31);
  int tok = -1;
#ifndef TETRIS_VERDICT_STAMP
  if (lane == 0 && b == (int)blockIdx.x) gstamp(a, 15);  // diagnostics: the first round trip is in
#endif
  if (mass > 0.0) {
    double T = u * mass;
    // chunk level (left to right), then warp level of the chosen chunk
    double P = 0.0;
    int cc = -1, last_pos = -1;
    auto step = [&](int c, double v) {
      if (v > 0.0) last_pos = c;
      if (cc < 0) {
        const double Pn = P + v;
        if (Pn > T) {
          T = T - P;
          cc = c;
        }
        P = Pn;
      }
    };
    for (int c = 0; c < nch; ++c) step(c, __shfl_sync(kFull, c < 32 ? s_lo : s_hi, c & 31));
    if (cc < 0) {
      cc = last_pos;
      T = __longlong_as_double(0x7ff0000000000000ll);
    }
    DESCENT_PROBE(2);
    // the 8 warp sums of the chosen chunk (from lane cc's registers, or lanes 0..7 load them, then broadcast)
    double Wc[kChunkWarps];
    double sg = 0.0;  // segment mode: lane l holds segment l of the chosen chunk
    if (segm) {
      const int c0 = cc < 0 ? 0 : cc;
      sg = c0 == 0 ? wv[0] : c0 == 1 ? wv[1] : c0 == 2 ? wv[2] : wv[3];
      // the warp sums, folded as the publisher folds them (four segments left to right), lanes 0..7
      double xw = 0.0;
#pragma unroll
      for (int q = 0; q < kWarpSegs; ++q) xw = xw + __shfl_sync(kFull, sg, (lane & 7) * kWarpSegs + q);
#pragma unroll
      for (int w = 0; w < kChunkWarps; ++w) Wc[w] = __shfl_sync(kFull, xw, w);
    } else if (one_trip) {
      const int c0 = cc < 0 ? 0 : cc, xr = c0 >> 2;
      const double src = xr == 0 ? wv[0] : xr == 1 ? wv[1] : xr == 2 ? wv[2] : wv[3];
#pragma unroll
      for (int w = 0; w < kChunkWarps; ++w) Wc[w] = __shfl_sync(kFull, src, 8 * (c0 & 3) + w);
    } else {
      const double wl = (cc >= 0 && lane < kChunkWarps) ? __ldcg(ws + (int64_t)cc * kChunkWarps + lane) : 0.0;
#pragma unroll
      for (int w = 0; w < kChunkWarps; ++w) Wc[w] = __shfl_sync(kFull, wl, w);
    }
    const int ww = seq_find(Wc, kChunkWarps, T);
    DESCENT_PROBE(3);
    double G[kWarpSegs];
#pragma unroll
    for (int q = 0; q < kWarpSegs; ++q) G[q] = __shfl_sync(kFull, sg, ((ww < 0 ? 0 : ww) * kWarpSegs + q) & 31);
    if (cc >= 0 && ww >= 0) {
      const int64_t e0 = (int64_t)cc * kChunkElems + ww * kWarpElems;
      const void* Pr = BF ? (const void*)(a.zp + prow * (int64_t)a.V) : (const void*)(a.p + prow * (int64_t)a.V);
      const void* Qr = !res ? nullptr
                       : BF ? (const void*)(a.zq + qrow * (int64_t)a.V) : (const void*)(a.q + qrow * (int64_t)a.V);
      if (segm)
        tok = res ? descend_seg<true, BF>(Pr, Qr, e0, a.V, lane, T, lp, lq, G)
                  : descend_seg<false, BF>(Pr, nullptr, e0, a.V, lane, T, lp, lq, G);
      else
        tok = res ? descend_global<true, BF>(Pr, Qr, e0, a.V, lane, T, lp, lq)
                  : descend_global<false, BF>(Pr, nullptr, e0, a.V, lane, T, lp, lq);
    }
  }
  DESCENT_PROBE(7);
  if (tok < 0) bad |= TETRIS_ST_DEGENERATE;
  if (lane == 0) {
    a.out_idx[b] = tok;
    if (a.mass_out) a.mass_out[b] = mass;
    if (a.accepted && off + acc < end) a.tokens[off + acc] = tok;  // the sample is emitted unless the cap cut it
    set_status(a.status, bad);
  }
}

// Producer helper: one item (request b, chunk c) of rows prow / qrow (qrow < 0: plain) into stage t; logits form: lp /
// lq are the rows' lse (loaded by the caller with the row indices, one item ahead).
template <bool BF>
__device__ __forceinline__ void issue_item(const StreamArgs& a, PersistShared& sh, uint8_t* stage_mem, int t, int b,
                                           int c, long long prow, long long qrow, int phase, uint64_t pol, float lp,
                                           float lq) {
  constexpr int S = Elem<BF>::kStages;
  const bool res = qrow >= 0;
  const int s = t % S;
  if (t >= S) mbar_wait(&sh.empty[s], (uint32_t)(((t / S) & 1) ^ 1u));
  const int n = min(kChunkElems, a.V - c * kChunkElems);
  const uint32_t bytes = (uint32_t)n * Elem<BF>::kBytes;
  sh.meta[s] = StageMeta{b, c, res ? 1 : 0, phase, lp, lq};
  uint8_t* sp = stage_mem + s * stage_bytes<BF>();
  const uint8_t* P = BF ? (const uint8_t*)a.zp : (const uint8_t*)a.p;
  const uint8_t* Q = BF ? (const uint8_t*)a.zq : (const uint8_t*)a.q;
  const int64_t eb = Elem<BF>::kBytes;
  mbar_arrive_expect_tx(&sh.full[s], res ? 2 * bytes : bytes);
  bulk_g2s_stream(sp, P + (prow * (int64_t)a.V + (int64_t)c * kChunkElems) * eb, bytes, &sh.full[s], pol);
  if (res)
    bulk_g2s_stream(sp + stage_row_bytes<BF>(), Q + (qrow * (int64_t)a.V + (int64_t)c * kChunkElems) * eb, bytes,
                    &sh.full[s], pol);
}

// Producer helper: stream the items (list[y], c), y < count, c < nch, taken one at a time from `work` in order with
// two items of look-ahead on the counter and one on the row lookup — the plain producer's schedule over a list.
// rows(b, prow, qrow) gives the rows of request b.  Returns the next stage index.
// Deeper producer schedule for the logits form (its items are half as many bytes, so the claim / row-lookup round
// trips must overlap more): C claims on the work counter and L row lookups in flight, kept in shift registers.
// req(i) -> request of item i; rows(b, prow, qrow, lse_p, lse_q).  Returns the next stage index.
template <bool BF, int L, int C, typename Req, typename Rows>
__device__ int stream_deep(const StreamArgs& a, PersistShared& sh, uint8_t* stage_mem, int t, long long total,
                           unsigned long long* work, int phase, uint64_t pol, Req req, Rows rows) {
  constexpr int D = L + C;
  long long ci[D], pr[D], qr[D];
  float lp[D], lq[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    ci[d] = (long long)atomicAdd(work, 1ull);
    pr[d] = 0;
    qr[d] = -1;
    lp[d] = lq[d] = 0.f;
  }
#pragma unroll
  for (int d = 0; d < L; ++d)
    if (ci[d] < total) rows(req(ci[d]), pr[d], qr[d], lp[d], lq[d]);
  for (;;) {
    const long long i = ci[0];  // one thread's claims increase: past the end, all later ones are too
    if (i >= total) break;
    const long long prow = pr[0], qrow = qr[0];
    const float l0 = lp[0], l1 = lq[0];
#pragma unroll
    for (int d = 0; d < D - 1; ++d) {
      ci[d] = ci[d + 1];
      pr[d] = pr[d + 1];
      qr[d] = qr[d + 1];
      lp[d] = lp[d + 1];
      lq[d] = lq[d + 1];
    }
    ci[D - 1] = (long long)atomicAdd(work, 1ull);
    if (ci[L - 1] < total) rows(req(ci[L - 1]), pr[L - 1], qr[L - 1], lp[L - 1], lq[L - 1]);
    issue_item<BF>(a, sh, stage_mem, t++, req(i), (int)(i % a.nch), prow, qrow, phase, pol, l0, l1);
  }
  return t;
}

template <bool BF, typename Rows>
__device__ int stream_list(const StreamArgs& a, PersistShared& sh, uint8_t* stage_mem, int t, const uint16_t* list,
                           int count, unsigned long long* work, int phase, uint64_t pol, Rows rows) {
  const int nch = a.nch;
  const long long total = (long long)count * nch;
  if (BF) return stream_deep<BF, 3, 3>(a, sh, stage_mem, t, total, work, phase, pol,
                                       [&](long long i) { return (int)list[i / nch]; }, rows);
  long long i_next = (long long)atomicAdd(work, 1ull);
  long long i_next2 = (long long)atomicAdd(work, 1ull);
  long long pn = 0, qn = -1;
  float lpn = 0.f, lqn = 0.f;
  if (i_next < total) rows((int)list[i_next / nch], pn, qn, lpn, lqn);
  for (;;) {
    const long long i = i_next;
    const long long prow = pn, qrow = qn;
    const float lp = lpn, lq = lqn;
    i_next = i_next2;
    if (i >= total) break;
    i_next2 = (long long)atomicAdd(work, 1ull);
    if (i_next < total) rows((int)list[i_next / nch], pn, qn, lpn, lqn);
    issue_item<BF>(a, sh, stage_mem, t++, (int)list[i / nch], (int)(i % nch), prow, qrow, phase, pol, lp, lq);
  }
  return t;
}

// ---- the selection fused into the sampler's launch (FUSED variant, B_sel * k <= kFusedMaxCells) ------------------
// fused_select.cuh's rank selection on all 576 threads, with this kernel's per-row epilogue: verify_token's first
// rejection among the selected positions (accept_model.py:309-313, sim_engine.py:397-401) from verdicts gathered in
// the selection's first round trip, the row to resample from, and the compaction offsets.  Every CTA counts itself in
// (ctl[0]) once its rows are written; the producers poll per-request ready words, the descents wait for the scans
// (ctl[1]).  The scans — win_offsets / PolicyStats (selector.py:150-170) and the compaction offsets over every CTA's
// published rows — are run in the last CTA to count itself in: by its extra scanner warp while the other warps stream
// (B_sel <= 32 * kFusedMaxRpt), else by its 16 consumer warps before they consume (global memory only: the prologue's
// shared scratch is the stage ring by then).
template <bool BF>
__device__ void fused_scans(const StreamArgs& a, int pt, int nt) {
  const FusedSel& f = a.fs;
  __shared__ long long s_tmp[33];
  if (pt == 0) gstamp(a, 11);
  int wr[kFusedMaxRpt], nr[kFusedMaxRpt];
  fused_load_windows(f, pt, nt, wr);  // both scans' inputs in one round trip
  const int R = a.R, rpl = (R + nt - 1) / nt, l0 = pt * rpl;
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i) {
    const int lr = l0 + i;
    nr[i] = (i < rpl && lr < R) ? __ldcg(f.accepted + lr) + 1 : 0;
    if (f.cap && i < rpl && lr < R) nr[i] = min(nr[i], max(__ldg(f.cap + lr), 0));
  }
  fused_win_scan(f, a.k, pt, nt, s_tmp, wr);
  long long my = 0;
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i) my += nr[i];
  long long etot;
  long long eex = fused_excl_scan<long long>(my, s_tmp, etot, pt, nt);
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i) {
    const int lr = l0 + i;
    if (i < rpl && lr < R) {
      f.offsets[lr] = (int32_t)eex;
      eex += nr[i];
    }
  }
  if (pt == 0) f.offsets[R] = (int32_t)etot;
  fused_release_done(f, pt, nt);
  if (pt == 0) gstamp(a, 12);
}

// The own cells' accept verdicts (verify_token, accept_model.py:309-313) by ONE warp — the publisher's, idle until
// streaming starts — while the other 17 warps build keys and ranks: its two dependent round trips (drafted tokens
// and uniforms, then the p / q gathers) overlap the selection instead of stalling it.  Verdict byte: bit0 accept,
// bit1 drafted token outside the vocabulary, bit2 uniform outside [0, 1).  4 cells per lane per round.
template <bool BF>
__device__ void fused_verdicts(const StreamArgs& a, const FusedView& v, int lane) {
  const FusedSel& f = a.fs;
  const int k = a.k, G = gridDim.x, g = blockIdx.x;
  for (int c0 = 0; c0 < v.ncell; c0 += 128) {
    int64_t ce[4];
    int t[4];
    double u[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int c = c0 + lane + 32 * x;
      ce[x] = -1;
      if (c < v.ncell) {
        const int oi = c / k, j = c - oi * k, lr = g + oi * G - f.row0;
        if (lr >= 0 && lr < a.R) ce[x] = (int64_t)lr * k + j;
      }
      t[x] = ce[x] >= 0 ? __ldg(a.d + ce[x]) : 0;
      u[x] = ce[x] >= 0 ? __ldg(f.u_acc + ce[x]) : 0.0;
    }
    double m[4], sq[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      m[x] = sq[x] = 0.0;
      if (ce[x] >= 0 && t[x] >= 0 && t[x] < a.V) {
        const int64_t e = ce[x], lr = e / k, prow = lr * (k + 1) + (e - lr * k);
        m[x] = gather_p(a, prow, t[x]);
        sq[x] = gather_q(a, e, t[x]);
      }
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int c = c0 + lane + 32 * x;
      if (c >= v.ncell) continue;
      uint8_t vb = 0;
      if (ce[x] >= 0) {
        vb = (u[x] >= 0.0 && u[x] < 1.0) ? 0 : 4;
        if (t[x] < 0 || t[x] >= a.V)
          vb |= 2;
        else
          vb |= ((sq[x] <= m[x]) || (u[x] < m[x] / sq[x])) ? 1 : 0;
      }
      v.verd[c] = vb;
    }
  }
}

template <bool BF>
__device__ uint32_t fused_select(const StreamArgs& a, uint8_t* smem) {
  const FusedSel& f = a.fs;
  const int tid = threadIdx.x, NT = blockDim.x, G = gridDim.x, g = blockIdx.x, k = a.k;
  const int NP = NT - 32;  // the selection's participants: warps 0 .. 16; warp 17 gathers the verdicts
  const FusedView v = fused_view(f, k, smem);
  __shared__ uint32_t s_epoch;
  // this launch's epoch (the previous grid is complete): loaded beside the scores, published after them (the barriers
  // before phase 3 make it visible)
  const uint32_t ep = tid == 0 ? (uint32_t)__ldcg(f.ctl + 2) : 0u;
  if (tid >= NP) {
    fused_verdicts<BF>(a, v, tid & 31);
#ifdef TETRIS_VERDICT_STAMP  // diagnostics only: slot 15 = the verdict warp done (instead of the descent's sums)
    if ((tid & 31) == 0) gstamp(a, 15);
#endif
  } else {
    fused_stage(f, k, v, tid, NP);
    if (tid == 0) s_epoch = ep + 1u;
    fused_bar(NP);
    if (tid == 0) gstamp(a, 8);
    fused_keys(f, k, v, tid, NP, a.status);
    fused_bar(NP);
    if (tid == 0) gstamp(a, 9);
    fused_ranks(k, v, tid, NP);
#ifdef TETRIS_FUSED_TWICE  // A/B timing only (wrong results): each phase again, warm, stamped into slots 11 / 12
    fused_bar(NP);
    if (tid == 0) gstamp(a, 10);
    fused_keys(f, k, v, tid, NP, a.status);
    fused_bar(NP);
    if (tid == 0) gstamp(a, 11);
    fused_ranks(k, v, tid, NP);
    fused_bar(NP);
    if (tid == 0) gstamp(a, 12);
#endif
  }
  __syncthreads();
  if (tid == 0) gstamp(a, 10);
  const uint32_t epoch = s_epoch;
  // phase 3: the own rows' windows, first rejection (sim_engine.py:397-401), row to resample from
  for (int oi = tid; oi < v.nown; oi += NT) {
    const int r = g + oi * G;
    const int w = fused_window(f, k, v, oi);
    f.windows[r] = w;
    const int lr = r - f.row0;
    if (lr >= 0 && lr < a.R) {
      uint32_t vbad = 0;
      int acc = w;
      for (int j = 0; j < w; ++j) {
        const uint8_t vb = v.verd[oi * k + j];
        vbad |= (vb & 2 ? TETRIS_ST_BAD_TOKEN : 0u) | (vb & 4 ? TETRIS_ST_BAD_UNIFORM : 0u);
        if (!(vb & 1)) {
          acc = j;
          break;
        }
      }
      f.accepted[lr] = acc;
      f.rowinfo[2 * (int64_t)lr] = (long long)lr * (k + 1) + acc;              // residual row / bonus row of p
      f.rowinfo[2 * (int64_t)lr + 1] = acc < w ? (long long)lr * k + acc : -1;  // draft row (residual only)
      if (BF) {
        f.rowlse[2 * (int64_t)lr] = __ldg(a.lse_p + (int64_t)lr * (k + 1) + acc);
        f.rowlse[2 * (int64_t)lr + 1] = acc < w ? __ldg(a.lse_q + (int64_t)lr * k + acc) : 0.f;
      }
      // the request's ready word: this launch's epoch + both rows, in one 8-byte store the producers poll
      __stcg(f.ready + lr, fused_ready_word(epoch, (long long)lr * (k + 1) + acc, acc < w ? (long long)lr * k + acc : -1));
      set_status(a.status, vbad);
    }
  }
  // the stage ring is written by the TMA engine (async proxy) after these generic shared-memory accesses
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  return epoch;  // this launch's epoch, for the producer's ready-word polls (no reload of ctl[2])
}

template <bool SPEC, bool BF, bool FUSED = false>
__global__ void __launch_bounds__(kPersistThreads + ((SPEC || FUSED) ? 32 : 0), 1)
    persist_stream_kernel(const StreamArgs a) {
  constexpr int kStages = Elem<BF>::kStages;
  extern __shared__ __align__(128) uint8_t stage_mem[];
  __shared__ PersistShared sh;
  __shared__ SpecShared sx;  // speculative variant only
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nch = a.nch, k = a.k, R = a.R;
  const long long total = (long long)R * nch;
  const int G = gridDim.x;
  // dynamic work distribution: items (request b, chunk c) are handed out in order from one global counter, so the
  // SMs stream neighbouring chunks at any moment (DRAM locality, like a round robin) and an SM that drew more
  // residual (p + q) items simply takes fewer items (balance).  The counter sits beside the grid barrier and is reset
  // by the barrier's last arrival.
  unsigned long long* work = reinterpret_cast<unsigned long long*>(a.grid_bar + 2);
  unsigned long long* work_a = reinterpret_cast<unsigned long long*>(a.grid_bar + 4);  // speculative phase A

  if (tid == 0) {
    gstamp(a, 0);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], kConsumerWarps);
    }
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&sh.ring_full[r], kConsumerWarps);
      mbar_init(&sh.ring_free[r], 1);
    }
    if (SPEC) mbar_init(&sx.listB_ready, 1);
    mbar_fence_init();
  }
  if (SPEC) {
    // This CTA's share of the phase-A set (requests b = blockIdx.x + x * G, one thread each): verify_token at drafted
    // position 0 (accept_model.py:309-313, the same arithmetic as the selector's accept test).  A rejected request
    // is appended to the global phase-A list (entry b + 1; 0 = not written yet) and its bit set in the global set;
    // then the CTA counts its requests as processed (release).  Every CTA starts streaming as soon as list entries
    // appear — no CTA waits for the whole set.
    const int nmine = blockIdx.x < R ? (R - 1 - (int)blockIdx.x) / G + 1 : 0;  // <= 32 (host-checked)
    if (warp == 0) {
      const int b = blockIdx.x + lane * G;
      bool rej = false;
      if (lane < nmine) {
        const bool drafted = (a.len ? a.len[b] : k) >= 1;
        const int t = drafted ? a.d[(int64_t)b * k] : 0;
        const double u = drafted ? a.u_acc[(int64_t)b * k] : 0.0;
        if (drafted) {
          if (t < 0 || t >= a.V) {
            rej = true;
          } else {
            const double s = gather_q(a, (int64_t)b * k, t);
            const double m = gather_p(a, (int64_t)b * (k + 1), t);
            rej = !((s <= m) || (u < m / s));
          }
        }
      }
      // the first of them the CTA streams itself, straight away (no list round trips before its first copy)
      const unsigned rj = __ballot_sync(kFull, rej);
      const int own = rj ? __ffs(rj) - 1 : -1;
      if (lane == 0) sx.own = own >= 0 ? (int)blockIdx.x + own * G : -1;
      if (rej) {
        atomicOr(a.spec_bitmap + (b >> 5), 1u << (b & 31));
        if (lane != own) {
          const int pos = atomicAdd(a.spec_ctl, 1);
          if (BF) {  // the entry's row lse travel with it (published by the release below)
            a.spec_lse[2 * pos] = a.lse_p[(int64_t)b * (k + 1)];
            a.spec_lse[2 * pos + 1] = a.lse_q[(int64_t)b * k];
          }
          asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(a.spec_list + pos), "r"(b + 1) : "memory");
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (nmine) asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(a.spec_ctl + 1), "r"(nmine) : "memory");
      gstamp(a, 7);
    }
  }
  __syncthreads();
  if (!SPEC) {
    // launched as a programmatic dependent of the selector (FUSED: of whatever precedes the step — it may have written
    // the inputs): wait for it (and its memory) before the first read of the row info it wrote; no-op for a plain
    // launch
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0) gstamp(a, 1);
  }
  long long f_i0 = 0, f_i1 = 0;
  uint32_t f_epoch = 0;
  if (FUSED) {
    // the producer's first two claims go out before the selection, so their round trip overlaps it (the counter was
    // reset by the previous launch, complete after griddepcontrol.wait)
    if (warp == kProducerWarp && lane == 0) {
      f_i0 = (long long)atomicAdd(work, 1ull);
      f_i1 = (long long)atomicAdd(work, 1ull);
    }
    f_epoch = fused_select<BF>(a, stage_mem);
  }

  if (warp == kProducerWarp) {
    // ---------------------------------------------------------------- producer
    if (FUSED) {
      if (lane == 0) {
        // items in order from the work counter, as the plain producer; each item's rows come from its request's ready
        // word (polled until it carries this launch's epoch — no wait for the other CTAs' selection work), the next
        // item's word read while the current copy waits for its stage
        const uint64_t pol = l2_evict_normal_policy();
        const uint32_t epoch = f_epoch;
        long long i = f_i0, i1 = f_i1;
        unsigned long long w = i < total ? fused_wait_ready(a.fs.ready + i / nch, epoch) : 0ull;
        gstamp(a, 7);
        int t = 0;
        while (i < total) {
          const unsigned long long w1 = i1 < total ? __ldcg(a.fs.ready + i1 / nch) : 0ull;
          const long long prow = (long long)((w >> 22) & 0x3FFFFFull), qrow = (long long)(w & 0x3FFFFFull) - 1;
          float lp = 0.f, lq = 0.f;
          if (BF) {
            lp = __ldg(a.lse_p + prow);
            lq = qrow >= 0 ? __ldg(a.lse_q + qrow) : 0.f;
          }
          if (t == 0) gstamp(a, 2);
          issue_item<BF>(a, sh, stage_mem, t++, (int)(i / nch), (int)(i % nch), prow, qrow, 0, pol, lp, lq);
          // the next claim goes out after the copy (its round trip is only needed a whole item later; issued before
          // the copy it delayed every copy: cfg2 22.40 -> 22.15 us, tools/gpurun_calls/r2az.sh)
          const long long i2 = (long long)atomicAdd(work, 1ull);
          i = i1;
          i1 = i2;
          if (i < total) w = fused_ready(w1, epoch) ? w1 : fused_wait_ready(a.fs.ready + i / nch, epoch);
        }
        const int st = t % kStages;  // end of stream: a sentinel stage without data
        if (t >= kStages) mbar_wait(&sh.empty[st], (uint32_t)(((t / kStages) & 1) ^ 1u));
        sh.meta[st] = StageMeta{-1, 0, 0, 0};
        mbar_arrive(&sh.full[st]);
        gstamp(a, 3);
      }
    } else if (SPEC) {
      if (lane == 0) {
        const uint64_t pol = l2_evict_first_policy();
        // phase A: residual rows at position 0 of the listed requests, item i = (entry i / nch, chunk i % nch),
        // taken one at a time with two items of look-ahead on the counter and one on the entry (a relaxed load
        // issued before the current copy waits for its stage); an entry not written yet is waited for until every
        // request has been processed (then the list is complete and the phase is over)
        auto entry = [&](long long i) -> int {  // request of item i, -1: past the end of the list
          const int y = (int)(i / nch);
          if (y >= R) return -1;
          for (;;) {
            int e, done;
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(e) : "l"(a.spec_list + y) : "memory");
            if (e) return e - 1;
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(done) : "l"(a.spec_ctl + 1) : "memory");
            if (done >= R) {
              asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(e) : "l"(a.spec_list + y) : "memory");
              return e ? e - 1 : -1;
            }
            __nanosleep(128);
          }
        };
        int t = 0;
        if (sx.own >= 0) {
          const int b = sx.own;
          const float lp = BF ? __ldg(a.lse_p + (int64_t)b * (k + 1)) : 0.f;
          const float lq = BF ? __ldg(a.lse_q + (int64_t)b * k) : 0.f;
          for (int cc = 0; cc < nch; ++cc) {
            if (t == 0) gstamp(a, 2);
            issue_item<BF>(a, sh, stage_mem, t++, b, cc, (long long)b * (k + 1), (long long)b * k, 1, pol, lp, lq);
          }
        }
        // logits form: an entry's lse pair is published with it (spec_lse[2y..]); read beside the entry (the
        // release/acquire of the entry orders them; an entry seen by the relaxed look-ahead load is re-read below)
        auto entry_lse = [&](long long i, float& lp, float& lq) {
          if (BF) {
            const int y = (int)(i / nch);
            lp = __ldcg(a.spec_lse + 2 * y);
            lq = __ldcg(a.spec_lse + 2 * y + 1);
          }
        };
        long long i_cur = (long long)atomicAdd(work_a, 1ull);
        long long i_nxt = (long long)atomicAdd(work_a, 1ull);
        int b_cur = entry(i_cur);
        float lp_cur = 0.f, lq_cur = 0.f;
        if (b_cur >= 0) entry_lse(i_cur, lp_cur, lq_cur);
        while (b_cur >= 0) {
          const long long i_nxt2 = (long long)atomicAdd(work_a, 1ull);
          // the next item's entry: its load is in flight while this item waits for a free stage
          const int y_nxt = (int)(i_nxt / nch);
          int e_nxt = 0;
          if (y_nxt < R) asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(e_nxt) : "l"(a.spec_list + y_nxt));
          float lp_nxt = 0.f, lq_nxt = 0.f;
          if (e_nxt) entry_lse(i_nxt, lp_nxt, lq_nxt);
          if (t == 0) gstamp(a, 2);
          issue_item<BF>(a, sh, stage_mem, t++, b_cur, (int)(i_cur % nch), (long long)b_cur * (k + 1),
                         (long long)b_cur * k, 1, pol, lp_cur, lq_cur);
          b_cur = e_nxt ? e_nxt - 1 : entry(i_nxt);
          if (!e_nxt && b_cur >= 0) entry_lse(i_nxt, lp_nxt, lq_nxt);
          lp_cur = lp_nxt;
          lq_cur = lq_nxt;
          i_cur = i_nxt;
          i_nxt = i_nxt2;
        }
        // phase B: everything else, from the selector's row info (listed by the planner warp)
        mbar_wait(&sx.listB_ready, 0);
        asm volatile("griddepcontrol.wait;" ::: "memory");  // the selector's row info (no-op by now)
        gstamp(a, 1);
        t = stream_list<BF>(a, sh, stage_mem, t, sx.listB, sx.countB, work, 0, pol,
                            [&](int b, long long& pr, long long& qr, float& lp, float& lq) {
                              pr = a.prow[(int64_t)b * a.row_stride];
                              qr = a.qrow ? a.qrow[(int64_t)b * a.row_stride] : -1;
                              if (BF) {
                                lp = a.rowlse[2 * (int64_t)b];
                                lq = a.rowlse[2 * (int64_t)b + 1];
                              }
                            });
        const int s = t % kStages;  // end of stream: a sentinel stage without data
        if (t >= kStages) mbar_wait(&sh.empty[s], (uint32_t)(((t / kStages) & 1) ^ 1u));
        sh.meta[s] = StageMeta{-1, 0, 0, 0};
        mbar_arrive(&sh.full[s]);
        gstamp(a, 3);
      }
    } else if (BF && lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int t = stream_deep<BF, 3, 3>(a, sh, stage_mem, 0, total, work, 0, pol,
                                    [&](long long i) { return (int)(i / nch); },
                                    [&](int b, long long& pr, long long& qr, float& lp, float& lq) {
                                      pr = __ldcg(a.prow + (int64_t)b * a.row_stride);
                                      qr = a.qrow ? __ldcg(a.qrow + (int64_t)b * a.row_stride) : -1;
                                      lp = __ldcg(a.rowlse + 2 * (int64_t)b);
                                      lq = __ldcg(a.rowlse + 2 * (int64_t)b + 1);
                                    });
      const int s = t % kStages;  // end of stream: a sentinel stage without data
      if (t >= kStages) mbar_wait(&sh.empty[s], (uint32_t)(((t / kStages) & 1) ^ 1u));
      sh.meta[s] = StageMeta{-1, 0, 0, 0};
      mbar_arrive(&sh.full[s]);
      gstamp(a, 3);
    } else if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      // two items of look-ahead on the counter and the row info, so neither round trip stalls the copies
      long long i_next = (long long)atomicAdd(work, 1ull);
      long long i_next2 = (long long)atomicAdd(work, 1ull);
      long long pn = 0, qn = -1;
      float lpn = 0.f, lqn = 0.f;
      auto rows = [&](long long ii) {
        const int bb = (int)(ii / nch);
        pn = __ldcg(a.prow + (int64_t)bb * a.row_stride);
        qn = a.qrow ? __ldcg(a.qrow + (int64_t)bb * a.row_stride) : -1;
        if (BF) {
          lpn = __ldcg(a.rowlse + 2 * (int64_t)bb);
          lqn = __ldcg(a.rowlse + 2 * (int64_t)bb + 1);
        }
      };
      if (i_next < total) rows(i_next);
      for (int t = 0;; ++t) {
        const long long i = i_next;
        const long long prow = pn, qrow = qn;
        const float lp = lpn, lq = lqn;
        i_next = i_next2;
        if (i < total) {
          i_next2 = (long long)atomicAdd(work, 1ull);
          if (i_next < total) rows(i_next);
        }
        if (i >= total) {  // end of stream: a sentinel stage without data
          const int s = t % kStages;
          if (t >= kStages) mbar_wait(&sh.empty[s], (uint32_t)(((t / kStages) & 1) ^ 1u));
          sh.meta[s] = StageMeta{-1, 0, 0, 0};
          mbar_arrive(&sh.full[s]);
          gstamp(a, 3);
          break;
        }
        if (t == 0) gstamp(a, 2);
        issue_item<BF>(a, sh, stage_mem, t, (int)(i / nch), (int)(i % nch), prow, qrow, 0, pol, lp, lq);
      }
    }
    __syncwarp();
  } else if (warp < kConsumerWarps) {
    // ---------------------------------------------------------------- consumers
    if (FUSED && a.fs.B_sel > 32 * kFusedMaxRpt) {  // large selections: the consumers count in and scan
      __shared__ int s_last;
      if (fused_publish(a.fs, tid, kConsumerWarps * 32, &s_last)) fused_scans<BF>(a, tid, kConsumerWarps * 32);
    }
    for (int t = 0;; ++t) {
      const int s = t % kStages;
      mbar_wait(&sh.full[s], (uint32_t)((t / kStages) & 1));
      const StageMeta m = sh.meta[s];
      const int slot = t % kRing;
      if (t >= kRing) mbar_wait(&sh.ring_free[slot], (uint32_t)(((t / kRing) & 1) ^ 1));
      if (m.b < 0) {  // forward the end of stream to the publisher
        if (lane == 0) {
          if (warp == 0) sh.ring_meta[slot] = m;
          mbar_arrive(&sh.ring_full[slot]);
        }
        break;
      }
      if (t == 0 && warp == 0 && lane == 0) gstamp(a, 4);
      const uint8_t* sp = stage_mem + s * stage_bytes<BF>();
      double Gs[kSegsPerConsumer];
#pragma unroll
      for (int x = 0; x < kSegsPerConsumer; ++x) {
        const int seg = warp * kSegsPerConsumer + x;
        Gs[x] = consume_segment<BF>(sp, sp + stage_row_bytes<BF>(), m.res != 0,
                                    (int64_t)m.c * kChunkElems + seg * kSegElems, seg * kSegElems, a.V, lane, m.lp,
                                    m.lq);
      }
      // the segments' balanced trees over the 32 lane sums (the contract's xor butterfly), level by level across the
      // segments so the shuffle latencies overlap
#pragma unroll
      for (int mm = 1; mm < 32; mm <<= 1) {
        double o[kSegsPerConsumer];
#pragma unroll
        for (int x = 0; x < kSegsPerConsumer; ++x) o[x] = __shfl_xor_sync(kFull, Gs[x], mm);
#pragma unroll
        for (int x = 0; x < kSegsPerConsumer; ++x) Gs[x] = Gs[x] + o[x];
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&sh.empty[s]);
#pragma unroll
        for (int x = 0; x < kSegsPerConsumer; ++x) sh.ring_g[slot][warp * kSegsPerConsumer + x] = Gs[x];
        if (warp == 0) sh.ring_meta[slot] = m;
        mbar_arrive(&sh.ring_full[slot]);
      }
      __syncwarp();
    }
  } else if (warp == kPublisherWarp) {
    // ---------------------------------------------------------------- publisher
    // One published chunk per iteration: lanes 0..7 fold a warp run each (4 segments left to right), lane 0 folds the
    // chunk sum over the 8 runs left to right, and the sums go to global memory for the descent.  Arrivals on the
    // per-request counters are batched: after 32 published chunks (and at the end) one release fence, then one
    // relaxed increment per chunk (lane i for the i-th pending chunk).  Phase-A chunks go to their own sums and
    // counters.
    int pend_b = 0, npend = 0;
#ifndef TETRIS_FLUSH_SMALL
#define TETRIS_FLUSH_SMALL 2  // A/B (tools/gpurun_calls/r2ar.sh): 1 / 2 / 4 / 32 -> cfg2 23.86 / 22.53 / 22.72 / 22.76 us
#endif
    // small streams (a few items per CTA): publish sooner, so a request's descent need not wait for the end of every
    // stream that carried one of its chunks
    const int flush_every = total <= 2048 ? TETRIS_FLUSH_SMALL : 32;
    auto flush = [&]() {
      if (npend == 0 || a.req_cnt == nullptr) return;
      __syncwarp();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (lane < npend) atomicAdd((pend_b < 0 ? a.req_cnt_spec : a.req_cnt) + (pend_b < 0 ? ~pend_b : pend_b), 1);
      npend = 0;
    };
    for (int t = 0;; ++t) {
      const int slot = t % kRing;
      mbar_wait(&sh.ring_full[slot], (uint32_t)((t / kRing) & 1));
      const StageMeta m = sh.ring_meta[slot];
      if (m.b < 0) break;
      double x = 0.0;
      if (lane < kChunkWarps) {
#pragma unroll
        for (int q = 0; q < kWarpSegs; ++q) x = x + sh.ring_g[slot][lane * kWarpSegs + q];
      }
      const double gl = sh.ring_g[slot][lane];  // segment `lane` (published instead of the warp sums for short rows)
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.ring_free[slot]);
      double S = 0.0;
#pragma unroll
      for (int w = 0; w < kChunkWarps; ++w) S = S + __shfl_sync(kFull, x, w);
      const int64_t cs = (int64_t)m.b * nch + m.c;
      double* wsum = (SPEC && m.phase) ? a.warp_sums_spec : a.warp_sums;
      double* csum = (SPEC && m.phase) ? a.chunk_sums_spec : a.chunk_sums;
      if (nch <= kSegSumMaxChunks)
        __stcg(&wsum[cs * kChunkSegs + lane], gl);
      else if (lane < kChunkWarps)
        __stcg(&wsum[cs * kChunkWarps + lane], x);
      if (lane == 0) __stcg(&csum[cs], S);
      if (lane == npend) pend_b = (SPEC && m.phase) ? ~m.b : m.b;
      if (++npend == flush_every) flush();
    }
    flush();
    if (lane == 0) gstamp(a, 5);
  } else if (SPEC) {
    // ---------------------------------------------------------------- planner (speculative variant)
    // After the selection: list B = the requests phase A did not cover — not in the phase-A set, or in it with a zero
    // window (then the bonus row p[b][0] is plain, not the residual phase A streamed).  Loads batched 16 per lane.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0) {  // every CTA's share of the phase-A set is in
      int done;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(done) : "l"(a.spec_ctl + 1) : "memory");
        if (done >= R) break;
        __nanosleep(128);
      }
    }
    __syncwarp();
    for (int w = lane; w < (R + 31) >> 5; w += 32) sx.inA[w] = __ldcg(a.spec_bitmap + w);
    __syncwarp();
    int base = 0;
    for (int b0 = 0; b0 < R; b0 += 32 * 16) {
      long long qv[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        const int b = b0 + 32 * x + lane;
        qv[x] = b < R ? a.qrow[(int64_t)b * a.row_stride] : -1;
      }
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        const int b = b0 + 32 * x + lane;
        const bool inA = b < R && ((sx.inA[b >> 5] >> (b & 31)) & 1u);
        const bool doneA = inA && qv[x] == (long long)b * k;
        const unsigned need = __ballot_sync(kFull, b < R && !doneA);
        if (b < R && !doneA) sx.listB[base + __popc(need & ((1u << lane) - 1u))] = (uint16_t)b;
        base += __popc(need);
      }
    }
    __syncwarp();
    if (lane == 0) {
      sx.countB = base;
      mbar_arrive(&sx.listB_ready);  // release (CTA scope): the list is visible to the producer's wait
    }
    __syncwarp();
  } else if (FUSED) {
    // ---------------------------------------------------------------- scanner (one-launch step)
    // Counts the CTA in (its rows were written before the prologue's last __syncthreads); in the last CTA to count in
    // it runs the scans while the other warps stream — no consumer waits for them (small selections; larger ones are
    // scanned by the consumers, above).
    if (a.fs.B_sel <= 32 * kFusedMaxRpt) {
      int last = 0;
      if (lane == 0) last = atomic_add_acq_rel_gpu(a.fs.ctl, 1) == (int)gridDim.x - 1;
      last = __shfl_sync(kFull, last, 0);
      if (last) {
        __threadfence();
        fused_scans<BF>(a, lane, 32);
      }
    }
  }
  if (a.req_cnt != nullptr) {
    // Descent, one warp per request (requests strided over the CTAs so the re-reads spread over all SMs), as soon
    // as the request's nch chunks are published.  A warp only ever waits for chunks already claimed from the work
    // counter by CTAs that are running, so no co-residency (cooperative launch) is needed.
    if (FUSED) {
      // the next launch on the stream may be scheduled onto the SMs as this grid's CTAs leave (it waits for the whole
      // grid before touching anything); the descents need the fused selection's offset scans
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
      if (tid == 0) spin_acquire_geq(a.fs.ctl + 1, 1);
    }
    __syncthreads();
    if (SPEC) asm volatile("griddepcontrol.wait;" ::: "memory");  // the selector's row info (no-op by now)
    const int nwarps = blockDim.x >> 5;
    for (int b = warp * G + blockIdx.x; b < R; b += G * nwarps) {
      const long long qrow = a.qrow ? __ldcg(a.qrow + (int64_t)b * a.row_stride) : -1;
      const bool inA = SPEC && ((sx.inA[b >> 5] >> (b & 31)) & 1u);
      const bool doneA = inA && qrow == (long long)b * k;
      if (lane == 0) {
        int seen;
        int* cnt = doneA ? a.req_cnt_spec + b : a.req_cnt + b;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
          if (seen >= nch) break;
          __nanosleep(64);
        }
        *cnt = 0;  // every arrival is in: ready for the next launch
        if (warp == 0 && b == (int)blockIdx.x) gstamp(a, 13);
        if (inA && !doneA) {  // phase A streamed this request for nothing: drain its counter too
          for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(a.req_cnt_spec + b) : "memory");
            if (seen >= nch) break;
            __nanosleep(64);
          }
          a.req_cnt_spec[b] = 0;
        }
      }
      __syncwarp();
      finalize_request<BF>(a, b, qrow >= 0, lane, doneA ? a.chunk_sums_spec : a.chunk_sums,
                           doneA ? a.warp_sums_spec : a.warp_sums);
      if (warp == 0 && lane == 0 && b == (int)blockIdx.x) gstamp(a, 14);
    }
    // the last CTA out resets the work counters and the phase-A list (every producer is done with them)
    __syncthreads();
    __shared__ int s_last;
    if (tid == 0) {
      gstamp(a, 6);
      unsigned* done = a.grid_bar;
      s_last = atomicAdd(done, 1u) == (unsigned)G - 1;
      if (s_last) {
        *work = 0ull;
        if (SPEC) *work_a = 0ull;
        if (FUSED) {
          a.fs.ctl[0] = 0;
          a.fs.ctl[1] = 0;
          a.fs.ctl[2] = a.fs.ctl[2] + 1;  // the epoch this launch used (every CTA has read it)
        }
        *done = 0u;
      }
    }
    if (SPEC) {
      __syncthreads();
      if (s_last) {
        const int n = __ldcg(a.spec_ctl);
        for (int y = tid; y < n; y += blockDim.x) a.spec_list[y] = 0;
        for (int w = tid; w < (R + 31) >> 5; w += blockDim.x) a.spec_bitmap[w] = 0u;
        __syncthreads();
        if (tid == 0) {
          a.spec_ctl[0] = 0;
          a.spec_ctl[1] = 0;
        }
      }
    }
  }
}

// One warp per request: mass, T = u*mass, descent (after persist_stream_kernel has published every chunk).
__global__ void __launch_bounds__(128) finalize_kernel(const StreamArgs a) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (b >= a.R) return;
  const long long qrow = a.qrow ? a.qrow[(int64_t)b * a.row_stride] : -1;
  finalize_request<false>(a, b, qrow >= 0, lane, a.chunk_sums, a.warp_sums);
}

// ---- pre-accept: verify_token on every drafted position, one thread each (runs before the selection) -----------
// The accept test of position (b, j) does not depend on the selection, so all B*k random gathers of p[b][j][d] and
// q[b][j][d] are issued at once by a full grid instead of serially by the selector's single cluster.  Verdict byte:
// bit0 accept (accept_model.py:311-313), bit1 draft token outside the vocabulary, bit2 uniform outside [0, 1).
__global__ void pre_accept_kernel(const SelectArgs a) {
  const int B = a.ep_rows, k = a.k, V = a.V;
  const int32_t* len = a.len ? a.len + a.ep_row0 : nullptr;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)B * k) return;
  const int b = (int)(e / k), j = (int)(e - (int64_t)b * k);
  const int L = len ? len[b] : k;
  if (j >= L) {
    a.acc_bytes[e] = 0;
    return;
  }
  const int t = a.d[e];
  const double u = a.u_acc[e];
  uint8_t v = (u >= 0.0 && u < 1.0) ? 0 : 4;
  if (t < 0 || t >= V) {
    v |= 2;  // rejected
  } else {
    const double s = gather_q(a, e, t);
    const double m = gather_p(a, (int64_t)b * (k + 1) + j, t);
    v |= ((s <= m) || (u < m / s)) ? 1 : 0;
  }
  a.acc_bytes[e] = v;
}

// ---- stand-alone accept test (verify_stochastic without the fused selector epilogue) ----------------------------
__global__ void accept_kernel(const float* __restrict__ p, const float* __restrict__ q, const int32_t* __restrict__ d,
                              const int32_t* __restrict__ windows, const int32_t* __restrict__ win_off,
                              const double* __restrict__ u_acc, int B, int k, int V, int32_t* __restrict__ accepted,
                              long long* __restrict__ rowinfo, uint32_t* status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  uint32_t bad = 0;
  int w = windows[b];
  if (w < 0 || w > k) {
    bad |= TETRIS_ST_BAD_WINDOW;
    w = w < 0 ? 0 : k;
  }
  const int64_t uoff = win_off ? (int64_t)win_off[b] : (int64_t)b * k;
  int acc = w;
  for (int j0 = 0; j0 < w && acc == w; j0 += 8) {
    int t[8];
    double u[8], s[8], m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = j0 + i;
      t[i] = (j < w) ? d[(int64_t)b * k + j] : 0;
      u[i] = (j < w) ? u_acc[uoff + j] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = j0 + i;
      const bool ok = (j < w) && t[i] >= 0 && t[i] < V;
      s[i] = ok ? (double)q[((int64_t)b * k + j) * V + t[i]] : 0.0;
      m[i] = ok ? (double)p[((int64_t)b * (k + 1) + j) * V + t[i]] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = j0 + i;
      if (j >= w || acc != w) continue;
      if (!(u[i] >= 0.0 && u[i] < 1.0)) bad |= TETRIS_ST_BAD_UNIFORM;
      bool rej;
      if (t[i] < 0 || t[i] >= V) {
        bad |= TETRIS_ST_BAD_TOKEN;
        rej = true;
      } else {
        rej = !(s[i] <= m[i]) && !(u[i] < m[i] / s[i]);  // accept_model.py:311-313
      }
      if (rej) acc = j;
    }
  }
  accepted[b] = acc;
  rowinfo[2 * (int64_t)b] = (long long)b * (k + 1) + acc;
  rowinfo[2 * (int64_t)b + 1] = acc < w ? (long long)b * k + acc : -1;
  set_status(status, bad);
}

}  // namespace tetris

// ---- host side ---------------------------------------------------------------------------------------------------
#include "abi_util.h"

namespace tetris {

int launch_persist_stream(const StreamArgs& a_in, cudaStream_t st) {
  if (a_in.R == 0) return TETRIS_OK;
  StreamArgs a = a_in;
  a.dbg = debug_buffer();
  const int g_num_sms = abi::device_sm_count();
  const bool spec = a.u_acc != nullptr && a.req_cnt != nullptr;
  if (spec && (a.R > kSpecMaxR || !a.req_cnt_spec || !a.chunk_sums_spec || !a.warp_sums_spec || !a.d ||
               !a.spec_ctl || !a.spec_bitmap || !a.spec_list ||
               (a.R + (int)std::min<long long>((long long)a.R * a.nch, g_num_sms) - 1) /
                       (int)std::min<long long>((long long)a.R * a.nch, g_num_sms) > 32))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "speculative sampler: R=%d > %d or missing buffers", a.R, kSpecMaxR);
  const bool bf = a.zp != nullptr;
  if (bf && (!a.lse_p || (a.qrow && (!a.zq || !a.lse_q)) || a.req_cnt == nullptr || !a.rowlse ||
             (spec && !a.spec_lse)))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "logits form: zq / lse_p / lse_q and the fused descent are required");
  const bool fused = a.fs.conf != nullptr;
  if (fused && (spec || a.req_cnt == nullptr || !a.accepted || !a.fs.ctl || !a.fs.ready || !a.fs.u_acc || !a.d ||
                (long long)a.fs.B_sel * a.k > kFusedMaxCells || (bf && !a.fs.rowlse)))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "fused step: B_sel * k > %d or missing buffers", kFusedMaxCells);
  const void* fn = fused ? (bf ? (const void*)persist_stream_kernel<false, true, true>
                               : (const void*)persist_stream_kernel<false, false, true>)
                   : spec ? (bf ? (const void*)persist_stream_kernel<true, true> : (const void*)persist_stream_kernel<true, false>)
                        : (bf ? (const void*)persist_stream_kernel<false, true> : (const void*)persist_stream_kernel<false, false>);
  cudaError_t e = abi::ensure_smem(fn, kPersistSmem);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  const long long items = (long long)a.R * a.nch;
  // fused: every SM (the selection's rank work is spread over the CTAs, and more CTAs shorten it)
  const int grid = fused ? g_num_sms : (int)(items < g_num_sms ? items : g_num_sms);
  const int threads = kPersistThreads + ((spec || fused) ? 32 : 0);  // + the planner / scanner warp
  if (a.req_cnt != nullptr) {
    // one launch: streaming + per-request completion counters + descent
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = kPersistSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap our launch with the selector's tail
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {(void*)&a};
    e = cudaLaunchKernelExC(&cfg, fn, args);
    if (e != cudaSuccess) return abi::cuda_fail(e);
    return abi::launch_check();
  }
  persist_stream_kernel<false, false><<<grid, kPersistThreads, kPersistSmem, st>>>(a);
  int rc = abi::launch_check();
  if (rc) return rc;
  finalize_kernel<<<(a.R + 3) / 4, 128, 0, st>>>(a);
  return abi::launch_check();
}

// requests one speculative call can take on the current device: its shared-memory lists hold kSpecMaxR, and each CTA
// evaluates at most 32 requests' position-0 verdicts in the prologue (ceil(R / grid) <= 32)
int spec_max_requests() { return std::min(kSpecMaxR, 32 * abi::device_sm_count()); }

bool fused_step_eligible(int B_sel, int k, int u_packed) {
  static const bool off = std::getenv("TETRIS_NO_FUSED") != nullptr;  // A/B timing switch: the two-launch step
  // (B_sel bounded too: with k = 0 every batch has 0 cells, but the scans hold at most kFusedMaxRpt rows per thread)
  return !u_packed && B_sel >= 1 && B_sel <= kFusedMaxRpt * 512 && (long long)B_sel * k <= kFusedMaxCells && !off;
}

bool persist_eligible(const float* p, const float* q, int V) {
  return (V % kLaneElems == 0) && (((uintptr_t)p & 15u) == 0) && (!q || (((uintptr_t)q & 15u) == 0)) &&
         n_chunks(V) <= 64;
}

int launch_pre_accept(const SelectArgs& a, cudaStream_t st) {
  const long long n = (long long)a.ep_rows * a.k;
  if (n == 0) return TETRIS_OK;
  pre_accept_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
  return abi::launch_check();
}

int launch_accept(const float* p, const float* q, const int32_t* d, const int32_t* windows, const int32_t* win_off,
                  const double* u_acc, int B, int k, int V, int32_t* accepted, long long* rowinfo, uint32_t* status,
                  cudaStream_t st) {
  accept_kernel<<<(B + 127) / 128, 128, 0, st>>>(p, q, d, windows, win_off, u_acc, B, k, V, accepted, rowinfo,
                                                 status);
  return abi::launch_check();
}

}  // namespace tetris
