// Stage (3) greedy verification as a persistent, warp-specialised TMA stream (sm_100a, fp32 rows, V % 8 == 0),
// with the compaction of stage (4) fused into the same launch.
//
// Greedy verification is verify_token on one-hot distributions (accept_model.py:309-313): position j of request b is
// accepted iff d[b][j] == argmax_v p[b][j][v] (numpy.argmax order: NaN ranks highest, ties -> lowest index), and the
// emitted token is the argmax at the first mismatch, or at w_b (the bonus position, sim_engine.py:407-409).  Every
// selected row 0..w_b is read in full once: HBM-bound, (Σ_b (w_b + 1)) · V · 4 bytes per call.
//
// The row list (rows 1..w_b of every request, in request order, their argmax keys zeroed) comes from the selector's
// epilogue (select1.cu) or from greedy_rowmap_kernel (one CTA); then persist_greedy_kernel, a programmatic dependent
// of the selector, one CTA per SM, 18 warps:
//   warp 16     producer: first row 0 of every request — always verified, so it streams before the selection
//               completes (its keys live in a fixed workspace region, left at zero) — then, after griddepcontrol.wait,
//               the listed rows; items (row, chunk) claimed 4 at a time from global counters, 1-D bulk copies
//               (cp.async.bulk, mbarrier complete_tx, L2 evict-first) of 8192-element chunks of p into a 6-stage
//               192 KB ring;
//   warps 0..15 consumers: the argmax key of 512 staged elements each (two segments), reduced over the warp;
//   warp 17     publisher: reduces the 16 keys of a chunk, folds it into the row's key with one atomicMax, and counts
//               the chunk on the request's arrival counter (one release fence per 32 chunks).
// The argmax travels as one 64-bit key whose unsigned order is numpy's: high word = the value's bits mapped to an
// unsigned order (NaN above +inf, -0.0 canonicalised to +0.0), low word = ~index (lower index wins a tie).
// Then, in the same launch, one warp per request (strided over the CTAs) waits for the request's (w_b + 1) · nch
// chunks, reads the w_b + 1 keys and writes accepted / out_tok; the last CTA out runs the compaction (offsets and
// tokens, compact_kernel's contract) when asked to.  One-launch step (the selection as this kernel's prologue, small
// batches): the windows' scan runs in the last CTA to publish its windows, during the stream; batches of at most
// kFinRows requests are finished by CTA 0 alone — every descent, then the compaction from shared memory.
#include <climits>

#include "common.cuh"
#include "fused_select.cuh"
#include "launch.h"

namespace tetris {

namespace {

constexpr int kGStages = 6;
constexpr int kGConsumers = 16;
constexpr int kSegsPerWarp = kChunkElems / kSegElems / kGConsumers;  // staged segments per consumer warp
constexpr int kGProducer = kGConsumers;
constexpr int kGThreads = (kGConsumers + 2) * 32;
constexpr int kFinRows = 36;  // one-launch batches up to this many requests: CTA 0 finishes them alone (2 per warp)
constexpr int kGRing = 64;
constexpr int kClaim = 4;  // work items (row chunks) per claim on the global counter
constexpr int kStaticItems = 8;  // calls with at most this many items per CTA use a static schedule
constexpr size_t kGStageBytes = (size_t)kChunkElems * sizeof(float);  // 32 KB
constexpr size_t kGSmem = kGStages * kGStageBytes;                    // 192 KB dynamic
static_assert(kSegsPerWarp * kGConsumers * kSegElems == kChunkElems, "consumers split a chunk evenly");

// diagnostics (tools/dbg_greedy.py): per-CTA %globaltimer stamps, a no-op unless a debug buffer is registered
__device__ __forceinline__ void gtime(const GreedyArgs& a, int slot) {
  if (a.dbg) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[64 + 8 * blockIdx.x + slot] = t;
  }
}

struct GMeta {
  int b, row, c, pad;  // request, row index b*(k+1)+j, chunk; pad 1: a row-0 item (phase A, key in key0)
};

struct GreedyShared {
  uint64_t full[kGStages];
  uint64_t empty[kGStages];
  uint64_t ring_full[kGRing];
  uint64_t ring_free[kGRing];
  GMeta meta[kGStages];
  GMeta ring_meta[kGRing];
  unsigned long long ring_key[kGRing][kGConsumers];
};

// numpy.argmax order of a value as an unsigned 32-bit word (larger wins): NaN above +inf, -0.0 equal to +0.0.
__device__ __forceinline__ uint32_t argmax_order(float v) {
  if (v != v) return 0xFFFFFFFFu;
  if (v == 0.f) v = 0.f;
  const uint32_t bits = __float_as_uint(v);
  return (bits >> 31) ? ~bits : (bits | 0x80000000u);
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long x) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    const unsigned long long y = __shfl_xor_sync(kFull, x, m);
    x = y > x ? y : x;
  }
  return x;
}

// The warp's argmax key over its SEGS staged segments (lane l: elements seg*256 + 8l .. +8 of each), as one 64-bit
// word whose unsigned order is numpy.argmax's: high word argmax_order(value), low word ~index (lower index wins a
// tie); 0 = no element.  Per element: one NaN-propagating max, then one compare + select for the first index equal
// to it; NaN rows take a separate (warp-uniform, rare) branch.  Elements at or past V (only in the row's last chunk)
// are read as -inf: they lose every comparison to a real element of the chunk, which always has one (V % 8 == 0).
template <int SEGS>
__device__ __forceinline__ unsigned long long warp_argmax(const float* __restrict__ sp, int chunk_e0, int seg0,
                                                          bool partial, int V, int lane) {
  float v[SEGS][8];
#pragma unroll
  for (int x = 0; x < SEGS; ++x) lds8_swz(sp + (seg0 + x) * kSegElems + lane * kLaneElems, lane, v[x]);
  const float kNegInf = __int_as_float(0xff800000);
  if (partial) {
#pragma unroll
    for (int x = 0; x < SEGS; ++x)
      if (chunk_e0 + (seg0 + x) * kSegElems + lane * kLaneElems >= V) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[x][i] = kNegInf;
      }
  }
  float bv = v[0][0];
#pragma unroll
  for (int x = 0; x < SEGS; ++x)
#pragma unroll
    for (int i = (x == 0 ? 1 : 0); i < 8; ++i) asm("max.NaN.f32 %0, %0, %1;" : "+f"(bv) : "f"(v[x][i]));
  int bl = 0;  // local position x * 8 + i of the first element equal to the max
  if (__any_sync(kFull, bv != bv)) {
    const bool nan = bv != bv;
#pragma unroll
    for (int x = SEGS - 1; x >= 0; --x)
#pragma unroll
      for (int i = 7; i >= 0; --i) bl = (nan ? (v[x][i] != v[x][i]) : (v[x][i] == bv)) ? x * 8 + i : bl;
  } else {
#pragma unroll
    for (int x = SEGS - 1; x >= 0; --x)
#pragma unroll
      for (int i = 7; i >= 0; --i) bl = (v[x][i] == bv) ? x * 8 + i : bl;
  }
  const uint32_t idx = (uint32_t)(chunk_e0 + (seg0 + (bl >> 3)) * kSegElems + lane * kLaneElems + (bl & 7));
  const uint32_t hi = argmax_order(bv);
  const uint32_t whi = __reduce_max_sync(kFull, hi);
  const uint32_t widx = __reduce_min_sync(kFull, hi == whi ? idx : 0xFFFFFFFFu);
  return ((unsigned long long)whi << 32) | (uint32_t)~widx;
}

}  // namespace

// Rows read by greedy verification — positions j0..w_b of every request, w_b clamped to [0, k] — in request order:
// rowmap[1 + r] = b << 8 | j, rowmap[0] = their count; the argmax key of each listed row is zeroed (keys != nullptr).
// j0 = 1 for the persistent stream (it streams row 0 of every request itself, before the selection completes).
// One CTA; each thread a contiguous block of requests.  Launched as a programmatic dependent of the selector.
__global__ void __launch_bounds__(1024, 1)
    greedy_rowmap_kernel(const int32_t* __restrict__ windows, int B, int k, int32_t* __restrict__ rowmap,
                         unsigned long long* __restrict__ keys, int j0) {
  __shared__ long long s_tmp[33];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int tid = threadIdx.x;
  const int R = (B + blockDim.x - 1) / blockDim.x;
  const int r0 = min(B, tid * R), r1 = min(B, r0 + R);
  long long local = 0;
  for (int b = r0; b < r1; ++b) {
    const int w = windows[b];
    local += (w < 0 ? 0 : (w > k ? k : w)) + 1 - j0;
  }
  long long total;
  const long long off0 = block_excl_scan<long long>(local, s_tmp, total);
  // the writes, one request at a time per warp with the lanes along the request's rows (coalesced): the owner lane
  // broadcasts each of its requests' row offset and window
  const int lane = tid & 31;
  long long off = off0;
  for (int src = 0; src < 32; ++src) {
    const int sb0 = __shfl_sync(kFull, r0, src), sb1 = __shfl_sync(kFull, r1, src);
    long long so = __shfl_sync(kFull, off, src);
    for (int b = sb0; b < sb1; ++b) {
      int w = windows[b];
      w = w < 0 ? 0 : (w > k ? k : w);
      for (int j = j0 + lane; j <= w; j += 32) {
        rowmap[1 + so + j - j0] = (b << 8) | j;
        if (keys) keys[(int64_t)b * (k + 1) + j] = 0ull;
      }
      so += w + 1 - j0;
    }
  }
  if (tid == 0) rowmap[0] = (int32_t)total;
}

// FUSED (the one-launch greedy step, B_sel * k <= kFusedMaxCells): the selection runs as a prologue on the consumer
// and publisher warps (fused_select.cuh) while the producer already streams row 0 of every request; the ring is 5
// stages and the 6th stage's 32 KB holds the selection's scratch.  The row list becomes per-request ready words (epoch
// | window): phase B claims every (request, row 1..k, chunk) item in order and skips the rows past the window.
template <bool FUSED>
__global__ void __launch_bounds__(kGThreads, 1) persist_greedy_kernel(const GreedyArgs a) {
  constexpr int kGStages = FUSED ? 5 : 6;
  extern __shared__ __align__(128) uint8_t stage_mem[];
  __shared__ GreedyShared sh;
  __shared__ long long s_tmp[33];
  __shared__ int s_last;
  __shared__ uint32_t s_epoch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nch = a.nch, V = a.V, k = a.k;
  const int G = gridDim.x;
  unsigned long long* work = reinterpret_cast<unsigned long long*>(a.grid_bar + 2);

  if (tid == 0) {
    gtime(a, 0);
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], kGConsumers);
    }
    for (int r = 0; r < kGRing; ++r) {
      mbar_init(&sh.ring_full[r], kGConsumers);
      mbar_init(&sh.ring_free[r], 1);
    }
    mbar_fence_init();
  }
  if (FUSED) {
    // the previous launch on the stream may have written the inputs: wait for it before the first read; the epoch
    // of this launch (the previous one's + 1, set by its last CTA out)
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  __syncthreads();

  if (FUSED && warp != kGProducer) {
    // the selection prologue on warps 0..15 and 17 (participant index: warp 17 -> 512..543)
    const int NP = kGThreads - 32, pt = warp < kGProducer ? tid : tid - 32;
    const FusedSel& f = a.fs;
    const FusedView v = fused_view(f, k, stage_mem + kGStages * kGStageBytes);
    // this launch's epoch (the previous one's + 1, set by its last CTA out): loaded beside the scores, published in
    // shared memory after them (the barriers before phase 3 and the descents make it visible)
    const uint32_t ep = pt == 0 ? (uint32_t)__ldcg(a.fs.ctl + 2) : 0u;
    fused_stage(f, k, v, pt, NP);
    if (pt == 0) s_epoch = ep + 1u;
    fused_bar(NP);
    fused_keys(f, k, v, pt, NP, a.status);
    fused_bar(NP);
    fused_ranks(k, v, pt, NP);
    fused_bar(NP);
    const uint32_t epoch = s_epoch;
    for (int oi = pt; oi < v.nown; oi += NP) {
      const int r = blockIdx.x + oi * G;
      const int w = fused_window(f, k, v, oi);
      f.windows[r] = w;
      const int lr = r - f.row0;
      if (lr >= 0 && lr < a.B) __stcg(f.ready + lr, fused_ready_word(epoch, w, -1));  // epoch | window
    }
    if (pt == 0) gtime(a, 5);
  }

  if (warp == kGProducer) {
    const uint64_t pol = l2_evict_first_policy();
    // the producer's own copy of this launch's epoch (it takes no part in the prologue's barriers); phase B needs it
    const uint32_t p_epoch = FUSED ? (uint32_t)__ldcg(a.fs.ctl + 2) + 1u : 0u;
    int t = 0;
    // one item (request b, listed row `row`, chunk c) into the next stage; phase 1: a row-0 item
    auto issue = [&](int b, int row, int cc, int phase) {
      const int s = t % kGStages;
      if (t >= kGStages) mbar_wait(&sh.empty[s], (uint32_t)(((t / kGStages) & 1) ^ 1u));
      const int n = min(kChunkElems, V - cc * kChunkElems);
      const uint32_t bytes = (uint32_t)n * sizeof(float);
      sh.meta[s] = GMeta{b, row, cc, phase};
      if (t == 0) gtime(a, 1);
      mbar_arrive_expect_tx(&sh.full[s], bytes);
      bulk_g2s_stream(stage_mem + s * kGStageBytes, a.p + (int64_t)row * V + (int64_t)cc * kChunkElems, bytes,
                      &sh.full[s], pol);
      ++t;
    };
    // Phase A, before the selection completes: row 0 of every request — always verified (positions 0..w_b) — as
    // items i = (b = i / nch, chunk i % nch), claimed 4 at a time (static when there are few)
    if (lane == 0) {
      const long long total_a = (long long)a.B * nch;
      if (total_a <= (long long)kStaticItems * G) {
        for (long long i = blockIdx.x; i < total_a; i += G) {
          const int b = (int)(i / nch);
          issue(b, b * (k + 1), (int)(i % nch), 1);
        }
      } else {
        unsigned long long* work_a = reinterpret_cast<unsigned long long*>(a.grid_bar2);
        long long c_cur = (long long)atomicAdd(work_a, (unsigned long long)kClaim);
        while (c_cur < total_a) {
          const long long c_next = (long long)atomicAdd(work_a, (unsigned long long)kClaim);
#pragma unroll
          for (int x = 0; x < kClaim; ++x) {
            const long long i = c_cur + x;
            if (i < total_a) {
              const int b = (int)(i / nch);
              issue(b, b * (k + 1), (int)(i % nch), 1);
            }
          }
          c_cur = c_next;
        }
      }
    }
    __syncwarp();
    if (FUSED) {
      // Phase B of the one-launch step: items (request b, row j = 1..k, chunk c) in order from the work counter; a
      // request's window comes from its ready word (polled until it carries this launch's epoch), rows past it are
      // skipped without a copy
      if (lane == 0) {
        const uint32_t epoch = p_epoch;
        const long long per_b = (long long)k * nch, total = (long long)a.B * per_b;
        long long i = (long long)atomicAdd(work, 1ull), i1 = (long long)atomicAdd(work, 1ull);
        int bcur = -1, wb = 0;
        while (i < total) {
          const long long i2 = (long long)atomicAdd(work, 1ull);
          const int b = (int)(i / per_b), rem = (int)(i - (long long)b * per_b), j = 1 + rem / nch, cc = rem % nch;
          if (b != bcur) {
            wb = (int)((fused_wait_ready(a.fs.ready + b, epoch) >> 22) & 0x3FFFFFull);
            bcur = b;
          }
          if (j <= wb) issue(b, b * (k + 1) + j, cc, 0);
          i = i1;
          i1 = i2;
        }
        gtime(a, 2);
      }
    }
    // Phase B: the listed rows 1..w_b, once the selection (and its row list) is complete
    if (!FUSED) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (lane == 0 && !FUSED) gtime(a, 2);
    const long long total = FUSED ? 0 : (long long)__ldcg(a.rowmap) * nch;
    if (FUSED) {
    } else if (lane == 0 && total <= (long long)kStaticItems * gridDim.x) {
      // small calls: a static schedule (items blockIdx.x + x * G) with every row lookup issued up front
      int rm[kStaticItems];
#pragma unroll
      for (int x = 0; x < kStaticItems; ++x) {
        const long long i = blockIdx.x + (long long)x * G;
        rm[x] = i < total ? __ldcg(a.rowmap + 1 + i / nch) : 0;
      }
#pragma unroll
      for (int x = 0; x < kStaticItems; ++x) {
        const long long i = blockIdx.x + (long long)x * G;
        if (i >= total) break;
        const int b = rm[x] >> 8, j = rm[x] & 0xFF;
        issue(b, b * (k + 1) + j, (int)(i % nch), 0);
      }
    } else if (lane == 0) {
      // Items are claimed kClaim at a time, one claim ahead: the counter's and the row map's round trips (each up to
      // ~1 us under full HBM load) overlap the copies of a whole claim instead of one 32 KB chunk each.
      // small calls (fewer than 16 items per CTA) claim one item at a time, so every SM gets a share
      const int claim = total >= 16LL * gridDim.x ? kClaim : 1;
      long long c_cur = (long long)atomicAdd(work, (unsigned long long)claim);
      int rm_cur[kClaim], rm_nx[kClaim];
#pragma unroll
      for (int x = 0; x < kClaim; ++x)
        rm_cur[x] = (x < claim && c_cur + x < total) ? __ldcg(a.rowmap + 1 + (c_cur + x) / nch) : 0;
      while (c_cur < total) {
        const long long c_next = (long long)atomicAdd(work, (unsigned long long)claim);
#pragma unroll
        for (int x = 0; x < kClaim; ++x) {
          const long long i = c_cur + x;
          if (x < claim && i < total) {
            const int b = rm_cur[x] >> 8, j = rm_cur[x] & 0xFF;
            issue(b, b * (k + 1) + j, (int)(i % nch), 0);
          }
          if (x == (claim > 1 ? 1 : 0)) {  // copies issued: fetch the next claim's rows (waits for the counter)
#pragma unroll
            for (int y = 0; y < kClaim; ++y)
              rm_nx[y] = (y < claim && c_next + y < total) ? __ldcg(a.rowmap + 1 + (c_next + y) / nch) : 0;
          }
        }
        c_cur = c_next;
#pragma unroll
        for (int x = 0; x < kClaim; ++x) rm_cur[x] = rm_nx[x];
      }
    }
    if (lane == 0) {  // end of stream: a sentinel stage without data
      const int s = t % kGStages;
      if (t >= kGStages) mbar_wait(&sh.empty[s], (uint32_t)(((t / kGStages) & 1) ^ 1u));
      sh.meta[s] = GMeta{-1, 0, 0, 0};
      mbar_arrive(&sh.full[s]);
      gtime(a, 3);
    }
    __syncwarp();
  } else if (warp < kGConsumers) {
    if (FUSED) {
      // the one-launch step: win_offsets / PolicyStats over every selected row's window, by the consumers of the last
      // CTA to publish its rows' windows — now, while the stream runs, not in the last CTA out's tail
      __shared__ int s_last_pub;
      if (fused_publish(a.fs, tid, kGConsumers * 32, &s_last_pub)) {
        int wr[kFusedMaxRpt];
        fused_load_windows(a.fs, tid, kGConsumers * 32, wr);
        fused_win_scan(a.fs, k, tid, kGConsumers * 32, s_tmp, wr);
      }
    }
    for (int t = 0;; ++t) {
      const int s = t % kGStages;
      mbar_wait(&sh.full[s], (uint32_t)((t / kGStages) & 1));
      const GMeta m = sh.meta[s];
      const int slot = t % kGRing;
      if (t >= kGRing) mbar_wait(&sh.ring_free[slot], (uint32_t)(((t / kGRing) & 1) ^ 1));
      if (m.b < 0) {  // forward the end of stream to the publisher
        if (lane == 0) {
          if (warp == 0) sh.ring_meta[slot] = m;
          mbar_arrive(&sh.ring_full[slot]);
        }
        break;
      }
      const float* sp = reinterpret_cast<const float*>(stage_mem + s * kGStageBytes);
      const int e0 = m.c * kChunkElems;
      const unsigned long long key =
          warp_argmax<kSegsPerWarp>(sp, e0, kSegsPerWarp * warp, e0 + kChunkElems > V, V, lane);
      if (lane == 0) {
        mbar_arrive(&sh.empty[s]);  // the staged data has been read
        sh.ring_key[slot][warp] = key;
        if (warp == 0) sh.ring_meta[slot] = m;
        mbar_arrive(&sh.ring_full[slot]);
      }
      __syncwarp();
    }
  } else {
    // publisher: one chunk per iteration; arrivals on the per-request counters batched behind one release fence
    int pend_b = 0, npend = 0;
    bool waited = false;
    auto flush = [&]() {
      if (npend == 0) return;
      __syncwarp();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (lane < npend) atomicAdd(a.req_cnt + pend_b, 1);
      npend = 0;
    };
    for (int t = 0;; ++t) {
      const int slot = t % kGRing;
      mbar_wait(&sh.ring_full[slot], (uint32_t)((t / kGRing) & 1));
      const GMeta m = sh.ring_meta[slot];
      if (m.b < 0) break;
      unsigned long long key = lane < kGConsumers ? sh.ring_key[slot][lane] : 0ull;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.ring_free[slot]);
      key = warp_max_u64(key);
      if (!FUSED && m.pad == 0 && !waited) {  // the row list's keys were zeroed by the selection: wait for it once
        asm volatile("griddepcontrol.wait;" ::: "memory");
        waited = true;
      }
      if (lane == 0) atomicMax(m.pad ? a.key0 + m.b : a.keys + m.row, key);
      if (lane == npend) pend_b = m.b;
      if (++npend == 32) flush();
    }
    flush();
  }

  // one warp per request as soon as its (w_b + 1) * nch chunks are in
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // windows (no-op by now)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next step's selector may be scheduled
  constexpr int kWarps = kGThreads / 32;
  // small one-launch batches: CTA 0 alone runs every request's descent (one round: B <= its warps x 2) and then the
  // compaction from shared memory — no last-CTA election, no reload of the results; the other CTAs leave at once
  const bool fin = FUSED && a.offsets != nullptr && a.B <= kFinRows;
  __shared__ int s_acc[kFinRows], s_tok[kFinRows];
  int32_t* ds = reinterpret_cast<int32_t*>(stage_mem);  // the stage ring is idle now: the drafted tokens
  if (fin && blockIdx.x == 0)
    for (int e = tid; e < a.B * k; e += kGThreads) ds[e] = __ldg(a.d + e);  // in flight while the counters fill
  for (int b = fin ? (blockIdx.x == 0 ? warp : a.B) : warp * G + blockIdx.x; b < a.B;
       b += fin ? kWarps : G * kWarps) {
    int w = FUSED ? (int)((fused_wait_ready(a.fs.ready + b, s_epoch) >> 22) & 0x3FFFFFull) : a.windows[b];
    uint32_t bad = (w < 0 || w > k) ? TETRIS_ST_BAD_WINDOW : 0u;
    w = w < 0 ? 0 : (w > k ? k : w);
    if (lane == 0) {
      const int need = (w + 1) * nch;
      int seen;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(a.req_cnt + b) : "memory");
        if (seen >= need) break;
        __nanosleep(64);
      }
      a.req_cnt[b] = 0;  // every arrival is in: ready for the next launch
    }
    __syncwarp();
    unsigned long long* kb = a.keys + (int64_t)b * (k + 1);
    int acc = w, tok = -1;
    for (int j0 = 0; j0 <= w; j0 += 32) {
      const int j = j0 + lane;
      const int am = j <= w ? (int)~(uint32_t)__ldcg(j == 0 ? a.key0 + b : kb + j) : -1;
      const int t = j < w ? a.d[(int64_t)b * k + j] : 0;
      const unsigned mis = __ballot_sync(kFull, j < w && t != am);
      if (mis) {
        const int l = __ffs(mis) - 1;
        acc = j0 + l;
        tok = __shfl_sync(kFull, am, l);
        const int tl = __shfl_sync(kFull, t, l);
        if (tl < 0 || tl >= V) bad |= TETRIS_ST_BAD_TOKEN;
        break;
      }
      if (w < j0 + 32) tok = __shfl_sync(kFull, am, w - j0);  // all accepted: the bonus position's argmax
    }
    for (int j = 1 + lane; j <= w; j += 32) kb[j] = 0ull;  // read: left at zero for the next launch
    if (lane == 0) {
      a.key0[b] = 0ull;  // read above (lane 0, j = 0): ready for the next launch
      a.accepted[b] = acc;
      a.out_tok[b] = tok;
      if (fin) {
        s_acc[b] = acc;
        s_tok[b] = tok;
      }
      set_status(a.status, bad);
    }
  }
  if (fin && blockIdx.x == 0) {
    __syncthreads();
    if (warp == 0) {  // compact_kernel's contract over <= 64 requests: n_b = accepted + 1 (capped), one warp scan
      int n[2], tot = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int b = lane + 32 * h;
        n[h] = b < a.B ? min(s_acc[b] + 1, a.cap ? max(__ldg(a.cap + b), 0) : INT_MAX) : 0;
      }
      int off[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int incl = warp_incl_scan<int>(n[h], lane);
        off[h] = tot + incl - n[h];
        tot += __shfl_sync(kFull, incl, 31);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int b = lane + 32 * h;
        if (b < a.B) {
          a.offsets[b] = off[h];
          for (int j = 0; j < n[h]; ++j) a.tokens[off[h] + j] = j < s_acc[b] ? ds[b * k + j] : s_tok[b];
        }
      }
      if (lane == 0) a.offsets[a.B] = tot;
    }
  }

  // the last CTA out resets the work counter and, when asked to, compacts the emitted tokens
  if (tid == 0) gtime(a, 4);
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    unsigned* done = a.grid_bar;
    const bool last = atomicAdd(done, 1u) == (unsigned)G - 1;
    if (last) {
      *work = 0ull;
      *reinterpret_cast<unsigned long long*>(a.grid_bar2) = 0ull;
      *done = 0u;
      if (FUSED) {
        a.fs.ctl[0] = 0;                  // the CTAs counted in by fused_publish
        a.fs.ctl[2] = (int)s_epoch;       // the epoch this launch used (every CTA has read it)
      }
      __threadfence();
    }
    s_last = last;
  }
  __syncthreads();
  if (!s_last || fin) return;
  if (tid == 0) gtime(a, 6);
  if (FUSED) {
    // the one-launch step (B <= kFusedMaxRows): the compaction with every load in ONE round trip (accepted, out_tok,
    // cap of the thread's rows [r0, r0 + rpt); the drafted tokens d staged in the now idle stage ring), then the
    // on-chip scan and the writes (win_offsets / PolicyStats were written during the stream)
    const int B = a.B, nt = blockDim.x, rpt = (B + nt - 1) / nt, r0 = tid * rpt;
    int acc[kFusedMaxRpt], tok[kFusedMaxRpt], nn[kFusedMaxRpt];
    int32_t* ds = reinterpret_cast<int32_t*>(stage_mem);
    if (a.offsets != nullptr) {
#pragma unroll
      for (int i = 0; i < kFusedMaxRpt; ++i) {
        const int r = r0 + i;
        const bool in = i < rpt && r < B;
        acc[i] = in ? __ldcg(a.accepted + r) : 0;
        tok[i] = in ? __ldcg(a.out_tok + r) : 0;
        nn[i] = in && a.cap ? __ldg(a.cap + r) : INT_MAX;
      }
      for (int e = tid; e < B * k; e += nt) ds[e] = __ldg(a.d + e);
    }
    if (a.offsets == nullptr) return;
    __syncthreads();
    long long local = 0;
#pragma unroll
    for (int i = 0; i < kFusedMaxRpt; ++i) {
      nn[i] = (i < rpt && r0 + i < B) ? min(acc[i] + 1, max(nn[i], 0)) : 0;
      local += nn[i];
    }
    long long total;
    long long off = block_excl_scan<long long>(local, s_tmp, total);
#pragma unroll
    for (int i = 0; i < kFusedMaxRpt; ++i) {
      const int r = r0 + i;
      if (i < rpt && r < B) {
        a.offsets[r] = (int32_t)off;
        for (int j = 0; j < nn[i]; ++j) a.tokens[off + j] = j < acc[i] ? ds[r * k + j] : tok[i];
        off += nn[i];
      }
    }
    if (tid == 0) {
      a.offsets[B] = (int32_t)total;
      gtime(a, 7);
    }
    return;
  }
  if (a.offsets == nullptr) return;
  // compact_kernel's contract: n_b = accepted[b] + 1 (capped), offsets = exclusive scan, tokens = d[b][0..a) ++ [x]
  const int B = a.B;
  const int R = (B + blockDim.x - 1) / blockDim.x;
  const int r0 = min(B, tid * R), r1 = min(B, r0 + R);
  long long local = 0;
  for (int r = r0; r < r1; ++r) {
    int n = __ldcg(a.accepted + r) + 1;
    if (a.cap) n = min(n, max(a.cap[r], 0));
    local += n;
  }
  long long total;
  long long off = block_excl_scan<long long>(local, s_tmp, total);
  for (int r = r0; r < r1; ++r) {
    const int acc = __ldcg(a.accepted + r);
    int n = acc + 1;
    if (a.cap) n = min(n, max(a.cap[r], 0));
    a.offsets[r] = (int32_t)off;
    const int x = __ldcg(a.out_tok + r);
    for (int i = 0; i < n; ++i) a.tokens[off + i] = i < acc ? a.d[(int64_t)r * k + i] : x;
    off += n;
  }
  if (tid == 0) a.offsets[B] = (int32_t)total;
}

}  // namespace tetris

// ---- host side ---------------------------------------------------------------------------------------------------
#include "abi_util.h"

namespace tetris {

// the one-launch greedy step keeps the selection's scratch in the 6th stage (32 KB)
// (and every own row's window is written by a consumer thread, which the win scan's barrier orders: <= 512 own rows)
bool greedy_fused_fits(int B_sel, int k) {
  const int G = abi::device_sm_count();
  return fused_scratch_bytes(B_sel, k, G) <= kGStageBytes && (B_sel + G - 1) / G <= kGConsumers * 32;
}

bool persist_greedy_eligible(const float* p, int V) {
  return (V % kLaneElems == 0) && (((uintptr_t)p & 15u) == 0);
}

static int launch_pdl(const void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, void** args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  return abi::launch_check();
}

int launch_greedy_rowmap(const int32_t* windows, int B, int k, int32_t* rowmap, unsigned long long* keys, int j0,
                         cudaStream_t st) {
  void* args[] = {(void*)&windows, (void*)&B, (void*)&k, (void*)&rowmap, (void*)&keys, (void*)&j0};
  return launch_pdl((const void*)greedy_rowmap_kernel, dim3(1), dim3(1024), 0, st, args);
}

int launch_persist_greedy(const GreedyArgs& a, cudaStream_t st) {
  const int num_sms = abi::device_sm_count();
  const bool fused = a.fs.conf != nullptr;
  if (fused && ((long long)a.fs.B_sel * a.k > kFusedMaxCells || !a.fs.ctl || !a.fs.ready ||
                fused_scratch_bytes(a.fs.B_sel, a.k, num_sms) > kGStageBytes))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "one-launch greedy step: B_sel * k > %d or missing buffers",
                     kFusedMaxCells);
  const void* fn = fused ? (const void*)persist_greedy_kernel<true> : (const void*)persist_greedy_kernel<false>;
  cudaError_t e = abi::ensure_smem(fn, kGSmem);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  // the listed-row count lives on the device; the bound B * (k + 1) * nch caps the useful grid (fused: every SM,
  // the selection's rank work is spread over the CTAs)
  const long long items = (long long)a.B * (a.k + 1) * a.nch;
  const int grid = fused ? num_sms : (int)(items < num_sms ? items : num_sms);
  GreedyArgs copy = a;
  copy.dbg = debug_buffer();
  void* args[] = {(void*)&copy};
  return launch_pdl(fn, dim3(grid), dim3(kGThreads), kGSmem, st, args);
}

}  // namespace tetris
