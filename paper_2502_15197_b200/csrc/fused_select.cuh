// The TETRIS selection as the prologue of a persistent verification launch (small batches: B_sel * k <=
// kFusedMaxCells), shared by the stochastic sampler (stream.cu) and the greedy argmax stream (greedy.cu).
//
// Same results as select1_kernel (cumulative_products, selector.py:95-110; select_tetris's global top-C under the
// _HeapItem order (-cum, row, depth) over each row's prefix-min envelope, selector.py:113-176), computed without a
// selector launch: the C smallest cells of the (key, cell index) order are exactly the cells of RANK < C, and a
// cell's rank is a count over all keys — independent per cell — so every CTA stages all B_sel rows' keys in shared
// memory and ranks only the cells of its own rows g, g + G, ...  Keys are non-decreasing along a row, so a row's
// selected cells are a prefix and its window is the number of its cells of rank < C.  The last CTA to publish its
// rows writes the scans (win_offsets, PolicyStats selector.py:150-170, and the kernel's own lists).
//
// Shared layout (caller-provided scratch): keys [B_sel][KS] u64 (KS = k | 1: odd row stride, conflict-free per-row
// walks; padding and cells past a row's length hold ~0 = never smaller), lens [B_sel], rank counters and accept
// verdicts of the own cells.  Every phase runs on the first `nt` participating threads (index `pt`), separated by
// named barrier 1, so a kernel can keep other warps (a TMA producer) out of it.
#pragma once
#include "common.cuh"
#include "launch.h"

namespace tetris {

constexpr int kFusedMaxRpt = 8;  // rows per thread in the scans: B_sel <= kFusedMaxCells <= 8 * 256
// the key of padding and of cells past a row's length: above every real key (real keys of scores in [0, 1] lie in
// [0x400F.., 0x7FFF..]), and still above them after the +1 of the rank test below
constexpr uint64_t kPadKey = 0xFFFFFFFFFFFFFFFEull;

__device__ __forceinline__ void fused_bar(int nt) { asm volatile("bar.sync 1, %0;" ::"r"(nt) : "memory"); }

// exclusive scan over the nt participants (pt = 0..nt-1, nt a multiple of 32, <= 1024); tmp >= 33
template <typename U>
__device__ U fused_excl_scan(U x, U* tmp, U& total, int pt, int nt) {
  const int lane = pt & 31, warp = pt >> 5, nw = nt >> 5;
  const U incl = warp_incl_scan(x, lane);
  if (lane == 31) tmp[warp] = incl;
  fused_bar(nt);
  if (warp == 0) {
    const U t = lane < nw ? tmp[lane] : U(0);
    const U ti = warp_incl_scan(t, lane);
    tmp[lane] = ti - t;
    if (lane == 31) tmp[32] = ti;
  }
  fused_bar(nt);
  const U r = tmp[warp] + incl - x;
  total = tmp[32];
  fused_bar(nt);
  return r;
}

struct FusedView {
  uint64_t* keys;
  int* lens;
  uint32_t* rk;
  uint8_t* verd;
  int KS, Np, nown, ncell;
};

__host__ __device__ inline size_t fused_scratch_bytes(int B_sel, int k, int G) {
  const int KS = k | 1, nown = (B_sel + G - 1) / G;
  return (size_t)(((size_t)B_sel * KS + 1) & ~(size_t)1) * 8 + (size_t)B_sel * 4 + (size_t)nown * k * 5;
}

__device__ inline FusedView fused_view(const FusedSel& f, int k, uint8_t* smem) {
  FusedView v;
  const int G = gridDim.x, g = blockIdx.x, Bs = f.B_sel;
  v.KS = k | 1;
  v.Np = Bs * v.KS;  // the array holds (Np + 1) & ~1 keys: 16-byte pairs, an odd Np padded with kPadKey
  v.nown = g < Bs ? (Bs - 1 - g) / G + 1 : 0;
  v.ncell = v.nown * k;
  v.keys = reinterpret_cast<uint64_t*>(smem);
  v.lens = reinterpret_cast<int*>(v.keys + ((v.Np + 1) & ~1));
  v.rk = reinterpret_cast<uint32_t*>(v.lens + Bs);
  v.verd = reinterpret_cast<uint8_t*>(v.rk + v.ncell);
  return v;
}

// phase 0: the [B_sel][k] scores and lengths (coalesced loads, all in flight together) and the rank counters cleared.
// The kernel issues its own per-cell loads (accept-test gathers) around this call, so they share the round trip.
__device__ inline void fused_stage(const FusedSel& f, int k, const FusedView& v, int pt, int nt) {
  const int N = f.B_sel * k, KS = v.KS;
  // the lengths' loads go out with the first batch of scores (one round trip, not two)
  int ln[kFusedMaxRpt];
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i) {
    const int r = pt + i * nt;
    ln[i] = r < f.B_sel ? (f.len ? __ldg(f.len + r) : k) : 0;
  }
  for (int e0 = 0; e0 < N; e0 += 4 * nt) {
    double x4[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int e = e0 + x * nt + pt;
      x4[x] = e < N ? __ldg(f.conf + e) : 0.0;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int e = e0 + x * nt + pt;
      if (e < N) {
        const int r = e / k;
        v.keys[r * KS + (e - r * k)] = (uint64_t)__double_as_longlong(x4[x]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i)
    if (pt + i * nt < f.B_sel) v.lens[pt + i * nt] = ln[i];
  for (int c = pt; c < v.ncell; c += nt) v.rk[c] = 0u;
}

// phase 1: per row, prefix products left to right (selector.py:104-108) and keys.  Scores are validated into [0, 1]
// (accept_model.py:55-59), so each product is <= the one before it (RN is monotone) and the prefix-min envelope of
// select1_kernel is the product itself; the key is desc_key's value for a non-negative double, ~(bits | sign)
// (which also maps -0.0 onto +0.0).  A row's values are read at once (KM unrolled), then the fp64 chain runs from
// registers.  Invalid rows only raise TETRIS_ST_BAD_VALUE (the reference raises ValueError).
__device__ __forceinline__ bool score_ok(uint64_t b) { return b <= 0x3FF0000000000000ull || b == 0x8000000000000000ull; }
__device__ __forceinline__ uint64_t key_of_nonneg(double v) {
  return ~((uint64_t)__double_as_longlong(v) | 0x8000000000000000ull);
}

// (rolled loop: this code runs once per launch, and every launch starts with a cold instruction cache — measured
// ~140 cycles per KB of straight-line code on B200, tools/micro/icache.cu — so compact code beats unrolled code here)
__device__ inline void fused_keys(const FusedSel& f, int k, const FusedView& v, int pt, int nt, uint32_t* status) {
  const int KS = v.KS;
  uint32_t bad = 0;
  for (int r = pt; r < f.B_sel; r += nt) {
    int L = v.lens[r];
    if (L < 0 || L > k) {
      bad |= TETRIS_ST_BAD_VALUE;
      L = L < 0 ? 0 : k;
      v.lens[r] = L;
    }
    uint64_t* row = v.keys + r * KS;
    double cum = 1.0;
    if (KS <= 9) {  // k <= 8: the row's values at once, then a branch-free chain (1.0 past the length)
      uint64_t x[9];
#pragma unroll
      for (int j = 0; j < 9; ++j) x[j] = j < L ? row[j] : 0x3FF0000000000000ull;
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        bad |= score_ok(x[j]) ? 0u : TETRIS_ST_BAD_VALUE;
        cum = __dmul_rn(cum, __longlong_as_double((long long)x[j]));
        if (j < KS) row[j] = j < L ? key_of_nonneg(cum) : kPadKey;
      }
    } else {
#pragma unroll 1
      for (int j = 0; j < KS; ++j) {
        uint64_t key = kPadKey;
        if (j < L) {
          const uint64_t xb = row[j];
          if (!score_ok(xb)) bad |= TETRIS_ST_BAD_VALUE;
          cum = __dmul_rn(cum, __longlong_as_double((long long)xb));
          key = key_of_nonneg(cum);
        }
        row[j] = key;
      }
    }
  }
  if (pt == 0 && (v.Np & 1)) v.keys[v.Np] = kPadKey;
  set_status(status, bad);
}

// phase 2: rank of each own cell m = #{o : key_o < key_m, or key_o == key_m and o < m} over every cell.  A group of
// warps per own row; each thread holds 8 of the row's cell keys in registers and walks a strided slice of all the
// other keys (coalesced loads) — keys before the row count when <= a cell's key, keys after it when < (the tie rule
// by index); within the row, cell j is preceded by exactly its j predecessors.  Warp sums (REDUX) go to the cells'
// counters.  ~3 instructions per (key, cell) pair, no shared-memory bottleneck.
// n + (a >= b) for unsigned 64-bit a, b: the borrow of a - b through the carry chain (sub.cc / subc.cc produce the
// carry of a + ~b + 1, i.e. 1 exactly when a >= b), added with addc — 3 instructions, no predicate, no select
__device__ __forceinline__ uint32_t add_ge(uint32_t n, uint64_t a, uint64_t b) {
  uint32_t r;
  asm("{\n\t.reg .u32 t0, t1;\n\t"
      "sub.cc.u32 t0, %1, %3;\n\t"
      "subc.cc.u32 t1, %2, %4;\n\t"
      "addc.u32 %0, %5, 0;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)a), "r"((uint32_t)(a >> 32)), "r"((uint32_t)b), "r"((uint32_t)(b >> 32)), "r"(n));
  return r;
}

// small non-negative integer quotient a / b (a, b <= 1024) without the integer-division subroutine: the float quotient
// is correctly rounded and at least 1/b away from the next integer, so truncation is exact
__device__ __forceinline__ int small_div(int a, int b) { return (int)__fdiv_rn((float)a, (float)b); }

__device__ inline void fused_ranks_rows(const FusedView& v, int k, int pt, int nt) {
  constexpr int KM = 8;  // cells per pass (a row of k cells takes ceil(k / 8) passes)
  if (v.nown == 0) return;
  const int W = nt >> 5, wid = pt >> 5, lane = pt & 31;
  const int wpr = v.nown <= W ? small_div(W, v.nown) : 1;  // warps per row
  const int rq = small_div(wid, wpr), wr = wid - rq * wpr;
  const int rpp = small_div(W, wpr);  // rows per pass
  const int sub = wr * 32 + lane, nsub = wpr * 32;
  const int G = gridDim.x, g = blockIdx.x, KS = v.KS, Np = v.Np;
  // after the warp reduction below, lane l holds the total of cell ((l >> 4) & 1) * 4 + ((l >> 3) & 1) * 2 +
  // ((l >> 2) & 1) of the pass
  const int my_cell = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  for (int oi = rq; oi < v.nown; oi += rpp) {
    const int r = g + oi * G, L = v.lens[r], rs = r * KS, re = rs + KS;
#pragma unroll 1
    for (int j0 = 0; j0 < L; j0 += KM) {
      // before the row: count key_o <= key_m (key_m >= key_o); after it: key_o < key_m (key_m - 1 >= key_o); real
      // keys are >= 0x400F.., so key_m - 1 does not wrap
      uint64_t km[KM], km1[KM];
      uint32_t n[KM];
#pragma unroll
      for (int j = 0; j < KM; ++j) {
        km[j] = j0 + j < L ? v.keys[rs + j0 + j] : 0ull;
        km1[j] = km[j] - 1;
        n[j] = 0u;
      }
      int o = sub;
      // one load per step: a thread scans Np / nsub keys (8 at cfg2, 64 at most), and this one-shot code runs from a
      // cold instruction cache — the 4-loads-in-flight variant's larger body was slower (cfg2 22.48 -> 22.41 us, cfg1
      // 11.39 -> 11.31 us without it, tools/gpurun_calls/r2aw.sh)
      for (; o < rs; o += nsub) {
        const uint64_t x = v.keys[o];
#pragma unroll
        for (int j = 0; j < KM; ++j) n[j] = add_ge(n[j], km[j], x);
      }
      o = re + sub;
      for (; o < Np; o += nsub) {
        const uint64_t x = v.keys[o];
#pragma unroll
        for (int j = 0; j < KM; ++j) n[j] = add_ge(n[j], km1[j], x);
      }
      // warp reduce-scatter of the 8 counters (xor 16, 8, 4 halve the set; xor 2, 1 finish the sum)
      const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t send = h16 ? n[j] : n[j + 4], keep = h16 ? n[j + 4] : n[j];
        n[j] = keep + __shfl_xor_sync(kFull, send, 16);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t send = h8 ? n[j] : n[j + 2], keep = h8 ? n[j + 2] : n[j];
        n[j] = keep + __shfl_xor_sync(kFull, send, 8);
      }
      {
        const uint32_t send = h4 ? n[0] : n[1], keep = h4 ? n[1] : n[0];
        n[0] = keep + __shfl_xor_sync(kFull, send, 4);
      }
      n[0] += __shfl_xor_sync(kFull, n[0], 2);
      n[0] += __shfl_xor_sync(kFull, n[0], 1);
      const int j = j0 + my_cell;
      const uint32_t t = n[0] + (wr == 0 ? (uint32_t)j : 0u);  // cell j's own-row predecessors, counted once
      if ((lane & 3) == 0 && j < L && t) atomicAdd(&v.rk[oi * k + j], t);
    }
  }
}

__device__ inline void fused_ranks(int k, const FusedView& v, int pt, int nt) { fused_ranks_rows(v, k, pt, nt); }

// the window of own row oi (after phase 2)
__device__ __forceinline__ int fused_window(const FusedSel& f, int k, const FusedView& v, int oi) {
  const int L = v.lens[blockIdx.x + oi * gridDim.x];
  int w = 0;
  for (int j = 0; j < L; ++j) w += (long long)v.rk[oi * k + j] < f.C ? 1 : 0;
  return w;
}

// after the own rows are written: count this CTA as published; true in every participant of the last CTA
__device__ __forceinline__ bool fused_publish(const FusedSel& f, int pt, int nt, int* s_flag) {
  fused_bar(nt);
  if (pt == 0) *s_flag = atomic_add_acq_rel_gpu(f.ctl, 1) == (int)gridDim.x - 1;  // releases the CTA's rows
  fused_bar(nt);
  const bool last = *s_flag != 0;
  if (last) __threadfence();
  return last;
}

// last CTA: win_offsets and the PolicyStats closed forms over all B_sel windows (select1.cu's packed scan); participant
// pt holds the windows of rows [pt * rpt, (pt + 1) * rpt)
// (windows loaded by the caller with fused_load_windows, in the same round trip as its own loads)
__device__ __forceinline__ void fused_load_windows(const FusedSel& f, int pt, int nt, int (&wr)[kFusedMaxRpt]) {
  const int Bs = f.B_sel, rpt = (Bs + nt - 1) / nt, r0 = pt * rpt;
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i) wr[i] = (i < rpt && r0 + i < Bs) ? __ldcg(f.windows + r0 + i) : 0;
}

__device__ inline void fused_win_scan(const FusedSel& f, int k, int pt, int nt, long long* tmp,
                                      const int (&wr)[kFusedMaxRpt]) {
  const int Bs = f.B_sel, rpt = (Bs + nt - 1) / nt, r0 = pt * rpt;
  long long pk = 0;
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i) {
    const int r = r0 + i;
    if (i < rpt && r < Bs) {
      int L = f.len ? __ldg(f.len + r) : k;  // (clamped as the keys phase did)
      L = L < 0 ? 0 : (L > k ? k : L);
      const int w = wr[i];
      pk += (long long)w | ((long long)(w - ((w == L && L > 0) ? 1 : 0)) << 24) | ((long long)(L > 0) << 48);
    }
  }
  long long ptot;
  long long pex = fused_excl_scan<long long>(pk, tmp, ptot, pt, nt);
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i) {
    const int r = r0 + i;
    if (i < rpt && r < Bs) {
      f.win_offsets[r] = (int32_t)(pex & 0xFFFFFF);
      pex += wr[i];
    }
  }
  if (pt == 0) {
    const long long tot_w = ptot & 0xFFFFFF;
    f.win_offsets[Bs] = (int32_t)tot_w;
    if (f.stats) {
      const long long nz = (ptot >> 48) & 0xFFFF, ins = (ptot >> 24) & 0xFFFFFF;
      const bool any = f.C > 0;
      f.stats[0] = any ? tot_w : 0;
      f.stats[1] = any ? nz + ins : 0;
      f.stats[2] = any ? nz : 0;
      f.stats[3] = -1;
    }
  }
}

__device__ __forceinline__ void fused_release_done(const FusedSel& f, int pt, int nt) {
  fused_bar(nt);
  if (pt == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(f.ctl + 1), "r"(1) : "memory");
  }
}

// A request's ready word (one-launch step): bits 63..44 the launch's epoch (low 20 bits), 43..22 its p row (greedy: its
// window), 21..0 its q row + 1 (0: bonus row).  Rows < 2^22 hold: R * (k + 1) <= 2 * kFusedMaxCells.  Epochs make the words self-resetting:
// a word from an earlier launch never carries this launch's epoch.
__device__ __forceinline__ unsigned long long fused_ready_word(uint32_t epoch, long long prow, long long qrow) {
  return ((unsigned long long)(epoch & 0xFFFFFu) << 44) | ((unsigned long long)prow << 22) |
         (unsigned long long)(qrow + 1);
}
__device__ __forceinline__ bool fused_ready(unsigned long long w, uint32_t epoch) {
  return (uint32_t)(w >> 44) == (epoch & 0xFFFFFu);
}
__device__ __forceinline__ unsigned long long fused_wait_ready(const unsigned long long* p, uint32_t epoch) {
  for (;;) {
    const unsigned long long w = __ldcg(p);
    if (fused_ready(w, epoch)) return w;
    __nanosleep(32);
  }
}

__device__ __forceinline__ void spin_acquire_geq(const int* p, int v) {
  int seen;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(p) : "memory");
    if (seen >= v) break;
    __nanosleep(32);
  }
}

}  // namespace tetris
