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
  return (size_t)B_sel * KS * 8 + (size_t)B_sel * 4 + (size_t)nown * k * 5;
}

__device__ inline FusedView fused_view(const FusedSel& f, int k, uint8_t* smem) {
  FusedView v;
  const int G = gridDim.x, g = blockIdx.x, Bs = f.B_sel;
  v.KS = k | 1;
  v.Np = Bs * v.KS;
  v.nown = g < Bs ? (Bs - 1 - g) / G + 1 : 0;
  v.ncell = v.nown * k;
  v.keys = reinterpret_cast<uint64_t*>(smem);
  v.lens = reinterpret_cast<int*>(v.keys + v.Np);
  v.rk = reinterpret_cast<uint32_t*>(v.lens + Bs);
  v.verd = reinterpret_cast<uint8_t*>(v.rk + v.ncell);
  return v;
}

// phase 0: the [B_sel][k] scores and lengths (coalesced loads, all in flight together) and the rank counters cleared.
// The kernel issues its own per-cell loads (accept-test gathers) around this call, so they share the round trip.
__device__ inline void fused_stage(const FusedSel& f, int k, const FusedView& v, int pt, int nt) {
  const int N = f.B_sel * k, KS = v.KS;
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
  for (int r = pt; r < f.B_sel; r += nt) v.lens[r] = f.len ? __ldg(f.len + r) : k;
  for (int c = pt; c < v.ncell; c += nt) v.rk[c] = 0u;
}

// phase 1: per row, prefix products left to right (selector.py:104-108), envelope, keys.  A row's values are read
// from shared memory all at once (up to 16), then the dependent fp64 chain runs from registers.
__device__ __forceinline__ void key_step(double x, int j, double& cum, double& env, uint64_t& key, uint32_t& bad) {
  if (!(x >= 0.0 && x <= 1.0)) bad |= TETRIS_ST_BAD_VALUE;  // accept_model.py:55-59
  cum = __dmul_rn(cum, x);
  env = (j == 0 || cum < env) ? cum : env;
  key = desc_key(env);
}

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
    double cum = 1.0, env = 0.0;
    if (KS <= 17) {
      double x[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = j < L ? __longlong_as_double((long long)row[j]) : 0.0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        uint64_t key = ~0ull;
        if (j < L) key_step(x[j], j, cum, env, key, bad);
        if (j < KS) row[j] = key;
      }
      if (KS == 17) row[16] = ~0ull;  // k == 16: the padding column
    } else {
      for (int j = 0; j < KS; ++j) {
        uint64_t key = ~0ull;
        if (j < L) key_step(__longlong_as_double((long long)row[j]), j, cum, env, key, bad);
        row[j] = key;
      }
    }
  }
  set_status(status, bad);
}

// phase 2: rank of each own cell m = #{o : key_o < key_m, or key_o == key_m and o < m} over every cell; the
// participants split (cell, key slice) pairs, lanes of a warp on consecutive cells of one slice (broadcast reads)
__device__ inline void fused_ranks(int k, const FusedView& v, int pt, int nt) {
  if (v.ncell == 0) return;
  const int G = gridDim.x, g = blockIdx.x, KS = v.KS, Np = v.Np;
  const int S = v.ncell >= nt ? 1 : nt / v.ncell;
  for (int wi = pt; wi < v.ncell * S; wi += nt) {
    const int c = wi % v.ncell, s = wi / v.ncell;
    const int oi = c / k, j = c - oi * k, r = g + oi * G;
    if (j >= v.lens[r]) continue;
    const int m = r * KS + j;
    const uint64_t km = v.keys[m];
    const int s0 = Np * s / S, s1 = Np * (s + 1) / S;  // Np * S <= 2 * kFusedMaxCells * 1024
    uint32_t n = 0;
    const int e1 = min(s1, m);
    int o = s0;
#pragma unroll 4
    for (; o < e1; ++o) n += v.keys[o] <= km ? 1u : 0u;
#pragma unroll 4
    for (o = max(s0, m + 1); o < s1; ++o) n += v.keys[o] < km ? 1u : 0u;
    if (n) atomicAdd(&v.rk[c], n);
  }
}

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

__device__ inline void fused_win_scan(const FusedSel& f, const FusedView& v, int pt, int nt, long long* tmp,
                                      const int (&wr)[kFusedMaxRpt]) {
  const int Bs = f.B_sel, rpt = (Bs + nt - 1) / nt, r0 = pt * rpt;
  long long pk = 0;
#pragma unroll
  for (int i = 0; i < kFusedMaxRpt; ++i) {
    const int r = r0 + i;
    if (i < rpt && r < Bs) {
      const int w = wr[i], L = v.lens[r];
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

__device__ __forceinline__ void spin_acquire_geq(const int* p, int v) {
  int seen;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(p) : "memory");
    if (seen >= v) break;
    __nanosleep(32);
  }
}

}  // namespace tetris
