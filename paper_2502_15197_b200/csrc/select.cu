// Stages (1)+(2): prefix products and TETRIS capacity-constrained selection (global top-C), sm_100a.
//
// Reference semantics: cumulative_products (selector.py:95-110) + select_tetris (selector.py:133-176) with the
// heap key (-cum, row, depth) of _HeapItem (selector.py:113-130).  The heap merge of per-row lists takes exactly
// the C smallest cells under key (env desc, row asc, depth asc), env = the row's prefix-min of cum (for prefix
// products env == cum because fp rounding is monotone).  Rows are monotone in that key, so the selection is a
// per-row prefix and the kernel never materialises a sorted order:
//   * one CTA (1024 threads) owns all rows, thread t a contiguous block of rows;
//   * an MSB-first 8-bit radix select on the 64-bit key keeps, per row, the sub-range [lo,hi) of cells matching
//     the current key prefix (a contiguous range because keys are non-decreasing along the row), so each pass only
//     touches still-undecided cells and histograms are built from run lengths;
//   * it stops as soon as the bucket holding the C-th cell is taken whole; if all 64 bits are resolved the remaining
//     `need` cells are exact key ties and are taken in row-major order (row asc, then depth asc).
#include <cmath>

#include "common.cuh"

namespace tetris {

constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;

__global__ void __launch_bounds__(kSelThreads, 1)
    select_kernel(const double* __restrict__ vals, const int32_t* __restrict__ len, int B, int k, long long C,
                  int vals_are_cum, int32_t* __restrict__ windows, int32_t* __restrict__ win_offsets,
                  double* __restrict__ cum_out, long long* __restrict__ stats, uint64_t* __restrict__ keys,
                  uint32_t* status) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t(*hist)[256] = reinterpret_cast<uint32_t(*)[256]>(smem);
  uint8_t* lo = smem + kSelWarps * 256 * sizeof(uint32_t);
  uint8_t* hi = lo + B;
  __shared__ long long s_tmp[33];
  __shared__ uint32_t s_wt[8];
  __shared__ int s_digit;
  __shared__ long long s_need;
  __shared__ int s_done;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = (B + kSelThreads - 1) / kSelThreads;
  const int r0 = min(B, tid * R), r1 = min(B, r0 + R);

  // ---- phase 0: prefix products (sequential, left to right, selector.py:104-108), envelope, keys ------------
  uint32_t bad = 0;
  long long nvalid = 0;
  for (int r = r0; r < r1; ++r) {
    int L = len ? len[r] : k;
    if (L < 0 || L > k) {
      bad |= TETRIS_ST_BAD_VALUE;
      L = L < 0 ? 0 : k;
    }
    const double* row = vals + (int64_t)r * k;
    double cum = 1.0, env = 0.0;
    for (int j = 0; j < L; ++j) {
      double v = row[j];
      if (vals_are_cum) {
        cum = v;
        if (isnan(v)) bad |= TETRIS_ST_BAD_VALUE;
      } else {
        if (!(v >= 0.0 && v <= 1.0)) bad |= TETRIS_ST_BAD_VALUE;  // accept_model.py:55-59
        cum = __dmul_rn(cum, v);
      }
      if (cum_out) cum_out[(int64_t)r * k + j] = cum;
      env = (j == 0 || cum < env) ? cum : env;
      keys[(int64_t)r * k + j] = desc_key(env);
    }
    lo[r] = 0;
    hi[r] = (uint8_t)L;
    nvalid += L;
  }
  set_status(status, bad);
  long long N;
  block_excl_scan<long long>(nvalid, s_tmp, N);

  // ---- phase 1: radix select ---------------------------------------------------------------------------------
  // mode 0: take nothing, 1: take everything (C >= N), 2: radix
  const int mode = (C <= 0 || N == 0) ? 0 : (C >= N ? 1 : 2);
  long long need = C;
  bool done = mode != 2;
  for (int pass = 0; pass < 8 && !done; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = lane; i < 256; i += 32) hist[warp][i] = 0;
    __syncwarp();
    for (int r = r0; r < r1; ++r) {
      int l = lo[r], h = hi[r];
      if (l >= h) continue;
      const uint64_t* kr = keys + (int64_t)r * k;
      uint32_t cur = (uint32_t)(kr[l] >> shift) & 255u, cnt = 1;
      for (int j = l + 1; j < h; ++j) {
        uint32_t dg = (uint32_t)(kr[j] >> shift) & 255u;
        if (dg == cur) {
          ++cnt;
        } else {
          atomicAdd(&hist[warp][cur], cnt);
          cur = dg;
          cnt = 1;
        }
      }
      atomicAdd(&hist[warp][cur], cnt);
    }
    __syncthreads();
    uint32_t x = 0, incl = 0;
    if (tid < 256) {
#pragma unroll 8
      for (int w = 0; w < kSelWarps; ++w) x += hist[w][tid];
      incl = warp_incl_scan<uint32_t>(x, lane);
      if (lane == 31) s_wt[warp] = incl;
    }
    __syncthreads();
    if (tid < 256) {
      uint32_t base = 0;
      for (int w = 0; w < warp; ++w) base += s_wt[w];
      long long excl = (long long)base + incl - x;
      if (excl < need && need <= excl + (long long)x) {
        s_digit = tid;
        s_need = need - excl;
        s_done = (need - excl == (long long)x);
      }
    }
    __syncthreads();
    const uint32_t D = (uint32_t)s_digit;
    need = s_need;
    const bool take_all = s_done;
    for (int r = r0; r < r1; ++r) {
      int l = lo[r], h = hi[r];
      const uint64_t* kr = keys + (int64_t)r * k;
      while (l < h && (((uint32_t)(kr[l] >> shift) & 255u) < D)) ++l;
      int e = l;
      while (e < h && (((uint32_t)(kr[e] >> shift) & 255u) == D)) ++e;
      // take_all: the whole digit-D bucket is selected, so the window ends at the end of that range
      lo[r] = (uint8_t)(take_all ? e : l);
      hi[r] = (uint8_t)e;
    }
    done = take_all;
    __syncthreads();
  }

  // ---- phase 2: windows ------------------------------------------------------------------------------------------
  // After the loop (mode 2): lo = cells strictly better than the threshold key (+ whole bucket if take_all);
  // [lo,hi) = exact ties with the threshold, taken in row-major order.
  long long ties = 0;
  if (mode == 2)
    for (int r = r0; r < r1; ++r) ties += hi[r] - lo[r];
  long long tie_total;
  long long tie_excl = block_excl_scan<long long>(ties, s_tmp, tie_total);
  const bool tie_mode = (mode == 2) && !done;
  long long wsum = 0, nz = 0, ins = 0;
  for (int r = r0; r < r1; ++r) {
    int L = len ? len[r] : k;
    L = L < 0 ? 0 : (L > k ? k : L);
    int w;
    if (mode == 0) {
      w = 0;
    } else if (mode == 1) {
      w = L;
    } else {
      w = lo[r];
      if (tie_mode) {
        long long t = hi[r] - lo[r];
        long long take = need - tie_excl;
        take = take < 0 ? 0 : (take > t ? t : take);
        w += (int)take;
        tie_excl += t;
      }
    }
    windows[r] = w;
    wsum += w;
    nz += (L > 0);
    ins += w - ((w == L && L > 0) ? 1 : 0);
  }
  long long tot_w, tot_nz, tot_ins;
  long long woff = block_excl_scan<long long>(wsum, s_tmp, tot_w);
  block_excl_scan<long long>(nz, s_tmp, tot_nz);
  block_excl_scan<long long>(ins, s_tmp, tot_ins);
  if (win_offsets) {
    for (int r = r0; r < r1; ++r) {
      win_offsets[r] = (int32_t)woff;
      woff += windows[r];
    }
    if (tid == 0) win_offsets[B] = (int32_t)tot_w;
  }
  if (stats && tid == 0) {
    // PolicyStats closed forms (selector.py:150-170): extracts = sum w; inserts = nz + sum(w - [w == L > 0]);
    // peak_queue = nz (the heap starts with every non-empty row and never grows); all zero when C == 0.
    const bool any = C > 0;
    stats[0] = any ? tot_w : 0;
    stats[1] = any ? tot_nz + tot_ins : 0;
    stats[2] = any ? tot_nz : 0;
    stats[3] = -1;
  }
}

// ---- exact heapq replay (accounting only) ------------------------------------------------------------------------
// Mirrors CPython heapq (heapify/_siftup/_siftdown) as driven by select_tetris (selector.py:151-170) and counts every
// _HeapItem.__lt__ (selector.py:128-130).  Single thread by construction: the count is a property of the sequential
// schedule.
struct HeapItem {
  double cum;
  int32_t row, depth;
};

__device__ __forceinline__ bool item_lt(const HeapItem& a, const HeapItem& b, long long& cmp) {
  ++cmp;
  double na = -a.cum, nb = -b.cum;  // key = (-cum, row, depth)
  if (na != nb) return na < nb;
  if (a.row != b.row) return a.row < b.row;
  return a.depth < b.depth;
}

__device__ void sift_down(HeapItem* h, int start, int pos, long long& cmp) {
  HeapItem nw = h[pos];
  while (pos > start) {
    int pp = (pos - 1) >> 1;
    HeapItem parent = h[pp];
    if (item_lt(nw, parent, cmp)) {
      h[pos] = parent;
      pos = pp;
      continue;
    }
    break;
  }
  h[pos] = nw;
}

__device__ void sift_up(HeapItem* h, int n, int pos, long long& cmp) {
  int start = pos;
  HeapItem nw = h[pos];
  int child = 2 * pos + 1;
  while (child < n) {
    int right = child + 1;
    if (right < n && !item_lt(h[child], h[right], cmp)) child = right;
    h[pos] = h[child];
    pos = child;
    child = 2 * pos + 1;
  }
  h[pos] = nw;
  sift_down(h, start, pos, cmp);
}

__global__ void heap_stats_kernel(const double* __restrict__ cum, const int32_t* __restrict__ len, int B, int k,
                                  long long C, long long* stats, HeapItem* heap) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  long long cmp = 0, extracts = 0, inserts = 0, peak = 0;
  if (C > 0) {
    int n = 0;
    for (int r = 0; r < B; ++r) {
      int L = len ? len[r] : k;
      if (L > 0) heap[n++] = HeapItem{cum[(int64_t)r * k], r, 1};
    }
    for (int i = n / 2 - 1; i >= 0; --i) sift_up(heap, n, i, cmp);
    inserts = n;
    peak = n;
    while (n > 0 && extracts < C) {
      // heappop
      HeapItem last = heap[--n];
      HeapItem item = last;
      if (n > 0) {
        item = heap[0];
        heap[0] = last;
        sift_up(heap, n, 0, cmp);
      }
      ++extracts;
      int r = item.row, j = item.depth;
      int L = len ? len[r] : k;
      if (j < L) {
        // heappush
        heap[n] = HeapItem{cum[(int64_t)r * k + j], r, j + 1};
        ++n;
        sift_down(heap, 0, n - 1, cmp);
        ++inserts;
        if (n > peak) peak = n;
      }
    }
  }
  stats[0] = extracts;
  stats[1] = inserts;
  stats[2] = peak;
  stats[3] = cmp;
}

// expected_accepted (selector.py:296-306): one running fp64 sum in row order; cum restarts per row.
__global__ void expected_accepted_kernel(const double* __restrict__ alpha, const int32_t* __restrict__ len,
                                         const int32_t* __restrict__ windows, int B, int k, double* out,
                                         uint32_t* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double value = 0.0;
  uint32_t bad = 0;
  for (int r = 0; r < B; ++r) {
    int L = len ? len[r] : k;
    int w = windows[r];
    if (w > L || w < 0) {
      bad |= TETRIS_ST_BAD_WINDOW;
      w = w < 0 ? 0 : L;
    }
    double cum = 1.0;
    for (int j = 0; j < w; ++j) {
      cum = __dmul_rn(cum, alpha[(int64_t)r * k + j]);
      value = __dadd_rn(value, cum);
    }
  }
  *out = value;
  set_status(status, bad);
}

}  // namespace tetris

// ---- C ABI ---------------------------------------------------------------------------------------------------------
#include "abi_util.h"

extern "C" int tetris_select_f64(const double* vals, const int32_t* len, int32_t B, int32_t k, int64_t C,
                                 int32_t vals_are_cum, int32_t* windows, int32_t* win_offsets, double* cum_out,
                                 int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                 tetris_stream_t stream) {
  using namespace tetris;
  if (C < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0, got %lld", (long long)C);
  if (B < 0 || B > TETRIS_MAX_SELECT_ROWS) return abi::fail(TETRIS_INVALID_ARGUMENT, "B=%d outside [0, 65535]", B);
  if (k < 0 || k > TETRIS_MAX_K) return abi::fail(TETRIS_INVALID_ARGUMENT, "k=%d outside [0, 255]", k);
  if (B == 0) {
    if (win_offsets) {
      cudaError_t e = cudaMemsetAsync(win_offsets, 0, sizeof(int32_t), (cudaStream_t)stream);
      if (e != cudaSuccess) return abi::cuda_fail(e);
    }
    if (stats4) {
      cudaError_t e = cudaMemsetAsync(stats4, 0, 4 * sizeof(int64_t), (cudaStream_t)stream);
      if (e != cudaSuccess) return abi::cuda_fail(e);
    }
    return TETRIS_OK;
  }
  if (!vals || !windows) return abi::fail(TETRIS_INVALID_ARGUMENT, "vals and windows are required");
  size_t need = tetris_workspace_bytes(TETRIS_OP_SELECT, B, k, 0);
  if (!ws || ws_bytes < need)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "workspace too small: %zu < %zu", ws_bytes, need);
  size_t smem = (size_t)kSelWarps * 256 * sizeof(uint32_t) + 2 * (size_t)B;
  cudaError_t e = abi::ensure_smem(select_kernel, smem);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  select_kernel<<<1, kSelThreads, smem, (cudaStream_t)stream>>>(
      vals, len, B, k, (long long)C, vals_are_cum, windows, win_offsets, cum_out, (long long*)stats4,
      (uint64_t*)abi::ws_region(ws, TETRIS_OP_SELECT, B, k, 0, abi::WS_KEYS), status);
  return abi::launch_check();
}

extern "C" int tetris_heap_stats_f64(const double* cum, const int32_t* len, int32_t B, int32_t k, int64_t C,
                                     int64_t* stats4, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  using namespace tetris;
  if (C < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0, got %lld", (long long)C);
  if (B < 0 || k < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "bad shape B=%d k=%d", B, k);
  if (!stats4) return abi::fail(TETRIS_INVALID_ARGUMENT, "stats4 is required");
  size_t need = tetris_workspace_bytes(TETRIS_OP_SELECT, B, k, 0);
  if (B > 0 && (!ws || ws_bytes < need))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "workspace too small: %zu < %zu", ws_bytes, need);
  heap_stats_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(
      cum, len, B, k, (long long)C, (long long*)stats4,
      (HeapItem*)abi::ws_region(ws, TETRIS_OP_SELECT, B, k, 0, abi::WS_KEYS));
  return abi::launch_check();
}

extern "C" int tetris_expected_accepted_f64(const double* alpha, const int32_t* len, const int32_t* windows,
                                            int32_t B, int32_t k, double* out, uint32_t* status,
                                            tetris_stream_t stream) {
  using namespace tetris;
  if (B < 0 || k < 0 || !out) return abi::fail(TETRIS_INVALID_ARGUMENT, "bad arguments");
  expected_accepted_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(alpha, len, windows, B, k, out, status);
  return abi::launch_check();
}
