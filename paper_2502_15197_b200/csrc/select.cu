// Stages (1)+(2): prefix products and TETRIS capacity-constrained selection (global top-C), sm_100a.
//
// Reference semantics: cumulative_products (selector.py:95-110) + select_tetris (selector.py:133-176) with the
// heap key (-cum, row, depth) of _HeapItem (selector.py:113-130).  The heap merge of per-row lists takes exactly
// the C smallest cells under key (env desc, row asc, depth asc), env = the row's prefix-min of cum (for prefix
// products env == cum because fp rounding is monotone).  Rows are monotone in that key, so the selection is a
// per-row prefix and the kernel never materialises a sorted order:
//   * a thread-block cluster of G CTAs (1..16, DSMEM) owns the batch; CTA g a contiguous block of rows whose 64-bit
//     keys live in its shared memory (column layout [depth][row], conflict-free);
//   * an MSB-first 8-bit radix select keeps, per row, the sub-range [lo,hi) of cells matching the current key
//     prefix (contiguous because keys are non-decreasing along a row), so a pass only touches undecided cells and
//     histograms are built from run lengths into per-warp copies; the cluster sums the CTA histograms over DSMEM;
//   * it stops as soon as the bucket holding the C-th cell is taken whole; if all 64 bits are resolved the
//     remaining `need` cells are exact key ties and are taken in row-major order (row asc, then depth asc).
// Optional epilogue (the fused step): verify_token's accept test on the selected window of every request, the
// first-rejection length, the row to resample from, and the compaction offsets + accepted-prefix tokens.
#include <cooperative_groups.h>

#include <cmath>

#include "common.cuh"
#include "launch.h"

namespace cg = cooperative_groups;

namespace tetris {

constexpr int kSelThreads = 1024;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kMaxCluster = 16;
constexpr size_t kSelHistBytes = (size_t)kSelWarps * 256 * sizeof(uint32_t);
constexpr size_t kSelKeyBudget = 192 * 1024;  // keys + lo/hi per CTA



struct SelShared {
  uint32_t cta_hist[2][256];
  long long part[8];
  long long tmp[33];
  uint32_t wt[8];
  int digit;
  long long need;
  int done;
};

// Cluster-wide exclusive scan over rows in row order.  Rows of CTA g are [g*RB, g*RB + nrows), thread t handles
// rows base + t.  `val(r)` gives a row's value, `use(r, excl)` consumes its exclusive prefix.  Returns the total.
template <typename ValF, typename UseF>
__device__ long long cluster_row_scan(cg::cluster_group& cluster, SelShared& sh, int slot, int nrows, ValF val,
                                      UseF use) {
  const int tid = threadIdx.x;
  long long local = 0;
  for (int base = 0; base < nrows; base += kSelThreads) {
    const int r = base + tid;
    local += (r < nrows) ? val(r) : 0;
  }
  long long cta_total;
  block_excl_scan<long long>(local, sh.tmp, cta_total);
  if (tid == 0) sh.part[slot] = cta_total;
  cluster.sync();
  long long before = 0, total = 0;
  const unsigned me = cluster.block_rank();
  for (unsigned g = 0; g < cluster.num_blocks(); ++g) {
    const long long v = *cluster.map_shared_rank(&sh.part[slot], g);
    if (g < me) before += v;
    total += v;
  }
  long long carry = before;
  for (int base = 0; base < nrows; base += kSelThreads) {
    const int r = base + tid;
    const long long v = (r < nrows) ? val(r) : 0;
    long long tot;
    const long long ex = block_excl_scan<long long>(v, sh.tmp, tot);
    if (r < nrows) use(r, carry + ex);
    carry += tot;
  }
  return total;
}

__global__ void __launch_bounds__(kSelThreads, 1) select_kernel(const SelectArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ SelShared sh;
  cg::cluster_group cluster = cg::this_cluster();
  uint32_t(*hist)[256] = reinterpret_cast<uint32_t(*)[256]>(smem);
  const int RB = a.RB, k = a.k;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem + kSelHistBytes);  // [k][RB]
  uint8_t* lo = reinterpret_cast<uint8_t*>(keys + (size_t)k * RB);
  uint8_t* hi = lo + RB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = (int)cluster.block_rank();
  const int row0 = g * RB;
  const int nrows = max(0, min(a.B, row0 + RB) - row0);

  // ---- phase 0: prefix products (sequential, left to right, selector.py:104-108), envelope, keys ------------
  uint32_t bad = 0;
  long long nvalid = 0;
  for (int r = tid; r < nrows; r += kSelThreads) {
    const int gr = row0 + r;
    int L = a.len ? a.len[gr] : k;
    if (L < 0 || L > k) {
      bad |= TETRIS_ST_BAD_VALUE;
      L = L < 0 ? 0 : k;
    }
    const double* row = a.vals + (int64_t)gr * k;
    double cum = 1.0, env = 0.0;
    for (int j = 0; j < L; ++j) {
      const double v = row[j];
      if (a.vals_are_cum) {
        cum = v;
        if (isnan(v)) bad |= TETRIS_ST_BAD_VALUE;
      } else {
        if (!(v >= 0.0 && v <= 1.0)) bad |= TETRIS_ST_BAD_VALUE;  // accept_model.py:55-59
        cum = __dmul_rn(cum, v);
      }
      if (a.cum_out) a.cum_out[(int64_t)gr * k + j] = cum;
      env = (j == 0 || cum < env) ? cum : env;
      keys[(size_t)j * RB + r] = desc_key(env);
    }
    lo[r] = 0;
    hi[r] = (uint8_t)L;
    nvalid += L;
  }
  set_status(a.status, bad);
  long long cta_valid;
  block_excl_scan<long long>(nvalid, sh.tmp, cta_valid);
  if (tid == 0) sh.part[0] = cta_valid;
  cluster.sync();
  long long N = 0;
  for (unsigned c = 0; c < cluster.num_blocks(); ++c) N += *cluster.map_shared_rank(&sh.part[0], c);

  // ---- phase 1: radix select ---------------------------------------------------------------------------------
  const int mode = (a.C <= 0 || N == 0) ? 0 : (a.C >= N ? 1 : 2);  // 0: nothing, 1: everything, 2: radix
  long long need = a.C;
  bool done = mode != 2;
  for (int pass = 0; pass < 8 && !done; ++pass) {
    const int shift = 56 - 8 * pass;
    const int buf = pass & 1;
    for (int i = lane; i < 256; i += 32) hist[warp][i] = 0;
    __syncwarp();
    for (int r = tid; r < nrows; r += kSelThreads) {
      const int l = lo[r], h = hi[r];
      if (l >= h) continue;
      uint32_t cur = (uint32_t)(keys[(size_t)l * RB + r] >> shift) & 255u, cnt = 1;
      for (int j = l + 1; j < h; ++j) {
        const uint32_t dg = (uint32_t)(keys[(size_t)j * RB + r] >> shift) & 255u;
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
    if (tid < 256) {
      uint32_t x = 0;
#pragma unroll 8
      for (int w = 0; w < kSelWarps; ++w) x += hist[w][tid];
      sh.cta_hist[buf][tid] = x;
    }
    cluster.sync();
    if (tid < 256) {
      uint32_t x = 0;
      for (unsigned c = 0; c < cluster.num_blocks(); ++c) x += cluster.map_shared_rank(&sh.cta_hist[buf][0], c)[tid];
      const uint32_t incl = warp_incl_scan<uint32_t>(x, lane);
      if (lane == 31) sh.wt[warp] = incl;
      asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 histogram warps only
      uint32_t base = 0;
      for (int w = 0; w < warp; ++w) base += sh.wt[w];
      const long long excl = (long long)base + incl - x;
      if (excl < need && need <= excl + (long long)x) {
        sh.digit = tid;
        sh.need = need - excl;
        sh.done = (need - excl == (long long)x);
      }
    }
    __syncthreads();
    const uint32_t D = (uint32_t)sh.digit;
    need = sh.need;
    const bool take_all = sh.done;
    for (int r = tid; r < nrows; r += kSelThreads) {
      int l = lo[r];
      const int h = hi[r];
      while (l < h && (((uint32_t)(keys[(size_t)l * RB + r] >> shift) & 255u) < D)) ++l;
      int e = l;
      while (e < h && (((uint32_t)(keys[(size_t)e * RB + r] >> shift) & 255u) == D)) ++e;
      // take_all: the whole digit-D bucket is selected, so the window ends at the end of that range
      lo[r] = (uint8_t)(take_all ? e : l);
      hi[r] = (uint8_t)e;
    }
    done = take_all;
  }
  __syncthreads();

  // ---- phase 2: windows -----------------------------------------------------------------------------------------
  // lo = cells strictly better than the threshold (+ the whole bucket when take_all); [lo,hi) = exact key ties,
  // taken in row-major order while the tie budget `need` lasts.
  const bool tie_mode = (mode == 2) && !done;
  auto row_len = [&](int r) {
    const int L = a.len ? a.len[row0 + r] : k;
    return L < 0 ? 0 : (L > k ? k : L);
  };
  if (tie_mode) {
    cluster_row_scan(
        cluster, sh, 1, nrows, [&](int r) { return (long long)(hi[r] - lo[r]); },
        [&](int r, long long ex) {
          const long long t = hi[r] - lo[r];
          long long take = need - ex;
          take = take < 0 ? 0 : (take > t ? t : take);
          lo[r] = (uint8_t)(lo[r] + take);
        });
  }
  for (int r = tid; r < nrows; r += kSelThreads) {
    const int w = mode == 0 ? 0 : (mode == 1 ? row_len(r) : lo[r]);
    a.windows[row0 + r] = w;
    lo[r] = (uint8_t)w;  // lo now holds the window
  }
  __syncthreads();
  // win_offsets (exclusive scan of windows) + PolicyStats closed forms (selector.py:150-170):
  // extracts = sum w; inserts = nz + sum(w - [w == L > 0]); peak_queue = nz; all zero when C == 0.
  long long nz_loc = 0, ins_loc = 0;
  for (int r = tid; r < nrows; r += kSelThreads) {
    const int L = row_len(r), w = lo[r];
    nz_loc += (L > 0);
    ins_loc += w - ((w == L && L > 0) ? 1 : 0);
  }
  {
    long long t;
    block_excl_scan<long long>(nz_loc, sh.tmp, t);
    if (tid == 0) sh.part[3] = t;
    block_excl_scan<long long>(ins_loc, sh.tmp, t);
    if (tid == 0) sh.part[4] = t;
  }
  const long long tot_w = cluster_row_scan(
      cluster, sh, 2, nrows, [&](int r) { return (long long)lo[r]; },
      [&](int r, long long ex) {
        if (a.win_offsets) a.win_offsets[row0 + r] = (int32_t)ex;
      });
  if (g == (int)cluster.num_blocks() - 1 && tid == 0 && a.win_offsets) a.win_offsets[a.B] = (int32_t)tot_w;
  if (a.stats && g == 0 && tid == 0) {
    long long nz = 0, ins = 0;
    for (unsigned c = 0; c < cluster.num_blocks(); ++c) {
      nz += *cluster.map_shared_rank(&sh.part[3], c);
      ins += *cluster.map_shared_rank(&sh.part[4], c);
    }
    const bool any = a.C > 0;
    a.stats[0] = any ? tot_w : 0;
    a.stats[1] = any ? nz + ins : 0;
    a.stats[2] = any ? nz : 0;
    a.stats[3] = -1;
  }

  // ---- optional epilogue: accept test + first rejection + compaction offsets (fused step) ----------------------
  if (a.p != nullptr) {
    uint32_t vbad = 0;
    const int ep0 = a.ep_row0, ep1 = a.ep_row0 + a.ep_rows;
    __syncthreads();
    for (int r = tid; r < nrows; r += kSelThreads) {
      const int gr = row0 + r;
      if (gr < ep0 || gr >= ep1) continue;
      const int lr = gr - ep0;
      const int w = lo[r];
      const int64_t uoff = a.u_packed ? (int64_t)a.win_offsets[gr] : (int64_t)lr * k;
      int acc = w;
      for (int j0 = 0; j0 < w && acc == w; j0 += 8) {
        int t[8];
        double u[8], s[8], m[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int j = j0 + i;
          t[i] = (j < w) ? a.d[(int64_t)lr * k + j] : 0;
          u[i] = (j < w) ? a.u_acc[uoff + j] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int j = j0 + i;
          const bool ok = (j < w) && t[i] >= 0 && t[i] < a.V;
          s[i] = ok ? (double)a.q[((int64_t)lr * k + j) * a.V + t[i]] : 0.0;
          m[i] = ok ? (double)a.p[((int64_t)lr * (k + 1) + j) * a.V + t[i]] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int j = j0 + i;
          if (j >= w || acc != w) continue;
          if (!(u[i] >= 0.0 && u[i] < 1.0)) vbad |= TETRIS_ST_BAD_UNIFORM;
          bool rej;
          if (t[i] < 0 || t[i] >= a.V) {
            vbad |= TETRIS_ST_BAD_TOKEN;
            rej = true;
          } else {
            rej = !(s[i] <= m[i]) && !(u[i] < m[i] / s[i]);  // accept_model.py:311-313
          }
          if (rej) acc = j;
        }
      }
      a.accepted[lr] = acc;
      a.rowinfo[2 * (int64_t)lr] = (long long)lr * (k + 1) + acc;              // residual row / bonus row of p
      a.rowinfo[2 * (int64_t)lr + 1] = acc < w ? (long long)lr * k + acc : -1;  // draft row (residual only)
      hi[r] = (uint8_t)acc;
    }
    set_status(a.status, vbad);
    __syncthreads();
    auto emitted = [&](int r) -> long long {
      const int gr = row0 + r;
      if (gr < ep0 || gr >= ep1) return 0;
      int n = hi[r] + 1;
      if (a.cap) n = min(n, max(a.cap[gr - ep0], 0));
      return n;
    };
    const long long tot_tok = cluster_row_scan(cluster, sh, 5, nrows, emitted, [&](int r, long long ex) {
      const int gr = row0 + r;
      if (gr < ep0 || gr >= ep1) return;
      const int lr = gr - ep0;
      a.offsets[lr] = (int32_t)ex;
      const int acc = hi[r];
      const int n = (int)emitted(r);
      for (int i = 0; i < min(acc, n); ++i) a.tokens[ex + i] = a.d[(int64_t)lr * k + i];
    });
    if (g == (int)cluster.num_blocks() - 1 && tid == 0) a.offsets[a.ep_rows] = (int32_t)tot_tok;
  }
  cluster.sync();  // keep every CTA's shared memory alive until the cluster is done reading it
}

// ---- exact heapq replay (accounting only) ------------------------------------------------------------------------
// Mirrors CPython heapq (heapify/_siftup/_siftdown) as driven by select_tetris (selector.py:151-170) and counts every
// _HeapItem.__lt__ (selector.py:128-130).  Single thread by construction: the count is a property of the sequential
// schedule.
struct HeapItem {
  double cum;
  int32_t row, depth;
};

__device__ __forceinline__ bool item_lt(const HeapItem& x, const HeapItem& y, long long& cmp) {
  ++cmp;
  const double nx = -x.cum, ny = -y.cum;  // key = (-cum, row, depth)
  if (nx != ny) return nx < ny;
  if (x.row != y.row) return x.row < y.row;
  return x.depth < y.depth;
}

__device__ void sift_down(HeapItem* h, int start, int pos, long long& cmp) {
  HeapItem nw = h[pos];
  while (pos > start) {
    const int pp = (pos - 1) >> 1;
    const HeapItem parent = h[pp];
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
  const int start = pos;
  const HeapItem nw = h[pos];
  int child = 2 * pos + 1;
  while (child < n) {
    const int right = child + 1;
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
      const int L = len ? len[r] : k;
      if (L > 0) heap[n++] = HeapItem{cum[(int64_t)r * k], r, 1};
    }
    for (int i = n / 2 - 1; i >= 0; --i) sift_up(heap, n, i, cmp);
    inserts = n;
    peak = n;
    while (n > 0 && extracts < C) {
      const HeapItem last = heap[--n];
      HeapItem item = last;
      if (n > 0) {  // heappop
        item = heap[0];
        heap[0] = last;
        sift_up(heap, n, 0, cmp);
      }
      ++extracts;
      const int r = item.row, j = item.depth;
      const int L = len ? len[r] : k;
      if (j < L) {  // heappush
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
    const int L = len ? len[r] : k;
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

namespace tetris {

// Cluster size: enough CTAs that every CTA's keys fit its shared-memory budget.
int select_cluster_size(int B, int k) {
  const size_t cells = (size_t)B * (size_t)(k > 0 ? k : 1);
  const int G = (int)((cells * 8 + kSelKeyBudget - 1) / kSelKeyBudget);
  return G < 1 ? 1 : G;
}

int launch_select(const SelectArgs& args_in, cudaStream_t st) {
  SelectArgs a = args_in;
  const int G = select_cluster_size(a.B, a.k);
  if (G > kMaxCluster)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "B*k=%lld cells exceed the selector's cluster capacity",
                     (long long)a.B * a.k);
  a.RB = (a.B + G - 1) / G;
  const size_t smem = kSelHistBytes + (size_t)a.RB * a.k * 8 + 2 * (size_t)a.RB;
  cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  if (G > 8) {
    e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return abi::cuda_fail(e);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(kSelThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, select_kernel, a);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  return abi::launch_check();
}

}  // namespace tetris

extern "C" int tetris_select_f64(const double* vals, const int32_t* len, int32_t B, int32_t k, int64_t C,
                                 int32_t vals_are_cum, int32_t* windows, int32_t* win_offsets, double* cum_out,
                                 int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                 tetris_stream_t stream) {
  using namespace tetris;
  (void)ws;
  (void)ws_bytes;  // the selector keeps everything in (distributed) shared memory
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
  SelectArgs a = {};
  a.vals = vals;
  a.len = len;
  a.B = B;
  a.k = k;
  a.C = (long long)C;
  a.vals_are_cum = vals_are_cum;
  a.windows = windows;
  a.win_offsets = win_offsets;
  a.cum_out = cum_out;
  a.stats = (long long*)stats4;
  a.status = status;
  return launch_select(a, (cudaStream_t)stream);
}

extern "C" int tetris_heap_stats_f64(const double* cum, const int32_t* len, int32_t B, int32_t k, int64_t C,
                                     int64_t* stats4, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  using namespace tetris;
  if (C < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0, got %lld", (long long)C);
  if (B < 0 || k < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "bad shape B=%d k=%d", B, k);
  if (!stats4) return abi::fail(TETRIS_INVALID_ARGUMENT, "stats4 is required");
  const size_t need = tetris_workspace_bytes(TETRIS_OP_SELECT, B, k, 0);
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
