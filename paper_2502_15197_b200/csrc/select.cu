// Stages (1)+(2): prefix products and TETRIS capacity-constrained selection (global top-C), sm_100a.
//
// Reference semantics: cumulative_products (selector.py:95-110) + select_tetris (selector.py:133-176) with the
// heap key (-cum, row, depth) of _HeapItem (selector.py:113-130).  The heap merge of per-row lists takes exactly
// the C smallest cells under key (env desc, row asc, depth asc), env = the row's prefix-min of cum (for prefix
// products env == cum because fp rounding is monotone).  Rows are monotone in that key, so the selection is a
// per-row prefix and the kernel never materialises a sorted order:
//   * a thread-block cluster of G CTAs (1..16) owns the batch, one row per thread: the work is instruction-bound,
//     so the rows are spread over up to 16 SMs; keys live in registers (k <= 16) or, for deep / very large
//     batches, in shared memory ([depth][row], row stride padded to 1 mod 16: conflict-free both ways);
//   * an MSB-first 8-bit radix select keeps, per row, the sub-range [lo,hi) of cells matching the current key
//     prefix (contiguous because keys are non-decreasing along a row), so a pass only touches undecided cells;
//     each CTA folds its per-warp histograms and adds them with DSMEM atomics into CTA 0's triple-buffered
//     cluster histogram — one cluster barrier per pass — and every CTA then derives the same digit;
//   * it stops as soon as the bucket holding the C-th cell is taken whole; if all 64 bits are resolved the
//     remaining `need` cells are exact key ties and are taken in row-major order (row asc, then depth asc).
// Optional epilogue (the fused step): the first rejection of every request from the accept verdicts (computed by
// extra CTAs of the same cooperative launch, one thread per drafted position, concurrently with the selection),
// the row to resample from, and the compaction offsets.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace cg = cooperative_groups;

namespace tetris {

constexpr int kSelMaxThreads = 1024;
constexpr int kMaxCluster = 16;
constexpr int kRegK = 16;                       // register path: k <= 16 and one row per thread
constexpr size_t kSelKeyBudget = 160 * 1024;    // shared-memory path: keys + lo/hi per CTA

struct SelShared {
  uint32_t cl_hist[3][256];  // cluster histogram (meaningful in CTA 0), triple-buffered by pass
  long long part[8];
  long long tmp[33];
  uint32_t wt[8];
};

// Cluster barrier; a plain CTA barrier when the cluster is a single CTA (no cluster-scope release/acquire fence).
__device__ __forceinline__ void cl_sync(cg::cluster_group& cluster) {
  if (cluster.num_blocks() == 1)
    __syncthreads();
  else
    cluster.sync();
}

// Cluster-wide exclusive scan over rows in row order.  Rows of CTA g are [g*RB, g*RB + nrows), thread t handles
// rows base + t.  `val(r)` gives a row's value, `use(r, excl)` consumes its exclusive prefix.  Returns the total.
template <typename ValF, typename UseF>
__device__ long long cluster_row_scan(cg::cluster_group& cluster, SelShared& sh, int slot, int nrows, ValF val,
                                      UseF use) {
  const int tid = threadIdx.x, nt = blockDim.x;
  long long local = 0;
  for (int base = 0; base < nrows; base += nt) {
    const int r = base + tid;
    local += (r < nrows) ? val(r) : 0;
  }
  long long cta_total;
  block_excl_scan<long long>(local, sh.tmp, cta_total);
  if (tid == 0) sh.part[slot] = cta_total;
  cl_sync(cluster);
  long long before = 0, total = 0;
  const unsigned me = cluster.block_rank();
  for (unsigned g = 0; g < cluster.num_blocks(); ++g) {
    const long long v = *cluster.map_shared_rank(&sh.part[slot], g);
    if (g < me) before += v;
    total += v;
  }
  long long carry = before;
  for (int base = 0; base < nrows; base += nt) {
    const int r = base + tid;
    const long long v = (r < nrows) ? val(r) : 0;
    long long tot;
    const long long ex = block_excl_scan<long long>(v, sh.tmp, tot);
    if (r < nrows) use(r, carry + ex);
    carry += tot;
  }
  return total;
}

// One radix pass' digit decision from the cluster histogram `h` (256 bins): every CTA computes the same result.
// Threads 0..127 (warps 0..3) each own bins 2t, 2t+1.  Returns via sh-free registers of the calling threads only;
// the caller broadcasts with __syncthreads through `out`.
__device__ __forceinline__ void pick_digit(const uint32_t* h, long long need, SelShared& sh, int* out_digit,
                                           long long* out_need, int* out_done) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 128) {
    const uint32_t x0 = h[2 * tid], x1 = h[2 * tid + 1];
    const uint32_t x = x0 + x1;
    const uint32_t incl = warp_incl_scan<uint32_t>(x, lane);
    if (lane == 31) sh.wt[warp] = incl;
    asm volatile("bar.sync 1, 128;" ::: "memory");  // warps 0..3 only
    uint32_t base = 0;
    for (int w = 0; w < warp; ++w) base += sh.wt[w];
    const long long e0 = (long long)base + incl - x;  // bins before 2*tid
    if (e0 < need && need <= e0 + x0) {
      *out_digit = 2 * tid;
      *out_need = need - e0;
      *out_done = (need - e0 == (long long)x0);
    } else if (e0 + x0 < need && need <= e0 + x) {
      *out_digit = 2 * tid + 1;
      *out_need = need - e0 - x0;
      *out_done = (need - e0 - x0 == (long long)x1);
    }
  }
}

constexpr int kRegMaxThreads = 512;  // register path: <= 512 threads so each may hold 128 registers

template <bool REG>
__global__ void __launch_bounds__(REG ? kRegMaxThreads : kSelMaxThreads, 1) select_kernel(const SelectArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ SelShared sh;
  __shared__ int s_digit, s_done;
  __shared__ long long s_need;
  cg::cluster_group cluster = cg::this_cluster();
  const int nt = blockDim.x, nw = nt >> 5;
  uint32_t(*hist)[256] = reinterpret_cast<uint32_t(*)[256]>(smem);  // per-warp histograms
  const int RB = a.RB, k = a.k;
  // shared-memory path: keys [k][KS], KS = RB padded to 1 (mod 16) so the transposing stores of the staging loop
  // and the per-row accesses are both bank-conflict free; register path: no key array
  const int KS = REG ? 0 : (RB | 15) + 2;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem + (size_t)nw * 256 * sizeof(uint32_t));
  uint8_t* lo = reinterpret_cast<uint8_t*>(keys + (size_t)k * KS);
  uint8_t* hi = lo + RB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = (int)cluster.block_rank();
  if (blockIdx.x >= cluster.num_blocks()) {
    // ---- accept role (clusters 1..): verify_token on every drafted position of the local rows, one thread per
    //      position, concurrently with the selection in cluster 0.  Verdict byte: bit0 accept
    //      (accept_model.py:311-313), bit1 draft token outside the vocabulary, bit2 uniform outside [0, 1).
    const int acta = blockIdx.x - cluster.num_blocks();
    const int64_t n = (int64_t)a.ep_rows * k, stride = (int64_t)a.accept_ctas * nt;
    const int32_t* llen = a.len ? a.len + a.ep_row0 : nullptr;
    for (int64_t e = (int64_t)acta * nt + tid; e < n; e += stride) {
      const int b = (int)(e / k), j = (int)(e - (int64_t)b * k);
      const int L = llen ? llen[b] : k;
      uint8_t v = 0;
      if (j < L) {
        const int t = a.d[e];
        const double u = a.u_acc[e];
        v = (u >= 0.0 && u < 1.0) ? 0 : 4;
        if (t < 0 || t >= a.V) {
          v |= 2;
        } else {
          const double s = gather_q(a, e, t);
          const double m = gather_p(a, (int64_t)b * (k + 1) + j, t);
          v |= ((s <= m) || (u < m / s)) ? 1 : 0;
        }
      }
      a.acc_bytes[e] = v;
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(a.acc_counter, 1);
    }
    return;
  }
  const int row0 = g * RB;
  const int nrows = max(0, min(a.B, row0 + RB) - row0);
  const bool stamp = a.dbg != nullptr && g == 0 && tid == 0;
  if (stamp) a.dbg[0] = clock64();
  for (int i = tid; i < 3 * 256; i += nt) (&sh.cl_hist[0][0])[i] = 0;

  uint64_t key[REG ? kRegK : 1];  // register path: this thread's row (row tid of the CTA)
  int lo_r = 0, hi_r = 0;
  uint32_t bad = 0;
  long long nvalid = 0;
  if constexpr (REG) {
    // ---- phase 0 (register path): the row's k values loaded at once, prefix products, envelope, keys ----------
    const int r = tid;
    int L = 0;
    if (r < nrows) {
      const int gr = row0 + r;
      L = a.len ? a.len[gr] : k;
      if (L < 0 || L > k) {
        bad |= TETRIS_ST_BAD_VALUE;
        L = L < 0 ? 0 : k;
      }
      const double* row = a.vals + (int64_t)gr * k;
      double v[kRegK];
#pragma unroll
      for (int j = 0; j < kRegK; ++j) v[j] = j < L ? row[j] : 0.0;
      double cum = 1.0, env = 0.0;
#pragma unroll
      for (int j = 0; j < kRegK; ++j) {
        if (j < L) {
          if (a.vals_are_cum) {
            cum = v[j];
            if (isnan(cum)) bad |= TETRIS_ST_BAD_VALUE;
          } else {
            if (!(v[j] >= 0.0 && v[j] <= 1.0)) bad |= TETRIS_ST_BAD_VALUE;  // accept_model.py:55-59
            cum = __dmul_rn(cum, v[j]);  // selector.py:104-108, left to right
          }
          if (a.cum_out) a.cum_out[(int64_t)gr * k + j] = cum;
          env = (j == 0 || cum < env) ? cum : env;
          key[j] = desc_key(env);
        } else {
          key[j] = ~0ull;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < kRegK; ++j) key[j] = ~0ull;
    }
    lo_r = 0;
    hi_r = L;
    nvalid = L;
  } else {
    // ---- phase 0 (shared-memory path): coalesced staging into [depth][row], then products / keys in place ------
    const double* src = a.vals + (int64_t)row0 * k;
    const int n = nrows * k;
    for (int e0 = 0; e0 < n; e0 += 8 * nt) {  // 8 independent loads in flight per thread
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = e0 + i * nt + tid;
        v[i] = e < n ? src[e] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = e0 + i * nt + tid;
        if (e < n) {
          const int r = e / k, j = e - r * k;
          keys[(size_t)j * KS + r] = (uint64_t)__double_as_longlong(v[i]);
        }
      }
    }
    __syncthreads();
    for (int r = tid; r < nrows; r += nt) {
      const int gr = row0 + r;
      int L = a.len ? a.len[gr] : k;
      if (L < 0 || L > k) {
        bad |= TETRIS_ST_BAD_VALUE;
        L = L < 0 ? 0 : k;
      }
      double cum = 1.0, env = 0.0;
      for (int j = 0; j < L; ++j) {
        const double v = __longlong_as_double((long long)keys[(size_t)j * KS + r]);
        if (a.vals_are_cum) {
          cum = v;
          if (isnan(v)) bad |= TETRIS_ST_BAD_VALUE;
        } else {
          if (!(v >= 0.0 && v <= 1.0)) bad |= TETRIS_ST_BAD_VALUE;  // accept_model.py:55-59
          cum = __dmul_rn(cum, v);
        }
        if (a.cum_out) a.cum_out[(int64_t)gr * k + j] = cum;
        env = (j == 0 || cum < env) ? cum : env;
        keys[(size_t)j * KS + r] = desc_key(env);
      }
      lo[r] = 0;
      hi[r] = (uint8_t)L;
      nvalid += L;
    }
  }
  set_status(a.status, bad);
  if (stamp) a.dbg[1] = clock64();
  long long cta_valid;
  block_excl_scan<long long>(nvalid, sh.tmp, cta_valid);
  if (tid == 0) sh.part[0] = cta_valid;
  cl_sync(cluster);  // also orders the cl_hist zeroing before any remote add
  long long N = 0;
  for (unsigned c = 0; c < cluster.num_blocks(); ++c) N += *cluster.map_shared_rank(&sh.part[0], c);

  // ---- phase 1: radix select ---------------------------------------------------------------------------------
  const int mode = (a.C <= 0 || N == 0) ? 0 : (a.C >= N ? 1 : 2);  // 0: nothing, 1: everything, 2: radix
  long long need = a.C;
  bool done = mode != 2;
  if (stamp) a.dbg[2] = clock64();
  int npass = 0;
  uint32_t* h0 = cluster.map_shared_rank(&sh.cl_hist[0][0], 0);  // CTA 0's cluster histogram buffers
  for (int pass = 0; pass < 8 && !done; ++pass) {
    ++npass;
    const int shift = 56 - 8 * pass;
    const int buf = pass % 3;
    for (int i = lane; i < 256; i += 32) hist[warp][i] = 0;
    __syncwarp();
    if constexpr (REG) {
      if (lo_r < hi_r) {  // run lengths of the row's undecided cells (digits are non-decreasing along the row)
        uint32_t cur = 0xFFFFFFFFu, cnt = 0;
#pragma unroll
        for (int j = 0; j < kRegK; ++j) {
          if (j >= lo_r && j < hi_r) {
            const uint32_t dg = (uint32_t)(key[j] >> shift) & 255u;
            if (dg == cur) {
              ++cnt;
            } else {
              if (cnt) atomicAdd(&hist[warp][cur], cnt);
              cur = dg;
              cnt = 1;
            }
          }
        }
        atomicAdd(&hist[warp][cur], cnt);
      }
    } else {
      for (int r = tid; r < nrows; r += nt) {
        const int l = lo[r], h = hi[r];
        if (l >= h) continue;
        uint32_t cur = (uint32_t)(keys[(size_t)l * KS + r] >> shift) & 255u, cnt = 1;
        for (int j = l + 1; j < h; ++j) {
          const uint32_t dg = (uint32_t)(keys[(size_t)j * KS + r] >> shift) & 255u;
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
    }
    __syncthreads();
    // fold the warp histograms and add them into CTA 0's cluster histogram (DSMEM atomics)
    for (int bin = tid; bin < 256; bin += nt) {
      uint32_t x = 0;
      for (int w = 0; w < nw; ++w) x += hist[w][bin];
      if (x) atomicAdd(h0 + buf * 256 + bin, x);
    }
    cl_sync(cluster);
    // CTA 0 clears the buffer of pass+2 (last read in pass-1, before this barrier; next written after pass+1's)
    if (g == 0)
      for (int i = tid; i < 256; i += nt) sh.cl_hist[(pass + 2) % 3][i] = 0;
    pick_digit(h0 + buf * 256, need, sh, &s_digit, &s_need, &s_done);
    __syncthreads();
    const uint32_t D = (uint32_t)s_digit;
    need = s_need;
    const bool take_all = s_done;
    if constexpr (REG) {
      int nless = 0, neq = 0;
#pragma unroll
      for (int j = 0; j < kRegK; ++j) {
        if (j >= lo_r && j < hi_r) {
          const uint32_t dg = (uint32_t)(key[j] >> shift) & 255u;
          nless += dg < D;
          neq += dg == D;
        }
      }
      const int l = lo_r + nless, e = l + neq;
      lo_r = take_all ? e : l;  // take_all: the whole digit-D bucket is selected
      hi_r = e;
    } else {
      for (int r = tid; r < nrows; r += nt) {
        int l = lo[r];
        const int h = hi[r];
        while (l < h && (((uint32_t)(keys[(size_t)l * KS + r] >> shift) & 255u) < D)) ++l;
        int e = l;
        while (e < h && (((uint32_t)(keys[(size_t)e * KS + r] >> shift) & 255u) == D)) ++e;
        lo[r] = (uint8_t)(take_all ? e : l);
        hi[r] = (uint8_t)e;
      }
    }
    done = take_all;
  }
  if constexpr (REG) {
    if (tid < nrows) {
      lo[tid] = (uint8_t)lo_r;
      hi[tid] = (uint8_t)hi_r;
    }
  }
  __syncthreads();
  if (stamp) {
    a.dbg[3] = clock64();
    a.dbg[9] = npass;
  }

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
  // windows, win_offsets and the PolicyStats closed forms (selector.py:150-170) in ONE scan of a packed value:
  // window (bits 0..23) | inserts term (24..47) | non-empty row (48..63); no field can overflow (B*k < 2^24).
  // extracts = sum w; inserts = nz + sum(w - [w == L > 0]); peak_queue = nz; all zero when C == 0.
  const long long packed_total = cluster_row_scan(
      cluster, sh, 2, nrows,
      [&](int r) {
        const int L = row_len(r);
        const int w = mode == 0 ? 0 : (mode == 1 ? L : lo[r]);
        const long long ins = w - ((w == L && L > 0) ? 1 : 0);
        return (long long)w | (ins << 24) | ((long long)(L > 0) << 48);
      },
      [&](int r, long long ex) {
        const int L = row_len(r);
        const int w = mode == 0 ? 0 : (mode == 1 ? L : lo[r]);
        a.windows[row0 + r] = w;
        if (a.win_offsets) a.win_offsets[row0 + r] = (int32_t)(ex & 0xFFFFFF);
        lo[r] = (uint8_t)w;  // lo now holds the window
      });
  const long long tot_w = packed_total & 0xFFFFFF;
  if (g == (int)cluster.num_blocks() - 1 && tid == 0 && a.win_offsets) a.win_offsets[a.B] = (int32_t)tot_w;
  if (a.stats && g == 0 && tid == 0) {
    const long long nz = (packed_total >> 48) & 0xFFFF, ins = (packed_total >> 24) & 0xFFFFFF;
    const bool any = a.C > 0;
    a.stats[0] = any ? tot_w : 0;
    a.stats[1] = any ? nz + ins : 0;
    a.stats[2] = any ? nz : 0;
    a.stats[3] = -1;
  }
  if (stamp) a.dbg[4] = clock64();

  // ---- optional epilogue: first rejection, row to resample from, compaction offsets (fused step) ---------------
  if (a.p != nullptr || a.zp != nullptr) {
    uint32_t vbad = 0;
    const int ep0 = a.ep_row0, ep1 = a.ep_row0 + a.ep_rows;
    if (a.accept_ctas > 0 && tid == 0) {
      // the accept CTAs of this launch run concurrently (cooperative launch => co-resident); wait for all of them
      int seen;
      do {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(a.acc_counter) : "memory");
        if (seen < a.accept_ctas) __nanosleep(200);
      } while (seen < a.accept_ctas);
    }
    __syncthreads();
    for (int r = tid; r < nrows; r += nt) {
      const int gr = row0 + r;
      if (gr < ep0 || gr >= ep1) continue;
      const int lr = gr - ep0;
      const int w = lo[r];
      int acc = w;
      if (a.acc_bytes) {
        // verdicts precomputed by pre_accept_kernel: bit0 accept, bit1 bad token, bit2 bad uniform
        const uint8_t* ab = a.acc_bytes + (int64_t)lr * k;
        for (int j0 = 0; j0 < w && acc == w; j0 += 16) {
          uint8_t v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = (j0 + i < w) ? ab[j0 + i] : (uint8_t)1;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (acc != w || j0 + i >= w) continue;
            vbad |= (v[i] & 2 ? TETRIS_ST_BAD_TOKEN : 0u) | (v[i] & 4 ? TETRIS_ST_BAD_UNIFORM : 0u);
            if (!(v[i] & 1)) acc = j0 + i;
          }
        }
      } else {
        const int64_t uoff = a.u_packed ? (int64_t)a.win_offsets[gr] : (int64_t)lr * k;
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
            s[i] = ok ? gather_q(a, (int64_t)lr * k + j, t[i]) : 0.0;
            m[i] = ok ? gather_p(a, (int64_t)lr * (k + 1) + j, t[i]) : 0.0;
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
      }
      a.accepted[lr] = acc;
      a.rowinfo[2 * (int64_t)lr] = (long long)lr * (k + 1) + acc;              // residual row / bonus row of p
      a.rowinfo[2 * (int64_t)lr + 1] = acc < w ? (long long)lr * k + acc : -1;  // draft row (residual only)
      if (a.rowlse) {  // logits form: the two rows' lse beside their indices (one load round for the producer)
        a.rowlse[2 * (int64_t)lr] = a.lse_p[(int64_t)lr * (k + 1) + acc];
        a.rowlse[2 * (int64_t)lr + 1] = acc < w ? a.lse_q[(int64_t)lr * k + acc] : 0.f;
      }
      hi[r] = (uint8_t)acc;
    }
    set_status(a.status, vbad);
    __syncthreads();
    if (stamp) a.dbg[5] = clock64();
    auto emitted = [&](int r) -> long long {
      const int gr = row0 + r;
      if (gr < ep0 || gr >= ep1) return 0;
      int n = hi[r] + 1;
      if (a.cap) n = min(n, max(a.cap[gr - ep0], 0));
      return n;
    };
    const long long tot_tok = cluster_row_scan(cluster, sh, 5, nrows, emitted, [&](int r, long long ex) {
      const int gr = row0 + r;
      if (gr >= ep0 && gr < ep1) a.offsets[gr - ep0] = (int32_t)ex;
    });
    if (g == (int)cluster.num_blocks() - 1 && tid == 0) a.offsets[a.ep_rows] = (int32_t)tot_tok;
  }
  if (stamp) a.dbg[6] = clock64();
  cluster.sync();  // keep every CTA's shared memory alive until the cluster is done reading it
  if (a.accept_ctas > 0 && g == 0 && tid == 0) *a.acc_counter = 0;  // every CTA of cluster 0 is past its wait
}

// ---- exact heapq replay (accounting only) ------------------------------------------------------------------------
// Mirrors CPython heapq (heapify/_siftup/_siftdown) as driven by select_tetris (selector.py:151-170) and counts every
// _HeapItem.__lt__ (selector.py:128-130).  Single thread by construction: the count is a property of the sequential
// schedule.
// Items carry the selection's integer key instead of the double: desc_key(cum) orders like -cum (with -0.0 == +0.0,
// as Python compares them) and the tie word row << 8 | depth like (row, depth), so one _HeapItem.__lt__ is a 96-bit
// integer compare (no fp64 compare in the dependent chain).  Scores are validated (no NaN) before this runs.
struct HeapItem {
  uint64_t key;
  uint32_t tie;
  uint32_t pad;
};

__device__ __forceinline__ bool item_lt(const HeapItem& x, const HeapItem& y, long long& cmp) {
  ++cmp;
  return x.key < y.key || (x.key == y.key && x.tie < y.tie);  // key = (-cum, row, depth)
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

// The replay is one dependent chain of heap accesses, so their latency is the cost: the heap (16 B per row), the
// cells' keys and the row lengths live in shared memory when they fit (staged by the whole CTA first), otherwise
// the heap and the keys in the workspace.
__global__ void heap_stats_kernel(const double* __restrict__ cum_g, const int32_t* __restrict__ len_g, int B, int k,
                                  long long C, long long* stats, HeapItem* heap_g, uint64_t* keys_g,
                                  int in_smem) {
  extern __shared__ __align__(16) uint8_t hs_smem[];
  HeapItem* heap = in_smem ? (HeapItem*)hs_smem : heap_g;
  uint64_t* keys = in_smem ? (uint64_t*)(hs_smem + (size_t)B * sizeof(HeapItem)) : keys_g;
  int* lens = in_smem ? (int*)(keys + (size_t)B * k) : nullptr;
  for (long long i = threadIdx.x; i < (long long)B * k; i += blockDim.x) keys[i] = desc_key(cum_g[i]);
  if (lens)
    for (int r = threadIdx.x; r < B; r += blockDim.x) lens[r] = len_g ? len_g[r] : k;
  __syncthreads();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  auto L_of = [&](int r) { return lens ? lens[r] : (len_g ? len_g[r] : k); };
  long long cmp = 0, extracts = 0, inserts = 0, peak = 0;
  if (C > 0) {
    int n = 0;
    for (int r = 0; r < B; ++r)
      if (L_of(r) > 0) heap[n++] = HeapItem{keys[(int64_t)r * k], (uint32_t)r << 8 | 1u, 0u};
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
      const int r = (int)(item.tie >> 8), j = (int)(item.tie & 0xFFu);
      if (j < L_of(r)) {  // heappush
        heap[n] = HeapItem{keys[(int64_t)r * k + j], (uint32_t)r << 8 | (uint32_t)(j + 1), 0u};
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

// Launch shape: the register path spreads the rows over up to 16 CTAs (one row per thread, >= 128 threads per CTA);
// the shared-memory path sizes the cluster so every CTA's keys fit its shared memory.
struct SelShape {
  int G, T, RB;
  bool reg;
};

SelShape select_shape(int B, int k) {
  SelShape s;
  s.reg = k <= kRegK && B <= kMaxCluster * kRegMaxThreads;
  if (s.reg) {
    s.G = B <= 128 ? 1 : (B + 127) / 128;
    if (s.G > kMaxCluster) s.G = kMaxCluster;
    s.RB = (B + s.G - 1) / s.G;
    s.T = 128;
    while (s.T < s.RB) s.T *= 2;
  } else {
    const size_t cells = (size_t)B * (size_t)(k > 0 ? k : 1);
    s.G = (int)((cells * 8 + kSelKeyBudget - 1) / kSelKeyBudget);
    if (s.G < 1) s.G = 1;
    s.RB = (B + s.G - 1) / s.G;
    s.T = kSelMaxThreads;
  }
  if (s.RB < 1) s.RB = 1;
  return s;
}

static long long* g_debug = nullptr;
void set_debug_buffer(long long* p) { g_debug = p; }
long long* debug_buffer() { return g_debug; }

int launch_select(const SelectArgs& args_in, cudaStream_t st) {
  if (select1_eligible(args_in.B, args_in.k)) return launch_select1(args_in, st);
  if (args_in.gscratch != nullptr) return launch_gselect(args_in, args_in.gscratch, st);
  SelectArgs a = args_in;
  a.dbg = g_debug;
  const SelShape sh = select_shape(a.B, a.k);
  const int G = sh.G;
  if (G > kMaxCluster)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "B*k=%lld cells exceed the selector's cluster capacity",
                     (long long)a.B * a.k);
  a.RB = sh.RB;
  const size_t KS = sh.reg ? 0 : (size_t)((a.RB | 15) + 2);
  const size_t smem = (size_t)(sh.T / 32) * 256 * 4 + KS * a.k * 8 + 2 * (size_t)a.RB;
  auto kern = sh.reg ? select_kernel<true> : select_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  if (G > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return abi::cuda_fail(e);
  }
  // accept CTAs (whole clusters after cluster 0): one thread per drafted position, within the co-resident limit
  int extra_clusters = 0;
  if (a.acc_bytes && a.accept_ctas > 0) {
    const int num_sms = abi::device_sm_count();
    const long long n = (long long)a.ep_rows * a.k;
    long long want = (n + sh.T - 1) / sh.T;
    const long long cap = (long long)(num_sms - G) / G * G;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    extra_clusters = (int)((want + G - 1) / G);
    a.accept_ctas = extra_clusters * G;
  } else {
    a.accept_ctas = 0;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G * (1 + extra_clusters), 1, 1);
  cfg.blockDim = dim3(sh.T, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // cluster 0 waits on the accept CTAs: they must be co-resident
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = extra_clusters > 0 ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess && extra_clusters > 0) {
    // cooperative cluster launch unavailable: run the verdicts as their own grid first, then the selection
    cudaGetLastError();
    int rc = launch_pre_accept(a, st);
    if (rc) return rc;
    a.accept_ctas = 0;
    cfg.gridDim = dim3(G, 1, 1);
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  if (e != cudaSuccess) return abi::cuda_fail(e);
  return abi::launch_check();
}

}  // namespace tetris

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
  if ((k > 0 && !vals) || !windows) return abi::fail(TETRIS_INVALID_ARGUMENT, "vals and windows are required");
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
  if (ws && ws_bytes >= abi::region_offset(TETRIS_OP_SELECT, B, k, 0, abi::WS_GSEL) + abi::kGselScratchBytes)
    a.gscratch = abi::ws_region(ws, TETRIS_OP_SELECT, B, k, 0, abi::WS_GSEL);
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
  constexpr size_t kMaxSmem = 200 * 1024;
  const size_t smem_all = (size_t)B * sizeof(HeapItem) + (size_t)B * k * 8 + (size_t)B * 4;
  const int in_smem = smem_all <= kMaxSmem;
  cudaError_t e = abi::ensure_smem(heap_stats_kernel, in_smem ? smem_all : 0);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  // workspace fallback: the heap in WS_KEYS ([B] items, 16 B each), the cell keys behind it
  uint8_t* base = (uint8_t*)abi::ws_region(ws, TETRIS_OP_SELECT, B, k, 0, abi::WS_KEYS);
  heap_stats_kernel<<<1, 256, in_smem ? smem_all : 0, (cudaStream_t)stream>>>(
      cum, len, B, k, (long long)C, (long long*)stats4, (HeapItem*)base,
      (uint64_t*)(base + (size_t)B * sizeof(HeapItem)), in_smem);
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
