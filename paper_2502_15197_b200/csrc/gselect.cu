// Stages (1)+(2) for large batches (B*k > 16384: cfg4, cfg5, the gathered multi-GPU selection): grid-wide
// prefix products + TETRIS global top-C on every SM (sm_100a).
//
// Same semantics as select1_kernel / select_kernel — cumulative_products (selector.py:95-110) + select_tetris
// (selector.py:133-176) under the _HeapItem key (-cum, row, depth) (selector.py:113-130) over each row's prefix-min
// envelope — spread over up to one CTA per SM so the per-row serial work (16 dependent multiplies per row) and the
// loads of the 1-2 MB score matrix run on every SM instead of one cluster:
//   * CTA g owns the contiguous rows [g*RB, (g+1)*RB), one row per thread, keys in shared memory [depth][row];
//   * MSB-first radix select with 11/11/11/11/10/10-bit digits: each CTA adds its histogram of the still-undecided
//     cells into one 2048-bin histogram in L2 (triple-buffered by pass), a grid barrier closes the pass, and every
//     CTA derives the same digit from the global histogram (warp-parallel pick) — no second barrier per pass;
//   * exact ties left after 64 bits, windows / win_offsets / PolicyStats and the compaction offsets are row-order
//     scans: CTA totals in L2, one grid barrier, each CTA adds the totals of the CTAs before it;
//   * the fused step's accept test runs at the start on the CTA's own rows (its gathers overlap the score loads), so
//     no separate accept CTAs are needed.
// The grid barrier is a generation barrier on two words of the workspace (left consistent for the next launch);
// the launch is cooperative, so all CTAs are co-resident.
#include <cooperative_groups.h>
#ifndef GSEL_CELLS_PER_CTA
#define GSEL_CELLS_PER_CTA 4096
#endif

#include "abi_util.h"
#include "common.cuh"
#include "launch.h"

namespace tetris {

constexpr int kGThreads = 512;
constexpr long long kGCellsPerCta = GSEL_CELLS_PER_CTA;
constexpr int kGBins = 2048;
constexpr int kGMaxGrid = 256;
constexpr size_t kGKeyBudget = 150 * 1024;  // keys + verdicts per CTA

struct GScratch {          // in the workspace (WS_GSEL), zero-initialised; every launch leaves it reusable
  uint32_t hist[3][kGBins];  // global radix histograms, triple-buffered by pass; zero between launches
  unsigned bar_count, bar_gen;  // barrier counter, exit counter
  long long part[2][kGMaxGrid];  // per-CTA totals of the row-order scans
};

static_assert(sizeof(GScratch) <= abi::kGselScratchBytes, "WS_GSEL region too small");

struct GShared {
  uint32_t hist[kGBins];
  long long tmp[33];
  long long before, total;
  int digit, done;
  long long need, N;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier over the whole (co-resident) grid: a counter that only grows within a launch — barrier i completes
// when it reaches (i + 1) * gridDim.x, so a waiting CTA needs no second round trip to learn it (about half the cost
// of a generation barrier, measured with tools/micro/gridbar.cu).  grid_exit() returns it to zero for the next
// launch once every CTA has passed its last barrier.  `nb` counts the barriers this CTA has passed (the same
// sequence in every CTA).
__device__ void grid_sync(GScratch* gs, unsigned& nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // release this CTA's writes (ordered before by the bar.sync)
    atomicAdd(&gs->bar_count, 1u);
    const unsigned target = (nb + 1u) * gridDim.x;
    while (ld_acquire_u32(&gs->bar_count) < target) {
    }
  }
  ++nb;
  __syncthreads();
}

__device__ void grid_exit(GScratch* gs) {
  if (threadIdx.x == 0 && atomicAdd(&gs->bar_gen, 1u) == gridDim.x - 1) {
    gs->bar_count = 0u;
    gs->bar_gen = 0u;
  }
}

// Cross-CTA exclusive prefix of a per-CTA total published in part[] before the last grid_sync: sh.before = sum over
// CTAs < blockIdx.x, sh.total = sum over all.  Warp 0 reads the totals; the caller __syncthreads() afterwards.
__device__ __forceinline__ void cta_prefix(const long long* part, GShared& sh) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    long long bf = 0, tot = 0;
    for (int c = lane; c < (int)gridDim.x; c += 32) {
      const long long v = __ldcg(part + c);
      tot += v;
      if (c < (int)blockIdx.x) bf += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bf += __shfl_xor_sync(kFull, bf, o);
      tot += __shfl_xor_sync(kFull, tot, o);
    }
    if (lane == 0) {
      sh.before = bf;
      sh.total = tot;
    }
  }
}

// Radix schedule.  Pass 0 is a CLAMPED digit of key bits 63..48: for a score in [2^-127, 1] those bits are its
// exponent and the top 4 mantissa bits (desc_key maps 1.0 to 0x400F..), so probabilities get 16 bins per binade
// instead of the 2 binades per bin a plain top-11-bit digit gives them (cfg4 data: one pass fewer); bin 0 collects
// every key below 0x4010 << 48 (scores >= 1.0, any cum above 1 in vals_are_cum mode) and bin 2047 every key from
// 0x480E << 48 up (scores below ~2^-127, zero, negative cums).  Every bin is an interval of keys, digits are monotone
// in the key, so the row-wise run-length histograms and range updates still apply.  After a middle bin (an exact
// 16-bit prefix) the passes refine bits 47..0 as 11/11/11/11/4; after an edge bin, bits 63..0 as 11/11/11/11/10/10.
struct GDigit {
  int shift;
  uint32_t mask;
  int clamp;
};
__device__ __forceinline__ uint32_t gdigit(uint64_t key, const GDigit& d) {
  if (d.clamp) {
    const long long x = (long long)(key >> 48) - 0x400F;
    return x < 0 ? 0u : (x > 2047 ? 2047u : (uint32_t)x);
  }
  return (uint32_t)(key >> d.shift) & d.mask;
}
__device__ __forceinline__ GDigit gpass(int pass, bool edge) {
  if (pass == 0) return GDigit{48, 2047u, 1};
  if (!edge) {  // bits 47..0
    const int sh = 48 - 11 * pass;
    return sh >= 0 ? GDigit{sh, 2047u, 0} : GDigit{0, 15u, 0};
  }
  const int w = pass <= 4 ? 11 : 10, sh = 64 - (pass <= 4 ? 11 * pass : 44 + 10 * (pass - 4));
  return GDigit{sh, (1u << w) - 1u, 0};
}
__device__ __forceinline__ int glast_pass(bool edge) { return edge ? 6 : 5; }

struct GArgs {
  SelectArgs a;
  GScratch* gs;
  int RB;
};

__global__ void __launch_bounds__(kGThreads, 1) gselect_kernel(const GArgs ga) {
  const SelectArgs& a = ga.a;
  GScratch* gs = ga.gs;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ __align__(16) GShared sh;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x, lane = tid & 31, k = a.k, B = a.B, RB = ga.RB;
  const int r0 = min(B, (int)blockIdx.x * RB), nr = max(0, min(B, r0 + RB) - r0);
  const int KS = (RB | 15) + 2;  // keys[j * KS + r]
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint8_t* verd = reinterpret_cast<uint8_t*>(keys + (size_t)k * KS);  // [RB][k] accept verdicts (epilogue)
  const bool row = tid < nr;
  const int gr = r0 + tid;
  const bool stamp = a.dbg != nullptr && blockIdx.x == 0 && tid == 0;
  if (stamp) a.dbg[0] = clock64();
  unsigned nb = 0;  // grid barriers passed

  // ---- accept verdicts of this CTA's rows in the epilogue range, issued first (two dependent gathers each) --------
  const int ep0 = a.ep_row0, ep1 = a.ep_row0 + a.ep_rows;
  if (a.p != nullptr || a.zp != nullptr) {
    const int lo_r = max(r0, ep0), hi_r = min(r0 + nr, ep1);
    for (int e = tid; e < (hi_r - lo_r) * k; e += kGThreads) {
      const int r = lo_r + e / k, j = e - (e / k) * k;
      const int lr = r - ep0;
      const int L = a.len ? a.len[r] : k;
      uint8_t v = 0;
      if (j < L) {
        const int64_t pos = (int64_t)lr * k + j;
        const int t = a.d[pos];
        const double u = a.u_acc[pos];
        v = (u >= 0.0 && u < 1.0) ? 0 : 4;
        if (t < 0 || t >= a.V) {
          v |= 2;
        } else {
          const double s = gather_q(a, pos, t);
          const double m = gather_p(a, (int64_t)lr * (k + 1) + j, t);
          v |= ((s <= m) || (u < m / s)) ? 1 : 0;  // accept_model.py:311-313
        }
      }
      verd[(r - r0) * k + j] = v;
    }
  }

  // ---- phase 0: the CTA's scores (coalesced), prefix products, keys, pass-0 digit histogram ---------------------
  for (int i = tid; i < kGBins; i += kGThreads) sh.hist[i] = 0;
  {
    const double* src = a.vals + (int64_t)r0 * k;
    const int n = nr * k;
    for (int e0 = 0; e0 < n; e0 += 8 * kGThreads) {
      double v[8];
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const int e = e0 + x * kGThreads + tid;
        v[x] = e < n ? __ldg(src + e) : 0.0;
      }
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const int e = e0 + x * kGThreads + tid;
        if (e < n) {
          const int r = e / k, j = e - r * k;
          keys[(size_t)j * KS + r] = (uint64_t)__double_as_longlong(v[x]);
        }
      }
    }
  }
  __syncthreads();
  const GDigit d0 = gpass(0, false);
  uint32_t bad = 0;
  int L = 0, lo = 0, hi = 0;
  if (row) {
    L = a.len ? a.len[gr] : k;
    if (L < 0 || L > k) {
      bad |= TETRIS_ST_BAD_VALUE;
      L = L < 0 ? 0 : k;
    }
    double cum = 1.0, env = 0.0;
    uint32_t cur = 0xFFFFFFFFu, cnt = 0;
    for (int j = 0; j < L; ++j) {
      const double v = __longlong_as_double((long long)keys[(size_t)j * KS + tid]);
      if (a.vals_are_cum) {
        cum = v;
        if (isnan(cum)) bad |= TETRIS_ST_BAD_VALUE;
      } else {
        if (!(v >= 0.0 && v <= 1.0)) bad |= TETRIS_ST_BAD_VALUE;  // accept_model.py:55-59
        cum = __dmul_rn(cum, v);                                  // selector.py:104-108, left to right
      }
      if (a.cum_out) a.cum_out[(int64_t)gr * k + j] = cum;
      env = (j == 0 || cum < env) ? cum : env;
      const uint64_t key = desc_key(env);
      keys[(size_t)j * KS + tid] = key;
      const uint32_t dg = gdigit(key, d0);
      if (dg == cur) {
        ++cnt;
      } else {
        if (cnt) atomicAdd(&sh.hist[cur], cnt);
        cur = dg;
        cnt = 1;
      }
    }
    if (cnt) atomicAdd(&sh.hist[cur], cnt);
    hi = L;
  }
  set_status(a.status, bad);
  __syncthreads();
  for (int i = tid; i < kGBins; i += kGThreads)
    if (sh.hist[i]) atomicAdd(&gs->hist[0][i], sh.hist[i]);
  if (stamp) a.dbg[1] = clock64();
  grid_sync(gs, nb);
  if (stamp) a.dbg[2] = clock64();

  // ---- phase 1: radix passes; one grid barrier each --------------------------------------------------------------
  long long need = a.C, N = 0;
  int mode = 0;  // 0: nothing selected, 1: everything, 2: radix
  bool done = false, edge = false;
  int npass = 0;
  for (int pass = 0; pass < 7; ++pass) {
    ++npass;
    const GDigit dg = gpass(pass, edge);
    // the global histogram, copied through L2 (other CTAs' atomics landed there before the barrier; L1 may hold a
    // stale line from an earlier pass)
    const uint32_t* H = gs->hist[pass % 3];
    for (int i = tid; i < kGBins; i += kGThreads) sh.hist[i] = __ldcg(H + i);
    __syncthreads();
    if (stamp) a.dbg[10 + 5 * pass] = clock64();
    if (tid < 32) {
      uint32_t tot;
      const long long nd = need < 1 ? 1 : (need > 0xFFFFFFFFll ? 0xFFFFFFFFll : need);
      pick_digit_warp(sh.hist, (uint32_t)nd, lane, &sh.digit, &sh.need, &sh.done, &tot);
      if (pass == 0 && lane == 0) sh.N = (long long)tot;
    } else if (blockIdx.x == 0) {
      uint32_t* Hz = gs->hist[(pass + 2) % 3];  // last read before the barrier that ended the previous pass
      for (int i = tid - 32; i < kGBins; i += kGThreads - 32) Hz[i] = 0u;
    }
    __syncthreads();
    if (stamp) a.dbg[11 + 5 * pass] = clock64();
    if (pass == 0) {
      N = sh.N;
      mode = (a.C <= 0 || N == 0) ? 0 : (a.C >= N ? 1 : 2);
      if (mode != 2) break;
    }
    const uint32_t D = (uint32_t)sh.digit;
    need = sh.need;
    const bool take_all = sh.done != 0;
    if (pass == 0) edge = D == 0u || D == 2047u;  // an edge bin is an interval, not a prefix: refine from bit 63
    if (row && lo < hi) {
      int l = lo;
      while (l < hi && gdigit(keys[(size_t)l * KS + tid], dg) < D) ++l;
      int e = l;
      while (e < hi && gdigit(keys[(size_t)e * KS + tid], dg) == D) ++e;
      lo = take_all ? e : l;
      hi = e;
    }
    done = take_all;
    if (done || pass == glast_pass(edge)) break;
    if (stamp) a.dbg[12 + 5 * pass] = clock64();
    // next digit's histogram of the still-undecided cells
    const GDigit nd = gpass(pass + 1, edge);
    __syncthreads();
    for (int i = tid; i < kGBins; i += kGThreads) sh.hist[i] = 0;
    __syncthreads();
    if (row && lo < hi) {
      uint32_t cur = gdigit(keys[(size_t)lo * KS + tid], nd), cnt = 1;
      for (int j = lo + 1; j < hi; ++j) {
        const uint32_t dg = gdigit(keys[(size_t)j * KS + tid], nd);
        if (dg == cur) {
          ++cnt;
        } else {
          atomicAdd(&sh.hist[cur], cnt);
          cur = dg;
          cnt = 1;
        }
      }
      atomicAdd(&sh.hist[cur], cnt);
    }
    __syncthreads();
    if (stamp) a.dbg[13 + 5 * pass] = clock64();
    uint32_t* Hn = gs->hist[(pass + 1) % 3];
    for (int i = tid; i < kGBins; i += kGThreads)
      if (sh.hist[i]) atomicAdd(&Hn[i], sh.hist[i]);
    grid_sync(gs, nb);
    if (stamp) a.dbg[14 + 5 * pass] = clock64();
  }
  if (stamp) {
    a.dbg[3] = clock64();
    a.dbg[9] = npass;
  }

  // ---- phase 2: exact ties in row-major order, then windows / win_offsets / PolicyStats ------------------------
  if (mode == 2 && !done) {
    long long tcnt;
    const long long ex = block_excl_scan<long long>(row ? hi - lo : 0, sh.tmp, tcnt);
    if (tid == 0) gs->part[0][blockIdx.x] = tcnt;
    grid_sync(gs, nb);
    cta_prefix(gs->part[0], sh);
    __syncthreads();
    if (row) {
      long long take = need - (sh.before + ex);
      const long long t = hi - lo;
      take = take < 0 ? 0 : (take > t ? t : take);
      lo += (int)take;
    }
  }
  const int w = !row ? 0 : (mode == 0 ? 0 : (mode == 1 ? L : lo));
  const long long pk = row ? ((long long)w | ((long long)(w - ((w == L && L > 0) ? 1 : 0)) << 24) |
                              ((long long)(L > 0) << 48))
                           : 0;
  long long ctot;
  const long long pex = block_excl_scan<long long>(pk, sh.tmp, ctot);
  if (tid == 0) gs->part[1][blockIdx.x] = ctot;
  grid_sync(gs, nb);
  cta_prefix(gs->part[1], sh);
  __syncthreads();
  if (row) {
    a.windows[gr] = w;
    if (a.win_offsets) a.win_offsets[gr] = (int32_t)((sh.before + pex) & 0xFFFFFF);
  }
  if (blockIdx.x == gridDim.x - 1 && tid == 0) {
    const long long ptot = sh.total;
    const long long tot_w = ptot & 0xFFFFFF;
    if (a.win_offsets) a.win_offsets[B] = (int32_t)tot_w;
    if (a.stats) {
      const long long nz = (ptot >> 48) & 0xFFFF, ins = (ptot >> 24) & 0xFFFFFF;
      const bool any = a.C > 0;
      a.stats[0] = any ? tot_w : 0;
      a.stats[1] = any ? nz + ins : 0;
      a.stats[2] = any ? nz : 0;
      a.stats[3] = -1;
    }
  }
  if (stamp) a.dbg[4] = clock64();

  // ---- epilogue (fused step): first rejection, the row to resample from, compaction offsets ----------------------
  if (a.p != nullptr || a.zp != nullptr) {
    uint32_t vbad = 0;
    const bool mine = row && gr >= ep0 && gr < ep1;
    int n_emit = 0;
    if (mine) {
      const int lr = gr - ep0;
      int acc = w;
      const uint8_t* vb = verd + tid * k;
      for (int j = 0; j < w; ++j) {
        const uint8_t v = vb[j];
        vbad |= (v & 2 ? TETRIS_ST_BAD_TOKEN : 0u) | (v & 4 ? TETRIS_ST_BAD_UNIFORM : 0u);
        if (!(v & 1)) {
          acc = j;
          break;
        }
      }
      a.accepted[lr] = acc;
      a.rowinfo[2 * (int64_t)lr] = (long long)lr * (k + 1) + acc;              // residual row / bonus row of p
      a.rowinfo[2 * (int64_t)lr + 1] = acc < w ? (long long)lr * k + acc : -1;  // draft row (residual only)
      if (a.rowlse) {  // logits form: the two rows' lse beside their indices (one load round for the producer)
        a.rowlse[2 * (int64_t)lr] = a.lse_p[(int64_t)lr * (k + 1) + acc];
        a.rowlse[2 * (int64_t)lr + 1] = acc < w ? a.lse_q[(int64_t)lr * k + acc] : 0.f;
      }
      n_emit = acc + 1;
      if (a.cap) n_emit = min(n_emit, max(a.cap[lr], 0));
    }
    set_status(a.status, vbad);
    long long etot;
    const long long eex = block_excl_scan<long long>(n_emit, sh.tmp, etot);
    if (tid == 0) gs->part[0][blockIdx.x] = etot;
    grid_sync(gs, nb);
    cta_prefix(gs->part[0], sh);
    __syncthreads();
    if (mine) a.offsets[gr - ep0] = (int32_t)(sh.before + eex);
    if (blockIdx.x == gridDim.x - 1 && tid == 0) a.offsets[a.ep_rows] = (int32_t)sh.total;
  }
  // leave the radix histograms zero for the next launch: hist[p % 3] of the passes run since the last zeroing
  if (blockIdx.x == 0 && npass > 0) {
    for (int i = tid; i < 3 * kGBins; i += kGThreads) (&gs->hist[0][0])[i] = 0u;
  }
  grid_exit(gs);
  if (stamp) a.dbg[5] = clock64();
}

bool gselect_shape(int B, int k, int num_sms, int* grid, int* RB) {
  const long long cells = (long long)B * (k > 0 ? k : 1);
  // cells per CTA: 1024 while that needs at most 64 CTAs (the selection's own latency is lowest with many CTAs),
  // else 4096 — fewer, fuller CTAs leave SMs to the sampler that overlaps a large gathered selection
  long long g = (cells + 1023) / 1024;
  if (g > 64) g = (cells + kGCellsPerCta - 1) / kGCellsPerCta;
  const long long g_rows = (B + kGThreads - 1) / kGThreads;                              // one row per thread
  const long long g_smem = (cells * 9 + (long long)kGKeyBudget - 1) / (long long)kGKeyBudget;  // keys + verdicts
  if (g < g_rows) g = g_rows;
  if (g < g_smem) g = g_smem;
  if (g > num_sms) g = num_sms;
  if (g < 1) g = 1;
  if (g > kGMaxGrid) return false;
  const int rb = (int)((B + g - 1) / g);
  if (rb > kGThreads) return false;
  if ((size_t)k * (size_t)((rb | 15) + 2) * 8 + (size_t)rb * k > kGKeyBudget + 16 * 1024) return false;
  *grid = (int)g;
  *RB = rb;
  return true;
}

int launch_gselect(const SelectArgs& args_in, void* scratch, cudaStream_t st) {
  const int num_sms = abi::device_sm_count();
  GArgs ga;
  ga.a = args_in;
  ga.a.dbg = debug_buffer();
  ga.gs = reinterpret_cast<GScratch*>(scratch);
  int grid = 0;
  if (!gselect_shape(ga.a.B, ga.a.k, num_sms, &grid, &ga.RB))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "B=%d k=%d exceeds the grid selector's shared-memory capacity",
                     ga.a.B, ga.a.k);
  const size_t smem = (size_t)ga.a.k * ((ga.RB | 15) + 2) * 8 + (size_t)ga.RB * ga.a.k;
  cudaError_t e = abi::ensure_smem(gselect_kernel, smem);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kGThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // grid barriers: every CTA co-resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, gselect_kernel, ga);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  return abi::launch_check();
}

size_t gselect_scratch_bytes() { return sizeof(GScratch); }

}  // namespace tetris
