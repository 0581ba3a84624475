// Stages (1)+(2) for batches whose keys fit one SM: single-CTA prefix products + TETRIS global top-C (sm_100a).
//
// Same semantics as select_kernel (select.cu) — cumulative_products (selector.py:95-110) + select_tetris
// (selector.py:133-176) under the _HeapItem key (-cum, row, depth) (selector.py:113-130) over each row's prefix-min
// envelope — but for B*k <= 16384 cells the whole batch lives in ONE CTA of 1024 threads, so every phase boundary is a
// __syncthreads instead of a cluster barrier and the launch is a plain (non-cluster, non-cooperative) kernel:
//   * thread t owns the contiguous rows [t*RPT, (t+1)*RPT) (row order == thread order, which the tie-break and every
//     offset scan need); keys live in shared memory as [depth][row] (conflict-free for RPT = 1);
//   * MSB-first radix select with 11/11/11/11/10/10-bit digits over one 2048-bin shared histogram: a pass only
//     touches the still-undecided sub-range [lo, hi) of each row (contiguous: keys are non-decreasing along a row),
//     and the select stops once the bucket holding the C-th cell is taken whole — on fp64 products that is after
//     the sign/exponent digit and one mantissa digit;
//   * exact key ties left after 64 bits are taken in row-major order (row asc, depth asc) by one block scan.
// Optional epilogue (the fused step), as in select.cu: first rejection from the accept verdicts that CTAs 1.. of the
// same launch compute concurrently (one thread per drafted position), the row to resample from, compaction offsets.
#include <cmath>

#include "common.cuh"
#include "abi_util.h"
#include "launch.h"

namespace tetris {

constexpr int kS1Threads = 1024;
constexpr int kS1MaxCells = 16384;
constexpr int kS1MaxRpt = 4;
constexpr int kS1Bins = 2048;

struct S1Shared {
  uint32_t hist[2][kS1Bins];  // double-buffered by radix pass
  long long tmp[33];
  int digit, done;
  long long need, total;
};

// The accept role (CTAs 1..): verify_token (accept_model.py:309-313) on every drafted position of the local rows.
// Verdict byte: bit0 accept, bit1 draft token outside the vocabulary, bit2 uniform outside [0, 1).
// CTA acta takes the contiguous positions [acta * per, (acta + 1) * per), per = ceil(n / nacta).
__device__ void accept_role(const SelectArgs& a, int acta, int nacta) {
  const int k = a.k, nt = blockDim.x, tid = threadIdx.x;
  const int64_t n = (int64_t)a.ep_rows * k, per = (n + nacta - 1) / nacta;
  const int64_t e0 = (int64_t)acta * per, e1 = e0 + per < n ? e0 + per : n;
  const int32_t* llen = a.len ? a.len + a.ep_row0 : nullptr;
  for (int64_t e = e0 + tid; e < e1; e += nt) {
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
  if (tid == 0) {  // release: the CTA's verdict stores (ordered by the barrier) before the arrival
    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.acc_counter) : "memory");
  }
}

// NT threads per CTA: 1024, or 256 / 128 for batches of at most 256 / 128 rows — every phase costs about
// (instructions per thread) x (warps per scheduler), so a small batch runs faster on fewer, busier threads.
template <int RPT, int NT = kS1Threads>
__global__ void __launch_bounds__(NT, 1) select1_kernel(const SelectArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ __align__(16) S1Shared sh;
  // programmatic dependent launch: the sampler that follows may be scheduled onto the SMs this grid leaves idle and
  // run its prologue; it reads nothing of ours before its griddepcontrol.wait (= this grid complete and flushed)
  // launched itself as a programmatic dependent of whatever precedes it (the previous step's sampler lets it be
  // scheduled early, during its descents): nothing is read or written before that grid has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (blockIdx.x > 0) {
    accept_role(a, blockIdx.x - 1, gridDim.x - 1);
    return;
  }
  const int tid = threadIdx.x, lane = tid & 31, k = a.k, B = a.B;
  // key row stride: keys[j * KS + r]; KS = 1 (mod 16) in 8-byte words, so both the transposing stores of the
  // coalesced staging loop and the per-row accesses (consecutive r across a warp) are bank-conflict free
  const int KS = (B | 15) + 2;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);
  uint8_t* lo = reinterpret_cast<uint8_t*>(keys + (size_t)k * KS);
  uint8_t* hi = lo + B;
  const int r0 = tid * RPT;
  const bool stamp = a.dbg != nullptr && tid == 0;
  if (stamp) {
    a.dbg[0] = clock64();
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    a.dbg[48] = g;
  }

  // ---- phase 0: every global load of the selector in flight at once (row lengths + the [B][k] values, 16-byte
  //      loads where aligned), transposed into keys[j][r]; histogram 0 cleared meanwhile ----------------------------
  int Lr[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) Lr[i] = (r0 + i < B) ? (a.len ? a.len[r0 + i] : k) : 0;
  for (int i = tid; i < kS1Bins; i += NT) sh.hist[0][i] = 0;
  {
    const int n = B * k;
    const bool vec = ((reinterpret_cast<uintptr_t>(a.vals) & 15) == 0) && (n % 2 == 0);
    if (vec) {
      const double2* v2 = reinterpret_cast<const double2*>(a.vals);
      const int n2 = n / 2;
      for (int e0 = 0; e0 < n2; e0 += 8 * NT) {
        double2 v[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const int e = e0 + x * NT + tid;
          v[x] = e < n2 ? __ldg(v2 + e) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          const int e = 2 * (e0 + x * NT + tid);
          if (e < n) {
            int r = e / k, j = e - r * k;
            keys[(size_t)j * KS + r] = (uint64_t)__double_as_longlong(v[x].x);
            if (++j == k) j = 0, ++r;
            keys[(size_t)j * KS + r] = (uint64_t)__double_as_longlong(v[x].y);
          }
        }
      }
    } else {
      for (int e0 = 0; e0 < n; e0 += 16 * NT) {
        double v[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) {
          const int e = e0 + x * NT + tid;
          v[x] = e < n ? __ldg(a.vals + e) : 0.0;
        }
#pragma unroll
        for (int x = 0; x < 16; ++x) {
          const int e = e0 + x * NT + tid;
          if (e < n) {
            const int r = e / k, j = e - r * k;
            keys[(size_t)j * KS + r] = (uint64_t)__double_as_longlong(v[x]);
          }
        }
      }
    }
  }
  __syncthreads();
  if (stamp) a.dbg[5] = clock64();

  // ---- per row: prefix products (selector.py:104-108, left to right), envelope, keys, and the first radix digit
  //      (bits 63..53) counted on the fly (run lengths: digits are non-decreasing along a row) --------------------
  constexpr int kShift0 = 53;
  uint32_t bad = 0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = r0 + i;
    if (r >= B) break;
    int L = Lr[i];
    if (L < 0 || L > k) {
      bad |= TETRIS_ST_BAD_VALUE;
      L = L < 0 ? 0 : k;
      Lr[i] = L;
    }
    double cum = 1.0, env = 0.0;
    uint32_t cur = 0xFFFFFFFFu, cnt = 0;
    for (int j0 = 0; j0 < L; j0 += 8) {
      double v[8];
#pragma unroll
      for (int x = 0; x < 8; ++x)
        v[x] = j0 + x < L ? __longlong_as_double((long long)keys[(size_t)(j0 + x) * KS + r]) : 0.0;
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const int j = j0 + x;
        if (j >= L) break;
        if (a.vals_are_cum) {
          cum = v[x];
          if (isnan(cum)) bad |= TETRIS_ST_BAD_VALUE;
        } else {
          if (!(v[x] >= 0.0 && v[x] <= 1.0)) bad |= TETRIS_ST_BAD_VALUE;  // accept_model.py:55-59
          cum = __dmul_rn(cum, v[x]);
        }
        if (a.cum_out) a.cum_out[(int64_t)r * k + j] = cum;
        env = (j == 0 || cum < env) ? cum : env;
        const uint64_t key = desc_key(env);
        keys[(size_t)j * KS + r] = key;
        const uint32_t dg = (uint32_t)(key >> kShift0);
        if (dg == cur) {
          ++cnt;
        } else {
          if (cnt) atomicAdd(&sh.hist[0][cur], cnt);
          cur = dg;
          cnt = 1;
        }
      }
    }
    if (cnt) atomicAdd(&sh.hist[0][cur], cnt);
    lo[r] = 0;
    hi[r] = (uint8_t)L;
  }
  set_status(a.status, bad);
  if (stamp) a.dbg[1] = clock64();

  // ---- phase 1: radix select of the C-th key, 11/11/11/11/10/10-bit digits; 2 barriers per pass: [count into
  //      hist[p&1]] | warp 0 picks the digit while the others clear hist[(p+1)&1] | [narrow each row's [lo, hi)] --
  long long need = a.C, N = 0;
  int mode = 0;  // 0: nothing selected, 1: everything, 2: radix
  bool done = false;
  int npass = 0;
  int shift = 64;
  for (int pass = 0; pass < 6 && !done; ++pass) {
    ++npass;
    const int width = pass < 4 ? 11 : 10;
    shift -= width;
    const uint32_t mask = (1u << width) - 1u;
    uint32_t* H = sh.hist[pass & 1];
    if (pass > 0) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r = r0 + i;
        if (r >= B) break;
        const int l = lo[r], h = hi[r];
        if (l >= h) continue;
        uint32_t cur = (uint32_t)(keys[(size_t)l * KS + r] >> shift) & mask, cnt = 1;
        for (int j = l + 1; j < h; ++j) {
          const uint32_t dg = (uint32_t)(keys[(size_t)j * KS + r] >> shift) & mask;
          if (dg == cur) {
            ++cnt;
          } else {
            atomicAdd(&H[cur], cnt);
            cur = dg;
            cnt = 1;
          }
        }
        atomicAdd(&H[cur], cnt);
      }
    }
    __syncthreads();
    if (stamp) a.dbg[10 + 3 * pass] = clock64();
    if (tid < 32) {
      uint32_t tot;
      const long long nd = need < 1 ? 1 : (need > kS1MaxCells ? kS1MaxCells + 1 : need);
      pick_digit_warp(H, (uint32_t)nd, lane, &sh.digit, &sh.need, &sh.done, &tot);
      if (pass == 0 && lane == 0) sh.total = (long long)tot;
    } else {
      uint32_t* Hn = sh.hist[(pass + 1) & 1];
      for (int i = tid - 32; i < kS1Bins; i += NT - 32) Hn[i] = 0;
    }
    __syncthreads();
    if (stamp) a.dbg[11 + 3 * pass] = clock64();
    if (pass == 0) {
      N = sh.total;
      mode = (a.C <= 0 || N == 0) ? 0 : (a.C >= N ? 1 : 2);
      if (mode != 2) break;
    }
    const uint32_t D = (uint32_t)sh.digit;
    need = sh.need;
    const bool take_all = sh.done != 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = r0 + i;
      if (r >= B) break;
      int l = lo[r];
      const int h = hi[r];
      if (l >= h) continue;
      while (l < h && (((uint32_t)(keys[(size_t)l * KS + r] >> shift) & mask) < D)) ++l;
      int e = l;
      while (e < h && (((uint32_t)(keys[(size_t)e * KS + r] >> shift) & mask) == D)) ++e;
      lo[r] = (uint8_t)(take_all ? e : l);
      hi[r] = (uint8_t)e;
    }
    done = take_all;
    if (stamp) a.dbg[12 + 3 * pass] = clock64();
  }
  __syncthreads();  // lo/hi of every row final before the scans below read neighbours' (tie mode) values
  if (stamp) {
    a.dbg[2] = clock64();
    a.dbg[9] = npass;
  }

  // ---- phase 2: windows ------------------------------------------------------------------------------------------
  // [lo, hi) are exact key ties after all 64 bits: take them in row-major order while `need` lasts.
  if (mode == 2 && !done) {
    long long t_my = 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (r0 + i < B) t_my += hi[r0 + i] - lo[r0 + i];
    long long tt;
    long long ex = block_excl_scan<long long>(t_my, sh.tmp, tt);
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = r0 + i;
      if (r >= B) break;
      const long long t = hi[r] - lo[r];
      long long take = need - ex;
      take = take < 0 ? 0 : (take > t ? t : take);
      lo[r] = (uint8_t)(lo[r] + take);
      ex += t;
    }
  }
  // windows, win_offsets and the PolicyStats closed forms (selector.py:150-170) in one scan of a packed value:
  // window (bits 0..23) | inserts term (24..47) | non-empty row (48..63).
  int wr[RPT];
  long long pk = 0;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = r0 + i;
    const int L = Lr[i];
    const int w = r >= B ? 0 : (mode == 0 ? 0 : (mode == 1 ? L : lo[r]));
    wr[i] = w;
    if (r < B) pk += (long long)w | ((long long)(w - ((w == L && L > 0) ? 1 : 0)) << 24) | ((long long)(L > 0) << 48);
  }
  long long ptot;
  long long pex = block_excl_scan<long long>(pk, sh.tmp, ptot);
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = r0 + i;
    if (r >= B) break;
    a.windows[r] = wr[i];
    if (a.win_offsets) a.win_offsets[r] = (int32_t)(pex & 0xFFFFFF);
    pex += wr[i];
  }
  const long long tot_w = ptot & 0xFFFFFF;
  if (tid == 0) {
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
  if (stamp) a.dbg[3] = clock64();

  // ---- optional greedy epilogue: the row list of greedy verification over the local rows -------------------------
  if (a.rowmap != nullptr) {
    const int ep0 = a.ep_row0, ep1 = a.ep_row0 + a.ep_rows;
    const int f = max(r0, ep0), l = min(min(r0 + RPT, B), ep1);  // this thread's local rows [f, l)
    const int nb = l > f ? l - f : 0;
    int wl[RPT];
    long long my = 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      int w = 0;
#pragma unroll
      for (int x = 0; x < RPT; ++x) w = (r0 + x == f + i) ? wr[x] : w;
      wl[i] = i < nb ? w : 0;
      my += i < nb ? w : 0;  // rows 1..w (row 0 of every request is streamed before the selection completes)
    }
    long long rtot;
    const long long roff = block_excl_scan<long long>(my, sh.tmp, rtot);
    rowmap_write_warp<RPT>(wl, f - ep0, nb, roff, k, a.rowmap, a.gkeys, lane);
    if (tid == 0) a.rowmap[0] = (int32_t)rtot;
  }

  // ---- optional epilogue: first rejection, row to resample from, compaction offsets --------------------------------
  if (a.p != nullptr || a.zp != nullptr) {
    uint32_t vbad = 0;
    const int ep0 = a.ep_row0, ep1 = a.ep_row0 + a.ep_rows;
    if (a.accept_ctas > 0) {
      if (tid == 0) {
        int seen;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(seen) : "l"(a.acc_counter) : "memory");
          if (seen >= a.accept_ctas) break;
          __nanosleep(100);
        }
      }
      __syncthreads();
    }
    if (stamp) a.dbg[6] = clock64();
    int nr[RPT];
    long long my_emit = 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = r0 + i;
      nr[i] = 0;
      if (r >= B || r < ep0 || r >= ep1) continue;
      const int lr = r - ep0;
      const int w = wr[i];
      int acc = w;
      if (a.acc_bytes) {
        // verdicts of 16 positions per round trip (independent loads), then the first rejection among them
        const uint8_t* ab = a.acc_bytes + (int64_t)lr * k;
        for (int j0 = 0; j0 < w && acc == w; j0 += 16) {
          uint8_t v[16];
#pragma unroll
          for (int x = 0; x < 16; ++x) v[x] = (j0 + x < w) ? __ldcg(ab + j0 + x) : (uint8_t)1;
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            if (acc != w || j0 + x >= w) continue;
            vbad |= (v[x] & 2 ? TETRIS_ST_BAD_TOKEN : 0u) | (v[x] & 4 ? TETRIS_ST_BAD_UNIFORM : 0u);
            if (!(v[x] & 1)) acc = j0 + x;
          }
        }
      } else {
        const int64_t uoff = a.u_packed ? (int64_t)a.win_offsets[r] : (int64_t)lr * k;
        for (int j = 0; j < w; ++j) {
          const int t = a.d[(int64_t)lr * k + j];
          const double u = a.u_acc[uoff + j];
          if (!(u >= 0.0 && u < 1.0)) vbad |= TETRIS_ST_BAD_UNIFORM;
          bool rej;
          if (t < 0 || t >= a.V) {
            vbad |= TETRIS_ST_BAD_TOKEN;
            rej = true;
          } else {
            const double s = gather_q(a, (int64_t)lr * k + j, t);
            const double m = gather_p(a, (int64_t)lr * (k + 1) + j, t);
            rej = !(s <= m) && !(u < m / s);  // accept_model.py:311-313
          }
          if (rej) {
            acc = j;
            break;
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
      int n = acc + 1;
      if (a.cap) n = min(n, max(a.cap[lr], 0));
      nr[i] = n;
      my_emit += n;
    }
    set_status(a.status, vbad);
    long long etot;
    long long eex = block_excl_scan<long long>(my_emit, sh.tmp, etot);
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = r0 + i;
      if (r >= B || r < ep0 || r >= ep1) continue;
      a.offsets[r - ep0] = (int32_t)eex;
      eex += nr[i];
    }
    if (tid == 0) {
      a.offsets[a.ep_rows] = (int32_t)etot;
      if (a.accept_ctas > 0) *a.acc_counter = 0;  // every accept CTA has arrived; ready for the next launch
    }
  }
  if (stamp) {
    a.dbg[4] = clock64();
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    a.dbg[49] = g;
  }
}

bool select1_eligible(int B, int k) {
  return B >= 1 && (long long)B * k <= kS1MaxCells && B <= kS1Threads * kS1MaxRpt;
}

int launch_select1(const SelectArgs& args_in, cudaStream_t st) {
  SelectArgs a = args_in;
  a.dbg = debug_buffer();
  const int rpt = (a.B + kS1Threads - 1) / kS1Threads;
  const int nt = a.B <= 128 ? 128 : (a.B <= 256 ? 256 : kS1Threads);
  const size_t smem = (size_t)a.k * ((a.B | 15) + 2) * 8 + 2 * (size_t)a.B;
  int naccept = 0;
  if (a.acc_bytes && a.accept_ctas > 0) {
    const int num_sms = abi::device_sm_count();
    const long long n = (long long)a.ep_rows * a.k;
    // one drafted position (two gathers) per thread; or, when the inputs are mapped host memory (the staged step),
    // every SM but CTA 0's: each scattered read there is a GPU TLB miss over a host pool of many GB, and the misses an
    // SM can have in flight, not the link, bound the rate — 32768 reads take ~880 us from 8-16 SMs, ~132 us from 147
    // (tools/micro/h2d_scalars.cu)
    long long want = a.accept_spread ? (n + 63) / 64 : (n + nt - 1) / nt;
    if (want > num_sms - 1) want = num_sms - 1;
    if (want < 1) want = 1;
    naccept = (int)want;
  }
  a.accept_ctas = naccept;
  // the accept CTAs only ever wait for nothing; CTA 0 waits for them.  They are tiny and need no co-residency
  // guarantee beyond eventually being scheduled, which a plain launch gives (CTA 0 holds one SM).
  auto launch = [&](auto kern) -> int {
    cudaError_t e = abi::ensure_smem(kern, smem);
    if (e != cudaSuccess) return abi::cuda_fail(e);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1 + naccept, 1, 1);
    cfg.blockDim = dim3(nt, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, a);
    if (e != cudaSuccess) return abi::cuda_fail(e);
    return abi::launch_check();
  };
  if (nt == 128) return launch(select1_kernel<1, 128>);
  if (nt == 256) return launch(select1_kernel<1, 256>);
  switch (rpt) {
    case 1:
      return launch(select1_kernel<1>);
    case 2:
      return launch(select1_kernel<2>);
    case 3:
    case 4:
      return launch(select1_kernel<4>);
  }
  return abi::fail(TETRIS_INVALID_ARGUMENT, "B=%d too large for the single-CTA selector", a.B);
}

}  // namespace tetris
