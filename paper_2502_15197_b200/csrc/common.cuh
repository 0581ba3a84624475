// Shared device helpers for the TETRIS B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tetris_b200.h"

namespace tetris {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kLaneElems = TETRIS_LANE_ELEMS;
constexpr int kSegElems = TETRIS_SEG_ELEMS;
constexpr int kWarpSegs = TETRIS_WARP_SEGS;
constexpr int kChunkWarps = TETRIS_CHUNK_WARPS;
constexpr int kChunkElems = TETRIS_CHUNK_ELEMS;
constexpr int kWarpElems = kSegElems * kWarpSegs;  // 1024
constexpr int kStreamThreads = kChunkWarps * 32;   // 256
constexpr int kMaxChunks = 64;                      // V <= 524288

static_assert(kLaneElems == 8, "lane = one 256-bit fp32 load");

__host__ __device__ inline int n_chunks(int V) { return (V + kChunkElems - 1) / kChunkElems; }

// ---- selection key --------------------------------------------------------------------------------------------
// Ascending uint64 order == (cum descending); -0.0 is canonicalised to +0.0 so it ties with +0.0 exactly as the
// reference's float comparison does (selector.py:123 compares -cum).
__device__ __forceinline__ uint64_t desc_key(double v) {
  if (v == 0.0) v = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(v);
  uint64_t o = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending in v
  return ~o;                                                    // descending in v
}

// ---- 256-bit streaming loads (LDG.E.256 on sm_100a) --------------------------------------------------------------
__device__ __forceinline__ void ldg8(const float* p, float (&v)[8]) {
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
      : "l"(p));
}
__device__ __forceinline__ void ldg8(const double* p, double (&v)[8]) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
      : "l"(p));
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
      : "l"(p + 4));
}

// Load the 8 elements of one lane starting at row element e (e is a multiple of 8).  VEC requires V % 8 == 0 (fp32)
// or V % 4 == 0 (fp64) and a 32-byte aligned row base, so a lane is either fully inside the row or fully outside.
template <typename T, bool VEC>
__device__ __forceinline__ void load_lane(const T* __restrict__ row, int64_t e, int V, T (&v)[8]) {
  if (VEC) {
    if (e < V) {
      ldg8(row + e, v);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = T(0);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = (e + i < V) ? __ldg(row + e + i) : T(0);
  }
}

// ---- element weights (sampling contract, tetris_b200.h) --------------------------------------------------------
// residual: max(0, (double)p - (double)q)  (accept_model.py:321 clip(pM - pS, 0))
// plain:    max(0, (double)p)
__device__ __forceinline__ double w_res(double p, double q) {
  double x = p - q;
  return x > 0.0 ? x : 0.0;
}
__device__ __forceinline__ double w_plain(double p) { return p > 0.0 ? p : 0.0; }
// The same weights from fp32 inputs with the sign test in fp32: (double)p - (double)q > 0 exactly when p > q (both
// widenings are exact and the fp64 difference of two distinct floats never rounds to zero), NaN compares false.
// Saves the fp64-pipe compare per element in the streaming consumers.
__device__ __forceinline__ double w_res32(float p, float q) { return p > q ? (double)p - (double)q : 0.0; }
__device__ __forceinline__ double w_plain32(float p) { return p > 0.f ? (double)p : 0.0; }

// Left-to-right fold over the 8 lane elements (the contract's ((0 + w0) + w1) + ...; weights are +0.0 or positive,
// never -0.0, so 0 + w0 == w0 exactly and the fold starts from w0).
__device__ __forceinline__ double fold8(const double (&w)[8]) {
  double o = w[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) o = o + w[i];
  return o;
}

// Segment = balanced binary tree over the 32 lane sums (xor butterfly; every node a contiguous lane range).
__device__ __forceinline__ double seg_sum(double x) {
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) x = x + __shfl_xor_sync(kFull, x, m);
  return x;
}

// Left-to-right node search: first child whose running prefix exceeds T; T becomes T - prefix_before.
// No qualifying child -> last child with positive mass and T = +inf (last-positive-leaf mode).  Returns -1 only
// when every child is zero.
__device__ __forceinline__ int seq_find(const double* v, int n, double& T) {
  double P = 0.0;
  for (int i = 0; i < n; ++i) {
    double Pn = P + v[i];
    if (Pn > T) {
      T = T - P;
      return i;
    }
    P = Pn;
  }
  int last = -1;
  for (int i = 0; i < n; ++i)
    if (v[i] > 0.0) last = i;
  T = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  return last;
}

// ---- logits -> probabilities (the logits contract, tetris_b200.h) ------------------------------------------------
__device__ __forceinline__ float bf16_bits_to_f32(uint32_t z16) { return __uint_as_float(z16 << 16); }

// fp32 -> bf16 bits rounded toward +inf / -inf (integer ops only; finite inputs)
__host__ __device__ __forceinline__ uint32_t bf16_round_up(uint32_t b) {
  const uint32_t h = b >> 16;
  return ((b & 0xffffu) && !(b >> 31)) ? h + 1u : h;
}
__host__ __device__ __forceinline__ uint32_t bf16_round_down(uint32_t b) {
  const uint32_t h = b >> 16;
  return ((b & 0xffffu) && (b >> 31)) ? h + 1u : h;
}

// The row's clamp bounds as bf16 bits: lo = up(lse - 86), hi = down(lse + 88), so that x = z' - lse lies in
// [TETRIS_EXP_LO, TETRIS_EXP_HI] for z' = min(max(z, lo), hi)
struct ExpBounds {
  uint32_t lo, hi;
};
__device__ __forceinline__ ExpBounds exp_bounds(float lse) {
  return ExpBounds{bf16_round_up(__float_as_uint(__fadd_rn(lse, TETRIS_EXP_LO))),
                   bf16_round_down(__float_as_uint(__fadd_rn(lse, TETRIS_EXP_HI)))};
}

// x -> prob for an already clamped x (shared tail of the scalar and packed forms)
__device__ __forceinline__ float exp_tail(float x) {
  const float t = __fmaf_rn(x, TETRIS_EXP_L2E, TETRIS_EXP_MAGIC);
  const float j = __fadd_rn(t, -TETRIS_EXP_MAGIC);
  const float r = __fmaf_rn(j, -TETRIS_EXP_LN2, x);
  float e = __fmaf_rn(TETRIS_EXP_C5, r, TETRIS_EXP_C4);
  e = __fmaf_rn(e, r, TETRIS_EXP_C3);
  e = __fmaf_rn(e, r, TETRIS_EXP_C2);
  e = __fmaf_rn(e, r, TETRIS_EXP_C1);
  e = __fmaf_rn(e, r, TETRIS_EXP_C0);
  return __uint_as_float((__float_as_uint(t) << 23) + __float_as_uint(e));
}

// Scalar prob(z, lse) (gathers: the accept test, the descent's recomputation).  The clamp compares the bf16 values as
// floats (exact): maxNum / minNum semantics like max.bf16x2 / min.bf16x2 (a NaN logit takes the lower bound).
__device__ __forceinline__ float prob_from_logit(uint32_t z16, float lse) {
  const ExpBounds bd = exp_bounds(lse);
  float z = bf16_bits_to_f32(z16);
  z = fminf(fmaxf(z, bf16_bits_to_f32(bd.lo)), bf16_bits_to_f32(bd.hi));
  return exp_tail(__fadd_rn(z, -lse));
}

// Packed fp32x2 (FFMA2 / FADD2 on sm_100a): two elements per instruction on the FMA pipe; elementwise IEEE RN, so the
// results are the scalar function's bits.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(f32x2 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Per-row constants of the packed form: the clamp bounds duplicated into both bf16 halves, and -lse in both lanes
struct ExpRow {
  uint32_t lo2, hi2;
  f32x2 nlse2;
};
__device__ __forceinline__ ExpRow exp_row(float lse) {
  const ExpBounds bd = exp_bounds(lse);
  return ExpRow{bd.lo | (bd.lo << 16), bd.hi | (bd.hi << 16), pk2(-lse, -lse)};
}

// prob(z, lse) for the two bf16 logits packed in `w` (element 0 in the low half): the clamp is one max.bf16x2 and
// one min.bf16x2 on the packed logits.
__device__ __forceinline__ void prob2_from_bf16(uint32_t w, const ExpRow& row, float& p0, float& p1) {
  asm("max.bf16x2 %0, %0, %1;" : "+r"(w) : "r"(row.lo2));
  asm("min.bf16x2 %0, %0, %1;" : "+r"(w) : "r"(row.hi2));
  const f32x2 x = add2(pk2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u)), row.nlse2);
  const f32x2 t = fma2(x, pk2(TETRIS_EXP_L2E, TETRIS_EXP_L2E), pk2(TETRIS_EXP_MAGIC, TETRIS_EXP_MAGIC));
  const f32x2 j = add2(t, pk2(-TETRIS_EXP_MAGIC, -TETRIS_EXP_MAGIC));
  const f32x2 r = fma2(j, pk2(-TETRIS_EXP_LN2, -TETRIS_EXP_LN2), x);
  f32x2 e = fma2(pk2(TETRIS_EXP_C5, TETRIS_EXP_C5), r, pk2(TETRIS_EXP_C4, TETRIS_EXP_C4));
  e = fma2(e, r, pk2(TETRIS_EXP_C3, TETRIS_EXP_C3));
  e = fma2(e, r, pk2(TETRIS_EXP_C2, TETRIS_EXP_C2));
  e = fma2(e, r, pk2(TETRIS_EXP_C1, TETRIS_EXP_C1));
  e = fma2(e, r, pk2(TETRIS_EXP_C0, TETRIS_EXP_C0));
  float t0, t1, e0, e1;
  upk2(t, t0, t1);
  upk2(e, e0, e1);
  p0 = __uint_as_float((__float_as_uint(t0) << 23) + __float_as_uint(e0));
  p1 = __uint_as_float((__float_as_uint(t1) << 23) + __float_as_uint(e1));
}

// 8 consecutive bf16 logits (one 16-byte word) -> 8 probabilities
__device__ __forceinline__ void prob8_from_bf16(const uint4 raw, const ExpRow& row, float (&v)[8]) {
  prob2_from_bf16(raw.x, row, v[0], v[1]);
  prob2_from_bf16(raw.y, row, v[2], v[3]);
  prob2_from_bf16(raw.z, row, v[4], v[5]);
  prob2_from_bf16(raw.w, row, v[6], v[7]);
}

// Logits-form weights: every probability is a positive normal float (>= ~exp(-86)), so the residual weight
// max(0, (double)p - (double)q) is (double)p - (double)min(p, q) (p <= q gives p - p = +0 exactly) and the bonus
// weight is (double)p: the same values as w_res32 / w_plain32 without the compare-and-select.
// Exact fp32 -> fp64 widening of a positive NORMAL float with integer ops (ALU pipe) instead of F2F.F64.F32, which
// runs at a quarter rate on the MIO queue shared with the consumers' shared-memory loads: the exponent is rebiased
// (+896 << 52) and the mantissa shifted into place.
__device__ __forceinline__ double widen_pos_normal(float f) {
  const uint32_t b = __float_as_uint(f);
  return __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29));
}
__device__ __forceinline__ double w_res_pos(float p, float q) {
  return widen_pos_normal(p) - widen_pos_normal(fminf(p, q));
}

// The probability of token t in row `row` of the target (p) / draft (q) input, whichever form the kernel was given:
// fp32 probabilities, or bf16 logits + per-row lse (A: SelectArgs / StreamArgs).
template <typename A>
__device__ __forceinline__ double gather_p(const A& a, int64_t row, int t) {
  if (a.zp) return (double)prob_from_logit(a.zp[row * a.V + t], a.lse_p[row]);
  return (double)a.p[row * a.V + t];
}
template <typename A>
__device__ __forceinline__ double gather_q(const A& a, int64_t row, int t) {
  if (a.zq) return (double)prob_from_logit(a.zq[row * a.V + t], a.lse_q[row]);
  return (double)a.q[row * a.V + t];
}

__device__ __forceinline__ void set_status(uint32_t* status, uint32_t bits) {
  if (status && bits) atomicOr(status, bits);
}

// ---- block-wide helpers for 1024-thread single-CTA kernels ------------------------------------------------------
template <typename U>
__device__ __forceinline__ U warp_incl_scan(U x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    U y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Exclusive scan across the block (blockDim.x == 1024); also returns the block total.  `tmp` >= 33 elements.
template <typename U>
__device__ U block_excl_scan(U x, U* tmp, U& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  U incl = warp_incl_scan(x, lane);
  if (lane == 31) tmp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    U t = lane < nw ? tmp[lane] : U(0);
    U ti = warp_incl_scan(t, lane);
    tmp[lane] = ti - t;
    if (lane == 31) tmp[32] = ti;
  }
  __syncthreads();
  U r = tmp[warp] + incl - x;
  total = tmp[32];
  __syncthreads();
  return r;
}

// Warp 0: the digit holding the need-th undecided cell of histogram h[0..2048).  Lane l owns bins [64l, 64l+64)
// (loaded in a rotated order so 8 consecutive lanes hit 8 distinct bank groups); a warp scan of the lane totals finds
// the owning 64-bin block, then the whole warp scans that block (2 bins per lane) to find the bin.  Also returns
// the histogram total.  Counts fit 32 bits (at most 16384 cells).
__device__ __forceinline__ void pick_digit_warp(const uint32_t* h, uint32_t need, int lane, int* digit,
                                                long long* need_out, int* done, uint32_t* total) {
  const uint4* h4 = reinterpret_cast<const uint4*>(h) + lane * 16;
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const uint4 x = h4[(c + lane) & 15];
    s += x.x + x.y + x.z + x.w;
  }
  const uint32_t incl = warp_incl_scan<uint32_t>(s, lane);
  *total = __shfl_sync(kFull, incl, 31);
  const unsigned own = __ballot_sync(kFull, incl - s < need && need <= incl);
  const int ol = own ? __ffs(own) - 1 : 0;
  const uint32_t before = __shfl_sync(kFull, incl - s, ol);  // cells in blocks before the owning block
  const uint2 b2 = reinterpret_cast<const uint2*>(h)[ol * 32 + lane];  // bins 64*ol + 2*lane, +1
  const uint32_t pair = b2.x + b2.y;
  const uint32_t pin = warp_incl_scan<uint32_t>(pair, lane) + before;
  const uint32_t pex = pin - pair;
  const unsigned hit = __ballot_sync(kFull, own != 0 && pex < need && need <= pin);
  if (hit && lane == __ffs(hit) - 1) {
    const bool first = need <= pex + b2.x;
    const uint32_t base = first ? pex : pex + b2.x, cnt = first ? b2.x : b2.y;
    *digit = ol * 64 + 2 * lane + (first ? 0 : 1);
    *need_out = (long long)(need - base);
    *done = (need - base == cnt);
  }
}

// Lane l's 8 elements are two 16-byte halves; lanes with bit 2 set read the upper half first, so each quarter-warp
// phase of an LDS.128 touches 8 distinct 4-bank groups (no 2-way conflict between lanes l and l+4).
__device__ __forceinline__ void lds8_swz(const float* p, int lane, float (&v)[8]) {
  const int sw = (lane >> 2) & 1;
  const float4 x = *reinterpret_cast<const float4*>(p + 4 * sw);
  const float4 y = *reinterpret_cast<const float4*>(p + 4 * (1 - sw));
  const float4 lo = sw ? y : x, hi = sw ? x : y;
  v[0] = lo.x, v[1] = lo.y, v[2] = lo.z, v[3] = lo.w, v[4] = hi.x, v[5] = hi.y, v[6] = hi.z, v[7] = hi.w;
}

// Greedy verification's row list (greedy.cu): rowmap[1 + o_b + j - J0] = b << 8 | j for j = J0..w_b, o_b =
// Σ_{b' < b} (w_b' + 1 - J0), and the argmax key of each listed row zeroed (J0 = 1: row 0 of every request is
// streamed separately, before the selection completes).  Warp-cooperative: every lane passes its own block of
// requests [b0, b0 + nb) (nb <= N) with clamped windows w[0..nb) and the row offset of b0; the warp writes each
// request's rows with the lanes along the rows (coalesced stores).
template <int N, int J0 = 1>
__device__ __forceinline__ void rowmap_write_warp(const int (&w)[N], int b0, int nb, long long off, int k,
                                                  int32_t* __restrict__ rowmap, unsigned long long* __restrict__ keys,
                                                  int lane) {
  for (int src = 0; src < 32; ++src) {
    const int sb0 = __shfl_sync(kFull, b0, src), snb = __shfl_sync(kFull, nb, src);
    long long so = __shfl_sync(kFull, off, src);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const int wi = __shfl_sync(kFull, w[i], src);
      if (i < snb) {
        const int b = sb0 + i;
        for (int j = J0 + lane; j <= wi; j += 32) {
          rowmap[1 + so + j - J0] = (b << 8) | j;
          if (keys) keys[(int64_t)b * (k + 1) + j] = 0ull;
        }
        so += wi + 1 - J0;
      }
    }
  }
}

}  // namespace tetris

// ---- mbarrier + bulk-copy (TMA engine) helpers -------------------------------------------------------------------
namespace tetris {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared on the TMA engine, completion signalled as transaction bytes on `bar`.
// Addresses 16-byte aligned, size a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The same copy with an L2 eviction-priority hint: streamed rows are read once, so they go in as evict-first and do
// not push out what the next step needs again (the kernels' code, the small per-request tensors).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Small batches (the one-launch step: tens of MB, well inside the 126 MB L2): normal priority, so the descent's
// re-read of one warp run per request hits L2 instead of going back to HBM at the tail of the step.
__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ int atomic_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void lds8(const float* p, float (&v)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  const float4 b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
}

}  // namespace tetris
