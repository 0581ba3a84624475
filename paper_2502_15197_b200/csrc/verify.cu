#include <stdlib.h>
// Stage (3): batched verification + residual / bonus resampling, and the row sampler it is built on (sm_100a).
//
// The HBM-bound part of the path.  For every request exactly one vocabulary row (bonus: p[b][w]) or row pair
// (residual after a rejection: p[b][a], q[b][a]) is streamed, once, with 256-bit loads (LDG.E.256).  Grid =
// (chunks of 8192 elements) x (requests); a CTA of 8 warps owns one chunk, a warp 4 consecutive 256-element
// segments, a lane 8 consecutive elements — exactly the nodes of the sampling contract in tetris_b200.h, so pass 1
// produces the chunk's warp and chunk sums with no extra traffic.  The last CTA of a request to arrive (arrival
// counter in the workspace) folds the chunk sums into the mass, draws T = u*mass and descends the hierarchy;
// only the one 1024-element warp run that holds the sample is re-read (L2-hot).  No second launch, no host sync.
//
// Reference semantics: verify_token (accept_model.py:291-313), residual_distribution (accept_model.py:316-327),
// Generator.choice inverse CDF (accept_model.py:364,368), apply_verification's first-rejection cascade
// (sim_engine.py:388-403), bonus token (sim_engine.py:407-409).
#include <climits>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace tetris {


// ---- pass 1: the 4 segment sums of one warp run and its left-to-right total ---------------------------------------
template <typename T, bool VEC, bool RES>
__device__ __forceinline__ double warp_run_sum(const T* __restrict__ P, const T* __restrict__ Q, int64_t e0, int V,
                                               int lane, double (&G)[kWarpSegs]) {
  constexpr int kBatch = sizeof(T) == 4 ? kWarpSegs : 1;  // fp32: all 8 (or 4) 256-bit loads in flight per thread
#pragma unroll
  for (int s0 = 0; s0 < kWarpSegs; s0 += kBatch) {
    T pv[kBatch][8], qv[kBatch][8];
#pragma unroll
    for (int s = 0; s < kBatch; ++s) {
      const int64_t e = e0 + (int64_t)(s0 + s) * kSegElems + lane * kLaneElems;
      load_lane<T, VEC>(P, e, V, pv[s]);
      if (RES) load_lane<T, VEC>(Q, e, V, qv[s]);
    }
#pragma unroll
    for (int s = 0; s < kBatch; ++s) {
      double w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = RES ? w_res((double)pv[s][i], (double)qv[s][i]) : w_plain((double)pv[s][i]);
      G[s0 + s] = seg_sum(fold8(w));
    }
  }
  double W = 0.0;
#pragma unroll
  for (int s = 0; s < kWarpSegs; ++s) W = W + G[s];
  return W;
}

// ---- the descent below the warp level (all lanes, uniform T) -------------------------------------------------------
template <typename T, bool VEC, bool RES>
__device__ int warp_descend(const T* __restrict__ P, const T* __restrict__ Q, int64_t e0, int V, int lane, double T_) {
  double G[kWarpSegs];
  warp_run_sum<T, VEC, RES>(P, Q, e0, V, lane, G);
  double Tv = T_;
  const int s = seq_find(G, kWarpSegs, Tv);
  if (s < 0) return -1;
  const int64_t eb = e0 + (int64_t)s * kSegElems;
  T pv[8], qv[8];
  load_lane<T, VEC>(P, eb + lane * kLaneElems, V, pv);
  if (RES) load_lane<T, VEC>(Q, eb + lane * kLaneElems, V, qv);
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
    const double R = __shfl_sync(kFull, lv[t], g + (1 << t));
    if (!(L > Tv || R == 0.0)) {
      Tv = Tv - L;
      g += 1 << t;
    }
  }
  double Tl = Tv;
  const int li_own = seq_find(w, 8, Tl);
  const int li = __shfl_sync(kFull, li_own, g);
  if (li < 0) return -1;
  return (int)(eb + g * kLaneElems + li);
}

// ---- stochastic verify (FUSED) / explicit-row sampler ------------------------------------------------------------
template <typename T, bool VEC, bool FUSED>
__global__ void __launch_bounds__(kStreamThreads)
    sample_kernel(const T* __restrict__ p, const T* __restrict__ q, const int32_t* __restrict__ d,
                  const int32_t* __restrict__ windows, const int32_t* __restrict__ win_off,
                  const double* __restrict__ u_acc, int k, int32_t* __restrict__ accepted,
                  const int64_t* __restrict__ p_row, const int64_t* __restrict__ q_row,
                  const double* __restrict__ u_res, int V, int32_t* __restrict__ out_idx,
                  double* __restrict__ mass_out, uint32_t* status, int* __restrict__ counters,
                  double* __restrict__ chunk_sums, double* __restrict__ warp_sums) {
  const int c = blockIdx.x, b = blockIdx.y, nch = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ long long s_prow, s_qrow;
  __shared__ int s_acc, s_last;
  __shared__ double s_w[kChunkWarps];
  __shared__ double s_S[kMaxChunks];

  if (FUSED) {
    if (warp == 0) {
      // verify_token over the selected window, all positions in parallel; first rejection via ballot
      uint32_t bad = 0;
      int w = windows[b];
      if (w < 0 || w > k) {
        bad |= TETRIS_ST_BAD_WINDOW;
        w = w < 0 ? 0 : k;
      }
      int a = w;
      const int64_t uoff = win_off ? (int64_t)win_off[b] : (int64_t)b * k;
      for (int j0 = 0; j0 < w; j0 += 32) {
        const int j = j0 + lane;
        bool rej = false;
        if (j < w) {
          const int t = d[(int64_t)b * k + j];
          const double u = u_acc[uoff + j];
          if (!(u >= 0.0 && u < 1.0)) bad |= TETRIS_ST_BAD_UNIFORM;
          if (t < 0 || t >= V) {
            bad |= TETRIS_ST_BAD_TOKEN;
            rej = true;
          } else {
            const double s = (double)q[((int64_t)b * k + j) * V + t];
            const double m = (double)p[((int64_t)b * (k + 1) + j) * V + t];
            rej = !(s <= m) && !(u < m / s);  // accept_model.py:311-313
          }
        }
        const unsigned mask = __ballot_sync(kFull, rej);
        if (mask) {
          a = j0 + __ffs(mask) - 1;
          break;
        }
      }
      bad = __reduce_or_sync(kFull, bad);
      if (lane == 0) {
        s_acc = a;
        if (a < w) {  // rejected at depth a: residual of (p, q) at that position
          s_prow = (long long)b * (k + 1) + a;
          s_qrow = (long long)b * k + a;
        } else {      // everything accepted: bonus token from the target at position w
          s_prow = (long long)b * (k + 1) + w;
          s_qrow = -1;
        }
        if (c == 0) set_status(status, bad);  // every chunk CTA derives the same verdict; report once
      }
    }
  } else if (tid == 0) {
    s_prow = p_row[b];
    s_qrow = (q != nullptr && q_row != nullptr) ? q_row[b] : -1;
  }
  __syncthreads();

  const T* P = p + s_prow * (int64_t)V;
  const bool res = s_qrow >= 0;
  const T* Q = res ? q + s_qrow * (int64_t)V : nullptr;
  const int64_t e0 = (int64_t)c * kChunkElems + warp * kWarpElems;
  double G[kWarpSegs];
  const double W = res ? warp_run_sum<T, VEC, true>(P, Q, e0, V, lane, G)
                       : warp_run_sum<T, VEC, false>(P, Q, e0, V, lane, G);
  if (lane == 0) s_w[warp] = W;
  __syncthreads();
  if (tid == 0) {
    double S = 0.0;
#pragma unroll
    for (int w = 0; w < kChunkWarps; ++w) S = S + s_w[w];
    const int64_t slot = (int64_t)b * nch + c;
    __stcg(&chunk_sums[slot], S);
#pragma unroll
    for (int w = 0; w < kChunkWarps; ++w) __stcg(&warp_sums[slot * kChunkWarps + w], s_w[w]);
    __threadfence();
    const int prev = atomicAdd(&counters[b], 1);
    s_last = (prev == nch - 1);
  }
  __syncthreads();
  if (!s_last || warp != 0) return;
  __threadfence();

  // ---- last CTA of request b: mass, T = u*mass, descent ------------------------------------------------------
  for (int i = lane; i < nch; i += 32) s_S[i] = __ldcg(&chunk_sums[(int64_t)b * nch + i]);
  __syncwarp();
  double mass = 0.0;
  for (int i = 0; i < nch; ++i) mass = mass + s_S[i];
  int tok = -1;
  uint32_t bad = 0;
  const double u = u_res[b];
  if (!(u >= 0.0 && u < 1.0)) bad |= TETRIS_ST_BAD_UNIFORM;
  if (mass > 0.0) {
    double Tv = u * mass;
    const int cc = seq_find(s_S, nch, Tv);
    double Wc[kChunkWarps];
#pragma unroll
    for (int w = 0; w < kChunkWarps; ++w) Wc[w] = __ldcg(&warp_sums[((int64_t)b * nch + cc) * kChunkWarps + w]);
    const int ww = seq_find(Wc, kChunkWarps, Tv);
    const int64_t e0s = (int64_t)cc * kChunkElems + ww * kWarpElems;
    tok = res ? warp_descend<T, VEC, true>(P, Q, e0s, V, lane, Tv) : warp_descend<T, VEC, false>(P, Q, e0s, V, lane, Tv);
  }
  if (tok < 0) bad |= TETRIS_ST_DEGENERATE;
  if (lane == 0) {
    counters[b] = 0;
    out_idx[b] = tok;
    if (mass_out) mass_out[b] = mass;
    if (FUSED) accepted[b] = s_acc;
    set_status(status, bad);
  }
}

// ---- greedy verify ----------------------------------------------------------------------------------------------
// numpy.argmax order: NaN ranks above every number (first NaN wins), otherwise larger value, ties -> lower index.
__device__ __forceinline__ bool arg_better(float av, int ai, float bv, int bi) {
  if (ai == INT_MAX) return false;
  if (bi == INT_MAX) return true;
  const bool an = isnan(av), bn = isnan(bv);
  if (an != bn) return an;
  if (!an && av != bv) return av > bv;
  return ai < bi;
}

// Greedy verify fallback (V % 8 != 0 or unaligned p; the product path is persist_greedy_kernel, greedy.cu): grid
// (chunks, selected rows): one CTA per (row chunk) of the rows listed by greedy_rowmap_kernel (no
// empty CTAs for the positions beyond a request's window); the last CTA of a request to finish combines the argmaxes.
template <bool VEC>
__global__ void __launch_bounds__(kStreamThreads)
    greedy_kernel(const float* __restrict__ p, const int32_t* __restrict__ d, const int32_t* __restrict__ windows,
                  int k, int V, int32_t* __restrict__ accepted, int32_t* __restrict__ out_tok, uint32_t* status,
                  int* __restrict__ counters, float* __restrict__ arg_val, int32_t* __restrict__ arg_idx,
                  const int32_t* __restrict__ rowmap) {
  const int nch = n_chunks(V);
  const int y = (int)(blockIdx.x / nch), c = (int)(blockIdx.x - (unsigned)y * nch);
  if (y >= __ldg(rowmap)) return;
  const int rm = __ldg(rowmap + 1 + y);
  const int j = rm & 0xFF, b = rm >> 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ float s_v[kChunkWarps];
  __shared__ int s_i[kChunkWarps];
  __shared__ int s_last;
  __shared__ int s_am[TETRIS_MAX_K + 1];
  int w = windows[b];
  const bool bad_w = (w < 0 || w > k);
  w = w < 0 ? 0 : (w > k ? k : w);

  const float* row = p + ((int64_t)b * (k + 1) + j) * V;
  const int64_t e0 = (int64_t)c * kChunkElems + warp * kWarpElems;
  float v[kWarpSegs][8];
#pragma unroll
  for (int s = 0; s < kWarpSegs; ++s) load_lane<float, VEC>(row, e0 + s * kSegElems + lane * kLaneElems, V, v[s]);
  // lane argmax in two cheap passes (the per-element numpy-order comparison made this kernel issue-bound): the
  // NaN-propagating max of the lane's 32 elements, then the first element equal to it (a NaN max matches the first
  // NaN) — numpy.argmax order.  Elements past V are -inf and lose every tie on index.
  const float kNegInf = __int_as_float(0xff800000);
  float bv = kNegInf;
#pragma unroll
  for (int s = 0; s < kWarpSegs; ++s) {
    const int64_t e = e0 + s * kSegElems + lane * kLaneElems;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (e + i >= V) v[s][i] = kNegInf;
      asm("max.NaN.f32 %0, %0, %1;" : "+f"(bv) : "f"(v[s][i]));
    }
  }
  const bool bnan = bv != bv;
  int bi = INT_MAX;
#pragma unroll
  for (int s = kWarpSegs - 1; s >= 0; --s) {
    const int e = (int)(e0 + s * kSegElems + lane * kLaneElems);
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      const bool hit = bnan ? (v[s][i] != v[s][i]) : (v[s][i] == bv);
      bi = hit ? e + i : bi;
    }
  }
  if (bi >= V) bi = INT_MAX;  // only padding in this lane
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) {
    const float ov = __shfl_xor_sync(kFull, bv, m);
    const int oi = __shfl_xor_sync(kFull, bi, m);
    if (arg_better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s_v[warp] = bv;
    s_i[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    float cv = s_v[0];
    int ci = s_i[0];
    for (int x = 1; x < kChunkWarps; ++x)
      if (arg_better(s_v[x], s_i[x], cv, ci)) {
        cv = s_v[x];
        ci = s_i[x];
      }
    const int64_t slot = ((int64_t)b * (k + 1) + j) * nch + c;
    __stcg(&arg_val[slot], cv);
    __stcg(&arg_idx[slot], ci);
    __threadfence();
    const int prev = atomicAdd(&counters[b], 1);
    s_last = (prev == (w + 1) * nch - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int jj = tid; jj <= w; jj += blockDim.x) {
    const int64_t base = ((int64_t)b * (k + 1) + jj) * nch;
    float cv = __ldcg(&arg_val[base]);
    int ci = __ldcg(&arg_idx[base]);
    for (int x = 1; x < nch; ++x) {
      const float ov = __ldcg(&arg_val[base + x]);
      const int oi = __ldcg(&arg_idx[base + x]);
      if (arg_better(ov, oi, cv, ci)) {
        cv = ov;
        ci = oi;
      }
    }
    s_am[jj] = ci;
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t bad = bad_w ? TETRIS_ST_BAD_WINDOW : 0u;
    int a = w;
    for (int jj = 0; jj < w; ++jj) {
      const int t = d[(int64_t)b * k + jj];
      if (t < 0 || t >= V) bad |= TETRIS_ST_BAD_TOKEN;
      if (t != s_am[jj]) {
        a = jj;
        break;
      }
    }
    accepted[b] = a;
    out_tok[b] = s_am[a];
    counters[b] = 0;
    set_status(status, bad);
  }
}

// ---- residual normalisation (residual_distribution's diff / mass, accept_model.py:321-327) ------------------------
__global__ void residual_norm_kernel(const double* __restrict__ ps, const double* __restrict__ pt, int V,
                                     const double* __restrict__ mass, double* __restrict__ out) {
  const int r = blockIdx.y;
  const double m = mass[r];
  if (!(m > 0.0)) return;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (int64_t)r * V + v;
    out[o] = w_res(pt[o], ps[o]) / m;
  }
}

__global__ void identity_rows_kernel(int64_t* a, int64_t* b, double* u, int R) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < R) {
    a[i] = i;
    b[i] = i;
    u[i] = 0.0;
  }
}

}  // namespace tetris

// ---- C ABI ---------------------------------------------------------------------------------------------------------
#include "abi_util.h"

namespace {
using namespace tetris;

inline bool aligned32(const void* ptr) { return ((uintptr_t)ptr & 31u) == 0; }

int check_verify_ws(int B, int k, int V, void* ws, size_t ws_bytes) {
  size_t need = tetris_workspace_bytes(TETRIS_OP_VERIFY, B, k, V);
  if (!ws || ws_bytes < need)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "workspace too small: %zu < %zu", ws_bytes, need);
  return TETRIS_OK;
}

int check_shape(int B, int k, int V) {
  if (B < 0 || B > 65535) return abi::fail(TETRIS_INVALID_ARGUMENT, "B=%d outside [0, 65535]", B);
  if (k < 0 || k > TETRIS_MAX_K) return abi::fail(TETRIS_INVALID_ARGUMENT, "k=%d outside [0, 255]", k);
  if (V < 1 || V > kMaxChunks * kChunkElems)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "V=%d outside [1, %d]", V, kMaxChunks * kChunkElems);
  return TETRIS_OK;
}

template <typename T>
int sample_rows_impl(const T* p, const T* q, const int64_t* p_row, const int64_t* q_row, const double* u, int R,
                     int V, int32_t* out_idx, double* mass_out, uint32_t* status, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  int rc = check_shape(R, 0, V);
  if (rc) return rc;
  if (R == 0) return TETRIS_OK;
  if (!p || !p_row || !u || !out_idx) return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if ((rc = check_verify_ws(R, 0, V, ws, ws_bytes))) return rc;
  const bool vec = (V % kLaneElems == 0) && aligned32(p) && (!q || aligned32(q));  // whole lanes only
  dim3 grid(n_chunks(V), R);
  int* cnt = (int*)abi::ws_region(ws, TETRIS_OP_VERIFY, R, 0, V, abi::WS_COUNTERS);
  double* cs = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, R, 0, V, abi::WS_CHUNK_SUMS);
  double* wsum = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, R, 0, V, abi::WS_WARP_SUMS);
  if (vec)
    sample_kernel<T, true, false><<<grid, kStreamThreads, 0, st>>>(p, q, nullptr, nullptr, nullptr, nullptr, 0,
                                                                   nullptr, p_row, q_row, u, V, out_idx, mass_out,
                                                                   status, cnt, cs, wsum);
  else
    sample_kernel<T, false, false><<<grid, kStreamThreads, 0, st>>>(p, q, nullptr, nullptr, nullptr, nullptr, 0,
                                                                    nullptr, p_row, q_row, u, V, out_idx, mass_out,
                                                                    status, cnt, cs, wsum);
  return abi::launch_check();
}
}  // namespace

extern "C" int tetris_verify_stochastic_f32(const float* p, const float* q, const int32_t* d, const int32_t* windows,
                                            const int32_t* win_offsets, const double* u_acc, const double* u_res,
                                            int32_t B, int32_t k, int32_t V, int32_t* accepted, int32_t* out_tok,
                                            double* mass_out, uint32_t* status, void* ws, size_t ws_bytes,
                                            tetris_stream_t stream) {
  int rc = check_shape(B, k, V);
  if (rc) return rc;
  if (B == 0) return TETRIS_OK;
  // with k == 0 nothing is drafted: the [B][0] tensors (d, u_acc) may be null
  if (!p || (k > 0 && (!d || !u_acc || !q)) || !windows || !u_res || !accepted || !out_tok)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if ((rc = check_verify_ws(B, k, V, ws, ws_bytes))) return rc;
  int* cnt = (int*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_COUNTERS);
  double* cs = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_CHUNK_SUMS);
  double* wsum = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_WARP_SUMS);
  cudaStream_t st = (cudaStream_t)stream;
  if (persist_eligible(p, q, V)) {
    // accept test -> row choice -> persistent TMA-pipelined sampler
    long long* rowinfo = (long long*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWINFO);
    if ((rc = launch_accept(p, q, d, windows, win_offsets, u_acc, B, k, V, accepted, rowinfo, status, st))) return rc;
    StreamArgs a = {};
    a.p = p;
    a.q = q;
    a.V = V;
    a.nch = n_chunks(V);
    a.R = B;
    a.prow = rowinfo;
    a.qrow = rowinfo + 1;
    a.row_stride = 2;
    a.u = u_res;
    a.out_idx = out_tok;
    a.mass_out = mass_out;
    a.status = status;
    a.counters = cnt;
    a.chunk_sums = cs;
    a.warp_sums = wsum;
    a.grid_bar = (unsigned*)cnt + abi::kSlotGridCount;
    a.req_cnt = cnt;
    return launch_persist_stream(a, st);
  }
  const bool vec = (V % 8 == 0) && aligned32(p) && aligned32(q);
  dim3 grid(n_chunks(V), B);
  if (vec)
    sample_kernel<float, true, true><<<grid, kStreamThreads, 0, st>>>(p, q, d, windows, win_offsets, u_acc, k,
                                                                      accepted, nullptr, nullptr, u_res, V, out_tok,
                                                                      mass_out, status, cnt, cs, wsum);
  else
    sample_kernel<float, false, true><<<grid, kStreamThreads, 0, st>>>(p, q, d, windows, win_offsets, u_acc, k,
                                                                       accepted, nullptr, nullptr, u_res, V,
                                                                       out_tok, mass_out, status, cnt, cs, wsum);
  return abi::launch_check();
}

// The step's inputs: fp32 probabilities p / q, or bf16 logits zp / zq with per-row lse (the logits contract).
struct ProbIn {
  const float* p;
  const float* q;
  const uint16_t* zp;
  const uint16_t* zq;
  const float* lse_p;
  const float* lse_q;
  bool logits() const { return zp != nullptr; }
  const void* pbase() const { return logits() ? (const void*)zp : (const void*)p; }
  const void* qbase() const { return logits() ? (const void*)zq : (const void*)q; }
};

static bool aligned16(const void* ptr) { return ((uintptr_t)ptr & 15u) == 0; }

// the TMA sampler's requirements: whole 16-byte lanes per row (V % 8 == 0) and 16-byte aligned row bases
static bool persist_eligible_in(const ProbIn& in, int V) {
  if (!in.logits()) return persist_eligible(in.p, in.q, V);
  return V % 8 == 0 && n_chunks(V) <= 64 && aligned16(in.zp) && (!in.zq || aligned16(in.zq)) && in.lse_p;
}

static int select_accept_impl(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                              int32_t row0, int32_t B, const ProbIn& in, const int32_t* d, const double* u_acc,
                              int32_t u_packed, const int32_t* cap, int32_t V, int32_t* windows, int32_t* win_offsets,
                              int32_t* accepted, int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status,
                              void* ws, size_t ws_bytes, tetris_stream_t stream, bool host_inputs = false) {
  int rc = check_shape(B, k, V);
  if (rc) return rc;
  if (C < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0, got %lld", (long long)C);
  if (B == 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "empty batch");
  if (B_sel < B || B_sel > TETRIS_MAX_SELECT_ROWS || row0 < 0 || row0 + B > B_sel)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "local rows [%d, %d) outside the %d selected rows", row0, row0 + B, B_sel);
  if (u_packed && B != B_sel) return abi::fail(TETRIS_INVALID_ARGUMENT, "packed uniforms need the whole batch");
  if ((k > 0 && (!conf || !d || !u_acc || !in.qbase() || (in.logits() && !in.lse_q))) || !in.pbase() ||
      (in.logits() && !in.lse_p) || !windows || !win_offsets || !accepted || !offsets || !tokens)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if ((rc = check_verify_ws(B, k, V, ws, ws_bytes))) return rc;
  SelectArgs sa = {};
  sa.vals = conf;
  sa.len = len;
  sa.B = B_sel;
  sa.k = k;
  sa.C = (long long)C;
  sa.windows = windows;
  sa.win_offsets = win_offsets;
  sa.stats = (long long*)stats4;
  sa.status = status;
  sa.ep_row0 = row0;
  sa.ep_rows = B;
  sa.p = in.p;
  sa.q = in.q;
  sa.zp = in.zp;
  sa.zq = in.zq;
  sa.lse_p = in.lse_p;
  sa.lse_q = in.lse_q;
  sa.d = d;
  sa.u_acc = u_acc;
  sa.u_packed = u_packed;
  sa.V = V;
  sa.cap = cap;
  sa.accepted = accepted;
  sa.rowinfo = (long long*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWINFO);
  if (in.logits()) sa.rowlse = (float*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWLSE);
  sa.gscratch = abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_GSEL);
  sa.offsets = offsets;
  (void)tokens;  // the accepted-prefix tokens are written by tetris_resample_f32's finalize kernel
  if (!u_packed) {
    // dense uniforms: every position's verdict is independent of the selection, so extra CTAs of the same launch
    // compute them (one thread per position) while cluster 0 selects
    sa.acc_bytes = (uint8_t*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ACCBYTES);
    sa.acc_counter = (int*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_COUNTERS) + abi::kSlotAccCounter;
    sa.accept_ctas = 1;
    sa.accept_spread = host_inputs ? 1 : 0;
  }
  return launch_select(sa, (cudaStream_t)stream);
}

extern "C" int tetris_select_accept_f32(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                                        int32_t row0, int32_t B, const float* p, const float* q, const int32_t* d,
                                        const double* u_acc, int32_t u_packed, const int32_t* cap, int32_t V,
                                        int32_t* windows, int32_t* win_offsets, int32_t* accepted, int32_t* offsets,
                                        int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                        tetris_stream_t stream) {
  const ProbIn in = {p, q, nullptr, nullptr, nullptr, nullptr};
  return select_accept_impl(conf, len, B_sel, k, C, row0, B, in, d, u_acc, u_packed, cap, V, windows, win_offsets,
                            accepted, offsets, tokens, stats4, status, ws, ws_bytes, stream);
}

extern "C" int tetris_select_accept_bf16(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                                         int32_t row0, int32_t B, const uint16_t* zp, const float* lse_p,
                                         const uint16_t* zq, const float* lse_q, const int32_t* d, const double* u_acc,
                                         int32_t u_packed, const int32_t* cap, int32_t V, int32_t* windows,
                                         int32_t* win_offsets, int32_t* accepted, int32_t* offsets, int32_t* tokens,
                                         int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                         tetris_stream_t stream) {
  const ProbIn in = {nullptr, nullptr, zp, zq, lse_p, lse_q};
  return select_accept_impl(conf, len, B_sel, k, C, row0, B, in, d, u_acc, u_packed, cap, V, windows, win_offsets,
                            accepted, offsets, tokens, stats4, status, ws, ws_bytes, stream);
}

constexpr long long kSpecMinChunks = 4096;  // see tetris_step_stochastic_f32

static int resample_impl(const ProbIn& in, const double* u_res, const double* u_acc_spec, const int32_t* len_spec,
                         int B, int k, int V, const int32_t* d, const int32_t* accepted, const int32_t* offsets,
                         int32_t* out_tok, double* mass_out, int32_t* tokens, uint32_t* status, void* ws,
                         size_t ws_bytes, cudaStream_t st) {
  int rc = check_shape(B, k, V);
  if (rc) return rc;
  if (B == 0) return TETRIS_OK;
  if (!in.pbase() || (k > 0 && !in.qbase()) || !u_res || !out_tok)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if ((rc = check_verify_ws(B, k, V, ws, ws_bytes))) return rc;
  if (!persist_eligible_in(in, V))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "the streaming sampler needs V %% 8 == 0 and 16-byte aligned rows");
  long long* rowinfo = (long long*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWINFO);
  int* cnt = (int*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_COUNTERS);
  StreamArgs a = {};
  a.p = in.p;
  a.q = in.q;
  a.zp = in.zp;
  a.zq = in.zq;
  a.lse_p = in.lse_p;
  a.lse_q = in.lse_q;
  if (in.logits()) a.rowlse = (const float*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWLSE);
  a.V = V;
  a.nch = n_chunks(V);
  a.R = B;
  a.k = k;
  a.d = d;
  a.prow = rowinfo;
  a.qrow = rowinfo + 1;
  a.row_stride = 2;
  a.u = u_res;
  a.out_idx = out_tok;
  a.mass_out = mass_out;
  a.status = status;
  a.counters = cnt;
  a.chunk_sums = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_CHUNK_SUMS);
  a.warp_sums = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_WARP_SUMS);
  a.grid_bar = (unsigned*)cnt + abi::kSlotGridCount;
  a.req_cnt = cnt;
  if (tokens) {
    if (!accepted || !offsets || (k > 0 && !d))
      return abi::fail(TETRIS_INVALID_ARGUMENT, "tokens needs accepted, offsets, d");
    a.accepted = accepted;
    a.offsets = offsets;
    a.tokens = tokens;
  }
  if (u_acc_spec && d && B <= spec_max_requests()) {
    double* sums = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_SPEC_SUMS);
    a.u_acc = u_acc_spec;
    a.len = len_spec;
    a.req_cnt_spec = cnt + abi::kSlotSpecCnt;
    a.chunk_sums_spec = sums;
    a.warp_sums_spec = sums + (size_t)B * a.nch;
    a.spec_ctl = cnt + abi::kSlotSpecCtl;
    a.spec_bitmap = (uint32_t*)(cnt + abi::kSlotSpecBitmap);
    a.spec_list = cnt + abi::kSlotSpecList;
    if (in.logits()) a.spec_lse = (float*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_SPEC_LSE);
  }
  return launch_persist_stream(a, st);
}

extern "C" int tetris_resample_f32(const float* p, const float* q, const double* u_res, int32_t B, int32_t k, int32_t V,
                                   const int32_t* d, const int32_t* accepted, const int32_t* offsets, int32_t* out_tok,
                                   double* mass_out, int32_t* tokens, uint32_t* status, void* ws, size_t ws_bytes,
                                   tetris_stream_t stream) {
  const ProbIn in = {p, q, nullptr, nullptr, nullptr, nullptr};
  return resample_impl(in, u_res, nullptr, nullptr, B, k, V, d, accepted, offsets, out_tok, mass_out, tokens, status,
                       ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int tetris_resample_spec_f32(const float* p, const float* q, const double* u_res, const double* u_acc,
                                        const int32_t* len, int32_t B, int32_t k, int32_t V, const int32_t* d,
                                        const int32_t* accepted, const int32_t* offsets, int32_t* out_tok,
                                        double* mass_out, int32_t* tokens, uint32_t* status, void* ws,
                                        size_t ws_bytes, tetris_stream_t stream) {
  if (k > 0 && (!u_acc || !d)) return abi::fail(TETRIS_INVALID_ARGUMENT, "the speculative sampler needs u_acc and d");
  const ProbIn in = {p, q, nullptr, nullptr, nullptr, nullptr};
  return resample_impl(in, u_res, u_acc, len, B, k, V, d, accepted, offsets, out_tok, mass_out, tokens, status, ws,
                       ws_bytes, (cudaStream_t)stream);
}

extern "C" int tetris_resample_bf16(const uint16_t* zp, const float* lse_p, const uint16_t* zq, const float* lse_q,
                                    const double* u_res, const double* u_acc, const int32_t* len, int32_t B,
                                    int32_t k, int32_t V, const int32_t* d, const int32_t* accepted,
                                    const int32_t* offsets, int32_t* out_tok, double* mass_out, int32_t* tokens,
                                    uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  if (u_acc && k > 0 && !d) return abi::fail(TETRIS_INVALID_ARGUMENT, "the speculative sampler needs d");
  if (u_acc && B > spec_max_requests())
    return abi::fail(TETRIS_INVALID_ARGUMENT, "speculative sampler: B=%d > %d", B, spec_max_requests());
  const ProbIn in = {nullptr, nullptr, zp, zq, lse_p, lse_q};
  return resample_impl(in, u_res, u_acc, len, B, k, V, d, accepted, offsets, out_tok, mass_out, tokens, status, ws,
                       ws_bytes, (cudaStream_t)stream);
}

static int step_stochastic_impl(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                                int32_t row0, int32_t B, const ProbIn& in, const int32_t* d, const double* u_acc,
                                int32_t u_packed, const double* u_res, const int32_t* cap, int32_t V, int32_t* windows,
                                int32_t* win_offsets, int32_t* accepted, int32_t* out_tok, double* mass_out,
                                int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws,
                                size_t ws_bytes, tetris_stream_t stream);

// Small batches (B_sel * k <= kFusedMaxCells, dense uniforms): the whole step in ONE launch — the selection, accept
// test, row choice and offset scans run as the persistent sampler's prologue (stream.cu, fused_select), so the step
// pays one launch and no selector latency chain.  Same arguments, checks and results as the two-launch step.
static int fused_step_impl(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C, int32_t row0,
                           int32_t B, const ProbIn& in, const int32_t* d, const double* u_acc, const double* u_res,
                           const int32_t* cap, int32_t V, int32_t* windows, int32_t* win_offsets, int32_t* accepted,
                           int32_t* out_tok, double* mass_out, int32_t* offsets, int32_t* tokens, int64_t* stats4,
                           uint32_t* status, void* ws, size_t ws_bytes, cudaStream_t st) {
  int rc = check_shape(B, k, V);
  if (rc) return rc;
  if (C < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0, got %lld", (long long)C);
  if (B_sel < B || B_sel > TETRIS_MAX_SELECT_ROWS || row0 < 0 || row0 + B > B_sel)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "local rows [%d, %d) outside the %d selected rows", row0, row0 + B, B_sel);
  if ((k > 0 && (!conf || !d || !u_acc || !in.qbase() || (in.logits() && !in.lse_q))) || !in.pbase() ||
      (in.logits() && !in.lse_p) || !windows || !win_offsets || !accepted || !offsets || !tokens)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if ((rc = check_verify_ws(B, k, V, ws, ws_bytes))) return rc;
  long long* rowinfo = (long long*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWINFO);
  int* cnt = (int*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_COUNTERS);
  StreamArgs a = {};
  a.p = in.p;
  a.q = in.q;
  a.zp = in.zp;
  a.zq = in.zq;
  a.lse_p = in.lse_p;
  a.lse_q = in.lse_q;
  float* rowlse = in.logits() ? (float*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWLSE) : nullptr;
  a.rowlse = rowlse;
  a.V = V;
  a.nch = n_chunks(V);
  a.R = B;
  a.k = k;
  a.d = d;
  a.prow = rowinfo;
  a.qrow = rowinfo + 1;
  a.row_stride = 2;
  a.u = u_res;
  a.out_idx = out_tok;
  a.mass_out = mass_out;
  a.status = status;
  a.counters = cnt;
  a.chunk_sums = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_CHUNK_SUMS);
  a.warp_sums = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_WARP_SUMS);
  a.grid_bar = (unsigned*)cnt + abi::kSlotGridCount;
  a.req_cnt = cnt;
  a.accepted = accepted;
  a.offsets = offsets;
  a.tokens = tokens;
  FusedSel& f = a.fs;
  static const double kNoScores = 0.0;  // k == 0: nothing is read through these
  f.conf = conf ? conf : &kNoScores;
  f.len = len;
  f.u_acc = u_acc ? u_acc : &kNoScores;
  f.B_sel = B_sel;
  f.row0 = row0;
  f.C = (long long)C;
  f.windows = windows;
  f.win_offsets = win_offsets;
  f.stats = (long long*)stats4;
  f.cap = cap;
  f.accepted = accepted;
  f.rowinfo = rowinfo;
  f.rowlse = rowlse;
  f.offsets = offsets;
  f.ctl = cnt + abi::kSlotFusedCtl;
  f.ready = reinterpret_cast<unsigned long long*>(cnt + abi::kSlotFusedReady);
  if (k == 0) a.d = d ? d : (const int32_t*)&kNoScores;
  return launch_persist_stream(a, st);
}

extern "C" int tetris_step_stochastic_f32(const double* conf, const int32_t* len, int32_t B_sel, int32_t k,
                                          int64_t C, int32_t row0, int32_t B, const float* p, const float* q,
                                          const int32_t* d, const double* u_acc, int32_t u_packed,
                                          const double* u_res, const int32_t* cap, int32_t V, int32_t* windows,
                                          int32_t* win_offsets, int32_t* accepted, int32_t* out_tok,
                                          double* mass_out, int32_t* offsets, int32_t* tokens, int64_t* stats4,
                                          uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  const ProbIn in = {p, q, nullptr, nullptr, nullptr, nullptr};
  return step_stochastic_impl(conf, len, B_sel, k, C, row0, B, in, d, u_acc, u_packed, u_res, cap, V, windows,
                              win_offsets, accepted, out_tok, mass_out, offsets, tokens, stats4, status, ws, ws_bytes,
                              stream);
}

static int step_stochastic_impl(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                                int32_t row0, int32_t B, const ProbIn& in, const int32_t* d, const double* u_acc,
                                int32_t u_packed, const double* u_res, const int32_t* cap, int32_t V, int32_t* windows,
                                int32_t* win_offsets, int32_t* accepted, int32_t* out_tok, double* mass_out,
                                int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws,
                                size_t ws_bytes, tetris_stream_t stream) {
  if (!persist_eligible_in(in, V))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "fused step needs V %% 8 == 0 and 16-byte aligned rows");
  if (!u_res || !out_tok) return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if (fused_step_eligible(B_sel, k, u_packed) && B >= 1)
    return fused_step_impl(conf, len, B_sel, k, C, row0, B, in, d, u_acc, u_res, cap, V, windows, win_offsets,
                           accepted, out_tok, mass_out, offsets, tokens, stats4, status, ws, ws_bytes,
                           (cudaStream_t)stream);
  int rc = select_accept_impl(conf, len, B_sel, k, C, row0, B, in, d, u_acc, u_packed, cap, V, windows, win_offsets,
                              accepted, offsets, tokens, stats4, status, ws, ws_bytes, stream);
  if (rc) return rc;
  // dense uniforms: the sampler streams the selection-independent rows while the selector runs — when there is
  // enough to stream for the early start to pay for its set-up (measured: cfg3, 16384 chunks, 158.8 -> 154.3 us per
  // step; cfg2, 1024 chunks, 30.3 -> 32.8 us)
  const bool spec = !u_packed && B <= spec_max_requests() && (long long)B * n_chunks(V) >= kSpecMinChunks;
  return resample_impl(in, u_res, spec ? u_acc : nullptr, spec && len ? len + row0 : nullptr, B, k, V, d, accepted,
                       offsets, out_tok, mass_out, tokens, status, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int tetris_step_stochastic_bf16(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                                           int32_t row0, int32_t B, const uint16_t* zp, const float* lse_p,
                                           const uint16_t* zq, const float* lse_q, const int32_t* d,
                                           const double* u_acc, int32_t u_packed, const double* u_res,
                                           const int32_t* cap, int32_t V, int32_t* windows, int32_t* win_offsets,
                                           int32_t* accepted, int32_t* out_tok, double* mass_out, int32_t* offsets,
                                           int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws,
                                           size_t ws_bytes, tetris_stream_t stream) {
  const ProbIn in = {nullptr, nullptr, zp, zq, lse_p, lse_q};
  return step_stochastic_impl(conf, len, B_sel, k, C, row0, B, in, d, u_acc, u_packed, u_res, cap, V, windows,
                              win_offsets, accepted, out_tok, mass_out, offsets, tokens, stats4, status, ws, ws_bytes,
                              stream);
}

static int verify_greedy_impl(const float* p, const int32_t* d, const int32_t* windows, const int32_t* cap, int B,
                              int k, int V, int32_t* accepted, int32_t* out_tok, int32_t* offsets, int32_t* tokens,
                              uint32_t* status, void* ws, size_t ws_bytes, cudaStream_t st) {
  int rc = check_shape(B, k, V);
  if (rc) return rc;
  if (B == 0) {
    if (offsets) {
      cudaError_t e = cudaMemsetAsync(offsets, 0, sizeof(int32_t), st);
      if (e != cudaSuccess) return abi::cuda_fail(e);
    }
    return TETRIS_OK;
  }
  if (!p || (k > 0 && !d) || !windows || !accepted || !out_tok)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if (offsets && !tokens) return abi::fail(TETRIS_INVALID_ARGUMENT, "tokens is required with offsets");
  if ((rc = check_verify_ws(B, k, V, ws, ws_bytes))) return rc;
  int* cnt = (int*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_COUNTERS);
  float* av = (float*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ARG_VAL);
  int32_t* ai = (int32_t*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ARG_IDX);
  int32_t* rowmap = (int32_t*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWMAP);
  if (persist_greedy_eligible(p, V)) {
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(av);
    if ((rc = launch_greedy_rowmap(windows, B, k, rowmap, keys, 1, st))) return rc;
    GreedyArgs a = {};
    a.p = p;
    a.d = d;
    a.windows = windows;
    a.cap = cap;
    a.B = B;
    a.k = k;
    a.V = V;
    a.nch = n_chunks(V);
    a.rowmap = rowmap;
    a.keys = keys;
    a.key0 = (unsigned long long*)(cnt + abi::kSlotGreedyKey0);
    a.grid_bar2 = (unsigned*)cnt + abi::kSlotWorkSpec;
    a.req_cnt = cnt;
    a.grid_bar = (unsigned*)cnt + abi::kSlotGridCount;
    a.accepted = accepted;
    a.out_tok = out_tok;
    a.offsets = offsets;
    a.tokens = tokens;
    a.status = status;
    return launch_persist_greedy(a, st);
  }
  if ((rc = launch_greedy_rowmap(windows, B, k, rowmap, nullptr, 0, st))) return rc;
  // one CTA per (selected row, chunk); the selected-row count Σ (w_b + 1) lives on the device, so the grid covers
  // the bound B * (k + 1) and CTAs past the count exit at once
  const long long rows_max = (long long)B * (k + 1);
  dim3 grid((unsigned)(rows_max * n_chunks(V)), 1, 1);
  if ((V % 8 == 0) && aligned32(p))
    greedy_kernel<true><<<grid, kStreamThreads, 0, st>>>(p, d, windows, k, V, accepted, out_tok, status, cnt, av, ai,
                                                         rowmap);
  else
    greedy_kernel<false><<<grid, kStreamThreads, 0, st>>>(p, d, windows, k, V, accepted, out_tok, status, cnt, av,
                                                          ai, rowmap);
  if ((rc = abi::launch_check())) return rc;
  return offsets ? tetris_compact(accepted, out_tok, d, cap, B, k, offsets, tokens, st) : TETRIS_OK;
}

// ---- host-buffer steps: the needed host rows are gathered by SM loads of the mapped host memory ----------------
// The stochastic step for HOST-resident p / q (the end-to-end path): the selector's accept test gathers its scalars
// from the mapped host memory; then stage_rows_kernel copies the row each request resamples from (rowinfo, left in the
// workspace by the selector epilogue) from the mapped host tensors into `staging` (request b: rows 2b, 2b+1) and
// rewrites rowinfo as staging rows, and the sampler runs on device memory.  Everything stays stream-ordered: no host
// synchronisation, capturable in a CUDA graph.  Measured on this box (tools/micro/h2d_rows.cu, 1800 rows of 513 KB):
// SM gather 51 GB/s, one cudaMemcpyAsync per row 37 GB/s (a ~4.5 us fixed cost per copy on the copy engine, whatever
// the stream count), one contiguous copy 55 GB/s (the link's ceiling, not reachable for scattered rows).
__device__ __forceinline__ void copy_row_h2d(const int4* __restrict__ src, int4* __restrict__ dst, long long words) {
  constexpr int U = 4;  // 16-byte loads in flight per thread
  for (long long i = threadIdx.x; i < words; i += U * blockDim.x) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * blockDim.x < words) v[u] = __ldcv(src + i + u * blockDim.x);  // host memory: never a stale line
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * blockDim.x < words) dst[i + u * blockDim.x] = v[u];
  }
}

// item 2b + t: request b's p row (t = 0) or q row (t = 1, absent for a bonus row) into staging row 2b + t
__global__ void __launch_bounds__(512) stage_rows_kernel(const char* __restrict__ p_map, const char* __restrict__ q_map,
                                                         const float* __restrict__ lsep_map,
                                                         const float* __restrict__ lseq_map, long long* rowinfo,
                                                         int B, long long row_bytes, char* staging,
                                                         float* lse_staging) {
  for (int it = blockIdx.x; it < 2 * B; it += gridDim.x) {
    const int b = it >> 1, t = it & 1;
    const long long r = rowinfo[2 * b + t];
    if (r < 0) continue;  // bonus: no q row
    copy_row_h2d((const int4*)((t ? q_map : p_map) + r * row_bytes), (int4*)(staging + (long long)it * row_bytes),
                 row_bytes / 16);
    __syncthreads();  // every thread has read rowinfo[it] before it is rewritten
    if (threadIdx.x == 0) {
      if (lse_staging) lse_staging[it] = (t ? lseq_map : lsep_map)[r];
      rowinfo[2 * b + t] = it;
    }
  }
}

// greedy: item b*(k+1) + j copies p[b][j] for j <= windows[b] into the same place of p_dev
__global__ void __launch_bounds__(512) stage_greedy_rows_kernel(const char* __restrict__ p_map,
                                                                const int32_t* __restrict__ windows, int B, int k,
                                                                long long row_bytes, char* p_dev) {
  const int n = B * (k + 1);
  for (int it = blockIdx.x; it < n; it += gridDim.x) {
    const int b = it / (k + 1), j = it - b * (k + 1);
    if (j > windows[b]) continue;
    copy_row_h2d((const int4*)(p_map + (long long)it * row_bytes), (int4*)(p_dev + (long long)it * row_bytes),
                 row_bytes / 16);
  }
}

static int stage_grid(long long items) {
  const long long g = 4LL * abi::device_sm_count();
  return (int)(items < g ? (items > 0 ? items : 1) : g);
}

template <typename T>
static int staged_impl(const double* conf, const int32_t* len, int32_t B, int32_t k, int64_t C, const T* p_host,
                       const T* q_host, const float* lsep_host, const float* lseq_host, const int32_t* d,
                       const double* u_acc, const double* u_res, const int32_t* cap, int32_t V, T* staging,
                       float* lse_staging, int32_t* windows, int32_t* win_offsets, int32_t* accepted, int32_t* out_tok,
                       double* mass_out, int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status,
                       void* ws, size_t ws_bytes, tetris_stream_t stream) {
  constexpr bool kLogits = sizeof(T) == 2;
  int rc = check_shape(B, k, V);
  if (rc) return rc;
  if (!p_host || (k > 0 && !q_host) || !staging ||
      (kLogits && (!lsep_host || (k > 0 && !lseq_host) || !lse_staging)))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if (V % 8 != 0 || !aligned16(staging) || !aligned16(p_host) || (q_host && !aligned16(q_host)))
    return abi::fail(TETRIS_INVALID_ARGUMENT,
                     "staged step needs V %% 8 == 0 and 16-byte aligned host tensors and staging buffer");
  cudaStream_t st = (cudaStream_t)stream;
  void *p_map = nullptr, *q_map = nullptr, *lp_map = nullptr, *lq_map = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&p_map, (void*)p_host, 0);
  if (e == cudaSuccess && q_host) e = cudaHostGetDevicePointer(&q_map, (void*)q_host, 0);
  if (kLogits && e == cudaSuccess) e = cudaHostGetDevicePointer(&lp_map, (void*)lsep_host, 0);
  if (kLogits && e == cudaSuccess && lseq_host) e = cudaHostGetDevicePointer(&lq_map, (void*)lseq_host, 0);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  const ProbIn mapped = kLogits ? ProbIn{nullptr, nullptr, (const uint16_t*)p_map, (const uint16_t*)q_map,
                                         (const float*)lp_map, (const float*)lq_map}
                                : ProbIn{(const float*)p_map, (const float*)q_map, nullptr, nullptr, nullptr, nullptr};
  if ((rc = select_accept_impl(conf, len, B, k, C, 0, B, mapped, d, u_acc, 0, cap, V, windows, win_offsets, accepted,
                               offsets, tokens, stats4, status, ws, ws_bytes, stream, /*host_inputs=*/true)))
    return rc;
  // the rows the selection chose, host -> staging (request b: rows 2b, 2b+1), rowinfo rewritten as staging rows
  long long* rowinfo = (long long*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWINFO);
  stage_rows_kernel<<<stage_grid(2LL * B), 512, 0, st>>>((const char*)p_map, (const char*)q_map,
                                                         (const float*)lp_map, (const float*)lq_map, rowinfo, B,
                                                         (long long)V * sizeof(T), (char*)staging,
                                                         kLogits ? lse_staging : nullptr);
  if ((rc = abi::launch_check())) return rc;
  const ProbIn staged = kLogits ? ProbIn{nullptr, nullptr, (const uint16_t*)staging, (const uint16_t*)staging,
                                         lse_staging, lse_staging}
                                : ProbIn{(const float*)staging, (const float*)staging, nullptr, nullptr, nullptr,
                                         nullptr};
  return resample_impl(staged, u_res, nullptr, nullptr, B, k, V, d, accepted, offsets, out_tok, mass_out, tokens,
                       status, ws, ws_bytes, st);
}

extern "C" int tetris_step_stochastic_staged_f32(const double* conf, const int32_t* len, int32_t B, int32_t k,
                                                 int64_t C, const float* p_host, const float* q_host,
                                                 const int32_t* d, const double* u_acc, const double* u_res,
                                                 const int32_t* cap, int32_t V, float* staging, int32_t* windows,
                                                 int32_t* win_offsets, int32_t* accepted, int32_t* out_tok,
                                                 double* mass_out, int32_t* offsets, int32_t* tokens, int64_t* stats4,
                                                 uint32_t* status, void* ws, size_t ws_bytes,
                                                 tetris_stream_t stream) {
  return staged_impl<float>(conf, len, B, k, C, p_host, q_host, nullptr, nullptr, d, u_acc, u_res, cap, V, staging,
                            nullptr, windows, win_offsets, accepted, out_tok, mass_out, offsets, tokens, stats4,
                            status, ws, ws_bytes, stream);
}

extern "C" int tetris_step_stochastic_staged_bf16(const double* conf, const int32_t* len, int32_t B, int32_t k,
                                                  int64_t C, const uint16_t* zp_host, const float* lse_p_host,
                                                  const uint16_t* zq_host, const float* lse_q_host, const int32_t* d,
                                                  const double* u_acc, const double* u_res, const int32_t* cap,
                                                  int32_t V, uint16_t* staging, float* lse_staging, int32_t* windows,
                                                  int32_t* win_offsets, int32_t* accepted, int32_t* out_tok,
                                                  double* mass_out, int32_t* offsets, int32_t* tokens,
                                                  int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                                  tetris_stream_t stream) {
  return staged_impl<uint16_t>(conf, len, B, k, C, zp_host, zq_host, lse_p_host, lse_q_host, d, u_acc, u_res, cap, V,
                               staging, lse_staging, windows, win_offsets, accepted, out_tok, mass_out, offsets,
                               tokens, stats4, status, ws, ws_bytes, stream);
}

// The greedy step (select -> greedy verification -> compaction) in 2 launches when the selector is the single-CTA one
// (its epilogue writes the row list) and p qualifies for the persistent stream; otherwise select + row list + stream.
extern "C" int tetris_step_greedy_f32(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                                      int32_t row0, int32_t B, const float* p, const int32_t* d, const int32_t* cap,
                                      int32_t V, int32_t* windows, int32_t* win_offsets, int32_t* accepted,
                                      int32_t* out_tok, int32_t* offsets, int32_t* tokens, int64_t* stats4,
                                      uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  int rc = check_shape(B, k, V);
  if (rc) return rc;
  if (C < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0, got %lld", (long long)C);
  if (B == 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "empty batch");
  if (B_sel < B || B_sel > TETRIS_MAX_SELECT_ROWS || row0 < 0 || row0 + B > B_sel)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "local rows [%d, %d) outside the %d selected rows", row0, row0 + B, B_sel);
  if ((k > 0 && (!conf || !d)) || !p || !windows || !accepted || !out_tok || !offsets || !tokens)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if ((rc = check_verify_ws(B, k, V, ws, ws_bytes))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (!persist_greedy_eligible(p, V)) {
    if ((rc = tetris_select_f64(conf, len, B_sel, k, C, 0, windows, win_offsets, nullptr, stats4, status, ws, ws_bytes,
                                stream)))
      return rc;
    return verify_greedy_impl(p, d, windows + row0, cap, B, k, V, accepted, out_tok, offsets, tokens, status, ws,
                              ws_bytes, st);
  }
  int* cnt = (int*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_COUNTERS);
  unsigned long long* keys = (unsigned long long*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ARG_VAL);
  int32_t* rowmap = (int32_t*)abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_ROWMAP);
  GreedyArgs a = {};
  a.p = p;
  a.d = d;
  a.windows = windows + row0;
  a.cap = cap;
  a.B = B;
  a.k = k;
  a.V = V;
  a.nch = n_chunks(V);
  a.rowmap = rowmap;
  a.keys = keys;
  a.key0 = (unsigned long long*)(cnt + abi::kSlotGreedyKey0);
  a.grid_bar2 = (unsigned*)cnt + abi::kSlotWorkSpec;
  a.req_cnt = cnt;
  a.grid_bar = (unsigned*)cnt + abi::kSlotGridCount;
  a.accepted = accepted;
  a.out_tok = out_tok;
  a.offsets = offsets;
  a.tokens = tokens;
  a.status = status;
  if (fused_step_eligible(B_sel, k, 0) && greedy_fused_fits(B_sel, k)) {
    // small batch: ONE launch — the selection as the argmax stream's prologue (greedy.cu, FUSED)
    FusedSel& f = a.fs;
    static const double kNoScores = 0.0;  // k == 0: nothing is read through it
    f.conf = conf ? conf : &kNoScores;
    f.len = len;
    f.B_sel = B_sel;
    f.row0 = row0;
    f.C = (long long)C;
    f.windows = windows;
    f.win_offsets = win_offsets;
    f.stats = (long long*)stats4;
    f.ctl = cnt + abi::kSlotFusedCtl;
    f.ready = reinterpret_cast<unsigned long long*>(cnt + abi::kSlotFusedReady);
    if (k == 0 && !d) a.d = (const int32_t*)&kNoScores;
    return launch_persist_greedy(a, st);
  }
  SelectArgs sa = {};
  sa.vals = conf;
  sa.len = len;
  sa.B = B_sel;
  sa.k = k;
  sa.C = (long long)C;
  sa.windows = windows;
  sa.win_offsets = win_offsets;
  sa.stats = (long long*)stats4;
  sa.status = status;
  sa.ep_row0 = row0;
  sa.ep_rows = B;
  sa.gscratch = abi::ws_region(ws, TETRIS_OP_VERIFY, B, k, V, abi::WS_GSEL);
  const bool fused_rows = select1_eligible(B_sel, k);
  if (fused_rows) {
    sa.rowmap = rowmap;
    sa.gkeys = keys;
  }
  if ((rc = launch_select(sa, st))) return rc;
  if (!fused_rows && (rc = launch_greedy_rowmap(windows + row0, B, k, rowmap, keys, 1, st))) return rc;
  return launch_persist_greedy(a, st);
}

extern "C" int tetris_verify_greedy_f32(const float* p, const int32_t* d, const int32_t* windows, int32_t B,
                                        int32_t k, int32_t V, int32_t* accepted, int32_t* out_tok,
                                        uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  return verify_greedy_impl(p, d, windows, nullptr, B, k, V, accepted, out_tok, nullptr, nullptr, status, ws, ws_bytes,
                            (cudaStream_t)stream);
}

extern "C" int tetris_verify_greedy_compact_f32(const float* p, const int32_t* d, const int32_t* windows,
                                                const int32_t* cap, int32_t B, int32_t k, int32_t V,
                                                int32_t* accepted, int32_t* out_tok, int32_t* offsets,
                                                int32_t* tokens, uint32_t* status, void* ws, size_t ws_bytes,
                                                tetris_stream_t stream) {
  if (!offsets) return abi::fail(TETRIS_INVALID_ARGUMENT, "offsets is required");
  return verify_greedy_impl(p, d, windows, cap, B, k, V, accepted, out_tok, offsets, tokens, status, ws, ws_bytes,
                            (cudaStream_t)stream);
}

extern "C" int tetris_sample_rows_f64(const double* p, const double* q, const int64_t* p_row, const int64_t* q_row,
                                      const double* u, int32_t R, int32_t V, int32_t* out_idx, double* mass_out,
                                      uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  return sample_rows_impl<double>(p, q, p_row, q_row, u, R, V, out_idx, mass_out, status, ws, ws_bytes,
                                  (cudaStream_t)stream);
}

extern "C" int tetris_sample_rows_f32(const float* p, const float* q, const int64_t* p_row, const int64_t* q_row,
                                      const double* u, int32_t R, int32_t V, int32_t* out_idx, double* mass_out,
                                      uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  if (R > 0 && R <= 65535 && V >= 1 && p && p_row && u && out_idx && persist_eligible(p, q, V) &&
      ws_bytes >= tetris_workspace_bytes(TETRIS_OP_VERIFY, R, 0, V) && ws) {
    StreamArgs a = {};
    a.p = p;
    a.q = q;
    a.V = V;
    a.nch = n_chunks(V);
    a.R = R;
    a.prow = (const long long*)p_row;
    a.qrow = (q && q_row) ? (const long long*)q_row : nullptr;
    a.row_stride = 1;
    a.u = u;
    a.out_idx = out_idx;
    a.mass_out = mass_out;
    a.status = status;
    a.counters = (int*)abi::ws_region(ws, TETRIS_OP_VERIFY, R, 0, V, abi::WS_COUNTERS);
    a.chunk_sums = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, R, 0, V, abi::WS_CHUNK_SUMS);
    a.warp_sums = (double*)abi::ws_region(ws, TETRIS_OP_VERIFY, R, 0, V, abi::WS_WARP_SUMS);
    a.grid_bar = (unsigned*)a.counters + abi::kSlotGridCount;
    a.req_cnt = a.counters;
    return launch_persist_stream(a, (cudaStream_t)stream);
  }
  return sample_rows_impl<float>(p, q, p_row, q_row, u, R, V, out_idx, mass_out, status, ws, ws_bytes,
                                 (cudaStream_t)stream);
}

extern "C" int tetris_residual_f64(const double* p_draft, const double* p_target, int32_t R, int32_t V, double* out,
                                   double* mass_out, uint32_t* status, void* ws, size_t ws_bytes,
                                   tetris_stream_t stream) {
  // mass via the sampler (u = 0 -> first positive element, discarded), then out = max(0, pt - ps) / mass.
  int rc = check_shape(R, 0, V);
  if (rc) return rc;
  if (R == 0) return TETRIS_OK;
  if (!p_draft || !p_target || !out || !mass_out) return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if ((rc = check_verify_ws(R, 0, V, ws, ws_bytes))) return rc;
  char* x = (char*)abi::ws_region(ws, TETRIS_OP_VERIFY, R, 0, V, abi::WS_SCRATCH);
  int64_t* prow = (int64_t*)x;
  int64_t* qrow = (int64_t*)(x + abi::align_up((size_t)R * 8));
  double* u = (double*)(x + 2 * abi::align_up((size_t)R * 8));
  int32_t* idx = (int32_t*)(x + 3 * abi::align_up((size_t)R * 8));
  cudaStream_t st = (cudaStream_t)stream;
  // rows r -> r for both operands; uniforms 0
  identity_rows_kernel<<<(R + 255) / 256, 256, 0, st>>>(prow, qrow, u, R);
  // weights = max(0, p - q) with p = p_target, q = p_draft
  rc = sample_rows_impl<double>(p_target, p_draft, prow, qrow, u, R, V, idx, mass_out, status, ws, ws_bytes, st);
  if (rc) return rc;
  dim3 grid((V + 255) / 256 < 1024 ? (V + 255) / 256 : 1024, R);
  residual_norm_kernel<<<grid, 256, 0, st>>>(p_draft, p_target, V, mass_out, out);
  return abi::launch_check();
}

// The greedy step for host-resident p: selection, then stage_greedy_rows_kernel copies each request's verified rows
// p[b][0..w_b] from the mapped host tensor into the same place of p_dev, then the greedy verification + compaction
// on p_dev.  Stream-ordered, no host synchronisation.
extern "C" int tetris_step_greedy_staged_f32(const double* conf, const int32_t* len, int32_t B, int32_t k, int64_t C,
                                             const float* p_host, const int32_t* d, const int32_t* cap, int32_t V,
                                             float* p_dev, int32_t* windows, int32_t* win_offsets, int32_t* accepted,
                                             int32_t* out_tok, int32_t* offsets, int32_t* tokens, int64_t* stats4,
                                             uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  using namespace tetris;
  int rc = check_shape(B, k, V);
  if (rc) return rc;
  if (C < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0, got %lld", (long long)C);
  if (B == 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "empty batch");
  if ((k > 0 && (!conf || !d)) || !p_host || !p_dev || !windows || !accepted || !out_tok || !offsets || !tokens)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  if (V % 4 != 0 || !aligned16(p_dev) || !aligned16(p_host))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "staged greedy step needs V %% 4 == 0 and 16-byte aligned p_host, p_dev");
  if ((rc = check_verify_ws(B, k, V, ws, ws_bytes))) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  void* p_map = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&p_map, (void*)p_host, 0);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  if ((rc = tetris_select_f64(conf, len, B, k, C, 0, windows, win_offsets, nullptr, stats4, status, ws, ws_bytes,
                              stream)))
    return rc;
  stage_greedy_rows_kernel<<<stage_grid((long long)B * (k + 1)), 512, 0, st>>>(
      (const char*)p_map, windows, B, k, (long long)V * sizeof(float), (char*)p_dev);
  if ((rc = abi::launch_check())) return rc;
  return verify_greedy_impl(p_dev, d, windows, cap, B, k, V, accepted, out_tok, offsets, tokens, status, ws, ws_bytes,
                            st);
}

// ---- the logits contract materialised: prob(z, lse) for R rows of V bf16 logits (tests, adapters) ---------------
__global__ void probs_from_logits_kernel(const uint16_t* __restrict__ z, const float* __restrict__ lse, int64_t R,
                                         int V, float* __restrict__ out) {
  const int64_t n = R * (int64_t)V;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = tetris::prob_from_logit(z[e], lse[e / V]);
}

extern "C" int tetris_probs_from_logits_bf16(const uint16_t* z, const float* lse, int64_t R, int32_t V, float* out,
                                             tetris_stream_t stream) {
  using namespace tetris;
  if (R < 0 || V < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "bad shape R=%lld V=%d", (long long)R, V);
  if (R == 0 || V == 0) return TETRIS_OK;
  if (!z || !lse || !out) return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  const int64_t n = R * (int64_t)V;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  probs_from_logits_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(z, lse, R, V, out);
  return abi::launch_check();
}
