// Stage (3) streaming: the persistent, warp-specialised residual / bonus sampler (sm_100a, fp32 rows, V % 8 == 0).
//
// One CTA per SM, 10 warps:
//   warp 8      producer: walks this CTA's work items (request b, chunk c) and issues 1-D bulk copies on the TMA
//               engine (cp.async.bulk + mbarrier complete_tx) of the chunk of the row to resample from — p[b][a_b]
//               and q[b][a_b] after a rejection, p[b][w_b] for the bonus — into a 3-stage shared-memory ring;
//   warps 0..7  consumers: each folds one 1024-element warp run of the staged chunk into the sampling-contract
//               sums (lane: 8 elements left to right; segment: xor butterfly; warp: 4 segments left to right) and
//               hands the 8 warp sums to the finalizer through a shared-memory ring;
//   warp 9      finalizer: folds the chunk sum, publishes chunk + warp sums, bumps the request's arrival counter
//               (atom.acq_rel.gpu, result consumed one item later so its latency overlaps) and, for the last chunk of
//               a request, runs the descent T = u*mass -> chunk -> warp -> segment -> lane -> element, re-reading only
//               the one 1024-element warp run that holds the sample.
// HBM is touched once per streamed element; the descent's re-read is 4-8 KB per request.  The accept test and the
// row choice come from the select kernel's epilogue (rowinfo), so the producer never waits on a dependent gather.
#include "common.cuh"
#include "launch.h"

namespace tetris {

constexpr int kStages = 3;
constexpr int kConsumerWarps = kChunkWarps;  // 8
constexpr int kProducerWarp = 8;
constexpr int kFinalWarp = 9;
constexpr int kPersistThreads = 10 * 32;
constexpr int kRing = 32;
constexpr size_t kStageRowBytes = (size_t)kChunkElems * sizeof(float);  // 32 KB
constexpr size_t kStageBytes = 2 * kStageRowBytes;                         // p + q chunk
constexpr size_t kPersistSmem = kStages * kStageBytes;                     // 192 KB dynamic



struct StageMeta {
  int b, c, res, pad;
};

struct PersistShared {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t ring_full[kRing];
  uint64_t ring_free[kRing];
  StageMeta meta[kStages];
  StageMeta ring_meta[kRing];
  double ring_w[kRing][kChunkWarps];
};

__device__ __forceinline__ void consume_warp_run(const float* __restrict__ sp, const float* __restrict__ sq, bool res,
                                                 int64_t e0, int off0, int V, int lane, double (&G)[kWarpSegs]) {
#pragma unroll
  for (int s = 0; s < kWarpSegs; ++s) {
    const int off = off0 + s * kSegElems + lane * kLaneElems;
    double w[8];
    if (e0 + s * kSegElems + lane * kLaneElems < V) {
      float pv[8];
      lds8(sp + off, pv);
      if (res) {
        float qv[8];
        lds8(sq + off, qv);
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = w_res((double)pv[i], (double)qv[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = w_plain((double)pv[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = 0.0;
    }
    G[s] = seg_sum(fold8(w));
  }
}

// descent below the warp level, reading the warp run from global memory (all 32 lanes, T uniform)
template <bool RES>
__device__ int descend_global(const float* __restrict__ P, const float* __restrict__ Q, int64_t e0, int V, int lane,
                              double T) {
  double G[kWarpSegs];
  float pv[kWarpSegs][8], qv[kWarpSegs][8];
#pragma unroll
  for (int s = 0; s < kWarpSegs; ++s) {
    load_lane<float, true>(P, e0 + s * kSegElems + lane * kLaneElems, V, pv[s]);
    if (RES) load_lane<float, true>(Q, e0 + s * kSegElems + lane * kLaneElems, V, qv[s]);
  }
  double wl[kWarpSegs][8];
#pragma unroll
  for (int s = 0; s < kWarpSegs; ++s) {
#pragma unroll
    for (int i = 0; i < 8; ++i) wl[s][i] = RES ? w_res((double)pv[s][i], (double)qv[s][i]) : w_plain((double)pv[s][i]);
    G[s] = seg_sum(fold8(wl[s]));
  }
  const int s = seq_find(G, kWarpSegs, T);
  if (s < 0) return -1;
  double w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double x = wl[0][i];
#pragma unroll
    for (int ss = 1; ss < kWarpSegs; ++ss) x = (s == ss) ? wl[ss][i] : x;
    w[i] = x;
  }
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
    const double Rr = __shfl_sync(kFull, lv[t], g + (1 << t));
    if (!(L > T || Rr == 0.0)) {
      T = T - L;
      g += 1 << t;
    }
  }
  double Tl = T;
  const int li_own = seq_find(w, 8, Tl);
  const int li = __shfl_sync(kFull, li_own, g);
  if (li < 0) return -1;
  return (int)(e0 + s * kSegElems + g * kLaneElems + li);
}

// The last chunk of request b has been published: mass, T = u*mass, descent, outputs (finalizer warp).
__device__ void finalize_request(const StreamArgs& a, int b, bool res, int lane) {
  const int nch = a.nch;
  const long long prow = a.prow[(int64_t)b * a.row_stride];
  const long long qrow = a.qrow ? a.qrow[(int64_t)b * a.row_stride] : -1;
  double S[64];
  double mass = 0.0;
  for (int c = 0; c < nch; ++c) {
    S[c] = __ldcg(&a.chunk_sums[(int64_t)b * nch + c]);
    mass = mass + S[c];
  }
  uint32_t bad = 0;
  const double u = a.u[b];
  if (!(u >= 0.0 && u < 1.0)) bad |= TETRIS_ST_BAD_UNIFORM;
  int tok = -1;
  if (mass > 0.0) {
    double T = u * mass;
    const int cc = seq_find(S, nch, T);
    double Wc[kChunkWarps];
#pragma unroll
    for (int w = 0; w < kChunkWarps; ++w) Wc[w] = __ldcg(&a.warp_sums[((int64_t)b * nch + cc) * kChunkWarps + w]);
    const int ww = seq_find(Wc, kChunkWarps, T);
    const int64_t e0 = (int64_t)cc * kChunkElems + ww * kWarpElems;
    const float* P = a.p + prow * (int64_t)a.V;
    tok = res ? descend_global<true>(P, a.q + qrow * (int64_t)a.V, e0, a.V, lane, T)
              : descend_global<false>(P, nullptr, e0, a.V, lane, T);
  }
  if (tok < 0) bad |= TETRIS_ST_DEGENERATE;
  if (lane == 0) {
    a.counters[b] = 0;
    a.out_idx[b] = tok;
    if (a.mass_out) a.mass_out[b] = mass;
    if (a.accepted) {
      const int acc = a.accepted[b];
      const int pos = a.offsets[b] + acc;
      if (pos < a.offsets[b + 1]) a.tokens[pos] = tok;  // the sample is emitted unless the cap cut it
    }
    set_status(a.status, bad);
  }
}

__global__ void __launch_bounds__(kPersistThreads, 1) persist_stream_kernel(const StreamArgs a) {
  extern __shared__ __align__(128) uint8_t stage_mem[];
  __shared__ PersistShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nch = a.nch;
  const long long total = (long long)a.R * nch;
  const int G = gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sh.full[s], 1);
      mbar_init(&sh.empty[s], kConsumerWarps);
    }
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&sh.ring_full[r], kConsumerWarps);
      mbar_init(&sh.ring_free[r], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kProducerWarp) {
    // ---------------------------------------------------------------- producer
    long long pr_p = 0, pr_q = -1;
    int t = 0;
    for (long long i = blockIdx.x; i < total; i += G, ++t) {
      if ((t & 31) == 0) {  // refill 32 items of row info, one per lane
        const long long ii = i + (long long)lane * G;
        if (ii < total) {
          const int bb = (int)(ii / nch);
          pr_p = a.prow[(int64_t)bb * a.row_stride];
          pr_q = a.qrow ? a.qrow[(int64_t)bb * a.row_stride] : -1;
        }
      }
      const long long prow = __shfl_sync(kFull, pr_p, t & 31);
      const long long qrow = __shfl_sync(kFull, pr_q, t & 31);
      const int s = t % kStages;
      const uint32_t ph = (uint32_t)((t / kStages) & 1);
      if (t >= kStages) mbar_wait(&sh.empty[s], ph ^ 1u);
      if (lane == 0) {
        const int b = (int)(i / nch), c = (int)(i % nch);
        const int n = min(kChunkElems, a.V - c * kChunkElems);
        const uint32_t bytes = (uint32_t)n * sizeof(float);
        const bool res = qrow >= 0;
        sh.meta[s] = StageMeta{b, c, res ? 1 : 0, 0};
        float* sp = reinterpret_cast<float*>(stage_mem + s * kStageBytes);
        mbar_arrive_expect_tx(&sh.full[s], res ? 2 * bytes : bytes);
        bulk_g2s(sp, a.p + prow * (int64_t)a.V + (int64_t)c * kChunkElems, bytes, &sh.full[s]);
        if (res) bulk_g2s(sp + kChunkElems, a.q + qrow * (int64_t)a.V + (int64_t)c * kChunkElems, bytes, &sh.full[s]);
      }
      __syncwarp();
    }
  } else if (warp < kConsumerWarps) {
    // ---------------------------------------------------------------- consumers
    int t = 0;
    for (long long i = blockIdx.x; i < total; i += G, ++t) {
      const int s = t % kStages;
      mbar_wait(&sh.full[s], (uint32_t)((t / kStages) & 1));
      const StageMeta m = sh.meta[s];
      const float* sp = reinterpret_cast<const float*>(stage_mem + s * kStageBytes);
      double Gs[kWarpSegs];
      const int off0 = warp * kWarpElems;
      consume_warp_run(sp, sp + kChunkElems, m.res != 0, (int64_t)m.c * kChunkElems + off0, off0, a.V, lane, Gs);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[s]);
      double W = 0.0;
#pragma unroll
      for (int x = 0; x < kWarpSegs; ++x) W = W + Gs[x];
      const int slot = t % kRing;
      if (t >= kRing) mbar_wait(&sh.ring_free[slot], (uint32_t)(((t / kRing) & 1) ^ 1));
      if (lane == 0) {
        sh.ring_w[slot][warp] = W;
        if (warp == 0) sh.ring_meta[slot] = m;
        mbar_arrive(&sh.ring_full[slot]);
      }
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- finalizer
    int prev_b = -1, prev_res = 0, prev_old = -1;
    int t = 0;
    for (long long i = blockIdx.x; i < total; i += G, ++t) {
      const int slot = t % kRing;
      mbar_wait(&sh.ring_full[slot], (uint32_t)((t / kRing) & 1));
      const StageMeta m = sh.ring_meta[slot];
      __syncwarp();
      int old = 0;
      if (lane == 0) {
        double W[kChunkWarps];
        double S = 0.0;
#pragma unroll
        for (int w = 0; w < kChunkWarps; ++w) {
          W[w] = sh.ring_w[slot][w];
          S = S + W[w];
        }
        mbar_arrive(&sh.ring_free[slot]);
        const int64_t cs = (int64_t)m.b * nch + m.c;
        __stcg(&a.chunk_sums[cs], S);
#pragma unroll
        for (int w = 0; w < kChunkWarps; ++w) __stcg(&a.warp_sums[cs * kChunkWarps + w], W[w]);
        old = atomic_add_acq_rel_gpu(&a.counters[m.b], 1);
      }
      // the previous item's arrival result has landed by now; finalize its request if it was the last chunk
      const int po = __shfl_sync(kFull, prev_old, 0);
      if (prev_b >= 0 && po == nch - 1) finalize_request(a, prev_b, prev_res != 0, lane);
      prev_b = m.b;
      prev_res = m.res;
      prev_old = old;
    }
    const int po = __shfl_sync(kFull, prev_old, 0);
    if (prev_b >= 0 && po == nch - 1) finalize_request(a, prev_b, prev_res != 0, lane);
  }
}

// ---- stand-alone accept test (verify_stochastic without the fused selector epilogue) ----------------------------
__global__ void accept_kernel(const float* __restrict__ p, const float* __restrict__ q, const int32_t* __restrict__ d,
                              const int32_t* __restrict__ windows, const int32_t* __restrict__ win_off,
                              const double* __restrict__ u_acc, int B, int k, int V, int32_t* __restrict__ accepted,
                              long long* __restrict__ rowinfo, uint32_t* status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  uint32_t bad = 0;
  int w = windows[b];
  if (w < 0 || w > k) {
    bad |= TETRIS_ST_BAD_WINDOW;
    w = w < 0 ? 0 : k;
  }
  const int64_t uoff = win_off ? (int64_t)win_off[b] : (int64_t)b * k;
  int acc = w;
  for (int j0 = 0; j0 < w && acc == w; j0 += 8) {
    int t[8];
    double u[8], s[8], m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = j0 + i;
      t[i] = (j < w) ? d[(int64_t)b * k + j] : 0;
      u[i] = (j < w) ? u_acc[uoff + j] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = j0 + i;
      const bool ok = (j < w) && t[i] >= 0 && t[i] < V;
      s[i] = ok ? (double)q[((int64_t)b * k + j) * V + t[i]] : 0.0;
      m[i] = ok ? (double)p[((int64_t)b * (k + 1) + j) * V + t[i]] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = j0 + i;
      if (j >= w || acc != w) continue;
      if (!(u[i] >= 0.0 && u[i] < 1.0)) bad |= TETRIS_ST_BAD_UNIFORM;
      bool rej;
      if (t[i] < 0 || t[i] >= V) {
        bad |= TETRIS_ST_BAD_TOKEN;
        rej = true;
      } else {
        rej = !(s[i] <= m[i]) && !(u[i] < m[i] / s[i]);  // accept_model.py:311-313
      }
      if (rej) acc = j;
    }
  }
  accepted[b] = acc;
  rowinfo[2 * (int64_t)b] = (long long)b * (k + 1) + acc;
  rowinfo[2 * (int64_t)b + 1] = acc < w ? (long long)b * k + acc : -1;
  set_status(status, bad);
}

}  // namespace tetris

// ---- host side ---------------------------------------------------------------------------------------------------
#include "abi_util.h"

namespace tetris {

static int g_num_sms = 0;

int launch_persist_stream(const StreamArgs& a, cudaStream_t st) {
  if (a.R == 0) return TETRIS_OK;
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  cudaError_t e =
      cudaFuncSetAttribute(persist_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPersistSmem);
  if (e != cudaSuccess) return abi::cuda_fail(e);
  const long long items = (long long)a.R * a.nch;
  const int grid = (int)(items < g_num_sms ? items : g_num_sms);
  persist_stream_kernel<<<grid, kPersistThreads, kPersistSmem, st>>>(a);
  return abi::launch_check();
}

bool persist_eligible(const float* p, const float* q, int V) {
  return (V % kLaneElems == 0) && (((uintptr_t)p & 15u) == 0) && (!q || (((uintptr_t)q & 15u) == 0)) &&
         n_chunks(V) <= 64;
}

int launch_accept(const float* p, const float* q, const int32_t* d, const int32_t* windows, const int32_t* win_off,
                  const double* u_acc, int B, int k, int V, int32_t* accepted, long long* rowinfo, uint32_t* status,
                  cudaStream_t st) {
  accept_kernel<<<(B + 127) / 128, 128, 0, st>>>(p, q, d, windows, win_off, u_acc, B, k, V, accepted, rowinfo,
                                                 status);
  return abi::launch_check();
}

}  // namespace tetris
