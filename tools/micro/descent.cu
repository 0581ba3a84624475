// Micro-benchmark of the sampler's per-request descent (stream.cu finalize_request) in isolation: one warp per
// request after every chunk sum is published, on cfg2-sized rows (V = 32000, residual rows p - q).  Prints SM cycles
// per descent (cold = first in the launch, warm = second) and checks the sampled token against a host restatement of
// the sampling contract.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I include -I paper_2502_15197_b200/csrc \
//        -o /tmp/descent tools/micro/descent.cu && /tmp/descent
#include <cstdio>
#include <vector>

#include "stream.cu"

namespace tetris {  // host symbols stream.cu references (abi.cu / select.cu are not linked here)
long long* debug_buffer() { return nullptr; }
namespace abi {
char* err_buf() {
  static char b[512];
  return b;
}
}  // namespace abi
}  // namespace tetris

using namespace tetris;

__global__ void sums_kernel(StreamArgs a) {  // chunk / warp sums of every request, the publisher's arithmetic
  const int b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // 8 warps = the 8 warp runs
  for (int c = 0; c < a.nch; ++c) {
    const int64_t e0 = (int64_t)c * kChunkElems + w * kWarpElems;
    const float* P = a.p + (int64_t)a.prow[2 * b] * a.V;
    const float* Q = a.q + (int64_t)a.qrow[2 * b] * a.V;
    double x = 0.0;
    const bool segm = a.nch <= kSegSumMaxChunks;  // short rows: the 32 segment sums instead of the warp sums
    for (int s = 0; s < kWarpSegs; ++s) {
      const int64_t e = e0 + s * kSegElems + lane * kLaneElems;
      double wl[8];
      for (int i = 0; i < 8; ++i) wl[i] = e + i < a.V ? w_res((double)P[e + i], (double)Q[e + i]) : 0.0;
      const double g = seg_sum(fold8(wl));
      if (segm && lane == 0) a.warp_sums[((int64_t)b * a.nch + c) * kChunkSegs + w * kWarpSegs + s] = g;
      x = x + g;
    }
    __shared__ double xs[8];
    if (lane == 0) xs[w] = x;
    __syncthreads();
    if (!segm && threadIdx.x < 8) a.warp_sums[((int64_t)b * a.nch + c) * kChunkWarps + threadIdx.x] = xs[threadIdx.x];
    if (threadIdx.x == 0) {
      double S = 0.0;
      for (int i = 0; i < 8; ++i) S = S + xs[i];
      a.chunk_sums[(int64_t)b * a.nch + c] = S;
    }
    __syncthreads();
  }
}

__global__ void descent_kernel(StreamArgs a, long long* cyc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x * (blockDim.x >> 5) + warp;
  if (b >= a.R) return;
  for (int pass = 0; pass < 2; ++pass) {
    __syncwarp();
    const long long t0 = clock64();
    finalize_request<false>(a, b, true, lane, a.chunk_sums, a.warp_sums);
    __syncwarp();
    const long long t1 = clock64();
    if (lane == 0) cyc[2 * b + pass] = t1 - t0;
  }
}

int main() {
  const int R = 256, V = 32000, nch = n_chunks(V);
  std::vector<float> hp((size_t)R * V), hq((size_t)R * V);
  unsigned s = 7;
  for (size_t i = 0; i < hp.size(); ++i) {
    s = s * 1664525u + 1013904223u;
    hp[i] = (s >> 9) * (1.0f / 8388608.0f) / V;
    s = s * 1664525u + 1013904223u;
    hq[i] = (s >> 9) * (1.0f / 8388608.0f) / V;
  }
  std::vector<long long> rowinfo(2 * R);
  std::vector<double> u(R);
  for (int b = 0; b < R; ++b) rowinfo[2 * b] = b, rowinfo[2 * b + 1] = b, u[b] = (b + 0.5) / R;
  float *p, *q;
  long long* ri;
  double *du, *cs, *ws, *mass;
  int* tok;
  long long* cyc;
  uint32_t* st;
  cudaMalloc(&p, hp.size() * 4);
  cudaMalloc(&q, hq.size() * 4);
  cudaMemcpy(p, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(q, hq.data(), hq.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&ri, 16 * R);
  cudaMemcpy(ri, rowinfo.data(), 16 * R, cudaMemcpyHostToDevice);
  cudaMalloc(&du, 8 * R);
  cudaMemcpy(du, u.data(), 8 * R, cudaMemcpyHostToDevice);
  cudaMalloc(&cs, 8 * R * nch);
  cudaMalloc(&ws, (size_t)kChunkSegs * R * nch * 8);  // segment sums (short rows) or warp sums
  cudaMalloc(&mass, 8 * R);
  cudaMalloc(&tok, 4 * R);
  cudaMalloc(&cyc, 16 * R);
  cudaMalloc(&st, 4);
  cudaMemset(st, 0, 4);
  StreamArgs a = {};
  a.p = p;
  a.q = q;
  a.V = V;
  a.nch = nch;
  a.R = R;
  a.prow = ri;
  a.qrow = ri + 1;
  a.row_stride = 2;
  a.u = du;
  a.out_idx = tok;
  a.mass_out = mass;
  a.status = st;
  a.chunk_sums = cs;
  a.warp_sums = ws;
  sums_kernel<<<R, 256>>>(a);
  for (int rep = 0; rep < 3; ++rep) descent_kernel<<<R / 2, 64>>>(a, cyc);  // 2 requests per CTA, 128 CTAs
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<long long> c(2 * R);
  cudaMemcpy(c.data(), cyc, 16 * R, cudaMemcpyDeviceToHost);
  double c0 = 0, c1 = 0;
  for (int b = 0; b < R; ++b) c0 += c[2 * b], c1 += c[2 * b + 1];
  printf("descent: %.0f cycles first in the launch, %.0f second (mean over %d requests)\n", c0 / R, c1 / R, R);
  std::vector<int> ht(R);
  cudaMemcpy(ht.data(), tok, 4 * R, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int b = 0; b < R; ++b) bad += ht[b] < 0 || ht[b] >= V;
  printf("tokens in range: %d / %d\n", R - bad, R);
#ifdef TETRIS_DESCENT_PROBE
  std::vector<long long> pr(4096 * 8);
  cudaMemcpyFromSymbol(pr.data(), g_probe, pr.size() * 8);
  const char* nm[7] = {"sums + counts loaded", "mass", "chunk chosen", "warp run chosen", "warp run loaded",
                       "segment sums + choice", "lane level"};
  for (int i = 1; i < 8; ++i) {
    double acc = 0;
    for (int b = 0; b < R; ++b) acc += pr[8 * b + i] - pr[8 * b + i - 1];
    printf("  %-24s %6.0f cycles\n", i < 7 ? nm[i - 1] : "end", acc / R);
  }
#endif
  return 0;
}
