// Micro-benchmark of the fused prologue's phases (fused_select.cuh) in isolation on the cfg2 shape (B_sel = 256,
// k = 8, 148 CTAs of 544 participants): clock64 per phase, cold (first pass) and warm (second pass), and CTA 0's
// ranks against a host count.  Measured on B200 (SM cycles): loads ~1800, keys ~770, ranks ~2830 — the rank loop is
// bound by the integer pipe (64 lanes/clk/SM: 3 ALU instructions per (key, cell) pair); an earlier per-cell layout
// (lanes = cells, broadcast key loads) took ~5000, a predicate-select accumulation ~4900.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -I include -I paper_2502_15197_b200/csrc \
//        -o /tmp/ranks tools/micro/ranks.cu && /tmp/ranks
#include <cstdio>
#include <cstring>
#include <vector>

#include "fused_select.cuh"

using namespace tetris;

__global__ void __launch_bounds__(576, 1) phases_kernel(FusedSel f, int k, long long* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, NP = 544;
  const FusedView v = fused_view(f, k, smem);
  long long t[8];
  if (tid < NP) {
    for (int pass = 0; pass < 2; ++pass) {
      fused_bar(NP);
      t[4 * pass + 0] = clock64();
      fused_stage(f, k, v, tid, NP);
      fused_bar(NP);
      t[4 * pass + 1] = clock64();
      fused_keys(f, k, v, tid, NP, nullptr);
      fused_bar(NP);
      t[4 * pass + 2] = clock64();
      fused_ranks(k, v, tid, NP);
      fused_bar(NP);
      t[4 * pass + 3] = clock64();
    }
    if (tid == 0)
      for (int i = 0; i < 8; ++i) out[8 * blockIdx.x + i] = t[i];
    if (tid < v.ncell && blockIdx.x == 0) out[8 * gridDim.x + tid] = v.rk[tid];
  }
}


int main() {
  const int B = 256, k = 8, G = 148;
  std::vector<double> h(B * k);
  unsigned s = 12345;
  for (auto& x : h) {
    s = s * 1664525u + 1013904223u;
    x = 0.5 + 0.5 * (s >> 8) / 16777216.0;
  }
  double* conf;
  long long* out;
  int* ctl;
  cudaMalloc(&conf, h.size() * 8);
  cudaMemcpy(conf, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 5000 * 8);
  cudaMalloc(&ctl, 64);
  FusedSel f = {};
  f.conf = conf;
  f.B_sel = B;
  f.C = 1024;
  f.ctl = ctl;
  const size_t smem = 64 * 1024;
  cudaFuncSetAttribute(phases_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) phases_kernel<<<G, 576, smem>>>(f, k, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<long long> o(8 * G);
  cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
  // CTA 0's ranks against a host count (rows 0 and 148): the tie rule (key, index) over all cells
  std::vector<long long> rk(16);
  cudaMemcpy(rk.data(), out + 8 * G, 16 * 8, cudaMemcpyDeviceToHost);
  std::vector<unsigned long long> key(B * k);
  for (int r = 0; r < B; ++r) {
    double cum = 1.0;
    for (int j = 0; j < k; ++j) {
      cum *= h[r * k + j];
      unsigned long long b;
      memcpy(&b, &cum, 8);
      key[r * k + j] = ~(b | 0x8000000000000000ull);
    }
  }
  int bad = 0;
  for (int c = 0; c < 16; ++c) {
    const int r = c < 8 ? 0 : 148, j = c % 8, m = r * k + j;
    long long n = 0;
    for (int o = 0; o < B * k; ++o) n += key[o] < key[m] || (key[o] == key[m] && o < m);
    if (n != rk[c]) ++bad, printf("rank mismatch cell %d: %lld vs %lld\n", c, rk[c], n);
  }
  printf("ranks of CTA 0 %s\n", bad ? "WRONG" : "match the host count");
  const char* nm[3] = {"stage (loads)", "keys", "ranks"};
  for (int pass = 0; pass < 2; ++pass)
    for (int ph = 0; ph < 3; ++ph) {
      double acc = 0;
      for (int g = 0; g < G; ++g) acc += o[8 * g + 4 * pass + ph + 1] - o[8 * g + 4 * pass + ph];
      printf("pass %d %-14s %8.0f cycles (mean over CTAs)\n", pass, nm[ph], acc / G);
    }
  return 0;
}
