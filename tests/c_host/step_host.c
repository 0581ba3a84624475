/* A plain C host driving one whole verification step on the GPU through the C ABI (no Python, no torch): device
 * buffers from cudaMalloc, a zeroed workspace, tetris_step_stochastic_f32 then tetris_step_greedy_f32 on the same
 * stream, results copied back and checked for the step's invariants (windows within the capacity and the depths,
 * accepted <= window, emitted = accepted + 1, the compacted stream = the accepted drafted tokens + the emitted one). */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tetris_b200.h"

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);     \
      return 10;                                                                \
    }                                                                           \
  } while (0)

static unsigned long long rng = 88172645463325252ull;
static double urand(void) {  /* xorshift64, [0, 1) */
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return (double)(rng >> 11) * (1.0 / 9007199254740992.0);
}

int main(void) {
  enum { B = 64, K = 6, V = 4096 };
  const long long C = 160;
  float* p = malloc(sizeof(float) * B * (K + 1) * V);
  float* q = malloc(sizeof(float) * B * K * V);
  double conf[B * K], u_acc[B * K], u_res[B];
  int32_t d[B * K], len[B];
  for (int r = 0; r < B * (K + 1); ++r) {  /* target rows: a spike on token (r * 7) % V over a flat floor */
    for (int v = 0; v < V; ++v) p[(size_t)r * V + v] = 0.5f / V;
    p[(size_t)r * V + (r * 7) % V] += 0.5f;
  }
  for (int b = 0; b < B; ++b) {
    len[b] = 1 + b % K;
    for (int j = 0; j < K; ++j) {
      const int r = b * K + j;
      for (int v = 0; v < V; ++v) q[(size_t)r * V + v] = 1.0f / V;
      d[r] = (int)(urand() * V);
      conf[r] = 0.2 + 0.8 * urand();
      u_acc[r] = urand();
    }
    u_res[b] = urand();
  }
  float *dp, *dq;
  double *dconf, *dua, *dur, *dmass;
  int32_t *dd, *dlen, *win, *woff, *acc, *tok, *off, *toks;
  int64_t* stats;
  uint32_t* status;
  CK(cudaMalloc((void**)&dp, sizeof(float) * B * (K + 1) * V));
  CK(cudaMalloc((void**)&dq, sizeof(float) * B * K * V));
  CK(cudaMalloc((void**)&dconf, sizeof conf));
  CK(cudaMalloc((void**)&dua, sizeof u_acc));
  CK(cudaMalloc((void**)&dur, sizeof u_res));
  CK(cudaMalloc((void**)&dmass, sizeof(double) * B));
  CK(cudaMalloc((void**)&dd, sizeof d));
  CK(cudaMalloc((void**)&dlen, sizeof len));
  CK(cudaMalloc((void**)&win, sizeof(int32_t) * B));
  CK(cudaMalloc((void**)&woff, sizeof(int32_t) * (B + 1)));
  CK(cudaMalloc((void**)&acc, sizeof(int32_t) * B));
  CK(cudaMalloc((void**)&tok, sizeof(int32_t) * B));
  CK(cudaMalloc((void**)&off, sizeof(int32_t) * (B + 1)));
  CK(cudaMalloc((void**)&toks, sizeof(int32_t) * B * (K + 1)));
  CK(cudaMalloc((void**)&stats, sizeof(int64_t) * 4));
  CK(cudaMalloc((void**)&status, sizeof(uint32_t)));
  CK(cudaMemcpy(dp, p, sizeof(float) * B * (K + 1) * V, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dq, q, sizeof(float) * B * K * V, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dconf, conf, sizeof conf, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dua, u_acc, sizeof u_acc, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dur, u_res, sizeof u_res, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dd, d, sizeof d, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dlen, len, sizeof len, cudaMemcpyHostToDevice));
  CK(cudaMemset(status, 0, sizeof(uint32_t)));
  const size_t wsb = tetris_workspace_bytes(TETRIS_OP_ALL, B, K, V);
  void* ws;
  CK(cudaMalloc(&ws, wsb));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  if (tetris_workspace_init(ws, wsb, (tetris_stream_t)st)) return 11;
  for (int mode = 0; mode < 2; ++mode) {
    int rc = mode == 0 ? tetris_step_stochastic_f32(dconf, dlen, B, K, C, 0, B, dp, dq, dd, dua, 0, dur, NULL, V, win,
                                                    woff, acc, tok, dmass, off, toks, stats, status, ws, wsb,
                                                    (tetris_stream_t)st)
                       : tetris_step_greedy_f32(dconf, dlen, B, K, C, 0, B, dp, dd, NULL, V, win, woff, acc, tok, off,
                                                toks, stats, status, ws, wsb, (tetris_stream_t)st);
    if (rc) {
      fprintf(stderr, "step %d: %s\n", mode, tetris_last_error());
      return 12;
    }
    CK(cudaStreamSynchronize(st));
    int32_t hw[B], ha[B], ht[B], ho[B + 1], hk[B * (K + 1)];
    uint32_t hs;
    CK(cudaMemcpy(hw, win, sizeof hw, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ha, acc, sizeof ha, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ht, tok, sizeof ht, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ho, off, sizeof ho, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hk, toks, sizeof hk, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&hs, status, sizeof hs, cudaMemcpyDeviceToHost));
    if (hs) return 13;
    long long sel = 0;
    for (int b = 0; b < B; ++b) {
      sel += hw[b];
      if (hw[b] < 0 || hw[b] > len[b] || ha[b] < 0 || ha[b] > hw[b] || ht[b] < 0 || ht[b] >= V) return 14;
      if (ho[b + 1] - ho[b] != ha[b] + 1) return 15;
      for (int j = 0; j < ha[b]; ++j)
        if (hk[ho[b] + j] != d[b * K + j]) return 16;
      if (hk[ho[b] + ha[b]] != ht[b]) return 17;
      if (mode == 1 && ha[b] < hw[b] && ht[b] != ((b * (K + 1) + ha[b]) * 7) % V) return 18; /* greedy: the argmax */
    }
    if (sel != C) return 19; /* C < total drafted cells: exactly C selected */
  }
  printf("ok\n");
  return 0;
}
