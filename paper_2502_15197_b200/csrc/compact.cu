// Stage (4) compaction and the matrix-level cascade verification (sm_100a).
//
// compact: emitted count n_b = accepted[b] + 1 (the bonus / correction token, sim_engine.py:407-409), optionally
// capped by the request's remaining budget (`min(acc + 1, remaining)`, sim_engine.py:469); offsets = exclusive scan;
// tokens = d[b][0..a) ++ [x_b] truncated to n_b.  One CTA of 1024 threads, each a contiguous block of requests.
//
// verify_matrix: apply_verification (sim_engine.py:374-404).  Row b reads its uniforms at the exclusive scan of the
// windows, which reproduces numpy's `rng.random(w_b)` per row in row order (0 draws for w_b = 0, :393-396).
#include "common.cuh"

namespace tetris {

__global__ void __launch_bounds__(1024, 1)
    compact_kernel(const int32_t* __restrict__ accepted, const int32_t* __restrict__ out_tok,
                   const int32_t* __restrict__ d, const int32_t* __restrict__ cap, int B, int k,
                   int32_t* __restrict__ offsets, int32_t* __restrict__ tokens) {
  __shared__ long long s_tmp[33];
  const int tid = threadIdx.x;
  const int R = (B + blockDim.x - 1) / blockDim.x;
  const int r0 = min(B, tid * R), r1 = min(B, r0 + R);
  long long local = 0;
  for (int r = r0; r < r1; ++r) {
    int n = accepted[r] + 1;
    if (cap) n = min(n, max(cap[r], 0));
    local += n;
  }
  long long total;
  long long off = block_excl_scan<long long>(local, s_tmp, total);
  for (int r = r0; r < r1; ++r) {
    const int a = accepted[r];
    int n = a + 1;
    if (cap) n = min(n, max(cap[r], 0));
    offsets[r] = (int32_t)off;
    for (int i = 0; i < n; ++i) tokens[off + i] = i < a ? d[(int64_t)r * k + i] : out_tok[r];
    off += n;
  }
  if (tid == 0) offsets[B] = (int32_t)total;
}

// Baseline policies on the tensor API: one common window for every request, clamped to what the
// request drafted — select_fixed_window (selector.py:179-190) / the simulator's sd policy min(k, depth)
// (sim_engine.py:358-360) and select_dsd's common window clamped the same way (:361-368).  Writes windows and their
// exclusive scan (the uniform / token offsets of the verification).  Same one-CTA layout as compact_kernel.
__global__ void __launch_bounds__(1024, 1)
    uniform_windows_kernel(const int32_t* __restrict__ len, int B, int k, int window, int32_t* __restrict__ windows,
                           int32_t* __restrict__ win_offsets) {
  __shared__ long long s_tmp[33];
  const int tid = threadIdx.x;
  const int R = (B + blockDim.x - 1) / blockDim.x;
  const int r0 = min(B, tid * R), r1 = min(B, r0 + R);
  long long local = 0;
  for (int r = r0; r < r1; ++r) {
    const int L = len ? len[r] : k;
    const int w = window < L ? window : L;
    windows[r] = w < 0 ? 0 : w;
    local += w < 0 ? 0 : w;
  }
  long long total;
  long long off = block_excl_scan<long long>(local, s_tmp, total);
  if (win_offsets) {
    for (int r = r0; r < r1; ++r) {
      win_offsets[r] = (int32_t)off;
      off += windows[r];
    }
    if (tid == 0) win_offsets[B] = (int32_t)total;
  }
}

__global__ void verify_matrix_kernel(const double* __restrict__ alpha, const int32_t* __restrict__ len,
                                     const int32_t* __restrict__ windows, const int32_t* __restrict__ win_off,
                                     const double* __restrict__ u, int B, int k, int32_t* __restrict__ accepted,
                                     uint32_t* status) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= B) return;
  const int L = len ? len[r] : k;
  int w = windows[r];
  uint32_t bad = 0;
  if (w < 0 || w > L) {  // sim_engine.py:389-392
    bad |= TETRIS_ST_BAD_WINDOW;
    w = w < 0 ? 0 : L;
  }
  const int64_t o = win_off[r];
  int count = 0;
  for (int j = 0; j < w; ++j) {
    if (u[o + j] < alpha[(int64_t)r * k + j])
      ++count;
    else
      break;
  }
  accepted[r] = count;
  set_status(status, bad);
}

__global__ void verify_tokens_kernel(const double* __restrict__ ps, const double* __restrict__ pt,
                                     const int32_t* __restrict__ token, const double* __restrict__ u, int R, int V,
                                     int32_t* __restrict__ accepted, uint32_t* status) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int t = token[r];
  const double ur = u[r];
  uint32_t bad = 0;
  if (t < 0 || t >= V) bad |= TETRIS_ST_BAD_TOKEN;         // accept_model.py:305-306
  if (!(ur >= 0.0 && ur < 1.0)) bad |= TETRIS_ST_BAD_UNIFORM;  // accept_model.py:307-308
  int acc = 0;
  if (!(bad & TETRIS_ST_BAD_TOKEN)) {
    const double s = ps[(int64_t)r * V + t], m = pt[(int64_t)r * V + t];
    acc = (s <= m) || (ur < m / s);  // accept_model.py:309-313
  }
  accepted[r] = acc;
  set_status(status, bad);
}

}  // namespace tetris

#include "abi_util.h"

extern "C" int tetris_compact(const int32_t* accepted, const int32_t* out_tok, const int32_t* d, const int32_t* cap,
                              int32_t B, int32_t k, int32_t* offsets, int32_t* tokens, tetris_stream_t stream) {
  using namespace tetris;
  if (B < 0 || k < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "bad shape B=%d k=%d", B, k);
  if (!offsets) return abi::fail(TETRIS_INVALID_ARGUMENT, "offsets is required");
  if (B > 0 && (!accepted || !out_tok || !tokens || (k > 0 && !d)))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  compact_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(accepted, out_tok, d, cap, B, k, offsets, tokens);
  return abi::launch_check();
}

extern "C" int tetris_uniform_windows(const int32_t* len, int32_t B, int32_t k, int32_t window, int32_t* windows,
                                      int32_t* win_offsets, tetris_stream_t stream) {
  using namespace tetris;
  if (B < 0 || k < 0 || window < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "bad shape B=%d k=%d window=%d", B, k, window);
  if (B == 0) {
    if (win_offsets) {
      cudaError_t e = cudaMemsetAsync(win_offsets, 0, sizeof(int32_t), (cudaStream_t)stream);
      if (e != cudaSuccess) return abi::cuda_fail(e);
    }
    return TETRIS_OK;
  }
  if (!windows) return abi::fail(TETRIS_INVALID_ARGUMENT, "windows is required");
  uniform_windows_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(len, B, k, window, windows, win_offsets);
  return abi::launch_check();
}

extern "C" int tetris_verify_matrix_f64(const double* alpha, const int32_t* len, const int32_t* windows,
                                        const int32_t* win_offsets, const double* u, int32_t B, int32_t k,
                                        int32_t* accepted, uint32_t* status, tetris_stream_t stream) {
  using namespace tetris;
  if (B < 0 || k < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "bad shape B=%d k=%d", B, k);
  if (B == 0) return TETRIS_OK;
  if (!alpha || !windows || !win_offsets || !accepted) return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  verify_matrix_kernel<<<(B + 255) / 256, 256, 0, (cudaStream_t)stream>>>(alpha, len, windows, win_offsets, u, B, k,
                                                                          accepted, status);
  return abi::launch_check();
}

extern "C" int tetris_verify_tokens_f64(const double* p_draft, const double* p_target, const int32_t* token,
                                        const double* u, int32_t R, int32_t V, int32_t* accepted, uint32_t* status,
                                        tetris_stream_t stream) {
  using namespace tetris;
  if (R < 0 || V < 1) return abi::fail(TETRIS_INVALID_ARGUMENT, "bad shape R=%d V=%d", R, V);
  if (R == 0) return TETRIS_OK;
  if (!p_draft || !p_target || !token || !u || !accepted) return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  verify_tokens_kernel<<<(R + 255) / 256, 256, 0, (cudaStream_t)stream>>>(p_draft, p_target, token, u, R, V, accepted,
                                                                          status);
  return abi::launch_check();
}
