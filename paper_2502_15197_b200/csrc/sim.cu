// GPU-resident simulator step: everything run_step (sim_engine.py:454-495) does after the draft
// phase, on device, for one batch of up to 1024 active requests — the baseline policies' windows (sd: min(k, depth),
// sim_engine.py:358-360; dsd: select_dsd's common window, selector.py:193-222, clamped to each depth, :361-368; tetris
// windows come from the selection kernel), apply_verification's cascade over the flat uniform stream
// (sim_engine.py:374-404), expected_accepted (selector.py:286-306), the credit min(acc + 1, remaining) (:467-471),
// the DSD estimate update (:473-478) and refill_batch (:428-451: survivors keep their order, replacements are
// appended with the next target lengths of the stream and arrival = step + 1), plus the next step's draft depths
// min(k + extra, remaining) (:343).  Single CTA, one request per thread; all cross-request order (uniform offsets,
// the running expected sum, the refill order) follows the reference's row order exactly.
#include "abi_util.h"
#include "common.cuh"

namespace tetris {

constexpr int kSimThreads = 1024;

// counters[]: 0 uniform offset, 1 length-stream offset, 2 next request id, 3 step, 4 completions of this step,
// 5 tokens sent this step, 6 tokens accepted this step
struct SimArgs {
  const double* truth;
  const int32_t* truth_len;
  int B, K, policy, k_base;
  long long capacity;
  double dsd_decay;
  const double* uniforms;
  long long n_uniforms;
  const int32_t* lengths;
  long long n_lengths;
  int32_t* windows;
  long long* ids;
  int32_t* target;
  int32_t* served;
  int32_t* arrival;
  double* alpha_hat;
  long long* counters;
  int32_t* accepted;
  int32_t* credited;
  double* expected;
  long long* done_ids;
  int32_t* done_arrival;
  int32_t* next_depths;
  uint32_t* status;
};

// select_dsd (selector.py:193-222): the window k in [1, k_max] maximising sum_{j<=k} alpha^j, first maximum wins;
// 0 when not even one token per row fits.  Same running products and sums as the reference, in fp64.
__device__ int dsd_window(double alpha, int n_rows, long long capacity, int depth_limit) {
  const long long per_row = capacity / n_rows;
  const int k_max = (int)(depth_limit < per_row ? depth_limit : per_row);
  if (k_max < 1) return 0;
  int best_k = 1;
  double best = alpha, value = alpha, power = alpha;
  for (int k = 2; k <= k_max; ++k) {
    power = __dmul_rn(power, alpha);
    value = __dadd_rn(value, power);
    if (value > best) {
      best = value;
      best_k = k;
    }
  }
  return best_k;
}

__global__ void __launch_bounds__(kSimThreads, 1) sim_step_kernel(const SimArgs a) {
  __shared__ long long tmp[33];
  __shared__ int s_common;
  const int t = threadIdx.x, B = a.B, K = a.K;
  const bool row = t < B;
  uint32_t bad = 0;
  const long long u_off = a.counters[0], len_off = a.counters[1], next_id = a.counters[2], step = a.counters[3];
  if (t == 0 && a.policy == 2) s_common = dsd_window(*a.alpha_hat, B, a.capacity, K);
  __syncthreads();

  // ---- windows of the baseline policies ------------------------------------------------------------------------
  int L = 0, w = 0, tgt = 0, srv = 0;
  if (row) {
    L = a.truth_len[t];
    tgt = a.target[t];
    srv = a.served[t];
    const int rem = tgt - srv;
    if (L != (K < rem ? K : rem) || L < 0) bad |= TETRIS_ST_BAD_WINDOW;  // depth must be min(k + extra, remaining)
    if (a.policy == 1)
      w = a.k_base < L ? a.k_base : L;
    else if (a.policy == 2)
      w = s_common < L ? s_common : L;
    else
      w = a.windows[t];
    if (w < 0 || w > L) {
      bad |= TETRIS_ST_BAD_WINDOW;
      w = w < 0 ? 0 : L;
    }
    if (a.policy != 0) a.windows[t] = w;
  }

  // ---- apply_verification: row t reads uniforms [u_off + excl(w), + w) ------------------------------------------
  long long sent;
  const long long wex = block_excl_scan<long long>(row ? w : 0, tmp, sent);
  int acc = 0;
  if (row) {
    if (u_off + wex + w > a.n_uniforms) {
      bad |= TETRIS_ST_STREAM_EXHAUSTED;
    } else {
      const double* u = a.uniforms + u_off + wex;
      const double* al = a.truth + (int64_t)t * K;
      while (acc < w && u[acc] < al[acc]) ++acc;  // sim_engine.py:397-401
    }
    a.accepted[t] = acc;
  }
  long long acc_sum;
  block_excl_scan<long long>(row ? acc : 0, tmp, acc_sum);

  // ---- credit (sim_engine.py:467-471) and completion ----------------------------------------------------------
  int cred = 0;
  bool done = false;
  if (row) {
    const int rem = tgt - srv;
    cred = acc + 1 < rem ? acc + 1 : rem;
    srv += cred;
    a.credited[t] = cred;
    done = tgt - srv <= 0;
  }
  long long n_done;
  const long long drank = block_excl_scan<long long>(done ? 1 : 0, tmp, n_done);
  // ---- expected_accepted: one running fp64 sum over the selected cells in row order (selector.py:302-305) -------
  if (t == 0) {
    double value = 0.0;
    for (int r = 0; r < B; ++r) {
      const int wr = a.windows[r];
      const double* al = a.truth + (int64_t)r * K;
      double cum = 1.0;
      for (int j = 0; j < wr; ++j) {
        cum = __dmul_rn(cum, al[j]);
        value = __dadd_rn(value, cum);
      }
    }
    *a.expected = value;
    // DSD estimate (sim_engine.py:473-478)
    if (sent > 0) {
      const double rate = (double)acc_sum / (double)sent;
      *a.alpha_hat = __dadd_rn(__dmul_rn(a.dsd_decay, *a.alpha_hat), __dmul_rn(__dadd_rn(1.0, -a.dsd_decay), rate));
    }
  }
  if (n_done > 0 && len_off + n_done > a.n_lengths) bad |= (t == 0) ? TETRIS_ST_STREAM_EXHAUSTED : 0u;
  // ---- refill_batch (sim_engine.py:428-451): survivors in order, then one replacement per completion ----------
  long long my_id = 0;
  int my_arr = 0;
  if (row) {
    my_id = a.ids[t];
    my_arr = a.arrival[t];
  }
  __syncthreads();  // every row's state is in registers before the compaction overwrites it
  if (row) {
    if (done) {
      a.done_ids[drank] = my_id;
      a.done_arrival[drank] = my_arr;
      const int slot = (int)(B - n_done + drank);
      const long long li = len_off + drank;
      const int nt = li < a.n_lengths ? a.lengths[li] : 1;
      a.ids[slot] = next_id + drank;
      a.target[slot] = nt;
      a.served[slot] = 0;
      a.arrival[slot] = (int)(step + 1);
      a.next_depths[slot] = K < nt ? K : nt;
    } else {
      const int slot = (int)(t - drank);
      a.ids[slot] = my_id;
      a.target[slot] = tgt;
      a.served[slot] = srv;
      a.arrival[slot] = my_arr;
      const int rem = tgt - srv;
      a.next_depths[slot] = K < rem ? K : rem;
    }
  }
  if (t == 0) {
    a.counters[0] = u_off + sent;
    a.counters[1] = len_off + n_done;
    a.counters[2] = next_id + n_done;
    a.counters[3] = step + 1;
    a.counters[4] = n_done;
    a.counters[5] = sent;
    a.counters[6] = acc_sum;
  }
  set_status(a.status, bad);
}

}  // namespace tetris

extern "C" int tetris_sim_step(const double* truth, const int32_t* truth_len, int32_t B, int32_t K, int32_t policy,
                               int32_t k_base, int64_t capacity, double dsd_decay, const double* uniforms,
                               int64_t n_uniforms, const int32_t* length_stream, int64_t n_lengths, int32_t* windows,
                               int64_t* ids, int32_t* target, int32_t* served, int32_t* arrival, double* alpha_hat,
                               int64_t* counters, int32_t* accepted, int32_t* credited, double* expected,
                               int64_t* done_ids, int32_t* done_arrival, int32_t* next_depths, uint32_t* status,
                               tetris_stream_t stream) {
  using namespace tetris;
  if (B < 1 || B > kSimThreads) return abi::fail(TETRIS_INVALID_ARGUMENT, "B=%d outside [1, %d]", B, kSimThreads);
  if (K < 1 || K > TETRIS_MAX_K) return abi::fail(TETRIS_INVALID_ARGUMENT, "K=%d outside [1, %d]", K, TETRIS_MAX_K);
  if (policy < 0 || policy > 2) return abi::fail(TETRIS_INVALID_ARGUMENT, "unknown policy %d", policy);
  if (capacity < 0) return abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0");
  if (!truth || !truth_len || !uniforms || !length_stream || !windows || !ids || !target || !served || !arrival ||
      !alpha_hat || !counters || !accepted || !credited || !expected || !done_ids || !done_arrival || !next_depths)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "null argument");
  SimArgs a = {truth,   truth_len, B,        K,      policy,   k_base,   (long long)capacity,     dsd_decay,
               uniforms, (long long)n_uniforms, length_stream, (long long)n_lengths, windows, (long long*)ids,
               target,   served,    arrival,  alpha_hat, (long long*)counters, accepted, credited, expected,
               (long long*)done_ids, done_arrival, next_depths, status};
  sim_step_kernel<<<1, kSimThreads, 0, (cudaStream_t)stream>>>(a);
  return abi::launch_check();
}
