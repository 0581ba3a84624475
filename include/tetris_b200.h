/*
 * tetris_b200.h — C ABI of the B200-native TETRIS batch speculative-decoding hot path.
 *
 * The reference (arXiv 2502.15197, package `tetris_sched` 0.1.0 under /root/reference/pkg) exposes this path as
 * plain Python module functions; there is no FFI of its own.  Each entry point below names the reference function
 * whose semantics it implements (file:line, paths relative to /root/reference/pkg/src/tetris_sched/).  The Python
 * drop-in adapters in paper_2502_15197_b200/{selector,accept_model,sim_engine}.py bind these symbols through ctypes
 * and keep the reference's names, argument meaning and exceptions.
 *
 * Conventions
 *   - All pointers are DEVICE pointers (or host pointers registered/mapped for device access) owned by the caller;
 *     the library allocates nothing persistent.  Scratch space comes from a caller-provided workspace that must be
 *     zeroed once with tetris_workspace_init() (kernels leave their arrival counters at zero after every call).
 *   - Everything is stream-ordered on the caller's `stream`; no entry point synchronises the host.  The ABI is
 *     reentrant: no mutable globals besides the thread-local last-error string and write-once per-device caches (SM
 *     count, kernel shared-memory attributes), and the NCCL symbol table of the sharded entry points (resolved once).
 *   - Host-checkable argument errors return TETRIS_INVALID_ARGUMENT immediately.  Data-dependent errors found on the
 *     device are OR-ed into the caller's device word `status` (TETRIS_ST_* bits); the host adapter reads it when it
 *     materialises results and raises the reference's exception.
 *   - Layouts are row-major and dense: conf/cum/alpha [B][k] f64, lengths [B] i32, draft tokens d [B][k] i32,
 *     target probabilities p [B][k+1][V] (the extra position is the bonus row), draft probabilities q [B][k][V].
 */
#ifndef TETRIS_B200_H_
#define TETRIS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tetris_stream_t; /* == cudaStream_t */

/* ---- return codes (host) ---------------------------------------------------------------------------------- */
#define TETRIS_OK 0
#define TETRIS_INVALID_ARGUMENT 1   /* -> ValueError (selector.py:145-146, accept_model.py:284-288, :304-308) */
#define TETRIS_DEGENERATE_RESIDUAL 2 /* -> DegenerateResidualError (accept_model.py:28-29, :323-326)           */
#define TETRIS_CUDA_ERROR 3
#define TETRIS_NCCL_ERROR 4         /* NCCL missing or a collective failed (tetris_dist_*)                       */

/* ---- device status bits (OR-ed into *status by kernels) ----------------------------------------------------- */
#define TETRIS_ST_BAD_VALUE 1u     /* alpha / cum NaN or (conf mode) outside [0,1]  (accept_model.py:55-59)       */
#define TETRIS_ST_DEGENERATE 2u    /* residual / bonus row with zero mass           (accept_model.py:323-326)     */
#define TETRIS_ST_BAD_TOKEN 4u     /* draft token outside [0,V)                     (accept_model.py:305-306)     */
#define TETRIS_ST_BAD_UNIFORM 8u   /* uniform outside [0,1)                         (accept_model.py:307-308)     */
#define TETRIS_ST_BAD_WINDOW 16u   /* window deeper than the row                    (sim_engine.py:389-392)       */
#define TETRIS_ST_STREAM_EXHAUSTED 32u /* tetris_sim_step: uniform or target-length stream too short               */

/* ---- the sampling contract ---------------------------------------------------------------------------------
 * Inverse-CDF sampling of a weight row w[0..V) with a uniform u (accept_model.py:364,368 use numpy's
 * Generator.choice = searchsorted(cumsum(p)/cumsum[-1], u, 'right')).  The GPU and the CPU oracle
 * (oracle/tetris_oracle.c) both follow ONE fixed fp64 summation hierarchy, every node a contiguous index range:
 *   lane  = TETRIS_LANE_ELEMS consecutive elements, summed left to right;
 *   seg   = 32 lanes, balanced binary tree (xor-butterfly order);
 *   warp  = TETRIS_WARP_SEGS consecutive segs, summed left to right;
 *   chunk = TETRIS_CHUNK_WARPS consecutive warps, summed left to right;
 *   row   = ceil(V / TETRIS_CHUNK_ELEMS) chunks, summed left to right -> mass.
 * T = u*mass; descend: at a left-to-right node take the first child whose running prefix exceeds T (T -= prefix
 * before it); at a binary node go left iff left > T or right == 0 (else T -= left).  When no child qualifies the
 * descent takes the last child with positive mass and continues with T = +inf (i.e. last positive leaf). */
#define TETRIS_LANE_ELEMS 8
#define TETRIS_SEG_ELEMS (32 * TETRIS_LANE_ELEMS)                   /* 256  */
#define TETRIS_WARP_SEGS 4
#define TETRIS_CHUNK_WARPS 8
#define TETRIS_CHUNK_ELEMS (TETRIS_SEG_ELEMS * TETRIS_WARP_SEGS * TETRIS_CHUNK_WARPS) /* 8192 */

/* ---- the logits contract (bf16 entry points) --------------------------------------------------------------
 * Entry points taking bf16 logits z (raw uint16 bf16 bits) and a caller-supplied fp32 log-sum-exp per row define each
 * probability as the fp32 value prob(z, lse) below (every operation IEEE fp32 round-to-nearest-even, FMA fused), then
 * apply the fp32 contract above to it unchanged (accept test, residual / bonus weights, sampling):
 *   lo = bf16_round_up(lse + TETRIS_EXP_LO);  hi = bf16_round_down(lse + TETRIS_EXP_HI)   (per row; toward +-inf)
 *   z' = min(max(z, lo), hi) on the bf16 values (maxNum / minNum: a NaN logit takes lo)
 *   x = (float)z' + (-lse)                                    (so x lies in [TETRIS_EXP_LO, TETRIS_EXP_HI])
 *   t = fma(x, TETRIS_EXP_L2E, TETRIS_EXP_MAGIC);  j = t + (-TETRIS_EXP_MAGIC);  r = fma(j, -TETRIS_EXP_LN2, x)
 *   e = fma(fma(fma(fma(fma(C5, r, C4), r, C3), r, C2), r, C1), r, C0)
 *   bits(prob) = bits(t) * 2^23 + bits(e)   (uint32 arithmetic, i.e. e * 2^round(x * log2(e)))
 * Relative error against exp(x) <= 1e-6; logits below lse - 86 read as ~exp(-86) (every probability is a positive
 * normal float).  lse must be finite.  The CPU oracle (oracle/tetris_oracle.c, oracle_probs_from_logits_bf16)
 * computes the same bits with C fmaf(). */
#define TETRIS_EXP_LO (-86.0f)
#define TETRIS_EXP_HI 88.0f
#define TETRIS_EXP_L2E 0x1.715476p+0f
#define TETRIS_EXP_LN2 0x1.62e430p-1f
#define TETRIS_EXP_MAGIC 0x1.8p+23f
#define TETRIS_EXP_C0 0x1p+0f
#define TETRIS_EXP_C1 0x1.ffffdep-1f
#define TETRIS_EXP_C2 0x1.fffde6p-2f
#define TETRIS_EXP_C3 0x1.556974p-3f
#define TETRIS_EXP_C4 0x1.571f3cp-5f
#define TETRIS_EXP_C5 0x1.08822ap-7f

#define TETRIS_MAX_K 255        /* depth fits the 8-bit tie-break field of the selection key                  */
#define TETRIS_MAX_SELECT_ROWS 65535

/* ---- workspace ------------------------------------------------------------------------------------------- */
#define TETRIS_OP_SELECT 1
#define TETRIS_OP_VERIFY 2   /* verify_stochastic / verify_greedy / sample_rows / residual                      */
#define TETRIS_OP_ALL 3
size_t tetris_workspace_bytes(int op, int32_t B, int32_t k, int32_t V);
int tetris_workspace_init(void* ws, size_t ws_bytes, tetris_stream_t stream);

const char* tetris_last_error(void);

/* Zero-copy access to host-resident inputs: returns in *dev_ptr the device address of pinned host memory
 * [host_ptr, host_ptr+bytes) (registering it as mapped/portable when it is not pinned yet), so the streaming kernels
 * can read p/q rows straight from host RAM over PCIe/C2C and only the touched rows cross the link. */
int tetris_map_host(void* host_ptr, size_t bytes, void** dev_ptr);
/* Releases a registration tetris_map_host made itself (no-op for memory the caller pinned or never mapped). */
int tetris_unmap_host(void* host_ptr);
int tetris_abi_version(void);
/* Largest B the speculative sampler (tetris_resample_spec_f32) takes on the current device: min(4096, 32 x SMs).
 * tetris_step_stochastic_f32 falls back to the plain sampler above it. */
int tetris_spec_max_requests(void);

/* Diagnostics (tools/dbg_*.py): when dev_buf != NULL the selector writes clock64() stamps of its phases (CTA 0) into
 * dev_buf[0..49] and the persistent kernels per-CTA %globaltimer / clock64() stamps from dev_buf[64] on; dev_buf must
 * hold 64 + 32 x (SM count) int64.  NULL turns them off (the default). */
int tetris_debug_timestamps(void* dev_buf);

/* Stages (1)+(2): prefix products and capacity-constrained greedy selection.
 * Replaces cumulative_products (selector.py:95-110) + select_tetris (selector.py:133-176).
 * vals_are_cum = 0: vals are acceptance rates alpha (AcceptanceMatrix rows, accept_model.py:37-70) and
 *   cum[b][j] = ((alpha[b][0]*alpha[b][1])*...)*alpha[b][j] left to right in fp64 (selector.py:104-108).
 * vals_are_cum = 1: vals are given Candidate.cum scores (selector.py:32-39), used as-is.
 * The selection is the global top-C under key (cum desc, row asc, depth asc) (_HeapItem, selector.py:113-130)
 * over each row's prefix-min envelope, which equals the heap merge exactly.  len may be NULL (all rows = k).
 * Outputs: windows[B]; optional win_offsets[B+1] (exclusive scan of windows), cum_out[B][k] (raw cum; cells
 * past len untouched), stats4 = {extracts, inserts, peak_queue, -1} (PolicyStats, selector.py:85-92; the heapq
 * comparison count is produced only by tetris_heap_stats_f64). */
int tetris_select_f64(const double* vals, const int32_t* len, int32_t B, int32_t k, int64_t C,
                      int32_t vals_are_cum, int32_t* windows, int32_t* win_offsets, double* cum_out,
                      int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream);

/* Exact replay of select_tetris's heapq schedule (selector.py:151-170) to produce PolicyStats including
 * `comparisons` (every _HeapItem.__lt__ call, selector.py:128-130).  Single-thread device kernel; accounting
 * only — not on the hot path.  cum[B][k] raw Candidate.cum values. */
int tetris_heap_stats_f64(const double* cum, const int32_t* len, int32_t B, int32_t k, int64_t C,
                          int64_t* stats4, void* ws, size_t ws_bytes, tetris_stream_t stream);

/* expected_accepted (selector.py:286-306): one fp64 running sum over the selected cells in row order. */
int tetris_expected_accepted_f64(const double* alpha, const int32_t* len, const int32_t* windows, int32_t B,
                                 int32_t k, double* out, uint32_t* status, tetris_stream_t stream);

/* Matrix-level cascade verification, apply_verification (sim_engine.py:374-404).  Row b consumes the uniforms
 * u[win_offsets[b] .. win_offsets[b]+windows[b]) (== numpy rng.random(w_b) per row in row order); accepted[b] is
 * the count before the first u >= alpha. */
int tetris_verify_matrix_f64(const double* alpha, const int32_t* len, const int32_t* windows,
                             const int32_t* win_offsets, const double* u, int32_t B, int32_t k,
                             int32_t* accepted, uint32_t* status, tetris_stream_t stream);

/* Token-level verify_token (accept_model.py:291-313) for R independent (draft row, target row, token, u) tuples:
 * s = p_draft[r][token[r]], m = p_target[r][token[r]]; accepted[r] = (s <= m) || (u[r] < m / s).  Rows are V f64. */
int tetris_verify_tokens_f64(const double* p_draft, const double* p_target, const int32_t* token, const double* u,
                             int32_t R, int32_t V, int32_t* accepted, uint32_t* status, tetris_stream_t stream);

/* Stage (3) stochastic: per request b, positions j < windows[b] are tested with verify_token's rule
 * (accept_model.py:309-313): s=(double)q[b][j][d], m=(double)p[b][j][d]; accept iff s<=m or u<m/s.
 * accepted[b] = first rejection (or windows[b]).  On rejection the emitted token is sampled (sampling contract
 * above, uniform u_res[b]) from max(0, p[b][a]-q[b][a]) (residual_distribution, accept_model.py:316-327);
 * if every selected token is accepted it is sampled from p[b][windows[b]] (bonus; sim_engine.py:407-409).
 * u_acc layout: win_offsets == NULL -> dense u_acc[b*k + j]; else packed u_acc[win_offsets[b] + j].
 * mass_out[b] (nullable) receives the row mass.  out_tok[b] = -1 with TETRIS_ST_DEGENERATE on zero mass. */
int tetris_verify_stochastic_f32(const float* p, const float* q, const int32_t* d, const int32_t* windows,
                                 const int32_t* win_offsets, const double* u_acc, const double* u_res,
                                 int32_t B, int32_t k, int32_t V, int32_t* accepted, int32_t* out_tok,
                                 double* mass_out, uint32_t* status, void* ws, size_t ws_bytes,
                                 tetris_stream_t stream);

/* The whole stochastic step in two launches (the product hot path), also callable as its two halves:
 *   tetris_select_accept_f32 — the selector (select1_kernel, one CTA, for B_sel*k <= 16384; else the grid selector
 *      gselect_kernel in the workspace's scratch; the cluster/DSMEM select_kernel only when no workspace is given)
 *      with its epilogue: prefix products, global top-C windows +
 *      win_offsets + stats, the accept test of every selected position, accepted[b], the row to resample from
 *      (kept in the workspace) and the compaction offsets (n_b = accepted[b]+1, capped by cap[b] when cap != NULL);
 *      with dense uniforms the accept test of every drafted position runs first in a full-grid pre_accept_kernel;
 *   tetris_resample_f32 — persist_stream_kernel (the TMA-pipelined residual / bonus sampler over the rows chosen by
 *      the previous tetris_select_accept_f32 on the same workspace) + finalize_kernel (one warp per request: the
 *      descent, out_tok[b], mass_out and, when tokens != NULL, the compacted stream d[b][0..a_b) ++ [out_tok[b]],
 *      cut at offsets[b+1]).
 * Same results as tetris_select_f64 + tetris_verify_stochastic_f32 + tetris_compact (u_packed selects the
 * uniform layout as win_offsets != NULL does there).  Requires V % 8 == 0 and 16-byte aligned p, q.
 * Request sharding: the selection runs over all B_sel rows of conf/len (every shard's scores, gathered) with the
 * global capacity C and writes windows/win_offsets for all of them; the verification tensors (p, q, d, u_acc, u_res,
 * cap, accepted, out_tok, mass_out, offsets, tokens) cover only this shard's rows [row0, row0 + B). */
int tetris_select_accept_f32(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                             int32_t row0, int32_t B, const float* p, const float* q, const int32_t* d,
                             const double* u_acc, int32_t u_packed, const int32_t* cap, int32_t V, int32_t* windows,
                             int32_t* win_offsets, int32_t* accepted, int32_t* offsets, int32_t* tokens,
                             int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream);
int tetris_resample_f32(const float* p, const float* q, const double* u_res, int32_t B, int32_t k, int32_t V,
                        const int32_t* d, const int32_t* accepted, const int32_t* offsets, int32_t* out_tok, double* mass_out,
                        int32_t* tokens, uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream);
/* tetris_resample_f32 with the speculative start (same results): the rows of requests whose first drafted token is
 * rejected do not depend on the selection, so the kernel finds them itself (verify_token at position 0 with the
 * dense uniforms u_acc[b][0] of the local rows; len: their drafted depths, nullable) and streams them while the
 * preceding tetris_select_accept_f32 is still running; the rest follows the selection.  B <= tetris_spec_max_requests()
 * (larger batches: TETRIS_INVALID_ARGUMENT).  tetris_step_stochastic_f32 uses it for dense uniforms. */
int tetris_resample_spec_f32(const float* p, const float* q, const double* u_res, const double* u_acc,
                             const int32_t* len, int32_t B, int32_t k, int32_t V, const int32_t* d,
                             const int32_t* accepted, const int32_t* offsets, int32_t* out_tok, double* mass_out,
                             int32_t* tokens, uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream);
int tetris_step_stochastic_f32(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                               int32_t row0, int32_t B, const float* p, const float* q, const int32_t* d,
                               const double* u_acc, int32_t u_packed, const double* u_res, const int32_t* cap,
                               int32_t V, int32_t* windows, int32_t* win_offsets, int32_t* accepted, int32_t* out_tok,
                               double* mass_out, int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status,
                               void* ws, size_t ws_bytes, tetris_stream_t stream);

/* The same stochastic step on LOGITS ("fused logits -> probs"): zp [B][k+1][V] and zq [B][k][V] are
 * bf16 logits (raw uint16 bits) with a caller-supplied fp32 log-sum-exp per row, lse_p [B][k+1] and lse_q [B][k]
 * (the LM head's softmax normaliser).  Every probability the step reads is prob(z, lse) of the logits contract above,
 * computed on the fly inside the kernels (the accept-test gathers, the streamed rows, the descent): the results equal
 * tetris_step_stochastic_f32's on p = prob(zp, lse_p), q = prob(zq, lse_q) bit for bit, while the streamed bytes
 * halve.  V % 8 == 0 and 16-byte aligned zp / zq.  Also as its two halves (tetris_select_accept_bf16, then
 * tetris_resample_bf16 with u_acc / len non-NULL for the speculative start, B <= tetris_spec_max_requests()). */
int tetris_step_stochastic_bf16(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                                int32_t row0, int32_t B, const uint16_t* zp, const float* lse_p, const uint16_t* zq,
                                const float* lse_q, const int32_t* d, const double* u_acc, int32_t u_packed,
                                const double* u_res, const int32_t* cap, int32_t V, int32_t* windows,
                                int32_t* win_offsets, int32_t* accepted, int32_t* out_tok, double* mass_out,
                                int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws,
                                size_t ws_bytes, tetris_stream_t stream);
int tetris_select_accept_bf16(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C,
                              int32_t row0, int32_t B, const uint16_t* zp, const float* lse_p, const uint16_t* zq,
                              const float* lse_q, const int32_t* d, const double* u_acc, int32_t u_packed,
                              const int32_t* cap, int32_t V, int32_t* windows, int32_t* win_offsets, int32_t* accepted,
                              int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws,
                              size_t ws_bytes, tetris_stream_t stream);
int tetris_resample_bf16(const uint16_t* zp, const float* lse_p, const uint16_t* zq, const float* lse_q,
                         const double* u_res, const double* u_acc, const int32_t* len, int32_t B, int32_t k, int32_t V,
                         const int32_t* d, const int32_t* accepted, const int32_t* offsets, int32_t* out_tok,
                         double* mass_out, int32_t* tokens, uint32_t* status, void* ws, size_t ws_bytes,
                         tetris_stream_t stream);
/* The logits contract materialised: out[r][v] = prob(z[r][v], lse[r]) for R rows of V (fp32 out). */
int tetris_probs_from_logits_bf16(const uint16_t* z, const float* lse, int64_t R, int32_t V, float* out,
                                  tetris_stream_t stream);

/* Stage (3) greedy: verify_token on one-hot distributions (accept_model.py:309-313): position j is accepted iff
 * d[b][j] == argmax_v p[b][j][v] (first maximal index, NaN ranks highest as in numpy.argmax); the emitted token is
 * the argmax at the first mismatch, or at windows[b] (bonus). */
int tetris_verify_greedy_f32(const float* p, const int32_t* d, const int32_t* windows, int32_t B, int32_t k,
                             int32_t V, int32_t* accepted, int32_t* out_tok, uint32_t* status, void* ws,
                             size_t ws_bytes, tetris_stream_t stream);
/* The same verification with the compaction of tetris_compact fused into its launch (offsets[B+1], tokens; cap
 * nullable): the greedy product path is 2 launches after the selection (row list, persistent argmax stream). */
int tetris_verify_greedy_compact_f32(const float* p, const int32_t* d, const int32_t* windows, const int32_t* cap,
                                     int32_t B, int32_t k, int32_t V, int32_t* accepted, int32_t* out_tok,
                                     int32_t* offsets, int32_t* tokens, uint32_t* status, void* ws, size_t ws_bytes,
                                     tetris_stream_t stream);

/* The stochastic step for HOST-resident p / q (the end-to-end path): p_host [B][k+1][V], q_host [B][k][V] pinned and
 * device-mapped (tetris_map_host), 16-byte aligned, V % 8 == 0.  The selector's accept test gathers its scalars through
 * the mapping; then one gather kernel copies the row each request resamples from (residual: p[b][a_b] and q[b][a_b];
 * bonus: p[b][w_b]) from host memory into the device buffer `staging` (>= 2*B rows of V; request b uses rows 2b, 2b+1)
 * with 16-byte SM loads over the host link (51 GB/s measured, vs 37 GB/s for one DMA copy per row), then the sampler
 * runs on device memory.  No host synchronisation (capturable).  Same results as tetris_step_stochastic_f32 with dense
 * uniforms. */
int tetris_step_stochastic_staged_f32(const double* conf, const int32_t* len, int32_t B, int32_t k, int64_t C,
                                      const float* p_host, const float* q_host, const int32_t* d,
                                      const double* u_acc, const double* u_res, const int32_t* cap, int32_t V,
                                      float* staging, int32_t* windows, int32_t* win_offsets, int32_t* accepted,
                                      int32_t* out_tok, double* mass_out, int32_t* offsets, int32_t* tokens,
                                      int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                      tetris_stream_t stream);

/* tetris_step_stochastic_staged_f32 for HOST-resident LOGITS: zp_host / zq_host bf16 and lse_p_host / lse_q_host f32,
 * all pinned and device-mapped; staging [2B][V] bf16 and lse_staging [2B] f32 on the device.  Same results as
 * tetris_step_stochastic_bf16 on device copies; half the host-link bytes of the fp32 form. */
int tetris_step_stochastic_staged_bf16(const double* conf, const int32_t* len, int32_t B, int32_t k, int64_t C,
                                       const uint16_t* zp_host, const float* lse_p_host, const uint16_t* zq_host,
                                       const float* lse_q_host, const int32_t* d, const double* u_acc,
                                       const double* u_res, const int32_t* cap, int32_t V, uint16_t* staging,
                                       float* lse_staging, int32_t* windows, int32_t* win_offsets, int32_t* accepted,
                                       int32_t* out_tok, double* mass_out, int32_t* offsets, int32_t* tokens,
                                       int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                       tetris_stream_t stream);

/* The greedy step for HOST-resident p ([B][k+1][V], pinned and device-mapped, 16-byte aligned, V % 4 == 0): the
 * selection, then a gather kernel copies each request's verified rows p[b][0 .. windows[b]] from host memory into the
 * same place of the device buffer p_dev ([B][k+1][V]; rows not needed are left untouched), then the greedy
 * verification + compaction on p_dev.  No host synchronisation.  Same results as tetris_step_greedy_f32. */
int tetris_step_greedy_staged_f32(const double* conf, const int32_t* len, int32_t B, int32_t k, int64_t C,
                                  const float* p_host, const int32_t* d, const int32_t* cap, int32_t V, float* p_dev,
                                  int32_t* windows, int32_t* win_offsets, int32_t* accepted, int32_t* out_tok,
                                  int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws,
                                  size_t ws_bytes, tetris_stream_t stream);

/* The greedy step in 2 launches (select1 with the row-list epilogue, then the persistent argmax stream with the
 * verdicts and the compaction; V % 8 == 0 and 16-byte aligned p, else the stage-by-stage fallback): the selection of
 * tetris_select_f64 over all B_sel rows of conf/len (sharded steps: every shard's scores, gathered) with capacity C,
 * then tetris_verify_greedy_compact_f32 over the local rows [row0, row0 + B) (p, d, cap, accepted, out_tok, offsets,
 * tokens are local; windows / win_offsets cover all B_sel rows). */
int tetris_step_greedy_f32(const double* conf, const int32_t* len, int32_t B_sel, int32_t k, int64_t C, int32_t row0,
                           int32_t B, const float* p, const int32_t* d, const int32_t* cap, int32_t V,
                           int32_t* windows, int32_t* win_offsets, int32_t* accepted, int32_t* out_tok,
                           int32_t* offsets, int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws,
                           size_t ws_bytes, tetris_stream_t stream);

/* Row sampler (the building block of the above, exposed for the token-level adapters):
 * for r < R: weights = max(0, p[p_row[r]] - q[q_row[r]]) if q != NULL and q_row[r] >= 0, else max(0, p[p_row[r]]);
 * out_idx[r] = sample(weights, u[r]); mass_out[r] = row mass.  Rows are V elements, row index in units of V. */
int tetris_sample_rows_f64(const double* p, const double* q, const int64_t* p_row, const int64_t* q_row,
                           const double* u, int32_t R, int32_t V, int32_t* out_idx, double* mass_out,
                           uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream);
int tetris_sample_rows_f32(const float* p, const float* q, const int64_t* p_row, const int64_t* q_row,
                           const double* u, int32_t R, int32_t V, int32_t* out_idx, double* mass_out,
                           uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream);

/* residual_distribution (accept_model.py:316-327) for R row pairs: out[r][v] = max(0, pt[r][v]-ps[r][v]) / mass[r]
 * with mass from the contract hierarchy; rows with zero mass set TETRIS_ST_DEGENERATE and are left untouched. */
int tetris_residual_f64(const double* p_draft, const double* p_target, int32_t R, int32_t V, double* out,
                        double* mass_out, uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream);

/* Stage (4) compaction (sim_engine.py:467-471): n_b = accepted[b]+1, capped by cap[b] when cap != NULL;
 * offsets[B+1] = exclusive scan of n_b; tokens[offsets[b] + i] = (d[b][0..accepted[b]) ++ [out_tok[b]])[i]. */
int tetris_compact(const int32_t* accepted, const int32_t* out_tok, const int32_t* d, const int32_t* cap,
                   int32_t B, int32_t k, int32_t* offsets, int32_t* tokens, tetris_stream_t stream);

/* Baseline policies (select_fixed_window, selector.py:179-190; the simulator's sd / dsd windows, sim_engine.py:358-368):
 * windows[b] = min(window, len[b]) (len NULL: k) and, when win_offsets != NULL, their exclusive scan [B+1].  The DSD
 * common window is select_dsd's scalar argmax (selector.py:193-222), computed by the caller. */
int tetris_uniform_windows(const int32_t* len, int32_t B, int32_t k, int32_t window, int32_t* windows,
                           int32_t* win_offsets, tetris_stream_t stream);

/* GPU-resident simulator step (everything run_step, sim_engine.py:454-495, does after the draft phase) for B <= 1024
 * active requests in the reference's row order.  truth[B][K] (K = k + extra) holds the step's truth acceptance rows,
 * truth_len[B] their depths, which must equal min(K, target - served) (sim_engine.py:343).  policy: 0 = tetris
 * (windows[] given, e.g. by tetris_select_f64 on the surrogate), 1 = sd (min(k_base, depth), :358-360), 2 = dsd
 * (select_dsd's common window from *alpha_hat, selector.py:193-222, clamped to each depth, :361-368).  Verification
 * consumes uniforms[counters[0] ..) in row order (apply_verification, :374-404); accepted[], credited[] = min(acc + 1,
 * remaining) (:467-471), *expected = expected_accepted (selector.py:286-306), *alpha_hat updated (:473-478); then
 * refill_batch (:428-451) rewrites ids/target/served/arrival in place (survivors in order, then one replacement per
 * completion with the next length_stream[counters[1] ..] entry and arrival = step + 1), listing the completed requests
 * in done_ids/done_arrival, and next_depths[] = the next step's draft depths.  counters[7] (device):
 * {uniform offset, length offset, next id, step, completions, sent, accepted}. */
int tetris_sim_step(const double* truth, const int32_t* truth_len, int32_t B, int32_t K, int32_t policy,
                    int32_t k_base, int64_t capacity, double dsd_decay, const double* uniforms, int64_t n_uniforms,
                    const int32_t* length_stream, int64_t n_lengths, int32_t* windows, int64_t* ids, int32_t* target,
                    int32_t* served, int32_t* arrival, double* alpha_hat, int64_t* counters, int32_t* accepted,
                    int32_t* credited, double* expected, int64_t* done_ids, int32_t* done_arrival,
                    int32_t* next_depths, uint32_t* status, tetris_stream_t stream);

/* ---- request-sharded steps over NCCL (north_star: "allgather of per-shard candidates + local select")
 * One process per GPU; rank g of W owns requests [g*B_local, (g+1)*B_local).  `nccl_comm` is the caller's ncclComm_t
 * (cast to void*; e.g. torch ProcessGroupNCCL's, or ncclCommInitRank's); the library resolves ncclAllGather /
 * ncclGroupStart / ncclGroupEnd / ncclCommCount / ncclCommUserRank from the libnccl.so.2 already loaded in the process
 * (else dlopen("libnccl.so.2") or $TETRIS_NCCL_LIB) and links no NCCL itself.  The exchange is ONE NCCL group of two
 * all-gathers on `stream`: every rank's conf [B_local][k] f64 and len [B_local] i32 into conf_all [W*B_local][k] /
 * len_all [W*B_local] (caller-owned; len_local == NULL: all rows k, nothing gathered, and every rank must pass NULL).
 * The selection then runs over the gathered W*B_local rows with the GLOBAL capacity C on every rank (identical
 * inputs => identical windows_all [W*B_local] and win_offsets_all [W*B_local+1] on all ranks, equal to the
 * single-device selection); verification, resampling and compaction cover the local rows only: p, q, zp, zq, d,
 * u_acc (dense [B_local][k]), u_res, cap, accepted, out_tok, mass_out, offsets, tokens are the shard's.  The workspace
 * is sized for B = W*B_local.  Capturable in a CUDA graph (NCCL supports stream capture).  The python replacement
 * for the reference's global selection call (selector.py:133-176 over all requests) is paper_2502_15197_b200.dist. */
int tetris_nccl_comm_info(void* nccl_comm, int32_t* rank, int32_t* world);
int tetris_dist_gather_scores(const double* conf_local, const int32_t* len_local, int32_t B_local, int32_t k,
                              void* nccl_comm, double* conf_all, int32_t* len_all, tetris_stream_t stream);
int tetris_dist_select_f64(const double* vals_local, const int32_t* len_local, int32_t B_local, int32_t k, int64_t C,
                           int32_t vals_are_cum, void* nccl_comm, double* vals_all, int32_t* len_all,
                           int32_t* windows_all, int32_t* win_offsets_all, int64_t* stats4, uint32_t* status, void* ws,
                           size_t ws_bytes, tetris_stream_t stream);
int tetris_dist_step_stochastic_f32(const double* conf_local, const int32_t* len_local, int32_t B_local, int32_t k,
                                    int64_t C, const float* p, const float* q, const int32_t* d, const double* u_acc,
                                    const double* u_res, const int32_t* cap, int32_t V, void* nccl_comm,
                                    double* conf_all, int32_t* len_all, int32_t* windows_all, int32_t* win_offsets_all,
                                    int32_t* accepted, int32_t* out_tok, double* mass_out, int32_t* offsets,
                                    int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                    tetris_stream_t stream);
int tetris_dist_step_stochastic_bf16(const double* conf_local, const int32_t* len_local, int32_t B_local, int32_t k,
                                     int64_t C, const uint16_t* zp, const float* lse_p, const uint16_t* zq,
                                     const float* lse_q, const int32_t* d, const double* u_acc, const double* u_res,
                                     const int32_t* cap, int32_t V, void* nccl_comm, double* conf_all, int32_t* len_all,
                                     int32_t* windows_all, int32_t* win_offsets_all, int32_t* accepted,
                                     int32_t* out_tok, double* mass_out, int32_t* offsets, int32_t* tokens,
                                     int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                     tetris_stream_t stream);
int tetris_dist_step_greedy_f32(const double* conf_local, const int32_t* len_local, int32_t B_local, int32_t k,
                                int64_t C, const float* p, const int32_t* d, const int32_t* cap, int32_t V,
                                void* nccl_comm, double* conf_all, int32_t* len_all, int32_t* windows_all,
                                int32_t* win_offsets_all, int32_t* accepted, int32_t* out_tok, int32_t* offsets,
                                int32_t* tokens, int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                tetris_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TETRIS_B200_H_ */
