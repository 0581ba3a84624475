// Launch-level declarations shared by the kernel translation units (host + device visible).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tetris {

struct SelectArgs {
  const double* vals;
  const int32_t* len;
  int B, k;
  long long C;
  int vals_are_cum;
  int32_t* windows;
  int32_t* win_offsets;
  double* cum_out;
  long long* stats;
  uint32_t* status;
  int RB;  // rows per CTA
  // fused accept + compaction epilogue (p == nullptr: off) for the local rows [ep_row0, ep_row0 + ep_rows); the
  // per-request tensors below are indexed by local row (global row - ep_row0)
  int ep_row0, ep_rows;
  const float* p;
  const float* q;
  const uint16_t* zp;   // logits form (nullptr: fp32 probabilities p / q): bf16 logits + per-row lse
  const uint16_t* zq;
  const float* lse_p;
  const float* lse_q;
  const int32_t* d;
  const double* u_acc;
  int u_packed;
  int V;
  const int32_t* cap;
  int32_t* accepted;
  long long* rowinfo;  // [B][2]: p row, q row (-1: bonus)
  float* rowlse;       // logits form: [B][2] the lse of those rows (written beside rowinfo)
  int32_t* offsets;    // [B+1]
  uint8_t* acc_bytes;  // pre-accept verdicts [ep_rows][k] (nullptr: gather in the epilogue)
  int accept_ctas;     // > 0: CTAs after cluster 0 compute acc_bytes concurrently with the selection
  int accept_spread;   // select1: spread the accept CTAs over every SM (inputs in mapped host memory, see select1.cu)
  int* acc_counter;    // arrivals of those CTAs (zero between launches)
  long long* dbg;      // diagnostics: per-phase clock64() stamps of CTA 0 (nullptr: off)
  void* gscratch;      // workspace region WS_GSEL (grid selector), zero-initialised
  // greedy epilogue (select1 only; rowmap == nullptr: off): the row list of greedy verification over the local rows
  // [ep_row0, ep_row0 + ep_rows) and their zeroed argmax keys (greedy.cu, rowmap_write_warp)
  int32_t* rowmap;
  unsigned long long* gkeys;
};

void set_debug_buffer(long long* p);
long long* debug_buffer();

// The selection fused into the sampler's launch (persist_stream_kernel<.., FUSED>, small batches: B_sel * k <=
// kFusedMaxCells): every CTA computes the keys of all B_sel rows, the exact rank of the cells of its own rows
// (g, g + G, ...) and from them the rows' windows, accept verdicts and row choice; the last CTA to publish writes
// the offset scans and the PolicyStats.  conf == nullptr: off.
struct FusedSel {
  const double* conf;   // [B_sel][k]
  const int32_t* len;   // [B_sel] nullable (k)
  const double* u_acc;  // [R][k] dense accept uniforms
  int B_sel, row0;      // selected rows; local rows [row0, row0 + R)
  long long C;
  int32_t* windows;     // [B_sel]
  int32_t* win_offsets; // [B_sel + 1]
  long long* stats;     // [4] nullable
  const int32_t* cap;   // [R] nullable
  int32_t* accepted;    // [R]
  long long* rowinfo;   // [R][2]
  float* rowlse;        // [R][2] logits form
  int32_t* offsets;     // [R + 1]
  int* ctl;             // [3] CTAs counted in, scans done (zero, left at zero), the last launch's epoch
  unsigned long long* ready;  // [R] per-request ready words (fused_ready_word), self-resetting by epoch
};
constexpr int kFusedMaxCells = 2048;

struct StreamArgs {
  const float* p;
  const float* q;
  const uint16_t* zp;  // logits form (the bf16 kernels): bf16 logits rows + per-row lse; p / q unused
  const uint16_t* zq;
  const float* lse_p;
  const float* lse_q;
  int V, nch, R;
  const long long* prow;     // p row of request b at prow[b * row_stride]
  const long long* qrow;     // q row (-1: plain / bonus row) at qrow[b * row_stride]; nullptr: all plain
  const float* rowlse;       // logits form: [R][2] the lse of request b's p row / q row (beside the row info)
  float* spec_lse;           // logits form, speculative variant: [R][2] the lse of phase-A list entry y's rows
  int row_stride;
  const double* u;           // [R]
  int32_t* out_idx;
  double* mass_out;
  uint32_t* status;
  int* counters;
  double* chunk_sums;
  double* warp_sums;
  // fused compaction (accepted == nullptr: off): tokens[offsets[b] ..) = d[b][0..a_b) ++ [sample], cut at the cap
  const int32_t* accepted;
  const int32_t* offsets;
  int32_t* tokens;
  const int32_t* d;
  int k;
  unsigned* grid_bar;  // [0]: CTAs done, [2..3]: 64-bit work counter (zero-initialised workspace, left at zero)
  int* req_cnt;        // [R] per-request published-chunk counters (zero, left at zero): the descent runs in the same
                       // launch as each request completes; nullptr -> a separate finalize_kernel launch
  long long* dbg;      // diagnostics: per-CTA %globaltimer stamps at dbg[64 + 8 * cta + slot] (nullptr: off)
  // speculative variant (u_acc != nullptr; R <= spec_max_requests()): the requests whose first drafted token is
  // rejected are streamed before the selection completes (stream.cu); dense u_acc[R][k], len[R] (nullable: k)
  const double* u_acc;
  const int32_t* len;
  int* req_cnt_spec;         // [R] their completion counters (zero, left at zero)
  double* chunk_sums_spec;   // [R][nch] and [R][nch][8]: their sums
  double* warp_sums_spec;
  int* spec_ctl;             // [2]: phase-A list length, requests processed (zero, left at zero)
  uint32_t* spec_bitmap;     // [ceil(R / 32)]: the phase-A set (zero, left at zero)
  int* spec_list;            // [R]: the phase-A list, entry b + 1 (zero, left at zero)
  FusedSel fs;               // fused selection (fs.conf != nullptr; not with the speculative variant)
};
bool fused_step_eligible(int B_sel, int k, int u_packed);
int spec_max_requests();

// Greedy verification (greedy.cu): the persistent argmax stream over the rows listed by greedy_rowmap_kernel.
struct GreedyArgs {
  const float* p;             // [B][k+1][V]
  const int32_t* d;           // [B][k]
  const int32_t* windows;     // [B]
  const int32_t* cap;         // [B] nullable: emitted-token cap of the fused compaction
  int B, k, V, nch;
  const int32_t* rowmap;      // [0]: listed-row count, then b << 8 | j
  unsigned long long* keys;   // [B][k+1] argmax keys of the listed rows (zeroed by the row-map kernel)
  unsigned long long* key0;   // [B] argmax keys of row 0 (streamed before the selection; zero, left at zero)
  unsigned* grid_bar2;        // [0..1]: 64-bit counter of the row-0 items (zero, left at zero)
  long long* dbg;             // diagnostics: per-CTA %globaltimer stamps at dbg[64 + 8 * cta + slot] (nullptr: off)
  int* req_cnt;               // [B] per-request published-chunk counters (zero, left at zero)
  unsigned* grid_bar;         // [0]: CTAs done, [2..3]: 64-bit work counter (zero, left at zero)
  int32_t* accepted;
  int32_t* out_tok;
  int32_t* offsets;           // [B+1] nullable: fused compaction off
  int32_t* tokens;
  uint32_t* status;
  FusedSel fs;                // one-launch step (fs.conf != nullptr): the selection as the kernel's prologue
};

int launch_select(const SelectArgs& a, cudaStream_t st);
bool select1_eligible(int B, int k);
int launch_select1(const SelectArgs& a, cudaStream_t st);  // single-CTA selector (select1.cu)
int launch_gselect(const SelectArgs& a, void* scratch, cudaStream_t st);  // grid-wide selector (gselect.cu)
size_t gselect_scratch_bytes();
int launch_persist_stream(const StreamArgs& a, cudaStream_t st);
bool persist_eligible(const float* p, const float* q, int V);
bool persist_greedy_eligible(const float* p, int V);
bool greedy_fused_fits(int B_sel, int k);
int launch_greedy_rowmap(const int32_t* windows, int B, int k, int32_t* rowmap, unsigned long long* keys, int j0,
                         cudaStream_t st);
int launch_persist_greedy(const GreedyArgs& a, cudaStream_t st);
int launch_pre_accept(const SelectArgs& a, cudaStream_t st);
int launch_accept(const float* p, const float* q, const int32_t* d, const int32_t* windows, const int32_t* win_off,
                  const double* u_acc, int B, int k, int V, int32_t* accepted, long long* rowinfo, uint32_t* status,
                  cudaStream_t st);

}  // namespace tetris
