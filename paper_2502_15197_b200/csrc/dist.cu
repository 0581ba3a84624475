// Request-sharded multi-GPU steps as native entry points: the one exchange the global capacity
// budget needs, then the single-device step over the gathered scores.
//
// Rank g of W owns requests [g*B_local, (g+1)*B_local).  The only data every rank needs from the others is their
// candidate scores: conf [B_local][k] f64 and the drafted depths len [B_local] i32 (B_local*(8k+4) bytes per rank,
// 2.1 MB at cfg5 = 16384 x 16).  They go out as ONE NCCL group of two all-gathers on the caller's stream (one
// launch; NVLink / NVSwitch, NVLS when NCCL picks it), into the caller's [W*B_local] buffers in rank order, so the
// gathered row index IS the global row id and the reference's (cum desc, row asc, depth asc) tie-break
// (selector.py:113-130) holds across shards.  Every rank then runs the identical selection kernel over bit-identical
// inputs, so the windows equal the single-GPU selection (and the CPU reference's) for any W by construction, and the
// verification / resampling / compaction that follow touch only the local rows (no further exchange).
//
// Why gather the scores and not per-shard top-m candidates: a candidate key is 16 bytes (score + global row/depth),
// a score 8 bytes; at cfg5 a shard's top-m (m = min(C, B_local*k)) is every one of its cells for W >= 2, so the
// score gather is the smaller message.  A threshold all-reduce (radix histograms, one round per 8-bit digit) would
// cut the per-rank selection work to the local rows but costs 6-8 dependent NCCL latencies (~10 us each on NVLink)
// against one all-gather plus a ~20 us replicated selection that the speculative sampler already overlaps.
//
// NCCL binding: the library does not link NCCL.  The communicator comes from the caller (ncclComm_t as void*), and
// the NCCL functions used (ncclAllGather, ncclGroupStart / End, ncclCommCount, ncclCommUserRank, and
// ncclCommGetAsyncError for non-blocking communicators) are resolved at first use from the libnccl.so.2 ALREADY LOADED in the process (the
// one that created the communicator: torch's bundled NCCL under Python, the host's own otherwise), falling back to
// dlopen("libnccl.so.2") -- or $TETRIS_NCCL_LIB when set.  Using a communicator with a different NCCL build than
// the one that created it is undefined, hence RTLD_NOLOAD first.
#include <dlfcn.h>
#include <stdlib.h>

#include <mutex>

#include "abi_util.h"

namespace tetris {
namespace nccl {

// NCCL C API subset (nccl.h; stable since 2.0): enums as int, the communicator as an opaque pointer
typedef int (*AllGatherFn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*GroupFn)(void);
typedef int (*CommIntFn)(const void*, int*);
typedef const char* (*ErrStrFn)(int);
typedef int (*AsyncErrFn)(void*, int*);
constexpr int kInt8 = 0;        // ncclInt8
constexpr int kInProgress = 7;  // ncclInProgress: a non-blocking communicator is still working on the call

struct Api {
  AllGatherFn all_gather = nullptr;
  GroupFn group_start = nullptr, group_end = nullptr;
  CommIntFn comm_count = nullptr, comm_rank = nullptr;
  ErrStrFn err_str = nullptr;
  AsyncErrFn async_err = nullptr;
  char why[256] = {0};
  bool ok = false;
};

static const Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("TETRIS_NCCL_LIB");
    void* h = nullptr;
    if (env && *env) {
      h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    } else {
      h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (the communicator's creator)
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      snprintf(a.why, sizeof a.why, "cannot load NCCL (%s): %s", env && *env ? env : "libnccl.so.2", dlerror());
      return;
    }
    a.all_gather = (AllGatherFn)dlsym(h, "ncclAllGather");
    a.group_start = (GroupFn)dlsym(h, "ncclGroupStart");
    a.group_end = (GroupFn)dlsym(h, "ncclGroupEnd");
    a.comm_count = (CommIntFn)dlsym(h, "ncclCommCount");
    a.comm_rank = (CommIntFn)dlsym(h, "ncclCommUserRank");
    a.err_str = (ErrStrFn)dlsym(h, "ncclGetErrorString");
    a.async_err = (AsyncErrFn)dlsym(h, "ncclCommGetAsyncError");
    a.ok = a.all_gather && a.group_start && a.group_end && a.comm_count && a.comm_rank;
    if (!a.ok) snprintf(a.why, sizeof a.why, "libnccl.so.2 lacks the NCCL collective API");
  });
  return a;
}

static int nccl_fail(const Api& a, int r, const char* what) {
  return abi::fail(TETRIS_NCCL_ERROR, "NCCL %s failed: %s (%d)", what, a.err_str ? a.err_str(r) : "?", r);
}

// A communicator created non-blocking (ncclConfig_t.blocking = 0) may answer ncclInProgress: wait for the call's
// completion the way NCCL prescribes (poll ncclCommGetAsyncError), then report its final state.
static int settle(const Api& a, void* comm, int r) {
  if (r != kInProgress || !a.async_err) return r;
  int st = kInProgress;
  do {
    if (a.async_err(comm, &st) != 0) return st == 0 ? kInProgress : st;
  } while (st == kInProgress);
  return st;
}

// rank / world of the communicator
static int comm_info(void* comm, int* rank, int* world) {
  const Api& a = api();
  if (!a.ok) return abi::fail(TETRIS_NCCL_ERROR, "%s", a.why);
  if (!comm) return abi::fail(TETRIS_INVALID_ARGUMENT, "null NCCL communicator");
  int r;
  if ((r = settle(a, comm, a.comm_count(comm, world))) != 0) return nccl_fail(a, r, "ncclCommCount");
  if ((r = settle(a, comm, a.comm_rank(comm, rank))) != 0) return nccl_fail(a, r, "ncclCommUserRank");
  return TETRIS_OK;
}

// The exchange: conf (and len when non-NULL) of every rank into the gathered buffers, one NCCL group.
static int gather_scores(const double* conf, const int32_t* len, int B_local, int k, void* comm, double* conf_all,
                         int32_t* len_all, cudaStream_t st) {
  const Api& a = api();
  if (!a.ok) return abi::fail(TETRIS_NCCL_ERROR, "%s", a.why);
  const size_t cb = (size_t)B_local * k * sizeof(double), lb = (size_t)B_local * sizeof(int32_t);
  int r;
  if ((r = a.group_start()) != 0) return nccl_fail(a, r, "ncclGroupStart");
  int r1 = cb ? a.all_gather(conf, conf_all, cb, kInt8, comm, st) : 0;
  int r2 = len ? a.all_gather(len, len_all, lb, kInt8, comm, st) : 0;
  if ((r = settle(a, comm, a.group_end())) != 0) return nccl_fail(a, r, "ncclGroupEnd");
  if (r1 && r1 != kInProgress) return nccl_fail(a, r1, "ncclAllGather(conf)");
  if (r2 && r2 != kInProgress) return nccl_fail(a, r2, "ncclAllGather(len)");
  return TETRIS_OK;
}

// Shared argument checks + the exchange; *row0 / *B_sel describe the gathered selection for the local step.
static int prologue(const double* conf, const int32_t* len, int32_t B_local, int32_t k, void* comm, double* conf_all,
                    int32_t* len_all, cudaStream_t st, int32_t* row0, int32_t* B_sel) {
  if (B_local <= 0 || k < 0 || k > TETRIS_MAX_K)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "bad shard shape B_local=%d k=%d", B_local, k);
  if ((k > 0 && (!conf || !conf_all)) || (len && !len_all))
    return abi::fail(TETRIS_INVALID_ARGUMENT, "conf / conf_all (and len_all when len is given) are required");
  int rank = 0, world = 0;
  int rc = comm_info(comm, &rank, &world);
  if (rc) return rc;
  if ((long long)B_local * world > TETRIS_MAX_SELECT_ROWS)
    return abi::fail(TETRIS_INVALID_ARGUMENT, "W*B_local=%lld exceeds %d selected rows", (long long)B_local * world,
                     TETRIS_MAX_SELECT_ROWS);
  if ((rc = gather_scores(conf, len, B_local, k, comm, conf_all, len_all, st))) return rc;
  *row0 = rank * B_local;
  *B_sel = world * B_local;
  return TETRIS_OK;
}

}  // namespace nccl
}  // namespace tetris

using tetris::nccl::prologue;

extern "C" int tetris_nccl_comm_info(void* comm, int32_t* rank, int32_t* world) {
  if (!rank || !world) return tetris::abi::fail(TETRIS_INVALID_ARGUMENT, "null rank / world");
  int r = 0, w = 0;
  int rc = tetris::nccl::comm_info(comm, &r, &w);
  if (rc) return rc;
  *rank = r;
  *world = w;
  return TETRIS_OK;
}

extern "C" int tetris_dist_gather_scores(const double* conf_local, const int32_t* len_local, int32_t B_local,
                                         int32_t k, void* nccl_comm, double* conf_all, int32_t* len_all,
                                         tetris_stream_t stream) {
  int32_t row0, B_sel;
  return prologue(conf_local, len_local, B_local, k, nccl_comm, conf_all, len_all, (cudaStream_t)stream, &row0,
                  &B_sel);
}

extern "C" int tetris_dist_select_f64(const double* vals_local, const int32_t* len_local, int32_t B_local, int32_t k,
                                      int64_t C, int32_t vals_are_cum, void* nccl_comm, double* vals_all,
                                      int32_t* len_all, int32_t* windows_all, int32_t* win_offsets_all,
                                      int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                      tetris_stream_t stream) {
  if (C < 0) return tetris::abi::fail(TETRIS_INVALID_ARGUMENT, "capacity must be >= 0, got %lld", (long long)C);
  int32_t row0, B_sel;
  int rc = prologue(vals_local, len_local, B_local, k, nccl_comm, vals_all, len_all, (cudaStream_t)stream, &row0,
                    &B_sel);
  if (rc) return rc;
  return tetris_select_f64(vals_all, len_local ? len_all : nullptr, B_sel, k, C, vals_are_cum, windows_all,
                           win_offsets_all, nullptr, stats4, status, ws, ws_bytes, stream);
}

extern "C" int tetris_dist_step_stochastic_f32(const double* conf_local, const int32_t* len_local, int32_t B_local,
                                               int32_t k, int64_t C, const float* p, const float* q, const int32_t* d,
                                               const double* u_acc, const double* u_res, const int32_t* cap,
                                               int32_t V, void* nccl_comm, double* conf_all, int32_t* len_all,
                                               int32_t* windows_all, int32_t* win_offsets_all, int32_t* accepted,
                                               int32_t* out_tok, double* mass_out, int32_t* offsets, int32_t* tokens,
                                               int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                               tetris_stream_t stream) {
  int32_t row0, B_sel;
  int rc = prologue(conf_local, len_local, B_local, k, nccl_comm, conf_all, len_all, (cudaStream_t)stream, &row0,
                    &B_sel);
  if (rc) return rc;
  return tetris_step_stochastic_f32(conf_all, len_local ? len_all : nullptr, B_sel, k, C, row0, B_local, p, q, d,
                                    u_acc, 0, u_res, cap, V, windows_all, win_offsets_all, accepted, out_tok, mass_out,
                                    offsets, tokens, stats4, status, ws, ws_bytes, stream);
}

extern "C" int tetris_dist_step_stochastic_bf16(const double* conf_local, const int32_t* len_local, int32_t B_local,
                                                int32_t k, int64_t C, const uint16_t* zp, const float* lse_p,
                                                const uint16_t* zq, const float* lse_q, const int32_t* d,
                                                const double* u_acc, const double* u_res, const int32_t* cap,
                                                int32_t V, void* nccl_comm, double* conf_all, int32_t* len_all,
                                                int32_t* windows_all, int32_t* win_offsets_all, int32_t* accepted,
                                                int32_t* out_tok, double* mass_out, int32_t* offsets, int32_t* tokens,
                                                int64_t* stats4, uint32_t* status, void* ws, size_t ws_bytes,
                                                tetris_stream_t stream) {
  int32_t row0, B_sel;
  int rc = prologue(conf_local, len_local, B_local, k, nccl_comm, conf_all, len_all, (cudaStream_t)stream, &row0,
                    &B_sel);
  if (rc) return rc;
  return tetris_step_stochastic_bf16(conf_all, len_local ? len_all : nullptr, B_sel, k, C, row0, B_local, zp, lse_p,
                                     zq, lse_q, d, u_acc, 0, u_res, cap, V, windows_all, win_offsets_all, accepted,
                                     out_tok, mass_out, offsets, tokens, stats4, status, ws, ws_bytes, stream);
}

extern "C" int tetris_dist_step_greedy_f32(const double* conf_local, const int32_t* len_local, int32_t B_local,
                                           int32_t k, int64_t C, const float* p, const int32_t* d, const int32_t* cap,
                                           int32_t V, void* nccl_comm, double* conf_all, int32_t* len_all,
                                           int32_t* windows_all, int32_t* win_offsets_all, int32_t* accepted,
                                           int32_t* out_tok, int32_t* offsets, int32_t* tokens, int64_t* stats4,
                                           uint32_t* status, void* ws, size_t ws_bytes, tetris_stream_t stream) {
  int32_t row0, B_sel;
  int rc = prologue(conf_local, len_local, B_local, k, nccl_comm, conf_all, len_all, (cudaStream_t)stream, &row0,
                    &B_sel);
  if (rc) return rc;
  return tetris_step_greedy_f32(conf_all, len_local ? len_all : nullptr, B_sel, k, C, row0, B_local, p, d, cap, V,
                                windows_all, win_offsets_all, accepted, out_tok, offsets, tokens, stats4, status, ws,
                                ws_bytes, stream);
}
