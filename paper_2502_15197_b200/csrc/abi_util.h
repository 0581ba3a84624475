// Host-side helpers shared by the C-ABI wrappers: thread-local last error, launch checks, workspace layout.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>

#include <atomic>
#include <mutex>

#include "tetris_b200.h"

namespace tetris {
namespace abi {

char* err_buf();  // thread-local, defined in abi.cu

inline int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err_buf(), 512, fmt, ap);
  va_end(ap);
  return code;
}

// the call site (file:line of the ABI code) is part of the message, so a failing launch can be located
inline int cuda_fail(cudaError_t e, const char* file = __builtin_FILE(), int line = __builtin_LINE()) {
  const char* base = file;
  for (const char* c = file; *c; ++c)
    if (*c == '/') base = c + 1;
  return fail(TETRIS_CUDA_ERROR, "CUDA error: %s (%s:%d)", cudaGetErrorString(e), base, line);
}

inline int launch_check(const char* file = __builtin_FILE(), int line = __builtin_LINE()) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, file, line);
  return TETRIS_OK;
}

// Raise the kernel's dynamic shared-memory limit to `bytes` when needed.  The 48 KB default covers static + dynamic
// together, so any dynamic size is set explicitly (a kernel with 17 KB of static shared memory fails to launch with
// 40 KB dynamic otherwise); the largest size set so far per kernel is remembered to skip redundant driver calls.
template <typename K>
inline cudaError_t ensure_smem(K kernel, size_t bytes) {
  struct Entry {
    const void* fn;
    int dev;  // the attribute is per device
    size_t max;
  };
  static Entry table[64];
  static std::mutex mu;  // host threads may launch concurrently (the ABI is reentrant)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  const void* fn = reinterpret_cast<const void*>(kernel);
  int slot = -1;
  for (int i = 0; i < 64; ++i) {
    if (table[i].fn == fn && table[i].dev == dev) {
      if (table[i].max >= bytes) return cudaSuccess;
      slot = i;
      break;
    }
    if (table[i].fn == nullptr) {
      slot = i;
      break;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && slot >= 0) table[slot] = Entry{fn, dev, bytes};
  return e;
}

// SM count of the CURRENT device, cached per device (a process may drive GPUs / MIG slices of different sizes;
// grids sized from another device's count would break the cooperative launches' co-residency).  Lock-free: racing
// first calls write the same value.
inline int device_sm_count() {
  static std::atomic<int> cache[128];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 128) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;
    }
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

enum Region { WS_KEYS, WS_COUNTERS, WS_GSEL, WS_CHUNK_SUMS, WS_WARP_SUMS, WS_ARG_VAL, WS_ARG_IDX, WS_SCRATCH, WS_ROWINFO, WS_ACCBYTES, WS_ROWMAP, WS_SPEC_SUMS, WS_ROWLSE, WS_SPEC_LSE, WS_END };

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Workspace layout.  The arrival counters sit in a fixed-size region at offset 0 (one slot per possible request),
// so a workspace reused across calls of different shapes never finds stale sums where counters must be zero.
constexpr size_t kRequestSlots = 65536;                 // per-request arrival counters [0, 65536)
constexpr size_t kSlotAccCounter = kRequestSlots;        // accept-CTA arrivals of the fused select launch
constexpr size_t kSlotGridCount = kRequestSlots + 2;     // grid barrier of the persistent sampler: arrivals
constexpr size_t kSlotGridGen = kRequestSlots + 3;       //   ... and generation
constexpr size_t kSlotWorkCounter = kRequestSlots + 4;   // the sampler's dynamic work counter (64-bit, 2 slots)
constexpr size_t kSlotWorkSpec = kRequestSlots + 6;      // the speculative sampler's phase-A counter (64-bit, 2 slots)
constexpr size_t kSlotSpecCnt = kRequestSlots + 64;      // its per-request completion counters [64 + 0, 64 + 4096)
constexpr size_t kSpecSlots = 4096;
constexpr size_t kSlotSpecCtl = kRequestSlots + 8;       // [2]: phase-A list length, requests processed
constexpr size_t kSlotFusedCtl = kRequestSlots + 10;     // [3]: fused step: CTAs counted in, scans done, epoch
constexpr size_t kSlotSpecBitmap = kSlotSpecCnt + kSpecSlots;   // [kSpecSlots / 32]: the phase-A set
constexpr size_t kSlotSpecList = kSlotSpecBitmap + kSpecSlots / 32;  // [kSpecSlots]: the phase-A list
constexpr size_t kSlotGreedyKey0 = kSlotSpecList + kSpecSlots;  // [2 * 65536]: greedy row-0 argmax keys (u64)
constexpr size_t kSlotFusedReady = kSlotGreedyKey0 + 2 * kRequestSlots;  // [2 * 4096]: fused step ready words (u64)
constexpr size_t kCounterSlots = kSlotFusedReady + 2 * 4096;
static_assert(kSlotGreedyKey0 % 2 == 0 && kSlotFusedReady % 2 == 0, "8-byte aligned greedy keys / ready words");
constexpr size_t kGselScratchBytes = 32 * 1024;  // grid selector: radix histograms, barrier words, CTA totals
static_assert(kSlotGridGen == kSlotGridCount + 1, "grid_barrier reads the generation at bar + 1");
static_assert(kSlotWorkCounter == kSlotGridCount + 2 && (kSlotWorkCounter % 2) == 0,
              "persist_stream_kernel reads its 8-byte-aligned work counter at grid_bar + 2");
static_assert(kSlotWorkSpec == kSlotGridCount + 4, "persist_stream_kernel reads its phase-A counter at grid_bar + 4");

inline size_t region_offset(int op, int B, int k, int V, Region which) {
  const size_t nch = (size_t)((V + TETRIS_CHUNK_ELEMS - 1) / TETRIS_CHUNK_ELEMS);
  size_t sizes[WS_END] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  sizes[WS_COUNTERS] = kCounterSlots * 4;
  sizes[WS_GSEL] = kGselScratchBytes;  // shape-independent, right after the counters: a fixed offset in every layout
  if (op & TETRIS_OP_SELECT) {
    // radix keys; or the heap replay's items (16 B per row) followed by its cell keys
    const size_t keys = (size_t)B * k * 8, heap = (size_t)B * 16;
    sizes[WS_KEYS] = keys + heap;
  }
  if (op & TETRIS_OP_VERIFY) {
    // rows processed by one verify call: B requests (stochastic/greedy) or R sampled rows (sample_rows)
    sizes[WS_CHUNK_SUMS] = (size_t)B * nch * 8;
    // warp sums; rows of <= kSegSumMaxChunks chunks: the 32 segment sums of every chunk instead (stream.cu)
    const size_t per_chunk = nch <= 4 ? (size_t)TETRIS_CHUNK_WARPS * TETRIS_WARP_SEGS : (size_t)TETRIS_CHUNK_WARPS;
    sizes[WS_WARP_SUMS] = (size_t)B * nch * per_chunk * 8;
    sizes[WS_ARG_VAL] = (size_t)B * (k + 1) * (nch > 1 ? nch : 2) * 4;  // also the greedy argmax keys (8 B per row)
    sizes[WS_ARG_IDX] = (size_t)B * (k + 1) * nch * 4;
    sizes[WS_SCRATCH] = align_up((size_t)B * 8) * 3 + align_up((size_t)B * 4);  // residual: rows, u, idx
    sizes[WS_ROWINFO] = (size_t)B * 16;  // accept result: row to resample from (p row, q row)
    sizes[WS_ACCBYTES] = (size_t)B * k;  // pre-accept verdicts
    sizes[WS_ROWMAP] = 256 + (size_t)B * (k + 1) * 4;  // greedy: [0] selected-row count, then row -> (b, j)
    // speculative sampler: the phase-A chunk sums then warp sums (B <= kSpecSlots)
    sizes[WS_SPEC_SUMS] = B <= (int)kSpecSlots ? (size_t)B * nch * 8 * (1 + per_chunk) : 0;
    // logits form: the lse of each request's two rows beside the row info, and of each phase-A list entry's rows
    sizes[WS_ROWLSE] = (size_t)B * 8;
    sizes[WS_SPEC_LSE] = B <= (int)kSpecSlots ? (size_t)B * 8 : 0;
  }
  const Region order[WS_END] = {WS_COUNTERS, WS_GSEL,    WS_KEYS,    WS_CHUNK_SUMS, WS_WARP_SUMS,
                                WS_ARG_VAL,  WS_ARG_IDX, WS_SCRATCH, WS_ROWINFO,    WS_ACCBYTES,
                                WS_ROWMAP,   WS_SPEC_SUMS, WS_ROWLSE, WS_SPEC_LSE};
  size_t off = 0;
  for (int i = 0; i < WS_END; ++i) {
    if (order[i] == which) return off;
    off += align_up(sizes[order[i]]);
  }
  return off;  // WS_END -> total
}

inline void* ws_region(void* ws, int op, int B, int k, int V, Region which) {
  return (char*)ws + region_offset(op, B, k, V, which);
}

}  // namespace abi
}  // namespace tetris
