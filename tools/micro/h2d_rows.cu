// Host->device row gather, the e2e step's transfer: 2048 rows of R bytes at random positions of a pinned host
// buffer into a dense device staging buffer.  Compares (1) one contiguous copy of the same bytes (ceiling),
// (2) one cudaMemcpyAsync per row over S streams, (3) an SM gather kernel reading the mapped host memory with
// 16-byte loads (G CTAs x T threads), (4) the two at once (a fraction of the rows by DMA, the rest by the kernel).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o h2d_rows h2d_rows.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);             \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// one CTA per row slice: rows [r0, r1) of the list, each row's 16-byte words strided over the CTA, 4 in flight
__global__ void gather_kernel(const int4* __restrict__ host, const long long* __restrict__ src_row, int4* dst,
                              int nrows, long long row_words) {
  for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int4* s = host + src_row[r] * row_words;
    int4* d = dst + (long long)r * row_words;
    for (long long i = threadIdx.x; i < row_words; i += 4 * blockDim.x) {
      int4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * blockDim.x < row_words) v[u] = __ldcv(s + i + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u * blockDim.x < row_words) d[i + u * blockDim.x] = v[u];
    }
  }
}

// TMA variant: each CTA moves whole rows through a ring of shared-memory stages with bulk copies, host -> shared
// (cp.async.bulk from the mapped host address) then shared -> device (cp.async.bulk.global.shared::cta)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int S, int CH>
__global__ void __launch_bounds__(32) tma_gather_kernel(const char* __restrict__ host, const long long* src_row,
                                                        char* dst, int nrows, long long row_bytes) {
  extern __shared__ __align__(128) char stage[];
  __shared__ __align__(8) unsigned long long full[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long nch = (row_bytes + CH - 1) / CH;
  long long t = 0;
  // items (row r of this CTA, chunk c): issue up to S loads ahead, then for each landed stage a bulk store
  auto issue = [&](long long it) {
    const int r = blockIdx.x + (int)(it / nch) * gridDim.x;
    const long long c = it % nch;
    const long long off = c * CH, n = row_bytes - off < CH ? row_bytes - off : CH;
    const int s = (int)(it % S);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"((uint32_t)n));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(stage + (size_t)s * CH)),
                 "l"(host + src_row[r] * row_bytes + off), "r"((uint32_t)n), "r"(smem_u32(&full[s]))
                 : "memory");
  };
  const int myrows = blockIdx.x < nrows ? (nrows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const long long items = (long long)myrows * nch;
  for (; t < items && t < S; ++t) issue(t);
  (void)t;
  for (long long it = 0; it < items; ++it) {
    const int s = (int)(it % S);
    const uint32_t par = (uint32_t)((it / S) & 1);
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
                     smem_u32(&full[s])),
                 "r"(par)
                 : "memory");
    const int r = blockIdx.x + (int)(it / nch) * gridDim.x;
    const long long c = it % nch;
    const long long off = c * CH, n = row_bytes - off < CH ? row_bytes - off : CH;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (long long)r * row_bytes + off),
                 "r"(smem_u32(stage + (size_t)s * CH)), "r"((uint32_t)n)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // refill the PREVIOUS item's stage once its store has read it (the newest store may still be in flight)
    if (it >= 1 && it - 1 + S < items) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(it - 1 + S);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const long long row_bytes = argc > 1 ? atoll(argv[1]) : 128256 * 4;
  const int nrows = argc > 2 ? atoi(argv[2]) : 1800;
  const int pool_rows = 8 * nrows;  // rows to pick from (the p/q tensors are far larger than what one step reads)
  const size_t pool = (size_t)pool_rows * row_bytes;
  char* host;
  CK(cudaHostAlloc(&host, pool, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < pool; i += 4096) host[i] = (char)i;
  char* hdev;
  CK(cudaHostGetDevicePointer((void**)&hdev, host, 0));
  char* dst;
  CK(cudaMalloc(&dst, (size_t)nrows * row_bytes));
  std::vector<long long> rows(nrows);
  srand(1);
  for (int r = 0; r < nrows; ++r) rows[r] = (long long)(rand() % pool_rows);
  long long* drows;
  CK(cudaMalloc(&drows, nrows * sizeof(long long)));
  CK(cudaMemcpy(drows, rows.data(), nrows * sizeof(long long), cudaMemcpyHostToDevice));
  cudaStream_t st[16];
  for (int i = 0; i < 16; ++i) CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  cudaEvent_t e0, e1, ej[16];
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 16; ++i) CK(cudaEventCreateWithFlags(&ej[i], cudaEventDisableTiming));
  const double gb = (double)nrows * row_bytes / 1e9;
  auto report = [&](const char* what, int reps) {
    float ms;
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    printf("%-44s %8.3f ms  %6.1f GB/s\n", what, ms, gb / (ms / 1e3));
  };
  const int reps = 5;
  // (1) one contiguous copy of the same byte count
  for (int w = 0; w < 2; ++w) {
    CK(cudaEventRecord(e0, st[0]));
    for (int r = 0; r < reps; ++r)
      CK(cudaMemcpyAsync(dst, host, (size_t)nrows * row_bytes, cudaMemcpyHostToDevice, st[0]));
    CK(cudaEventRecord(e1, st[0]));
    if (w) report("one contiguous copy", reps);
  }
  // (2) one copy per row over S streams
  for (int S : {1, 2, 4, 8, 16}) {
    for (int w = 0; w < 2; ++w) {
      CK(cudaEventRecord(e0, st[0]));
      for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(ej[0], st[0]));
        for (int s = 1; s < S; ++s) CK(cudaStreamWaitEvent(st[s], ej[0], 0));
        for (int i = 0; i < nrows; ++i)
          CK(cudaMemcpyAsync(dst + (size_t)i * row_bytes, host + rows[i] * row_bytes, row_bytes,
                             cudaMemcpyHostToDevice, st[i % S]));
        for (int s = 1; s < S; ++s) {
          CK(cudaEventRecord(ej[s], st[s]));
          CK(cudaStreamWaitEvent(st[0], ej[s], 0));
        }
      }
      CK(cudaEventRecord(e1, st[0]));
      char name[64];
      snprintf(name, 64, "per-row copies, %d streams", S);
      if (w) report(name, reps);
    }
  }
  // (3) gather kernel
  const long long words = row_bytes / 16;
  for (int G : {148, 296, 592, 1184}) {
    for (int T : {256, 512, 1024}) {
      for (int w = 0; w < 2; ++w) {
        CK(cudaEventRecord(e0, st[0]));
        for (int r = 0; r < reps; ++r)
          gather_kernel<<<G, T, 0, st[0]>>>((const int4*)hdev, drows, (int4*)dst, nrows, words);
        CK(cudaEventRecord(e1, st[0]));
        CK(cudaGetLastError());
        char name[64];
        snprintf(name, 64, "gather kernel %d x %d", G, T);
        if (w) report(name, reps);
      }
    }
  }
  // (3b) TMA gather: one CTA (one thread) per SM-slot, S stages of CH bytes
  {
    constexpr int S = 6, CH = 32768;
    CK(cudaFuncSetAttribute(tma_gather_kernel<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH));
    for (int G : {148, 296, 592}) {
      for (int w = 0; w < 2; ++w) {
        CK(cudaEventRecord(e0, st[0]));
        for (int r = 0; r < reps; ++r)
          tma_gather_kernel<S, CH><<<G, 32, S * CH, st[0]>>>(hdev, drows, dst, nrows, row_bytes);
        CK(cudaEventRecord(e1, st[0]));
        CK(cudaGetLastError());
        char name[64];
        snprintf(name, 64, "TMA gather %d CTAs x %d x %d KB", G, S, CH / 1024);
        if (w) report(name, reps);
      }
    }
  }
  // (4) split: the first f of the rows by DMA (8 streams), the rest by the kernel, concurrently
  for (double f : {0.2, 0.35, 0.5}) {
    const int nd = (int)(f * nrows);
    for (int w = 0; w < 2; ++w) {
      CK(cudaEventRecord(e0, st[0]));
      for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(ej[0], st[0]));
        for (int s = 1; s < 9; ++s) CK(cudaStreamWaitEvent(st[s], ej[0], 0));
        gather_kernel<<<592, 512, 0, st[0]>>>((const int4*)hdev, drows + nd, (int4*)(dst + (size_t)nd * row_bytes),
                                              nrows - nd, words);
        for (int i = 0; i < nd; ++i)
          CK(cudaMemcpyAsync(dst + (size_t)i * row_bytes, host + rows[i] * row_bytes, row_bytes,
                             cudaMemcpyHostToDevice, st[1 + i % 8]));
        for (int s = 1; s < 9; ++s) {
          CK(cudaEventRecord(ej[s], st[s]));
          CK(cudaStreamWaitEvent(st[0], ej[s], 0));
        }
      }
      CK(cudaEventRecord(e1, st[0]));
      char name[64];
      snprintf(name, 64, "split: %.0f%% DMA + gather kernel", f * 100);
      if (w) report(name, reps);
    }
  }
  return 0;
}
