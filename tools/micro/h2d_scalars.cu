// Scattered 4-byte reads of mapped pinned host memory (the staged step's accept test: p[b][j][d], q[b][j][d] through
// the mapping): N reads at random rows of a pool of R rows x 513 KB, one read per thread, G CTAs of 1024 threads.
// Compares pool sizes (GPU TLB reach) and reads per thread.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o s h2d_scalars.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                      \
  do {                                                             \
    cudaError_t e_ = (x);                                          \
    if (e_ != cudaSuccess) {                                       \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); \
      exit(1);                                                     \
    }                                                              \
  } while (0)

template <int U>
__global__ void reads(const float* host, const long long* idx, float* out, int n) {
  const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * U;
  float v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = i0 + u < n ? host[idx[i0 + u]] : 0.f;
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) s += v[u];
  if (i0 < n) out[i0 / U] = s;
}

int main() {
  const long long row = 128256;  // floats per row
  const int n = 32768;
  for (long long rows : {128LL, 2048LL, 17408LL * 2}) {
    const size_t bytes = (size_t)rows * row * 4;
    float* host;
    if (cudaHostAlloc(&host, bytes, cudaHostAllocMapped) != cudaSuccess) {
      printf("alloc %zu failed\n", bytes);
      cudaGetLastError();
      continue;
    }
    for (size_t i = 0; i < bytes / 4; i += 1024) host[i] = 1.f;
    float* hdev;
    CK(cudaHostGetDevicePointer((void**)&hdev, host, 0));
    std::vector<long long> idx(n);
    srand(3);
    for (int i = 0; i < n; ++i) idx[i] = (long long)(rand() % rows) * row + rand() % row;
    long long* didx;
    float* out;
    CK(cudaMalloc(&didx, n * 8));
    CK(cudaMalloc(&out, n * 4));
    CK(cudaMemcpy(didx, idx.data(), n * 8, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto run = [&](auto kern, int U, const char* nm) {
      const int threads = n / U, G = (threads + 1023) / 1024;
      for (int w = 0; w < 3; ++w) {
        CK(cudaEventRecord(a));
        kern<<<G, 1024>>>(hdev, didx, out, n);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
      }
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      printf("pool %6.1f GB, %d reads, %s (%d CTAs): %8.1f us  (%.1f M reads/s)\n", bytes / 1e9, n, nm, G, ms * 1e3,
             n / (ms * 1e3));
    };
    run(reads<1>, 1, "1 read/thread");
    run(reads<4>, 4, "4 reads/thread");
    run(reads<16>, 16, "16 reads/thread");
    // spread over G CTAs of n / G threads (every SM issues a share)
    for (int G : {64, 128, 147, 296}) {
      const int T = (n + G - 1) / G;
      for (int w = 0; w < 3; ++w) {
        CK(cudaEventRecord(a));
        reads<1><<<G, T>>>(hdev, didx, out, n);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
      }
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      printf("pool %6.1f GB, %d reads, 1 read/thread, %d CTAs x %d: %8.1f us  (%.1f M reads/s)\n", bytes / 1e9, n, G, T,
             ms * 1e3, n / (ms * 1e3));
    }
    CK(cudaFreeHost(host));
    CK(cudaFree(didx));
    CK(cudaFree(out));
  }
  return 0;
}
