// Microbenchmark: cycles for ONE CTA (1024 threads) to bring 128 KB from cold DRAM into shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o load128k load128k.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_load(const double* __restrict__ src, long long* out, double* sink) {
  extern __shared__ __align__(128) double buf[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int n = 16384;
  long long t0 = clock64();
  if (MODE == 0) {  // 8B coalesced, 16 per thread in flight
    double v[16];
#pragma unroll
    for (int x = 0; x < 16; ++x) v[x] = __ldg(src + x * 1024 + tid);
#pragma unroll
    for (int x = 0; x < 16; ++x) buf[x * 1024 + tid] = v[x];
  } else if (MODE == 1) {  // 16B coalesced, 8 per thread
    double2 v[8];
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int x = 0; x < 8; ++x) v[x] = __ldg(s2 + x * 1024 + tid);
#pragma unroll
    for (int x = 0; x < 8; ++x) reinterpret_cast<double2*>(buf)[x * 1024 + tid] = v[x];
  } else {  // bulk copies: MODE-1 pieces
    const int pieces = MODE == 2 ? 1 : (MODE == 3 ? 8 : 64);
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(n * 8) : "memory");
    }
    __syncthreads();
    if (tid < pieces) {
      const int bytes = n * 8 / pieces;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32((char*)buf + tid * bytes)),
                   "l"((const char*)src + tid * bytes), "r"(bytes), "r"(smem_u32(&bar))
                   : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nWAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra WAIT;\n}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[MODE] = t1 - t0;
  if (buf[(tid * 7) % n] == 12345.0) sink[0] = 1.0;
}

int main() {
  const size_t big = (size_t)1 << 30;  // 1 GB, pick a fresh 128 KB slice per launch (cold in L2)
  double* src;
  cudaMalloc(&src, big);
  cudaMemset(src, 0, big);
  long long* out;
  cudaMallocManaged(&out, 8 * sizeof(long long));
  double* sink;
  cudaMalloc(&sink, 8);
  void (*ks[5])(const double*, long long*, double*) = {k_load<0>, k_load<1>, k_load<2>, k_load<3>, k_load<4>};
  const char* names[5] = {"8B coalesced x16", "16B coalesced x8", "1 bulk 128KB", "8 bulk 16KB", "64 bulk 2KB"};
  // flush L2 between runs by touching a 256 MB buffer
  char* flush;
  cudaMalloc(&flush, 256 << 20);
  for (int m = 0; m < 5; ++m) {
    cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    long long best = 1LL << 60, sum = 0;
    for (int it = 0; it < 10; ++it) {
      cudaMemsetAsync(flush, it, 256 << 20);
      const double* s = src + ((size_t)(it * 5 + m) * 16384 * 3) % (big / 8 - 16384);
      ks[m]<<<1, 1024, 131072>>>(s, out, sink);
      cudaDeviceSynchronize();
      best = out[m] < best ? out[m] : best;
      sum += out[m];
    }
    printf("%-20s best %lld cycles, mean %lld\n", names[m], best, sum / 10);
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
