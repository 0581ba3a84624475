// Microbenchmark: cost of a warp-0-only shared-memory scan phase inside a 1024-thread CTA, with and without a
// preceding histogram-atomics phase.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pick pick.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t wscan(uint32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(long long* out, int* sink, int natom) {
  __shared__ __align__(16) uint32_t h[2][2048];
  extern __shared__ uint8_t dyn[];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 4096; i += 1024) (&h[0][0])[i] = 0;
  __syncthreads();
  long long t0 = clock64();
  if (MODE >= 1) {
    for (int i = 0; i < natom; ++i) atomicAdd(&h[0][(tid * 7 + i * 13) & (MODE == 2 ? 31 : 2047)], 1u);
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t res = 0;
  if (tid < 32) {
    const uint4* h4 = reinterpret_cast<const uint4*>(h[0]) + lane * 16;
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const uint4 x = h4[(c + lane) & 15];
      s += x.x + x.y + x.z + x.w;
    }
    long long ta = clock64();
    const uint32_t incl = wscan(s, lane);
    const unsigned own = __ballot_sync(0xffffffffu, incl > 100);
    res = incl + own;
    long long tb = clock64();
    if (tid == 0) { out[4] = ta - t1; out[5] = tb - ta; }
  } else {
    for (int i = tid - 32; i < 2048; i += 992) h[1][i] = 0;
  }
  __syncthreads();
  long long t2 = clock64();
  if (tid == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
  }
  if (res == 123456789) sink[0] = 1;
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 16 * sizeof(long long));
  int* sink;
  cudaMalloc(&sink, 4);
  char* flush;
  cudaMalloc(&flush, 512 << 20);
  const char* names[3] = {"no atomics", "atomics spread", "atomics 32 bins"};
  void (*ks[3])(long long*, int*, int) = {k<0>, k<1>, k<2>};
  for (int dynsm : {0}) {
  printf("dynamic smem %d\n", dynsm);
  for (int m = 0; m < 3; ++m) {
    for (int natom : {4, 16}) {
      for (int it = 0; it < 4; ++it) {
        cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
        if (it >= 2) cudaMemset(flush, it, 512 << 20);
        ks[m]<<<1, 1024, dynsm>>>(out, sink, natom);
        cudaDeviceSynchronize();
        printf("%-16s natom %2d it %d%s: atom phase %lld, pick phase %lld (loads %lld, scan %lld)\n", names[m], natom,
               it, it >= 2 ? " (after L2 flush)" : "", out[0], out[1], out[4], out[5]);
      }
    }
  }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
