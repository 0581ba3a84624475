// Instruction-fetch micro-benchmark (B200): a straight-line block of N dependent-free integer instructions
// (N * 16 bytes of code) run twice in one launch by every warp of a 576-thread CTA on all SMs; clock64 around each
// pass shows whether first-pass code fetch (cold instruction cache) dominates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/icache tools/micro/icache.cu && /tmp/icache
#include <cstdio>
#include <cuda_runtime.h>

#define R4(X) X X X X
#define R16(X) R4(R4(X))
#define R256(X) R16(R16(X))
#define R1024(X) R4(R256(X))

template <int K>
__device__ __forceinline__ void block(float& a, float& b, float& c, float& d, float m, float n) {
  // K x 1024 x 4 FMAs on 4 independent accumulators (fp, so nothing can be folded)
#pragma unroll
  for (int k = 0; k < K; ++k) {
    R1024(asm volatile("fma.rn.f32 %0, %0, %4, %5; fma.rn.f32 %1, %1, %4, %5; fma.rn.f32 %2, %2, %4, %5; "
                       "fma.rn.f32 %3, %3, %4, %5;"
                       : "+f"(a), "+f"(b), "+f"(c), "+f"(d) : "f"(m), "f"(n));)
  }
}

template <int K>
__global__ void __launch_bounds__(576, 1) icache_kernel(long long* out, unsigned* sink) {
  float a = threadIdx.x, b = 1, c = 2, d = 3;
  const float m = 1.0f + 1e-7f * (float)blockIdx.x, n = 1e-3f;
  long long t[3];
  for (int pass = 0; pass < 2; ++pass) {
    __syncthreads();
    t[pass] = clock64();
    block<K>(a, b, c, d, m, n);
  }
  __syncthreads();
  t[2] = clock64();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t[1] - t[0];
    out[2 * blockIdx.x + 1] = t[2] - t[1];
  }
  if (a + b + c + d == 1234.5f) sink[0] = 1;
}

template <int K>
void run(long long* o, unsigned* s, int nsm) {
  for (int rep = 0; rep < 3; ++rep) icache_kernel<K><<<nsm, 576>>>(o, s);
  cudaDeviceSynchronize();
  long long h[2 * 148];
  cudaMemcpy(h, o, sizeof(long long) * 2 * nsm, cudaMemcpyDeviceToHost);
  double p0 = 0, p1 = 0;
  for (int i = 0; i < nsm; ++i) p0 += h[2 * i], p1 += h[2 * i + 1];
  const double ninst = 4096.0 * K;
  printf("code %6.0f KB (%6.0f instr/warp): pass 1 %8.0f cycles, pass 2 %8.0f cycles (18 warps; ideal issue %6.0f)\n",
         ninst * 16 / 1024, ninst, p0 / nsm, p1 / nsm, ninst * 18 / 4);
}

int main() {
  long long* o;
  unsigned* s;
  cudaMalloc(&o, 4096);
  cudaMalloc(&s, 16);
  int nsm = 148;
  run<1>(o, s, nsm);
  run<2>(o, s, nsm);
  run<4>(o, s, nsm);
  return 0;
}
