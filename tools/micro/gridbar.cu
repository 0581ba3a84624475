// Microbenchmark: cost of a software grid barrier (generation counter in global memory) across G co-resident CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridbar gridbar.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int atom_acqrel(int* p, int v) {
  int o;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}
template <int MODE>
__device__ void gsync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (MODE == 0) {  // generation barrier
      const unsigned g0 = ld_acq(bar + 1);
      const int old = atom_acqrel((int*)bar, 1);
      if ((unsigned)old == gridDim.x - 1) {
        bar[0] = 0;
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(g0 + 1) : "memory");
      } else {
        while (ld_acq(bar + 1) == g0) {
        }
      }
    } else {  // monotonic counter: target = G * (index + 1)
      __shared__ unsigned idx;
      if (MODE == 1) {
        static __device__ unsigned dummy;
        (void)dummy;
      }
      const unsigned target = (bar[3] + 1) * gridDim.x;  // bar[3]: per-CTA local count kept in smem instead
      (void)target;
    }
  }
  __syncthreads();
}

__global__ void k_bar(unsigned* bar, int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) gsync<0>(bar);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_mono(unsigned* cnt, int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(cnt, 1u);
      __threadfence();
      const unsigned target = (unsigned)(i + 1) * gridDim.x;
      while (ld_acq(cnt) < target) {
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = t1 - t0;
}

int main() {
  unsigned* bar;
  cudaMalloc(&bar, 64);
  long long* out;
  cudaMallocManaged(&out, 16);
  for (int G : {16, 64, 148}) {
    for (int T : {256, 512}) {
      cudaMemset(bar, 0, 64);
      void* args[] = {&bar, nullptr, &out};
      int iters = 100;
      args[1] = &iters;
      cudaLaunchCooperativeKernel((void*)k_bar, G, T, args, 0, 0);
      cudaDeviceSynchronize();
      cudaMemset(bar, 0, 64);
      cudaLaunchCooperativeKernel((void*)k_mono, G, T, args, 0, 0);
      cudaDeviceSynchronize();
      printf("G=%3d T=%3d: generation barrier %6.0f cycles, monotonic counter %6.0f cycles per barrier\n", G, T,
             out[0] / 100.0, out[1] / 100.0);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
