// Microbenchmark: per-SM throughput of F2F.F64.F32 (float->double), DADD, DMNMX-style max, and FADD on this B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64 fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* in, double* out, int iters, long long* cyc) {
  float f[8];
  double d[8];
  for (int i = 0; i < 8; ++i) {
    f[i] = in[threadIdx.x * 8 + i];
    d[i] = (double)f[i];
  }
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {
        d[i] += (double)f[i];  // F2F (+ DADD to keep it live)
        f[i] = f[i] * 1.0000001f;
      } else if (OP == 1) {
        d[i] = d[i] + 1.0000001;  // DADD
      } else if (OP == 2) {
        d[i] = d[i] > 0.5 ? d[i] - 0.25 : d[i] + 0.25;  // compare/select chain
      } else {
        f[i] = f[i] + 1.0000001f;  // FADD
      }
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += d[i] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[OP] = t1 - t0;
}

int main() {
  float* in;
  double* out;
  long long* cyc;
  cudaMalloc(&in, 1 << 20);
  cudaMemset(in, 0, 1 << 20);
  cudaMalloc(&out, 1 << 22);
  cudaMallocManaged(&cyc, 64);
  const int iters = 4096, threads = 1024;
  const char* names[4] = {"F2F+DADD+FMUL", "DADD", "DSETP+DADD+SEL", "FADD"};
  void (*ks[4])(float*, double*, int, long long*) = {k<0>, k<1>, k<2>, k<3>};
  for (int op = 0; op < 4; ++op) {
    ks[op]<<<1, threads>>>(in, out, iters, cyc);
    cudaDeviceSynchronize();
    ks[op]<<<1, threads>>>(in, out, iters, cyc);
    cudaDeviceSynchronize();
    const double ops = (double)iters * 8 * threads;
    printf("%-16s %6.2f ops/clk/SM (1 CTA x %d threads)\n", names[op], ops / cyc[op], threads);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
