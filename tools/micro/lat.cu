// Latency micro-benchmark (B200): dependent chains of the operations the small-batch step's prologue and descent are
// built from, timed with clock64 in one warp (SM cycles per operation).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/micro/lat.cu && /tmp/lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* dbuf, unsigned long long* gbuf, int* ibuf, long long* out, int n) {
  __shared__ unsigned long long sh[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) sh[i] = (unsigned long long)((i * 7 + 1) & 1023);
  __syncthreads();
  if (tid >= 32) {
    // the other warps: take part in the named-barrier test below only
    for (int it = 0; it < n; ++it) asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x));
    return;
  }
  long long t0, t1;
  // DMUL chain
  double x = dbuf[0], y = dbuf[1];
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
  t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / n;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / n;
  // LDS pointer chase
  unsigned long long p = tid;
  t0 = clock64();
  for (int i = 0; i < n; ++i) p = sh[p];
  t1 = clock64();
  if (tid == 0) out[2] = (t1 - t0) / n;
  // shfl chain
  double s = x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1.0;
  t1 = clock64();
  if (tid == 0) out[3] = (t1 - t0) / n;
  // global (L2-resident) pointer chase
  unsigned long long q = tid;
  t0 = clock64();
  for (int i = 0; i < n; ++i) q = __ldcg(gbuf + q);
  t1 = clock64();
  if (tid == 0) out[4] = (t1 - t0) / n;
  // atom.add.acq_rel.gpu round trips (lane 0)
  if (tid == 0) {
    int v = 0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
      int old;
      asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(ibuf + (v & 1)), "r"(1) : "memory");
      v += old;
    }
    t1 = clock64();
    out[5] = (t1 - t0) / n;
    // relaxed atomics
    t0 = clock64();
    for (int i = 0; i < n; ++i) v += atomicAdd(ibuf + 2 + (v & 1), 1);
    t1 = clock64();
    out[6] = (t1 - t0) / n;
    // fence.acq_rel.gpu after a store
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
      ibuf[4] = i;
      __threadfence();
    }
    t1 = clock64();
    out[7] = (t1 - t0) / n;
    out[10] = v;
  }
  __syncwarp();
  // __nanosleep(32 / 256 / 1000) as polling loops use it
  if (tid == 0) {
    t0 = clock64();
    for (int i = 0; i < 64; ++i) __nanosleep(32);
    t1 = clock64();
    out[11] = (t1 - t0) / 64;
    t0 = clock64();
    for (int i = 0; i < 64; ++i) __nanosleep(256);
    t1 = clock64();
    out[12] = (t1 - t0) / 64;
    t0 = clock64();
    for (int i = 0; i < 16; ++i) __nanosleep(1000);
    t1 = clock64();
    out[13] = (t1 - t0) / 16;
  }
  __syncwarp();
  // named barrier over the whole block (every warp arrives every iteration)
  t0 = clock64();
  for (int it = 0; it < n; ++it) asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x));
  t1 = clock64();
  if (tid == 0) out[8] = (t1 - t0) / n;
  if (tid == 0) out[9] = (long long)(x + s + (double)p + (double)q);
}

int main() {
  double* d;
  unsigned long long* g;
  int* ib;
  long long* o;
  cudaMalloc(&d, 16);
  cudaMalloc(&g, 1 << 20);
  cudaMalloc(&ib, 64);
  cudaMalloc(&o, 256);
  double h[2] = {1.0000001, 0.9999999};
  cudaMemcpy(d, h, 16, cudaMemcpyHostToDevice);
  unsigned long long hg[131072];
  for (int i = 0; i < 131072; ++i) hg[i] = (unsigned long long)((i * 97 + 13) % 131072);
  cudaMemcpy(g, hg, sizeof(hg), cudaMemcpyHostToDevice);
  cudaMemset(ib, 0, 64);
  for (int rep = 0; rep < 2; ++rep) lat_kernel<<<1, 576>>>(d, g, ib, o, 256);
  cudaDeviceSynchronize();
  long long r[14];
  cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: DMUL %lld  DADD %lld  LDS %lld  SHFL+DADD %lld  LDG.cg (L2) %lld  "
         "atom.acq_rel.gpu %lld  atomicAdd %lld  store+fence.gpu %lld  bar.sync(576 thr) %lld\n",
         r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], r[8]);
  printf("cycles per __nanosleep(32) %lld, (256) %lld, (1000) %lld\n", r[11], r[12], r[13]);
  return 0;
}
