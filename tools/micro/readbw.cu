// Microbenchmark: achievable DRAM read bandwidth on this B200 (pure read, no write): (a) LDG.256 grid-stride sum,
// (b) persistent TMA 1-D bulk copies (32 KB chunks, 3-stage ring, one CTA per SM) into shared memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o readbw readbw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_ldg(const float* __restrict__ p, size_t n8, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n8; i += (size_t)gridDim.x * blockDim.x) {
    float v[8];
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p + i * 8));
    acc += v[0] + v[1] + v[2] + v[3] + v[4] + v[5] + v[6] + v[7];
  }
  if (acc == 1234.5f) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(64, 1) k_tma(const char* __restrict__ p, size_t nchunks, float* out) {
  extern __shared__ __align__(128) char buf[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid != 0) return;
  int t = 0;
  float acc = 0.f;
  // issue STAGES ahead, consume (touch one word) and re-issue
  size_t next = blockIdx.x;
  for (int s = 0; s < STAGES && next < nchunks; ++s, next += gridDim.x) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(buf + s * CHUNK)), "l"(p + next * CHUNK), "r"(CHUNK), "r"(su32(&full[s]))
                 : "memory");
  }
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++t) {
    const int s = t % STAGES;
    const uint32_t ph = (t / STAGES) & 1;
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(
                     su32(&full[s])), "r"(ph) : "memory");
    acc += *(volatile float*)(buf + s * CHUNK);
    if (next < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(buf + s * CHUNK)), "l"(p + next * CHUNK), "r"(CHUNK), "r"(su32(&full[s]))
                   : "memory");
      next += gridDim.x;
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const size_t bytes = (size_t)8 << 30;
  char* p;
  cudaMalloc(&p, bytes);
  cudaMemset(p, 0, bytes);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-34s %8.1f GB/s\n", name, bytes / (best * 1e-3) / 1e9);
  };
  for (int bpsm : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "LDG.256 %d CTAs/SM x 512 thr", bpsm);
    run(nm, [&] { k_ldg<<<sms * bpsm, 512>>>((const float*)p, bytes / 32, out); });
  }
  {
    auto kern = k_tma<3, 65536>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    run("TMA 3x64KB per SM", [&] { kern<<<sms, 64, 3 * 65536>>>(p, bytes / 65536, out); });
    auto kern2 = k_tma<6, 32768>;
    cudaFuncSetAttribute(kern2, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    run("TMA 6x32KB per SM", [&] { kern2<<<sms, 64, 6 * 32768>>>(p, bytes / 32768, out); });
    auto kern3 = k_tma<4, 32768>;
    cudaFuncSetAttribute(kern3, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    run("TMA 4x32KB per SM", [&] { kern3<<<sms, 64, 4 * 32768>>>(p, bytes / 32768, out); });
  }
  {  // copy for reference (read + write)
    char* q;
    cudaMalloc(&q, bytes / 2);
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
      cudaEventRecord(a);
      cudaMemcpyAsync(q, p, bytes / 2, cudaMemcpyDeviceToDevice);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-34s %8.1f GB/s (read+write)\n", "cudaMemcpy D2D", bytes / (best * 1e-3) / 1e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
