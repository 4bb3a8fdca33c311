// Probe (measurement tool): latency and throughput of the legacy warp MMA
// mma.sync.m16n8k32.s8 and of dp4a on this GPU.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void mma_s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int CHAINS>
__global__ void mma_kernel(int iters, int* out, long long* cyc) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u};
  int c[CHAINS][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) mma_s8(c[k], a, (uint32_t)i + k, (uint32_t)k);
  long long t1 = clock64();
  int s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void dp4a_kernel(int iters, int* out) {
  int acc[8] = {};
  uint32_t x = threadIdx.x;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = __dp4a((int)(x + k), (int)(i * 3 + k), acc[k]);
  int s = 0;
  for (int k = 0; k < 8; ++k) s += acc[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaMalloc(&cyc, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  long long hc;
  // latency: one warp, one chain
  mma_kernel<1><<<1, 32>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("mma.sync m16n8k32 s8 latency: %.1f cycles\n", (double)hc / iters);
  mma_kernel<8><<<1, 32>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("8 chains, 1 warp: %.1f cycles per mma\n", (double)hc / iters / 8);
  // throughput: all SMs, 8 warps per block, 4 blocks per SM, 8 chains
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    mma_kernel<8><<<148 * 4, 256>>>(iters, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * (148 * 4 * 8);
  printf("mma.sync s8 throughput: %.1f TOPS\n", ops / ms / 1e9);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    dp4a_kernel<<<148 * 8, 256>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  ops = 2.0 * 4 * 8.0 * iters * (148.0 * 8 * 256);
  printf("dp4a throughput: %.1f TOPS\n", ops / ms / 1e9);
  return 0;
}
