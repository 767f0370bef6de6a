// microbenchmark: POPC vs ALU throughput on sm_100a (scratch, not product)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_popc(uint32_t *out, uint32_t seed, int iters) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t a4 = a0 * 9u, a5 = a0 * 11u, a6 = a0 * 13u, a7 = a0 * 15u;
  uint32_t m0 = 99, m1 = 99, m2 = 99, m3 = 99, m4=99,m5=99,m6=99,m7=99;
  for (int i = 0; i < iters; ++i) {
    uint32_t c = seed + i;
#define CHK(a,m) m = min(m, (uint32_t)__popc(a ^ c));
    CHK(a0,m0) CHK(a1,m1) CHK(a2,m2) CHK(a3,m3) CHK(a4,m4) CHK(a5,m5) CHK(a6,m6) CHK(a7,m7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = m0+m1+m2+m3+m4+m5+m6+m7;
}
// ALU-only d=3 test: popc(x) >= 3  <=>  (x & (x-1)) & ((x&(x-1))-1) != 0
__global__ void k_alu3(uint32_t *out, uint32_t seed, int iters) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t a4 = a0 * 9u, a5 = a0 * 11u, a6 = a0 * 13u, a7 = a0 * 15u;
  uint32_t m0 = ~0u, m1 = ~0u, m2 = ~0u, m3 = ~0u, m4=~0u,m5=~0u,m6=~0u,m7=~0u;
  for (int i = 0; i < iters; ++i) {
    uint32_t c = seed + i;
#define CHK3(a,m) { uint32_t x = a ^ c; uint32_t y = x & (x - 1u); y = y & (y - 1u); m = min(m, y); }
    CHK3(a0,m0) CHK3(a1,m1) CHK3(a2,m2) CHK3(a3,m3) CHK3(a4,m4) CHK3(a5,m5) CHK3(a6,m6) CHK3(a7,m7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = m0|m1|m2|m3|m4|m5|m6|m7;
}
// mixed: half popc half alu
__global__ void k_mix(uint32_t *out, uint32_t seed, int iters) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  uint32_t a4 = a0 * 9u, a5 = a0 * 11u, a6 = a0 * 13u, a7 = a0 * 15u;
  uint32_t m0 = 99, m1 = 99, m2 = 99, m3 = 99, m4=~0u,m5=~0u,m6=~0u,m7=~0u;
  for (int i = 0; i < iters; ++i) {
    uint32_t c = seed + i;
    CHK(a0,m0) CHK(a1,m1) CHK(a2,m2) CHK(a3,m3) CHK3(a4,m4) CHK3(a5,m5) CHK3(a6,m6) CHK3(a7,m7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = m0+m1+m2+m3+(m4|m5|m6|m7);
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%s SMs=%d clock(kHz)=%d\n", p.name, p.multiProcessorCount, clk);
  uint32_t *out; cudaMalloc(&out, 1 << 26);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 1 << 16;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[3] = {"popc", "alu3", "mix"};
  for (int kk = 0; kk < 3; ++kk) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (kk == 0) k_popc<<<blocks, threads>>>(out, 12345, iters);
      if (kk == 1) k_alu3<<<blocks, threads>>>(out, 12345, iters);
      if (kk == 2) k_mix<<<blocks, threads>>>(out, 12345, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double checks = (double)blocks * threads * iters * 8;
      printf("%s: %.3f ms  %.3e checks/s  %.2f checks/clk/SM @maxclk\n", names[kk], ms, checks / (ms * 1e-3),
             checks / (ms * 1e-3) / (p.multiProcessorCount * (double)clk * 1e3));
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
