// tools/popc_peak.cu -- measured peak of the candidate-codeword check on sm_100a.
//
// The check is "popc(v ^ c) < d".  Two arithmetic forms are timed, each with many
// independent candidates per thread and a warp-uniform codeword stream (as in the kernel):
//   popc   : m = min(m, popc(v ^ c))                        (LOP3 + POPC + IMNMX)
//   mix<D> : half the candidates as popc, half as the bit-clearing form
//            m = min(m, clear_low<D>(v ^ c))  (x &= x - 1, D - 1 times; 0 iff popc < D)
// The reported rate (checks/clk/SM at the clock the run held) is the roofline denominator
// bench.py uses: popc for d > 4, mix<d> for 2 <= d <= 4.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o popc_peak tools/popc_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int D>
__device__ __forceinline__ uint32_t clear_low(uint32_t x) {
#pragma unroll
    for (int i = 0; i < D - 1; ++i) x &= x - 1u;
    return x;
}

constexpr int kC = 8;   // candidates per thread

template <int MIX>
__global__ void k_check(uint32_t *out, uint32_t seed, int iters) {
    uint32_t v[kC], m[kC];
#pragma unroll
    for (int r = 0; r < kC; ++r) { v[r] = (seed ^ threadIdx.x) * (2u * r + 3u); m[r] = 0xffffffffu; }
    for (int i = 0; i < iters; ++i) {
        const uint32_t c = seed + (uint32_t)i * 0x9e3779b9u;      // warp-uniform codeword
#pragma unroll
        for (int r = 0; r < kC; ++r) {
            if (MIX && (r & 1)) m[r] = min(m[r], clear_low<MIX>(v[r] ^ c));
            else m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c));
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int r = 0; r < kC; ++r) acc += m[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MIX>
double run(uint32_t *out, int blocks, int threads, int iters, double clk_hz, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_check<MIX><<<blocks, threads>>>(out, 12345u + rep, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double checks = (double)blocks * threads * iters * kC;
        const double per_clk_sm = checks / (ms * 1e-3) / (sms * clk_hz);
        if (per_clk_sm > best) best = per_clk_sm;
    }
    return best;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double clk = clk_khz * 1e3;
    uint32_t *out;
    cudaMalloc(&out, 1 << 26);
    const int sms = p.multiProcessorCount, blocks = sms * 8, threads = 256, iters = 1 << 15;
    printf("%s SMs=%d clock=%.0f MHz (rates below are per clk at this clock)\n", p.name, sms, clk / 1e6);
    printf("popc   : %.2f checks/clk/SM\n", run<0>(out, blocks, threads, iters, clk, sms));
    printf("mix<2> : %.2f checks/clk/SM\n", run<2>(out, blocks, threads, iters, clk, sms));
    printf("mix<3> : %.2f checks/clk/SM\n", run<3>(out, blocks, threads, iters, clk, sms));
    printf("mix<4> : %.2f checks/clk/SM\n", run<4>(out, blocks, threads, iters, clk, sms));
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
