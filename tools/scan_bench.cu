// tools/scan_bench.cu -- development microbenchmark: full-scan throughput of the screen's inner
// loop (true survivors: no candidate dies) for two data layouts, on sm_100a.
//   shfl<R,MIX>  : lane holds R candidates; the warp reads 32 codewords per coalesced load and
//                  broadcasts each by SHFL (the round-1 p_scan)
//   lhc<R,NA,U>  : lane holds ONE codeword per step (coalesced load, no shuffle); the R
//                  candidates are warp-uniform registers; NA of them use the ALU form
//                  (x &= x-1, d-1 times); vote every U steps (32*U codewords)
// Codebook: 8M random 28-bit words in global memory (L2-resident), grid = #SMs x 512 threads,
// each warp scans 2048-codeword sub-ranges.  Prints checks/clk/SM at the current clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/scan_bench tools/scan_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr uint32_t kD = 3;
constexpr int kSub = 2048;

template <int D>
__device__ __forceinline__ uint32_t clear_low(uint32_t x) {
#pragma unroll
    for (int i = 0; i < D - 1; ++i) x &= x - 1u;
    return x;
}

template <int R, int MIX>
__global__ void __launch_bounds__(512, 1) k_shfl(const uint32_t *__restrict__ cb, uint32_t M, int items,
                                                 uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (int it = gw; it < items; it += nw) {
        uint32_t v[R], m[R];
#pragma unroll
        for (int r = 0; r < R; ++r) { v[r] = (it * 64 + r * 32 + lane) * 2654435761u >> 4; m[r] = ~0u; }
        const long long hi = ((long long)it * kSub) % (M - kSub) + kSub, lo = hi - kSub;
        long long top = hi;
        uint32_t cur = __ldcg(cb + top - 1 - lane);
        while (top > lo) {
            const long long ntop = top - 32;
            const uint32_t nxt = ntop > lo ? __ldcg(cb + ntop - 1 - lane) : 0u;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint32_t c = __shfl_sync(0xffffffffu, cur, k);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (MIX && (r & 1)) m[r] = min(m[r], clear_low<MIX>(v[r] ^ c));
                    else m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c));
                }
            }
            bool done = true;
#pragma unroll
            for (int r = 0; r < R; ++r) done &= (MIX && (r & 1)) ? m[r] == 0 : m[r] < kD;
            if (__all_sync(0xffffffffu, done)) break;
            cur = nxt;
            top = ntop;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) acc += m[r];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// R uniform candidates, lane-owned codewords; candidates r < NA use the ALU form
template <int R, int NA, int U>
__global__ void __launch_bounds__(512, 1) k_lhc(const uint32_t *__restrict__ cb, uint32_t M, int items,
                                                uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (int it = gw; it < items; it += nw) {
        uint32_t v[R], m[R];
#pragma unroll
        for (int r = 0; r < R; ++r) { v[r] = (it * R + r) * 2654435761u >> 4; m[r] = ~0u; }
        const long long hi = ((long long)it * kSub) % (M - kSub) + kSub, lo = hi - kSub;
        long long top = hi;
        uint32_t c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = __ldcg(cb + top - 1 - lane - 32 * u);
        while (top > lo) {
            const long long ntop = top - 32 * U;
            uint32_t nx[U];
#pragma unroll
            for (int u = 0; u < U; ++u) nx[u] = ntop > lo ? __ldcg(cb + ntop - 1 - lane - 32 * u) : 0u;
#pragma unroll
            for (int u = 0; u < U; ++u) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r < NA) m[r] = min(m[r], clear_low<kD>(v[r] ^ c[u]));
                    else m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c[u]));
                }
            }
            bool done = true;
#pragma unroll
            for (int r = 0; r < R; ++r) done &= __any_sync(0xffffffffu, r < NA ? m[r] == 0 : m[r] < kD);
            if (done) break;
#pragma unroll
            for (int u = 0; u < U; ++u) c[u] = nx[u];
            top = ntop;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) acc += m[r];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// lane holds R candidates; codewords read by warp-UNIFORM 128-bit loads (4 per load, L1
// broadcast), U loads per block, next block prefetched; ALU form for candidates r with bit r
// of PAT set
template <int R, int PAT, int U>
__global__ void __launch_bounds__(512, 1) k_bcast(const uint32_t *__restrict__ cb, uint32_t M, int items,
                                                  uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (int it = gw; it < items; it += nw) {
        uint32_t v[R], m[R];
#pragma unroll
        for (int r = 0; r < R; ++r) { v[r] = (it * 32 * R + r * 32 + lane) * 2654435761u >> 4; m[r] = ~0u; }
        const long long hi = ((long long)it * kSub) % (M - kSub) + kSub, lo = hi - kSub;
        // blocks of 4U codewords, newest first (hi and lo multiples of 4 here)
        long long top = hi;
        uint4 c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = __ldcg(reinterpret_cast<const uint4 *>(cb + top - 4 * (u + 1)));
        while (top > lo) {
            const long long ntop = top - 4 * U;
            uint4 nx[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                nx[u] = ntop > lo ? __ldcg(reinterpret_cast<const uint4 *>(cb + ntop - 4 * (u + 1))) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t cw[4] = {c[u].w, c[u].z, c[u].y, c[u].x};
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        if ((PAT >> r) & 1) m[r] = min(m[r], clear_low<kD>(v[r] ^ cw[k]));
                        else m[r] = min(m[r], (uint32_t)__popc(v[r] ^ cw[k]));
                    }
            }
            bool done = true;
#pragma unroll
            for (int r = 0; r < R; ++r) done &= ((PAT >> r) & 1) ? m[r] == 0 : m[r] < kD;
            if (__all_sync(0xffffffffu, done)) break;
#pragma unroll
            for (int u = 0; u < U; ++u) c[u] = nx[u];
            top = ntop;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) acc += m[r];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename F>
static void timeit(const char *name, F launch, double checks, double clk, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaDeviceSynchronize();
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double r = checks / (ms * 1e-3) / (sms * clk);
        if (r > best) best = r;
    }
    printf("%-22s %6.2f checks/clk/SM  (%s)\n", name, best, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double clk = clk_khz * 1e3;
    const int sms = p.multiProcessorCount;
    const uint32_t M = 1u << 23;
    uint32_t *cb, *out;
    cudaMalloc(&cb, M * 4ull);
    cudaMalloc(&out, sms * 512 * 4);
    // random 28-bit codewords, all at distance >= 3 from the candidates with high probability
    // is NOT required: the bench never breaks early unless every candidate died
    {
        uint32_t *h = new uint32_t[M];
        uint64_t s = 88172645463325252ull;
        for (uint32_t i = 0; i < M; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)s & 0x0fffffffu; }
        cudaMemcpy(cb, h, M * 4ull, cudaMemcpyHostToDevice);
        delete[] h;
    }
    printf("%s SMs=%d clock=%.0f MHz, d=%u, sub-range %d codewords\n", p.name, sms, clk / 1e6, kD, kSub);
    const int nw = sms * 16;
    const int items = nw * 8;
#define SHFL(R, MIX) timeit("shfl<" #R "," #MIX ">", [&] { k_shfl<R, MIX><<<sms, 512>>>(cb, M, items, out); }, \
                            (double)items * 32 * R * kSub, clk, sms)
#define LHC(R, NA, U) timeit("lhc<" #R "," #NA "," #U ">", [&] { k_lhc<R, NA, U><<<sms, 512>>>(cb, M, items, out); }, \
                             (double)items * R * kSub, clk, sms)
#define BC(R, PAT, U) timeit("bcast<" #R "," #PAT "," #U ">", [&] { k_bcast<R, PAT, U><<<sms, 512>>>(cb, M, items, out); }, \
                            (double)items * 32 * R * kSub, clk, sms)
    BC(2, 0, 8);
    BC(2, 2, 8);
    BC(2, 2, 4);
    BC(2, 2, 16);
    BC(2, 1, 8);
    BC(3, 2, 8);
    BC(3, 5, 8);
    BC(3, 6, 8);
    BC(4, 10, 8);
    BC(4, 8, 8);
    BC(4, 14, 8);
    BC(4, 12, 8);
    BC(1, 0, 8);
    SHFL(2, 0);
    SHFL(2, 3);
    SHFL(4, 3);
    LHC(4, 0, 4);
    LHC(8, 0, 4);
    LHC(8, 4, 4);
    LHC(8, 3, 4);
    LHC(8, 2, 4);
    LHC(8, 4, 8);
    LHC(16, 8, 2);
    LHC(16, 6, 2);
    LHC(12, 4, 4);
    LHC(12, 5, 4);
    LHC(12, 6, 4);
    return 0;
}
