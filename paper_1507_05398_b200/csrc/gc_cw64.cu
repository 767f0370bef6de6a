// gc_cw64.cu -- constant-weight greedy codes on 64-bit words, 33 <= n <= 63 (SURVEY.md Sec. 8(f)
// row 4: "verified the published results on constant weight codes of length up-to 35",
// PAPER.md:240; the problem of PAPER.md:57 restricted to one weight class).
//
// The candidates are the weight-w vectors of F_2^n in ascending value (lex / graded-lex: lex
// restricted to one weight is graded-lex within it) or descending value (graded-revlex), unranked
// directly from their rank in the class (combinatorial number system, 64-bit binomials).  One
// cooperative kernel runs the whole construction: tiles of candidates are screened by every warp
// of the grid against the committed codebook (XOR + 64-bit POPC, newest-first
// warp items with warp-vote early exit), then CTA 0 decides the tile's survivors in rank order
// against the words accepted earlier in the tile and appends them.  Tiles with
// more survivors than one resolve buffer are cut after them (the rest is screened again with
// the next tile): tile boundaries never change the result.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gc_internal.h"

namespace cg = cooperative_groups;

namespace gc {

constexpr int kWThreads = 512;
constexpr int kWWarps = kWThreads / 32;
constexpr uint32_t kWTileMax = 1u << 16;
constexpr uint32_t kWTileMin = 64;
constexpr uint32_t kWMaxS = 1024;           // survivors decided per tile (resolve buffer)
constexpr uint32_t kWSub = 4096;            // codewords per screen work item
constexpr uint32_t kWTargetS = 256;         // tiles sized toward this many survivors

struct WState {
    unsigned long long M, t, tiles, checks, survivors;
    unsigned int K, error;
};

struct WArgs {
    int n, d, w;
    int desc;                               // descending values within the class (graded-revlex)
    unsigned long long total;               // C(n, w) candidates
    unsigned long long nmask;               // 2^n - 1
    const unsigned long long *binom;        // C(p, k), p, k <= 63, [64][64]
    unsigned long long *codebook;           // [capacity]
    unsigned long long capacity;
    unsigned int *kill;                     // [kWTileMax / 32]
    WState *st;
};

// the q-th (0-based) weight-k vector of F_2^n in ascending value: bits p_k > ... > p_1 with
// q = sum_j C(p_j, j) (combinatorial number system)
__device__ __forceinline__ unsigned long long w_unrank(const unsigned long long (*C)[64], int n, int k,
                                                       unsigned long long q) {
    unsigned long long v = 0;
    int p = n - 1;
    for (int j = k; j >= 1; --j) {
        while (C[p][j] > q) --p;
        v |= 1ull << p;
        q -= C[p][j];
        --p;
    }
    return v;
}

__device__ __forceinline__ unsigned long long w_candidate(const WArgs &a, const unsigned long long (*C)[64],
                                                          unsigned long long r) {
    if (!a.desc) return w_unrank(C, a.n, a.w, r);
    // descending weight-w values = complements of the ascending weight-(n - w) values
    return ~w_unrank(C, a.n, a.n - a.w, r) & a.nmask;
}

__global__ void __launch_bounds__(kWThreads, 1) k_cw64(WArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned long long C[64][64];
    __shared__ unsigned long long s_val[kWMaxS];
    __shared__ unsigned char s_acc[kWMaxS];
    __shared__ unsigned int s_ws[kWWarps + 1];
    __shared__ unsigned long long s_t0, s_M;
    __shared__ unsigned int s_K;
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) C[i / 64][i % 64] = a.binom[i];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned gwarp = blockIdx.x * kWWarps + wid, nwarps = gridDim.x * kWWarps;
    unsigned long long my_checks = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            s_t0 = __ldcg(&a.st->t);
            s_K = __ldcg(&a.st->K);
            s_M = __ldcg(&a.st->M);
        }
        __syncthreads();
        const unsigned long long t0 = s_t0, M = s_M;
        if (t0 >= a.total) break;
        const uint32_t K = (uint32_t)min((unsigned long long)s_K, a.total - t0);
        // ---- screen: (batch of 32 candidates) x (newest-first sub-range of kWSub codewords)
        const uint32_t nb = (K + 31) / 32;
        const uint32_t nsub = M ? (uint32_t)((M + kWSub - 1) / kWSub) : 0u;
        for (unsigned long long it = gwarp; it < (unsigned long long)nb * nsub; it += nwarps) {
            const uint32_t b = (uint32_t)(it % nb), j = (uint32_t)(it / nb);
            const uint32_t q = b * 32 + lane;
            const bool live = q < K;
            const unsigned long long v = live ? w_candidate(a, C, t0 + q) : 0ull;
            const long long hi = (long long)M - (long long)j * kWSub, lo = max(0ll, hi - (long long)kWSub);
            int m = live ? 64 : 0;
            for (long long top = hi; top > lo; top -= 32) {
                const long long k = top - 1 - lane;
                const unsigned long long c = k >= lo ? __ldcg(a.codebook + k) : 0ull;
                const int nv = (int)min(32ll, top - lo);
                for (int e = 0; e < nv; ++e) m = min(m, __popcll(v ^ __shfl_sync(0xffffffffu, c, e)));
                my_checks += (unsigned long long)nv;
                if (__all_sync(0xffffffffu, m < a.d)) break;
            }
            const unsigned dead = __ballot_sync(0xffffffffu, live && m < a.d);
            if (lane == 0 && dead) atomicOr(a.kill + b, dead);
        }
        grid.sync();
        // ---- resolve (CTA 0): survivors in rank order, decided against the tile's accepted words
        if (blockIdx.x == 0) {
            __shared__ unsigned int s_cut;
            if (threadIdx.x == 0) s_cut = K;
            __syncthreads();
            // ordered gather: one pass per 32-candidate word, a block-wide scan of the counts
            unsigned int base = 0;
            for (uint32_t w0 = 0; w0 < nb; w0 += blockDim.x) {
                const uint32_t wi = w0 + threadIdx.x;
                unsigned int alive = 0;
                if (wi < nb) {
                    alive = ~__ldcg(a.kill + wi);
                    if (wi * 32 + 32 > K) alive &= (1u << (K - wi * 32)) - 1u;
                }
                const unsigned int cnt = __popc(alive);
                unsigned int inc = cnt;
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                if (lane == 31) s_ws[wid] = inc;
                __syncthreads();
                if (wid == 0) {
                    unsigned int x = lane < kWWarps ? s_ws[lane] : 0u, xi = x;
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned int y = __shfl_up_sync(0xffffffffu, xi, o);
                        if (lane >= o) xi += y;
                    }
                    if (lane < kWWarps) s_ws[lane] = xi - x;
                    if (lane == 31) s_ws[kWWarps] = xi;
                }
                __syncthreads();
                unsigned int pos = base + s_ws[wid] + inc - cnt;
                while (alive) {
                    const int bit = __ffs(alive) - 1;
                    alive &= alive - 1;
                    const uint32_t i = wi * 32 + bit;
                    if (pos < kWMaxS) s_val[pos] = w_candidate(a, C, t0 + i);
                    else if (pos == kWMaxS) s_cut = i;        // first survivor left for the next tile
                    ++pos;
                }
                base += s_ws[kWWarps];
                __syncthreads();
            }
            const uint32_t S = min(base, kWMaxS);
            const uint32_t K_used = base > kWMaxS ? s_cut : K;
            // warp 0: survivors in rank order; accepted iff no earlier ACCEPTED survivor of the
            // tile is closer than d (the screen removed those with a committed word closer)
            if (wid == 0) {
                unsigned int A = 0;
                for (uint32_t j = 0; j < S; ++j) {
                    const unsigned long long v = s_val[j];
                    bool conflict = false;
                    for (uint32_t k = lane; k < j; k += 32)
                        conflict |= s_acc[k] && __popcll(v ^ s_val[k]) < a.d;
                    conflict = __any_sync(0xffffffffu, conflict);
                    if (lane == 0) s_acc[j] = conflict ? 0 : 1;
                    A += conflict ? 0u : 1u;
                    __syncwarp();
                }
                // ordered append
                unsigned int pos = 0;
                for (uint32_t j0 = 0; j0 < S; j0 += 32) {
                    const uint32_t j = j0 + lane;
                    const bool acc = j < S && s_acc[j];
                    const unsigned bal = __ballot_sync(0xffffffffu, acc);
                    if (acc) {
                        const unsigned long long p = M + pos + __popc(bal & ((1u << lane) - 1u));
                        if (p < a.capacity) a.codebook[p] = s_val[j];
                        else a.st->error = 1;
                    }
                    pos += __popc(bal);
                }
                if (lane == 0) {
                    const unsigned long long M1 = min(M + A, a.capacity);
                    WState *st = a.st;
                    st->M = M1;
                    st->t = t0 + K_used;
                    st->tiles += 1;
                    st->survivors += S;
                    // next tile: toward kWTargetS survivors, a power of two in [kWTileMin, kWTileMax]
                    unsigned long long want = S ? (unsigned long long)K_used * kWTargetS / S : 2ull * K;
                    uint32_t Kn = kWTileMin;
                    while (Kn < kWTileMax && (unsigned long long)Kn * 2 <= want && Kn < 2 * K) Kn <<= 1;
                    st->K = Kn;
                }
            }
            for (uint32_t wi = threadIdx.x; wi < nb; wi += blockDim.x) a.kill[wi] = 0;
        }
        __threadfence();
        grid.sync();
    }
    for (int o = 16; o > 0; o >>= 1) my_checks += __shfl_down_sync(0xffffffffu, my_checks, o);
    if (lane == 0 && my_checks) atomicAdd(&a.st->checks, my_checks);
}

// ------------------------------------------------------------------ host side

#define WCK(call)                                                                             \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
            return e_ == cudaErrorMemoryAllocation ? GC_ENOMEM : GC_ECUDA;                   \
        }                                                                                     \
    } while (0)

namespace {
struct WContext {
    unsigned long long *binom = nullptr, *cb = nullptr;
    unsigned long long cb_cap = 0;
    unsigned int *kill = nullptr;
    WState *st = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::mutex mu;
};
std::mutex g_wmu;
WContext *g_wctx[64];
}  // namespace

bool cw64_supported(const RunArgs &a) {
    return a.constant_weight >= 0 && !a.use_basis && !a.self_orthogonal && a.world == 1 &&
           (a.ordering == GC_LEX || a.ordering == GC_GRADED_LEX || a.ordering == GC_GRADED_REVLEX) && a.n <= 63;
}

int cw64_run(const RunArgs &r, uint64_t *out_codewords, uint64_t *out_count, gc_stats *stats) {
    int device;
    WCK(cudaGetDevice(&device));
    WContext *cx;
    {
        std::lock_guard<std::mutex> g(g_wmu);
        if (device < 0 || device >= 64) { set_error("device index out of range"); return GC_EINVAL; }
        if (!g_wctx[device]) {
            WContext *c = new WContext;
            WCK(cudaMalloc(&c->binom, 64 * 64 * sizeof(unsigned long long)));
            WCK(cudaMalloc(&c->kill, kWTileMax / 32 * sizeof(unsigned int)));
            WCK(cudaMalloc(&c->st, sizeof(WState)));
            WCK(cudaEventCreate(&c->ev0));
            WCK(cudaEventCreate(&c->ev1));
            std::vector<unsigned long long> C(64 * 64, 0);
            for (int p = 0; p < 64; ++p) {
                C[p * 64] = 1;
                for (int k = 1; k <= p && k < 64; ++k) C[p * 64 + k] = C[(p - 1) * 64 + k - 1] + (k < p ? C[(p - 1) * 64 + k] : 0);
            }
            WCK(cudaMemcpy(c->binom, C.data(), C.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
            g_wctx[device] = c;
        }
        cx = g_wctx[device];
    }
    std::lock_guard<std::mutex> lock(cx->mu);
    const int n = (int)r.n, w = r.constant_weight;
    // C(n, w) with n <= 63: exact in 64 bits (C(63, 31) < 2^63), by Pascal's rule
    std::vector<unsigned long long> row(64, 0);
    row[0] = 1;
    for (int p = 1; p <= n; ++p)
        for (int k = std::min(p, 63); k >= 1; --k) row[k] += row[k - 1];
    const unsigned long long total = row[w];
    const unsigned long long cap_host = *out_count;
    const unsigned long long cap = std::min<unsigned long long>(total, 1ull << 27);   // device buffer (1 GiB max)
    if (cx->cb_cap < cap) {
        if (cx->cb) WCK(cudaFree(cx->cb));
        cx->cb = nullptr;
        cx->cb_cap = 0;
        WCK(cudaMalloc(&cx->cb, cap * sizeof(unsigned long long)));
        cx->cb_cap = cap;
    }
    cudaStream_t s = (cudaStream_t)r.stream;
    WState h{};
    h.K = kWTileMin;
    WCK(cudaMemcpyAsync(cx->st, &h, sizeof h, cudaMemcpyHostToDevice, s));
    WCK(cudaMemsetAsync(cx->kill, 0, kWTileMax / 32 * sizeof(unsigned int), s));
    WArgs a;
    a.n = n; a.d = (int)r.d; a.w = w;
    a.desc = r.ordering == GC_GRADED_REVLEX;
    a.total = total;
    a.nmask = (1ull << n) - 1ull;
    a.binom = cx->binom;
    a.codebook = cx->cb;
    a.capacity = cap;
    a.kill = cx->kill;
    a.st = cx->st;
    int sms = 0, per_sm = 0;
    WCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    WCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cw64, kWThreads, 0));
    if (per_sm < 1) { set_error("k_cw64 cannot be resident"); return GC_ECUDA; }
    void *args[] = {&a};
    WCK(cudaEventRecord(cx->ev0, s));
    WCK(cudaLaunchCooperativeKernel((const void *)k_cw64, dim3(sms), dim3(kWThreads), args, 0, s));
    WCK(cudaEventRecord(cx->ev1, s));
    WCK(cudaMemcpyAsync(&h, cx->st, sizeof h, cudaMemcpyDeviceToHost, s));
    WCK(cudaStreamSynchronize(s));
    if (h.error) { *out_count = h.M + 1; set_error("constant-weight codebook exceeds 2^27 words"); return GC_ENOSPC; }
    *out_count = h.M;
    if (h.M > cap_host) { set_error("output buffer too small"); return GC_ENOSPC; }
    if (h.M) WCK(cudaMemcpy(out_codewords, cx->cb, h.M * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    if (stats) {
        float ms = 0;
        WCK(cudaEventElapsedTime(&ms, cx->ev0, cx->ev1));
        gc_stats *o = stats;
        const uint32_t sz = o->struct_size;
        memset(o, 0, sizeof *o);
        o->struct_size = sz ? sz : sizeof(gc_stats);
        o->n_ranks = 1;
        o->device_ms = ms;
        o->screen_ms = ms;
        o->M = h.M;
        o->tiles = h.tiles;
        o->phases = h.tiles;
        o->checks_exec = h.checks;
        o->survivors = h.survivors;
        o->launches = 1;
        o->screen_launches = 1;
    }
    return GC_OK;
}

}  // namespace gc
