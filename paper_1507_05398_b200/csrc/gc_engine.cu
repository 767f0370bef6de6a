// gc_engine.cu -- the B200 (sm_100a) hot path of the greedy code construction
// (Sec. 4; inner check PAPER.md:71/73 Sec. 4.1; XOR+popcount PAPER.md:155).
//
// One construction scans ranks 0 .. 2^n-1 in TILES of K consecutive candidates
// (SURVEY.md Sec. 8(a)).  Per tile, all enqueued on one stream, no host round trip:
//
//   k_gen_tile        a1: rank -> vector for the K candidates (gc_order.cuh)
//   k_screen  x P     a2/a2': every candidate against the codebook committed before the
//                     tile, NEWEST FIRST, in geometrically growing windows
//                     [M-W0,M), [M-3W0,M-W0), [M-7W0,M-3W0), ... the last one down to 0;
//                     XOR + POPC + min per check, warp-vote early exit, a candidate is
//                     dropped from later windows as soon as one codeword is closer than d
//   k_compact x P-1   survivors of a window -> dense list for the next window
//   k_gather          survivors of the tile in rank order
//   k_edges           all survivor pairs at distance < d (multi-CTA)
//   k_commit          a3/a4: in-tile ordered resolve (lexicographically-first maximal
//                     independent set of the conflict graph, computed in rounds) and
//                     append to the codebook in rank order; M += accepted
//
// The "selective kernel launch" of PAPER.md:159 (first 10% of the output, then the
// rest) is the two-window special case of the window schedule; here the windows start
// at the NEWEST codewords (which reject most candidates) and grow
// geometrically, so a rejected candidate costs at most ~2x its first-witness depth.
// None of this changes the result: a candidate is accepted iff it is at distance >= d
// from every codeword accepted before it (the tile's own earlier survivors included).
//
// Multi-GPU (gc_generate_rank): each rank screens 1/world of every tile's candidates
// against its replicated codebook; the K-bit dead masks are all-gathered (NCCL) once
// per tile; gather/edges/commit then run redundantly and identically on every rank.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gc_internal.h"
#include "gc_order.cuh"

namespace gc {

// ------------------------------------------------------------------ constants
constexpr int kScreenThreads = 128;   // threads per screen CTA
constexpr int kScreenR = 2;           // candidates per thread
constexpr int kScreenCB = kScreenThreads * kScreenR;   // candidates per work item
constexpr int kChunk = 1024;          // codewords per work item (4 KiB of smem)
constexpr int kMaxPhases = 40;
constexpr int kMaxParts = 64;
constexpr uint32_t kEdgeCap = 1u << 22;   // in-tile conflict edges (32 MiB)
constexpr int kResolveThreads = 1024;
constexpr int kEdgeBlock = 128;

// Device-resident counters of one construction.
struct DevCounters {
    unsigned long long M;               // committed codewords
    unsigned long long checks_exec;     // screen lane-checks executed
    unsigned long long survivors;
    unsigned long long conflicts;
    unsigned long long resolve_checks;
    unsigned long long w_def;           // sum over accepted of (2^n - 1 - rank)
    unsigned int S;                     // survivors of the current tile
    unsigned int E;                     // conflict edges of the current tile
    unsigned int edge_overflow;
    unsigned int error;                 // 1 = capacity exceeded
    unsigned int list_count[kMaxParts * kMaxPhases];
    unsigned long long phase_checks[kMaxPhases];   // diagnostics (GC_DEBUG_PHASES)
    unsigned long long phase_alive[kMaxPhases];
};

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
            return e_ == cudaErrorMemoryAllocation ? GC_ENOMEM : GC_ECUDA;                   \
        }                                                                                     \
    } while (0)

// ================================================================== kernels

// a1: vals[i] = vector of rank t0 + i (i < K); mask the padding i in [K, Kpad) as dead.
__global__ void k_gen_tile(const OrderTables *__restrict__ tab, int ord, int n, unsigned long long t0,
                           uint32_t K, uint32_t Kpad, uint32_t *__restrict__ vals, uint32_t *__restrict__ dead,
                           DevCounters *ctr) {
    __shared__ uint32_t C[33][33];
    __shared__ uint64_t off[34];
    if (ord >= GRADED_LEX) {
        for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) C[i / 33][i % 33] = tab->binom[i / 33][i % 33];
        for (int i = threadIdx.x; i < 34; i += blockDim.x) off[i] = tab->off[i];
        __syncthreads();
    }
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    for (uint32_t i = tid; i < Kpad; i += stride)
        vals[i] = i < K ? rank_to_vector32(ord, n, C, off, t0 + i) : 0u;
    const uint32_t words = Kpad / 32;
    for (uint32_t w = tid; w < words; w += stride) {
        uint32_t lo = w * 32, m = 0;
        if (lo + 32 > K) m = (lo >= K) ? 0xffffffffu : (0xffffffffu << (K - lo));
        dead[w] = m;
    }
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < kMaxParts * kMaxPhases; i += blockDim.x) ctr->list_count[i] = 0;
        if (threadIdx.x == 0) { ctr->S = 0; ctr->E = 0; ctr->edge_overflow = 0; }
    }
}

// a2: screen a list of candidates against the codebook window of phase p.
//   list == nullptr: the implicit list idx = part_lo + i, i < part_n (phase 0)
//   window: newest-first positions [b_p, b_{p+1}) with b_p = W0 (2^p - 1); last phase to 0.
// Work item = (block of kScreenCB candidates) x (chunk of kChunk codewords).
__global__ void __launch_bounds__(kScreenThreads)
k_screen(int p, int P, uint32_t W0, int growth, bool early_exit, const uint32_t *__restrict__ codebook,
         const uint32_t *__restrict__ vals, const uint2 *__restrict__ list, const unsigned int *list_count,
         uint32_t part_lo, uint32_t part_n, uint32_t *dead, DevCounters *ctr, uint32_t d) {
    __shared__ __align__(16) uint32_t cw[kChunk];
    const long long M = (long long)ctr->M;
    long long hi, lo;
    if (!early_exit) {
        hi = M; lo = 0;
    } else {
        long long bp = 0, w = W0;
        for (int i = 0; i < p; ++i) { bp += w; w <<= growth; }
        const long long bq = bp + w;
        hi = M - bp;
        lo = (p == P - 1) ? 0 : M - bq;
        if (lo < 0) lo = 0;
    }
    if (hi <= lo) return;
    const uint32_t L = list ? *list_count : part_n;
    if (L == 0) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&ctr->phase_alive[p], (unsigned long long)L);
    const uint32_t wlen = (uint32_t)(hi - lo);
    const uint32_t nchunks = (wlen + kChunk - 1) / kChunk;
    const uint32_t ncb = (L + kScreenCB - 1) / kScreenCB;
    const unsigned long long nitems = (unsigned long long)nchunks * ncb;
    const int lane = threadIdx.x & 31;
    unsigned long long my_checks = 0;

    for (unsigned long long item = blockIdx.x; item < nitems; item += gridDim.x) {
        const uint32_t chunk = (uint32_t)(item % nchunks);          // chunk 0 = newest
        const uint32_t cb = (uint32_t)(item / nchunks);
        const long long c_hi = hi - (long long)chunk * kChunk;
        const long long c_lo = max(lo, c_hi - kChunk);
        const uint32_t len = (uint32_t)(c_hi - c_lo);
        // stage the chunk in shared memory (coalesced); pad to a multiple of 4 with a
        // duplicate codeword (a duplicate cannot change a minimum)
        for (uint32_t i = threadIdx.x; i < kChunk; i += kScreenThreads) {
            uint32_t src = i < len ? i : 0;
            if (i < ((len + 3) & ~3u)) cw[i] = codebook[c_lo + src];
        }
        __syncthreads();

        uint32_t v[kScreenR], m[kScreenR], idx[kScreenR];
        bool live[kScreenR];
#pragma unroll
        for (int r = 0; r < kScreenR; ++r) {
            const uint32_t li = cb * kScreenCB + r * kScreenThreads + threadIdx.x;
            live[r] = li < L;
            if (live[r]) {
                if (list) { uint2 e = list[li]; idx[r] = e.x; v[r] = e.y; }
                else { idx[r] = part_lo + li; v[r] = vals[idx[r]]; }
                live[r] = !((dead[idx[r] >> 5] >> (idx[r] & 31)) & 1u);
            } else {
                idx[r] = 0; v[r] = 0;
            }
            m[r] = live[r] ? 64u : 0u;
        }
        const uint4 *cw4 = reinterpret_cast<const uint4 *>(cw);
        const int ng = (int)((len + 3) >> 2);
        int g = ng - 1;
        // newest first: highest index in the chunk first
        for (; g >= 0; --g) {
            if (early_exit && ((g & 7) == 7 || g == ng - 1)) {
                bool done = true;
#pragma unroll
                for (int r = 0; r < kScreenR; ++r) done &= (m[r] < d);
                if (__all_sync(0xffffffffu, done)) break;
            }
            const uint4 c = cw4[g];
#pragma unroll
            for (int r = 0; r < kScreenR; ++r) {
                m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c.x));
                m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c.y));
                m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c.z));
                m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c.w));
            }
        }
        if (lane == 0) my_checks += (unsigned long long)(ng - 1 - g) * 4 * 32 * kScreenR;
#pragma unroll
        for (int r = 0; r < kScreenR; ++r) {
            const bool kill = live[r] && m[r] < d;
            if (!list) {
                // implicit list: the warp's 32 candidates are one aligned mask word
                const unsigned b = __ballot_sync(0xffffffffu, kill);
                if (lane == 0 && b) atomicOr(&dead[idx[r] >> 5], b);
            } else if (kill) {
                atomicOr(&dead[idx[r] >> 5], 1u << (idx[r] & 31));
            }
        }
        __syncthreads();   // before the next item overwrites cw
    }
    if (lane == 0 && my_checks) {
        atomicAdd(&ctr->checks_exec, my_checks);
        atomicAdd(&ctr->phase_checks[p], my_checks);
    }
}

// survivors of a window -> dense list for the next window (order irrelevant here)
__global__ void k_compact(const uint32_t *__restrict__ vals, const uint2 *__restrict__ list_in,
                          const unsigned int *count_in, uint32_t part_lo, uint32_t part_n,
                          const uint32_t *__restrict__ dead, uint2 *__restrict__ list_out, unsigned int *count_out) {
    const uint32_t L = list_in ? *count_in : part_n;
    const int lane = threadIdx.x & 31;
    for (uint32_t base = blockIdx.x * blockDim.x; base < L; base += gridDim.x * blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        uint2 e = make_uint2(0, 0);
        bool alive = false;
        if (i < L) {
            if (list_in) e = list_in[i];
            else { e.x = part_lo + i; e.y = vals[e.x]; }
            alive = !((dead[e.x >> 5] >> (e.x & 31)) & 1u);
        }
        const unsigned b = __ballot_sync(0xffffffffu, alive);
        unsigned pos = 0;
        if (lane == 0 && b) pos = atomicAdd(count_out, __popc(b));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (alive) list_out[pos + __popc(b & ((1u << lane) - 1u))] = e;
    }
}

// block-wide exclusive scan of one value per thread (blockDim.x == kResolveThreads)
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t *total, uint32_t *warp_sums) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u, si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += y;
        }
        if (lane < (int)(blockDim.x >> 5)) warp_sums[lane] = si - s;
        if (lane == 31) warp_sums[32] = si;
    }
    __syncthreads();
    const uint32_t res = warp_sums[wid] + inc - x;
    *total = warp_sums[32];
    __syncthreads();
    return res;
}

// survivors of the tile, in rank order: surv[j] = (tile index, vector)
__global__ void __launch_bounds__(kResolveThreads)
k_gather(uint32_t Kpad, const uint32_t *__restrict__ dead, const uint32_t *__restrict__ vals,
         uint2 *__restrict__ surv, DevCounters *ctr) {
    __shared__ uint32_t ws[33];
    const uint32_t words = Kpad / 32;
    uint32_t base = 0;
    for (uint32_t w0 = 0; w0 < words; w0 += kResolveThreads) {
        const uint32_t w = w0 + threadIdx.x;
        uint32_t alive = w < words ? ~dead[w] : 0u;
        uint32_t tot;
        uint32_t pos = base + block_exclusive_scan(__popc(alive), &tot, ws);
        while (alive) {
            const int b = __ffs(alive) - 1;
            alive &= alive - 1;
            const uint32_t i = w * 32 + b;
            surv[pos++] = make_uint2(i, vals[i]);
        }
        base += tot;
    }
    if (threadIdx.x == 0) { ctr->S = base; ctr->survivors += base; }
}

// all survivor pairs k < j at distance < d -> edges (k, j)
__global__ void __launch_bounds__(kEdgeBlock)
k_edges(const uint2 *__restrict__ surv, uint2 *__restrict__ edges, uint32_t d, DevCounters *ctr) {
    __shared__ uint32_t kv[kEdgeBlock];
    const uint32_t S = ctr->S;
    if (S < 2) return;
    const uint32_t nb = (S + kEdgeBlock - 1) / kEdgeBlock;
    const unsigned long long npairs = (unsigned long long)nb * (nb + 1) / 2;
    unsigned long long my_checks = 0;
    for (unsigned long long x = blockIdx.x; x < npairs; x += gridDim.x) {
        // decode lower-triangular block pair (bj >= bk)
        uint32_t bj = (uint32_t)((sqrt(8.0 * (double)x + 1.0) - 1.0) / 2.0);
        while ((unsigned long long)(bj + 1) * (bj + 2) / 2 <= x) ++bj;
        while ((unsigned long long)bj * (bj + 1) / 2 > x) --bj;
        const uint32_t bk = (uint32_t)(x - (unsigned long long)bj * (bj + 1) / 2);
        const uint32_t k0 = bk * kEdgeBlock;
        const uint32_t kn = min((uint32_t)kEdgeBlock, S - k0);
        if (threadIdx.x < kn) kv[threadIdx.x] = surv[k0 + threadIdx.x].y;
        __syncthreads();
        const uint32_t j = bj * kEdgeBlock + threadIdx.x;
        if (j < S) {
            const uint32_t vj = surv[j].y;
            const uint32_t kend = min(kn, j > k0 ? j - k0 : 0u);
            for (uint32_t t = 0; t < kend; ++t) {
                if ((uint32_t)__popc(vj ^ kv[t]) < d) {
                    const uint32_t e = atomicAdd(&ctr->E, 1u);
                    if (e < kEdgeCap) edges[e] = make_uint2(k0 + t, j);
                    else ctr->edge_overflow = 1;
                }
            }
            my_checks += kend;
        }
        __syncthreads();
    }
    // one atomic per warp
    for (int o = 16; o > 0; o >>= 1) my_checks += __shfl_down_sync(0xffffffffu, my_checks, o);
    if ((threadIdx.x & 31) == 0 && my_checks) atomicAdd(&ctr->resolve_checks, my_checks);
}

enum : uint8_t { UNDEC = 0, ACC = 1, REJ = 2 };

// a3 + a4: ordered resolve of the tile's survivors and commit to the codebook.
// Accept s_j iff no ACCEPTED s_k (k < j) is at distance < d (PAPER.md:59 applied inside
// the tile; Example 1, is the K = 1 case).
__global__ void __launch_bounds__(kResolveThreads)
k_commit(const uint2 *__restrict__ surv, const uint2 *__restrict__ edges, uint8_t *status, uint8_t *blocked,
         uint32_t *codebook, unsigned long long capacity, uint32_t d, unsigned long long t0,
         unsigned long long Nm1, bool force_seq, DevCounters *ctr, unsigned long long tile_index,
         volatile unsigned long long *host_latest) {
    __shared__ uint32_t ws[33];
    __shared__ unsigned long long s_wdef;
    const uint32_t S = ctr->S, E = ctr->E;
    const unsigned long long M0 = ctr->M;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) s_wdef = 0;
    uint32_t A = 0;

    if (force_seq || ctr->edge_overflow) {
        // sequential fallback (exact, slow): candidate by candidate against the tile's accepted list
        __shared__ uint32_t sA;
        if (tid == 0) sA = 0;
        __syncthreads();
        for (uint32_t j = 0; j < S; ++j) {
            const uint2 e = surv[j];
            const uint32_t a = sA;
            bool conflict = false;
            for (uint32_t t = tid; t < a; t += kResolveThreads)
                conflict |= (uint32_t)__popc(e.y ^ codebook[M0 + t]) < d;
            conflict = __syncthreads_or(conflict);
            if (tid == 0 && !conflict) {
                if (M0 + a < capacity) codebook[M0 + a] = e.y;
                else ctr->error = 1;
                sA = a + 1;
                s_wdef += Nm1 - (t0 + e.x);
            }
            __syncthreads();
        }
        A = sA;
    } else {
        for (uint32_t j = tid; j < S; j += kResolveThreads) { status[j] = E ? UNDEC : ACC; blocked[j] = 0; }
        __syncthreads();
        if (E) {
            // rounds: an undecided node is accepted once all its earlier neighbours are
            // decided and none is accepted; rejected as soon as one earlier neighbour is accepted.
            int any;
            do {
                for (uint32_t e = tid; e < E; e += kResolveThreads) {
                    const uint2 kj = edges[e];
                    const uint8_t sk = status[kj.x];
                    if (sk == ACC) status[kj.y] = REJ;
                    else if (sk == UNDEC) blocked[kj.y] = 1;
                }
                __syncthreads();
                any = 0;
                for (uint32_t j = tid; j < S; j += kResolveThreads) {
                    if (status[j] == UNDEC) {
                        if (!blocked[j]) status[j] = ACC;
                        else any = 1;
                    }
                    blocked[j] = 0;
                }
                any = __syncthreads_or(any);
            } while (any);
            if (tid == 0) ctr->conflicts += E;
        }
        // ordered append of the accepted survivors
        unsigned long long wdef = 0;
        for (uint32_t j0 = 0; j0 < S; j0 += kResolveThreads) {
            const uint32_t j = j0 + tid;
            const uint32_t acc = (j < S && status[j] == ACC) ? 1u : 0u;
            uint32_t tot;
            const uint32_t pos = A + block_exclusive_scan(acc, &tot, ws);
            if (acc) {
                const uint2 e = surv[j];
                if (M0 + pos < capacity) codebook[M0 + pos] = e.y;
                else ctr->error = 1;
                wdef += Nm1 - (t0 + e.x);
            }
            A += tot;
        }
        if (wdef) atomicAdd(&s_wdef, wdef);
        __syncthreads();
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long M1 = M0 + A;
        if (M1 > capacity) M1 = capacity;
        ctr->M = M1;
        ctr->w_def += s_wdef;
        if (host_latest) *host_latest = (M1 << 24) | ((tile_index + 1) & 0xffffffull);
    }
}

__global__ void k_finish(const DevCounters *ctr, unsigned long long *d_count, unsigned long long capacity) {
    *d_count = ctr->error ? capacity + 1 : ctr->M;     // above capacity: incomplete code (gc.h)
}

__global__ void k_unrank(const OrderTables *__restrict__ tab, int ord, int n, unsigned long long first,
                         unsigned long long count, uint32_t *__restrict__ out) {
    __shared__ uint32_t C[33][33];
    __shared__ uint64_t off[34];
    for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) C[i / 33][i % 33] = tab->binom[i / 33][i % 33];
    for (int i = threadIdx.x; i < 34; i += blockDim.x) off[i] = tab->off[i];
    __syncthreads();
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < count;
         i += (unsigned long long)gridDim.x * blockDim.x)
        out[i] = rank_to_vector32(ord, n, C, off, first + i);
}

// ============================================================ host: context

struct DeviceContext {
    int device = -1;
    int sm_count = 148;
    uint32_t tile_cap = 0;     // allocated for tiles up to this K
    uint32_t *vals = nullptr, *dead = nullptr;
    uint2 *list[2] = {nullptr, nullptr};
    uint2 *surv = nullptr, *edges = nullptr;
    uint8_t *status = nullptr, *blocked = nullptr;
    DevCounters *ctr = nullptr;
    OrderTables *tabs = nullptr;   // device copy
    int tabs_n = -1;
    unsigned long long *host_latest = nullptr;       // pinned, mapped
    unsigned long long *host_latest_dev = nullptr;   // its device alias
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> tev;   // GC_FLAG_KERNEL_TIMING event pool (pairs)
    std::mutex mu;

    int timing_event(size_t i, cudaEvent_t *e) {
        while (tev.size() <= i) {
            cudaEvent_t x;
            CK(cudaEventCreate(&x));
            tev.push_back(x);
        }
        *e = tev[i];
        return GC_OK;
    }

    void release() {
        cudaFree(vals); cudaFree(dead); cudaFree(list[0]); cudaFree(list[1]);
        cudaFree(surv); cudaFree(edges); cudaFree(status); cudaFree(blocked);
        vals = dead = nullptr; list[0] = list[1] = nullptr; surv = edges = nullptr;
        status = blocked = nullptr; tile_cap = 0;
    }
    int ensure(uint32_t K) {
        if (!ctr) {
            CK(cudaMalloc(&ctr, sizeof(DevCounters)));
            CK(cudaMalloc(&tabs, sizeof(OrderTables)));
            CK(cudaHostAlloc(&host_latest, sizeof(unsigned long long), cudaHostAllocMapped));
            CK(cudaHostGetDevicePointer(&host_latest_dev, host_latest, 0));
            CK(cudaEventCreate(&ev0));
            CK(cudaEventCreate(&ev1));
            CK(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device));
            CK(cudaMalloc(&edges, (size_t)kEdgeCap * sizeof(uint2)));
        }
        if (K <= tile_cap) return GC_OK;
        cudaFree(vals); cudaFree(dead); cudaFree(list[0]); cudaFree(list[1]);
        cudaFree(surv); cudaFree(status); cudaFree(blocked);
        tile_cap = 0;
        CK(cudaMalloc(&vals, (size_t)K * 4));
        CK(cudaMalloc(&dead, (size_t)K / 8 + 4));
        CK(cudaMalloc(&list[0], (size_t)K * sizeof(uint2)));
        CK(cudaMalloc(&list[1], (size_t)K * sizeof(uint2)));
        CK(cudaMalloc(&surv, (size_t)K * sizeof(uint2)));
        CK(cudaMalloc(&status, K));
        CK(cudaMalloc(&blocked, K));
        tile_cap = K;
        return GC_OK;
    }
};

static std::mutex g_ctx_mu;
static std::map<int, std::unique_ptr<DeviceContext>> g_ctx;

static DeviceContext *context_for(int device) {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    auto &p = g_ctx[device];
    if (!p) { p.reset(new DeviceContext); p->device = device; }
    return p.get();
}

// tile size for the tile starting at rank t0 (host-side, deterministic)
static uint32_t tile_size(const Options &o, unsigned long long t0) {
    uint32_t K = o.tile_min;
    while (K < o.tile_max && (unsigned long long)K * 8 <= t0) K <<= 1;
    return K;
}

static int phases_for(unsigned long long M_ub, uint32_t W0, uint32_t growth) {
    if (M_ub == 0) return 0;
    int P = 1;
    unsigned long long depth = W0, w = W0;
    while (P < kMaxPhases && depth < M_ub) { w <<= growth; depth += w; ++P; }
    return P;
}

// ============================================================== host: engine

int engine_run(const RunArgs &a_in) {
    auto wall0 = std::chrono::steady_clock::now();
    // Engine choice by measurement (profiles/r02ap_knob_engines.log): d = 3 codes in lexicographic
    // or Gray order up to n = 25 on one rank run on the tile-barrier engine, whose tiles are cut after
    // 512 survivors (24,3,lex 81 -> 61 ms, 24,3,gray 91 -> 71 ms); from n = 26 the pipelined engine
    // wins (28,3,lex 590 vs 810 ms).  GC_FLAG_PIPELINED keeps the pipelined engine.
    RunArgs a = a_in;
    if (!(a.opt.flags & (GC_FLAG_PIPELINED | GC_FLAG_TILE_BARRIERS)) && a.world <= 1 && a.opt.emulate_ranks <= 1 &&
        !a.extended() && (a.ordering == GC_LEX || a.ordering == GC_GRAY) && a.d == 3 && a.n <= 25)
        a.opt.flags |= GC_FLAG_TILE_BARRIERS;
    // default: the pipelined engine (one GPU, emulated ranks, or one rank per GPU with attached
    // peers); then the tile-barrier engines (GC_FLAG_TILE_BARRIERS, or ranks without peers)
    if (pipeline_supported(a)) {
        int rc = pipeline_run(a);
        if (a.stats) a.stats->wall_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
        return rc;
    }
    if (persistent_partitioned_supported(a)) {
        int rc = persistent_run_partitioned(a);
        if (a.stats) a.stats->wall_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
        return rc;
    }
    if (a.extended() && !pipeline_supported(a) && !persistent_supported(a)) {
        set_error("B-ordering / self-orthogonal / constant-weight problems run on the persistent engines "
                  "only (not with launched tiles, no-early-exit or sequential-resolve flags)");
        return GC_EUNSUPPORTED;
    }
    if (persistent_supported(a)) {
        int rc = persistent_run(a);
        if (a.stats) a.stats->wall_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
        return rc;
    }
    int device;
    CK(cudaGetDevice(&device));
    DeviceContext *cx = context_for(device);
    std::lock_guard<std::mutex> lock(cx->mu);
    cudaStream_t st = (cudaStream_t)a.stream;
    Options o = a.opt;
    if (!o.tile_max) o.tile_max = 65536;
    if (o.tile_min > o.tile_max) o.tile_min = o.tile_max;
    const unsigned parts_local = (a.world > 1) ? 1u : o.emulate_ranks;   // partitions screened here
    const unsigned G = (a.world > 1) ? (unsigned)a.world : o.emulate_ranks; // partitions per tile
    const uint32_t Kpad_max = std::max<uint32_t>(o.tile_max, 32u * G);
    int rc = cx->ensure(Kpad_max);
    if (rc) return rc;
    if (cx->tabs_n != (int)a.n) {
        OrderTables t;
        build_order_tables((int)a.n, &t);
        CK(cudaMemcpy(cx->tabs, &t, sizeof t, cudaMemcpyHostToDevice));
        cx->tabs_n = (int)a.n;
    }
    CK(cudaMemsetAsync(cx->ctr, 0, sizeof(DevCounters), st));
    *cx->host_latest = 0;

    const unsigned long long N = 1ull << a.n;
    const bool early = !(o.flags & GC_FLAG_NO_EARLY_EXIT);
    const bool force_seq = (o.flags & GC_FLAG_FORCE_SEQ_RESOLVE) != 0;
    const int screen_grid = cx->sm_count * 8;
    const int edge_grid = cx->sm_count * 8;
    const unsigned long long cap_bound = a.capacity;
    std::vector<unsigned long long> tile_end;   // ranks covered after each tile
    unsigned long long phases_total = 0, launches = 0, screen_launches = 0;
    const bool timing = (o.flags & GC_FLAG_KERNEL_TIMING) != 0;
    size_t nev = 0;

    CK(cudaEventRecord(cx->ev0, st));
    unsigned long long t0 = 0, tile = 0;
    while (t0 < N) {
        uint32_t K = tile_size(o, t0);
        if ((unsigned long long)K > N - t0) K = (uint32_t)(N - t0);
        uint32_t Kpad = 0, part = 0, plo0 = 0;
        if (gc_tile_partition(K, (int)G, 0, &plo0, &part, &Kpad) != GC_OK) return GC_EINTERNAL;
        // upper bound on M before this tile: last completed tile's M + ranks since
        // (multi-process: only the deterministic bound, so every rank launches the same
        // phases and the same collectives; the last phase always reaches codeword 0, so
        // the bound only affects efficiency, never the result)
        unsigned long long M_ub = std::min(t0, cap_bound);
        const unsigned long long lat = (a.world > 1) ? 0ull : *(volatile unsigned long long *)cx->host_latest;
        if (lat) {
            const unsigned long long done = (lat & 0xffffffull);   // tiles completed (mod 2^24)
            const unsigned long long Mk = lat >> 24;
            // map to the most recent tile with that low-24-bit count
            if (done >= 1 && done <= tile) {
                const unsigned long long k = done - 1;
                M_ub = std::min(M_ub, Mk + (t0 - tile_end[k]));
            }
        }
        int P = early ? phases_for(M_ub, o.window0, o.growth ? o.growth : 2u) : 1;
        if (t0 == 0) P = 0;            // empty codebook before the first tile
        else if (P < 1) P = 1;

        k_gen_tile<<<std::min<uint32_t>((Kpad + 255) / 256, (uint32_t)cx->sm_count * 4), 256, 0, st>>>(
            cx->tabs, a.ordering, (int)a.n, t0, K, Kpad, cx->vals, cx->dead, cx->ctr);
        for (unsigned pl = 0; pl < parts_local; ++pl) {
            const unsigned g = (a.world > 1) ? (unsigned)a.rank : pl;
            uint32_t plo = 0, plen = 0, kp = 0;
            if (gc_tile_partition(K, (int)G, (int)g, &plo, &plen, &kp) != GC_OK) return GC_EINTERNAL;
            const uint2 *lin = nullptr;
            const unsigned int *cin = nullptr;
            for (int p = 0; p < P; ++p) {
                cudaEvent_t ea = nullptr, eb = nullptr;
                if (timing) {
                    if ((rc = cx->timing_event(nev++, &ea)) || (rc = cx->timing_event(nev++, &eb))) return rc;
                    CK(cudaEventRecord(ea, st));
                }
                k_screen<<<screen_grid, kScreenThreads, 0, st>>>(p, P, o.window0, (int)(o.growth ? o.growth : 2u), early, a.d_codebook, cx->vals,
                                                                lin, cin, plo, part, cx->dead, cx->ctr, a.d);
                if (timing) CK(cudaEventRecord(eb, st));
                ++launches;
                ++screen_launches;
                if (p + 1 < P) {
                    uint2 *lout = cx->list[p & 1];
                    unsigned int *cout = &cx->ctr->list_count[g * kMaxPhases + p];
                    const uint32_t L_ub = part;
                    k_compact<<<std::min<uint32_t>((L_ub + 255) / 256, (uint32_t)cx->sm_count * 4), 256, 0, st>>>(
                        cx->vals, lin, cin, plo, part, cx->dead, lout, cout);
                    ++launches;
                    lin = lout;
                    cin = cout;
                }
            }
            phases_total += P;
        }
        if (a.world > 1 && P > 0) {
            // every rank's dead bits for its own partition -> the full tile mask
            const uint32_t seg = part / 32;
            rc = nccl_allgather_u32(cx->dead + (size_t)a.rank * seg, cx->dead, seg, a.nccl_comm, st);
            if (rc) return rc;
        }
        k_gather<<<1, kResolveThreads, 0, st>>>(Kpad, cx->dead, cx->vals, cx->surv, cx->ctr);
        k_edges<<<edge_grid, kEdgeBlock, 0, st>>>(cx->surv, cx->edges, a.d, cx->ctr);
        k_commit<<<1, kResolveThreads, 0, st>>>(cx->surv, cx->edges, cx->status, cx->blocked, a.d_codebook,
                                                a.capacity, a.d, t0, N - 1, force_seq, cx->ctr, tile,
                                                cx->host_latest_dev);
        launches += 4;   // gen, gather, edges, commit
        CK(cudaGetLastError());
        t0 += K;
        tile_end.push_back(t0);
        ++tile;
        if (o.flags & GC_FLAG_SYNC_TILES) CK(cudaStreamSynchronize(st));
    }
    k_finish<<<1, 1, 0, st>>>(cx->ctr, (unsigned long long *)a.d_count, a.capacity);
    ++launches;
    CK(cudaEventRecord(cx->ev1, st));
    CK(cudaGetLastError());

    if (a.stats) {
        CK(cudaStreamSynchronize(st));
        DevCounters h;
        CK(cudaMemcpy(&h, cx->ctr, sizeof h, cudaMemcpyDeviceToHost));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, cx->ev0, cx->ev1));
        gc_stats *s = a.stats;
        s->struct_size = sizeof(gc_stats);
        s->n_ranks = G;
        s->device_ms = ms;
        s->M = h.M;
        s->tiles = tile;
        s->phases = phases_total;
        s->checks_exec = h.checks_exec;
        s->survivors = h.survivors;
        s->conflicts = h.conflicts;
        s->resolve_checks = h.resolve_checks;
        s->w_def = (double)h.w_def;
        s->launches = launches;
        s->screen_launches = screen_launches;
        s->screen_ms = 0;
        for (size_t i = 0; i + 1 < nev; i += 2) {
            float t = 0;
            CK(cudaEventElapsedTime(&t, cx->tev[i], cx->tev[i + 1]));
            s->screen_ms += t;
        }
        s->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
        if (o.flags & GC_FLAG_DEBUG_PHASES) {
            for (int p = 0; p < kMaxPhases; ++p)
                if (h.phase_alive[p])
                    fprintf(stderr, "[gc] phase %2d: alive %.4g  checks %.4g  (%.1f%% of screen)\n", p,
                            (double)h.phase_alive[p], (double)h.phase_checks[p],
                            100.0 * (double)h.phase_checks[p] / (double)(h.checks_exec ? h.checks_exec : 1));
        }
        if (h.error) { set_error("codebook capacity exceeded"); return GC_ENOSPC; }
    }
    return GC_OK;
}

int engine_ranks_to_vectors_device(int ordering, uint32_t n, uint64_t first, uint64_t count, uint32_t *d_out,
                                   void *stream) {
    int device;
    CK(cudaGetDevice(&device));
    DeviceContext *cx = context_for(device);
    std::lock_guard<std::mutex> lock(cx->mu);
    int rc = cx->ensure(32);
    if (rc) return rc;
    OrderTables t;
    build_order_tables((int)n, &t);
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemcpyAsync(cx->tabs, &t, sizeof t, cudaMemcpyHostToDevice, st));
    cx->tabs_n = (int)n;
    const unsigned long long blocks = std::min<unsigned long long>((count + 255) / 256, 148ull * 16);
    k_unrank<<<(unsigned)blocks, 256, 0, st>>>(cx->tabs, ordering, (int)n, first, count, d_out);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return GC_OK;
}

}  // namespace gc

using namespace gc;

// host-buffer construction shared by gc_generate_ex and gc_construct (args validated)
static int host_construct(RunArgs &a, uint64_t *out_codewords, uint64_t *out_count, gc_stats *stats);

extern "C" int gc_construct(const gc_problem *problem, const gc_options *opt, uint64_t *out_codewords,
                            uint64_t *out_count, gc_stats *stats) {
    clear_error();
    if (!out_count) { set_error("out_count is NULL"); return GC_EINVAL; }
    if (!out_codewords && *out_count) { set_error("out_codewords is NULL with capacity > 0"); return GC_EINVAL; }
    gc_problem base{};
    RunArgs a;
    int rc = gc_problem_to_args(problem, &a);
    (void)base;
    if (rc) return rc;
    rc = resolve_options(opt, &a.opt);
    if (rc) return rc;
    if (a.wide()) return cw64_supported(a) ? cw64_run(a, out_codewords, out_count, stats) : GC_EUNSUPPORTED;
    return host_construct(a, out_codewords, out_count, stats);
}

extern "C" int gc_generate_ex(uint32_t n, uint32_t d, gc_ordering ordering, const gc_options *opt,
                              uint64_t *out_codewords, uint64_t *out_count, gc_stats *stats) {
    clear_error();
    if (!out_count) { set_error("out_count is NULL"); return GC_EINVAL; }
    if (!out_codewords && *out_count) { set_error("out_codewords is NULL with capacity > 0"); return GC_EINVAL; }
    if (ordering < GC_LEX || ordering > GC_GRADED_REVLEX) { set_error("unknown ordering"); return GC_EINVAL; }
    if (n == 0) { set_error("n must be >= 1"); return GC_EINVAL; }
    if (d == 0 || d > n) { set_error("d must be in [1, n]"); return GC_EINVAL; }
    if (n > 32) { set_error("the GPU path supports n <= 32"); return GC_EUNSUPPORTED; }
    RunArgs a;
    int rc = resolve_options(opt, &a.opt);
    if (rc) return rc;
    a.n = n; a.d = d; a.ordering = ordering;
    return host_construct(a, out_codewords, out_count, stats);
}

// Host-buffer path: device codebook, count and a pinned staging buffer are cached per device
// (grown on demand) so a call pays no allocation; the code comes back through pinned memory
// and is widened to u64 by a few host threads.
namespace {
struct HostPathCache {
    uint32_t *d_cb = nullptr;
    uint64_t cap = 0;
    unsigned long long *d_cnt = nullptr;
    uint32_t *h_pin = nullptr;
    uint64_t pin_cap = 0;
    std::mutex mu;
};
std::mutex g_hp_mu;
std::map<int, std::unique_ptr<HostPathCache>> g_hp;

HostPathCache *host_cache(int dev) {
    std::lock_guard<std::mutex> g(g_hp_mu);
    auto &p = g_hp[dev];
    if (!p) p.reset(new HostPathCache);
    return p.get();
}

void widen(const uint32_t *src, uint64_t *dst, uint64_t M) {
    const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    const uint64_t per = (M + hw - 1) / hw;
    if (M < (1u << 16) || hw == 1) {
        for (uint64_t i = 0; i < M; ++i) dst[i] = src[i];
        return;
    }
    std::vector<std::thread> th;
    for (unsigned t = 0; t < hw; ++t) {
        const uint64_t b = t * per, e = std::min(M, b + per);
        if (b >= e) break;
        th.emplace_back([=] { for (uint64_t i = b; i < e; ++i) dst[i] = src[i]; });
    }
    for (auto &x : th) x.join();
}
}  // namespace

static int host_construct(RunArgs &a, uint64_t *out_codewords, uint64_t *out_count, gc_stats *stats) {
    int rc;
    const uint32_t n = a.n, d = a.d;
    const uint64_t cap = gc_capacity_bound(n, d);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    HostPathCache *hc = host_cache(dev);
    std::lock_guard<std::mutex> lock(hc->mu);
    if (hc->cap < cap) {
        if (hc->d_cb) cudaFree(hc->d_cb);
        hc->d_cb = nullptr;
        hc->cap = 0;
        CK(cudaMalloc(&hc->d_cb, cap * sizeof(uint32_t)));
        hc->cap = cap;
    }
    if (!hc->d_cnt) CK(cudaMalloc(&hc->d_cnt, sizeof(unsigned long long)));
    gc_stats local{};
    a.d_codebook = hc->d_cb; a.capacity = cap; a.d_count = (uint64_t *)hc->d_cnt;
    a.stream = nullptr; a.stats = stats ? stats : &local;
    rc = engine_run(a);
    unsigned long long M = 0;
    if (rc == GC_OK) {
        cudaError_t e = cudaMemcpy(&M, hc->d_cnt, sizeof M, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); rc = GC_ECUDA; }
    }
    if (rc == GC_OK) {
        if (M > *out_count) {
            *out_count = M;
            rc = GC_ENOSPC;
        } else if (M) {
            if (hc->pin_cap < M) {
                if (hc->h_pin) cudaFreeHost(hc->h_pin);
                hc->h_pin = nullptr;
                hc->pin_cap = 0;
                if (cudaHostAlloc(&hc->h_pin, cap * sizeof(uint32_t), cudaHostAllocDefault) == cudaSuccess)
                    hc->pin_cap = cap;
            }
            std::vector<uint32_t> pageable;
            uint32_t *h = hc->h_pin;
            if (!h) { pageable.resize(M); h = pageable.data(); }      // pinned allocation failed
            cudaError_t e = cudaMemcpy(h, hc->d_cb, M * sizeof(uint32_t), cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); rc = GC_ECUDA; }
            else {
                widen(h, out_codewords, M);
                *out_count = M;
            }
        } else {
            *out_count = 0;
        }
    }
    return rc;
}
