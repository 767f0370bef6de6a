// gc_persistent.cu -- the device-resident construction: ONE cooperative kernel runs the
// whole greedy scan, tile after tile, with no host round trip.  This is
// the B200 replacement of the paper's per-vector host loop and of its
// dynamic-parallelism parent kernel: the loop itself lives on the GPU.
//
// Per tile of K consecutive ranks [t0, t0+K):
//   levels l = 0 .. L-1   a1+a2: every candidate against the codebook committed before the
//                         tile, newest first, in geometrically growing windows
//                         [M - W0(2^l - 1) - W0 2^l, M - W0(2^l - 1)), the last one down to 0.
//                         Work items are WARP-granular: (64 candidates, <= kSub codewords);
//                         codewords are read with warp-uniform 128-bit loads (L1/L2 broadcast),
//                         XOR + POPC + min per check, warp-vote early exit.  The warp that
//                         completes a batch's last item pushes the batch's live candidates to
//                         the next level's list, so no compaction pass/barrier is needed.
//   grid barrier after each level (the dead bits of level l decide level l+1's list)
//   resolve (CTA 0)       a3: survivors in rank order; a survivor with no earlier in-tile
//                         conflict is accepted outright, the others are decided in rank order
//                         against the accepted ones (PAPER.md:59 inside the tile); a4: append.
//   grid barrier          the commit is visible to every CTA before the next tile.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include "gc_internal.h"
#include "gc_order.cuh"

namespace cg = cooperative_groups;

namespace gc {

constexpr int kPThreads = 512;              // threads per CTA (16 warps); grid = #SMs
constexpr int kPWarps = kPThreads / 32;
constexpr int kPR = 2;                      // candidates per lane
constexpr int kPBatch = 32 * kPR;           // candidates per warp item
constexpr uint32_t kPSub = 512;             // codewords per warp item
constexpr int kPMaxLevels = 32;
constexpr uint32_t kPMaxTile = 1u << 13;    // largest tile for this engine (survivors fit in smem)
constexpr uint32_t kPMaxBatches = kPMaxTile / kPBatch;
constexpr size_t kPDynSmem = kPMaxTile * 7;     // s_val (4 B) + s_idx (2 B) + s_status (1 B)

struct PState {
    unsigned long long M;
    unsigned long long checks_exec;
    unsigned long long survivors;
    unsigned long long conflicts;
    unsigned long long resolve_checks;
    unsigned long long w_def;
    unsigned long long tiles;
    unsigned long long levels;
    unsigned int error;
    unsigned int q_count[kPMaxLevels + 1];
    unsigned int bfin[kPMaxLevels][kPMaxBatches];
};

struct PArgs {
    int n, ord;
    uint32_t d;
    unsigned long long N;           // 2^n
    uint32_t tile_min, tile_max, W0;
    uint32_t *codebook;
    unsigned long long capacity;
    const OrderTables *tabs;
    uint32_t *vals;                 // [kPMaxTile]
    uint32_t *dead;                 // [kPMaxTile / 32]
    uint2 *q0, *q1;                 // level lists (ping-pong), [kPMaxTile] each
    uint2 *surv;                    // [kPMaxTile]
    uint8_t *status;                // [kPMaxTile]
    PState *st;
    unsigned long long *d_count;
};

__device__ __forceinline__ uint32_t p_tile_size(const PArgs &a, unsigned long long t0) {
    uint32_t K = a.tile_min;
    while (K < a.tile_max && (unsigned long long)K * 8 <= t0) K <<= 1;
    if ((unsigned long long)K > a.N - t0) K = (uint32_t)(a.N - t0);
    return K;
}

// number of levels needed to reach codeword 0 from the newest, windows W0 * 2^l
__device__ __forceinline__ int p_levels(unsigned long long M, uint32_t W0) {
    if (M == 0) return 0;
    int L = 1;
    while (L < kPMaxLevels && (unsigned long long)W0 * ((1ull << L) - 1) < M) ++L;
    return L;
}

// scan codewords [a, b) newest first for the lane's kPR candidates; returns the number of
// codewords scanned (for the work counter).  Early exit when every lane's candidates are dead.
__device__ __forceinline__ uint32_t p_scan(const uint32_t *__restrict__ cb, long long a, long long b,
                                           const uint32_t (&v)[kPR], uint32_t (&m)[kPR], uint32_t d) {
    long long hi = b;
    uint32_t scanned = 0;
    // unaligned top part (scalar) so that the body is 16-byte aligned
    while (hi > a && (hi & 3)) {
        const uint32_t c = __ldcg(cb + hi - 1);
#pragma unroll
        for (int r = 0; r < kPR; ++r) m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c));
        --hi;
        ++scanned;
    }
    const uint4 *cb4 = reinterpret_cast<const uint4 *>(cb);
    long long g = hi >> 2;                    // groups [a4, g)
    const long long a4 = (a + 3) >> 2;
    int it = 0;
    while (g > a4) {
        if ((it++ & 7) == 0) {
            bool done = true;
#pragma unroll
            for (int r = 0; r < kPR; ++r) done &= (m[r] < d);
            if (__all_sync(0xffffffffu, done)) return scanned;
        }
        const uint4 c = __ldcg(cb4 + g - 1);
#pragma unroll
        for (int r = 0; r < kPR; ++r) {
            m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c.w));
            m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c.z));
            m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c.y));
            m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c.x));
        }
        --g;
        scanned += 4;
    }
    hi = g << 2;
    while (hi > a) {                          // unaligned bottom part
        const uint32_t c = __ldcg(cb + hi - 1);
#pragma unroll
        for (int r = 0; r < kPR; ++r) m[r] = min(m[r], (uint32_t)__popc(v[r] ^ c));
        --hi;
        ++scanned;
    }
    return scanned;
}

// block-wide exclusive scan (blockDim.x == kPThreads); *total = block sum
__device__ __forceinline__ uint32_t p_block_scan(uint32_t x, uint32_t *total, uint32_t *ws) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint32_t s = lane < kPWarps ? ws[lane] : 0u, si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += y;
        }
        if (lane < kPWarps) ws[lane] = si - s;
        if (lane == 31) ws[32] = si;
    }
    __syncthreads();
    const uint32_t r = ws[wid] + inc - x;
    *total = ws[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kPThreads, 1) k_construct(PArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t C[33][33];
    __shared__ uint64_t off[34];
    __shared__ uint32_t s_ws[33];
    extern __shared__ __align__(16) uint8_t p_dyn[];        // resolve scratch (kPDynSmem bytes)
    uint32_t *s_val = reinterpret_cast<uint32_t *>(p_dyn);
    uint16_t *s_idx = reinterpret_cast<uint16_t *>(p_dyn + kPMaxTile * 4);
    uint8_t *s_status = p_dyn + kPMaxTile * 6;
    PState *st = a.st;
    const bool graded = a.ord >= GRADED_LEX;
    if (graded) {
        for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) C[i / 33][i % 33] = a.tabs->binom[i / 33][i % 33];
        for (int i = threadIdx.x; i < 34; i += blockDim.x) off[i] = a.tabs->off[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t gwarp = blockIdx.x * kPWarps + (threadIdx.x >> 5);
    const uint32_t nwarps = gridDim.x * kPWarps;
    unsigned long long my_checks = 0;

    unsigned long long t0 = 0;
    while (t0 < a.N) {
        const uint32_t K = p_tile_size(a, t0);
        const unsigned long long M = __ldcg(&st->M);
        const int L = p_levels(M, a.W0);
        const uint32_t W0 = a.W0;

        for (int l = 0; l < L; ++l) {
            // window of level l (newest-first positions), last level reaches 0
            const long long bp = (long long)W0 * ((1ll << l) - 1);
            const long long hi = (long long)M - bp;
            long long lo = (l == L - 1) ? 0 : hi - ((long long)W0 << l);
            if (lo < 0) lo = 0;
            const uint32_t n_l = (l == 0) ? K : __ldcg(&st->q_count[l]);
            const uint2 *qin = (l == 0) ? nullptr : ((l & 1) ? a.q1 : a.q0);
            uint2 *qout = (l & 1) ? a.q0 : a.q1;
            const uint32_t B = (n_l + kPBatch - 1) / kPBatch;
            // sub-ranges aligned to absolute multiples of kPSub
            const long long c_top = (hi + kPSub - 1) / kPSub, c_bot = lo / kPSub;
            const uint32_t nsub = (hi > lo) ? (uint32_t)(c_top - c_bot) : 0u;
            const unsigned long long items = (unsigned long long)B * nsub;
            for (unsigned long long it = gwarp; it < items; it += nwarps) {
                const uint32_t j = (uint32_t)(it / B), b = (uint32_t)(it % B);
                // candidates of batch b
                uint32_t v[kPR], m[kPR], idx[kPR];
                bool live[kPR];
#pragma unroll
                for (int r = 0; r < kPR; ++r) {
                    const uint32_t pos = b * kPBatch + r * 32 + lane;
                    live[r] = pos < n_l;
                    idx[r] = 0; v[r] = 0;
                    if (live[r]) {
                        if (qin) { const uint2 e = __ldcg(qin + pos); idx[r] = e.x; v[r] = e.y; }
                        else {
                            idx[r] = pos;
                            v[r] = rank_to_vector32(a.ord, a.n, C, off, t0 + pos);
                            if (j == 0) a.vals[pos] = v[r];
                        }
                        live[r] = !((__ldcg(a.dead + (idx[r] >> 5)) >> (idx[r] & 31)) & 1u);
                    }
                    m[r] = live[r] ? 64u : 0u;
                }
                const long long cidx = c_top - 1 - (long long)j;          // j = 0: newest chunk
                const long long s_lo = max(lo, cidx * (long long)kPSub);
                const long long s_hi = min(hi, (cidx + 1) * (long long)kPSub);
                bool any = false;
#pragma unroll
                for (int r = 0; r < kPR; ++r) any |= live[r];
                if (__any_sync(0xffffffffu, any)) {
                    const uint32_t sc = p_scan(a.codebook, s_lo, s_hi, v, m, a.d);
                    my_checks += (unsigned long long)sc * kPR;   // per lane; summed over lanes below
#pragma unroll
                    for (int r = 0; r < kPR; ++r) {
                        const bool kill = live[r] && m[r] < a.d;
                        if (!qin) {
                            const unsigned bb = __ballot_sync(0xffffffffu, kill);
                            if (lane == 0 && bb) atomicOr(&a.dead[idx[r] >> 5], bb);
                        } else if (kill) {
                            atomicOr(&a.dead[idx[r] >> 5], 1u << (idx[r] & 31));
                        }
                    }
                }
                if (l + 1 < L) {
                    // the warp finishing batch b's last item pushes its live candidates
                    __threadfence();
                    unsigned last = 0;
                    if (lane == 0) last = (atomicAdd(&st->bfin[l][b], 1u) + 1u == nsub);
                    last = __shfl_sync(0xffffffffu, last, 0);
                    if (last) {
                        __threadfence();
#pragma unroll
                        for (int r = 0; r < kPR; ++r) {
                            const uint32_t pos = b * kPBatch + r * 32 + lane;
                            bool alive = pos < n_l;
                            uint2 e = make_uint2(0, 0);
                            if (alive) {
                                if (qin) e = __ldcg(qin + pos);
                                else { e.x = pos; e.y = v[r]; }
                                alive = !((__ldcg(a.dead + (e.x >> 5)) >> (e.x & 31)) & 1u);
                            }
                            const unsigned bb = __ballot_sync(0xffffffffu, alive);
                            unsigned base = 0;
                            if (lane == 0 && bb) base = atomicAdd(&st->q_count[l + 1], (unsigned)__popc(bb));
                            base = __shfl_sync(0xffffffffu, base, 0);
                            if (alive) qout[base + __popc(bb & ((1u << lane) - 1u))] = e;
                        }
                    }
                }
            }
            grid.sync();
        }

        // ------------------------------------------------ resolve + commit (CTA 0)
        if (blockIdx.x == 0) {
            const uint32_t tid = threadIdx.x;
            const uint32_t words = (K + 31) / 32;
            if (L == 0) {      // empty codebook: no level generated the candidates
                for (uint32_t i = tid; i < K; i += blockDim.x) a.vals[i] = rank_to_vector32(a.ord, a.n, C, off, t0 + i);
                __syncthreads();
            }
            // survivors in rank order -> s_val / s_idx
            uint32_t S = 0;
            for (uint32_t w0 = 0; w0 < words; w0 += blockDim.x) {
                const uint32_t w = w0 + tid;
                uint32_t alive = 0;
                if (w < words) {
                    alive = ~__ldcg(a.dead + w);
                    if (w * 32 + 32 > K) alive &= (1u << (K - w * 32)) - 1u;
                }
                uint32_t tot;
                uint32_t pos = S + p_block_scan(__popc(alive), &tot, s_ws);
                while (alive) {
                    const int bit = __ffs(alive) - 1;
                    alive &= alive - 1;
                    const uint32_t i = w * 32 + bit;
                    s_idx[pos] = (uint16_t)i;
                    s_val[pos] = __ldcg(a.vals + i);
                    ++pos;
                }
                S += tot;
            }
            __syncthreads();
            // status: 1 = accepted (no earlier in-tile conflict), 2 = undecided (has one)
            unsigned long long rchk = 0, confl = 0;
            for (uint32_t j = tid; j < S; j += blockDim.x) {
                const uint32_t vj = s_val[j];
                uint32_t has = 0;
                for (uint32_t k = 0; k < j; ++k) has |= (uint32_t)__popc(vj ^ s_val[k]) < a.d;
                rchk += j;
                s_status[j] = has ? 2 : 1;
                confl += has;
            }
            __syncthreads();
            // undecided survivors in rank order (warp 0): accepted iff no earlier ACCEPTED
            // survivor is within distance < d
            if (tid < 32) {
                for (uint32_t j = 0; j < S; ++j) {
                    if (s_status[j] != 2) continue;      // uniform across the warp
                    const uint32_t vj = s_val[j];
                    bool c = false;
                    for (uint32_t k = lane; k < j; k += 32)
                        c |= (s_status[k] == 1) && (uint32_t)__popc(vj ^ s_val[k]) < a.d;
                    c = __any_sync(0xffffffffu, c);
                    if (lane == 0) s_status[j] = c ? 0 : 1;
                    __syncwarp();
                }
            }
            __syncthreads();
            // ordered append
            const unsigned long long M0 = __ldcg(&st->M);
            uint32_t A = 0;
            unsigned long long wdef = 0;
            for (uint32_t j0 = 0; j0 < S; j0 += blockDim.x) {
                const uint32_t j = j0 + tid;
                const uint32_t acc = (j < S && s_status[j] == 1) ? 1u : 0u;
                uint32_t tot;
                const uint32_t pos = A + p_block_scan(acc, &tot, s_ws);
                if (acc) {
                    if (M0 + pos < a.capacity) a.codebook[M0 + pos] = s_val[j];
                    else st->error = 1;
                    wdef += a.N - 1 - (t0 + s_idx[j]);
                }
                A += tot;
            }
            // clear per-tile state for the next tile
            for (uint32_t w = tid; w < kPMaxTile / 32; w += blockDim.x) a.dead[w] = 0;
            for (int l = 0; l < L; ++l)
                for (uint32_t b = tid; b < kPMaxBatches; b += blockDim.x) st->bfin[l][b] = 0;
            for (int l = tid; l <= kPMaxLevels; l += blockDim.x) st->q_count[l] = 0;
            if (rchk) atomicAdd(&st->resolve_checks, rchk);
            if (confl) atomicAdd(&st->conflicts, confl);
            if (wdef) atomicAdd(&st->w_def, wdef);
            __syncthreads();
            if (tid == 0) {
                unsigned long long M1 = M0 + A;
                if (M1 > a.capacity) M1 = a.capacity;
                st->M = M1;
                st->survivors += S;
                st->tiles += 1;
                st->levels += L;
            }
            __threadfence();
        }
        grid.sync();
        t0 += K;
    }
    // work counter: lanes hold per-lane counts
    for (int o = 16; o > 0; o >>= 1) my_checks += __shfl_down_sync(0xffffffffu, my_checks, o);
    if (lane == 0 && my_checks) atomicAdd(&st->checks_exec, my_checks);
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.d_count = st->M;
}

// ------------------------------------------------------------------ host side

struct PContext {
    int device = -1, sms = 0;
    uint32_t *vals = nullptr, *dead = nullptr;
    uint2 *q0 = nullptr, *q1 = nullptr, *surv = nullptr;
    uint8_t *status = nullptr;
    PState *st = nullptr;
    OrderTables *tabs = nullptr;
    int tabs_n = -1;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::mutex mu;
};

#define PCK(call)                                                                             \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
            return e_ == cudaErrorMemoryAllocation ? GC_ENOMEM : GC_ECUDA;                   \
        }                                                                                     \
    } while (0)

static std::mutex g_pmu;
static PContext *g_pctx[64];

static int p_context(int device, PContext **out) {
    std::lock_guard<std::mutex> g(g_pmu);
    if (device < 0 || device >= 64) { set_error("device index out of range"); return GC_EINVAL; }
    PContext *c = g_pctx[device];
    if (!c) {
        c = new PContext;
        c->device = device;
        PCK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
        PCK(cudaMalloc(&c->vals, kPMaxTile * 4));
        PCK(cudaMalloc(&c->dead, kPMaxTile / 8));
        PCK(cudaMalloc(&c->q0, kPMaxTile * sizeof(uint2)));
        PCK(cudaMalloc(&c->q1, kPMaxTile * sizeof(uint2)));
        PCK(cudaMalloc(&c->surv, kPMaxTile * sizeof(uint2)));
        PCK(cudaMalloc(&c->status, kPMaxTile));
        PCK(cudaMalloc(&c->st, sizeof(PState)));
        PCK(cudaMalloc(&c->tabs, sizeof(OrderTables)));
        PCK(cudaEventCreate(&c->ev0));
        PCK(cudaEventCreate(&c->ev1));
        g_pctx[device] = c;
    }
    *out = c;
    return GC_OK;
}

constexpr uint32_t kPDefaultTile = 4096;

bool persistent_supported(const RunArgs &a) {
    return a.world == 1 && a.opt.emulate_ranks == 1 && a.opt.tile_max <= kPMaxTile &&
           a.opt.tile_min <= std::max(a.opt.tile_max, kPDefaultTile) &&
           !(a.opt.flags & (GC_FLAG_NO_EARLY_EXIT | GC_FLAG_FORCE_SEQ_RESOLVE | GC_FLAG_LAUNCHED_TILES));
}

int persistent_run(const RunArgs &r) {
    int device;
    PCK(cudaGetDevice(&device));
    PContext *cx;
    int rc = p_context(device, &cx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(cx->mu);
    cudaStream_t s = (cudaStream_t)r.stream;
    if (cx->tabs_n != (int)r.n) {
        OrderTables t;
        build_order_tables((int)r.n, &t);
        PCK(cudaMemcpy(cx->tabs, &t, sizeof t, cudaMemcpyHostToDevice));
        cx->tabs_n = (int)r.n;
    }
    PCK(cudaMemsetAsync(cx->st, 0, sizeof(PState), s));
    PCK(cudaMemsetAsync(cx->dead, 0, kPMaxTile / 8, s));
    PArgs a;
    a.n = (int)r.n; a.ord = r.ordering; a.d = r.d;
    a.N = 1ull << r.n;
    a.tile_min = r.opt.tile_min; a.tile_max = r.opt.tile_max ? r.opt.tile_max : kPDefaultTile;
    a.W0 = r.opt.window0;
    a.codebook = r.d_codebook; a.capacity = r.capacity;
    a.tabs = cx->tabs; a.vals = cx->vals; a.dead = cx->dead;
    a.q0 = cx->q0; a.q1 = cx->q1; a.surv = cx->surv; a.status = cx->status;
    a.st = cx->st; a.d_count = (unsigned long long *)r.d_count;
    int per_sm = 0;
    PCK(cudaFuncSetAttribute(k_construct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPDynSmem));
    PCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_construct, kPThreads, kPDynSmem));
    if (per_sm < 1) { set_error("k_construct cannot be resident"); return GC_ECUDA; }
    void *args[] = {&a};
    PCK(cudaEventRecord(cx->ev0, s));
    PCK(cudaLaunchCooperativeKernel((const void *)k_construct, dim3(cx->sms), dim3(kPThreads), args, kPDynSmem, s));
    PCK(cudaEventRecord(cx->ev1, s));
    if (r.stats) {
        PCK(cudaStreamSynchronize(s));
        PState h;
        PCK(cudaMemcpy(&h, cx->st, offsetof(PState, q_count), cudaMemcpyDeviceToHost));
        float ms = 0;
        PCK(cudaEventElapsedTime(&ms, cx->ev0, cx->ev1));
        gc_stats *o = r.stats;
        o->struct_size = sizeof(gc_stats);
        o->n_ranks = 1;
        o->device_ms = ms;
        o->M = h.M;
        o->tiles = h.tiles;
        o->phases = h.levels;
        o->checks_exec = h.checks_exec;
        o->survivors = h.survivors;
        o->conflicts = h.conflicts;
        o->resolve_checks = h.resolve_checks;
        o->w_def = (double)h.w_def;
        o->launches = 1;
        o->screen_launches = 1;
        o->screen_ms = ms;
        if (h.error) { set_error("codebook capacity exceeded"); return GC_ENOSPC; }
    }
    return GC_OK;
}

}  // namespace gc
