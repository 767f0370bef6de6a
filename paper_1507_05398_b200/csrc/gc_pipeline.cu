// gc_pipeline.cu -- the pipelined device-resident construction: the default single-GPU
// engine.  ONE persistent kernel runs the whole greedy scan with no host round
// trip (the paper's lesson of PAPER.md:157, taken further), and -- unlike k_construct, where
// every CTA screens one tile, waits at a grid barrier and then waits for CTA 0's resolve --
// the screen of later tiles overlaps the resolve of earlier ones:
//
//   CTA 0 (resolver)   tiles in rank order: waits until tile i is screened, then the in-tile
//                      ordered resolve and the commit (a4); at the
//                      commit of tile i it publishes the descriptor of tile i + D (its ranks and
//                      the codebook size M_i it is screened against) and the count of committed
//                      tiles (release).
//   CTAs 1.. (screen)  any published tile: its levels (a1 + a2 + a2') against codebook[0, M_s),
//                      warp items claimed from per-tile, per-level counters, the last warp of a
//                      level merges its kills and opens the next level (arrival counters, no
//                      grid barrier).
//
// A tile is screened against the codebook committed D tiles before it; the resolve checks its
// survivors against the words committed since (codebook[M_s, M)) before the in-tile greedy.
// Exact: the screen only ever REMOVES candidates that have an earlier codeword closer than d,
// and the resolve applies the rest of "distance >= d from every previous choice"
// in rank order.  The result is independent of D and of timing; the schedule (tile sizes, the
// codebook each screen sees) is a deterministic function of the problem and D.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "gc_screen.cuh"

namespace gc {

constexpr int kQRing = 16;          // tile slots; the pipeline depth D <= kQRing
constexpr uint32_t kQWords = kPMaxTile / 32;

// One tile in flight (global memory).  The descriptor fields are written by the resolver before
// it releases `phase`; `items[l]` / `nlive[l]` for l >= 1 by the warp that finished level l - 1
// before it releases `phase`.  Every reader acquires `phase` first and reads the rest from L2.
struct QSlot {
    unsigned long long phase;                   // (tile + 1) << 8 | level; level >= L: screened
    unsigned long long t0, M_s, base;           // first rank; screened against codebook[base, M_s)
    uint32_t K, L;                              // candidates; levels
    uint32_t items[kPMaxLevels];                // warp items of each level
    uint32_t nlive[kPMaxLevels];                // live candidates at the start of each level
    uint32_t done[kPMaxLevels];                 // items finished (arrival counter)
    unsigned long long claim[kPMaxLevels];      // ((tile + 1) mod 2^32) << 32 | items claimed
};
struct QCtl {
    unsigned long long committed;               // tiles committed (release; the resolver only)
    unsigned int finished;                      // every tile committed
    unsigned int pad;
    unsigned long long resolve_wait_ns;         // diagnostics: resolver time waiting for screens
    unsigned long long resolve_busy_ns;         //              and resolving
    QSlot slot[kQRing];
};

__device__ __forceinline__ unsigned long long q_ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int q_ld_acquire32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void q_st_release(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void q_st_release32(unsigned int *p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Resolver thread 0: publish tile i (ranks [t0, t0 + K)) to be screened against
// codebook[base, M_s).  Level 0 plans all K candidates; a tile with nothing to screen
// (L == 0) is published as already screened.
__device__ __forceinline__ void q_publish(const PArgs &a, QCtl *q, unsigned long long i, unsigned long long t0,
                                          uint32_t K, unsigned long long M_s, unsigned long long base) {
    QSlot &sl = q->slot[i % kQRing];
    const int L = p_levels(M_s - base, a.W0, a.growth);
    sl.t0 = t0; sl.K = K; sl.M_s = M_s; sl.base = base; sl.L = (uint32_t)L;
    const unsigned long long tag = (i + 1) & 0xffffffffull;
    for (int l = 0; l < L; ++l) { sl.claim[l] = tag << 32; sl.done[l] = 0; sl.items[l] = 0; sl.nlive[l] = 0; }
    if (L > 0) {
        long long hi, lo;
        p_level_window(a, M_s, base, L, 0, hi, lo);
        sl.items[0] = (uint32_t)p_plan(a, K, hi - lo, a.plan_warps).items();
        sl.nlive[0] = K;
    }
    __threadfence();
    q_st_release(&sl.phase, (i + 1) << 8);           // level 0 (>= L when L == 0: screened)
}

// The warp that finished the last item of level l of tile i: merge the level's kills into the
// tile's dead mask, count the live candidates, plan level l + 1 and open it (or mark the tile
// screened when nothing is left to screen).
__device__ __forceinline__ void q_finish_level(const PArgs &a, QSlot *sl, unsigned long long i, int l, int L,
                                               uint32_t K, unsigned long long M_s, unsigned long long base,
                                               uint32_t *dead, uint32_t *kill) {
    __threadfence();                                  // acquire side of the items' release
    const int lane = threadIdx.x & 31;
    const uint32_t words = (K + 31) / 32;
    uint32_t live = 0;
    for (uint32_t w = lane; w < words; w += 32) {
        const uint32_t k = __ldcg(kill + w);
        uint32_t dd = __ldcg(dead + w);
        if (k) {
            dd |= k;
            __stcg(dead + w, dd);
            __stcg(kill + w, 0u);
        }
        uint32_t lv = ~dd;
        if (w * 32 + 32 > K) lv &= (1u << (K - w * 32)) - 1u;
        live += __popc(lv);
    }
    live = __reduce_add_sync(0xffffffffu, live);
    int nl = l + 1;
    uint32_t items = 0;
    if (nl < L && live > 0) {
        long long hi, lo;
        p_level_window(a, M_s, base, L, nl, hi, lo);
        items = (uint32_t)p_plan(a, live, hi - lo, a.plan_warps).items();
    }
    if (items == 0) nl = L;                           // nothing left to screen
    __threadfence();
    __syncwarp();
    if (lane == 0) {
        if (nl < L) {
            sl->items[nl] = items;
            sl->nlive[nl] = live;
        }
        __threadfence();
        q_st_release(&sl->phase, ((i + 1) << 8) | (unsigned)nl);
    }
    __syncwarp();
}

template <int kMinBlocks>
__global__ void __launch_bounds__(kPThreads, kMinBlocks) k_pipeline(PArgs a) {
    const uint32_t kPChunk = a.chunk;
    __shared__ uint32_t C[33][33];
    __shared__ uint64_t off[34];
    __shared__ uint32_t s_ws[33];
    __shared__ uint32_t s_basis[32];
    extern __shared__ __align__(16) uint8_t p_dyn[];
    uint32_t *s_pre = reinterpret_cast<uint32_t *>(p_dyn + p_scratch_smem(kPChunk));
    uint32_t *s_live = s_pre + kPMaxTile / 32 + 4;
    uint2 *s_sup = reinterpret_cast<uint2 *>(p_dyn + p_dyn_smem(kPChunk));     // [a.nsup_smem]
    PState *st = a.st;
    QCtl *q = a.q;
    if (threadIdx.x < 32) s_basis[threadIdx.x] = a.basis[threadIdx.x];
    if (a.ord >= GRADED_LEX) {
        for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) C[i / 33][i % 33] = a.tabs->binom[i / 33][i % 33];
        for (int i = threadIdx.x; i < 34; i += blockDim.x) off[i] = a.tabs->off[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned long long my_checks = 0, my_tests = 0;

    if (blockIdx.x == 0) {
        // ------------------------------------------------------------------ resolver
        PSmem sm;
        sm.C = C; sm.off = off; sm.s_basis = s_basis; sm.s_ws = s_ws;
        sm.s_val = reinterpret_cast<uint32_t *>(p_dyn);
        sm.s_idx = reinterpret_cast<uint16_t *>(p_dyn + kPChunk * 4);
        sm.s_status = p_dyn + kPChunk * 6;
        sm.s_cnt = reinterpret_cast<uint32_t *>(p_dyn + kPChunk * 8);
        sm.s_adj = reinterpret_cast<uint16_t *>(p_dyn + kPChunk * 12);
        sm.chunk = kPChunk;
        sm.s_tmp = s_pre;                      // this CTA never screens: the level prefix area is free
        sm.tmp_words = kPTmpMaxWords;
        __shared__ PCount pc;
        __shared__ unsigned long long s_t0[kQRing], s_Ms[kQRing];
        __shared__ uint32_t s_K[kQRing], s_L[kQRing];
        __shared__ unsigned long long s_next, s_issued;
        __shared__ uint32_t s_klast;
        if (threadIdx.x == 0) {
            p_count_load(pc, st);
            s_next = a.t_begin;
            s_issued = 0;
            s_klast = a.tile_min;
            // the first D tiles are screened against the empty codebook (nothing to screen)
            for (int i = 0; i < a.depth && s_next < a.t_end; ++i) {
                const uint32_t K = (uint32_t)min((unsigned long long)a.tile_min, a.t_end - s_next);
                s_t0[i] = s_next; s_K[i] = K; s_Ms[i] = 0; s_L[i] = 0;
                q_publish(a, q, (unsigned long long)i, s_next, K, 0, 0);
                s_next += K;
                ++s_issued;
            }
        }
        unsigned long long t_wait = 0, t_busy = 0, t_pub = 0;
        PTimers tmr;
        if (a.timing && threadIdx.x == 0) memset(&tmr, 0, sizeof tmr);
        PTimers *timer = (a.timing && threadIdx.x == 0) ? &tmr : nullptr;
        for (unsigned long long i = 0;; ++i) {
            __syncthreads();
            if (i >= s_issued) break;
            const int si = (int)(i % kQRing);
            QSlot *sl = &q->slot[si];
            if (threadIdx.x == 0) {
                const unsigned long long tw = p_now();
                for (;;) {
                    const unsigned long long ph = q_ld_acquire(&sl->phase);
                    if ((ph >> 8) == i + 1 && (uint32_t)(ph & 0xff) >= s_L[si]) break;
                    __nanosleep(32);
                }
                const unsigned long long tb = p_now();
                t_wait += tb - tw;
                t_busy -= tb;
            }
            __syncthreads();
            uint32_t *dead = a.qdead + (size_t)si * kQWords;
            p_resolve(a, sm, s_t0[si], s_K[si], (int)s_L[si], pc, timer, 0, false, dead, s_Ms[si]);
            if (threadIdx.x == 0) {
                const unsigned long long tp = timer ? clock64() : 0;
                // next descriptor: tile s_issued, screened against the codebook as of now
                if (s_next < a.t_end) {
                    uint32_t Kn = p_next_tile(a, s_klast, pc.S_tile, pc.A_tile, s_t0[si] + s_K[si], pc.M, pc.S_last,
                                              pc.K_last ? pc.K_last : 1u);
                    s_klast = Kn;
                    if ((unsigned long long)Kn > a.t_end - s_next) Kn = (uint32_t)(a.t_end - s_next);
                    const unsigned long long base = p_base(a, s_next, pc.M);
                    const int sj = (int)(s_issued % kQRing);
                    s_t0[sj] = s_next; s_K[sj] = Kn; s_Ms[sj] = pc.M;
                    s_L[sj] = (uint32_t)p_levels(pc.M - base, a.W0, a.growth);
                    q_publish(a, q, s_issued, s_next, Kn, pc.M, base);
                    s_next += Kn;
                    ++s_issued;
                }
                __threadfence();
                q_st_release(&q->committed, i + 1);
                t_busy += p_now();
                if (timer) t_pub += clock64() - tp;
            }
        }
        if (threadIdx.x == 0) {
            q_st_release32(&q->finished, 1u);
            p_count_store(pc, st);
            *a.d_count = __ldcg(&st->error) ? a.capacity + 1 : pc.M;   // above capacity: incomplete (gc.h)
            q->resolve_wait_ns = t_wait;
            q->resolve_busy_ns = t_busy;
            if (timer) {
                for (int k = 0; k < 8; ++k) st->t_r[k] = tmr.r[k];
                st->t_sync = t_pub;
            }
        }
    } else {
        // ------------------------------------------------------------------ screen
        __shared__ unsigned long long s_tile, s_t0, s_Ms, s_base;
        __shared__ uint32_t s_K, s_L;
        __shared__ int s_lvl;
        unsigned long long hint = 0, supM = 0;
        for (;;) {
            if (threadIdx.x == 0) {
                int lvl = -1;
                unsigned long long pick = 0;
                unsigned int nap = 32;
                for (;;) {
                    const unsigned long long com = q_ld_acquire(&q->committed);
                    if (hint < com) hint = com;
                    for (unsigned long long i = hint; i < com + (unsigned long long)a.depth; ++i) {
                        QSlot *sl = &q->slot[i % kQRing];
                        const unsigned long long ph = q_ld_acquire(&sl->phase);
                        if ((ph >> 8) != i + 1) break;           // not published yet
                        const uint32_t l = (uint32_t)(ph & 0xff);
                        if (l >= __ldcg(&sl->L)) {                   // screened
                            if (i == hint) ++hint;
                            continue;
                        }
                        const unsigned long long c = __ldcg(&sl->claim[l]);
                        if ((c >> 32) == ((i + 1) & 0xffffffffull) && (uint32_t)c < __ldcg(&sl->items[l])) {
                            pick = i;
                            lvl = (int)l;
                            break;
                        }
                    }
                    if (lvl >= 0) break;
                    if (q_ld_acquire32(&q->finished)) { lvl = -2; break; }
                    __nanosleep(nap);
                    if (nap < 512) nap *= 2;
                }
                s_lvl = lvl;
                if (lvl >= 0) {
                    QSlot *sl = &q->slot[pick % kQRing];
                    s_tile = pick;
                    s_t0 = __ldcg(&sl->t0); s_Ms = __ldcg(&sl->M_s); s_base = __ldcg(&sl->base);
                    s_K = __ldcg(&sl->K); s_L = __ldcg(&sl->L);
                }
            }
            __syncthreads();
            const int l = s_lvl;
            if (l == -2) break;
            const unsigned long long i = s_tile, M_s = s_Ms, base = s_base, t0 = s_t0;
            const uint32_t K = s_K;
            const int L = (int)s_L;
            const int si = (int)(i % kQRing);
            QSlot *sl = &q->slot[si];
            const unsigned long long tag = (i + 1) & 0xffffffffull;
            uint32_t *dead = a.qdead + (size_t)si * kQWords, *kill = a.qkill + (size_t)si * kQWords;
            if (a.nsup_smem && M_s > supM) {
                // super-block summaries the commits since the last refresh changed (a summary that
                // also covers words beyond M_s is still valid: it only widens)
                const long long s0 = (long long)(supM >> 10);
                const long long s1 = min((long long)a.nsup_smem, (long long)((M_s + 1023) >> 10));
                for (long long x = s0 + threadIdx.x; x < s1; x += blockDim.x) s_sup[x] = __ldcg(a.ssum + x);
                supM = M_s;
            }
            long long hi, lo;
            p_level_window(a, M_s, base, L, l, hi, lo);
            uint32_t n_l = K;
            if (l > 0) n_l = p_live_prefix(dead, 0, K, s_live, s_pre, s_ws);    // ends with a barrier
            else __syncthreads();
            const PPlan pl = p_plan(a, n_l, hi - lo, a.plan_warps);
            PLevel lv;
            lv.l = l; lv.n_l = n_l; lv.B = pl.B; lv.nsub = pl.nsub;
            lv.hi = hi; lv.lo = lo; lv.sub = pl.sub; lv.t0 = t0; lv.head = pl.head; lv.J0 = pl.J0;
            lv.s_pre = s_pre; lv.s_live = s_live; lv.words = (K + 31) / 32; lv.basis = s_basis;
            lv.stage = reinterpret_cast<uint32_t *>(p_dyn); lv.s_sup = s_sup; lv.c_lo = 0; lv.w_base = 0;
            lv.kill = kill; lv.vals = a.qvals + (size_t)si * kPMaxTile;
            lv.win = nullptr; lv.wsum = nullptr; lv.win_lo = 0;
            if (p_window_in_smem(a, l, hi, lo))
                p_copy_window(a, lv, reinterpret_cast<uint32_t *>(p_dyn + (size_t)kPWarps * kPWarpStage * 4), hi, lo);
            const unsigned long long items = pl.items();
            for (;;) {
                unsigned long long c = 0;
                if (lane == 0) c = atomicAdd(&sl->claim[l], 1ull);
                c = __shfl_sync(0xffffffffu, c, 0);
                if ((c >> 32) != tag || (uint32_t)c >= items) break;
                p_run_item(a, lv, pl.R, (uint32_t)c, C, off, my_checks, my_tests);
                __threadfence();                              // this item's kills before its arrival
                __syncwarp();
                uint32_t dn = 0;
                if (lane == 0) dn = atomicAdd(&sl->done[l], 1u);
                dn = __shfl_sync(0xffffffffu, dn, 0);
                if (dn + 1 == (uint32_t)items) q_finish_level(a, sl, i, l, L, K, M_s, base, dead, kill);
            }
            __syncthreads();                                  // shared memory is reused by the next pick
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        my_checks += __shfl_down_sync(0xffffffffu, my_checks, o);
        my_tests += __shfl_down_sync(0xffffffffu, my_tests, o);
    }
    if (lane == 0 && my_checks) atomicAdd(&st->checks_exec, my_checks);
    if (lane == 0 && my_tests) atomicAdd(&st->bound_tests, my_tests);
}

// ------------------------------------------------------------------ host side

struct QContext {
    int device = -1, sms = 0;
    uint2 *surv = nullptr;
    uint32_t *bsum = nullptr;
    size_t bsum_words = 0;
    PState *st = nullptr;
    OrderTables *tabs = nullptr;
    int tabs_n = -1;
    QCtl *q = nullptr;
    uint32_t *qdead = nullptr, *qkill = nullptr, *qvals = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::mutex mu;
};

#define QCK(call)                                                                             \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
            return e_ == cudaErrorMemoryAllocation ? GC_ENOMEM : GC_ECUDA;                   \
        }                                                                                     \
    } while (0)

static std::mutex g_qmu;
static QContext *g_qctx[64];

static int q_context(QContext **out) {
    int device;
    QCK(cudaGetDevice(&device));
    std::lock_guard<std::mutex> g(g_qmu);
    if (device < 0 || device >= 64) { set_error("device index out of range"); return GC_EINVAL; }
    QContext *c = g_qctx[device];
    if (!c) {
        c = new QContext;
        c->device = device;
        QCK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
        QCK(cudaMalloc(&c->surv, kPMaxTile * sizeof(uint2)));
        QCK(cudaMalloc(&c->st, sizeof(PState)));
        QCK(cudaMalloc(&c->tabs, sizeof(OrderTables)));
        QCK(cudaMalloc(&c->q, sizeof(QCtl)));
        QCK(cudaMalloc(&c->qdead, (size_t)kQRing * kQWords * 4));
        QCK(cudaMalloc(&c->qkill, (size_t)kQRing * kQWords * 4));
        QCK(cudaMalloc(&c->qvals, (size_t)kQRing * kPMaxTile * 4));
        QCK(cudaEventCreate(&c->ev0));
        QCK(cudaEventCreate(&c->ev1));
        g_qctx[device] = c;
    }
    *out = c;
    return GC_OK;
}

bool pipeline_supported(const RunArgs &a) {
    return a.world == 1 && a.opt.emulate_ranks == 1 && a.opt.tile_max <= kPMaxTile &&
           !(a.opt.flags & (GC_FLAG_NO_EARLY_EXIT | GC_FLAG_FORCE_SEQ_RESOLVE | GC_FLAG_LAUNCHED_TILES |
                            GC_FLAG_TILE_BARRIERS));
}

int pipeline_run(const RunArgs &r) {
    QContext *cx;
    int rc = q_context(&cx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(cx->mu);       // setup, launch and read-back (gc.h)
    cudaStream_t s = (cudaStream_t)r.stream;
    if (cx->tabs_n != (int)r.n) {
        OrderTables t;
        build_order_tables((int)r.n, &t);
        QCK(cudaMemcpy(cx->tabs, &t, sizeof t, cudaMemcpyHostToDevice));
        cx->tabs_n = (int)r.n;
    }
    QCK(cudaMemsetAsync(cx->st, 0, sizeof(PState), s));
    QCK(cudaMemsetAsync(cx->q, 0, sizeof(QCtl), s));
    QCK(cudaMemsetAsync(cx->qdead, 0, (size_t)kQRing * kQWords * 4, s));
    QCK(cudaMemsetAsync(cx->qkill, 0, (size_t)kQRing * kQWords * 4, s));
    // block-bound summaries (AND = all ones, OR = 0 before any append), as in gc_persistent.cu
    const size_t nsup = (size_t)((r.capacity + 1023) / 1024) + 1, nblk = nsup * 32;
    const size_t need = 2 * (nblk + nsup);
    if (cx->bsum_words < need) {
        if (cx->bsum) QCK(cudaFree(cx->bsum));
        cx->bsum = nullptr;
        cx->bsum_words = 0;
        QCK(cudaMalloc(&cx->bsum, need * 4));
        cx->bsum_words = need;
    }
    QCK(cudaMemsetAsync(cx->bsum, 0, need * 4, s));
    QCK(cudaMemset2DAsync(cx->bsum, 8, 0xff, 4, nblk + nsup, s));
    PArgs a;
    p_fill_args(r, &a);
    a.bsum = reinterpret_cast<uint2 *>(cx->bsum);
    a.ssum = reinterpret_cast<uint2 *>(cx->bsum) + nblk;
    a.tabs = cx->tabs;
    a.surv = cx->surv;
    a.st = cx->st;
    a.vals = nullptr;
    a.dead = nullptr;
    a.q = cx->q;
    a.qdead = cx->qdead; a.qkill = cx->qkill; a.qvals = cx->qvals;
    a.depth = (int)std::min<uint32_t>(r.opt.pipeline_depth ? r.opt.pipeline_depth : 4u, (uint32_t)kQRing);
    a.chunk = 2048u;
    const void *kfn = (const void *)k_pipeline<1>;
    size_t smem = p_dyn_smem(a.chunk);
    a.nsup_smem = 0;
    if (a.bound) {
        cudaFuncAttributes fa;
        int optin = 0;
        QCK(cudaFuncGetAttributes(&fa, kfn));
        QCK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cx->device));
        const long long room = (long long)optin - (long long)fa.sharedSizeBytes - (long long)smem;
        const unsigned long long want = (r.capacity + 1023) / 1024 + 1;
        if (room >= 8) a.nsup_smem = (uint32_t)std::min<unsigned long long>(want, (unsigned long long)(room / 8));
        smem += (size_t)a.nsup_smem * 8;
    }
    QCK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    QCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kPThreads, smem));
    if (per_sm < 1) { set_error("k_pipeline cannot be resident"); return GC_ECUDA; }
    int grid = cx->sms;
    if (r.opt.grid_ctas) grid = std::max(2, std::min(grid, (int)r.opt.grid_ctas));   // >= 1 screening CTA
    const uint32_t screen_warps = (uint32_t)(grid - 1) * kPWarps;
    a.plan_warps = r.opt.plan_warps ? r.opt.plan_warps : std::max<uint32_t>(kPWarps, screen_warps / (uint32_t)a.depth);
    void *args[] = {&a};
    QCK(cudaEventRecord(cx->ev0, s));
    QCK(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kPThreads), args, smem, s));
    QCK(cudaEventRecord(cx->ev1, s));
    if (r.stats) {
        QCK(cudaStreamSynchronize(s));
        PState h;
        QCK(cudaMemcpy(&h, cx->st, sizeof(PState), cudaMemcpyDeviceToHost));
        QCtl hq;
        QCK(cudaMemcpy(&hq, cx->q, offsetof(QCtl, slot), cudaMemcpyDeviceToHost));
        float ms = 0;
        QCK(cudaEventElapsedTime(&ms, cx->ev0, cx->ev1));
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
        o->bound_tests = h.bound_tests;
        o->resolve_wait_ms = hq.resolve_wait_ns * 1e-6;
        o->resolve_busy_ms = hq.resolve_busy_ns * 1e-6;
        o->pipeline_depth = (uint32_t)a.depth;
        if (a.timing) {
            PState f;
            QCK(cudaMemcpy(&f, cx->st, sizeof(PState), cudaMemcpyDeviceToHost));
            const double T = (double)f.tiles, c = 1965.0;
            fprintf(stderr, "[gc] pipeline: %llu tiles, depth %d, %.2f us/tile; resolver per tile: wait %.2f busy %.2f us\n",
                    f.tiles, a.depth, ms * 1e3 / T, hq.resolve_wait_ns / T / 1e3, hq.resolve_busy_ns / T / 1e3);
            fprintf(stderr, "[gc]   resolve: gather %.2f conflicts %.2f prior+status %.2f rounds %.2f sequential %.2f "
                    "append %.2f clear+stats %.2f publish %.2f us (SM cycles at 1965 MHz)\n", f.t_r[0] / T / c,
                    f.t_r[1] / T / c, f.t_r[5] / T / c, f.t_r[6] / T / c, f.t_r[2] / T / c, f.t_r[3] / T / c,
                    f.t_r[4] / T / c, f.t_sync / T / c);
            fprintf(stderr, "[gc]   per tile: survivors %.1f, accepted %.1f, resolve checks %.0f, levels %.2f; "
                    "largest S %llu, %llu multi-chunk tiles, %.2f rounds, %.2f sequential\n", f.survivors / T, f.M / T,
                    f.resolve_checks / T, f.levels / T, f.s_max, f.n_chunked, f.n_rounds / T, f.n_seq / T);
        }
        if (h.error) { set_error("codebook capacity exceeded"); return GC_ENOSPC; }
    }
    return GC_OK;
}

}  // namespace gc
