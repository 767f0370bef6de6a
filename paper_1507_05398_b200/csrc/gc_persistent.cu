// gc_persistent.cu -- the device-resident construction: ONE cooperative kernel runs the
// whole greedy scan, tile after tile, with no host round trip.  This is
// the B200 replacement of the paper's per-vector host loop and of its
// dynamic-parallelism parent kernel: the loop itself lives on the GPU.
//
// Per tile of K consecutive ranks [t0, t0+K):
//   levels l = 0 .. L-1   a1+a2: every candidate against the codebook committed before the
//                         tile, newest first, in growing windows, the last one down to 0
//                         (lex with d <= 3: one window).  Work items are WARP-granular:
//                         (64 candidates, one sub-range of the window), claimed from a
//                         per-CTA counter.  A block of 32 codewords is skipped when its
//                         bit-consensus bound is >= d; the blocks that pass are staged in
//                         shared memory and checked (XOR + POPC + min, warp-vote early exit).
//                         Level 0's window is copied to shared memory once per CTA; deeper
//                         levels find their live candidates through a per-CTA prefix of
//                         the tile's dead mask.
//   grid barrier after each level (the dead bits of level l decide level l+1's live set)
//   resolve (CTA 0)       a3: survivors in rank order (tiles with more than 512 are cut after
//                         them); conflict masks, parallel rounds, warp-sequential tail
//                         (PAPER.md:59 inside the tile); a4: append + block summaries.
//   commit token          CTA 0 publishes M and the next tile size (release); the others
//                         wait for it (acquire) -- the commit needs no second barrier.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "gc_screen.cuh"

namespace cg = cooperative_groups;

namespace gc {


template <int kMinBlocks>
__global__ void __launch_bounds__(kPThreads, kMinBlocks) k_construct(PArgs a) {
    const uint32_t kPChunk = a.chunk;
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t C[33][33];
    __shared__ uint64_t off[34];
    __shared__ uint32_t s_ws[33];
    extern __shared__ __align__(16) uint8_t p_dyn[];        // resolve scratch (kPDynSmem bytes)
    uint32_t *s_val = reinterpret_cast<uint32_t *>(p_dyn);
    uint16_t *s_idx = reinterpret_cast<uint16_t *>(p_dyn + kPChunk * 4);
    uint8_t *s_status = p_dyn + kPChunk * 6;
    uint32_t *s_cnt = reinterpret_cast<uint32_t *>(p_dyn + kPChunk * 8);
    uint16_t *s_adj = reinterpret_cast<uint16_t *>(p_dyn + kPChunk * 12);
    uint32_t *s_pre = reinterpret_cast<uint32_t *>(p_dyn + p_scratch_smem(kPChunk));
    uint32_t *s_live = s_pre + kPMaxTile / 32 + 4;
    uint2 *s_sup = reinterpret_cast<uint2 *>(p_dyn + p_dyn_smem(kPChunk));     // [a.nsup_smem]
    __shared__ uint32_t s_basis[32];
    __shared__ unsigned int s_claim;            // per-level item claims of this CTA
    PState *st = a.st;
    if (threadIdx.x < 32) s_basis[threadIdx.x] = a.basis[threadIdx.x];
    const bool graded = a.ord >= GRADED_LEX;
    if (graded) {
        for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) C[i / 33][i % 33] = a.tabs->binom[i / 33][i % 33];
        for (int i = threadIdx.x; i < 34; i += blockDim.x) off[i] = a.tabs->off[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t nwarps = gridDim.x * kPWarps;
    unsigned long long my_checks = 0, my_tests = 0;
    PSmem sm;
    sm.C = C; sm.off = off; sm.s_basis = s_basis; sm.s_ws = s_ws; sm.s_val = s_val; sm.s_idx = s_idx;
    sm.s_status = s_status; sm.s_cnt = s_cnt; sm.s_adj = s_adj; sm.chunk = kPChunk;
    sm.s_tmp = s_pre;                            // the level prefix is not used during a resolve
    sm.tmp_words = 2 * (kPMaxTile / 32);

    __shared__ PCount pc;                     // CTA 0: commit-side state (see PCount)
    if (blockIdx.x == 0 && threadIdx.x == 0) p_count_load(pc, st);
    // diagnostics accumulate in CTA 0's shared memory (only its thread 0 touches them)
    __shared__ PTimers tmr;
    if (a.timing && blockIdx.x == 0 && threadIdx.x == 0) memset(&tmr, 0, sizeof tmr);
    // tile state every thread carries: the codebook size and the next tile size, as published
    // by the commit token (no barrier and no load of M / K_next after a resolve)
    unsigned long long curM = __ldcg(&st->M);
    uint32_t curK = __ldcg(&st->K_next);
    unsigned long long supM = 0;            // the shared super-block mirror is final below supM
    unsigned long long tile_no = 0;
    __shared__ unsigned long long s_tok;
    __shared__ uint32_t s_kused;
    unsigned long long t0 = a.part_mode ? a.t_single : a.t_begin;
    while (t0 < a.t_end) {
        const unsigned long long M = curM;
        uint32_t K = a.part_mode ? a.K_single : curK;
        if (a.nsup_smem) {
            // refresh the mirrored super-block summaries the last commits changed (the partial one
            // and the new ones); every level syncs the CTA before its items read them
            const long long s0 = (long long)(supM >> 10);
            const long long s1 = min((long long)a.nsup_smem, (long long)((M + 1023) >> 10));
            for (long long q = s0 + threadIdx.x; q < s1; q += blockDim.x) s_sup[q] = __ldcg(a.ssum + q);
            supM = M;
        }
        if ((unsigned long long)K > a.t_end - t0) K = (uint32_t)(a.t_end - t0);
        // candidate range screened by this launch: the tile, or one rank's partition of it
        const uint32_t c_lo = a.part_mode ? min(a.part_lo, K) : 0u;
        const uint32_t c_hi = a.part_mode ? min(a.part_lo + a.part_len, K) : K;
        const uint32_t w_lo = c_lo / 32;
        // Weight bound (graded orders, GC_FLAG_NO_WEIGHT_BOUND unset): the codebook is sorted
        // by weight and |wt(v) - wt(c)| <= dist(v, c), so codewords of weight < w_lo - (d-1)
        // (w_lo = weight of the tile's first candidate) are at distance >= d from every
        // candidate of the tile: the screen stops at the first codeword of weight
        // >= w_lo - d + 1.  Exact -- only checks whose outcome is known are skipped.
        const unsigned long long base = p_base(a, t0, M);
        const int L = p_levels(M - base, a.W0, a.growth);
        PTimers *timer = (a.timing && blockIdx.x == 0 && threadIdx.x == 0) ? &tmr : nullptr;
        unsigned long long tm = timer ? p_now() : 0, tm_tile = tm;

        for (int l = 0; l < L; ++l) {
            long long hi, lo;
            p_level_window(a, M, base, L, l, hi, lo);
            // live candidates of this level: level 0 all of them; deeper levels from the dead
            // mask, compacted through a per-CTA prefix over the mask words (every CTA builds it)
            uint32_t n_l = c_hi - c_lo;
            const uint32_t pwords = (c_hi + 31) / 32 - w_lo;      // mask words of the range
            if (l > 0) n_l = p_live_prefix(a.dead, c_lo, c_hi, s_live, s_pre, s_ws);
            const PPlan pl = p_plan(a, n_l, hi - lo, nwarps);
            const int R = pl.R;
            const unsigned long long checks_before = my_checks;
            PLevel lv;
            lv.l = l; lv.n_l = n_l; lv.B = pl.B; lv.nsub = pl.nsub;
            lv.hi = hi; lv.lo = lo; lv.sub = pl.sub; lv.t0 = t0; lv.head = pl.head; lv.J0 = pl.J0;
            lv.s_pre = s_pre; lv.s_live = s_live; lv.words = pwords; lv.basis = s_basis;
            lv.stage = reinterpret_cast<uint32_t *>(p_dyn); lv.s_sup = s_sup; lv.c_lo = c_lo; lv.w_base = w_lo * 32;
            lv.kill = a.dead; lv.vals = a.vals;
            lv.win = nullptr; lv.wsum = nullptr; lv.win_lo = 0;
            if (p_window_in_smem(a, l, hi, lo)) {
                // level 0 with the block bound: every item scans part of the same small window,
                // so each CTA copies it (and its block summaries) to shared memory once
                p_copy_window(a, lv, reinterpret_cast<uint32_t *>(p_dyn + (size_t)kPWarps * kPWarpStage * 4), hi, lo);
            }
            const unsigned long long items = pl.items();
            if (timer) {
                const unsigned long long t = p_now();
                timer->prefix[l] += t - tm;
                timer->live[l] += n_l;
                timer->items_n[l] += items;
            }
            unsigned long long t_it = a.timing ? p_now() : 0;
            // items: CTA c owns items c, c + G, c + 2G, ...; its warps claim them in order from a
            // shared-memory counter (dynamic balance inside the CTA, no global atomics -- one
            // global counter for ~2400 warps serialises at L2 for microseconds)
            if (threadIdx.x == 0) s_claim = 0;
            __syncthreads();
            while (true) {
                unsigned int q = 0;
                if (lane == 0) q = atomicAdd(&s_claim, 1u);
                q = __shfl_sync(0xffffffffu, q, 0);
                const unsigned long long it = blockIdx.x + (unsigned long long)q * gridDim.x;
                if (it >= items) break;
                p_run_item(a, lv, R, it, C, off, my_checks, my_tests);
                if (a.timing && (threadIdx.x & 31) == 0) {
                    const unsigned long long t = p_now();
                    atomicAdd(&st->t_item_sum[l], t - t_it);
                    atomicMax(&st->t_item_max[l & 1], t - t_it);
                    t_it = t;
                }
            }
            if (a.timing) {
                unsigned long long dc = my_checks - checks_before;
                for (int o = 16; o > 0; o >>= 1) dc += __shfl_down_sync(0xffffffffu, dc, o);
                if ((threadIdx.x & 31) == 0 && dc) atomicAdd(&st->c_level[l], dc);
                if ((threadIdx.x & 31) == 0) atomicMax(&st->t_item_end[l & 1], p_now());
            }
            grid.sync();
            if (timer) {
                const unsigned long long t = p_now(), e = __ldcg(&st->t_item_end[l & 1]);
                st->t_item_end[l & 1] = 0;
                timer->item_max[l] += __ldcg(&st->t_item_max[l & 1]);
                st->t_item_max[l & 1] = 0;
                st->scan_max_sum[l] += __ldcg(&st->item_scan_max[l & 1]);
                st->item_scan_max[l & 1] = 0;
                timer->level[l] += t - tm;
                timer->items[l] += e > tm ? e - tm : 0;
                tm = t;
            }
        }

        if (a.part_mode) break;       // the host runs the exchange and k_resolve_tile
        // ------------------------------------------------ resolve + commit (CTA 0)
        // Commit token instead of a grid barrier: every other CTA finished this tile's levels
        // (the last level's barrier), so the commit only has to be broadcast.  CTA 0 resolves,
        // then publishes (release) the token carrying M and log2(K_next); the others wait for it
        // (acquire) and take M and K from it -- no second barrier, no load of M / K_next.
        ++tile_no;
        const unsigned long long gen = tile_no & ((1ull << 24) - 1);
        uint32_t K_used = K;
        if (blockIdx.x == 0) {
            p_resolve(a, sm, t0, K, L, pc, timer, tm, true, a.dead, M);  // ends with __syncthreads
            const bool partial = pc.K_used != K;
            if (threadIdx.x == 0) {
                if (partial) st->K_used = pc.K_used;
                const unsigned long long tok = (gen << 40) | ((unsigned long long)partial << 39) |
                                               ((unsigned long long)(31 - __clz(pc.K_next)) << 34) | pc.M;
                __threadfence();
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&st->token), "l"(tok) : "memory");
            }
            curM = pc.M;
            curK = pc.K_next;
            K_used = pc.K_used;
            if (timer) { const unsigned long long t = p_now(); timer->resolve += t - tm; tm = t; }
        } else {
            if (threadIdx.x == 0) {
                unsigned long long tok;
                do {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(tok) : "l"(&st->token) : "memory");
                } while ((tok >> 40) != gen);
                s_tok = tok;
                s_kused = ((tok >> 39) & 1) ? __ldcg(&st->K_used) : K;
            }
            __syncthreads();
            curM = s_tok & ((1ull << 34) - 1);
            curK = 1u << ((s_tok >> 34) & 31);
            K_used = s_kused;
        }
        if (timer) { const unsigned long long t = p_now(); timer->tile += t - tm_tile; }
        t0 += K_used;
    }
    // work counter: lanes hold per-lane counts
    for (int o = 16; o > 0; o >>= 1) {
        my_checks += __shfl_down_sync(0xffffffffu, my_checks, o);
        my_tests += __shfl_down_sync(0xffffffffu, my_tests, o);
    }
    if (lane == 0 && my_checks) atomicAdd(&st->checks_exec, my_checks);
    if (lane == 0 && my_tests) atomicAdd(&st->bound_tests, my_tests);
    if (!a.part_mode && blockIdx.x == 0 && threadIdx.x == 0) {
        p_count_store(pc, st);
        // capacity overflow: report a count above capacity (gc.h), never a silently truncated code
        *a.d_count = __ldcg(&st->error) ? a.capacity + 1 : pc.M;
    }
    if (a.timing && blockIdx.x == 0 && threadIdx.x == 0) {
        for (int l = 0; l < kPMaxLevels; ++l) {
            st->t_level[l] = tmr.level[l]; st->t_items[l] = tmr.items[l];
            st->t_prefix[l] = tmr.prefix[l]; st->n_live[l] = tmr.live[l]; st->n_items[l] = tmr.items_n[l];
            st->t_itmax[l] = tmr.item_max[l];
        }
        for (int i = 0; i < 8; ++i) st->t_r[i] = tmr.r[i];
        st->t_resolve = tmr.resolve; st->t_sync = tmr.sync; st->t_tile = tmr.tile;
    }
}

// partition mode, one tile: survivors -> resolve -> commit by one CTA (all ranks identically)
__global__ void __launch_bounds__(kPThreads, 1) k_resolve_tile(PArgs a) {
    __shared__ uint32_t C[33][33];
    __shared__ uint64_t off[34];
    __shared__ uint32_t s_ws[33];
    __shared__ uint32_t s_basis[32];
    extern __shared__ __align__(16) uint8_t p_dyn[];
    const uint32_t kPChunk = a.chunk;
    if (threadIdx.x < 32) s_basis[threadIdx.x] = a.basis[threadIdx.x];
    if (a.ord >= GRADED_LEX) {
        for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) C[i / 33][i % 33] = a.tabs->binom[i / 33][i % 33];
        for (int i = threadIdx.x; i < 34; i += blockDim.x) off[i] = a.tabs->off[i];
    }
    __syncthreads();
    PSmem sm;
    sm.C = C; sm.off = off; sm.s_basis = s_basis; sm.s_ws = s_ws;
    sm.s_val = reinterpret_cast<uint32_t *>(p_dyn);
    sm.s_idx = reinterpret_cast<uint16_t *>(p_dyn + kPChunk * 4);
    sm.s_status = p_dyn + kPChunk * 6;
    sm.s_cnt = reinterpret_cast<uint32_t *>(p_dyn + kPChunk * 8);
    sm.s_adj = reinterpret_cast<uint16_t *>(p_dyn + kPChunk * 12);
    sm.chunk = kPChunk;
    sm.s_tmp = reinterpret_cast<uint32_t *>(p_dyn + p_resolve_smem(kPChunk));
    sm.tmp_words = kPResolveTmp;
    __shared__ PCount pc;
    if (threadIdx.x == 0) p_count_load(pc, a.st);
    __syncthreads();
    const unsigned long long M = pc.M;
    uint32_t K = a.K_single;
    if ((unsigned long long)K > a.t_end - a.t_single) K = (uint32_t)(a.t_end - a.t_single);
    const int L = p_levels(M - p_base(a, a.t_single, M), a.W0, a.growth);
    p_resolve(a, sm, a.t_single, K, L, pc, nullptr, 0, false, a.dead, M);
    if (threadIdx.x == 0) {
        p_count_store(pc, a.st);
        *a.d_count = __ldcg(&a.st->error) ? a.capacity + 1 : pc.M;
    }
}

// ------------------------------------------------------------------ host side

struct PContext {
    int device = -1, sms = 0;
    uint32_t *vals = nullptr, *dead = nullptr;
    uint2 *surv = nullptr;
    uint32_t *bsum = nullptr;       // block-bound summaries: (AND, OR) per block, then per super-block
    size_t bsum_words = 0;          // allocated u32 words
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
        PCK(cudaMalloc(&c->surv, kPMaxTile * sizeof(uint2)));
        PCK(cudaMalloc(&c->st, sizeof(PState)));
        PCK(cudaMalloc(&c->tabs, sizeof(OrderTables)));
        PCK(cudaEventCreate(&c->ev0));
        PCK(cudaEventCreate(&c->ev1));
        g_pctx[device] = c;
    }
    *out = c;
    return GC_OK;
}

constexpr uint32_t kPDefaultTile = kPMaxTile;   // adaptive tiles up to this size

bool persistent_supported(const RunArgs &a) {
    return a.world == 1 && a.opt.emulate_ranks == 1 && (a.opt.tile_max == 0 || a.opt.tile_max <= kPMaxTile) &&
           !(a.opt.flags & (GC_FLAG_NO_EARLY_EXIT | GC_FLAG_FORCE_SEQ_RESOLVE | GC_FLAG_LAUNCHED_TILES));
}

static int p_setup(const RunArgs &r, PContext *cx, PArgs *pa);
static int persistent_run_locked(const RunArgs &r, PContext *cx, PArgs &a);

static int p_current_context(PContext **pcx) {
    int device;
    PCK(cudaGetDevice(&device));
    return p_context(device, pcx);
}

// Every call holds the device context's lock from p_setup (which rewrites the shared
// per-device scratch: order tables, PState, masks, summaries) through the launch and the
// stats read-back, so concurrent calls on one device serialise (gc.h).
int persistent_run(const RunArgs &r) {
    PContext *cx;
    int rc = p_current_context(&cx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(cx->mu);
    PArgs a;
    rc = p_setup(r, cx, &a);
    if (rc) return rc;
    return persistent_run_locked(r, cx, a);
}

// caller holds cx->mu
static int p_setup(const RunArgs &r, PContext *cx, PArgs *pa) {
    cudaStream_t s = (cudaStream_t)r.stream;
    // the context's buffers are reused by every call on this device: order this call after the
    // previous one's kernels even when the callers use different streams
    PCK(cudaStreamWaitEvent(s, cx->ev1, 0));
    if (cx->tabs_n != (int)r.n) {
        OrderTables t;
        build_order_tables((int)r.n, &t);
        PCK(cudaMemcpy(cx->tabs, &t, sizeof t, cudaMemcpyHostToDevice));
        cx->tabs_n = (int)r.n;
    }
    PCK(cudaMemsetAsync(cx->st, 0, sizeof(PState), s));
    {
        const uint32_t k0 = std::min<uint32_t>(r.opt.tile_min, r.opt.tile_max ? r.opt.tile_max : kPDefaultTile);
        PCK(cudaMemcpyAsync((char *)cx->st + offsetof(PState, K_next), &k0, sizeof k0, cudaMemcpyHostToDevice, s));
        PCK(cudaStreamSynchronize(s));   // k0 lives on this stack frame
    }
    PCK(cudaMemsetAsync(cx->dead, 0, kPMaxTile / 8, s));
    // block-bound summaries for the whole capacity, (AND, OR) pairs: AND = all ones, OR = 0
    // before any append.  Blocks padded to whole super-blocks (a super-block's 32 block
    // summaries are staged as one 256-byte run).
    const size_t nsup = (size_t)((r.capacity + 1023) / 1024) + 1, nblk = nsup * 32;
    const size_t need = 2 * (nblk + nsup);
    if (cx->bsum_words < need) {
        if (cx->bsum) PCK(cudaFree(cx->bsum));
        cx->bsum = nullptr;
        cx->bsum_words = 0;
        PCK(cudaMalloc(&cx->bsum, need * 4));
        cx->bsum_words = need;
    }
    PCK(cudaMemsetAsync(cx->bsum, 0, need * 4, s));
    PCK(cudaMemset2DAsync(cx->bsum, 8, 0xff, 4, nblk + nsup, s));     // the AND word of every pair
    PArgs a;
    p_fill_args(r, &a);
    a.bsum = reinterpret_cast<uint2 *>(cx->bsum);
    a.ssum = reinterpret_cast<uint2 *>(cx->bsum) + nblk;
    a.tabs = cx->tabs; a.vals = cx->vals; a.dead = cx->dead;
    a.surv = cx->surv;
    a.st = cx->st;
    *pa = a;
    return GC_OK;
}

// The problem and schedule fields of PArgs shared by the persistent engines (library-owned
// device buffers are set by each engine).  Defaults for every knob left 0 in gc_options.
void p_fill_args(const RunArgs &r, PArgs *pa) {
    PArgs a;
    memset(&a, 0, sizeof a);
    const Options &o = r.opt;
    a.nmask = r.n >= 32 ? 0xffffffffu : ((1u << r.n) - 1u);
    a.n = (int)r.n; a.ord = r.ordering; a.d = r.d;
    a.N = 1ull << r.n;
    a.tile_min = o.tile_min; a.tile_max = o.tile_max ? o.tile_max : kPDefaultTile;
    if (a.tile_min > a.tile_max) a.tile_min = a.tile_max;
    const bool graded = r.ordering >= GRADED_LEX && !r.use_basis;
    // lexicographic order, d <= 3, with the block bound: one level over the whole codebook (its tiles
    // candidates are consecutive integers, so a warp's 64 share all but their low 6 bits and the
    // bound alone prunes the deep part; a separate newest-first level costs more than it saves)
    const bool lex_single = !o.window0_set && r.ordering == LEX && r.d <= 3 && !r.use_basis && !r.self_orthogonal &&
                            !(o.flags & GC_FLAG_NO_BLOCK_BOUND);
    a.W0 = lex_single ? (1u << 24) : o.window0;
    // default window growth: without the block bound x4 per level; with it, two levels (newest
    // W0, then everything) for lex / Gray / B-orderings, where the bound skips almost all of a
    // deep window, and x16 for graded orders, where it skips less and compaction pays
    const bool bnd = !r.self_orthogonal && !(o.flags & GC_FLAG_NO_BLOCK_BOUND);
    a.growth = (int)(o.growth ? o.growth : !bnd ? 2u : graded ? 4u : 12u);
    a.mix = (r.d >= 2 && r.d <= 4 && !(o.flags & GC_FLAG_POPC_ONLY)) ? (int)r.d : 0;
    a.codebook = r.d_codebook; a.capacity = r.capacity;
    a.d_count = (unsigned long long *)r.d_count;
    a.timing = (o.flags & GC_FLAG_DEBUG_PHASES) ? 1 : 0;
    a.bound = bnd;
    // with the block bound most of a window is skipped by summary tests: one item per warp and
    // long sub-ranges keep a level to a few dependent round trips
    // (graded orders, whose deep windows pass more blocks, balance better with more, smaller items:
    // warps claim them dynamically)
    a.items_per_warp = o.items_per_warp ? (int)o.items_per_warp : !a.bound ? 2 : graded ? 4 : 1;
    a.sub_max_bound = o.sub_max ? o.sub_max : 262144u;
    a.nsup_smem = 0;                // set by the launcher when shared memory has room
    a.split_bits = o.split_bits ? (int)o.split_bits : lex_single ? kPSplitBits - 2 : kPSplitBits;
    a.geo_head = o.geo_head ? o.geo_head : 8192u;
    a.partial_s = o.partial_s ? o.partial_s : graded ? 1024u : 512u;
    a.burst_chunk = o.burst_chunk ? o.burst_chunk : 512u;
    a.par = (a.bound && r.n <= 30 && !(o.flags & GC_FLAG_NO_PARITY_BOUND)) ? 1 : 0;
    a.target_accepted = o.target_accepted ? o.target_accepted
                        : r.use_basis ? kPTargetAccepted
                        : r.ordering >= GRADED_LEX ? 4 * kPTargetAccepted
                        : r.ordering == GRAY ? 2 * kPTargetAccepted : kPTargetAccepted;
    a.use_basis = r.use_basis;
    for (int i = 0; i < 32; ++i) a.basis[i] = r.basis[i];
    a.so = r.self_orthogonal;
    a.cw = r.constant_weight;
    a.wdef_valid = !(r.self_orthogonal || r.constant_weight >= 0);
    // the weight bound is a distance argument: not valid for the orthogonality constraint
    a.weight_bound = graded && !r.self_orthogonal && !(o.flags & GC_FLAG_NO_WEIGHT_BOUND);
    a.t_begin = 0;
    a.t_end = a.N;
    if (r.constant_weight >= 0 && graded) {
        OrderTables t;
        build_order_tables((int)r.n, &t);
        a.t_begin = t.off[r.constant_weight];        // graded orders: the weight class is one
        a.t_end = t.off[r.constant_weight + 1];      // contiguous block of ranks
    }
    if (a.mix && r.self_orthogonal) a.mix = 0;
    *pa = a;
}

static int persistent_run_locked(const RunArgs &r, PContext *cx, PArgs &a) {
    cudaStream_t s = (cudaStream_t)r.stream;
    int per_sm = 0;
    const void *kfn = (const void *)k_construct<1>;      // one CTA of 16 warps per SM
    a.chunk = 2048u;            // partial tiles keep a persistent tile's survivors <= 1024
    size_t smem = p_dyn_smem(a.chunk);
    // mirror as many super-block summaries in shared memory as fit (one CTA per SM)
    a.nsup_smem = 0;
    if (a.bound && !(r.opt.flags & GC_FLAG_NO_SUP_SMEM)) {
        cudaFuncAttributes fa;
        int optin = 0;
        PCK(cudaFuncGetAttributes(&fa, kfn));
        PCK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cx->device));
        const long long room = (long long)optin - (long long)fa.sharedSizeBytes - (long long)smem;
        const unsigned long long need = (r.capacity + 1023) / 1024 + 1;
        if (room >= 8) a.nsup_smem = (uint32_t)std::min<unsigned long long>(need, (unsigned long long)(room / 8));
        smem += (size_t)a.nsup_smem * 8;
    }
    PCK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kPThreads, smem));
    if (per_sm < 1) { set_error("k_construct cannot be resident"); return GC_ECUDA; }
    void *args[] = {&a};
    PCK(cudaEventRecord(cx->ev0, s));
    int grid = cx->sms;
    if (r.opt.grid_ctas) grid = std::max(1, std::min(grid, (int)r.opt.grid_ctas));
    PCK(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kPThreads), args, smem, s));
    PCK(cudaEventRecord(cx->ev1, s));
    if (r.stats) {
        PCK(cudaStreamSynchronize(s));
        PState h;
        PCK(cudaMemcpy(&h, cx->st, sizeof(PState), cudaMemcpyDeviceToHost));
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
        o->bound_tests = h.bound_tests;
        if (a.timing) {
            PState full;
            PCK(cudaMemcpy(&full, cx->st, sizeof(PState), cudaMemcpyDeviceToHost));
            const double T = (double)full.tiles;
            fprintf(stderr, "[gc] persistent: %llu tiles, per tile: total %.2f us, resolve %.2f us, final sync %.2f us\n",
                    full.tiles, full.t_tile / T / 1e3, full.t_resolve / T / 1e3, full.t_sync / T / 1e3);
            fprintf(stderr, "[gc]   resolve: gather %.2f conflicts %.2f status %.2f rounds %.2f sequential %.2f append %.2f "
                    "clear+stats %.2f us (SM cycles at 1965 MHz)\n", full.t_r[0] / T / 1965.0, full.t_r[1] / T / 1965.0,
                    full.t_r[5] / T / 1965.0, full.t_r[6] / T / 1965.0, full.t_r[2] / T / 1965.0, full.t_r[3] / T / 1965.0,
                    full.t_r[4] / T / 1965.0);
            fprintf(stderr, "[gc]   resolve: per tile %.2f adjacency overflows, %.2f rounds, %.2f sequential nodes; "
                    "largest S %llu, %llu multi-chunk tiles, most rounds %llu\n",
                    full.n_overflow / T, full.n_rounds / T, full.n_seq / T, full.s_max, full.n_chunked, full.n_rounds_max);
            for (int l = 0; l < kPMaxLevels; ++l)
                if (full.t_level[l])
                    fprintf(stderr, "[gc]   level %2d: %.3f s total (%.2f us per tile, last item done at %.2f us), %.3g "
                            "checks, %.1f%% of the mixed/POPC peak (148 SM x 19.18/clk x 1965 MHz)\n", l, full.t_level[l] / 1e9,
                            full.t_level[l] / T / 1e3, full.t_items[l] / T / 1e3, (double)full.c_level[l],
                            100.0 * (double)full.c_level[l] / (full.t_level[l] * 1e-9) / (148.0 * 19.18 * 1.965e9));
            for (int l = 0; l < kPMaxLevels; ++l)
                if (full.t_level[l])
                    fprintf(stderr, "[gc]   level %2d: per tile %.1f live candidates, %.1f items; prefix %.2f us, "
                            "warp item mean %.2f us, longest %.2f us, most codewords scanned by one item %.0f\n", l, full.n_live[l] / T, full.n_items[l] / T,
                            full.t_prefix[l] / T / 1e3, full.t_item_sum[l] / (double)std::max(1ull, full.n_items[l]) / 1e3,
                            full.t_itmax[l] / T / 1e3, full.scan_max_sum[l] / T);
        }
        if (h.error) { set_error("codebook capacity exceeded"); return GC_ENOSPC; }
    }
    return GC_OK;
}

// Multi-GPU / emulated ranks: per tile, every local partition's screen (one cooperative
// launch of k_construct in partition mode each), the NCCL all-gather of the tile's dead
// mask words (world > 1), then k_resolve_tile (one CTA; identical on every rank).  The
// tile schedule is host-side and deterministic (every rank launches the same sequence).
bool persistent_partitioned_supported(const RunArgs &a) {
    return (a.world > 1 || a.opt.emulate_ranks > 1) && (a.opt.tile_max == 0 || a.opt.tile_max <= kPMaxTile) &&
           !(a.opt.flags & (GC_FLAG_NO_EARLY_EXIT | GC_FLAG_FORCE_SEQ_RESOLVE | GC_FLAG_LAUNCHED_TILES));
}

int persistent_run_partitioned(const RunArgs &r) {
    PContext *cx;
    int rc = p_current_context(&cx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(cx->mu);
    PArgs a;
    rc = p_setup(r, cx, &a);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)r.stream;
    const unsigned G = r.world > 1 ? (unsigned)r.world : r.opt.emulate_ranks;
    const unsigned parts_local = r.world > 1 ? 1u : G;
    a.part_mode = 1;
    a.chunk = 2048u;
    const uint32_t tile_max = r.opt.tile_max ? r.opt.tile_max : 16384u;
    const size_t smem = p_dyn_smem(a.chunk);
    PCK(cudaFuncSetAttribute((const void *)k_construct<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PCK(cudaFuncSetAttribute((const void *)k_resolve_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(p_resolve_smem(a.chunk) + kPResolveTmp * 4)));
    int per_sm = 0;
    PCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_construct<1>, kPThreads, smem));
    if (per_sm < 1) { set_error("k_construct cannot be resident"); return GC_ECUDA; }
    unsigned long long launches = 0, tiles = 0;
    PCK(cudaEventRecord(cx->ev0, s));
    unsigned long long t0 = a.t_begin;
    while (t0 < a.t_end) {
        uint32_t K = r.opt.tile_min;
        while (K < tile_max && (unsigned long long)K * 8 <= t0 - a.t_begin) K <<= 1;
        if ((unsigned long long)K > a.t_end - t0) K = (uint32_t)(a.t_end - t0);
        uint32_t plo = 0, plen = 0, Kpad = 0;
        a.t_single = t0;
        a.K_single = K;
        for (unsigned pl = 0; pl < parts_local; ++pl) {
            const unsigned g = r.world > 1 ? (unsigned)r.rank : pl;
            if (gc_tile_partition(K, (int)G, (int)g, &plo, &plen, &Kpad) != GC_OK) return GC_EINTERNAL;
            a.part_lo = plo;
            a.part_len = plen;
            void *args[] = {&a};
            PCK(cudaLaunchCooperativeKernel((const void *)k_construct<1>, dim3(cx->sms), dim3(kPThreads), args,
                                            smem, s));
            ++launches;
        }
        if (r.world > 1) {
            if (gc_tile_partition(K, (int)G, r.rank, &plo, &plen, &Kpad) != GC_OK) return GC_EINTERNAL;
            const uint32_t seg = plen / 32;
            rc = nccl_allgather_u32(cx->dead + (size_t)r.rank * seg, cx->dead, seg, r.nccl_comm, s);
            if (rc) return rc;
        }
        k_resolve_tile<<<1, kPThreads, p_resolve_smem(a.chunk) + kPResolveTmp * 4, s>>>(a);
        ++launches;
        PCK(cudaGetLastError());
        t0 += K;
        ++tiles;
    }
    PCK(cudaEventRecord(cx->ev1, s));
    if (r.stats) {
        PCK(cudaStreamSynchronize(s));
        PState h;
        PCK(cudaMemcpy(&h, cx->st, sizeof(PState), cudaMemcpyDeviceToHost));
        float ms = 0;
        PCK(cudaEventElapsedTime(&ms, cx->ev0, cx->ev1));
        gc_stats *o = r.stats;
        o->struct_size = sizeof(gc_stats);
        o->n_ranks = G;
        o->device_ms = ms;
        o->M = h.M;
        o->tiles = tiles;
        o->phases = h.levels;
        o->checks_exec = h.checks_exec;
        o->survivors = h.survivors;
        o->conflicts = h.conflicts;
        o->resolve_checks = h.resolve_checks;
        o->w_def = (double)h.w_def;
        o->launches = launches;
        o->screen_launches = launches - tiles;
        o->screen_ms = ms;
        o->bound_tests = h.bound_tests;
        if (h.error) { set_error("codebook capacity exceeded"); return GC_ENOSPC; }
    }
    return GC_OK;
}

}  // namespace gc
