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

constexpr int kQRing = kQRingMax;   // tile slots; the pipeline depth D <= kQRing (multi-rank: D <= 7)
constexpr uint32_t kQChunk = 2048;  // survivors per resolve chunk (and per prepared tile)
constexpr uint32_t kQScreened = 0x80;   // QSlot::phase: the tile is screened (level field >= L)
constexpr uint32_t kQWords = kPMaxTile / 32;
constexpr unsigned long long kQM = (1ull << 40) - 1;   // QCtl::cm: committed tiles << 40 | M
// watchdog: the resolver gives up (st->error = 2) when one tile's screen, preparation or peer flags
// have not arrived after this long (a healthy tile takes microseconds to milliseconds)
constexpr unsigned long long kQStallNs = 30ull * 1000 * 1000 * 1000;

// QSlot::prep packs everything the resolver needs from a preparation into one word, so that
// its CAS (or the poll that sees it finished) is the only round trip:
//   tag (tile + 1, 12 bits) << 52 | state << 50 | (M_prep - M_s) (21 bits) << 29
//     | S_prep (13 bits) << 16 | xb (3 bits) << 13 | survivors of the screen (13 bits, saturated)
// (M_prep - M_s counts the words committed since the tile's screen: < depth tiles x 2^16; xb > 0:
// cross lists recorded against the prepared lists of the xb tiles before this one, which were
// not committed when the preparation read M_prep)
constexpr unsigned kPrepOpen = 0, kPrepBusy = 1, kPrepDone = 2, kPrepResolver = 3;
constexpr uint32_t kPrepTooMany = 0x1fff;           // S_prep: more survivors than one resolve chunk
__host__ __device__ constexpr unsigned long long q_pw(unsigned long long i, unsigned st, unsigned long long dM = 0,
                                                      uint32_t S = 0, uint32_t S_screen = 0, uint32_t xb = 0) {
    return (((i + 1) & 0xfffull) << 52) | ((unsigned long long)st << 50) | (dM << 29) |
           ((unsigned long long)S << 16) | ((unsigned long long)(xb & 7u) << 13) |
           (S_screen > 0x1fffu ? 0x1fffu : S_screen);
}
__device__ __forceinline__ unsigned q_pw_state(unsigned long long w) { return (unsigned)(w >> 50) & 3u; }
__device__ __forceinline__ unsigned long long q_pw_dM(unsigned long long w) { return (w >> 29) & ((1ull << 21) - 1); }
__device__ __forceinline__ uint32_t q_pw_S(unsigned long long w) { return (uint32_t)(w >> 16) & 0x1fffu; }
__device__ __forceinline__ uint32_t q_pw_xb(unsigned long long w) { return (uint32_t)(w >> 13) & 7u; }
__device__ __forceinline__ uint32_t q_pw_Sscreen(unsigned long long w) { return (uint32_t)(w & 0x1fffu); }

// One tile in flight (global memory).  The descriptor fields are written by the resolver before
// it releases `phase`; `items[l]` / `nlive[l]` for l >= 1 by the warp that finished level l - 1
// before it releases `phase`; the prepared survivors by the CTA that prepared the tile before it
// releases `prep`.  Every reader acquires `phase` (or `prep`) first and reads the rest from L2.
struct QSlot {
    unsigned long long phase;                   // (tile + 1) << 8 | level; level >= L: screened
    unsigned long long prep;                    // q_pw(tile, state, M_prep, S_prep)
    unsigned long long t_pub, t_scr;            // diagnostics (timing): descriptor published, screen done
    unsigned long long listw;                   // (tile + 1) << 16 | S_prep (0xffff: none): the prepared
                                                // list, published before the cross step (cross lists)
    unsigned long long t0, M_s, base;           // first rank; screened against codebook[base, M_s)
    uint32_t K, L;                              // candidates; levels
    unsigned int inside;                        // CTAs between validating a level and their last claim
    uint32_t cu;                                // 1: level L - 1 is the catch-up level over codebook[M_s, M_x)
    unsigned long long M_x;                     // catch-up: end of its window (set when the level opens)
    uint32_t items[kPMaxLevels];                // warp items of each level
    uint32_t nlive[kPMaxLevels];                // live candidates at the start of each level
    uint32_t done[kPMaxLevels];                 // items finished (arrival counter)
    unsigned long long claim[kPMaxLevels];      // ((tile + 1) mod 2^32) << 32 | items claimed
};
struct QCtl {
    unsigned long long cm;                      // committed tiles << 40 | M after them (release; resolver)
    unsigned int finished;                      // every tile committed
    unsigned int pad;
    unsigned long long resolve_wait_ns;         // diagnostics: resolver time waiting for screens
    unsigned long long resolve_busy_ns;         //              and resolving
    unsigned long long preps, prep_used;        // diagnostics: tiles prepared / resolved from a prep
    unsigned long long prep_rchk;               // resolve checks done by preparations
    unsigned long long busy_prep_ns;            // diagnostics: resolver busy time on prepared tiles
    unsigned long long n_xmode;                 // diagnostics (timing): tiles resolved in cross mode
    unsigned long long prep_ns, xcross_ns, n_xb;              // diagnostics (timing): stage A time, stage B
                                                // time, stage B count
    unsigned long long arr[4], scr_ns, lag_ns, n_scr;        // diagnostics (timing): resolver arrivals at a tile
                                                // unscreened / screened but open / prep busy / prep done;
                                                // publish -> screened; screened -> resolver arrival
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
__device__ __forceinline__ void q_st_release32(unsigned int *p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// a strong store that, after a fence, completes a release pattern (PTX memory model)
__device__ __forceinline__ void q_st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned int q_atom_add_acqrel(unsigned int *p, unsigned int v) {
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long q_cas_acqrel(unsigned long long *p, unsigned long long cmp,
                                                           unsigned long long val) {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "l"(p), "l"(cmp), "l"(val)
                 : "memory");
    return old;
}

// Release / acquire fence at GPU scope: every publication in this engine is data stores, this
// fence, then a relaxed flag store (or atomic), read back with ld.acquire -- the PTX release
// pattern, which needs no sequentially consistent fence (__threadfence is fence.sc.gpu)
__device__ __forceinline__ void q_fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned long long q_ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int q_ld_relaxed32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long q_ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void q_st_relaxed_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// This rank's share of a tile's screen: candidates [plo, plo + n0) of the K, whole 32-bit mask
// words (the partition of gc_tile_partition: K padded to 32 x world, equal parts in rank order).
__device__ __forceinline__ void q_part(const PArgs &a, uint32_t K, uint32_t &plo, uint32_t &n0) {
    if (a.world <= 1) { plo = 0; n0 = K; return; }
    const uint32_t qq = 32u * (uint32_t)a.world, kp = (K + qq - 1) / qq * qq, plen = kp / (uint32_t)a.world;
    plo = (uint32_t)a.rank * plen;
    n0 = plo < K ? min(plen, K - plo) : 0u;
}

// Every rank's partition of tile i (slot si) is in this rank's dead mask (multi-rank engine).
__device__ __forceinline__ bool q_peers_in(const PArgs &a, int si, unsigned long long i) {
    if (a.world <= 1) return true;
    const unsigned long long *f = a.peer_flag[a.rank] + (size_t)si * kMaxRanks;
    for (int g = 0; g < a.world; ++g)
        if (q_ld_acquire_sys(f + g) != i + 1) return false;
    return true;
}

// Multi-rank engine, one full warp: store this rank's partition words of tile i's dead mask into
// every other rank's ring (peer memory over NVLink / NVSwitch, or another emulated rank's
// buffer), then raise this rank's flag for the tile on every rank (after a system-scope fence).
// data = false: the partition has nothing to send (empty, or no level ran).
__device__ __forceinline__ void q_push(const PArgs &a, int si, unsigned long long i, uint32_t K, const uint32_t *dead,
                                       bool data) {
    if (a.world <= 1) return;
    const int lane = threadIdx.x & 31;
    if (data) {
        uint32_t plo, n0;
        q_part(a, K, plo, n0);
        const uint32_t w_lo = plo / 32, w_hi = (plo + n0 + 31) / 32;
        for (int g = 0; g < a.world; ++g) {
            if (g == a.rank) continue;
            uint32_t *dst = a.peer_qdead[g] + (size_t)si * kQWords;
            for (uint32_t w = w_lo + lane; w < w_hi; w += 32) __stcg(dst + w, __ldcg(dead + w));
        }
    }
    __threadfence_system();
    __syncwarp();
    if (lane < a.world) q_st_relaxed_sys(a.peer_flag[lane] + (size_t)si * kMaxRanks + a.rank, i + 1);
    __syncwarp();
}

// Resolver thread 0, multi-rank engine: tile i was published with nothing for this rank to screen
// (no level, or an empty partition): raise this rank's flag for it on every rank.
__device__ __forceinline__ void q_flag_empty(const PArgs &a, int si, unsigned long long i) {
    if (a.world <= 1) return;
    __threadfence_system();
    for (int g = 0; g < a.world; ++g) q_st_relaxed_sys(a.peer_flag[g] + (size_t)si * kMaxRanks + a.rank, i + 1);
}

// Resolver thread 0: make the slot of tile i reusable -- its previous tile is long committed, but
// CTAs that validated one of its levels may still be about to claim items from it (a claim is an
// add), so the counters are reset only once none is inside.  Done ahead of time (while waiting
// for a screen) when the ring is deeper than the pipeline.
// (nlev: the most levels a tile of this run can have, PArgs::reset_levels)
__device__ __forceinline__ void q_reset(QCtl *q, unsigned long long i, int nlev, unsigned int inside_seen = 1u) {
    QSlot &sl = q->slot[i % kQRing];
    // `inside` of a committed tile's slot only decreases: a 0 read earlier (acquire) stays valid
    if (inside_seen != 0)
        while (q_ld_acquire32(&sl.inside) != 0) __nanosleep(32);
    const unsigned long long tag = (i + 1) & 0xffffffffull;
    for (int l = 0; l < nlev; ++l) { sl.claim[l] = tag << 32; sl.done[l] = 0; }
}

// Levels of a tile screened against codebook[base, M_s): the window levels, plus (pipelined engine,
// one rank, GC_FLAG_NO_CATCHUP off) a last catch-up level over the words committed meanwhile.
__device__ __forceinline__ int q_levels(const PArgs &a, unsigned long long M_s, unsigned long long base, uint32_t &cu) {
    const int L = p_levels(M_s - base, a.W0, a.growth);
    cu = (a.cm && a.world <= 1 && L > 0 && L < kPMaxLevels) ? 1u : 0u;
    return L + (int)cu;
}
// window [lo, hi) of level l of a tile with L levels (cu, M_x: its catch-up level)
__device__ __forceinline__ void q_level_window(const PArgs &a, unsigned long long M_s, unsigned long long base, int L,
                                               uint32_t cu, unsigned long long M_x, int l, long long &hi, long long &lo) {
    if (cu && l == L - 1) { hi = (long long)M_x; lo = (long long)M_s; return; }
    p_level_window(a, M_s, base, L - (int)cu, l, hi, lo);
}

// Resolver thread 0: write the descriptor of tile i (ranks [t0, t0 + K)) to be screened against
// codebook[base, M_s) into its (reset) slot.  Level 0 plans all K candidates; a tile with nothing
// to screen (L == 0) is published as already screened.  Returns the phase word; the caller makes
// everything visible with a fence and then stores it.
__device__ __forceinline__ unsigned long long q_write(const PArgs &a, QCtl *q, unsigned long long i,
                                                      unsigned long long t0, uint32_t K, unsigned long long M_s,
                                                      unsigned long long base) {
    QSlot &sl = q->slot[i % kQRing];
    uint32_t cu;
    const int L = q_levels(a, M_s, base, cu);
    sl.t0 = t0; sl.K = K; sl.M_s = M_s; sl.base = base; sl.L = (uint32_t)L;
    sl.cu = cu; sl.M_x = 0;
    uint32_t plo, n0;
    q_part(a, K, plo, n0);
    if (L > 0 && n0 > 0) {
        long long hi, lo;
        p_level_window(a, M_s, base, L - (int)cu, 0, hi, lo);
        sl.items[0] = (uint32_t)p_plan(a, n0, hi - lo, a.plan_warps).items();
        sl.nlive[0] = n0;
    }
    sl.prep = q_pw(i, kPrepOpen, 0, 0);
    // the phase to open: level 0, or screened when this rank has nothing to screen
    return ((i + 1) << 8) | (L > 0 && n0 > 0 ? 0u : (kQScreened | (uint32_t)L));
}

// The warp that finished the last item of level l of tile i: merge the level's kills into the
// tile's dead mask, count the live candidates, plan level l + 1 and open it (or mark the tile
// screened when nothing is left to screen).
__device__ __forceinline__ void q_finish_level(const PArgs &a, QSlot *sl, unsigned long long i, int l, int L,
                                               uint32_t K, unsigned long long M_s, unsigned long long base,
                                               uint32_t *dead, uint32_t *kill) {
    q_fence();                                  // acquire side of the items' release
    const int lane = threadIdx.x & 31;
    uint32_t plo, n0;
    q_part(a, K, plo, n0);
    const uint32_t c_hi = plo + n0;
    uint32_t live = 0;
    for (uint32_t w = plo / 32 + lane; w < (c_hi + 31) / 32; w += 32) {
        const uint32_t k = __ldcg(kill + w);
        uint32_t dd = __ldcg(dead + w);
        if (k) {
            dd |= k;
            __stcg(dead + w, dd);
            __stcg(kill + w, 0u);
        }
        uint32_t lv = ~dd;
        if (w * 32 + 32 > c_hi) lv &= (1u << (c_hi - w * 32)) - 1u;
        live += __popc(lv);
    }
    live = __reduce_add_sync(0xffffffffu, live);
    int nl = l + 1;
    uint32_t items = 0;
    const uint32_t cu = __ldcg(&sl->cu);
    if (nl < L && live > 0) {
        long long hi, lo;
        if (cu && nl == L - 1) {
            // the catch-up level: the words committed since the descriptor (read now), so that the
            // preparation and the resolver check the survivors against fewer of them
            unsigned long long mx = 0;
            if (lane == 0) mx = q_ld_acquire(a.cm) & kQM;
            mx = __shfl_sync(0xffffffffu, mx, 0);
            hi = (long long)mx; lo = (long long)M_s;
            if (lane == 0) sl->M_x = mx;
        } else {
            p_level_window(a, M_s, base, L - (int)cu, nl, hi, lo);
        }
        if (hi > lo) items = (uint32_t)p_plan(a, live, hi - lo, a.plan_warps).items();
    }
    if (items == 0) nl = L;                           // nothing left to screen
    __syncwarp();
    if (nl >= L) q_push(a, (int)(i % kQRing), i, K, dead, true);   // multi-rank: share the partition
    if (lane == 0) {
        if (nl < L) {
            sl->items[nl] = items;
            sl->nlive[nl] = live;
        }
        if (a.timing && nl >= L) sl->t_scr = p_now();
        q_fence();
        q_st_relaxed(&sl->phase, ((i + 1) << 8) | (nl >= L ? kQScreened : 0u) | (unsigned)nl);
    }
    __syncwarp();
}

// Stage B of a preparation (cross lists), run by a preparing CTA on tile j = com + 1 while tile
// com is being resolved; stage A (p_prep, any time after the screen) left the tile's survivors
// checked against codebook[0, M_cA) in its prep buffer and published them as its list (word w).
// Stage B flags the survivors in conflict with the words committed since, codebook[M_cA, M_cB)
// (M_cB: the codebook after tile com - 1), and records their conflicts with the list of tile com
// -- a superset of the words tile com will add, at the positions the resolver decides it in
// (cross lists, kPX per survivor; xcnt = 0xff: flagged).  The resolver then needs no check
// against committed words at all.  Returns the new prep word: xb = 1 (M_prep = M_cB), or xb = 7
// when a survivor has more than kPX cross conflicts (the flags are kept, the cross lists are not
// used: the resolver checks codebook[M_cA, M) itself).  Ends with a barrier.
__device__ __forceinline__ unsigned long long q_stage_b(const PArgs &a, const PSmem &sm, unsigned long long j,
                                                        unsigned long long w, unsigned long long M_s,
                                                        unsigned long long M_cB, uint32_t S_prev, uint8_t *buf,
                                                        unsigned long long &rchk) {
    __shared__ XList s_xl[1];
    __shared__ int s_ovf;
    const uint32_t tid = threadIdx.x;
    const uint32_t S = q_pw_S(w);
    const unsigned long long M_cA = M_s + q_pw_dM(w);
    const uint32_t *val = reinterpret_cast<const uint32_t *>(buf);
    uint16_t *xadj = reinterpret_cast<uint16_t *>(buf + p_prep_xadj(sm.chunk));
    uint8_t *xcnt = buf + p_prep_xcnt(sm.chunk);
    for (uint32_t k = tid; k < S; k += blockDim.x) {
        sm.s_val[k] = __ldcg(val + k);
        sm.s_cnt[k] = 0;
    }
    if (tid == 0) {
        s_ovf = 0;
        s_xl[0].val = reinterpret_cast<const uint32_t *>(a.qprep + (size_t)((j - 1) % kQRing) * p_prep_bytes(sm.chunk));
        s_xl[0].S = S_prev;
    }
    __syncthreads();
    r_consensus(sm, S);
    r_prior(a, sm, S, M_cA, M_cB > M_cA ? M_cB : M_cA, false, rchk);   // s_status: flagged (zeroed first)
    if (S_prev) r_cross(a, sm, S, s_xl, 1, xadj, rchk);
    for (uint32_t k = tid; k < S; k += blockDim.x) {
        const uint32_t c = sm.s_cnt[k];
        const bool flagged = sm.s_status[k] != 0;
        if (!flagged && c > (uint32_t)kPX) s_ovf = 1;
        __stcg(xcnt + k, flagged ? (uint8_t)0xff : (uint8_t)min(c, 254u));
    }
    __syncthreads();
    return s_ovf ? q_pw(j, kPrepDone, q_pw_dM(w), S, q_pw_Sscreen(w), 7)
                 : q_pw(j, kPrepDone, (M_cB > M_cA ? M_cB : M_cA) - M_s, S, q_pw_Sscreen(w), 1);
}

// the resolve scratch of a CTA in the dynamic shared memory (the level stages alias it)
__device__ __forceinline__ PSmem q_smem(const PArgs &a, uint8_t *p_dyn, const uint32_t (*C)[33], const uint64_t *off,
                                        const uint32_t *s_basis, uint32_t *s_ws, uint32_t *s_pre) {
    PSmem sm;
    const uint32_t ch = a.chunk;
    sm.C = C; sm.off = off; sm.s_basis = s_basis; sm.s_ws = s_ws;
    sm.s_val = reinterpret_cast<uint32_t *>(p_dyn);
    sm.s_idx = reinterpret_cast<uint16_t *>(p_dyn + ch * 4);
    sm.s_status = p_dyn + ch * 6;
    sm.s_cnt = reinterpret_cast<uint32_t *>(p_dyn + ch * 8);
    sm.s_adj = reinterpret_cast<uint16_t *>(p_dyn + ch * 12);
    sm.chunk = ch;
    sm.s_tmp = s_pre;                      // the level prefix area is free outside a level
    sm.tmp_words = kPTmpMaxWords;
    return sm;
}

// The whole construction as one persistent kernel body; `bid` is the CTA's index within its rank
// (the kernel may hold several emulated ranks, each a group of CTAs).
__device__ __forceinline__ void q_body(const PArgs &a, int bid) {
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
    const PSmem sm = q_smem(a, p_dyn, C, off, s_basis, s_ws, s_pre);

    if (bid == 0) {
        // ------------------------------------------------------------------ resolver
        __shared__ PCount pc;
        __shared__ unsigned long long s_t0[kQRing], s_Ms[kQRing];
        __shared__ uint32_t s_K[kQRing], s_L[kQRing];
        __shared__ unsigned long long s_next, s_issued;
        __shared__ int s_mode;
        __shared__ unsigned long long s_plo;             // mode 0: survivors screened against codebook[0, s_plo)
        __shared__ PPrep s_pp;
        __shared__ uint32_t s_xbits[kPXRing][64];        // accepted positions of the last tiles' lists
        __shared__ unsigned long long s_listed[kPXRing]; // tile + 1 when resolved from its prepared list
        if (threadIdx.x < kPXRing) s_listed[threadIdx.x] = 0;
        const bool pre_reset = a.depth < kQRing;         // slot of tile i + D reset during tile i
        if (threadIdx.x == 0) {
            p_count_load(pc, st);
            s_next = a.t_begin;
            s_issued = 0;
            // the first D tiles are screened against the empty codebook (nothing to screen)
            for (int i = 0; i < a.depth && s_next < a.t_end; ++i) {
                const uint32_t K = (uint32_t)min((unsigned long long)a.tile_min, a.t_end - s_next);
                s_t0[i] = s_next; s_K[i] = K; s_Ms[i] = 0; s_L[i] = 0;
                q_reset(q, (unsigned long long)i, a.reset_levels);
                const unsigned long long ph = q_write(a, q, (unsigned long long)i, s_next, K, 0, 0);
                q_fence();
                q_st_relaxed(&q->slot[i].phase, ph);
                q_flag_empty(a, i, (unsigned long long)i);        // nothing to screen (L == 0)
                s_next += K;
                ++s_issued;
            }
        }
        unsigned long long t_wait = 0, t_busy = 0, t_pub = 0, n_used = 0, t_bprep = 0, tb0 = 0;
        unsigned long long w_ahead = 0;    // thread 0: the next tile's prep word, read ahead
        unsigned int in_ahead = 1u;        // thread 0: `inside` of the slot the next tile resets, read ahead
        PTimers tmr;
        if (a.timing && threadIdx.x == 0) memset(&tmr, 0, sizeof tmr);
        PTimers *timer = (a.timing && threadIdx.x == 0) ? &tmr : nullptr;
        unsigned long long t_top_p = 0, t_pub_p = 0, t_rp[8] = {0}, t_r0[8];   // diagnostics: prepared tiles
        __shared__ int s_stall;
        if (threadIdx.x == 0) s_stall = 0;
        for (unsigned long long i = 0;; ++i) {
            __syncthreads();
            if (i >= s_issued || s_stall) break;
            const int si = (int)(i % kQRing);
            QSlot *sl = &q->slot[si];
            if (threadIdx.x == 0) {
                const unsigned long long tw = p_now();
                {
                    if (a.timing) {      // what the resolver finds on arrival
                        const unsigned long long ph = q_ld_acquire(&sl->phase), pw = q_ld_acquire(&sl->prep);
                        const bool scr = (ph >> 8) == i + 1 && (uint32_t)(ph & 0xff) >= s_L[si];
                        const unsigned ps = q_pw_state(pw);
                        q->arr[!scr ? 0 : ps == kPrepOpen ? 1 : ps == kPrepBusy ? 2 : 3]++;
                        const unsigned long long ts = __ldcg(&sl->t_scr), tpb = __ldcg(&sl->t_pub);
                        if (scr && ts && tpb && ts > tpb) { q->scr_ns += ts - tpb; q->lag_ns += tw > ts ? tw - ts : 0; q->n_scr++; }
                    }
                    if (pre_reset && s_next < a.t_end) q_reset(q, i + a.depth, a.reset_levels, i ? in_ahead : 1u);
                    // Prepared by another CTA?  One CAS: it either hands over the finished preparation
                    // or takes the tile over (nobody started on it: this CTA does all of it).
                    int mode = 0;
                    bool need_phase = true;
                    if (a.prep_lead > 0) {
                        const unsigned long long open = q_pw(i, kPrepOpen, 0, 0);
                        // the word read (acquire) while the previous commit was being published: a
                        // finished preparation is final, anything else needs the CAS
                        unsigned long long w = w_ahead;
                        if (!(w >> 52 == ((i + 1) & 0xfffull) && q_pw_state(w) == kPrepDone))
                            w = q_cas_acqrel(&sl->prep, open, q_pw(i, kPrepResolver, 0, 0));
                        if (w != open) {
                            while (q_pw_state(w) != kPrepDone) {
                                __nanosleep(32);
                                w = q_ld_acquire(&sl->prep);
                                if (p_now() - tw > kQStallNs) { s_stall = 1; break; }
                            }
                            need_phase = false;               // prepared implies screened
                            if (q_pw_S(w) != kPrepTooMany) {
                                const uint8_t *buf = a.qprep + (size_t)si * p_prep_bytes(kPChunk);
                                s_pp.S = q_pw_S(w);
                                s_pp.S_screen = q_pw_Sscreen(w);
                                s_pp.M_prep = s_Ms[si] + q_pw_dM(w);
                                s_pp.val = reinterpret_cast<const uint32_t *>(buf);
                                s_pp.cnt = reinterpret_cast<const uint32_t *>(buf + (size_t)kPChunk * 4);
                                s_pp.idx = reinterpret_cast<const uint16_t *>(buf + (size_t)kPChunk * 8);
                                s_pp.adj = reinterpret_cast<const uint16_t *>(buf + (size_t)kPChunk * 10);
                                s_pp.xcnt = buf + p_prep_xcnt(kPChunk);
                                s_pp.xadj = reinterpret_cast<const uint16_t *>(buf + p_prep_xadj(kPChunk));
                                s_pp.xbits = s_xbits;
                                s_pp.tile = i;
                                // stage B ran (xb 1 or 7): xcnt flags the survivors in conflict with
                                // codebook[M_cA, M_prep); cross mode (xb 1): the tile before was
                                // resolved from its list (then codebook[M_prep, M) are exactly its
                                // accepted words, and the cross lists say which survivors they reject)
                                const uint32_t xb = q_pw_xb(w);
                                s_pp.xstage = xb != 0;
                                const bool xm = a.cross && xb == 1 && i >= 1 && s_listed[(i - 1) % kPXRing] == i;
                                s_pp.xmode = xm;
                                if (xm && a.timing) q->n_xmode++;
                                mode = 1;
                                ++n_used;
                            }
                        }
                    }
                    if (need_phase) {
                        for (;;) {
                            const unsigned long long ph = q_ld_acquire(&sl->phase);
                            if ((ph >> 8) == i + 1 && (uint32_t)(ph & 0xff) >= s_L[si] && q_peers_in(a, si, i)) break;
                            __nanosleep(32);
                            if (p_now() - tw > kQStallNs) { s_stall = 1; break; }
                        }
                    }
                    s_mode = mode;
                    // the screen covered codebook[0, M_x) when its catch-up level ran
                    s_plo = max(s_Ms[si], __ldcg(&sl->cu) ? __ldcg(&sl->M_x) : 0ull);
                    const unsigned long long tb = p_now();
                    if (mode) t_top_p += tb - tw;
                    t_wait += tb - tw;
                    t_busy -= tb;
                    tb0 = tb;
                }
            }
            __syncthreads();
            if (s_stall) break;          // watchdog: a screen, a preparation or a peer never arrived
            uint32_t *dead = a.qdead + (size_t)si * kQWords;
            if (timer)
                for (int k = 0; k < 8; ++k) t_r0[k] = tmr.r[k];
            p_resolve(a, sm, s_t0[si], s_K[si], (int)s_L[si], pc, timer, 0, false, dead, s_plo,
                      s_mode ? &s_pp : nullptr, (s_mode && a.cross) ? s_xbits[i % kPXRing] : nullptr);
            if (timer && s_mode)
                for (int k = 0; k < 8; ++k) t_rp[k] += tmr.r[k] - t_r0[k];
            if (threadIdx.x == 0) {
                const unsigned long long tp = timer ? clock64() : 0;
                // (a prepared burst decided in sub-chunks has no accepted positions in its list)
                s_listed[i % kPXRing] = (s_mode && !p_prep_big(a, s_pp)) ? i + 1 : 0;
                // next descriptor: tile s_issued, screened against the codebook as of now; its
                // size follows the tile just resolved (p_resolve's pc.K_next)
                unsigned long long ph = 0, *php = nullptr;
                if (s_next < a.t_end) {
                    uint32_t Kn = pc.K_next;
                    if ((unsigned long long)Kn > a.t_end - s_next) Kn = (uint32_t)(a.t_end - s_next);
                    const unsigned long long base = p_base(a, s_next, pc.M);
                    const int sj = (int)(s_issued % kQRing);
                    if (!pre_reset) q_reset(q, s_issued, a.reset_levels);
                    s_t0[sj] = s_next; s_K[sj] = Kn; s_Ms[sj] = pc.M;
                    uint32_t cu_;
                    s_L[sj] = (uint32_t)q_levels(a, pc.M, base, cu_);
                    ph = q_write(a, q, s_issued, s_next, Kn, pc.M, base);
                    if (a.timing) { q->slot[sj].t_pub = p_now(); q->slot[sj].t_scr = 0; }
                    php = &q->slot[sj].phase;
                    s_next += Kn;
                    ++s_issued;
                }
                // look at the next tile's preparation now: relaxed loads, both in flight at once; the
                // fence below completes after them and makes them acquires (fence.acq_rel after a
                // strong read is the PTX acquire pattern)
                if (a.prep_lead > 0 && i + 1 < s_issued) w_ahead = q_ld_relaxed(&q->slot[(i + 1) % kQRing].prep);
                if (pre_reset) in_ahead = q_ld_relaxed32(&q->slot[(i + 1 + a.depth) % kQRing].inside);
                // one fence releases the tile's appended words and summaries (the whole CTA's,
                // ordered by the barrier at the end of p_resolve) and the new descriptor
                q_fence();
                if (php) {
                    q_st_relaxed(php, ph);
                    if ((uint32_t)(ph & 0xff) >= s_L[(int)((s_issued - 1) % kQRing)])   // nothing to screen here
                        q_flag_empty(a, (int)((s_issued - 1) % kQRing), s_issued - 1);
                }
                q_st_relaxed(&q->cm, ((i + 1) << 40) | pc.M);
                const unsigned long long te = p_now();
                t_busy += te;
                if (s_mode) t_bprep += te - tb0;
                if (timer) { t_pub += clock64() - tp; if (s_mode) t_pub_p += clock64() - tp; }
            }
        }
        if (threadIdx.x == 0) {
            if (s_stall) st->error = 2;
            q_st_release32(&q->finished, 1u);
            pc.resolve_checks += __ldcg(&q->prep_rchk);   // every preparation was consumed (acquired)
            p_count_store(pc, st);
            *a.d_count = __ldcg(&st->error) ? a.capacity + 1 : pc.M;   // above capacity: incomplete (gc.h)
            q->resolve_wait_ns = t_wait;
            q->resolve_busy_ns = t_busy;
            q->prep_used = n_used;
            q->busy_prep_ns = t_bprep;
            if (timer) {
                for (int k = 0; k < 8; ++k) {
                    st->t_r[k] = tmr.r[k];
                    st->t_level[k] = t_rp[k];
                }
                st->t_sync = t_pub;
                st->t_level[8] = t_pub_p;
                st->t_level[9] = t_top_p;
            }
        }
    } else {
        // ------------------------------------------------------------------ screen / prep
        // CTAs 1 .. prep_ctas only prepare tiles for the resolver; the others screen, and prepare
        // too when a tile is ready and they are between levels.
        const bool prep_only = bid <= a.prep_ctas;
        __shared__ unsigned long long s_tile, s_t0, s_Ms, s_base, s_Mc, s_wA;
        __shared__ uint32_t s_K, s_L, s_Sprev, s_cu;
        __shared__ unsigned long long s_Mx;
        __shared__ int s_lvl;                 // >= 0: a level; -2: finished; -3: prepare s_tile (stage A); -4: stage B
        unsigned long long hint = 0, supM = 0, n_prep = 0;
        for (;;) {
            if (threadIdx.x == 0) {
                int lvl = -1;
                unsigned long long pick = 0, Mc = 0, c0 = 0;
                uint32_t sprev = 0;
                unsigned int nap = 32;
                for (;;) {
                    const unsigned long long cmv = q_ld_acquire(&q->cm);
                    const unsigned long long com = cmv >> 40;
                    // 0. stage B of the tile after the one being resolved (the resolver's next tile)
                    if (a.stage_b) {
                        const unsigned long long j = com + 1;
                        QSlot *sl = &q->slot[j % kQRing];
                        const unsigned long long w = q_ld_acquire(&sl->prep);
                        // (only when words were committed since its stage A)
                        if ((w >> 52) == ((j + 1) & 0xfffull) && q_pw_state(w) == kPrepDone && q_pw_xb(w) == 0 &&
                            q_pw_S(w) != kPrepTooMany && q_pw_S(w) != 0 && __ldcg(&sl->M_s) + q_pw_dM(w) < (cmv & kQM)) {
                            // cross lists need the list of the tile being resolved
                            const unsigned long long lw = a.cross ? q_ld_acquire(&q->slot[com % kQRing].listw) : 0ull;
                            if (!a.cross || ((lw >> 16) == com + 1 && (lw & 0xffffu) != 0xffffu)) {
                                const unsigned long long wb = (w & ~(3ull << 50)) | ((unsigned long long)kPrepBusy << 50);
                                if (atomicCAS(&sl->prep, w, wb) == w) {
                                    pick = j;
                                    Mc = cmv & kQM;
                                    c0 = w;
                                    sprev = a.cross ? (uint32_t)(lw & 0xffffu) : 0u;
                                    lvl = -4;
                                    break;
                                }
                            }
                        }
                    }
                    // 1. prepare (stage A) a screened tile the resolver reaches soon
                    for (unsigned long long j = com + 1; a.prep_lead > 0 && j <= com + (unsigned long long)a.prep_lead &&
                                                         j < com + (unsigned long long)a.depth; ++j) {
                        QSlot *sl = &q->slot[j % kQRing];
                        // one round trip: the phase and the prep word together, made acquires by
                        // the fence (the screened flag of the phase needs no load of L)
                        const unsigned long long ph = q_ld_relaxed(&sl->phase), pw = q_ld_relaxed(&sl->prep);
                        q_fence();
                        if ((ph >> 8) != j + 1 || !(ph & kQScreened)) continue;
                        if (!q_peers_in(a, (int)(j % kQRing), j)) continue;
                        const unsigned long long open = q_pw(j, kPrepOpen, 0, 0);
                        if (pw != open) continue;
                        if (atomicCAS(&sl->prep, open, q_pw(j, kPrepBusy, 0, 0)) == open) {
                            pick = j;
                            Mc = cmv & kQM;
                            lvl = -3;
                            break;
                        }
                    }
                    if (lvl == -3) break;
                    // 2. a level with items left
                    if (hint < com) hint = com;
                    for (unsigned long long i = hint; !prep_only && i < com + (unsigned long long)a.depth; ++i) {
                        QSlot *sl = &q->slot[i % kQRing];
                        const unsigned long long ph = q_ld_acquire(&sl->phase);
                        if ((ph >> 8) != i + 1) break;           // not published yet
                        const uint32_t l = (uint32_t)(ph & 0x7f);
                        if (ph & kQScreened) {                       // screened
                            if (i == hint) ++hint;
                            continue;
                        }
                        const unsigned long long c = __ldcg(&sl->claim[l]);
                        if ((c >> 32) == ((i + 1) & 0xffffffffull) && (uint32_t)c < __ldcg(&sl->items[l])) {
                            // validate with the slot pinned: once `inside` is raised the slot is not
                            // reset before this CTA's last claim
                            q_atom_add_acqrel(&sl->inside, 1u);
                            if (q_ld_acquire(&sl->phase) == ph) {
                                pick = i;
                                lvl = (int)l;
                                break;
                            }
                            atomicSub(&sl->inside, 1u);
                        }
                    }
                    if (lvl >= 0 || lvl == -4) break;
                    if (q_ld_acquire32(&q->finished)) { lvl = -2; break; }
                    __nanosleep(nap);
                    if (nap < (prep_only ? 64u : 512u)) nap *= 2;
                }
                s_lvl = lvl;
                if (lvl >= 0 || lvl <= -3) {
                    QSlot *sl = &q->slot[pick % kQRing];
                    s_tile = pick;
                    s_t0 = __ldcg(&sl->t0); s_Ms = __ldcg(&sl->M_s); s_base = __ldcg(&sl->base);
                    s_K = __ldcg(&sl->K); s_L = __ldcg(&sl->L);
                    s_cu = __ldcg(&sl->cu); s_Mx = __ldcg(&sl->M_x);
                    s_Mc = Mc;
                    s_wA = c0;
                    s_Sprev = sprev;
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
            uint32_t *dead = a.qdead + (size_t)si * kQWords, *kill = a.qkill + (size_t)si * kQWords;
            if (l == -4) {
                // ---- stage B of tile i (the resolver's next tile)
                unsigned long long rchk = 0;
                const unsigned long long tp0 = a.timing ? p_now() : 0;
                const unsigned long long wn = q_stage_b(a, sm, i, s_wA, M_s, s_Mc, s_Sprev,
                                                        a.qprep + (size_t)si * p_prep_bytes(kPChunk), rchk);
                for (int o = 16; o > 0; o >>= 1) rchk += __shfl_down_sync(0xffffffffu, rchk, o);
                if (lane == 0 && rchk) atomicAdd(&q->prep_rchk, rchk);
                if (threadIdx.x == 0) {
                    q_fence();
                    // (a CAS: the slot is never rewritten under a stage B, but do not rely on timing)
                    atomicCAS(&sl->prep, (s_wA & ~(3ull << 50)) | ((unsigned long long)kPrepBusy << 50), wn);
                    if (a.timing) { atomicAdd(&q->xcross_ns, p_now() - tp0); atomicAdd(&q->n_xb, 1ull); }
                }
                continue;
            }
            if (l == -3) {
                // ---- prepare tile i for the resolver
                unsigned long long rchk = 0;
                uint32_t S1 = 0;
                uint8_t *pbuf = a.qprep + (size_t)si * p_prep_bytes(kPChunk);
                const unsigned long long tp0 = a.timing ? p_now() : 0;
                const uint32_t S2 = p_prep(a, sm, t0, K, L, dead, max(M_s, s_cu ? s_Mx : 0ull), s_Mc, pbuf,
                                           a.qspill + (size_t)si * kPMaxTile, rchk, S1);
                if (a.cross && threadIdx.x == 0)          // the list, for the next tile's stage B
                    q_st_relaxed(&sl->listw, ((i + 1) << 16) | (S2 == 0xffffffffu ? 0xffffu : S2));
                if (a.timing && threadIdx.x == 0) atomicAdd(&q->prep_ns, p_now() - tp0);
                for (int o = 16; o > 0; o >>= 1) rchk += __shfl_down_sync(0xffffffffu, rchk, o);
                if (lane == 0 && rchk) atomicAdd(&q->prep_rchk, rchk);
                __syncthreads();
                if (threadIdx.x == 0) {
                    q_fence();
                    q_st_relaxed(&sl->prep, q_pw(i, kPrepDone, s_Mc - M_s, S2 == 0xffffffffu ? kPrepTooMany : S2, S1));
                    ++n_prep;
                }
                continue;
            }
            const unsigned long long tag = (i + 1) & 0xffffffffull;
            long long hi, lo;
            q_level_window(a, M_s, base, L, s_cu, s_Mx, l, hi, lo);
            const unsigned long long M_ref = max(M_s, (unsigned long long)hi);   // (catch-up level: hi = M_x)
            if (a.nsup_smem && M_ref > supM) {
                // super-block summaries the commits since the last refresh changed (a summary that
                // also covers words beyond the window is still valid: it only widens)
                const long long s0 = (long long)(supM >> 10);
                const long long s1 = min((long long)a.nsup_smem, (long long)((M_ref + 1023) >> 10));
                for (long long x = s0 + threadIdx.x; x < s1; x += blockDim.x) s_sup[x] = __ldcg(a.ssum + x);
                supM = M_ref;
            }
            uint32_t plo, n0;
            q_part(a, K, plo, n0);                            // this rank's candidates of the tile
            uint32_t n_l = n0;
            if (l > 0) n_l = p_live_prefix(dead, plo, plo + n0, s_live, s_pre, s_ws);    // ends with a barrier
            else __syncthreads();
            const PPlan pl = p_plan(a, n_l, hi - lo, a.plan_warps);
            PLevel lv;
            lv.l = l; lv.n_l = n_l; lv.B = pl.B; lv.nsub = pl.nsub;
            lv.hi = hi; lv.lo = lo; lv.sub = pl.sub; lv.t0 = t0; lv.head = pl.head; lv.J0 = pl.J0;
            lv.s_pre = s_pre; lv.s_live = s_live; lv.words = (plo + n0 + 31) / 32 - plo / 32; lv.basis = s_basis;
            lv.stage = reinterpret_cast<uint32_t *>(p_dyn); lv.s_sup = s_sup; lv.c_lo = plo; lv.w_base = plo;
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
                q_fence();                              // this item's kills before its arrival
                __syncwarp();
                uint32_t dn = 0;
                if (lane == 0) dn = atomicAdd(&sl->done[l], 1u);
                dn = __shfl_sync(0xffffffffu, dn, 0);
                if (dn + 1 == (uint32_t)items) q_finish_level(a, sl, i, l, L, K, M_s, base, dead, kill);
            }
            __syncthreads();                                  // shared memory is reused by the next pick
            if (threadIdx.x == 0) atomicSub(&sl->inside, 1u); // after this CTA's last claim on the slot
        }
        if (threadIdx.x == 0 && n_prep) atomicAdd(&q->preps, n_prep);
    }
    for (int o = 16; o > 0; o >>= 1) {
        my_checks += __shfl_down_sync(0xffffffffu, my_checks, o);
        my_tests += __shfl_down_sync(0xffffffffu, my_tests, o);
    }
    if (lane == 0 && my_checks) atomicAdd(&st->checks_exec, my_checks);
    if (lane == 0 && my_tests) atomicAdd(&st->bound_tests, my_tests);
}

// One rank per launch (single GPU, or one process of the multi-GPU engine).
template <int kMinBlocks>
__global__ void __launch_bounds__(kPThreads, kMinBlocks) k_pipeline(PArgs a) { q_body(a, (int)blockIdx.x); }

// Emulated ranks on one GPU (gc_options.emulate_ranks): gridDim.x / ngroups CTAs per rank, each
// group with its own arguments (its replica of the codebook and of the pipeline state).
template <int kMinBlocks>
__global__ void __launch_bounds__(kPThreads, kMinBlocks) k_pipeline_ranks(const PArgs *__restrict__ ga, int ngroups) {
    __shared__ PArgs s_a;
    const int per = (int)gridDim.x / ngroups, g = (int)blockIdx.x / per;
    const uint32_t *src = reinterpret_cast<const uint32_t *>(ga + g);
    uint32_t *dst = reinterpret_cast<uint32_t *>(&s_a);
    for (int k = threadIdx.x; k < (int)(sizeof(PArgs) / 4); k += blockDim.x) dst[k] = __ldg(src + k);
    __syncthreads();
    q_body(s_a, (int)blockIdx.x - g * per);
}

// ------------------------------------------------------------------ host side

// One rank's device state: this process's rank, or an emulated one (gc_options.emulate_ranks).
struct QRank {
    uint2 *surv = nullptr, *qspill = nullptr;
    uint32_t *bsum = nullptr;
    size_t bsum_words = 0;
    PState *st = nullptr;
    QCtl *q = nullptr;
    uint32_t *qdead = nullptr, *qkill = nullptr, *qvals = nullptr;
    uint8_t *qprep = nullptr;
    unsigned long long *qflags = nullptr;         // [kQRing][kMaxRanks]
    uint32_t *codebook = nullptr;                 // emulated ranks > 0: their replica of the codebook
    size_t cb_words = 0;
    unsigned long long *count = nullptr;
};

struct QContext {
    int device = -1, sms = 0;
    OrderTables *tabs = nullptr;
    int tabs_n = -1;
    QRank rk[kMaxRanks];
    PArgs *d_args = nullptr;                      // emulated ranks: their arguments
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

static int q_rank_alloc(QRank &k) {
    if (k.st) return GC_OK;
    QCK(cudaMalloc(&k.surv, kPMaxTile * sizeof(uint2)));
    QCK(cudaMalloc(&k.st, sizeof(PState)));
    QCK(cudaMalloc(&k.q, sizeof(QCtl)));
    QCK(cudaMalloc(&k.qdead, (size_t)kQRing * kQWords * 4));
    QCK(cudaMalloc(&k.qkill, (size_t)kQRing * kQWords * 4));
    QCK(cudaMalloc(&k.qvals, (size_t)kQRing * kPMaxTile * 4));
    QCK(cudaMalloc(&k.qprep, (size_t)kQRing * p_prep_bytes(kQChunk)));
    QCK(cudaMalloc(&k.qspill, (size_t)kQRing * kPMaxTile * sizeof(uint2)));
    QCK(cudaMalloc(&k.qflags, (size_t)kQRing * kMaxRanks * sizeof(unsigned long long)));
    QCK(cudaMalloc(&k.count, sizeof(unsigned long long)));
    return GC_OK;
}

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
        QCK(cudaMalloc(&c->tabs, sizeof(OrderTables)));
        QCK(cudaMalloc(&c->d_args, kMaxRanks * sizeof(PArgs)));
        QCK(cudaEventCreate(&c->ev0));
        QCK(cudaEventCreate(&c->ev1));
        int rc = q_rank_alloc(c->rk[0]);
        if (rc) return rc;
        g_qctx[device] = c;
    }
    *out = c;
    return GC_OK;
}

// ---- multi-GPU: the exchange buffers of rank 0 of this device's context, shared by CUDA IPC
int pipeline_peer_handles(uint8_t *out) {
    QContext *cx;
    int rc = q_context(&cx);
    if (rc) return rc;
    cudaIpcMemHandle_t h[2];
    QCK(cudaIpcGetMemHandle(&h[0], cx->rk[0].qdead));
    QCK(cudaIpcGetMemHandle(&h[1], cx->rk[0].qflags));
    static_assert(2 * sizeof(cudaIpcMemHandle_t) == kPeerHandleBytes, "handle blob size");
    memcpy(out, h, sizeof h);
    return GC_OK;
}

int pipeline_open_peers(PeerTable *t, const uint8_t *all, int world, int rank) {
    if (world < 2 || world > kMaxRanks || rank < 0 || rank >= world) {
        set_error("peers: world must be in [2, 8] and 0 <= rank < world");
        return GC_EINVAL;
    }
    pipeline_close_peers(t);
    for (int g = 0; g < world; ++g) {
        if (g == rank) continue;
        cudaIpcMemHandle_t h[2];
        memcpy(h, all + (size_t)g * kPeerHandleBytes, sizeof h);
        void *pd = nullptr, *pf = nullptr;
        QCK(cudaIpcOpenMemHandle(&pd, h[0], cudaIpcMemLazyEnablePeerAccess));
        QCK(cudaIpcOpenMemHandle(&pf, h[1], cudaIpcMemLazyEnablePeerAccess));
        t->qdead[g] = static_cast<uint32_t *>(pd);
        t->qflags[g] = static_cast<unsigned long long *>(pf);
    }
    t->world = world;
    t->rank = rank;
    t->ready = true;
    return GC_OK;
}

void pipeline_close_peers(PeerTable *t) {
    for (int g = 0; g < kMaxRanks; ++g) {
        if (t->qdead[g]) cudaIpcCloseMemHandle(t->qdead[g]);
        if (t->qflags[g]) cudaIpcCloseMemHandle(t->qflags[g]);
        t->qdead[g] = nullptr;
        t->qflags[g] = nullptr;
    }
    t->ready = false;
}

bool pipeline_supported(const RunArgs &a) {
    const bool ranks_ok = a.world == 1 ? (a.opt.emulate_ranks >= 1 && a.opt.emulate_ranks <= (uint32_t)kMaxRanks)
                                       : (a.world <= kMaxRanks && a.opt.emulate_ranks == 1 && a.peers && a.peers->ready &&
                                          a.peers->world == a.world && a.peers->rank == a.rank);
    return ranks_ok && a.opt.tile_max <= kPMaxTile &&
           !(a.opt.flags & (GC_FLAG_NO_EARLY_EXIT | GC_FLAG_FORCE_SEQ_RESOLVE | GC_FLAG_LAUNCHED_TILES |
                            GC_FLAG_TILE_BARRIERS));
}

// per-call state of one rank: counters, pipeline, summaries (AND = all ones, OR = 0 before any
// append, as in gc_persistent.cu)
static int q_rank_reset(QRank &k, const RunArgs &r, cudaStream_t s, size_t nblk, size_t nsup) {
    QCK(cudaMemsetAsync(k.st, 0, sizeof(PState), s));
    QCK(cudaMemsetAsync(k.q, 0, sizeof(QCtl), s));
    QCK(cudaMemsetAsync(k.qdead, 0, (size_t)kQRing * kQWords * 4, s));
    QCK(cudaMemsetAsync(k.qkill, 0, (size_t)kQRing * kQWords * 4, s));
    QCK(cudaMemsetAsync(k.qflags, 0, (size_t)kQRing * kMaxRanks * sizeof(unsigned long long), s));
    const size_t need = 2 * (nblk + nsup);
    if (k.bsum_words < need) {
        if (k.bsum) QCK(cudaFree(k.bsum));
        k.bsum = nullptr;
        k.bsum_words = 0;
        QCK(cudaMalloc(&k.bsum, need * 4));
        k.bsum_words = need;
    }
    QCK(cudaMemsetAsync(k.bsum, 0, need * 4, s));
    QCK(cudaMemset2DAsync(k.bsum, 8, 0xff, 4, nblk + nsup, s));
    return GC_OK;
}

int pipeline_run(const RunArgs &r) {
    QContext *cx;
    int rc = q_context(&cx);
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(cx->mu);       // setup, launch and read-back (gc.h)
    cudaStream_t s = (cudaStream_t)r.stream;
    // the context's buffers are reused by every call on this device: order this call after the
    // previous one's kernel even when the callers use different streams
    QCK(cudaStreamWaitEvent(s, cx->ev1, 0));
    if (cx->tabs_n != (int)r.n) {
        OrderTables t;
        build_order_tables((int)r.n, &t);
        QCK(cudaMemcpy(cx->tabs, &t, sizeof t, cudaMemcpyHostToDevice));
        cx->tabs_n = (int)r.n;
    }
    const int world = r.world > 1 ? r.world : (int)r.opt.emulate_ranks;   // ranks sharing each tile's screen
    const int local = r.world > 1 ? 1 : world;                             // of which run in this launch
    const size_t nsup = (size_t)((r.capacity + 1023) / 1024) + 1, nblk = nsup * 32;
    for (int g = 0; g < local; ++g) {
        QRank &k = cx->rk[g];
        if ((rc = q_rank_alloc(k))) return rc;
        if (g > 0 && k.cb_words < r.capacity) {     // an emulated rank's replica of the codebook
            if (k.codebook) QCK(cudaFree(k.codebook));
            k.codebook = nullptr;
            k.cb_words = 0;
            QCK(cudaMalloc(&k.codebook, (size_t)r.capacity * 4));
            k.cb_words = (size_t)r.capacity;
        }
        if ((rc = q_rank_reset(k, r, s, nblk, nsup))) return rc;
    }
    PArgs a;
    p_fill_args(r, &a);
    a.tabs = cx->tabs;
    a.vals = nullptr;
    a.dead = nullptr;
    const bool graded = (r.ordering == GRADED_LEX || r.ordering == GRADED_REVLEX) && !r.use_basis;
    // graded orders: their screens are the binding stage -- sub-ranges of 32768 words per warp item
    // (more items, shorter ones) and two more tiles in flight (tools/r02am.sh, r02an.sh:
    // 28,3,glex 2386 -> 1394 ms, 26,4,glex 342 -> 290 ms)
    // (not for constant weight, whose graded scan is one weight class: 24,6,glex,cw=12 26 -> 29 ms)
    const bool graded_screen = graded && r.constant_weight < 0;
    a.depth = (int)std::min<uint32_t>(r.opt.pipeline_depth ? r.opt.pipeline_depth : graded_screen ? 10u : 8u, (uint32_t)kQRing);
    if (graded_screen && !r.opt.sub_max) a.sub_max_bound = 32768u;
    // Gray order: ~448 accepted words per tile (the tile-barrier engine's 768 leaves the pipelined
    // resolver and preparation too much per tile: 28,3,gray 602 -> 571 ms, 26,4,gray 150 -> 142.5;
    // tools/r02bc.sh, profiles/r02bc_knob_target.log)
    if (r.ordering == GRAY && !r.use_basis && !r.opt.target_accepted) a.target_accepted = 448u;
    // ranks may run up to 2 x depth tiles apart; a slot is rewritten by a peer only after its
    // previous tile is committed everywhere when 2 x depth < the ring
    if (world > 1) a.depth = std::min(a.depth, kQRing / 2 - 1);
    a.chunk = kQChunk;
    // preparation lead: 1 tile for lex / Gray / B-orders (the resolver then checks only the last
    // tile's words), 2 for graded orders, whose screens are the binding stage and whose preparers
    // need the slack (tools/r02g.sh sweep, profiles/r02g_knob_sweep.log)
    a.prep_lead = (r.opt.flags & GC_FLAG_NO_PREP) ? 0 : (int)(r.opt.prep_lead ? r.opt.prep_lead : graded ? 2u : 1u);
    a.size_on_screen = (r.opt.flags & GC_FLAG_SIZE_ON_TRUE) ? 0 : 1;
    // cross lists (two-stage preparation): opt-in -- neutral to slightly slower on the measured
    // workloads (tools/r02ae.sh, profiles/r02_cross_catchup.md)
    a.cross = (a.prep_lead > 0 && (r.opt.flags & GC_FLAG_CROSS)) ? 1 : 0;
    {   // the most levels a tile can have: the window levels reaching a full codebook, plus the
        // catch-up level (q_reset rewrites only these slots' level counters)
        int L = 0;
        unsigned long long dsum = 0;
        while (L < kPMaxLevels && dsum < r.capacity) {
            const int sh = a.growth * L;
            dsum += sh >= 40 ? (1ull << 40) : std::min((unsigned long long)a.W0 << sh, 1ull << 40);
            ++L;
        }
        a.reset_levels = std::min(L + 1, kPMaxLevels);
    }
    // two-stage preparation: stage A as soon as a tile is screened (prep_lead tiles ahead, default 3),
    // stage B one tile ahead of the resolver flags the survivors hit by the words committed since
    a.stage_b = (a.prep_lead > 0 && (a.cross || (r.opt.flags & GC_FLAG_STAGE_B))) ? 1 : 0;
    if (a.stage_b && !r.opt.prep_lead) a.prep_lead = 3;
    a.world = world;
    a.rank = r.world > 1 ? r.rank : 0;
    for (int g = 0; g < kMaxRanks; ++g) { a.peer_qdead[g] = nullptr; a.peer_flag[g] = nullptr; }
    for (int g = 0; g < world; ++g) {
        const bool own = r.world > 1 ? g == r.rank : true;
        const QRank &k = cx->rk[r.world > 1 ? 0 : g];
        a.peer_qdead[g] = own ? k.qdead : r.peers->qdead[g];
        a.peer_flag[g] = own ? k.qflags : r.peers->qflags[g];
    }
    const void *kfn = local > 1 ? (const void *)k_pipeline_ranks<1> : (const void *)k_pipeline<1>;
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
    int per = cx->sms / local;                       // CTAs per rank in this launch
    if (r.opt.grid_ctas) per = std::max(2, std::min(per, (int)r.opt.grid_ctas));   // >= 1 screening CTA
    if (per < 2) { set_error("too many emulated ranks for this GPU"); return GC_EINVAL; }
    // dedicated preparing CTAs, leaving at least one screening CTA
    a.prep_ctas = a.prep_lead ? std::min((int)(r.opt.prep_ctas ? r.opt.prep_ctas : 2u), per - 2) : 0;
    if (a.prep_ctas < 0) a.prep_ctas = 0;
    const uint32_t screen_warps = (uint32_t)(per - 1 - a.prep_ctas) * kPWarps;
    a.plan_warps = r.opt.plan_warps ? r.opt.plan_warps : std::max<uint32_t>(kPWarps, screen_warps / (uint32_t)a.depth);
    PArgs ga[kMaxRanks];
    for (int g = 0; g < local; ++g) {
        const QRank &k = cx->rk[g];
        PArgs &b = ga[g];
        b = a;
        if (local > 1) b.rank = g;
        b.bsum = reinterpret_cast<uint2 *>(k.bsum);
        b.ssum = reinterpret_cast<uint2 *>(k.bsum) + nblk;
        b.surv = k.surv;
        b.st = k.st;
        b.q = k.q;
        b.qdead = k.qdead; b.qkill = k.qkill; b.qvals = k.qvals;
        b.qprep = k.qprep;
        // catch-up screening level, by default for graded orders (their screens are the binding stage;
        // 26,4,glex 359 -> 334 ms) and d = 4 (26,4,gray 160 -> 153 ms); not for d = 3 lex / Gray, whose
        // killers sit in the last one or two tiles, which no screen sees in time (28,3,lex +6 %), nor
        // for large d with tiny codebooks (24,8,lex +20 %)  (tools/r02aj.sh, profiles/r02_cross_catchup.md)
        const bool cu_default = graded_screen || r.d == 4;
        const bool cu = (r.opt.flags & GC_FLAG_CATCHUP) || (cu_default && !(r.opt.flags & GC_FLAG_NO_CATCHUP));
        b.cm = cu && !(r.opt.flags & GC_FLAG_NO_CATCHUP) ? &k.q->cm : nullptr;
        b.qspill = k.qspill;
        if (g > 0) { b.codebook = k.codebook; b.d_count = k.count; }
    }
    QCK(cudaEventRecord(cx->ev0, s));
    if (local > 1) {
        QCK(cudaMemcpyAsync(cx->d_args, ga, local * sizeof(PArgs), cudaMemcpyHostToDevice, s));
        const PArgs *dp = cx->d_args;
        int ng = local;
        void *args[] = {&dp, &ng};
        QCK(cudaLaunchCooperativeKernel(kfn, dim3(per * local), dim3(kPThreads), args, smem, s));
    } else {
        void *args[] = {&ga[0]};
        QCK(cudaLaunchCooperativeKernel(kfn, dim3(per), dim3(kPThreads), args, smem, s));
    }
    QCK(cudaEventRecord(cx->ev1, s));
    if (r.stats) {
        QCK(cudaStreamSynchronize(s));
        PState h;
        QCK(cudaMemcpy(&h, cx->rk[0].st, sizeof(PState), cudaMemcpyDeviceToHost));
        QCtl hq;
        QCK(cudaMemcpy(&hq, cx->rk[0].q, offsetof(QCtl, slot), cudaMemcpyDeviceToHost));
        float ms = 0;
        QCK(cudaEventElapsedTime(&ms, cx->ev0, cx->ev1));
        gc_stats *o = r.stats;
        o->struct_size = sizeof(gc_stats);
        o->n_ranks = (uint32_t)world;
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
        o->prep_used = hq.prep_used;
        for (int g = 1; g < local; ++g) {            // emulated ranks: their screen work counts too
            PState hg;
            QCK(cudaMemcpy(&hg, cx->rk[g].st, sizeof(PState), cudaMemcpyDeviceToHost));
            o->checks_exec += hg.checks_exec;
            o->bound_tests += hg.bound_tests;
            if (hg.M != h.M) { set_error("emulated ranks disagree on the code size"); return GC_EINTERNAL; }
        }
        if (a.timing) {
            PState f;
            QCK(cudaMemcpy(&f, cx->rk[0].st, sizeof(PState), cudaMemcpyDeviceToHost));
            const double T = (double)f.tiles, c = 1965.0;
            fprintf(stderr, "[gc] pipeline: %llu tiles, %d rank(s), depth %d, prep lead %d (%d CTAs), %.2f us/tile; "
                    "resolver per tile: wait %.2f busy %.2f us; %llu tiles prepared, %llu resolved from a prep (busy "
                    "%.2f us each; the others %.2f us each)\n", f.tiles, world, a.depth, a.prep_lead, a.prep_ctas,
                    ms * 1e3 / T, hq.resolve_wait_ns / T / 1e3, hq.resolve_busy_ns / T / 1e3, hq.preps, hq.prep_used,
                    hq.busy_prep_ns / 1e3 / (double)std::max(1ull, hq.prep_used),
                    (hq.resolve_busy_ns - hq.busy_prep_ns) / 1e3 / (double)std::max(1ull, f.tiles - hq.prep_used));
            fprintf(stderr, "[gc]   resolve: gather %.2f conflicts %.2f prior+status %.2f rounds %.2f sequential %.2f "
                    "append %.2f clear+stats %.2f publish %.2f us (SM cycles at 1965 MHz)\n", f.t_r[0] / T / c,
                    f.t_r[1] / T / c, f.t_r[5] / T / c, f.t_r[6] / T / c, f.t_r[2] / T / c, f.t_r[3] / T / c,
                    f.t_r[4] / T / c, f.t_sync / T / c);
            const double P = (double)std::max(1ull, hq.prep_used);
            fprintf(stderr, "[gc]   prepared tiles: CAS+reset %.2f (ns clock) load %.2f consensus+prior %.2f status %.2f "
                    "rounds %.2f sequential %.2f append %.2f stats %.2f publish %.2f us\n", f.t_level[9] / P / 1e3,
                    f.t_level[0] / P / c, f.t_level[1] / P / c, f.t_level[5] / P / c, f.t_level[6] / P / c,
                    f.t_level[2] / P / c, f.t_level[3] / P / c, f.t_level[4] / P / c, f.t_level[8] / P / c);
            fprintf(stderr, "[gc]   preparations: %llu stage A, %.2f us each; %llu stage B, %.2f us each; %llu tiles "
                    "resolved in cross mode\n", hq.preps, hq.prep_ns / 1e3 / (double)std::max(1ull, hq.preps), hq.n_xb,
                    hq.xcross_ns / 1e3 / (double)std::max(1ull, hq.n_xb), hq.n_xmode);
            fprintf(stderr, "[gc]   arrivals: %llu unscreened, %llu screened+open, %llu prep busy, %llu prep done; "
                    "screen latency %.2f us, screened -> arrival %.2f us\n", hq.arr[0], hq.arr[1], hq.arr[2], hq.arr[3],
                    hq.scr_ns / 1e3 / (double)std::max(1ull, hq.n_scr), hq.lag_ns / 1e3 / (double)std::max(1ull, hq.n_scr));
            fprintf(stderr, "[gc]   tail: %llu chunks entered it (%.1f undecided threads each), %.2f us per tile in the tail "
                    "itself\n", f.t_level[12], f.t_level[13] / (double)std::max(1ull, f.t_level[12]), f.t_r[7] / T / c);
            fprintf(stderr, "[gc]   per tile: survivors %.1f, accepted %.1f, resolve checks %.0f, levels %.2f; "
                    "largest S %llu, %llu multi-chunk tiles, %.2f rounds, %.2f sequential\n", f.survivors / T, f.M / T,
                    f.resolve_checks / T, f.levels / T, f.s_max, f.n_chunked, f.n_rounds / T, f.n_seq / T);
        }
        if (h.error == 2) { set_error("pipelined engine stalled: a screen, preparation or peer never arrived"); return GC_EINTERNAL; }
        if (h.error) { set_error("codebook capacity exceeded"); return GC_ENOSPC; }
    }
    return GC_OK;
}

}  // namespace gc
