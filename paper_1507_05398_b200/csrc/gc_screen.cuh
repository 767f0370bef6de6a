// gc_screen.cuh -- device pieces shared by the persistent engines (gc_persistent.cu:
// k_construct / k_resolve_tile, and gc_pipeline.cu: k_pipeline): the schedule arithmetic,
// the tile screen (SURVEY.md Sec. 8(a) a1, a2, a2'), the in-tile ordered resolve and the
// commit (a3, a4).  Everything here is __device__ __forceinline__ (or a constant / struct).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "gc_internal.h"
#include "gc_order.cuh"

namespace gc {

constexpr int kPThreads = 512;              // threads per CTA (16 warps); grid = #SMs
constexpr int kMaxRanks = 8;                // ranks of the multi-GPU pipelined engine (one node)
constexpr int kQRingMax = 16;               // tile slots of the pipelined engine
constexpr int kPWarps = kPThreads / 32;
constexpr uint32_t kPR2Min = 1;             // levels with >= this many candidates use 2 per lane
constexpr uint32_t kPSubMin = 64;           // codewords per warp item: at least ...
constexpr uint32_t kPSubMax = 2048;         // ... and at most
constexpr int kPMaxLevels = 32;
constexpr uint32_t kPMaxTile = 1u << 16;    // largest tile (tile indices fit in 16 bits)
// survivors resolved per chunk (shared memory): 4096 with one CTA per SM, 2048 with two
constexpr uint32_t kPMaxBatches = kPMaxTile / 32;
constexpr uint32_t kPTargetAccepted = 384;  // adaptive tiles grow up to ~2x this many accepted words
                                            // (Gray: twice that, graded orders: four times;
                                            // tools/sweep_knobs2.sh, profiles/r01j_knob_sweep.md)
constexpr uint32_t kPMaxPredictedSurvivors = 1024;
constexpr int kPAdj = 32;                       // earlier in-tile conflicts recorded per survivor
constexpr int kPX = 8;                          // cross conflicts (with earlier tiles' prepared survivors)
                                                // recorded per prepared survivor (pipelined engine)
constexpr int kPXRing = 8;                      // the resolver keeps the accepted bits of this many tiles
constexpr uint32_t kPStageWords = 32 * 32;      // per-warp stage: 32 blocks of 32 codewords (4 KiB)
constexpr uint32_t kPWarpStage = kPStageWords + 8 * 64 + 32;   // + 8 super-blocks' block summaries + a block queue
constexpr uint32_t kPWinWords = 16384 + 32;     // level-0 window copied to shared memory (words, then
                                                // kPWinWords / 32 + 1 block summaries)
constexpr int kPSplitBits = 12;                 // a warp's live candidates differing in more bits are
                                                // screened as two halves (block bound, p_item)
constexpr uint32_t kPOvf = 1024;                // overflow survivors decided warp-parallel (per chunk)
constexpr uint32_t kPChunkMaxGroups = 4096 / 32;  // groups of 32 survivors in the largest resolve chunk
constexpr uint32_t kPResolveTmp = 2048;         // k_resolve_tile: staging words after the scratch
constexpr uint32_t kPOvfMark = 0xffffffffu;     // s_cnt of a listed overflow survivor
constexpr uint32_t kPTmpMaxWords = 4096;        // prior words staged per round of the resolve (PSmem::tmp_words)
// resolve scratch: s_val (4 B) + s_idx (2 B) + s_status (1 B) + pad (1 B) + s_cnt (4 B) + s_adj (2 B x kPAdj)
__host__ __device__ constexpr size_t p_resolve_smem(uint32_t chunk) { return (size_t)chunk * (12 + 2 * kPAdj); }
// + level prefix: s_pre[kPMaxTile/32 + 1] and s_live[kPMaxTile/32]
// the level stages (kPWarpStage words per warp) alias the resolve scratch: a CTA never runs both
constexpr size_t kPLevelSmem = (size_t)kPWarps * kPWarpStage * 4 + kPWinWords * 4 + (kPWinWords / 32 + 1) * 8;
__host__ __device__ constexpr size_t p_scratch_smem(uint32_t chunk) {
    return p_resolve_smem(chunk) > kPLevelSmem ? p_resolve_smem(chunk) : kPLevelSmem;
}
__host__ __device__ constexpr size_t p_dyn_smem(uint32_t chunk) {
    return p_scratch_smem(chunk) + (size_t)(2 * (kPMaxTile / 32) + 4) * 4;
}

struct PState {
    unsigned long long M;
    unsigned long long checks_exec;
    unsigned long long bound_tests;            // block / super-block summary tests (lane evaluations)
    unsigned long long survivors;
    unsigned long long conflicts;
    unsigned long long resolve_checks;
    unsigned long long w_def;
    unsigned long long tiles;
    unsigned long long levels;
    unsigned long long t_level[kPMaxLevels];   // diagnostics: CTA 0's view, ns (%globaltimer)
    unsigned long long c_level[kPMaxLevels];   // diagnostics: lane-checks per level
    unsigned long long t_resolve, t_sync, t_tile;
    unsigned long long t_r[8];                 // resolve sub-steps
    unsigned long long t_items[kPMaxLevels];   // diagnostics: level start -> last item done (any warp)
    unsigned long long t_item_end[2];          // per-level scratch (alternating slots)
    unsigned long long t_item_max[2];          // per-level scratch: longest warp item
    unsigned long long item_scan_max[2];       // per-level scratch: most codewords one warp item scanned
    unsigned long long scan_max_sum[kPMaxLevels];
    unsigned long long t_item_sum[kPMaxLevels];
    unsigned long long t_prefix[kPMaxLevels], n_live[kPMaxLevels], n_items[kPMaxLevels], t_itmax[kPMaxLevels];
    unsigned long long n_overflow, n_seq, n_rounds;
    unsigned long long n_chunked, s_max, n_rounds_max;   // diagnostics: multi-chunk tiles, largest S
    unsigned int error;
    unsigned int K_next;                       // size of the next tile (set by CTA 0)
    unsigned long long token;                  // commit token: (tile + 1) << 40 | partial << 39 | log2(K_next) << 34 | M
    unsigned int K_used;                       // a partial tile's length (token bit 39)
    unsigned int S_last, K_last;               // last tile with survivors: its S and K
    unsigned int wfirst[33];                   // graded orders: 1 + index of the first codeword of weight w
};

struct PArgs {
    int n, ord;
    uint32_t d;
    unsigned long long N;           // 2^n
    uint32_t tile_min, tile_max, W0;
    int growth;
    int mix;                        // 2..4: half the checks via p_clear_low<d> (d <= 4), 0: POPC only
    uint32_t chunk;                 // survivors per resolve chunk
    int weight_bound;               // graded orders: stop the screen at the weight bound
    int items_per_warp;             // target work items per warp and level
    uint32_t target_accepted;       // adaptive tiles grow toward ~this many accepted words per tile
    uint32_t sub_max_bound;         // longest window sub-range per warp item with the block bound
    uint32_t partial_s;             // persistent engine: a tile with more survivors is cut after this many
    uint32_t geo_head;              // first (newest) window sub-range of a level; 0 = uniform sub-ranges
    int split_bits;                 // a warp whose live candidates vary in more bits screens two halves
    uint32_t nsup_smem;             // super-block summaries [0, nsup_smem) mirrored in every CTA's shared
                                    // memory (persistent mode; refreshed as commits change them)
    // partition mode (multi-GPU / emulated ranks): one tile's screen over one candidate range
    int part_mode;
    unsigned long long t_single;
    uint32_t K_single, part_lo, part_len;
    // SURVEY 8(f) extensions
    int use_basis;                  // B-ordering: rank -> XOR of basis[j] over set bits j
    uint32_t basis[32];
    int so;                         // self-orthogonal: also popc(v & c) even, wt(v) even
    int cw;                         // constant weight (-1: none)
    unsigned long long t_begin, t_end;   // ranks scanned (graded + constant weight: one class)
    int wdef_valid;                 // W_def counts every rank: only without filters
    // block bound: per aligned block of 32 codewords (and of 1024) the AND and the OR of its
    // words; a warp skips a block when popc((AND_blk & ~OR_c) | (AND_c & ~OR_blk)) >= d for
    // the AND/OR of its live candidates (GC_FLAG_NO_BLOCK_BOUND turns it off)
    int bound;
    uint32_t nmask;                 // 2^n - 1
    uint2 *bsum;                    // (AND, OR) per block of 32, [nblk] (multiple of 32)
    uint2 *ssum;                    // (AND, OR) per super-block of 1024
    uint32_t *codebook;
    unsigned long long capacity;
    const OrderTables *tabs;
    uint32_t *vals;                 // [kPMaxTile]
    uint32_t *dead;                 // [kPMaxTile / 32]
    uint2 *surv;                    // [kPMaxTile]
    PState *st;
    unsigned long long *d_count;
    int timing;
    // pipelined engine (k_pipeline, gc_pipeline.cu)
    struct QCtl *q;
    uint32_t *qdead, *qkill, *qvals;   // per ring slot: kPMaxTile/32, kPMaxTile/32 and kPMaxTile words
    int depth;                         // tiles in flight: tile i is screened against codebook[0, M after i - depth)
    uint32_t plan_warps;               // warps the level plans are sized for
    uint8_t *qprep;                    // per ring slot: p_prep_bytes(chunk) (a prepared tile)
    uint2 *qspill;                     // per ring slot: kPMaxTile (the preparer's survivors beyond one chunk)
    int prep_lead;                     // tile i is prepared once tile i - prep_lead is being resolved (0: never)
    int prep_ctas;                     // CTAs 1 .. prep_ctas only prepare tiles (never screen)
    uint32_t burst_chunk;              // survivors decided per sub-chunk of a tile with more than one chunk
    int par;                           // block-bound summaries carry the weight parity in bit 31 (n <= 30)
    const unsigned long long *cm;      // the resolver's commit word (committed tiles << 40 | M), or null:
                                       // pipelined engine, one rank: every tile's screen ends with a
                                       // catch-up level over the words committed since its descriptor
    int reset_levels;                  // pipelined engine: level counters reset per slot (levels + catch-up)
    int stage_b;                       // two-stage preparation (GC_FLAG_STAGE_B, or with cross lists)
    int cross;                         // preparations record cross conflicts with the prepared survivors of
                                       // the tiles still being resolved (GC_FLAG_NO_CROSS: 0)
    int size_on_screen;                // tile sizes bound the survivors of the (older-codebook) screen, which
                                       // the resolve handles, not only those left after the catch-up checks
    // multi-rank pipelined engine: the screen of every tile is split over `world` ranks (whole mask
    // words, gc_tile_partition); every rank resolves the whole tile, so the codebooks stay identical
    int world, rank;
    uint32_t *peer_qdead[kMaxRanks];          // each rank's qdead ring: this rank stores its partition's words into all
    unsigned long long *peer_flag[kMaxRanks]; // each rank's flags [kQRingMax][kMaxRanks]: tile + 1 once rank r's words are in
};

// Next tile size (a power of two in [tile_min, tile_max]) after a tile of K candidates
// with S survivors and A accepted, the construction now at rank t1 with M1 words.
//   cap: the density seen so far (M1 / t1) predicts ~kPTargetAccepted accepted words per
//        tile of size cap (sparse codes get long tiles, so little per-tile latency); also
//        cap <= t1/8 while the history is short;
//   K halves when false survivors (S - A) exceed A/4 -- each scans the whole codebook --
//   and grows back toward cap while S <= 9/8 A.
// Deterministic: a function of (K, S, A, t1, M1) only, never of timing.
__device__ __forceinline__ uint32_t p_next_tile(const PArgs &a, uint32_t K, uint32_t S, uint32_t A,
                                                unsigned long long t1, unsigned long long M1,
                                                uint32_t S_last, uint32_t K_last) {
    const unsigned long long want = M1 ? (unsigned long long)a.target_accepted * t1 / M1 : ~0ull;
    uint32_t cap = a.tile_min;
    // survivors predicted from the last tile that had any (bursty orders, e.g. graded ones at
    // large d, have long empty stretches): keep them <= kPMaxPredictedSurvivors
    while (cap < a.tile_max && (unsigned long long)cap * 2 <= want && (unsigned long long)cap * 16 <= t1 &&
           (unsigned long long)S_last * cap * 2 <= (unsigned long long)kPMaxPredictedSurvivors * K_last)
        cap <<= 1;
    uint32_t Kn = K;
    if (A > 0 && (unsigned long long)S * 4 > (unsigned long long)A * 5) Kn = K > a.tile_min ? K / 2 : K;
    else if (A == 0 || (unsigned long long)S * 8 <= (unsigned long long)A * 9) Kn = K * 2;
    if (Kn > cap) Kn = cap;
    if (Kn < a.tile_min) Kn = a.tile_min;
    return Kn;
}

// newest-first depth covered by levels 0 .. l-1: W0 (1 + g + ... + g^(l-1)), g = 2^growth
// (window sizes saturate at 2^40, far above any codebook)
__device__ __forceinline__ unsigned long long p_window(uint32_t W0, int growth, int l) {
    const int sh = growth * l;
    return sh >= 40 ? (1ull << 40) : min((unsigned long long)W0 << sh, 1ull << 40);
}
__device__ __forceinline__ unsigned long long p_depth(uint32_t W0, int growth, int l) {
    unsigned long long dsum = 0;
    for (int i = 0; i < l; ++i) dsum += p_window(W0, growth, i);
    return dsum;
}

// number of levels needed to reach codeword 0 from the newest
__device__ __forceinline__ int p_levels(unsigned long long M, uint32_t W0, int growth) {
    if (M == 0) return 0;
    int L = 1;
    while (L < kPMaxLevels && p_depth(W0, growth, L) < M) ++L;
    return L;
}

// x with its lowest D-1 set bits cleared: zero iff popc(x) < D (D - 1 applications of
// x & (x - 1)).  Runs on the integer ALU/FMA pipes instead of the POPC unit.
template <int D>
__device__ __forceinline__ uint32_t p_clear_low(uint32_t x) {
#pragma unroll
    for (int i = 0; i < D - 1; ++i) x &= x - 1u;
    return x;
}

// One candidate-codeword check, accumulated into m.  MIX = 0: m = min popc(v ^ c) (the
// candidate dies when m < d).  MIX = D (2..4) for odd r: m = min p_clear_low<D>(v ^ c),
// dies when m == 0 -- the same predicate popc(v ^ c) < d, evaluated without POPC so that
// the two halves of a warp's checks use different pipes.
template <int MIX>
__device__ __forceinline__ void p_check(uint32_t &m, uint32_t v, uint32_t c, int r) {
    if (MIX == 1) {
        // self-orthogonal: odd AND-parity counts as a violation (distance 0)
        m = min(m, (__popc(v & c) & 1) ? 0u : (uint32_t)__popc(v ^ c));
    } else if (MIX && (r & 1)) {
        m = min(m, p_clear_low<MIX>(v ^ c));
    } else {
        m = min(m, (uint32_t)__popc(v ^ c));
    }
}

template <int MIX>
__device__ __forceinline__ bool p_dead(uint32_t m, uint32_t d, int r) {
    return (MIX >= 2 && (r & 1)) ? (m == 0) : (m < d);
}

// scan codewords [a, b) newest first for the lane's R candidates; returns the number of
// codewords scanned (for the work counter).  The warp reads 32 codewords per coalesced
// 128-byte load (lane k holds codeword top-1-k), prefetches the next block while it works
// on this one, and broadcasts each codeword with a shuffle.  Early exit (warp vote) after
// every block once every lane's candidates are dead.
template <int R, int MIX>
__device__ __forceinline__ uint32_t p_scan(const uint32_t *__restrict__ cb, long long a, long long b,
                                           uint32_t cur, const uint32_t (&v)[R], uint32_t (&m)[R],
                                           uint32_t d) {
    const int lane = threadIdx.x & 31;
    long long top = b;
    uint32_t scanned = 0;
    while (top > a) {
        const long long ntop = top - 32;
        const uint32_t nxt = (ntop > a && ntop - 1 - lane >= a) ? __ldcg(cb + ntop - 1 - lane) : 0u;
        const long long nv = top - a;
        if (nv >= 32) {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const uint32_t c = __shfl_sync(0xffffffffu, cur, k);
#pragma unroll
                for (int r = 0; r < R; ++r) p_check<MIX>(m[r], v[r], c, r);
            }
            scanned += 32;
        } else {
            for (int k = 0; k < (int)nv; ++k) {
                const uint32_t c = __shfl_sync(0xffffffffu, cur, k);
#pragma unroll
                for (int r = 0; r < R; ++r) p_check<MIX>(m[r], v[r], c, r);
            }
            scanned += (uint32_t)nv;
        }
        bool done = true;
#pragma unroll
        for (int r = 0; r < R; ++r) done &= p_dead<MIX>(m[r], d, r);
        if (__all_sync(0xffffffffu, done)) break;
        cur = nxt;
        top = ntop;
    }
    return scanned;
}

// Block bound (exact): at a bit position where every codeword of a block has the value x and
// every live candidate of the warp has 1 - x, every candidate-codeword pair differs, so
//   dist(v, c) >= popc((AND_blk & ~OR_cand) | (AND_cand & ~OR_blk))   for all v, c.
// A block whose bound is >= d cannot hold a codeword closer than d to any of the candidates.
__device__ __forceinline__ uint32_t p_lb(uint32_t bA, uint32_t bO, uint32_t cA, uint32_t cO, uint32_t nmask) {
    return (uint32_t)__popc(((bA & ~cO) | (cA & ~bO)) & nmask);
}

// The same bound on the screen's parity-tagged summaries (a.par, n <= 30: bit 31 of every word
// that enters an AND / OR is the parity of its weight).  dist(v, c) = wt(v) + wt(c) mod 2, so when
// every codeword of the block and every candidate of the warp have one weight parity each (AND
// and OR agree in bit 31 on both sides), every distance has the parity of their sum and the
// bound rounds up to it (graded orders: a block inside one weight class, d = 4: a bound of 3
// between equal parities proves >= 4).
__device__ __forceinline__ uint32_t p_lbs(const PArgs &a, uint32_t bA, uint32_t bO, uint32_t cA, uint32_t cO) {
    uint32_t lb = (uint32_t)__popc(((bA & ~cO) | (cA & ~bO)) & a.nmask);
    if (a.par) {
        const uint32_t uniform = ~((bA ^ bO) | (cA ^ cO)) >> 31;
        lb += uniform & ((lb ^ ((bO ^ cO) >> 31)) & 1u);
    }
    return lb;
}

// a word with its weight parity in bit 31 (parity-tagged summaries, a.par)
__device__ __forceinline__ uint32_t p_ptag(const PArgs &a, uint32_t v) {
    return a.par ? (v | ((uint32_t)__popc(v) << 31)) : v;
}

// checks of the lane's R candidates against the (nv <= 32) codewords held by lanes 0..nv-1
template <int R, int MIX>
__device__ __forceinline__ void p_block(uint32_t cur, int nv, const uint32_t (&v)[R], uint32_t (&m)[R]) {
    if (nv == 32) {
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            const uint32_t c = __shfl_sync(0xffffffffu, cur, k);
#pragma unroll
            for (int r = 0; r < R; ++r) p_check<MIX>(m[r], v[r], c, r);
        }
    } else {
        for (int k = 0; k < nv; ++k) {
            const uint32_t c = __shfl_sync(0xffffffffu, cur, k);
#pragma unroll
            for (int r = 0; r < R; ++r) p_check<MIX>(m[r], v[r], c, r);
        }
    }
}

template <int R, int MIX>
__device__ __forceinline__ bool p_all_dead(const uint32_t (&m)[R], uint32_t d) {
    bool done = true;
#pragma unroll
    for (int r = 0; r < R; ++r) done &= p_dead<MIX>(m[r], d, r);
    return __all_sync(0xffffffffu, done);
}

// checks against the codewords stage[o_lo, o_hi) of one staged block (shared memory, the same
// address in every lane: broadcast reads, four codewords per 128-bit load for a full block)
template <int R, int MIX>
__device__ __forceinline__ void p_block_smem(const uint32_t *stage, int o_lo, int o_hi, const uint32_t (&v)[R],
                                             uint32_t (&m)[R]) {
    if (o_lo == 0 && o_hi == 32) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(stage);
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
            const uint4 c = s4[k4];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                p_check<MIX>(m[r], v[r], c.x, r);
                p_check<MIX>(m[r], v[r], c.y, r);
                p_check<MIX>(m[r], v[r], c.z, r);
                p_check<MIX>(m[r], v[r], c.w, r);
            }
        }
    } else {
        for (int k = o_lo; k < o_hi; ++k) {
            const uint32_t c = stage[k];
#pragma unroll
            for (int r = 0; r < R; ++r) p_check<MIX>(m[r], v[r], c, r);
        }
    }
}

__device__ __forceinline__ void p_cp_async16(uint32_t *dst, const uint32_t *src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void p_cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
}

// Aligned blocks kb..kt (newest first) of the codeword range [r_lo, r_hi): lane t tests block
// kt - t (32 blocks per round).  The codewords of block kt are fetched into registers together
// with the bounds (speculatively); every other passing block is copied at once into the warp's
// shared-memory stage (cp.async, 16 B per lane, L2 only) while block kt is checked, so a round
// costs two dependent round trips however many blocks pass.  Returns true once every candidate
// of the warp is dead.
template <int R, int MIX>
__device__ __forceinline__ bool p_scan_blocks(const PArgs &a, long long r_lo, long long r_hi, uint32_t cA, uint32_t cO,
                                              const uint32_t (&v)[R], uint32_t (&m)[R], uint32_t &scanned,
                                              uint32_t *stage, uint32_t &tests) {
    const int lane = threadIdx.x & 31;
    const long long kb = r_lo >> 5;
    for (long long kt = (r_hi - 1) >> 5; kt >= kb; kt -= 32) {
        const long long k = kt - lane;
        auto blk_top = [&](long long q) { return min(r_hi, (q + 1) << 5); };
        auto blk_bot = [&](long long q) { return max(r_lo, q << 5); };
        const long long i0 = blk_top(kt) - 1 - lane;
        const uint32_t cur = i0 >= blk_bot(kt) ? __ldcg(a.codebook + i0) : 0u;
        bool pass = false;
        if (k >= kb) {
            const uint2 bs = __ldcg(a.bsum + k);
            pass = p_lbs(a, bs.x, bs.y, cA, cO) < a.d;
            ++tests;
        }
        const uint32_t mask = __ballot_sync(0xffffffffu, pass);
        if (!mask) continue;
        const uint32_t rest = mask & ~1u;             // block kt (bit 0) is checked from registers
        const int nst = __popc(rest);
        // stage: slot s <- the s-th passing block after kt, 8 lanes x 16 B per block; a 16-byte
        // chunk reaching past the codebook's capacity is read word by word instead
        for (int p = lane; p < 8 * nst; p += 32) {
            const int sl = p >> 3, c4 = (p & 7) * 4;
            const long long q = kt - (long long)(__fns(rest, 0, sl + 1));
            const unsigned long long w0 = (unsigned long long)(q << 5) + c4;
            if (w0 + 4 <= a.capacity) {
                p_cp_async16(stage + sl * 32 + c4, a.codebook + w0);
            } else {
                for (int e = 0; e < 4; ++e)
                    if (w0 + e < a.capacity) stage[sl * 32 + c4 + e] = __ldcg(a.codebook + w0 + e);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        if (mask & 1u) {
            const int nv = (int)(blk_top(kt) - blk_bot(kt));
            p_block<R, MIX>(cur, nv, v, m);
            scanned += (uint32_t)nv;
            if (p_all_dead<R, MIX>(m, a.d)) { p_cp_async_wait_all(); return true; }
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        uint32_t mm = rest;
        for (int sl = 0; sl < nst; ++sl) {
            const int t = __ffs(mm) - 1;
            mm &= mm - 1;
            const long long q = kt - t;
            const int o_lo = (int)(blk_bot(q) - (q << 5)), o_hi = (int)(blk_top(q) - (q << 5));
            p_block_smem<R, MIX>(stage + sl * 32, o_lo, o_hi, v, m);
            scanned += (uint32_t)(o_hi - o_lo);
            if (p_all_dead<R, MIX>(m, a.d)) { __syncwarp(); return true; }
        }
        __syncwarp();      // the stage is rewritten by the next round
    }
    return false;
}

// Check the warp's candidates against the listed blocks blist[0, nb) of [lo, hi): all of
// them are copied into the stage at once (cp.async, 8 lanes x 16 B per block, L2 only), then
// scanned in list order.  Returns true once every candidate of the warp is dead.
template <int R, int MIX>
__device__ __forceinline__ bool p_scan_list(const PArgs &a, long long lo, long long hi, const uint32_t *blist, int nb,
                                            const uint32_t (&v)[R], uint32_t (&m)[R], uint32_t &scanned,
                                            uint32_t *stage) {
    const int lane = threadIdx.x & 31;
    for (int p = lane; p < 8 * nb; p += 32) {
        const int sl = p >> 3, c4 = (p & 7) * 4;
        const unsigned long long w0 = ((unsigned long long)blist[sl] << 5) + c4;
        if (w0 + 4 <= a.capacity) {
            p_cp_async16(stage + sl * 32 + c4, a.codebook + w0);
        } else {
            for (int e = 0; e < 4; ++e)
                if (w0 + e < a.capacity) stage[sl * 32 + c4 + e] = __ldcg(a.codebook + w0 + e);
        }
    }
    p_cp_async_wait_all();
    for (int sl = 0; sl < nb; ++sl) {
        const long long q = blist[sl];
        const int o_lo = (int)(max(lo, q << 5) - (q << 5)), o_hi = (int)(min(hi, (q + 1) << 5) - (q << 5));
        p_block_smem<R, MIX>(stage + sl * 32, o_lo, o_hi, v, m);
        scanned += (uint32_t)(o_hi - o_lo);
        if (p_all_dead<R, MIX>(m, a.d)) { __syncwarp(); return true; }
    }
    __syncwarp();      // the stage and the list are rewritten next
    return false;
}

// scan [lo, hi) newest first with the block bound, the window and its block summaries held in
// shared memory (level 0): lane t tests block kt - t, the warp checks the passing blocks
// straight from shared memory -- no global round trip at all
template <int R, int MIX>
__device__ __forceinline__ uint32_t p_scan_window(const PArgs &a, const uint32_t *win, const uint2 *wsum,
                                                  long long win_lo, long long lo, long long hi, uint32_t cA,
                                                  uint32_t cO, const uint32_t (&v)[R], uint32_t (&m)[R],
                                                  uint32_t &tests) {
    const int lane = threadIdx.x & 31;
    uint32_t scanned = 0;
    const long long kb = lo >> 5, k0 = win_lo >> 5;
    for (long long kt = (hi - 1) >> 5; kt >= kb; kt -= 32) {
        const long long k = kt - lane;
        bool pass = false;
        if (k >= kb) {
            const uint2 bs = wsum[k - k0];
            pass = p_lbs(a, bs.x, bs.y, cA, cO) < a.d;
            ++tests;
        }
        uint32_t mask = __ballot_sync(0xffffffffu, pass);
        while (mask) {
            const long long q = kt - (__ffs(mask) - 1);
            mask &= mask - 1;
            const int o_lo = (int)(max(lo, q << 5) - (q << 5)), o_hi = (int)(min(hi, (q + 1) << 5) - (q << 5));
            p_block_smem<R, MIX>(win + ((q << 5) - win_lo), o_lo, o_hi, v, m);
            scanned += (uint32_t)(o_hi - o_lo);
            if (p_all_dead<R, MIX>(m, a.d)) return scanned;
        }
    }
    return scanned;
}

// scan [lo, hi) newest first with the block bound.  Ranges up to 4096 codewords test their
// blocks directly (p_scan_blocks).  Longer ones go down a hierarchy, newest first, with a
// fixed number of dependent round trips per round whatever passes:
//   1. lane j tests super-block sg - j (1024 codewords) from its (AND, OR) summary;
//   2. the block summaries of up to 8 passing super-blocks are copied to shared memory at once
//      (256 B each) and tested there, one block per lane;
//   3. the passing blocks are queued; every 32 of them are staged and checked (p_scan_list).
template <int R, int MIX>
__device__ __forceinline__ uint32_t p_scan_bound(const PArgs &a, long long lo, long long hi, uint32_t cA, uint32_t cO,
                                                 const uint32_t (&v)[R], uint32_t (&m)[R], uint32_t *stage,
                                                 const uint2 *s_sup, uint32_t &tests) {
    const int lane = threadIdx.x & 31;
    uint32_t scanned = 0;
    if (hi - lo <= 4096) {
        p_scan_blocks<R, MIX>(a, lo, hi, cA, cO, v, m, scanned, stage, tests);
        return scanned;
    }
    uint32_t *sstage = stage + kPStageWords;                 // 8 super-blocks x 32 (AND, OR)
    uint32_t *blist = sstage + 8 * 64;                       // 32 queued block indices
    const long long sb_lo = lo >> 10, kb = lo >> 5, kt = (hi - 1) >> 5;
    int nb = 0;
    for (long long sg = (hi - 1) >> 10; sg >= sb_lo; sg -= 32) {
        const long long sb = sg - lane;
        bool pass = false;
        if (sb >= sb_lo) {
            const uint2 ss = sb < (long long)a.nsup_smem ? s_sup[sb] : __ldcg(a.ssum + sb);
            pass = p_lbs(a, ss.x, ss.y, cA, cO) < a.d;
            ++tests;
        }
        uint32_t smask = __ballot_sync(0xffffffffu, pass);
        while (smask) {
            const int ns = min(8, __popc(smask));
            for (int p = lane; p < 16 * ns; p += 32) {
                const int sl = p >> 4, c = p & 15;
                const long long s = sg - (long long)__fns(smask, 0, sl + 1);
                p_cp_async16(sstage + sl * 64 + c * 4, reinterpret_cast<const uint32_t *>(a.bsum + (s << 5)) + c * 4);
            }
            p_cp_async_wait_all();
            for (int sl = 0; sl < ns; ++sl) {
                const long long s = sg - (long long)(__ffs(smask) - 1);
                smask &= smask - 1;
                const long long k = (s << 5) + 31 - lane;            // newest block first
                bool bp = false;
                if (k >= kb && k <= kt) {
                    const uint32_t *e = sstage + sl * 64 + 2 * (31 - lane);
                    bp = p_lbs(a, e[0], e[1], cA, cO) < a.d;
                    ++tests;
                }
                const uint32_t bm = __ballot_sync(0xffffffffu, bp);
                if (!bm) continue;
                if (nb + __popc(bm) > 32) {
                    if (p_scan_list<R, MIX>(a, lo, hi, blist, nb, v, m, scanned, stage)) return scanned;
                    nb = 0;
                }
                if (bp) blist[nb + __popc(bm & ((1u << lane) - 1u))] = (uint32_t)k;
                nb += __popc(bm);
                __syncwarp();
            }
        }
    }
    if (nb) p_scan_list<R, MIX>(a, lo, hi, blist, nb, v, m, scanned, stage);
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

// u and v cannot both be in the code: distance < d, or (self-orthogonal) odd AND-parity
__device__ __forceinline__ bool p_conflict(const PArgs &a, uint32_t u, uint32_t v) {
    return (uint32_t)__popc(u ^ v) < a.d || (a.so && (__popc(u & v) & 1));
}

// candidate of rank r: the ordering's vector, or the B-ordering's XOR of basis vectors
__device__ __forceinline__ uint32_t p_gen(const PArgs &a, const uint32_t (*C)[33], const uint64_t *off,
                                          const uint32_t *basis, unsigned long long r) {
    if (a.use_basis) {
        uint32_t v = 0;
        for (uint32_t bits = (uint32_t)r; bits; bits &= bits - 1) v ^= basis[__ffs(bits) - 1];
        return v;
    }
    return rank_to_vector32(a.ord, a.n, C, off, r);
}

// candidate considered at all: constant weight, even weight if self-orthogonal
__device__ __forceinline__ bool p_allowed(const PArgs &a, uint32_t v) {
    const int w = __popc(v);
    return (a.cw < 0 || w == a.cw) && (!a.so || !(w & 1));
}

struct PLevel {
    int l;
    uint32_t n_l, B, nsub;
    long long hi, lo, sub;
    long long head;          // block bound: the first J0 sub-ranges (newest) are head, 2 head, 4 head,
    int J0;                  // ... < sub -- the newest words pass the bound most, so they are split finer
    unsigned long long t0;
    const uint32_t *s_pre;   // level >= 1: exclusive prefix of live candidates per mask word (smem)
    const uint32_t *s_live;  // level >= 1: live bits per mask word (smem)
    uint32_t words;
    const uint32_t *basis;   // B-ordering basis (smem)
    uint32_t *stage;         // block-bound staging, kPStageWords per warp (smem; aliases the resolve scratch)
    const uint2 *s_sup;      // shared-memory mirror of the first a.nsup_smem super-block summaries
    const uint32_t *win;     // level 0 with the block bound: the whole window, copied to shared memory
    const uint2 *wsum;       //   once per CTA (words [win_lo, hi), win_lo = lo & ~31) and its block summaries
    long long win_lo;
    uint32_t *kill;          // the level's kill mask (k_construct: the tile's dead mask)
    uint32_t *vals;          // candidate values stored by level 0 (graded orders)
    uint32_t c_lo;           // first tile index of the screened range
    uint32_t w_base;         // 32 * (first mask word of the range)
};

// tile index of the q-th live candidate of level >= 1 (q < n_l): the mask word w with
// s_pre[w] <= q < s_pre[w+1], then the (q - s_pre[w])-th set bit of s_live[w]
__device__ __forceinline__ uint32_t p_locate(const PLevel &lv, uint32_t q) {
    uint32_t lo = 0, hi = lv.words;          // s_pre[lo] <= q < s_pre[hi] (s_pre[words] = n_l)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (lv.s_pre[mid] <= q) lo = mid; else hi = mid;
    }
    uint32_t bits = lv.s_live[lo];
    for (uint32_t k = q - lv.s_pre[lo]; k > 0; --k) bits &= bits - 1;
    return lv.w_base + lo * 32 + (__ffs(bits) - 1);
}

// One warp item: batch b (32 R candidates) of the level's live candidates against sub-range
// j of the level's window.  Level 0 generates the candidates from their ranks; deeper levels
// find them through the CTA's prefix of the dead mask (no lists, no pushes).
template <int R, int MIX>
__device__ __forceinline__ void p_item(const PArgs &a, const PLevel &lv, unsigned long long it,
                                       const uint32_t (*C)[33], const uint64_t *off,
                                       unsigned long long &my_checks, unsigned long long &my_tests) {
    const int lane = threadIdx.x & 31;
    const uint32_t j = (uint32_t)(it / lv.B), b = (uint32_t)(it % lv.B);
    long long v0, vlen;                                               // j = 0: newest
    if ((int)j < lv.J0) { v0 = lv.head * ((1ll << j) - 1); vlen = lv.head << j; }
    else { v0 = lv.head * ((1ll << lv.J0) - 1) + (long long)(j - lv.J0) * lv.sub; vlen = lv.sub; }
    const long long s_hi = lv.hi - v0;
    const long long s_lo = max(lv.lo, s_hi - vlen);
    // first codeword block in flight while the candidates are fetched
    const uint32_t cur0 = (!a.bound || MIX == 1) && (s_hi - 1 - lane >= s_lo) ? __ldcg(a.codebook + s_hi - 1 - lane) : 0u;
    uint32_t v[R], m[R], idx[R];
    bool live[R], filtered[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t q = b * (32u * R) + r * 32 + lane;
        live[r] = q < lv.n_l;
        filtered[r] = false;
        idx[r] = 0; v[r] = 0;
        if (live[r]) {
            if (lv.l == 0) {
                idx[r] = lv.c_lo + q;
                v[r] = p_gen(a, C, off, lv.basis, lv.t0 + idx[r]);
                if (j == 0) lv.vals[idx[r]] = v[r];
                if (!p_allowed(a, v[r])) { filtered[r] = true; live[r] = false; }
            } else {
                idx[r] = p_locate(lv, q);
                // lex / Gray / B-ordering: regenerate from the rank (a few ALU ops, no round
                // trip); graded orders: load the value level 0 stored (unranking is O(n))
                v[r] = a.ord < GRADED_LEX || a.use_basis ? p_gen(a, C, off, lv.basis, lv.t0 + idx[r])
                                                         : __ldcg(lv.vals + idx[r]);
            }
            // another sub-range of this level may already have killed it (load issued in
            // parallel with the value / codeword loads)
            // (level 0 only: deeper levels hold mostly true survivors, and the load would sit
            // on their critical path)
            // (not with the block bound: level-0 items all run at once, the bit is rarely set
            // yet, and the load would delay the bound tests by a round trip)
            if (lv.l == 0 && lv.nsub > 1 && live[r] && (!a.bound || MIX == 1))
                live[r] = !((__ldcg(lv.kill + (idx[r] >> 5)) >> (idx[r] & 31)) & 1u);
        }
        m[r] = live[r] ? 0xffffffffu : 0u;      // dead lanes start "already dead" in both forms
    }
    bool any = false;
#pragma unroll
    for (int r = 0; r < R; ++r) any |= live[r];
    bool any_filtered = false;
#pragma unroll
    for (int r = 0; r < R; ++r) any_filtered |= filtered[r];
    const bool scan = __any_sync(0xffffffffu, any);
    if (scan || __any_sync(0xffffffffu, any_filtered)) {
        if (scan) {
            uint32_t sc;
            if (MIX != 1 && a.bound) {
                // AND / OR of the warp's live candidates (identity for the others)
                uint32_t la = ~0u, lo_ = 0u;
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (live[r]) { const uint32_t vt = p_ptag(a, v[r]); la &= vt; lo_ |= vt; }
                const uint32_t cA = __reduce_and_sync(0xffffffffu, la), cO = __reduce_or_sync(0xffffffffu, lo_);
                uint32_t *stg = lv.stage + (threadIdx.x >> 5) * kPWarpStage;
                uint32_t tests = 0;
                auto scan = [&](uint32_t sA, uint32_t sO, uint32_t (&mm)[R]) {
                    return lv.win ? p_scan_window<R, MIX>(a, lv.win, lv.wsum, lv.win_lo, s_lo, s_hi, sA, sO, v, mm, tests)
                                  : p_scan_bound<R, MIX>(a, s_lo, s_hi, sA, sO, v, mm, stg, lv.s_sup, tests);
                };
                const uint32_t vary = cO & ~cA & a.nmask;  // bits on which the live candidates differ
                // (not for graded orders: a weight class in colex order varies many bits by
                // nature, and the weight bound already cuts their windows)
                if (__popc(vary) <= a.split_bits || (a.ord >= GRADED_LEX && !a.use_basis)) {
                    sc = scan(cA, cO, m);
                } else {
                    // weak consensus (typically a batch straddling a carry of a high bit): scan
                    // the two halves split on the highest varying bit separately, each with its
                    // own, much stronger, consensus; the other half's lanes ride along as dead
                    const uint32_t hb = 1u << (31 - __clz(vary));
                    sc = 0;
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        uint32_t ha = ~0u, ho = 0u, mm[R];
                        bool any_h = false;
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const bool in = live[r] && (((v[r] & hb) != 0) == (half == 1));
                            mm[r] = in ? m[r] : 0u;
                            if (in) { const uint32_t vt = p_ptag(a, v[r]); ha &= vt; ho |= vt; any_h = true; }
                        }
                        if (!__any_sync(0xffffffffu, any_h)) continue;
                        const uint32_t hA = __reduce_and_sync(0xffffffffu, ha), hO = __reduce_or_sync(0xffffffffu, ho);
                        sc += scan(hA, hO, mm);
#pragma unroll
                        for (int r = 0; r < R; ++r)
                            if (live[r] && (((v[r] & hb) != 0) == (half == 1))) m[r] = mm[r];
                    }
                }
                my_tests += tests;                         // per lane: block-summary tests evaluated
            } else {
                sc = p_scan<R, MIX>(a.codebook, s_lo, s_hi, cur0, v, m, a.d);
            }
            my_checks += (unsigned long long)sc * R;   // per lane; summed over lanes at the end
            if (a.timing && (threadIdx.x & 31) == 0) atomicMax(&a.st->item_scan_max[lv.l & 1], (unsigned long long)sc);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool kill = filtered[r] || (live[r] && p_dead<MIX>(m[r], a.d, r));
            if (lv.l == 0) {
                // the warp's 32 candidates of this r are one aligned mask word
                const unsigned bb = __ballot_sync(0xffffffffu, kill);
                if (lane == 0 && bb) atomicOr(&lv.kill[idx[r] >> 5], bb);
            } else if (kill) {
                atomicOr(&lv.kill[idx[r] >> 5], 1u << (idx[r] & 31));
            }
        }
    }
}

// Item decomposition of one level: batches of 32 R live candidates x newest-first sub-ranges
// of the window [lo, hi), sized so that the level has ~items_per_warp items per warp of
// `nwarps` (the first J0 sub-ranges geometric: head, 2 head, 4 head, ... < sub).
// Deterministic: every CTA (and the level's publisher) derives the same plan.
struct PPlan {
    int R;
    uint32_t B, nsub;
    long long sub, head;
    int J0;
    __device__ __forceinline__ unsigned long long items() const { return (unsigned long long)B * nsub; }
};
__device__ __forceinline__ PPlan p_plan(const PArgs &a, uint32_t n_l, long long wlen, uint32_t nwarps) {
    PPlan p;
    p.R = (n_l >= kPR2Min) ? 2 : 1;
    const uint32_t batch = 32u * p.R;
    p.B = (n_l + batch - 1) / batch;
    p.sub = 0; p.head = 0; p.J0 = 0; p.nsub = 0;
    if (wlen > 0 && p.B > 0) {
        const long long want = ((long long)nwarps * a.items_per_warp + p.B - 1) / p.B;   // sub-ranges wanted
        long long sub = (wlen + want - 1) / want;
        sub = (sub + 31) & ~31ll;
        sub = max(sub, (long long)kPSubMin);
        sub = min(sub, a.bound ? (long long)a.sub_max_bound : (long long)kPSubMax);
        long long head = sub;
        int J0 = 0;
        if (a.bound && a.geo_head > 0 && sub > (long long)a.geo_head) {
            head = a.geo_head;
            while ((head << (J0 + 1)) <= sub && head * ((1ll << (J0 + 1)) - 1) < wlen) ++J0;
        }
        const long long headlen = head * ((1ll << J0) - 1);
        p.nsub = (uint32_t)J0 + (wlen > headlen ? (uint32_t)((wlen - headlen + sub - 1) / sub) : 0u);
        p.sub = sub; p.head = head; p.J0 = J0;
    }
    return p;
}

// window [lo, hi) of level l (newest-first positions) of a screen against codebook[base, M):
// level 0 the newest W0 words, each next one 2^growth times longer, the last reaches base
__device__ __forceinline__ void p_level_window(const PArgs &a, unsigned long long M, unsigned long long base, int L,
                                               int l, long long &hi, long long &lo) {
    const long long bp = (long long)p_depth(a.W0, a.growth, l);
    hi = (long long)M - bp;
    lo = (l == L - 1) ? (long long)base : hi - (long long)p_window(a.W0, a.growth, l);
    if (lo < (long long)base) lo = (long long)base;
}

// CTA-wide: live candidates of [c_lo, c_hi) (not set in `dead`) as per-word bits s_live and an
// exclusive prefix s_pre over the mask words from c_lo / 32 (s_pre[pwords] = total); returns
// the total.  Ends with a CTA barrier.
__device__ __forceinline__ uint32_t p_live_prefix(const uint32_t *dead, uint32_t c_lo, uint32_t c_hi, uint32_t *s_live,
                                                  uint32_t *s_pre, uint32_t *s_ws) {
    const uint32_t w_lo = c_lo / 32;
    const uint32_t pwords = (c_hi + 31) / 32 - w_lo;
    uint32_t tot_all = 0;
    for (uint32_t w0 = 0; w0 < pwords; w0 += blockDim.x) {
        const uint32_t wr = w0 + threadIdx.x;          // relative word
        uint32_t live = 0;
        if (wr < pwords) {
            const uint32_t w = w_lo + wr;
            live = ~__ldcg(dead + w);
            if (w * 32 + 32 > c_hi) live &= (1u << (c_hi - w * 32)) - 1u;
            if (w * 32 < c_lo) live &= ~((1u << (c_lo - w * 32)) - 1u);
            s_live[wr] = live;
        }
        uint32_t tot;
        const uint32_t pre = tot_all + p_block_scan(__popc(live), &tot, s_ws);
        if (wr < pwords) s_pre[wr] = pre;
        tot_all += tot;
    }
    if (threadIdx.x == 0) s_pre[pwords] = tot_all;
    __syncthreads();
    return tot_all;
}

// CTA-wide: copy the window [lo, hi) of the codebook and its block summaries to shared memory
// (win: kPWinWords words, then wsum); sets lv.win / wsum / win_lo.  Ends with a CTA barrier.
__device__ __forceinline__ void p_copy_window(const PArgs &a, PLevel &lv, uint32_t *win, long long hi, long long lo) {
    uint2 *wsum = reinterpret_cast<uint2 *>(win + kPWinWords);
    const long long wl = lo & ~31ll, nwd = hi - wl;
    for (long long c = threadIdx.x; c < (nwd + 3) / 4; c += blockDim.x) {
        const unsigned long long w0 = (unsigned long long)(wl + 4 * c);
        if (w0 + 4 <= a.capacity) {
            p_cp_async16(win + 4 * c, a.codebook + w0);
        } else {
            for (int e = 0; e < 4; ++e)
                if (w0 + e < a.capacity) win[4 * c + e] = __ldcg(a.codebook + w0 + e);
        }
    }
    const long long nbk = ((hi - 1) >> 5) - (wl >> 5) + 1;
    for (long long k = threadIdx.x; k < nbk; k += blockDim.x) wsum[k] = __ldcg(a.bsum + (wl >> 5) + k);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    lv.win = win; lv.wsum = wsum; lv.win_lo = wl;
}

// level 0 with the block bound copies its window to shared memory when it is this short
__device__ __forceinline__ bool p_window_in_smem(const PArgs &a, int l, long long hi, long long lo) {
    return l == 0 && a.bound && !a.so && hi > lo && hi - (lo & ~31ll) <= (long long)kPWinWords;
}

// one warp item of a level planned with R candidates per lane (dispatch on the check form)
__device__ __forceinline__ void p_run_item(const PArgs &a, const PLevel &lv, int R, unsigned long long it,
                                           const uint32_t (*C)[33], const uint64_t *off,
                                           unsigned long long &my_checks, unsigned long long &my_tests) {
    if (a.so) {
        if (R == 2) p_item<2, 1>(a, lv, it, C, off, my_checks, my_tests);
        else p_item<1, 1>(a, lv, it, C, off, my_checks, my_tests);
    } else if (R == 2) {
        switch (a.mix) {
            case 2: p_item<2, 2>(a, lv, it, C, off, my_checks, my_tests); break;
            case 3: p_item<2, 3>(a, lv, it, C, off, my_checks, my_tests); break;
            case 4: p_item<2, 4>(a, lv, it, C, off, my_checks, my_tests); break;
            default: p_item<2, 0>(a, lv, it, C, off, my_checks, my_tests); break;
        }
    } else {
        p_item<1, 0>(a, lv, it, C, off, my_checks, my_tests);
    }
}

__device__ __forceinline__ unsigned long long p_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// a3 + a4 for one tile, by ONE CTA: survivors in rank order (from the dead mask), in-tile
// ordered resolve, ordered append, M += A, next tile size, per-tile state cleared.
// first codeword the tile must be screened against (weight bound, graded orders), else 0
__device__ __forceinline__ unsigned long long p_base(const PArgs &a, unsigned long long t0, unsigned long long M) {
    if (!a.weight_bound) return 0;
    int w_lo = 0;
    while (t0 >= a.tabs->off[w_lo + 1]) ++w_lo;
    for (int w = max(0, w_lo - (int)a.d + 1); w <= a.n; ++w) {
        const unsigned int f = __ldcg(&a.st->wfirst[w]);
        if (f) return f - 1;
    }
    return M;
}

// Commit-side state and counters, kept by the CTA that resolves (thread 0) in its shared memory
// so the tile's critical path has no global read-modify-write; loaded from / flushed to PState
// once per kernel.  M and K_next are also published to PState every tile (fire-and-forget
// stores the grid barrier makes visible).
struct PCount {
    unsigned long long M, survivors, tiles, levels, resolve_checks, conflicts, w_def;
    unsigned int S_last, K_last, K_next, K_used;
    unsigned int S_tile, A_tile;         // the last resolved tile's survivors and accepted words
    unsigned int wfirst[33];
};
__device__ __forceinline__ void p_count_load(PCount &pc, const PState *st) {
    pc.M = st->M; pc.survivors = st->survivors; pc.tiles = st->tiles; pc.levels = st->levels;
    pc.resolve_checks = st->resolve_checks; pc.conflicts = st->conflicts; pc.w_def = st->w_def;
    pc.S_last = st->S_last; pc.K_last = st->K_last;
    for (int w = 0; w < 33; ++w) pc.wfirst[w] = st->wfirst[w];
}
__device__ __forceinline__ void p_count_store(const PCount &pc, PState *st) {
    st->M = pc.M; st->survivors = pc.survivors; st->tiles = pc.tiles; st->levels = pc.levels;
    st->resolve_checks = pc.resolve_checks; st->conflicts = pc.conflicts; st->w_def = pc.w_def;
    st->S_last = pc.S_last; st->K_last = pc.K_last;
    for (int w = 0; w < 33; ++w) st->wfirst[w] = pc.wfirst[w];
}

// diagnostics (GC_DEBUG_PHASES): accumulated by thread 0 of CTA 0 in local memory, written once
struct PTimers {
    unsigned long long level[kPMaxLevels], items[kPMaxLevels];
    unsigned long long prefix[kPMaxLevels], live[kPMaxLevels], items_n[kPMaxLevels], item_max[kPMaxLevels];
    unsigned long long resolve, sync, tile, r[8];
};

struct PSmem {
    const uint32_t (*C)[33];
    const uint64_t *off;
    const uint32_t *s_basis;
    uint32_t *s_ws, *s_val;
    uint16_t *s_idx;
    uint8_t *s_status;
    uint32_t *s_cnt;
    uint16_t *s_adj;
    uint32_t chunk;
    uint32_t *s_tmp;          // staging for words accepted in earlier chunks of a tile
    uint32_t tmp_words;
};

// Small scratch of the resolve stages (one static shared-memory allocation per kernel).
struct RShared {
    uint16_t ovf[kPOvf];
    uint32_t novf;
    uint32_t tsum[4];                                        // p_resolve: the tile's counters
    uint32_t und[3];                                         // r_decide: undecided survivors per round (mod 3)
    uint32_t wmin[33];                                       // graded orders: first position of each weight
    uint32_t gA[kPChunkMaxGroups], gO[kPChunkMaxGroups];     // survivor group consensus (AND / OR of 32)
    uint32_t qA[kPTmpMaxWords / 32], qO[kPTmpMaxWords / 32]; // staged prior-word blocks
};
__device__ __forceinline__ RShared &p_rsh() {
    __shared__ RShared r;
    return r;
}

// A tile prepared off the resolver's critical path (pipelined engine, gc_pipeline.cu): its
// survivors in rank order, already checked against codebook[.., M_prep), with their in-tile
// conflict lists -- laid out as the resolve keeps them in shared memory.
struct PPrep {
    uint32_t S;                       // survivors stored
    uint32_t S_screen;                // survivors of the tile's screen (before the preparer's check)
    unsigned long long M_prep;        // they have no conflict in codebook[0, M_prep)
    const uint32_t *val, *cnt;        // [S]
    const uint16_t *idx, *adj;        // [S], [S * kPAdj]
    // cross mode: codebook[M_prep, M) holds only the accepted words of the xb tiles before this one,
    // each resolved from its own prepared list; the preparer recorded every conflict of survivor j
    // with those lists (xcnt[j] <= kPX entries xadj[j * kPX + q] = b << 12 | position in the list of
    // tile `tile - b`), and xbits[(tile - b) % kPXRing] holds the accepted positions of that tile
    int xmode;
    int xstage;                       // stage B ran: xcnt[j] == 0xff flags a conflict in codebook[.., M_prep)
    unsigned long long tile;
    const uint8_t *xcnt;              // [S]
    const uint16_t *xadj;             // [S * kPX]
    const uint32_t (*xbits)[64];      // [kPXRing][64]: accepted positions of the last tiles
};
// a prepared tile decided in sub-chunks (p_resolve): more than two sub-chunks of survivors; not after
// a stage B (its flags only live in the prepared layout)
__device__ __forceinline__ bool p_prep_big(const PArgs &a, const PPrep &p) {
    return !p.xstage && p.S > 2u * max(32u, a.burst_chunk);
}
// per-slot layout of a prepared tile: val u32[chunk], cnt u32[chunk], idx u16[chunk], adj u16[chunk * kPAdj],
// xadj u16[chunk * kPX], xcnt u8[chunk]
__host__ __device__ constexpr size_t p_prep_bytes(uint32_t chunk) { return (size_t)chunk * (11 + 2 * kPAdj + 2 * kPX); }
__host__ __device__ constexpr size_t p_prep_xadj(uint32_t chunk) { return (size_t)chunk * (10 + 2 * kPAdj); }
__host__ __device__ constexpr size_t p_prep_xcnt(uint32_t chunk) { return (size_t)chunk * (10 + 2 * kPAdj + 2 * kPX); }

// a3.1 survivors of the tile in rank order (from its dead mask), values regenerated from their
// ranks (no load): the first `chunk` straight into shared memory (s_idx, s_val), any further ones
// to `spill` (a.surv for the resolving CTA; null: only counted).  L == 0 (empty codebook, no
// level ran): the candidate filters are applied here.  Returns S (CTA-uniform).  Ends with a
// barrier.
__device__ __forceinline__ uint32_t r_gather(const PArgs &a, const PSmem &sm, unsigned long long t0, uint32_t K,
                                             int L, uint32_t *dead, uint2 *spill) {
    const uint32_t tid = threadIdx.x, words = (K + 31) / 32;
    if (L == 0) {
        for (uint32_t i = tid; i < K; i += blockDim.x)
            if (!p_allowed(a, p_gen(a, sm.C, sm.off, sm.s_basis, t0 + i))) atomicOr(&dead[i >> 5], 1u << (i & 31));
        __syncthreads();
    }
    uint32_t S = 0;
    for (uint32_t w0 = 0; w0 < words; w0 += blockDim.x) {
        const uint32_t w = w0 + tid;
        uint32_t alive = 0;
        if (w < words) {
            alive = ~__ldcg(dead + w);
            if (w * 32 + 32 > K) alive &= (1u << (K - w * 32)) - 1u;
        }
        uint32_t tot;
        uint32_t pos = S + p_block_scan(__popc(alive), &tot, sm.s_ws);
        while (alive) {
            const int bit = __ffs(alive) - 1;
            alive &= alive - 1;
            const uint32_t i = w * 32 + bit;
            const uint32_t v = p_gen(a, sm.C, sm.off, sm.s_basis, t0 + i);
            if (pos < sm.chunk) { sm.s_idx[pos] = (uint16_t)i; sm.s_val[pos] = v; }
            else if (spill) spill[pos] = make_uint2(i, v);
            ++pos;
        }
        S += tot;
    }
    __syncthreads();
    return S;
}

// consensus (AND / OR) of every aligned group of 32 survivors s_val[0, Sc) (zero_status: their
// s_status too).  Ends with a barrier.
__device__ __forceinline__ void r_consensus(const PSmem &sm, uint32_t Sc, bool zero_status = false) {
    RShared &r = p_rsh();
    const int lane = threadIdx.x & 31;
    const uint32_t ng = (Sc + 31) / 32;
    for (uint32_t g = threadIdx.x >> 5; g < ng; g += blockDim.x >> 5) {
        const uint32_t k = 32 * g + lane;
        const uint32_t x = k < Sc ? sm.s_val[k] : 0u;
        if (zero_status && k < Sc) sm.s_status[k] = 0;
        const uint32_t gA = __reduce_and_sync(0xffffffffu, k < Sc ? x : ~0u);
        const uint32_t gO = __reduce_or_sync(0xffffffffu, x);
        if (lane == 0) { r.gA[g] = gA; r.gO[g] = gO; }
    }
    __syncthreads();
}

// a3.2 in-chunk conflicts: one warp task per (group jb of 32 survivors, earlier group kg <= jb):
// lane t holds survivor 32 jb + t, the survivors of group kg are broadcast by shuffles; a bit
// mask of the conflicting earlier ones is appended to j's adjacency list (s_adj, up to kPAdj
// entries, any order; s_cnt[j] > kPAdj marks an overflow).  Two groups whose consensus bound is
// >= d hold no conflicting pair (not for the orthogonality constraint).  Needs r_consensus.
// MIX (2..4, distance-only problems): odd columns use the ALU bit-clearing form of the same
// predicate, so the XU (POPC) and ALU pipes share the work.  Ends with a barrier.
__device__ __forceinline__ void r_units(const PArgs &a, const PSmem &sm, uint32_t Sc, unsigned long long &rchk) {
    RShared &r = p_rsh();
    const int lane = threadIdx.x & 31;
    for (uint32_t j = threadIdx.x; j < Sc; j += blockDim.x) sm.s_cnt[j] = 0;
    __syncthreads();
    const uint32_t ng = (Sc + 31) / 32;
    auto units = [&](auto so_tag, auto mix_tag) {
        constexpr bool SO = decltype(so_tag)::value;
        constexpr int MIXC = decltype(mix_tag)::value;
        auto cf = [&](uint32_t u, uint32_t w, int t) {
            if (MIXC >= 2 && (t & 1)) return p_clear_low<MIXC>(u ^ w) == 0u;
            return (uint32_t)__popc(u ^ w) < a.d || (SO && (__popc(u & w) & 1));
        };
        const uint32_t ntask = ng * (ng + 1) / 2;
        for (uint32_t p = threadIdx.x >> 5; p < ntask; p += blockDim.x >> 5) {
            uint32_t jb = (uint32_t)((sqrtf(8.0f * (float)p + 1.0f) - 1.0f) * 0.5f);
            while ((jb + 1) * (jb + 2) / 2 <= p) ++jb;
            while (jb * (jb + 1) / 2 > p) --jb;
            const uint32_t kg = p - jb * (jb + 1) / 2;
            const uint32_t j = 32 * jb + lane, k = 32 * kg + lane;
            if (!SO && p_lb(r.gA[jb], r.gO[jb], r.gA[kg], r.gO[kg], a.nmask) >= a.d) continue;
            const uint32_t vj = j < Sc ? sm.s_val[j] : 0u, vk = k < Sc ? sm.s_val[k] : 0u;
            uint32_t mask = 0;
#pragma unroll
            for (int t = 0; t < 32; ++t) mask |= (uint32_t)cf(vj, __shfl_sync(0xffffffffu, vk, t), t) << t;
            const uint32_t kmax = min(j, Sc);                 // earlier survivors only
            const uint32_t lim = kmax > 32 * kg ? min(32u, kmax - 32 * kg) : 0u;
            mask &= lim >= 32 ? 0xffffffffu : ((1u << lim) - 1u);
            if (j < Sc) rchk += lim;
            if (j < Sc && mask) {
                uint32_t q = atomicAdd(&sm.s_cnt[j], (uint32_t)__popc(mask));
                while (mask) {
                    const uint32_t t = __ffs(mask) - 1;
                    mask &= mask - 1;
                    if (q < kPAdj) sm.s_adj[j * kPAdj + q] = (uint16_t)(32 * kg + t);
                    ++q;
                }
            }
        }
    };
    if (a.so) units(std::true_type{}, std::integral_constant<int, 0>{});
    else if (a.mix == 2) units(std::false_type{}, std::integral_constant<int, 2>{});
    else if (a.mix == 3) units(std::false_type{}, std::integral_constant<int, 3>{});
    else if (a.mix == 4) units(std::false_type{}, std::integral_constant<int, 4>{});
    else units(std::false_type{}, std::integral_constant<int, 0>{});
    __syncthreads();
}

// An earlier tile's prepared list (pipelined engine, cross lists): its survivors val[0, S).
struct XList {
    const uint32_t *val;
    uint32_t S;
};

// Cross conflicts of a prepared tile (pipelined engine): its survivors s_val[0, S) (consensus in
// r.gA / r.gO, r_consensus) against the prepared lists xl[k] (shared memory) of the tiles b = k + 1
// before it, k < nl, which may still be unresolved: every conflicting pair is appended to
// xadj[j * kPX + q] (global) as b << 12 | position in that list, counted in sm.s_cnt[j] (zeroed by
// the caller; counts above kPX are overflows).  The lists are staged together in s_tmp (each from
// a multiple of 32, as many as fit per batch); a warp task is (group of 32 survivors, group of 32
// listed words), skipped when the consensus bound of the two is >= d (not for the orthogonality
// constraint).  Ends with a barrier.
__device__ __forceinline__ void r_cross(const PArgs &a, const PSmem &sm, uint32_t S, const XList *xl, uint32_t nl,
                                        uint16_t *xadj, unsigned long long &rchk) {
    RShared &r = p_rsh();
    __shared__ uint32_t s_xoff[kPXRing + 1];
    const int lane = threadIdx.x & 31;
    const uint32_t tid = threadIdx.x;
    const uint32_t ng = (S + 31) / 32;
    for (uint32_t k0 = 0; k0 < nl;) {
        uint32_t k1 = k0, tot = 0;                    // lists k0 .. k1 - 1 in this batch
        while (k1 < nl && tot + ((xl[k1].S + 31) & ~31u) <= sm.tmp_words) tot += (xl[k1++].S + 31) & ~31u;
        __syncthreads();                              // s_tmp / r.qA / s_xoff are free
        if (tid == 0) {
            uint32_t o = 0;
            for (uint32_t k = k0; k < k1; ++k) { s_xoff[k - k0] = o; o += (xl[k].S + 31) & ~31u; }
            s_xoff[k1 - k0] = o;
        }
        for (uint32_t k = k0, o = 0; k < k1; o += (xl[k].S + 31) & ~31u, ++k)
            for (uint32_t t = tid; t < xl[k].S; t += blockDim.x) sm.s_tmp[o + t] = __ldcg(xl[k].val + t);
        __syncthreads();
        const uint32_t nq = tot / 32, nk = k1 - k0;
        // the list of group q (warp-uniform), and the valid words in it
        auto qlist = [&](uint32_t q, uint32_t &e, uint32_t &pos0) {
            uint32_t k = 0;
            while (k + 1 < nk && s_xoff[k + 1] <= 32 * q) ++k;
            pos0 = 32 * q - s_xoff[k];
            e = min(32u, xl[k0 + k].S - pos0);
            return k0 + k;
        };
        for (uint32_t q = tid >> 5; q < nq; q += blockDim.x >> 5) {
            uint32_t e, pos0;
            qlist(q, e, pos0);
            const uint32_t x = (uint32_t)lane < e ? sm.s_tmp[32 * q + lane] : 0u;
            const uint32_t qA = __reduce_and_sync(0xffffffffu, (uint32_t)lane < e ? x : ~0u);
            const uint32_t qO = __reduce_or_sync(0xffffffffu, x);
            if (lane == 0) { r.qA[q] = qA; r.qO[q] = qO; }
        }
        __syncthreads();
        const uint32_t ntask = ng * nq;
        auto tasks = [&](auto so_tag, auto mix_tag) {
            constexpr bool SO = decltype(so_tag)::value;
            constexpr int MIXC = decltype(mix_tag)::value;
            auto cf = [&](uint32_t u, uint32_t w, int t) {
                if (MIXC >= 2 && (t & 1)) return p_clear_low<MIXC>(u ^ w) == 0u;
                return (uint32_t)__popc(u ^ w) < a.d || (SO && (__popc(u & w) & 1));
            };
            for (uint32_t p = tid >> 5; p < ntask; p += blockDim.x >> 5) {
                const uint32_t g = p / nq, q = p - g * nq;
                if (!SO && p_lb(r.gA[g], r.gO[g], r.qA[q], r.qO[q], a.nmask) >= a.d) continue;
                uint32_t e, pos0;
                const uint32_t b = qlist(q, e, pos0) + 1;
                const uint32_t j = 32 * g + lane;
                const uint32_t vj = j < S ? sm.s_val[j] : 0u;
                const uint4 *w4 = reinterpret_cast<const uint4 *>(sm.s_tmp + 32 * q);
                uint32_t mask = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint4 c = w4[k];
                    mask |= (uint32_t)cf(vj, c.x, 4 * k) << (4 * k);
                    mask |= (uint32_t)cf(vj, c.y, 4 * k + 1) << (4 * k + 1);
                    mask |= (uint32_t)cf(vj, c.z, 4 * k + 2) << (4 * k + 2);
                    mask |= (uint32_t)cf(vj, c.w, 4 * k + 3) << (4 * k + 3);
                }
                if (e < 32) mask &= (1u << e) - 1u;
                if (j < S) rchk += e;
                if (j < S && mask) {
                    uint32_t qq = atomicAdd(&sm.s_cnt[j], (uint32_t)__popc(mask));
                    while (mask) {
                        const uint32_t t = __ffs(mask) - 1;
                        mask &= mask - 1;
                        if (qq < (uint32_t)kPX)
                            __stcg(xadj + (size_t)j * kPX + qq, (uint16_t)((b << 12) | (pos0 + t)));
                        ++qq;
                    }
                }
            }
        };
        if (a.so) tasks(std::true_type{}, std::integral_constant<int, 0>{});
        else if (a.mix == 2) tasks(std::false_type{}, std::integral_constant<int, 2>{});
        else if (a.mix == 3) tasks(std::false_type{}, std::integral_constant<int, 3>{});
        else if (a.mix == 4) tasks(std::false_type{}, std::integral_constant<int, 4>{});
        else tasks(std::false_type{}, std::integral_constant<int, 0>{});
        k0 = k1;
    }
    __syncthreads();
}

// v in conflict with one of the words w[0, e) (shared memory, the same address in every lane):
// distance < d, or (SO) odd AND-parity.  A full block of 32 is read four words per 128-bit
// broadcast load, fully unrolled; with MIX (2..4) odd words use the ALU bit-clearing form of the
// distance test so that the POPC and ALU pipes share the work.
template <bool SO, int MIX>
__device__ __forceinline__ bool r_hit(uint32_t v, const uint32_t *w, uint32_t e, uint32_t d) {
    uint32_t m = 0xffffffffu;
    bool hit = false;
    if (e == 32) {
        const uint4 *w4 = reinterpret_cast<const uint4 *>(w);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint4 c = w4[k];
            const uint32_t cs[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (SO) hit |= (__popc(v & cs[u]) & 1) != 0;
                if (MIX >= 2 && (u & 1)) hit |= p_clear_low<MIX>(v ^ cs[u]) == 0u;
                else m = min(m, (uint32_t)__popc(v ^ cs[u]));
            }
        }
    } else {
        for (uint32_t t = 0; t < e; ++t) {
            const uint32_t c = w[t];
            if (SO) hit |= (__popc(v & c) & 1) != 0;
            m = min(m, (uint32_t)__popc(v ^ c));
        }
    }
    return hit || m < d;
}

// Survivors s_val[0, Sc) against committed words codebook[lo, hi) the screen did not see:
// s_status[j] |= 1 on a conflict (zeroed first unless `accumulate`).  The words are staged
// through shared memory newest first; a warp task is (group of 32 survivors, block of 32 staged
// words), skipped when the consensus bound of the two is >= d.  Needs r_consensus.  Ends with a
// barrier.
// first_loaded: the newest batch, codebook[hi - min(tmp_words, hi - lo), hi), is already in s_tmp.
// first_ready (with first_loaded and accumulate): its group consensus is in r.qA / r.qO too and a
// barrier has passed since -- the first batch's tasks start at once.
__device__ __forceinline__ void r_prior(const PArgs &a, const PSmem &sm, uint32_t Sc, unsigned long long lo,
                                        unsigned long long hi, bool accumulate, unsigned long long &rchk,
                                        bool first_loaded = false, bool first_ready = false) {
    RShared &r = p_rsh();
    const int lane = threadIdx.x & 31;
    const uint32_t tid = threadIdx.x;
    const uint32_t ng = (Sc + 31) / 32;
    if (!accumulate)
        for (uint32_t j = tid; j < Sc; j += blockDim.x) sm.s_status[j] = 0;
    for (unsigned long long top = hi; top > lo;) {
        const uint32_t nb = (uint32_t)min((unsigned long long)sm.tmp_words, top - lo);
        const unsigned long long b0 = top - nb;
        const uint32_t nq = (nb + 31) / 32;
        if (!(first_ready && top == hi)) {
            __syncthreads();
            if (!first_loaded || top != hi)
                for (uint32_t t = tid; t < nb; t += blockDim.x) sm.s_tmp[t] = __ldcg(a.codebook + b0 + t);
            __syncthreads();
            for (uint32_t q = tid >> 5; q < nq; q += blockDim.x >> 5) {
                const uint32_t k = 32 * q + lane;
                const uint32_t x = k < nb ? sm.s_tmp[k] : 0u;
                const uint32_t qA = __reduce_and_sync(0xffffffffu, k < nb ? x : ~0u);
                const uint32_t qO = __reduce_or_sync(0xffffffffu, x);
                if (lane == 0) { r.qA[q] = qA; r.qO[q] = qO; }
            }
            __syncthreads();
        }
        const uint32_t ntask = ng * nq;
        auto tasks = [&](auto so_tag, auto mix_tag) {
            constexpr bool SO = decltype(so_tag)::value;
            constexpr int MIX = decltype(mix_tag)::value;
            for (uint32_t p = tid >> 5; p < ntask; p += blockDim.x >> 5) {
                const uint32_t g = p / nq, q = p - g * nq;
                if (!SO && p_lb(r.gA[g], r.gO[g], r.qA[q], r.qO[q], a.nmask) >= a.d) continue;
                const uint32_t j = 32 * g + lane;
                const uint32_t vj = j < Sc ? sm.s_val[j] : 0u;
                const uint32_t e = min(32u, nb - 32 * q);
                const bool c = r_hit<SO, MIX>(vj, sm.s_tmp + 32 * q, e, a.d);
                if (j < Sc) {
                    rchk += e;
                    if (c) sm.s_status[j] = 1;
                }
            }
        };
        if (a.so) tasks(std::true_type{}, std::integral_constant<int, 0>{});
        else if (a.mix == 2) tasks(std::false_type{}, std::integral_constant<int, 2>{});
        else if (a.mix == 3) tasks(std::false_type{}, std::integral_constant<int, 3>{});
        else if (a.mix == 4) tasks(std::false_type{}, std::integral_constant<int, 4>{});
        else tasks(std::false_type{}, std::integral_constant<int, 0>{});
        top = b0;
    }
    __syncthreads();
}

// Stable compaction of the chunk s_val / s_idx [0, Sc) to the survivors with s_status == 0 (no
// conflict with a committed word), in place: a round reads its elements before any of them is
// overwritten and writes only below its own range.  Returns the count (CTA-uniform).  Ends with
// a barrier.
__device__ __forceinline__ uint32_t r_compact(const PSmem &sm, uint32_t Sc) {
    uint32_t out = 0;
    for (uint32_t j0 = 0; j0 < Sc; j0 += blockDim.x) {
        const uint32_t j = j0 + threadIdx.x;
        const bool keep = j < Sc && sm.s_status[j] == 0;
        const uint32_t v = keep ? sm.s_val[j] : 0u;
        const uint16_t ix = keep ? sm.s_idx[j] : (uint16_t)0;
        uint32_t tot;
        const uint32_t pos = out + p_block_scan(keep ? 1u : 0u, &tot, sm.s_ws);   // has barriers
        if (keep) { sm.s_val[pos] = v; sm.s_idx[pos] = ix; }
        out += tot;
        __syncthreads();
    }
    return out;
}

// a3.3 decide the chunk s_val[0, Sc) in rank order: s_status = 1 accepted / 0 rejected.
// On entry s_cnt / s_adj hold the in-chunk conflict lists and, when `prior`, s_status[j] != 0
// marks a survivor with a conflict outside the chunk (rejected outright; counted in pkill).
// Parallel rounds: an undecided survivor is rejected as soon as one earlier conflicting survivor
// is accepted, accepted once all of them are rejected; long chains are finished by warp 0 in
// rank order.  A survivor is accepted iff no earlier ACCEPTED survivor conflicts.
// Survivors with more than kPAdj earlier conflicts ("overflow") are listed (up to kPOvf) and
// decided by a whole warp per node.  Ends with a barrier.
__device__ __forceinline__ void r_decide(const PArgs &a, const PSmem &sm, uint32_t Sc, bool prior,
                                         unsigned long long &confl, unsigned long long &pkill, PTimers *timer,
                                         unsigned long long &tr) {
    RShared &r = p_rsh();
    PState *st = a.st;
    const int lane = threadIdx.x & 31;
    const uint32_t tid = threadIdx.x;
    uint8_t *s_status = sm.s_status;
    const uint32_t *s_val = sm.s_val;
    uint32_t *s_cnt = sm.s_cnt;
    const uint16_t *s_adj = sm.s_adj;
    if (tid == 0) { r.novf = 0; r.und[0] = 0; }
    __syncthreads();
    for (uint32_t j = tid; j < Sc; j += blockDim.x) {
        const bool prev = prior && s_status[j] != 0;
        const uint32_t cnt = s_cnt[j];
        s_status[j] = prev ? 0 : (cnt ? 2 : 1);
        confl += cnt;
        pkill += prev;
        if (cnt > kPAdj) {
            if (a.timing) atomicAdd(&st->n_overflow, 1ull);
            if (!prev) {
                const uint32_t o = atomicAdd(&r.novf, 1u);
                if (o < kPOvf) { r.ovf[o] = (uint16_t)j; s_cnt[j] = kPOvfMark; }
            }
        }
    }
    __syncthreads();
    const uint32_t novf = min(r.novf, kPOvf);
    if (timer) { const unsigned long long t_ = clock64(); timer->r[5] += t_ - tr; tr = t_; }
    // rounds read the statuses of one buffer and write the next one (the pad bytes after s_status),
    // so a round never reads a status another thread is writing
    uint8_t *cur = s_status, *nxt = s_status + sm.chunk;
    int left = 0, prev_cnt = 1 << 30;
    for (int round = 0; round < 8; ++round) {
        int undecided = 0;
        for (uint32_t j = tid; j < Sc; j += blockDim.x) {
            const uint8_t sj = cur[j];
            if (sj != 2) { nxt[j] = sj; continue; }
            const uint32_t cn = s_cnt[j];
            if (cn == kPOvfMark) { undecided = 1; continue; }     // a warp decides it below
            bool acc_nb = false, und_nb = false;
            if (cn <= kPAdj) {
                for (uint32_t t = 0; t < cn; ++t) {
                    const uint8_t sk = cur[s_adj[j * kPAdj + t]];
                    acc_nb |= sk == 1;
                    und_nb |= sk == 2;
                }
            } else {
                const uint32_t vj = s_val[j];
                for (uint32_t k = 0; k < j; ++k) {
                    if (p_conflict(a, vj, s_val[k])) {
                        const uint8_t sk = cur[k];
                        acc_nb |= sk == 1;
                        und_nb |= sk == 2;
                    }
                }
            }
            const uint8_t ns = acc_nb ? 0 : (!und_nb ? 1 : 2);
            nxt[j] = ns;
            undecided |= ns == 2;
        }
        for (uint32_t o = tid >> 5; o < novf; o += blockDim.x >> 5) {
            const uint32_t j = r.ovf[o];
            if (cur[j] != 2) continue;                            // warp-uniform (copied above)
            const uint32_t vj = s_val[j];
            bool acc_nb = false, und_nb = false;
            for (uint32_t k = lane; k < j; k += 32) {
                if (p_conflict(a, vj, s_val[k])) {
                    const uint8_t sk = cur[k];
                    acc_nb |= sk == 1;
                    und_nb |= sk == 2;
                }
            }
            acc_nb = __any_sync(0xffffffffu, acc_nb);
            und_nb = __any_sync(0xffffffffu, und_nb);
            if (lane == 0) nxt[j] = acc_nb ? 0 : (!und_nb ? 1 : 2);
            undecided |= !acc_nb && und_nb;
        }
        if (a.timing && tid == 0) {
            atomicAdd(&st->n_rounds, 1ull);
            atomicMax(&st->n_rounds_max, (unsigned long long)round + 1);
        }
        // threads still holding an undecided survivor; when many are left and a round settles less
        // than a quarter of them (long chains of conflicts, e.g. a tile just past a high-bit
        // boundary) the group-sequential tail below takes over.  Counted in r.und[round % 3]
        // (plain barriers only): the counter of round + 1 is zeroed before this round's barrier,
        // after every thread read it as the counter of round - 2.
        if (tid == 0) r.und[(round + 1) % 3] = 0;
        const uint32_t wu = (uint32_t)__popc(__ballot_sync(0xffffffffu, undecided));
        if (lane == 0 && wu) atomicAdd(&r.und[round % 3], wu);
        __syncthreads();
        const int cnt = (int)r.und[round % 3];
        uint8_t *t = cur; cur = nxt; nxt = t;
        left = cnt;
        if (!cnt || (round >= 1 && cnt > 96 && cnt * 4 > prev_cnt * 3)) break;
        prev_cnt = cnt;
    }
    if (cur != s_status) {
        for (uint32_t j = tid; j < Sc; j += blockDim.x) s_status[j] = cur[j];
        __syncthreads();
    }
    if (timer) { const unsigned long long t_ = clock64(); timer->r[6] += t_ - tr; tr = t_; }
    if (a.timing && tid == 0 && left) {          // diagnostics: tiles entering the tail, undecided threads
        atomicAdd(&st->t_level[12], 1ull);
        atomicAdd(&st->t_level[13], (unsigned long long)left);
    }
    if (left && left <= 64 && tid < 32) {
        // a few undecided survivors left: warp 0 decides them one by one, in rank order, finding
        // them 32 at a time by a ballot (lane t reads s_status[g0 + t]; lane 0 writes the decided
        // one, which every lane re-reads only after the __syncwarp below)
        for (uint32_t g0 = 0; g0 < Sc; g0 += 32) {
          unsigned und = __ballot_sync(0xffffffffu, g0 + lane < Sc && s_status[g0 + lane] == 2);
          __syncwarp();
          while (und) {
            const uint32_t j = g0 + (uint32_t)(__ffs(und) - 1);
            und &= und - 1;
            if (a.timing && lane == 0) atomicAdd(&st->n_seq, 1ull);
            const uint32_t cn = s_cnt[j];
            bool acc_nb = false;
            if (cn <= kPAdj) {
                if (lane < cn) acc_nb = s_status[s_adj[j * kPAdj + lane]] == 1;
            } else {
                const uint32_t vj = s_val[j];
                for (uint32_t k = lane; k < j; k += 32)
                    acc_nb |= (s_status[k] == 1) && p_conflict(a, vj, s_val[k]);
            }
            acc_nb = __any_sync(0xffffffffu, acc_nb);
            if (lane == 0) s_status[j] = acc_nb ? 0 : 1;
            __syncwarp();
          }
        }
    } else if (left && tid < 32) {
        // warp 0 finishes the undecided survivors group by group (32 consecutive ones, in rank
        // order): lane t owns survivor g0 + t.  A member is rejected by an accepted survivor
        // before the group -- its conflict list, or, for an overflow node (more conflicts than the
        // list holds), the values of the accepted survivors so far, kept in order in s_tmp (free
        // after the prior checks) -- else decided by the group's own greedy over a 32 x 32
        // conflict bit matrix held in registers.
        const bool use_list = Sc <= sm.tmp_words;
        uint32_t n_acc = 0;                                // accepted survivors before g0 (use_list)
        for (uint32_t g0 = 0; g0 < Sc; g0 += 32) {
            const uint32_t j = g0 + lane;
            const bool in = j < Sc;
            const uint32_t sj = in ? (uint32_t)s_status[j] : 0u;   // lane-owned until the write below
            const uint32_t vj = in ? s_val[j] : 0u;
            const unsigned und = __ballot_sync(0xffffffffu, in && sj == 2);
            unsigned acc = __ballot_sync(0xffffffffu, in && sj == 1);
            if (und) {
                if (a.timing && lane == 0) atomicAdd(&st->n_seq, 1ull);
                const uint32_t cn = in ? s_cnt[j] : 0u;
                bool pre = false;
                if (sj == 2 && cn <= kPAdj) {
                    for (uint32_t t = 0; t < cn; ++t) {
                        const uint32_t k = s_adj[j * kPAdj + t];
                        pre |= k < g0 && s_status[k] == 1;
                    }
                } else if (sj == 2 && use_list) {          // overflow node: the accepted list, newest first
                    for (uint32_t k = n_acc; k > 0 && !pre; --k) pre = p_conflict(a, vj, sm.s_tmp[k - 1]);
                }
                unsigned ovm = use_list ? 0u : __ballot_sync(0xffffffffu, sj == 2 && cn > kPAdj);
                while (ovm) {                              // (no room for the list) the warp scans
                    const int t = __ffs(ovm) - 1;
                    ovm &= ovm - 1;
                    const uint32_t vt = __shfl_sync(0xffffffffu, vj, t);
                    bool c = false;
                    for (uint32_t k = lane; k < g0; k += 32) c |= s_status[k] == 1 && p_conflict(a, vt, s_val[k]);
                    c = __any_sync(0xffffffffu, c);
                    if (lane == t) pre |= c;
                }
                uint32_t inmask = 0;                       // earlier members of the group in conflict
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const uint32_t vt = __shfl_sync(0xffffffffu, vj, t);
                    if (t < lane && p_conflict(a, vj, vt)) inmask |= 1u << t;
                }
                const unsigned prem = __ballot_sync(0xffffffffu, pre);
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    const uint32_t im = __shfl_sync(0xffffffffu, inmask, t);
                    if (((und & ~prem) >> t & 1u) && !(im & acc)) acc |= 1u << t;
                }
                if (sj == 2) s_status[j] = (acc >> lane & 1u) ? 1 : 0;
            }
            if (use_list) {                                // the group's accepted members, in order
                if (acc >> lane & 1u) sm.s_tmp[n_acc + __popc(acc & ((1u << lane) - 1u))] = vj;
                n_acc += __popc(acc);
            }
            __syncwarp();
        }
    }
    if (timer) { const unsigned long long t_ = clock64(); timer->r[7] += t_ - tr; }
    __syncthreads();
    if (timer) { const unsigned long long t_ = clock64(); timer->r[2] += t_ - tr; tr = t_; }
}

// a4 ordered append of the chunk's accepted survivors at codebook[M0 + A, ...); their values are
// also staged in order (in s_adj, free now) for the block-bound summaries: AND / OR per aligned
// block of 32 (a warp covers one block) and per super-block of 1024 -- appends only ever narrow
// the AND and widen the OR; fire-and-forget atomics published by the commit's release.
// Returns the new A (CTA-uniform).  Ends with a barrier.
__device__ __forceinline__ uint32_t r_append(const PArgs &a, const PSmem &sm, uint32_t Sc, unsigned long long M0,
                                             uint32_t A, unsigned long long t0, unsigned long long &sidx,
                                             uint32_t *accbits = nullptr) {
    RShared &r = p_rsh();
    PState *st = a.st;
    const int lane = threadIdx.x & 31;
    const uint32_t tid = threadIdx.x;
    uint32_t *s_stage = reinterpret_cast<uint32_t *>(sm.s_adj);
    const uint32_t A_start = A;
    for (uint32_t j0 = 0; j0 < Sc; j0 += blockDim.x) {
        const uint32_t j = j0 + tid;
        const uint32_t acc = (j < Sc && sm.s_status[j] == 1) ? 1u : 0u;
        if (accbits) {                         // accepted positions of the chunk, one word per warp
            const unsigned bal = __ballot_sync(0xffffffffu, acc);
            if (lane == 0 && (j >> 5) < 64) accbits[j >> 5] = bal;
        }
        uint32_t tot;
        const uint32_t pos = A + p_block_scan(acc, &tot, sm.s_ws);
        if (acc) {
            const unsigned long long p = M0 + pos;
            const uint32_t v = sm.s_val[j];
            s_stage[pos - A_start] = v;
            if (a.weight_bound) atomicMin(&r.wmin[__popc(v)], pos);
            if (p < a.capacity) {
                a.codebook[p] = v;
            } else {
                st->error = 1;
            }
            sidx += sm.s_idx[j];         // W_def of the tile = A (2^n - 1 - t0) - (sum of in-tile indices)
        }
        A += tot;
    }
    __syncthreads();
    if (a.bound && A > A_start) {
        const unsigned long long b = M0 + A_start, e = min(M0 + A, (unsigned long long)a.capacity);
        const unsigned long long p0 = b & ~31ull;
        for (unsigned long long p = p0 + tid; p < ((e + 31) & ~31ull); p += blockDim.x) {
            const bool in = p >= b && p < e;
            const uint32_t w = in ? p_ptag(a, s_stage[p - b]) : 0u;   // parity-tagged (a.par)
            const uint32_t an = __reduce_and_sync(0xffffffffu, in ? w : ~0u);
            const uint32_t orr = __reduce_or_sync(0xffffffffu, w);
            if (lane == 0) {
                atomicAnd(&a.bsum[p >> 5].x, an);
                atomicOr(&a.bsum[p >> 5].y, orr);
                atomicAnd(&a.ssum[p >> 10].x, an);
                atomicOr(&a.ssum[p >> 10].y, orr);
            }
        }
    }
    if (A > a.capacity - M0) A = (uint32_t)(a.capacity - M0);
    __threadfence_block();
    __syncthreads();
    return A;
}

// a3 + a4 for one tile, by ONE CTA: survivors in rank order (from the dead mask), in-tile
// ordered resolve, ordered append, M += A, next tile size, per-tile state cleared.
// dead: the tile's dead mask (read, then cleared for the next tile that uses it).
// prior_lo: survivors are also checked against the committed words codebook[prior_lo, M) --
//   the pipelined engine screens a tile against an older codebook, codebook[0, prior_lo)
//   (k_construct: prior_lo = M, nothing to check).
// prep (pipelined engine, may be null): the tile's survivors were gathered, checked against
//   codebook[prior_lo, prep->M_prep) and their conflict lists built by another CTA; they are
//   loaded instead, and only codebook[prep->M_prep, M) remains to be checked.
// On return (thread 0): pc.M / stats updated, pc.S_tile (survivors without a committed
// conflict) / pc.A_tile / pc.K_used set; the next tile size is the caller's decision.
__device__ __forceinline__ void p_resolve(const PArgs &a, const PSmem &sm, unsigned long long t0, uint32_t K, int L,
                                          PCount &pc, PTimers *timer, unsigned long long tm, bool allow_partial,
                                          uint32_t *dead, unsigned long long prior_lo, const PPrep *prep = nullptr,
                                          uint32_t *accbits = nullptr) {
    const uint32_t kPChunk = sm.chunk;
    PState *st = a.st;
    RShared &r = p_rsh();
    const int lane = threadIdx.x & 31;
    const uint32_t words = (K + 31) / 32;
    const uint32_t tid = threadIdx.x;
    const unsigned long long tg = timer ? clock64() : 0;
    uint32_t S;
    bool pre_loaded = false;
    // a prepared burst (more than two sub-chunks of survivors, typically just past a high-bit or a
    // weight-class boundary, where they conflict densely): decided sub-chunk by sub-chunk from the
    // prepared list like an unprepared multi-chunk tile -- the words accepted in the earlier sub-chunks
    // reject most of a later one before its conflict lists are built (the prepared lists are unused)
    const bool big = prep && p_prep_big(a, *prep);
    if (big) {
        S = prep->S;
        prior_lo = prep->M_prep;
    } else if (prep) {
        S = prep->S;
        prior_lo = prep->M_prep;
        // one round trip: the prepared survivors and the newest committed words they still have to
        // be checked against (r_prior's first batch)
        const unsigned long long M0 = pc.M;
        // the newest words (r_prior's first batch) and the survivors, each 32-group's consensus
        // (AND / OR) taken by the warp that loads it, statuses initialised: r_consensus and the
        // first batch of r_prior need no pass and no barrier of their own (pre_ready)
        if (!prep->xmode && M0 > prior_lo && S > 0) {
            const uint32_t nb = (uint32_t)min((unsigned long long)sm.tmp_words, M0 - prior_lo);
            for (uint32_t t0w = 0; t0w < nb; t0w += blockDim.x) {
                const uint32_t t = t0w + tid;
                const uint32_t x = t < nb ? __ldcg(a.codebook + M0 - nb + t) : 0u;
                if (t < nb) sm.s_tmp[t] = x;
                const uint32_t qA = __reduce_and_sync(0xffffffffu, t < nb ? x : ~0u);
                const uint32_t qO = __reduce_or_sync(0xffffffffu, x);
                if (lane == 0 && t < nb) { r.qA[t >> 5] = qA; r.qO[t >> 5] = qO; }
            }
            pre_loaded = true;
        }
        for (uint32_t j0 = 0; j0 < S; j0 += blockDim.x) {
            const uint32_t j = j0 + tid;
            const uint32_t x = j < S ? __ldcg(prep->val + j) : 0u;
            const uint32_t gA = __reduce_and_sync(0xffffffffu, j < S ? x : ~0u);
            const uint32_t gO = __reduce_or_sync(0xffffffffu, x);
            if (lane == 0 && j < S) { r.gA[j >> 5] = gA; r.gO[j >> 5] = gO; }
            if (j >= S) continue;
            sm.s_val[j] = x;
            sm.s_cnt[j] = __ldcg(prep->cnt + j);
            sm.s_idx[j] = __ldcg(prep->idx + j);
            if (!prep->xstage) sm.s_status[j] = 0;
            if (prep->xstage) {
                // stage B flagged the survivors in conflict with the words committed after stage A;
                // cross mode: also rejected iff one of its recorded conflicts in the list of the tile
                // before was accepted there (its accepted words are all of codebook[M_prep, M0))
                const uint32_t xc = __ldcg(prep->xcnt + j);
                bool hit = xc == 0xffu;
                for (uint32_t q = 0; prep->xmode && !hit && q < xc; ++q) {
                    const uint32_t e = __ldcg(prep->xadj + (size_t)j * kPX + q);
                    const uint32_t p = e & 0xfffu;
                    hit |= (prep->xbits[(prep->tile - (e >> 12)) % kPXRing][p >> 5] >> (p & 31)) & 1u;
                }
                sm.s_status[j] = hit ? 1 : 0;
            }
        }
        const uint4 *src = reinterpret_cast<const uint4 *>(prep->adj);
        uint4 *dst = reinterpret_cast<uint4 *>(sm.s_adj);
        for (uint32_t q = tid; q < S * (kPAdj / 8); q += blockDim.x) dst[q] = __ldcg(src + q);
        __syncthreads();
    } else {
        S = r_gather(a, sm, t0, K, L, dead, a.surv);
    }
    const uint32_t S_screen = prep ? prep->S_screen : S;
    // Partial tile (k_construct): with more survivors than one chunk, only the candidates ranked
    // before the first survivor of the second chunk are decided now; the tile is cut there
    // (K_used) and the rest is screened again as part of the next tile, against a codebook that
    // then holds this chunk's accepted words.  Exact (tile boundaries never change the result)
    // and it bounds a resolve to one chunk.
    uint32_t K_used = K;
    const uint32_t s_cut = min(kPChunk, a.partial_s);
    if (!prep && allow_partial && S > s_cut) {
        K_used = s_cut < kPChunk ? sm.s_idx[s_cut] : __ldcg(&a.surv[kPChunk].x);
        S = s_cut;
    }
    // resolve sub-steps timed with the SM cycle counter (one CTA: consistent, and cheap to read)
    unsigned long long tr = timer ? clock64() : 0;
#define P_TR(i) if (timer) { const unsigned long long t_ = clock64(); timer->r[i] += t_ - tr; tr = t_; }
    if (timer) timer->r[0] += tr - tg;
    if (a.timing && tid == 0) {
        atomicMax(&st->s_max, (unsigned long long)S);
        if (S > kPChunk) atomicAdd(&st->n_chunked, 1ull);
    }
    if (tid < 33) r.wmin[tid] = 0xffffffffu;
    unsigned long long rchk = 0, confl = 0, sidx = 0, pkill = 0;
    if (tid < 4) r.tsum[tid] = 0;
    const unsigned long long M0 = pc.M;
    uint32_t A = 0;                   // accepted so far in this tile (codebook[M0, M0+A))
    // More survivors than one chunk (a "burst": e.g. a tile just past a high-bit boundary, where
    // most candidates survive a screen against an older codebook and kill each other): decided in
    // sub-chunks of burst_chunk from a.surv -- each one checked against the words accepted in the
    // earlier ones first, so the in-chunk conflict lists (quadratic) stay small.
    const bool multi = S > kPChunk || big;
    const uint32_t step = multi ? min(kPChunk, max(32u, a.burst_chunk)) : kPChunk;
    if (multi && !big) {
        for (uint32_t j = tid; j < kPChunk; j += blockDim.x) a.surv[j] = make_uint2(sm.s_idx[j], sm.s_val[j]);
        __syncthreads();
    }
    for (uint32_t c0 = 0; c0 < S; c0 += step) {
        uint32_t Sc = min(step, S - c0);
        if (big) {
            for (uint32_t j = tid; j < Sc; j += blockDim.x) {
                sm.s_idx[j] = __ldcg(prep->idx + c0 + j);
                sm.s_val[j] = __ldcg(prep->val + c0 + j);
            }
        } else if (multi) {
            for (uint32_t j = tid; j < Sc; j += blockDim.x) {
                const uint2 e = __ldcg(a.surv + c0 + j);
                sm.s_idx[j] = (uint16_t)e.x;
                sm.s_val[j] = e.y;
            }
        }
        __syncthreads();
        const bool pc_prior = M0 > prior_lo, ch_prior = A > 0;
        if (prep && !big) {
            // the preparer built the conflict lists; the committed words it did not see only flag
            // (cross mode: the cross lists flagged them at the load)
            const bool xm = prep->xmode != 0;
            // (consensus of the survivors and of the newest words taken at the load; statuses zeroed
            // there, or set from stage B's flags)
            if (!xm && pc_prior && Sc) r_prior(a, sm, Sc, prior_lo, M0, true, rchk, pre_loaded, pre_loaded);
            P_TR(1)
            r_decide(a, sm, Sc, xm || prep->xstage || pc_prior, confl, pkill, timer, tr);
        } else {
            r_consensus(sm, Sc);
            // Survivors conflicting with a committed word the screen did not see are rejected first:
            // codebook[prior_lo, M0) (pipelined engine: the tile was screened against an older
            // codebook) and [M0, M0 + A) (words accepted in this tile's earlier chunks).  The rest
            // is compacted and only it gets in-tile conflict lists.  The first kind also leaves the
            // survivor count the tile size is chosen from (pkill).
            if (pc_prior || ch_prior) {
                if (pc_prior) r_prior(a, sm, Sc, prior_lo, M0, false, rchk, pre_loaded);
                if (ch_prior) {
                    if (pc_prior)
                        for (uint32_t j = tid; j < Sc; j += blockDim.x) pkill += sm.s_status[j] != 0;
                    r_prior(a, sm, Sc, M0, M0 + A, pc_prior, rchk);
                }
                const uint32_t Sc2 = r_compact(sm, Sc);
                if (pc_prior && !ch_prior && tid == 0) pkill += Sc - Sc2;
                Sc = Sc2;
                r_consensus(sm, Sc);
            }
            r_units(a, sm, Sc, rchk);
            P_TR(1)
            unsigned long long none = 0;
            r_decide(a, sm, Sc, false, confl, none, timer, tr);
        }
        A = r_append(a, sm, Sc, M0, A, t0, sidx, (prep && !big) ? accbits : nullptr);
        P_TR(3)
    }
    // clear per-tile state for the next tile (a prepared tile's mask was cleared by its preparer)
    if (!prep)
        for (uint32_t w = tid; w < words; w += blockDim.x) dead[w] = 0;
    // the tile's counters: each fits 32 bits (a tile has < 2^16 candidates, a resolve chunk checks
    // < 2^12 survivors against < 2^20 words), so one redux.sync per warp and one shared atomic each
    // replace 64-bit shuffle trees
    {
        const uint32_t w0 = __reduce_add_sync(0xffffffffu, (uint32_t)rchk);
        const uint32_t w1 = __reduce_add_sync(0xffffffffu, (uint32_t)confl);
        const uint32_t w2 = __reduce_add_sync(0xffffffffu, (uint32_t)sidx);
        const uint32_t w3 = __reduce_add_sync(0xffffffffu, (uint32_t)pkill);
        if (lane == 0) {
            if (w0) atomicAdd(&r.tsum[0], w0);
            if (w1) atomicAdd(&r.tsum[1], w1);
            if (w2) atomicAdd(&r.tsum[2], w2);
            if (w3) atomicAdd(&r.tsum[3], w3);
        }
    }
    __syncthreads();
    unsigned long long pk = 0;
    if (tid == 0) {
        pc.resolve_checks += r.tsum[0];
        pc.conflicts += r.tsum[1];
        if (a.wdef_valid) pc.w_def += (unsigned long long)A * (a.N - 1 - t0) - r.tsum[2];
        pk = r.tsum[3];
    }
    if (tid == 0) {
        const uint32_t S_true = S - (uint32_t)min(pk, (unsigned long long)S);
        unsigned long long M1 = M0 + A;
        if (M1 > a.capacity) M1 = a.capacity;
        pc.M = M1;
        st->M = M1;
        const uint32_t S_size = a.size_on_screen ? max(S_true, S_screen) : S_true;
        if (S_size) { pc.S_last = S_size; pc.K_last = K_used; }
        // (tile sizes stay powers of two: a partial tile's length is rounded down first)
        pc.K_next = p_next_tile(a, 1u << (31 - __clz(K_used)), S_true, A, t0 + K_used, M1, pc.S_last,
                                pc.K_last ? pc.K_last : 1u);
        pc.K_used = K_used;
        pc.S_tile = S_true;
        pc.A_tile = A;
        st->K_next = pc.K_next;
        pc.survivors += S_true;
        pc.tiles += 1;
        pc.levels += L;
    }
    P_TR(4)
#undef P_TR
    if (a.weight_bound && tid < 33 && r.wmin[tid] != 0xffffffffu && !pc.wfirst[tid] &&
        M0 + r.wmin[tid] < a.capacity) {
        // first codebook index of each weight (acceptance order is weight-sorted for graded
        // orders); stored +1, 0 = none yet
        pc.wfirst[tid] = (unsigned int)(M0 + r.wmin[tid] + 1);
        st->wfirst[tid] = pc.wfirst[tid];
    }
    __syncthreads();
}

// Prepare a tile for the resolver (pipelined engine; run by a whole CTA while earlier tiles are
// resolved): gather its survivors, reject those conflicting with the words committed since its
// screen (codebook[M_s, M_c)), compact the rest in rank order, build their in-tile conflict
// lists, and store everything in the slot's prep buffer (p_prep_bytes layout).  Survivors beyond
// one chunk are spilled to `spill` and checked chunk by chunk.  Returns the number stored, or
// 0xffffffff when more than one chunk is left after the checks (the resolver then does the whole
// tile itself, from the dead mask, which is left intact); otherwise the dead mask is cleared
// here.  S_screen: the survivors of the screen.  rchk: work counter.
__device__ __forceinline__ uint32_t p_prep(const PArgs &a, const PSmem &sm, unsigned long long t0, uint32_t K, int L,
                                           uint32_t *dead, unsigned long long M_s, unsigned long long M_c,
                                           uint8_t *buf, uint2 *spill, unsigned long long &rchk, uint32_t &S_screen) {
    const uint32_t tid = threadIdx.x;
    // the newest words the survivors are checked against (r_prior's first batch), with their group
    // consensus, staged while the survivors are gathered (s_tmp is not used by the gather)
    bool pre = false;
    if (M_c > M_s) {
        const int lane = tid & 31;
        RShared &r = p_rsh();
        const uint32_t nb = (uint32_t)min((unsigned long long)sm.tmp_words, M_c - M_s);
        for (uint32_t t0w = 0; t0w < nb; t0w += blockDim.x) {
            const uint32_t t = t0w + tid;
            const uint32_t x = t < nb ? __ldcg(a.codebook + M_c - nb + t) : 0u;
            if (t < nb) sm.s_tmp[t] = x;
            const uint32_t qA = __reduce_and_sync(0xffffffffu, t < nb ? x : ~0u);
            const uint32_t qO = __reduce_or_sync(0xffffffffu, x);
            if (lane == 0 && t < nb) { r.qA[t >> 5] = qA; r.qO[t >> 5] = qO; }
        }
        pre = true;
    }
    const uint32_t S = r_gather(a, sm, t0, K, L, dead, spill);
    S_screen = S;
    uint32_t *val = reinterpret_cast<uint32_t *>(buf);
    uint32_t *cnt = reinterpret_cast<uint32_t *>(buf + (size_t)sm.chunk * 4);
    uint16_t *idx = reinterpret_cast<uint16_t *>(buf + (size_t)sm.chunk * 8);
    uint4 *adj = reinterpret_cast<uint4 *>(buf + (size_t)sm.chunk * 10);
    const bool multi = S > sm.chunk;
    uint32_t out = 0;
    for (uint32_t c0 = 0; c0 < S; c0 += sm.chunk) {
        uint32_t Sc = min(sm.chunk, S - c0);
        if (c0 > 0) {
            for (uint32_t j = tid; j < Sc; j += blockDim.x) {
                const uint2 e = __ldcg(spill + c0 + j);
                sm.s_idx[j] = (uint16_t)e.x;
                sm.s_val[j] = e.y;
            }
            __syncthreads();
        }
        if (M_c > M_s && Sc > 0) {
            r_consensus(sm, Sc, true);
            r_prior(a, sm, Sc, M_s, M_c, true, rchk, pre && c0 == 0, pre && c0 == 0);
            Sc = r_compact(sm, Sc);
        }
        if (out + Sc > sm.chunk) return 0xffffffffu;
        if (multi) {          // collect the compacted chunks in the prep buffer
            for (uint32_t j = tid; j < Sc; j += blockDim.x) {
                __stcg(val + out + j, sm.s_val[j]);
                __stcg(idx + out + j, sm.s_idx[j]);
            }
            __syncthreads();
        }
        out += Sc;
    }
    if (multi) {
        for (uint32_t j = tid; j < out; j += blockDim.x) {
            sm.s_val[j] = __ldcg(val + j);
            sm.s_idx[j] = __ldcg(idx + j);
        }
        __syncthreads();
    }
    const uint32_t S2 = out;
    if (S2 > 0) {
        r_consensus(sm, S2);
        r_units(a, sm, S2, rchk);
    }
    for (uint32_t j = tid; j < S2; j += blockDim.x) {
        __stcg(val + j, sm.s_val[j]);
        __stcg(cnt + j, sm.s_cnt[j]);
        __stcg(idx + j, sm.s_idx[j]);
    }
    const uint4 *sa = reinterpret_cast<const uint4 *>(sm.s_adj);
    for (uint32_t q = tid; q < S2 * (kPAdj / 8); q += blockDim.x) __stcg(adj + q, sa[q]);
    // the mask is not read again: clear it for the next tile that uses the slot
    for (uint32_t w = tid; w < (K + 31) / 32; w += blockDim.x) dead[w] = 0;
    __syncthreads();
    return S2;
}

// host: the problem / schedule fields of PArgs (gc_persistent.cu)
void p_fill_args(const RunArgs &r, PArgs *a);

}  // namespace gc
