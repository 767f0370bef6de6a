/*
 * include/gc.h -- C ABI of libgc.so, the B200 (sm_100a) greedy binary-code engine.
 *
 * The operation (PAPER.md = arXiv 1507.05398 text, /root/reference/PAPER.md):
 *   "Given n, d ... construct the code C using different orderings in greedy
 *    approach" (Sec. 3).  "First step is ordering all the vectors of
 *    F_2^n.  Next, the vectors are appended to code C from the set F_2^n one by one
 *    starting from zero vector.  The vectors are checked to satisfy the constraint
 *    of minimum Hamming distance d from all the previous choices in code C.  The
 *    algorithm terminates when all the 2^n vectors are exhausted."
 *   Distance = popcount(u XOR v) (Sec. 5.2).  Orderings: lexicographic,
 *   Gray, graded-lexicographic, graded-reverse-lexicographic (Sec. 4.2).
 *
 * Vector encoding (reading R4): a vector of F_2^n is the unsigned integer
 * whose bit n-1-i holds coordinate i, so lexicographic order is ascending integers
 * (PAPER.md:89 lists {000, 001, ..., 111}).  Orderings (R1, R2):
 *   GC_LEX            rank r -> r
 *   GC_GRAY           rank r -> r ^ (r >> 1)            (binary reflected Gray code)
 *   GC_GRADED_LEX     weight ascending, then value ascending
 *   GC_GRADED_REVLEX  weight ascending, then value descending
 * Every ordering starts at the zero vector (rank 0).
 *
 * Result: the greedy code in ACCEPTANCE order (= increasing rank).  It is a pure
 * function of (n, d, ordering): no option below changes it (PAPER.md:159's
 * "selective kernel launch" and every other schedule only reorder the evaluation
 * of "distance >= d for all previous choices").
 *
 * Conventions for every entry point:
 *   - return value is a gc_status; no exception or signal crosses the ABI;
 *   - argument validation happens before any CUDA call (so it is testable
 *     without a GPU) and leaves outputs untouched on error;
 *   - gc_last_error() returns a thread-local message for the last failure;
 *   - one construction per device at a time (calls on one device serialise on an
 *     internal per-device context; the library owns its scratch device memory).
 */
#ifndef GC_H_
#define GC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GC_ABI_VERSION 1

typedef enum gc_ordering {
    GC_LEX = 0,            /* lexicographic                        */
    GC_GRAY = 1,           /* Gray order, reflected binary (R1)      */
    GC_GRADED_LEX = 2,     /* graded-lexicographic (R2)              */
    GC_GRADED_REVLEX = 3   /* graded-reverse-lexicographic (R2)      */
} gc_ordering;

typedef enum gc_status {
    GC_OK = 0,
    GC_EINVAL = 1,         /* invalid argument (NULL pointer, n == 0, d == 0, d > n, bad ordering, bad option) */
    GC_ERANGE = 2,         /* rank or vector out of [0, 2^n)                                                      */
    GC_ENOSPC = 3,         /* output capacity too small; *out_count receives the required size                    */
    GC_EUNSUPPORTED = 4,   /* n > 32 on the GPU path (device words are 32-bit)                                    */
    GC_ECUDA = 5,          /* CUDA runtime / launch error (no device, kernel fault, ...)                           */
    GC_ENOMEM = 6,         /* device or pinned host allocation failed                                              */
    GC_ENCCL = 7,          /* NCCL unavailable or a collective failed (multi-process entry points)                 */
    GC_EINTERNAL = 8       /* internal consistency check failed (a bug; please report)                             */
} gc_status;

/* Schedule knobs.  None of them changes the result.  Zero-initialise and set
 * struct_size = sizeof(gc_options); a zero field means "default". */
typedef struct gc_options {
    uint32_t struct_size;
    uint32_t tile_min;       /* smallest candidate tile K (power of 2, >= 32), default 256              */
    uint32_t tile_max;       /* largest candidate tile K (power of 2, <= 2^20), default 65536; the
                                persistent kernel (tiles <= 65536) sizes tiles adaptively for
                                ~384 accepted words per tile (768 Gray, 1536 graded) and cuts a
                                tile after 512 survivors (1024 graded); neither changes the code  */
    uint32_t window0;        /* first newest-first codebook window (power of 2, <= 2^24); default: 4096,
                                and for the persistent engine with the block bound in lexicographic
                                order with d <= 3 the whole codebook (one screening level)       */
    uint32_t emulate_ranks;  /* >1: split every tile's candidates into this many partitions on ONE GPU,
                                exactly as gc_generate_rank splits them across GPUs (testing), default 1 */
    uint32_t flags;          /* GC_FLAG_* below                                                          */
    uint32_t window_growth;  /* log2 of the factor by which each newest-first window grows over the
                                previous one (1 = doubling ... 12 = x4096); default 2, and for the
                                persistent engines with the block bound 4 (graded orders) or 12     */
    /* persistent engines (development / tuning knobs; 0 = default, none changes the code): */
    uint32_t pipeline_depth; /* pipelined engine: tile i is screened against the codebook committed
                                after tile i - depth, so `depth` tiles are screened while one is
                                resolved; 1..16, default 8 (graded orders 10)                       */
    uint32_t target_accepted;/* adaptive tiles grow toward ~this many accepted words per tile
                                (default 384; Gray 768 -- 448 on the pipelined engine --, graded
                                orders 1536)                                                     */
    uint32_t items_per_warp; /* screen work items per warp and level (default 1; graded orders 4;
                                2 without the block bound)                                         */
    uint32_t sub_max;        /* longest codeword sub-range of one work item with the block bound,
                                >= 64 (default 262144; pipelined engine, graded orders 32768)      */
    uint32_t geo_head;       /* first (newest) sub-range of a level with the block bound; the next
                                ones double up to sub_max (default 8192)                           */
    uint32_t split_bits;     /* a warp whose live candidates differ in more bits screens them as two
                                halves (default 10 for the one-level lexicographic schedule, else 12) */
    uint32_t partial_s;      /* tile-barrier engine: a tile is cut after this many survivors, >= 32
                                (default 512; graded orders 1024)                                  */
    uint32_t grid_ctas;      /* CTAs of the persistent kernel (default one per SM; the pipelined
                                engine uses >= 2: one resolves, the others screen)                 */
    uint32_t plan_warps;     /* pipelined engine: warps a level's work items are planned for
                                (default: screening warps / pipeline_depth)                        */
    uint32_t prep_lead;      /* pipelined engine: a screening CTA prepares tile i (survivors, their
                                check against the words committed since its screen, in-tile
                                conflict lists) once tile i - prep_lead is being resolved; the
                                resolver then checks only the newer words.  0 = default (1; graded
                                orders 2);
                                GC_FLAG_NO_PREP: the resolver does everything                    */
    uint32_t prep_ctas;      /* pipelined engine: CTAs that only prepare tiles (default 2; other
                                screening CTAs also prepare when idle)                           */
    uint32_t burst_chunk;    /* survivors decided per sub-chunk when a tile has more than one resolve
                                chunk of them, or a prepared tile more than two sub-chunks (>= 32,
                                default 512)                                                     */
} gc_options;

#define GC_FLAG_NO_EARLY_EXIT  0x1u  /* screen every candidate against the whole codebook, one phase     */
#define GC_FLAG_SYNC_TILES     0x2u  /* host waits after every tile (debugging)                         */
#define GC_FLAG_FORCE_SEQ_RESOLVE 0x4u /* in-tile resolve by the sequential fallback (testing)           */
#define GC_FLAG_LAUNCHED_TILES 0x10u /* host-launched tile kernels instead of the persistent
                                        device-resident construction kernel (testing / comparison) */
#define GC_FLAG_POPC_ONLY      0x20u /* every check by XOR+POPC (default for d <= 4: half of them
                                        by an ALU bit-clearing test of the same predicate)         */
#define GC_FLAG_NO_WEIGHT_BOUND 0x40u /* graded orders: screen the whole codebook (default: stop at the
                                        first codeword of weight >= wt(candidate) - d + 1, since the
                                        codebook is weight-sorted and |wt(u)-wt(v)| <= dist(u,v))     */
#define GC_FLAG_NO_BLOCK_BOUND 0x80u /* persistent engine: scan every codeword block of a window (default:
                                        skip a block of 32 codewords when the bit-consensus bound
                                        popc((AND_blk & ~OR_batch) | (AND_batch & ~OR_blk)) -- positions
                                        where every codeword of the block differs from every live
                                        candidate of the warp -- is already >= d; exact)            */
#define GC_FLAG_TILE_BARRIERS  0x100u /* the round-1 tile-synchronous persistent kernel (every CTA screens
                                        one tile, grid barrier, CTA 0 resolves while the rest wait)
                                        instead of the pipelined one (testing / comparison)          */
#define GC_FLAG_DEBUG_PHASES   0x200u /* tile-barrier engine: per-phase timing and counters on stderr     */
#define GC_FLAG_NO_SUP_SMEM    0x400u /* do not mirror the super-block summaries in shared memory          */
#define GC_FLAG_NO_PREP        0x800u /* pipelined engine: no preparation of tiles by screening CTAs   */
#define GC_FLAG_SIZE_ON_TRUE   0x1000u /* pipelined engine: size tiles on the survivors left after the
                                        checks against the newest words (default: on the survivors of
                                        the screen against the older codebook, which the resolve gets) */
#define GC_FLAG_NO_PARITY_BOUND 0x2000u /* block bound without the weight-parity refinement (n <= 30:
                                        when a block's codewords and a warp's candidates each have one
                                        weight parity, the bound rounds up to the parity of every
                                        distance)                                                    */
#define GC_FLAG_CROSS          0x4000u /* pipelined engine: two-stage preparation -- stage A (survivors, their
                                        check against the committed words, in-tile conflict lists) once
                                        a tile is screened, stage B one tile ahead of the resolver: the
                                        words committed since, and the conflicts with the previous
                                        tile's prepared list (cross lists), so the resolver checks no
                                        committed word (default off)                                */
#define GC_FLAG_NO_CATCHUP     0x8000u /* pipelined engine: no catch-up screening level (default for graded
                                        orders and d = 4: after its window levels a tile's live
                                        candidates are screened against the words committed since its
                                        descriptor, so fewer survivors reach the preparation)        */
#define GC_FLAG_CATCHUP        0x10000u /* pipelined engine: the catch-up level for every ordering          */
#define GC_FLAG_STAGE_B        0x40000u /* pipelined engine: two-stage preparation without cross lists --
                                        stage A (default 3 tiles ahead) once a tile is screened, stage B
                                        one tile ahead of the resolver flags the survivors hit by the
                                        words committed since stage A                               */
#define GC_FLAG_PIPELINED      0x20000u /* always the pipelined engine (default: d = 3 codes in lexicographic or
                                        Gray order with n <= 25 run on the tile-barrier engine, which is
                                        faster there)                                                */
#define GC_FLAG_KERNEL_TIMING  0x8u  /* bracket every screen launch with CUDA events on the launching
                                        stream; fills gc_stats.screen_ms (benchmarking)               */

/* Counters of one construction (filled when a gc_stats* is passed). */
typedef struct gc_stats {
    uint32_t struct_size;
    uint32_t n_ranks;        /* world size used (1, or emulate_ranks / world)                       */
    double device_ms;        /* device time between the first and the last kernel (CUDA events)       */
    double wall_ms;          /* host wall time of the call                                            */
    uint64_t M;              /* codewords produced                                                    */
    uint64_t tiles;          /* candidate tiles                                                       */
    uint64_t phases;         /* screen phases launched                                                */
    uint64_t checks_exec;    /* candidate-codeword distance evaluations executed by the screen (lane work) */
    uint64_t survivors;      /* candidates that passed the screen (sum over tiles)                    */
    uint64_t conflicts;      /* in-tile survivor pairs at distance < d (sum over tiles)                */
    uint64_t resolve_checks; /* survivor-survivor distance evaluations in the in-tile resolve         */
    double w_def;            /* definitional work sum_j (2^n - 1 - rank_j): every candidate against
                                every codeword accepted before it                       */
    uint64_t launches;       /* kernels this call launched                                            */
    uint64_t screen_launches;/* of which screen kernels (the dominant kernel)                         */
    double screen_ms;        /* summed device time of the screen launches (GC_FLAG_KERNEL_TIMING)     */
    uint64_t bound_tests;    /* block / super-block summary tests of the block bound (lane evaluations;
                                each covers 32 or 1024 codewords against a warp's candidates)        */
    double resolve_wait_ms;  /* pipelined engine: time the resolving CTA waited for screens          */
    double resolve_busy_ms;  /* pipelined engine: time it spent resolving and committing             */
    uint32_t pipeline_depth; /* pipelined engine: tiles in flight (0: another engine ran)             */
    uint32_t reserved;
    uint64_t prep_used;      /* pipelined engine: tiles resolved from a screening CTA's preparation   */
} gc_stats;

/* ------------------------------------------------------------------ generate */

/* The greedy code for (n, d, ordering) on the current CUDA device.
 *   n in [1, 32] on the GPU (GC_EUNSUPPORTED above), d in [1, n].
 *   out_codewords: caller-owned HOST buffer of *out_count elements (may be NULL iff *out_count == 0).
 *   in: *out_count = capacity; out: GC_OK -> *out_count = M and out_codewords[0..M) in acceptance order;
 *   GC_ENOSPC -> *out_count = M (required capacity), buffer contents unspecified.
 * gc_capacity_bound(n, d) elements always suffice. */
int gc_generate(uint32_t n, uint32_t d, gc_ordering ordering,
                uint64_t *out_codewords, uint64_t *out_count);

/* As gc_generate, with schedule options (NULL = defaults) and optional stats (NULL = none). */
int gc_generate_ex(uint32_t n, uint32_t d, gc_ordering ordering, const gc_options *opt,
                   uint64_t *out_codewords, uint64_t *out_count, gc_stats *stats);

/* Device-buffer variant for callers that own device memory and streams (PyTorch):
 *   d_codebook: DEVICE buffer of `capacity` uint32 words (the code, acceptance order);
 *   d_count:    DEVICE uint64 receiving M;  stream: cudaStream_t (NULL = legacy default stream).
 * Work is enqueued on `stream`.  With stats == NULL the call returns once everything is
 * enqueued (results valid when the stream reaches this point; device scratch stays owned
 * by the library and is reused by the next call on this device, which must be ordered
 * after this one -- e.g. the same stream).  With stats != NULL the call synchronises the
 * stream and fills *stats.  If M would exceed capacity, *d_count receives capacity + 1 (a value
 * above capacity: the code is incomplete) and, with stats != NULL, the call returns GC_ENOSPC.
 * capacity >= gc_capacity_bound(n, d) is safe.  d_codebook must be 16-byte aligned (GC_EINVAL). */
int gc_generate_device(uint32_t n, uint32_t d, gc_ordering ordering, const gc_options *opt,
                       uint32_t *d_codebook, uint64_t capacity, uint64_t *d_count,
                       void *stream, gc_stats *stats);

/* ------------------------------------------------ generalised problem */

/* The constructions of PAPER.md Sec. 3-4 beyond the base greedy:
 *   - B-ordering: ordering = GC_B_ORDERING and basis = n linearly
 *     independent vectors b_1..b_n (HOST memory, caller-owned, read during the call);
 *     rank r -> XOR of b_{j+1} over the set bits j of r, i.e. {0, b_1, b_2, b_2+b_1, ...};
 *   - self-orthogonal greedy codes: a candidate must also be orthogonal
 *     to itself (even weight) and to every accepted word (popcount(v & c) even);
 *   - constant-weight codes: only candidates of weight constant_weight.
 * The ordering still defines the scan; filtered candidates are never accepted.  Supported
 * by the persistent engines, single-GPU and partitioned (emulate_ranks > 1, world > 1);
 * GC_EUNSUPPORTED with GC_FLAG_LAUNCHED_TILES / NO_EARLY_EXIT / FORCE_SEQ_RESOLVE.
 * gc_stats.w_def is 0 for filtered problems (its definition counts every rank). */
#define GC_B_ORDERING 4
typedef struct gc_problem {
    uint32_t struct_size;        /* sizeof(gc_problem)                                        */
    uint32_t n, d;               /* 1 <= d <= n <= 32                                         */
    int32_t ordering;            /* gc_ordering value, or GC_B_ORDERING                        */
    const uint64_t *basis;       /* GC_B_ORDERING: n vectors < 2^n, independent over F_2       */
    int32_t constant_weight;     /* -1: no constraint, else 0..n                               */
    uint32_t self_orthogonal;    /* 0 or 1                                                     */
} gc_problem;

/* As gc_generate_ex / gc_generate_device for a gc_problem.  GC_EINVAL for a dependent or
 * out-of-range basis, a bad weight or flag. */
int gc_construct(const gc_problem *problem, const gc_options *opt, uint64_t *out_codewords,
                 uint64_t *out_count, gc_stats *stats);
int gc_construct_device(const gc_problem *problem, const gc_options *opt, uint32_t *d_codebook,
                        uint64_t capacity, uint64_t *d_count, void *stream, gc_stats *stats);

/* ------------------------------------------------ code analysis */

/* Properties of a code (weight, distance, minimum distance, linear [n,k]
 * codes; :123 orthogonality), computed on the GPU:
 *   weight_hist[w]   number of words of weight w
 *   gf2_rank         dimension of the span; is_linear = (M == 2^gf2_rank) (distinct words)
 *   min_distance     GC_ANALYZE_PAIRWISE: min over all pairs of popcount(u ^ v) (M(M-1)/2
 *                    XOR+POPC checks, the screen's kernel shape); otherwise, for a linear
 *                    code, the minimum nonzero weight; 0 if undetermined or M < 2
 *   self_orthogonal  1 every pair (and word) has even AND-parity, 0 not, 2 undetermined
 *                    (nonlinear code without GC_ANALYZE_PAIRWISE | GC_ANALYZE_ORTHOGONALITY) */
typedef struct gc_analysis {
    uint32_t struct_size;
    uint32_t min_distance;
    uint64_t M;
    uint64_t weight_hist[33];
    uint32_t gf2_rank;
    uint32_t is_linear;
    uint32_t self_orthogonal;
    uint32_t reserved;
    uint64_t pairs_checked;
} gc_analysis;
#define GC_ANALYZE_PAIRWISE      0x1u
#define GC_ANALYZE_ORTHOGONALITY 0x2u   /* with PAIRWISE: AND-parity of every pair too */

/* d_words: DEVICE array of M 32-bit words; synchronises `stream`.  GC_EINVAL for NULL
 * pointers (d_words may be NULL iff M == 0) or unknown flags. */
int gc_analyze_device(const uint32_t *d_words, uint64_t M, uint32_t flags, void *stream, gc_analysis *out);
/* words: HOST array of M words < 2^32 (copied to the device). */
int gc_analyze(const uint64_t *words, uint64_t M, uint32_t flags, gc_analysis *out);

/* Upper bound on M: the sphere-packing (Hamming) bound for (n, d); for even d the
 * bound of (n-1, d-1) (a code of even distance d and length n punctures to one of
 * length n-1 and distance d-1).  Clamped to 2^n.  Returns 0 if the arguments are invalid.
 * (28,3) -> 9,256,395; (26,4) -> 1,290,555; (24,8) -> 4,096. */
uint64_t gc_capacity_bound(uint32_t n, uint32_t d);

/* ---------------------------------------------------------- orderings (host) */

/* rank -> vector in `ordering`.  n in [1, 63]; GC_ERANGE if rank >= 2^n. */
int gc_rank_to_vector(gc_ordering ordering, uint32_t n, uint64_t rank, uint64_t *out_vec);

/* vector -> rank (inverse of gc_rank_to_vector).  GC_ERANGE if vec >= 2^n. */
int gc_vector_to_rank(gc_ordering ordering, uint32_t n, uint64_t vec, uint64_t *out_rank);

/* out[i] = gc_rank_to_vector(first + i), i < count, computed on the HOST. */
int gc_ranks_to_vectors(gc_ordering ordering, uint32_t n, uint64_t first, uint64_t count,
                        uint64_t *out);

/* The same map evaluated by the DEVICE candidate generator the screen uses:
 * d_out (DEVICE, count uint32) receives the vectors of ranks first .. first+count-1.
 * n in [1, 32].  Synchronises `stream` (NULL = legacy default stream). */
int gc_ranks_to_vectors_device(gc_ordering ordering, uint32_t n, uint64_t first, uint64_t count,
                               uint32_t *d_out, void *stream);

/* --------------------------------------------------------------- multi-GPU */

/* Size in bytes of the NCCL unique id (128).  0 if NCCL cannot be loaded. */
size_t gc_nccl_id_bytes(void);

/* Fill id[0..gc_nccl_id_bytes()) with a fresh NCCL unique id (call on one rank, broadcast
 * the bytes to the others, e.g. over a torch.distributed process group).  GC_ENCCL if NCCL
 * (libnccl.so.2, loaded at run time) is unavailable. */
int gc_nccl_unique_id(uint8_t *id, size_t id_bytes);

/* An NCCL communicator over `world` ranks (one process per GPU), created once and reused
 * by every construction.  nccl_id: the bytes from gc_nccl_unique_id on one rank, shared
 * with the others (e.g. broadcast over a torch.distributed process group); the current
 * CUDA device must be this rank's GPU.  world must be a power of two in [1, 64];
 * world == 1 needs no id (nccl_id may be NULL) and uses no NCCL.  GC_ENCCL on failure. */
typedef struct gc_comm gc_comm;
int gc_comm_create(const uint8_t *nccl_id, size_t id_bytes, int rank, int world, gc_comm **out_comm);
int gc_comm_destroy(gc_comm *comm);   /* NULL is a no-op */

/* One rank's part of a multi-GPU construction (comm == NULL: a single-GPU run).
 * Every rank screens 1/world of each tile's candidates against its full (replicated)
 * codebook; the per-tile survivor bit-masks are all-gathered with NCCL over NVLink once
 * per tile; every rank then resolves the tile identically, so all ranks end with the
 * same code in d_codebook.  Buffers/stream/stats as gc_generate_device; the call
 * synchronises `stream`.  Every rank must call with identical (n, d, ordering, opt). */
int gc_generate_rank(uint32_t n, uint32_t d, gc_ordering ordering, const gc_options *opt,
                     gc_comm *comm, uint32_t *d_codebook, uint64_t capacity, uint64_t *d_count,
                     void *stream, gc_stats *stats);

/* The candidate partition every rank uses inside a tile of K candidates (host-side, pure):
 * the tile is padded to Kpad = ceil(K / (32 world)) * 32 world candidates (padding is
 * never accepted) and rank r screens [r Kpad/world, (r+1) Kpad/world), a whole number of
 * 32-bit mask words, so the all-gather of the mask words rebuilds the tile's mask in rank
 * order.  GC_EINVAL for a bad world/rank or NULL outputs. */
/* Multi-GPU pipelined engine (one process per GPU of one node, 2..8 ranks): every rank runs the
 * persistent pipelined kernel on its own replica of the codebook and screens its partition of
 * every tile (gc_tile_partition); the partition's survivor-mask words are stored straight into
 * every peer's memory by the kernel (NVLink / NVSwitch peer stores, CUDA IPC mappings) with a
 * per-tile flag, and every rank resolves the whole tile -- no host round trip and no collective
 * in the data path.  Setup, once per communicator: every rank calls gc_peer_handles (the IPC
 * handles of its exchange buffers on the current device, gc_peer_handle_bytes() bytes), the
 * blobs are all-gathered in rank order (e.g. torch.distributed), and gc_comm_attach_peers opens
 * them.  Without attached peers gc_generate_rank uses the tile-barrier engine with one NCCL
 * all-gather per tile. */
size_t gc_peer_handle_bytes(void);
int gc_peer_handles(uint8_t *out, size_t out_bytes);
int gc_comm_attach_peers(gc_comm *comm, const uint8_t *all_handles, size_t bytes_per_rank);

int gc_tile_partition(uint32_t K, int world, int rank, uint32_t *part_lo, uint32_t *part_len,
                      uint32_t *Kpad);

/* ------------------------------------------------------------------- misc */
const char *gc_strerror(int status);
const char *gc_last_error(void);   /* thread-local detail of the last failure ("" if none) */
int gc_abi_version(void);          /* GC_ABI_VERSION */

#ifdef __cplusplus
}
#endif
#endif /* GC_H_ */
