// gc_abi.cpp -- the extern "C" boundary of libgc.so (include/gc.h): argument
// validation (always before any CUDA call), the host-side orderings, the capacity
// bound, error strings, and the run-time NCCL loader.  The construction itself is
// engine_run() in gc_engine.cu.
#include <dlfcn.h>
#include <string.h>

#include <chrono>
#include <mutex>
#include <string>

#include "gc_internal.h"

namespace gc {

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }

static bool is_pow2(uint32_t x) { return x && !(x & (x - 1)); }

int resolve_options(const gc_options *opt, Options *out) {
    Options o;
    if (opt) {
        if (opt->struct_size != 0 && opt->struct_size < sizeof(gc_options)) {
            set_error("gc_options.struct_size smaller than this library's gc_options");
            return GC_EINVAL;
        }
        if (opt->tile_min) o.tile_min = opt->tile_min;
        if (opt->tile_max) o.tile_max = opt->tile_max;
        if (opt->window0) { o.window0 = opt->window0; o.window0_set = true; }
        if (opt->emulate_ranks) o.emulate_ranks = opt->emulate_ranks;
        o.flags = opt->flags;
        if (opt->window_growth) o.growth = opt->window_growth;
        o.pipeline_depth = opt->pipeline_depth;
        o.target_accepted = opt->target_accepted;
        o.items_per_warp = opt->items_per_warp;
        o.sub_max = opt->sub_max;
        o.geo_head = opt->geo_head;
        o.split_bits = opt->split_bits;
        o.partial_s = opt->partial_s;
        o.grid_ctas = opt->grid_ctas;
        o.plan_warps = opt->plan_warps;
        o.prep_lead = opt->prep_lead;
        o.prep_ctas = opt->prep_ctas;
        o.burst_chunk = opt->burst_chunk;
    }
    if (o.pipeline_depth > 16 || (o.sub_max && o.sub_max < 64) || (o.partial_s && o.partial_s < 32) ||
        o.split_bits > 32 || o.prep_lead > 15 || o.prep_ctas > 64 || (o.burst_chunk && o.burst_chunk < 32)) {
        set_error("pipeline_depth must be <= 16, sub_max >= 64, partial_s >= 32, split_bits <= 32, prep_lead <= 15, "
                  "prep_ctas <= 64, burst_chunk >= 32");
        return GC_EINVAL;
    }
    if (o.growth > 12) {          // 0 = engine default
        set_error("window_growth must be in [1, 12]");
        return GC_EINVAL;
    }
    if (!is_pow2(o.tile_min) || o.tile_min < 32 || (o.tile_max && (!is_pow2(o.tile_max) || o.tile_max > (1u << 20) ||
        o.tile_min > o.tile_max))) {
        set_error("tile_min/tile_max must be powers of two with 32 <= tile_min <= tile_max <= 2^20");
        return GC_EINVAL;
    }
    if (!is_pow2(o.window0) || o.window0 > (1u << 24)) {
        set_error("window0 must be a power of two <= 2^24");
        return GC_EINVAL;
    }
    if (o.emulate_ranks < 1 || o.emulate_ranks > 64 || !is_pow2(o.emulate_ranks)) {
        set_error("emulate_ranks must be a power of two in [1, 64]");
        return GC_EINVAL;
    }
    if (o.flags & ~(uint32_t)(GC_FLAG_NO_EARLY_EXIT | GC_FLAG_SYNC_TILES | GC_FLAG_FORCE_SEQ_RESOLVE |
                              GC_FLAG_KERNEL_TIMING | GC_FLAG_LAUNCHED_TILES | GC_FLAG_POPC_ONLY |
                              GC_FLAG_NO_WEIGHT_BOUND | GC_FLAG_NO_BLOCK_BOUND | GC_FLAG_TILE_BARRIERS |
                              GC_FLAG_DEBUG_PHASES | GC_FLAG_NO_SUP_SMEM | GC_FLAG_NO_PREP |
                              GC_FLAG_SIZE_ON_TRUE | GC_FLAG_NO_PARITY_BOUND | GC_FLAG_CROSS | GC_FLAG_NO_CATCHUP |
                              GC_FLAG_CATCHUP | GC_FLAG_PIPELINED | GC_FLAG_STAGE_B)) {
        set_error("unknown bits in gc_options.flags");
        return GC_EINVAL;
    }
    *out = o;
    return GC_OK;
}

// ------------------------------------------------------ host orderings (n <= 63)
// Same maps as gc_order.cuh (which is limited to the device's 32-bit words), with
// 64-bit binomials: C(63,31) < 2^63.
namespace {
struct HostTables {
    uint64_t C[65][65];
    HostTables() {
        for (int p = 0; p <= 64; ++p)
            for (int k = 0; k <= 64; ++k)
                C[p][k] = (k == 0) ? 1 : (p == 0 ? 0 : C[p - 1][k - 1] + C[p - 1][k]);
    }
};
const HostTables &host_tables() {
    static HostTables t;
    return t;
}
int weight_class(const uint64_t (*C)[65], uint32_t n, uint64_t r, uint64_t *q) {
    int w = 0;
    while (r >= C[n][w]) { r -= C[n][w]; ++w; }
    *q = r;
    return w;
}
uint64_t unrank_colex64(const uint64_t (*C)[65], uint32_t n, int w, uint64_t q) {
    uint64_t v = 0;
    int p = (int)n - 1;
    for (int k = w; k >= 1; --k) {
        while (C[p][k] > q) --p;
        v |= 1ull << p;
        q -= C[p][k];
        --p;
    }
    return v;
}
uint64_t rank_colex64(const uint64_t (*C)[65], uint64_t v) {
    uint64_t q = 0;
    int k = 0;
    for (int p = 0; p < 64; ++p)
        if (v >> p & 1ull) { ++k; q += C[p][k]; }
    return q;
}
int check_order_args(int ordering, uint32_t n) {
    if (ordering < GC_LEX || ordering > GC_GRADED_REVLEX) { set_error("unknown ordering"); return GC_EINVAL; }
    if (n < 1 || n > 63) { set_error("n must be in [1, 63] for the host orderings"); return GC_EINVAL; }
    return GC_OK;
}
uint64_t host_rank_to_vector(int ord, uint32_t n, uint64_t r) {
    if (ord == GC_LEX) return r;
    if (ord == GC_GRAY) return r ^ (r >> 1);
    const auto &T = host_tables();
    uint64_t q;
    int w = weight_class(T.C, n, r, &q);
    if (ord == GC_GRADED_REVLEX) q = T.C[n][w] - 1 - q;
    return unrank_colex64(T.C, n, w, q);
}
}  // namespace

// ------------------------------------------------------------- NCCL loader
static NcclApi g_nccl;
static std::once_flag g_nccl_once;

const NcclApi *nccl_api() {
    std::call_once(g_nccl_once, [] {
        // Prefer the copy torch already loaded (same soname), else the system one.
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
        g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
        g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
        g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
        g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllGather && g_nccl.CommDestroy;
    });
    return g_nccl.ok ? &g_nccl : nullptr;
}

int nccl_comm_init(void **comm, int world, int rank, const uint8_t *id, size_t id_bytes) {
    const NcclApi *api = nccl_api();
    if (!api) { set_error("libnccl.so.2 could not be loaded"); return GC_ENCCL; }
    if (id_bytes != sizeof(NcclUid)) { set_error("NCCL id must be 128 bytes"); return GC_EINVAL; }
    NcclUid uid;
    memcpy(uid.internal, id, sizeof uid.internal);
    int rc = api->CommInitRank(comm, world, uid, rank);
    if (rc != 0) {
        set_error(std::string("ncclCommInitRank: ") + (api->GetErrorString ? api->GetErrorString(rc) : "?"));
        return GC_ENCCL;
    }
    return GC_OK;
}

int nccl_allgather_u32(const uint32_t *send, uint32_t *recv, size_t count, void *comm, void *stream) {
    const NcclApi *api = nccl_api();
    int rc = api->AllGather(send, recv, count, kNcclUint32, comm, stream);
    if (rc != 0) {
        set_error(std::string("ncclAllGather: ") + (api->GetErrorString ? api->GetErrorString(rc) : "?"));
        return GC_ENCCL;
    }
    return GC_OK;
}

void nccl_comm_destroy(void *comm) {
    if (comm && nccl_api()) nccl_api()->CommDestroy(comm);
}

// validate a gc_problem into RunArgs (before any CUDA call)
int gc_problem_to_args(const gc_problem *p, RunArgs *a) {
    if (!p) { set_error("problem is NULL"); return GC_EINVAL; }
    if (p->struct_size != 0 && p->struct_size < sizeof(gc_problem)) { set_error("gc_problem.struct_size too small"); return GC_EINVAL; }
    const int ord = p->ordering;
    if (ord < GC_LEX || ord > GC_B_ORDERING) { set_error("unknown ordering"); return GC_EINVAL; }
    if (p->n == 0) { set_error("n must be >= 1"); return GC_EINVAL; }
    if (p->d == 0 || p->d > p->n) { set_error("d must be in [1, n]"); return GC_EINVAL; }
    if (p->constant_weight < -1 || p->constant_weight > (int)p->n) { set_error("constant_weight must be -1 or in [0, n]"); return GC_EINVAL; }
    if (p->n > 63) { set_error("n must be <= 63"); return GC_EUNSUPPORTED; }
    if (p->n > 32 && (p->constant_weight < 0 || p->self_orthogonal || ord == GC_B_ORDERING || ord == GC_GRAY)) {
        set_error("n > 32 is supported for constant-weight problems in lex / graded orders only (64-bit words)");
        return GC_EUNSUPPORTED;
    }
    if (p->self_orthogonal > 1) { set_error("self_orthogonal must be 0 or 1"); return GC_EINVAL; }
    a->n = p->n; a->d = p->d;
    a->ordering = ord == GC_B_ORDERING ? GC_LEX : ord;
    a->constant_weight = p->constant_weight;
    a->self_orthogonal = p->self_orthogonal != 0;
    if (ord == GC_B_ORDERING) {
        if (!p->basis) { set_error("GC_B_ORDERING needs a basis"); return GC_EINVAL; }
        uint64_t red[64] = {0};
        for (uint32_t k = 0; k < p->n; ++k) {
            uint64_t x = p->basis[k];
            if (x >> p->n) { set_error("basis vector >= 2^n"); return GC_EINVAL; }
            for (int b = 63; b >= 0 && x; --b) {
                if (!(x >> b & 1ull)) continue;
                if (!red[b]) { red[b] = x; x = 0; break; }
                x ^= red[b];
            }

            a->basis[k] = (uint32_t)p->basis[k];
        }
        int rank = 0;
        for (int b = 0; b < 64; ++b) rank += red[b] != 0;
        if (rank != (int)p->n) { set_error("basis is not linearly independent over F_2"); return GC_EINVAL; }
        a->use_basis = true;
    }
    return GC_OK;
}

}  // namespace gc

using namespace gc;

// ======================================================================= ABI
extern "C" {

const char *gc_strerror(int s) {
    switch (s) {
        case GC_OK: return "ok";
        case GC_EINVAL: return "invalid argument";
        case GC_ERANGE: return "rank or vector out of range";
        case GC_ENOSPC: return "output capacity too small";
        case GC_EUNSUPPORTED: return "unsupported parameters (n > 32 on the GPU path)";
        case GC_ECUDA: return "CUDA error";
        case GC_ENOMEM: return "out of memory";
        case GC_ENCCL: return "NCCL error";
        case GC_EINTERNAL: return "internal error";
        default: return "unknown status";
    }
}

const char *gc_last_error(void) { return g_last_error.c_str(); }
int gc_abi_version(void) { return GC_ABI_VERSION; }

uint64_t gc_capacity_bound(uint32_t n, uint32_t d) {
    if (n < 1 || n > 63 || d < 1 || d > n) return 0;
    uint32_t nn = n, dd = d;
    if (dd % 2 == 0) { nn -= 1; dd -= 1; }     // even d: puncture to (n-1, d-1)
    uint32_t t = (dd - 1) / 2;
    const auto &T = host_tables();
    // sphere volume sum_{i<=t} C(nn, i); nn <= 62 so no overflow for the ranges used
    unsigned __int128 vol = 0;
    for (uint32_t i = 0; i <= t; ++i) vol += T.C[nn][i];
    unsigned __int128 space = (unsigned __int128)1 << nn;
    unsigned __int128 b = space / vol;
    if (b < 1) b = 1;
    unsigned __int128 lim = (unsigned __int128)1 << n;
    if (b > lim) b = lim;
    return (uint64_t)b;
}

int gc_rank_to_vector(gc_ordering ordering, uint32_t n, uint64_t rank, uint64_t *out_vec) {
    clear_error();
    int rc = check_order_args(ordering, n);
    if (rc) return rc;
    if (!out_vec) { set_error("out_vec is NULL"); return GC_EINVAL; }
    if (rank >> n) { set_error("rank >= 2^n"); return GC_ERANGE; }
    *out_vec = host_rank_to_vector(ordering, n, rank);
    return GC_OK;
}

int gc_vector_to_rank(gc_ordering ordering, uint32_t n, uint64_t vec, uint64_t *out_rank) {
    clear_error();
    int rc = check_order_args(ordering, n);
    if (rc) return rc;
    if (!out_rank) { set_error("out_rank is NULL"); return GC_EINVAL; }
    if (vec >> n) { set_error("vec >= 2^n"); return GC_ERANGE; }
    uint64_t r;
    if (ordering == GC_LEX) {
        r = vec;
    } else if (ordering == GC_GRAY) {
        r = vec;                       // inverse of r ^ (r >> 1): prefix XOR
        for (int s = 1; s < 64; s <<= 1) r ^= r >> s;
    } else {
        const auto &T = host_tables();
        int w = __builtin_popcountll(vec);
        uint64_t q = rank_colex64(T.C, vec);
        if (ordering == GC_GRADED_REVLEX) q = T.C[n][w] - 1 - q;
        uint64_t off = 0;
        for (int u = 0; u < w; ++u) off += T.C[n][u];
        r = off + q;
    }
    *out_rank = r;
    return GC_OK;
}

int gc_ranks_to_vectors(gc_ordering ordering, uint32_t n, uint64_t first, uint64_t count, uint64_t *out) {
    clear_error();
    int rc = check_order_args(ordering, n);
    if (rc) return rc;
    if (!out && count) { set_error("out is NULL"); return GC_EINVAL; }
    if (count && ((first >> n) || ((first + count - 1) >> n) || first + count < first)) {
        set_error("ranks out of [0, 2^n)");
        return GC_ERANGE;
    }
    for (uint64_t i = 0; i < count; ++i) out[i] = host_rank_to_vector(ordering, n, first + i);
    return GC_OK;
}

static int validate_nd(uint32_t n, uint32_t d, int ordering) {
    if (ordering < GC_LEX || ordering > GC_GRADED_REVLEX) { set_error("unknown ordering"); return GC_EINVAL; }
    if (n == 0) { set_error("n must be >= 1"); return GC_EINVAL; }
    if (d == 0 || d > n) { set_error("d must be in [1, n]"); return GC_EINVAL; }
    if (n > 32) { set_error("the GPU path supports n <= 32"); return GC_EUNSUPPORTED; }
    return GC_OK;
}

int gc_ranks_to_vectors_device(gc_ordering ordering, uint32_t n, uint64_t first, uint64_t count,
                               uint32_t *d_out, void *stream) {
    clear_error();
    if (ordering < GC_LEX || ordering > GC_GRADED_REVLEX) { set_error("unknown ordering"); return GC_EINVAL; }
    if (n < 1) { set_error("n must be >= 1"); return GC_EINVAL; }
    if (n > 32) { set_error("the device generator supports n <= 32"); return GC_EUNSUPPORTED; }
    if (!d_out && count) { set_error("d_out is NULL"); return GC_EINVAL; }
    if (count && ((first >> n) || ((first + count - 1) >> n) || first + count < first)) {
        set_error("ranks out of [0, 2^n)");
        return GC_ERANGE;
    }
    if (!count) return GC_OK;
    return engine_ranks_to_vectors_device(ordering, n, first, count, d_out, stream);
}

int gc_generate_device(uint32_t n, uint32_t d, gc_ordering ordering, const gc_options *opt,
                       uint32_t *d_codebook, uint64_t capacity, uint64_t *d_count, void *stream,
                       gc_stats *stats) {
    clear_error();
    int rc = validate_nd(n, d, ordering);
    if (rc) return rc;
    RunArgs a;
    rc = resolve_options(opt, &a.opt);
    if (rc) return rc;
    if (!d_codebook || !d_count || capacity == 0) { set_error("d_codebook/d_count NULL or capacity 0"); return GC_EINVAL; }
    if ((uintptr_t)d_codebook & 15u) { set_error("d_codebook must be 16-byte aligned"); return GC_EINVAL; }
    if (stats && stats->struct_size != 0 && stats->struct_size < sizeof(gc_stats)) {
        set_error("gc_stats.struct_size too small");
        return GC_EINVAL;
    }
    a.n = n; a.d = d; a.ordering = ordering;
    a.d_codebook = d_codebook; a.capacity = capacity; a.d_count = d_count;
    a.stream = stream; a.stats = stats;
    return engine_run(a);
}

int gc_generate_ex(uint32_t n, uint32_t d, gc_ordering ordering, const gc_options *opt,
                   uint64_t *out_codewords, uint64_t *out_count, gc_stats *stats);

int gc_construct_device(const gc_problem *problem, const gc_options *opt, uint32_t *d_codebook, uint64_t capacity,
                        uint64_t *d_count, void *stream, gc_stats *stats) {
    clear_error();
    RunArgs a;
    int rc = gc_problem_to_args(problem, &a);
    if (rc) return rc;
    if (a.wide()) { set_error("n > 32: 64-bit words, host buffers only (gc_construct)"); return GC_EUNSUPPORTED; }
    rc = resolve_options(opt, &a.opt);
    if (rc) return rc;
    if (!d_codebook || !d_count || capacity == 0) { set_error("d_codebook/d_count NULL or capacity 0"); return GC_EINVAL; }
    if ((uintptr_t)d_codebook & 15u) { set_error("d_codebook must be 16-byte aligned"); return GC_EINVAL; }
    if (stats && stats->struct_size != 0 && stats->struct_size < sizeof(gc_stats)) {
        set_error("gc_stats.struct_size too small");
        return GC_EINVAL;
    }
    a.d_codebook = d_codebook; a.capacity = capacity; a.d_count = d_count;
    a.stream = stream; a.stats = stats;
    return engine_run(a);
}

int gc_generate(uint32_t n, uint32_t d, gc_ordering ordering, uint64_t *out_codewords, uint64_t *out_count) {
    return gc_generate_ex(n, d, ordering, nullptr, out_codewords, out_count, nullptr);
}

size_t gc_nccl_id_bytes(void) { return nccl_api() ? sizeof(NcclUid) : 0; }

int gc_nccl_unique_id(uint8_t *id, size_t id_bytes) {
    clear_error();
    if (!id || id_bytes < sizeof(NcclUid)) { set_error("id buffer NULL or smaller than 128 bytes"); return GC_EINVAL; }
    const NcclApi *api = nccl_api();
    if (!api) { set_error("libnccl.so.2 could not be loaded"); return GC_ENCCL; }
    NcclUid uid;
    int rc = api->GetUniqueId(&uid);
    if (rc != 0) { set_error("ncclGetUniqueId failed"); return GC_ENCCL; }
    memcpy(id, uid.internal, sizeof uid.internal);
    return GC_OK;
}

int gc_tile_partition(uint32_t K, int world, int rank, uint32_t *part_lo, uint32_t *part_len, uint32_t *Kpad) {
    clear_error();
    if (!part_lo || !part_len || !Kpad) { set_error("NULL output"); return GC_EINVAL; }
    if (world < 1 || world > 64 || (world & (world - 1)) || rank < 0 || rank >= world) {
        set_error("world must be a power of two in [1, 64] and 0 <= rank < world");
        return GC_EINVAL;
    }
    const uint32_t q = 32u * (uint32_t)world;
    const uint32_t kp = (K + q - 1) / q * q;
    *Kpad = kp;
    *part_len = kp / (uint32_t)world;
    *part_lo = (uint32_t)rank * (kp / (uint32_t)world);
    return GC_OK;
}

struct gc_comm {
    int rank = 0, world = 1;
    void *nccl = nullptr;
    PeerTable peers;          // the peers' exchange buffers (gc_comm_attach_peers)
};

int gc_comm_create(const uint8_t *nccl_id, size_t id_bytes, int rank, int world, gc_comm **out_comm) {
    clear_error();
    if (!out_comm) { set_error("out_comm is NULL"); return GC_EINVAL; }
    if (world < 1 || world > 64 || (world & (world - 1)) || rank < 0 || rank >= world) {
        set_error("world must be a power of two in [1, 64] and 0 <= rank < world");
        return GC_EINVAL;
    }
    if (world > 1 && (!nccl_id || id_bytes != sizeof(NcclUid))) { set_error("nccl_id must be 128 bytes"); return GC_EINVAL; }
    gc_comm *c = new gc_comm;
    c->rank = rank;
    c->world = world;
    if (world > 1) {
        int rc = nccl_comm_init(&c->nccl, world, rank, nccl_id, id_bytes);
        if (rc) { delete c; return rc; }
    }
    *out_comm = c;
    return GC_OK;
}

size_t gc_peer_handle_bytes(void) { return kPeerHandleBytes; }

int gc_peer_handles(uint8_t *out, size_t out_bytes) {
    clear_error();
    if (!out || out_bytes < kPeerHandleBytes) { set_error("out must hold gc_peer_handle_bytes() bytes"); return GC_EINVAL; }
    return pipeline_peer_handles(out);
}

int gc_comm_attach_peers(gc_comm *comm, const uint8_t *all, size_t bytes_per_rank) {
    clear_error();
    if (!comm || !all) { set_error("comm / handles NULL"); return GC_EINVAL; }
    if (bytes_per_rank != kPeerHandleBytes) { set_error("bytes_per_rank must be gc_peer_handle_bytes()"); return GC_EINVAL; }
    if (comm->world < 2 || comm->world > 8) { set_error("peers need 2..8 ranks (one node)"); return GC_EUNSUPPORTED; }
    return pipeline_open_peers(&comm->peers, all, comm->world, comm->rank);
}

int gc_comm_destroy(gc_comm *comm) {
    if (!comm) return GC_OK;
    pipeline_close_peers(&comm->peers);
    nccl_comm_destroy(comm->nccl);
    delete comm;
    return GC_OK;
}

int gc_generate_rank(uint32_t n, uint32_t d, gc_ordering ordering, const gc_options *opt, gc_comm *comm,
                     uint32_t *d_codebook, uint64_t capacity, uint64_t *d_count, void *stream, gc_stats *stats) {
    clear_error();
    int rc = validate_nd(n, d, ordering);
    if (rc) return rc;
    RunArgs a;
    rc = resolve_options(opt, &a.opt);
    if (rc) return rc;
    if (comm && comm->world > 1 && a.opt.emulate_ranks != 1) { set_error("emulate_ranks needs a single rank"); return GC_EINVAL; }
    if (!d_codebook || !d_count || capacity == 0) { set_error("d_codebook/d_count NULL or capacity 0"); return GC_EINVAL; }
    if ((uintptr_t)d_codebook & 15u) { set_error("d_codebook must be 16-byte aligned"); return GC_EINVAL; }
    if (stats && stats->struct_size != 0 && stats->struct_size < sizeof(gc_stats)) {
        set_error("gc_stats.struct_size too small");
        return GC_EINVAL;
    }
    a.n = n; a.d = d; a.ordering = ordering;
    a.d_codebook = d_codebook; a.capacity = capacity; a.d_count = d_count;
    a.stream = stream;
    if (comm) {
        a.rank = comm->rank; a.world = comm->world; a.nccl_comm = comm->nccl;
        if (comm->peers.ready) a.peers = &comm->peers;
    }
    gc_stats local{};
    a.stats = stats ? stats : &local;   // the multi-process call always synchronises
    return engine_run(a);
}

}  // extern "C"
