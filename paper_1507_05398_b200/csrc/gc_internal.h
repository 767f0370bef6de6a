// gc_internal.h -- shared declarations between gc_abi.cpp (validation, host orderings,
// NCCL loader) and gc_engine.cu (device kernels and the tile scheduler).
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <string>

#include "../../include/gc.h"

namespace gc {

// thread-local last-error message (gc_last_error)
void set_error(const std::string &msg);
void clear_error();

// resolved schedule options (defaults applied, validated)
struct Options {
    uint32_t tile_min = 256;
    uint32_t tile_max = 0;          // 0 = engine default (persistent 4096, launched 65536)
    uint32_t window0 = 4096;
    bool window0_set = false;       // window0 given by the caller (else engine default)
    uint32_t emulate_ranks = 1;
    uint32_t flags = 0;
    uint32_t growth = 0;            // log2 window growth per level, 0 = engine default (launched
                                    // engine 2; persistent engines: see p_fill_args)
    // persistent engines (0 = default; gc.h gc_options)
    uint32_t pipeline_depth = 0, target_accepted = 0, items_per_warp = 0, sub_max = 0, geo_head = 0,
             split_bits = 0, partial_s = 0, grid_ctas = 0, plan_warps = 0, prep_lead = 0,
             prep_ctas = 0, burst_chunk = 0;
    bool geo_head_set = false;
};
int resolve_options(const gc_options *opt, Options *out);   // GC_OK / GC_EINVAL

// ---- NCCL, loaded with dlopen at first use (no link-time dependency) ----
struct NcclUid { char internal[128]; };   // layout of ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128)
constexpr int kNcclUint32 = 3;             // ncclDataType_t ncclUint32
struct NcclApi {
    bool ok = false;
    size_t id_bytes = 128;
    int (*GetUniqueId)(NcclUid *uid) = nullptr;
    int (*CommInitRank)(void **comm, int nranks, NcclUid id, int rank) = nullptr;
    int (*AllGather)(const void *send, void *recv, size_t count, int dtype, void *comm, void *stream) = nullptr;
    int (*CommDestroy)(void *comm) = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
};
const NcclApi *nccl_api();   // nullptr if libnccl.so.2 cannot be loaded
int nccl_comm_init(void **comm, int world, int rank, const uint8_t *id, size_t id_bytes);  // GC_OK/GC_ENCCL
int nccl_allgather_u32(const uint32_t *send, uint32_t *recv, size_t count_per_rank, void *comm, void *stream);
void nccl_comm_destroy(void *comm);

// ---- multi-GPU pipelined engine: the peers' tile-exchange buffers (CUDA IPC, gc_comm_attach_peers) ----
struct PeerTable {
    bool ready = false;
    int world = 1, rank = 0;
    uint32_t *qdead[8] = {nullptr};              // rank r's dead-mask ring (opened IPC mapping; own: null)
    unsigned long long *qflags[8] = {nullptr};   // rank r's screen flags
};
constexpr size_t kPeerHandleBytes = 128;         // two cudaIpcMemHandle_t (qdead ring, flags)
int pipeline_peer_handles(uint8_t *out);         // this process's handles (current device), kPeerHandleBytes
int pipeline_open_peers(PeerTable *t, const uint8_t *all, int world, int rank);
void pipeline_close_peers(PeerTable *t);

// ---- engine (gc_engine.cu) ----
struct RunArgs {
    uint32_t n, d;
    int ordering;
    Options opt;
    int rank = 0, world = 1;
    void *nccl_comm = nullptr;      // world > 1
    const PeerTable *peers = nullptr;  // world > 1: attached peers (pipelined engine over NVLink)
    uint32_t *d_codebook = nullptr; // device, capacity words
    uint64_t capacity = 0;
    uint64_t *d_count = nullptr;    // device
    void *stream = nullptr;
    gc_stats *stats = nullptr;      // non-null -> synchronise and fill
    // SURVEY 8(f) extensions (persistent engine only)
    bool use_basis = false;
    uint32_t basis[32] = {0};
    bool self_orthogonal = false;
    int constant_weight = -1;
    bool extended() const { return use_basis || self_orthogonal || constant_weight >= 0; }
    bool wide() const { return n > 32; }   // 64-bit words: constant-weight problems only (gc_cw64.cu)
};
int engine_run(const RunArgs &a);
int gc_problem_to_args(const gc_problem *p, RunArgs *a);   // gc_abi.cpp (validation, no CUDA)
int analyze_device(const uint32_t *d_words, uint64_t M, int pairwise, int orth, void *stream,
                   gc_analysis *out);                        // gc_analysis.cu
bool pipeline_supported(const RunArgs &a);     // gc_pipeline.cu (default single-GPU engine)
int pipeline_run(const RunArgs &a);
bool persistent_supported(const RunArgs &a);   // gc_persistent.cu
int persistent_run(const RunArgs &a);
bool persistent_partitioned_supported(const RunArgs &a);
int persistent_run_partitioned(const RunArgs &a);
bool cw64_supported(const RunArgs &a);        // gc_cw64.cu (constant weight, n <= 63, host buffers)
int cw64_run(const RunArgs &a, uint64_t *out_codewords, uint64_t *out_count, gc_stats *stats);
int engine_ranks_to_vectors_device(int ordering, uint32_t n, uint64_t first, uint64_t count,
                                   uint32_t *d_out, void *stream);

}  // namespace gc
