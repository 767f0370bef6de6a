// gc_analysis.cu -- SURVEY 8(f) row 3: GPU analysis of a code (the step after the path):
// minimum distance (all pairs, XOR + POPC -- the screen's kernel shape), weight
// distribution, GF(2) rank / linearity, self-orthogonality.  PAPER.md:56 defines weight,
// distance, minimum distance and linear codes; :123 orthogonality.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "gc_internal.h"

namespace gc {

#define ACK(call)                                                                             \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            set_error(std::string(#call) + ": " + cudaGetErrorString(e_));                    \
            return e_ == cudaErrorMemoryAllocation ? GC_ENOMEM : GC_ECUDA;                   \
        }                                                                                     \
    } while (0)

struct AState {
    unsigned int min_dist;          // min over pairs i < j of popc(w_i ^ w_j)
    unsigned int odd_pair;          // 1 if some pair (incl. i = j) has odd AND-parity
    unsigned long long hist[33];
    unsigned long long pairs;
};

// weight histogram + self-orthogonality of single words
__global__ void a_weights(const uint32_t *__restrict__ w, unsigned long long M, AState *st) {
    __shared__ unsigned long long h[33];
    for (int i = threadIdx.x; i < 33; i += blockDim.x) h[i] = 0;
    __syncthreads();
    unsigned int odd = 0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < M;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int c = __popc(w[i]);
        atomicAdd(&h[c], 1ull);
        odd |= c & 1;
    }
    if (odd) st->odd_pair = 1;
    __syncthreads();
    for (int i = threadIdx.x; i < 33; i += blockDim.x)
        if (h[i]) atomicAdd(&st->hist[i], h[i]);
}

// all pairs i < j: minimum distance and AND-parity.  Warp item = 32 words (one per lane) x
// a block of earlier words read 32 at a time and broadcast by shuffle.
__global__ void a_pairs(const uint32_t *__restrict__ w, unsigned long long M, int orth, AState *st) {
    const int lane = threadIdx.x & 31;
    const unsigned long long gw = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const unsigned long long nb = (M + 31) / 32;                 // 32-word blocks
    const unsigned long long items = nb * (nb + 1) / 2;          // block pairs (bi >= bj)
    unsigned int best = 64, odd = 0;
    unsigned long long pairs = 0;
    for (unsigned long long it = gw; it < items; it += nw) {
        unsigned long long bi = (unsigned long long)((sqrt(8.0 * (double)it + 1.0) - 1.0) / 2.0);
        while ((bi + 1) * (bi + 2) / 2 <= it) ++bi;
        while (bi * (bi + 1) / 2 > it) --bi;
        const unsigned long long bj = it - bi * (bi + 1) / 2;
        const unsigned long long i = bi * 32 + lane, j = bj * 32 + lane;
        const uint32_t wi = i < M ? w[i] : 0u;
        const uint32_t wj = j < M ? w[j] : 0u;
        for (int k = 0; k < 32; ++k) {
            const uint32_t c = __shfl_sync(0xffffffffu, wj, k);
            const unsigned long long jk = bj * 32 + k;
            if (i < M && jk < i) {
                best = min(best, (unsigned int)__popc(wi ^ c));
                if (orth) odd |= __popc(wi & c) & 1;
                ++pairs;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        best = min(best, __shfl_down_sync(0xffffffffu, best, o));
        odd |= __shfl_down_sync(0xffffffffu, odd, o);
        pairs += __shfl_down_sync(0xffffffffu, pairs, o);
    }
    if (lane == 0) {
        atomicMin(&st->min_dist, best);
        if (odd) st->odd_pair = 1;
        atomicAdd(&st->pairs, pairs);
    }
}

// GF(2) basis of each thread's words (strided), written out for the host-side merge
__global__ void a_basis(const uint32_t *__restrict__ w, unsigned long long M, uint32_t *bases) {
    uint32_t b[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) b[k] = 0;
    const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    for (unsigned long long i = tid; i < M; i += (unsigned long long)gridDim.x * blockDim.x) {
        uint32_t x = w[i];
#pragma unroll
        for (int k = 31; k >= 0; --k) {
            if (x >> k & 1u) {
                if (b[k]) x ^= b[k];
                else { b[k] = x; x = 0; }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) bases[tid * 32 + k] = b[k];
}

int analyze_device(const uint32_t *d_words, uint64_t M, int pairwise, int orth, void *stream, gc_analysis *out) {
    cudaStream_t s = (cudaStream_t)stream;
    int dev, sms = 148;
    ACK(cudaGetDevice(&dev));
    ACK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    AState *st = nullptr;
    uint32_t *bases = nullptr;
    const int bthreads = 256, bblocks = sms * 2;
    ACK(cudaMalloc(&st, sizeof(AState)));
    AState init{};
    init.min_dist = 0xffffffffu;
    ACK(cudaMemcpyAsync(st, &init, sizeof init, cudaMemcpyHostToDevice, s));
    if (cudaMalloc(&bases, (size_t)bthreads * bblocks * 32 * 4) != cudaSuccess) {
        cudaFree(st);
        set_error("cudaMalloc failed");
        return GC_ENOMEM;
    }
    if (M) {
        a_weights<<<sms * 4, 256, 0, s>>>(d_words, M, st);
        if (pairwise && M > 1) a_pairs<<<sms * 8, 256, 0, s>>>(d_words, M, orth, st);
        a_basis<<<bblocks, bthreads, 0, s>>>(d_words, M, bases);
    }
    cudaError_t e = cudaGetLastError();
    AState h{};
    std::vector<uint32_t> hb((size_t)bthreads * bblocks * 32);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, st, sizeof h, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hb.data(), bases, hb.size() * 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(st);
    cudaFree(bases);
    if (e != cudaSuccess) { set_error(cudaGetErrorString(e)); return GC_ECUDA; }
    // merge the per-thread bases (<= 32 vectors each)
    uint32_t b[32] = {0};
    int rank = 0;
    for (uint32_t x : hb) {
        for (int k = 31; k >= 0 && x; --k) {
            if (!(x >> k & 1u)) continue;
            if (b[k]) x ^= b[k];
            else { b[k] = x; x = 0; ++rank; }
        }
    }
    out->struct_size = sizeof(gc_analysis);
    out->M = M;
    for (int i = 0; i < 33; ++i) out->weight_hist[i] = M ? h.hist[i] : 0;
    out->gf2_rank = (uint32_t)rank;
    out->is_linear = (M > 0 && rank < 64 && M == (1ull << rank)) ? 1u : 0u;
    // minimum distance: pairwise if asked, else (linear codes) the minimum nonzero weight
    uint32_t md = 0;
    if (pairwise) md = (M > 1) ? h.min_dist : 0u;
    else if (out->is_linear) {
        for (int wgt = 1; wgt <= 32; ++wgt) if (h.hist[wgt]) { md = (uint32_t)wgt; break; }
    }
    out->min_distance = md;
    out->pairs_checked = h.pairs;
    // self-orthogonal: every word even and every pair even AND-parity; for a linear code
    // it suffices to check the basis (bilinearity), otherwise the pairwise pass decides
    uint32_t so = h.odd_pair ? 0u : 1u;
    if (so && !(pairwise && orth)) {
        if (out->is_linear) {
            for (int i = 0; i < 32 && so; ++i)
                for (int j = i; j < 32 && so; ++j)
                    if (b[i] && b[j] && (__builtin_popcount(b[i] & b[j]) & 1)) so = 0;
        } else {
            so = 2;   // unknown: not linear and no pairwise orthogonality pass
        }
    }
    out->self_orthogonal = so;
    return GC_OK;
}

}  // namespace gc

using namespace gc;

extern "C" int gc_analyze_device(const uint32_t *d_words, uint64_t M, uint32_t flags, void *stream,
                                 gc_analysis *out) {
    clear_error();
    if (!out || (!d_words && M)) { set_error("NULL pointer"); return GC_EINVAL; }
    if (flags & ~(GC_ANALYZE_PAIRWISE | GC_ANALYZE_ORTHOGONALITY)) { set_error("unknown analysis flags"); return GC_EINVAL; }
    return analyze_device(d_words, M, (flags & GC_ANALYZE_PAIRWISE) != 0, (flags & GC_ANALYZE_ORTHOGONALITY) != 0,
                          stream, out);
}

extern "C" int gc_analyze(const uint64_t *words, uint64_t M, uint32_t flags, gc_analysis *out) {
    clear_error();
    if (!out || (!words && M)) { set_error("NULL pointer"); return GC_EINVAL; }
    if (flags & ~(GC_ANALYZE_PAIRWISE | GC_ANALYZE_ORTHOGONALITY)) { set_error("unknown analysis flags"); return GC_EINVAL; }
    for (uint64_t i = 0; i < M; ++i)
        if (words[i] >> 32) { set_error("words must be < 2^32"); return GC_EINVAL; }
    std::vector<uint32_t> h(M);
    for (uint64_t i = 0; i < M; ++i) h[i] = (uint32_t)words[i];
    uint32_t *d = nullptr;
    if (M) ACK(cudaMalloc(&d, M * 4));
    cudaError_t e = M ? cudaMemcpy(d, h.data(), M * 4, cudaMemcpyHostToDevice) : cudaSuccess;
    if (e != cudaSuccess) { cudaFree(d); set_error(cudaGetErrorString(e)); return GC_ECUDA; }
    int rc = analyze_device(d, M, (flags & GC_ANALYZE_PAIRWISE) != 0, (flags & GC_ANALYZE_ORTHOGONALITY) != 0,
                            nullptr, out);
    cudaFree(d);
    return rc;
}
