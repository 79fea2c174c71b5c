// k_ragged.cu — phase 3 on a RAGGED backing (WSORT_ALGO_RAGGED): the paper's "vectors of strings"
// (§3.1: "the difference between them is the data structure. 1) Implemented based on vectors of
// strings; 2) implemented based on array char 3D"), measured against the fixed-width keys (the "array char
// 3D") the other algorithms sort.
//
// A sub-array element is a reference to the word in the text (its byte offset; the length is the bucket's),
// and every comparison reads both words through the references, letter groups of 4 from the text (L1 / L2),
// folded (reading A2), in unsigned byte order (A4); equal words compare by offset, so the order is stable
// (src_off comes out for free). Sort per length bucket: bitonic tiles of 1024 references in shared memory,
// then merge-path merges of sorted runs (the paper's merge) until each bucket is one run; emit
// copies each word from the text.
#include "wsort_internal.cuh"

namespace wsort {
namespace {

constexpr int kRT = 256;
constexpr uint32_t kRaggedTile = 1024;   // references per bitonic tile (4 per thread)
constexpr uint32_t kInf = 0xffffffffu;   // padding reference: after every word

// 4 letters of the text at byte p, folded, the first in the top byte (big-endian: unsigned compare = order)
__device__ __forceinline__ uint32_t letters4(const uint8_t *text, uint32_t p) {
    const uint32_t *w = reinterpret_cast<const uint32_t *>(text + (p & ~3u));
    const uint32_t v = __funnelshift_r(__ldg(w), __ldg(w + 1), 8u * (p & 3u)) | 0x20202020u;
    return __byte_perm(v, 0, 0x0123);
}

// a < b for two references to words of L letters (ties: the earlier text position first)
__device__ __forceinline__ bool ref_less(const uint8_t *text, uint32_t L, uint32_t a, uint32_t b) {
    if (a == kInf || b == kInf) return a != kInf && b == kInf;
    for (uint32_t i = 0; i < L; i += 4) {
        uint32_t x = letters4(text, a + i), y = letters4(text, b + i);
        if (L - i < 4) {   // the last group: only the word's own letters
            const uint32_t m = ~0u << (8u * (4u - (L - i)));
            x &= m;
            y &= m;
        }
        if (x != y) return x < y;
    }
    return a < b;
}

// bitonic sort of one tile of a bucket's references in shared memory
__global__ void __launch_bounds__(kRT) k_ragged_tiles(RaggedArgs a) {
    __shared__ uint32_t r[kRaggedTile];
    const TileDesc td = tile_from_prefix_cta(a.tile_pfx, blockIdx.x);
    const BucketInfo b = a.buckets[td.L];
    const uint32_t k0 = td.tile * kRaggedTile, n = min(kRaggedTile, b.n - k0);
    const uint32_t *src = a.in + b.word_off + k0;
    for (uint32_t i = threadIdx.x; i < kRaggedTile; i += kRT) r[i] = i < n ? src[i] : kInf;
    __syncthreads();
    for (uint32_t k = 2; k <= kRaggedTile; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < kRaggedTile; i += kRT) {
                const uint32_t p = i ^ j;
                if (p > i) {
                    const uint32_t x = r[i], y = r[p];
                    const bool up = (i & k) == 0;
                    if (up == ref_less(a.text, td.L, y, x)) {
                        r[i] = y;
                        r[p] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
    uint32_t *dst = a.out + b.word_off + k0;
    for (uint32_t i = threadIdx.x; i < n; i += kRT) dst[i] = r[i];
}

// one merge pass: sorted runs of `run` references -> runs of 2 run; block = 1024 outputs of one bucket,
// each thread 4 consecutive outputs from its merge-path split (binary search on the diagonal)
__global__ void __launch_bounds__(kRT) k_ragged_merge(RaggedArgs a) {
    const TileDesc td = tile_from_prefix_cta(a.tile_pfx, blockIdx.x);
    const BucketInfo b = a.buckets[td.L];
    const uint32_t L = td.L, run = a.run;
    const uint32_t *in = a.in + b.word_off;
    uint32_t *out = a.out + b.word_off;
    const uint32_t o0 = td.tile * kRaggedTile + threadIdx.x * 4u;
    if (o0 >= b.n) return;
    const uint32_t s = o0 / (2 * run) * (2 * run);            // the pair of runs holding output o0
    const uint32_t na = min(run, b.n - s), nb = min(run, b.n - s - na);
    const uint32_t *A = in + s, *B = in + s + na;
    const uint32_t d = o0 - s;                                 // diagonal
    uint32_t lo = d > nb ? d - nb : 0u, hi = min(d, na);       // i = elements taken from A
    while (lo < hi) {
        const uint32_t i = (lo + hi) >> 1;
        if (ref_less(a.text, L, B[d - i - 1], A[i])) hi = i;   // A[i] is after B[d-i-1]: take fewer from A
        else lo = i + 1;
    }
    uint32_t i = lo, j = d - lo;
    for (uint32_t k = 0; k < 4u && o0 + k < min(b.n, s + na + nb); k++) {
        const bool takeA = i < na && (j >= nb || !ref_less(a.text, L, B[j], A[i]));
        out[o0 + k] = takeA ? A[i++] : B[j++];
    }
}

// "word\n" of every reference (copied from the text, folded); src_off = global offsets
__global__ void __launch_bounds__(kRT) k_ragged_emit(RaggedArgs a) {
    const TileDesc td = tile_from_prefix_cta(a.tile_pfx, blockIdx.x);
    const BucketInfo b = a.buckets[td.L];
    const uint32_t L = td.L;
    const uint32_t k = td.tile * kRaggedTile + threadIdx.x * 4u;
    for (uint32_t q = 0; q < 4u && k + q < b.n; q++) {
        const uint32_t p = a.in[b.word_off + k + q];
        uint8_t *o = a.words + b.byte_off + (uint64_t)(k + q) * (L + 1);
        for (uint32_t i = 0; i < L; i++) o[i] = a.text[p + i] | 0x20u;
        o[L] = '\n';
        if (a.src_off) a.src_off[b.word_off + k + q] = a.global_base + p;
    }
}

}  // namespace

uint32_t ragged_tile() { return kRaggedTile; }
cudaError_t launch_ragged_tiles(const RaggedArgs &a, cudaStream_t s) {
    if (a.ntiles) k_ragged_tiles<<<a.ntiles, kRT, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_ragged_merge(const RaggedArgs &a, cudaStream_t s) {
    if (a.ntiles) k_ragged_merge<<<a.ntiles, kRT, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_ragged_emit(const RaggedArgs &a, cudaStream_t s) {
    if (a.ntiles) k_ragged_emit<<<a.ntiles, kRT, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace wsort
