// k_dist.cu — the multi-GPU exchange step: a sample sort over the global order
// (length, key, source rank). It replaces the paper's MPI master/slave scatter-gather (PAPER.md:76,
// §4: "the master will send the data to the slaves ... merges all the chunks"), which would
// serialise on one device, by a symmetric exchange: every rank sends every other rank the keys that
// fall between two global splitters, then sorts what it received.
//
//   k_sample         regular sample of a rank's packed keys: records [L, rank, key words, 0-pad]
//   k_part_count     per tile, how many keys go to each destination; totals per (dest, length)
//   k_part_scatter   each key to the send buffer laid out [dest][length][keys]
//   k_regroup        received [src][length][keys] ranges -> per-length buckets (src order)
// Splitter order: (L, key words, rank) lexicographic; a key equal to a splitter in (L, key) goes to
// the lower side iff its source rank <= the splitter's rank. Identical keys from one rank share a
// destination, so the output (concatenation in rank order) equals the one-GPU output.
#include "wsort_internal.cuh"

namespace wsort {
namespace {

constexpr int kDT = 256;

// true iff splitter record s < element (L, key[kw], rank)
__device__ __forceinline__ bool split_lt(const uint32_t *s, uint32_t L, const uint32_t *key, uint32_t kw,
                                         uint32_t rank) {
    if (s[0] != L) return s[0] < L;
    for (uint32_t u = 0; u < kw; u++) {
        const uint32_t a = s[2 + u], b = key[u];
        if (a != b) return a < b;
    }
    return s[1] < rank;
}

__device__ __forceinline__ uint32_t dest_of(const DistArgs &a, uint32_t L, const uint32_t *key, uint32_t kw) {
    uint32_t lo = a.split_lo[L], hi = a.split_hi[L];   // splitters with length < L / <= L
    while (lo < hi) {                                   // number of splitters < element
        const uint32_t mid = (lo + hi) >> 1;
        if (split_lt(a.splitters + (size_t)mid * a.rec_words, L, key, kw, a.rank)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kDT) k_sample(DistArgs a) {
    const uint32_t i = blockIdx.x * kDT + threadIdx.x;
    if (i >= a.nsamples) return;
    uint32_t *rec = a.records + (size_t)i * a.rec_words;
    for (uint32_t u = 0; u < a.rec_words; u++) rec[u] = 0;
    if (a.n_words == 0) return;
    const uint64_t g = ((2ull * i + 1) * a.n_words) / (2ull * a.nsamples);   // regular positions
    uint32_t lo = 1, hi = 256;                      // largest L with off[L] <= g (off[256] = W > g)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a.off[mid] <= g) lo = mid;
        else hi = mid;
    }
    const uint32_t L = lo;
    const BucketInfo b = a.buckets[L];
    const uint32_t *key = a.keys + b.key_off + (g - b.word_off) * b.kw;
    rec[0] = L;
    rec[1] = a.rank;
    for (uint32_t u = 0; u < b.kw && 2 + u < a.rec_words; u++) rec[2 + u] = key[u];
}

__global__ void __launch_bounds__(kDT) k_part_count(DistArgs a) {
    __shared__ uint32_t cnt[kMaxRanks];
    const int t = threadIdx.x;
    const TileDesc td = a.tiles[blockIdx.x];
    const BucketInfo b = a.buckets[td.L];
    const uint32_t k0 = td.tile * kDistTileKeys, nk = min(kDistTileKeys, b.n - k0);
    if (a.split_lo[td.L] == a.split_hi[td.L]) {   // no splitter inside this bucket: one destination
        if (t == 0) atomicAdd(&a.counts[(size_t)a.split_lo[td.L] * 256 + td.L], nk);
        return;
    }
    for (uint32_t d = t; d < a.nparts; d += kDT) cnt[d] = 0;
    __syncthreads();
    const uint32_t *keys = a.keys + b.key_off;
    for (uint32_t k = t; k < nk; k += kDT) atomicAdd(&cnt[dest_of(a, td.L, keys + (uint64_t)(k0 + k) * b.kw, b.kw)], 1u);
    __syncthreads();
    for (uint32_t d = t; d < a.nparts; d += kDT)
        if (cnt[d]) atomicAdd(&a.counts[(size_t)d * 256 + td.L], cnt[d]);
}

__global__ void __launch_bounds__(kDT) k_part_scatter(DistArgs a) {
    __shared__ uint32_t cnt[kMaxRanks], base[kMaxRanks];
    const int t = threadIdx.x;
    const TileDesc td = a.tiles[blockIdx.x];
    const BucketInfo b = a.buckets[td.L];
    const uint32_t L = td.L, kw = b.kw;
    const uint32_t k0 = td.tile * kDistTileKeys, nk = min(kDistTileKeys, b.n - k0);
    const uint32_t *keys = a.keys + b.key_off;
    const bool one = a.split_lo[L] == a.split_hi[L];
    for (uint32_t d = t; d < a.nparts; d += kDT) cnt[d] = 0;
    __syncthreads();
    uint32_t dst[kDistTileKeys / kDT], slot[kDistTileKeys / kDT];
#pragma unroll
    for (int r = 0; r < kDistTileKeys / kDT; r++) {
        const uint32_t k = t + r * kDT;
        dst[r] = 0;
        slot[r] = 0;
        if (k < nk) {
            dst[r] = one ? a.split_lo[L] : dest_of(a, L, keys + (uint64_t)(k0 + k) * kw, kw);
            slot[r] = atomicAdd(&cnt[dst[r]], 1u);
        }
    }
    __syncthreads();
    for (uint32_t d = t; d < a.nparts; d += kDT)
        base[d] = cnt[d] ? atomicAdd(&a.cursor[(size_t)d * 256 + L], cnt[d]) : 0u;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kDistTileKeys / kDT; r++) {
        const uint32_t k = t + r * kDT;
        if (k < nk) {
            const uint32_t d = dst[r];
            uint32_t *o = a.send + a.send_base[(size_t)d * 256 + L] + (uint64_t)(base[d] + slot[r]) * kw;
            const uint32_t *src = keys + (uint64_t)(k0 + k) * kw;
            for (uint32_t u = 0; u < kw; u++) o[u] = src[u];
        }
    }
}

// Copy received ranges into per-length buckets: range r = (src, L) of `len` words from recv + from
// to keys + to. One CTA per 4096-word chunk of a range.
__global__ void __launch_bounds__(kDT) k_regroup(const CopyRange *ranges, const uint32_t *recv, uint32_t *keys) {
    const CopyRange r = ranges[blockIdx.x];
    for (uint32_t i = threadIdx.x; i < r.len; i += kDT) keys[r.to + i] = __ldg(recv + r.from + i);
}

}  // namespace

cudaError_t launch_sample(const DistArgs &a, cudaStream_t s) {
    if (a.nsamples == 0) return cudaSuccess;
    k_sample<<<(a.nsamples + kDT - 1) / kDT, kDT, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_part_count(const DistArgs &a, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    k_part_count<<<a.ntiles, kDT, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_part_scatter(const DistArgs &a, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    k_part_scatter<<<a.ntiles, kDT, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_regroup(const CopyRange *ranges, uint32_t nranges, const uint32_t *recv, uint32_t *keys,
                           cudaStream_t s) {
    if (nranges == 0) return cudaSuccess;
    k_regroup<<<nranges, kDT, 0, s>>>(ranges, recv, keys);
    return cudaGetLastError();
}

}  // namespace wsort
