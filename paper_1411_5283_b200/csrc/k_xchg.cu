// k_xchg.cu — the multi-GPU exchange of the long words, on the table of
// distinct words each rank's K1 built (k_hash.cuh).
//
// The paper's MPI version sends chunks of a sub-array to slaves and merges them back (§4).
// Here every rank holds the DISTINCT long words of its text shard with their counts; the ranks agree on
// splitters over (length, word) and every distinct word goes, with its count, to the one rank that owns
// its range; equal words from all ranks meet there and their counts add. So only (word, count) records
// cross NVLink, not every occurrence.
//   KX1 k_xchg_sample     count-weighted systematic sample of this rank's distinct words
//   KX2 k_xchg_rank       (all ranks' samples, all-gathered) rank of each sample in (length, word, index)
//   KX3 k_xchg_split      the P-1 splitters at the weighted quantiles (identical on every rank)
//   KX4 k_xchg_count      destination of every distinct word; records per destination
//   KX5 k_xchg_write      (after the all-gather of the record counts) every record stored straight into
//                         its destination's receive window (peer memory over NVLink: P2P stores), at an
//                         offset from a device-side scan of the count matrix — no host read-back
//   KX6 k_xchg_absorb     (after a barrier) the received records counted into this rank's table
#include "k_hash.cuh"

namespace wsort {
namespace {

constexpr int kXT = 256;

// (L, key) of distinct word j of the gathered buckets (keys_a layout; tile_from_prefix over dist_pfx)
__device__ __forceinline__ void word_of(const XchgArgs &a, uint32_t j, uint32_t &L, const uint32_t *&key) {
    const TileDesc td = tile_from_prefix(a.dist_pfx, j);
    L = td.L;
    key = a.keys + a.kbuckets[L].key_off + (uint64_t)td.tile * ((L + 5u) / 6u);
}

// -1 / 0 / 1: (La, ka) against (Lb, kb), length first (readings A4/A5)
__device__ __forceinline__ int cmp_word(uint32_t La, const uint32_t *ka, uint32_t Lb, const uint32_t *kb) {
    if (La != Lb) return La < Lb ? -1 : 1;
    const uint32_t kw = (La + 5u) / 6u;
    for (uint32_t q = 0; q < kw; q++) {
        const uint32_t x = ka[q], y = kb[q];
        if (x != y) return x < y ? -1 : 1;
    }
    return 0;
}

// KX1: sample k = the word holding count-quantile (2k+1)/(2s) of this rank's long words (prefix = inclusive
// prefix of the counts in gathered order); record [L, weight lo, weight hi, key...], weight = total / s
__global__ void __launch_bounds__(kXT) k_xchg_sample(XchgArgs a) {
    const uint32_t k = blockIdx.x * kXT + threadIdx.x;
    if (k >= a.nsamples) return;
    uint32_t *rec = a.samples + (size_t)k * a.rec_words;
    for (uint32_t q = 0; q < a.rec_words; q++) rec[q] = 0;
    const uint64_t total = a.D ? a.prefix[a.D - 1] : 0;
    if (!total) return;   // (L = 0: an empty sample, ranked below every word and never a splitter)
    const uint64_t target = ((2ull * k + 1ull) * total) / (2ull * a.nsamples);
    uint32_t lo = 0, hi = a.D - 1;   // first j with prefix[j] > target
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a.prefix[mid] > target) hi = mid;
        else lo = mid + 1;
    }
    uint32_t L;
    const uint32_t *key;
    word_of(a, lo, L, key);
    rec[0] = L;
    const uint64_t w = total / a.nsamples + 1ull;
    rec[1] = (uint32_t)w;
    rec[2] = (uint32_t)(w >> 32);
    for (uint32_t q = 0; q < (L + 5u) / 6u; q++) rec[3 + q] = key[q];
}

// KX2: rank of every all-gathered sample i in (L, key, i) order -> order[rank] = i
__global__ void __launch_bounds__(kXT) k_xchg_rank(XchgArgs a) {
    const uint32_t i = blockIdx.x * kXT + threadIdx.x;
    if (i >= a.nall) return;
    const uint32_t *ri = a.all_samples + (size_t)i * a.rec_words;
    uint32_t rank = 0;
    for (uint32_t j = 0; j < a.nall; j++) {
        const uint32_t *rj = a.all_samples + (size_t)j * a.rec_words;
        const int c = cmp_word(rj[0], rj + 3, ri[0], ri + 3);
        rank += c < 0 || (c == 0 && j < i);
    }
    a.order[rank] = i;
}

// KX3 (one block): walk the samples in order with their cumulative weight; splitter d (1..P-1) = the first
// sample whose cumulative weight reaches d/P of the total. Record [L, key...] (rec_words - 2 words).
__global__ void __launch_bounds__(1024) k_xchg_split(XchgArgs a) {
    __shared__ unsigned long long ws[32];
    __shared__ unsigned long long s_total, s_run;
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {
        s_total = 0;
        s_run = 0;
    }
    __syncthreads();
    for (uint32_t i = t; i < a.nall; i += 1024) {
        const uint32_t *r = a.all_samples + (size_t)i * a.rec_words;
        atomicAdd(&s_total, (unsigned long long)r[1] | ((unsigned long long)r[2] << 32));
    }
    __syncthreads();
    const unsigned long long total = s_total;
    for (uint32_t b0 = 0; b0 < a.nall; b0 += 1024) {
        const uint32_t i = b0 + t;
        unsigned long long w = 0;
        if (i < a.nall) {
            const uint32_t *r = a.all_samples + (size_t)a.order[i] * a.rec_words;
            w = (unsigned long long)r[1] | ((unsigned long long)r[2] << 32);
        }
        unsigned long long x = w;   // inclusive scan over the block
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned long long v = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= (uint32_t)o) v += y;
            }
            ws[lane] = v;
        }
        __syncthreads();
        const unsigned long long run = s_run, incl = run + x + (warp ? ws[warp - 1] : 0ull), excl = incl - w;
        if (i < a.nall && w) {
            for (uint32_t d = 1; d < a.nparts; d++) {   // the sample where d/P of the weight is first reached
                const unsigned long long q = (total * d) / a.nparts;
                if (excl < q + 1ull && incl >= q + 1ull) {
                    const uint32_t *r = a.all_samples + (size_t)a.order[i] * a.rec_words;
                    uint32_t *sp = a.splitters + (size_t)(d - 1) * (a.rec_words - 2);
                    sp[0] = r[0];
                    for (uint32_t qq = 3; qq < a.rec_words; qq++) sp[qq - 2] = r[qq];
                }
            }
        }
        __syncthreads();
        if (t == 1023) s_run = incl;
        __syncthreads();
    }
}

// destination of (L, key): how many splitters are <= it
__device__ __forceinline__ uint32_t dest_of(const XchgArgs &a, uint32_t L, const uint32_t *key) {
    uint32_t lo = 0, hi = a.nparts - 1;   // first splitter > word
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t *sp = a.splitters + (size_t)mid * (a.rec_words - 2);
        if (cmp_word(sp[0], sp + 1, L, key) > 0) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// KX4: destination of every distinct word (dest[j]) and records per destination
__global__ void __launch_bounds__(kXT) k_xchg_count(XchgArgs a) {
    __shared__ uint32_t cnt[kMaxRanks];
    if (threadIdx.x < kMaxRanks) cnt[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t j = blockIdx.x * kXT + threadIdx.x;
    if (j < a.D) {
        uint32_t L;
        const uint32_t *key;
        word_of(a, j, L, key);
        const uint32_t d = dest_of(a, L, key);
        a.dest[j] = (uint8_t)d;
        atomicAdd(&cnt[d], 1u);
    }
    __syncthreads();
    if (threadIdx.x < a.nparts && cnt[threadIdx.x]) atomicAdd(a.send_counts + threadIdx.x, cnt[threadIdx.x]);
}

// cursor[d] = records the ranks before this one send to d (matrix[src][d] all-gathered, src-major)
__global__ void k_xchg_offsets(XchgArgs a) {
    const uint32_t d = threadIdx.x;
    if (d >= a.nparts) return;
    uint32_t off = 0;
    for (uint32_t src = 0; src < a.rank; src++) off += a.matrix[src * a.nparts + d];
    a.cursor[d] = off;
    if (d == 0) {   // records this rank receives
        uint32_t n = 0;
        for (uint32_t src = 0; src < a.nparts; src++) n += a.matrix[src * a.nparts + a.rank];
        a.recv_n[0] = n;
    }
}

// KX5: every distinct word's record [L, count, 0, key...] stored into its destination's window (P2P)
__global__ void __launch_bounds__(kXT) k_xchg_write(XchgArgs a) {
    const uint32_t j = blockIdx.x * kXT + threadIdx.x;
    if (j >= a.D) return;
    uint32_t L;
    const uint32_t *key;
    word_of(a, j, L, key);
    const uint32_t d = a.dest[j];
    const uint32_t pos = atomicAdd(a.cursor + d, 1u);
    if ((uint64_t)pos >= a.win_cap) {   // (cannot happen: windows hold every rank's distinct words)
        atomicExch(a.flag, 1u);
        return;
    }
    uint32_t *rec = a.peer_win[d] + (size_t)pos * a.rec_words;
    const uint32_t c = a.counts[j];
    rec[0] = L;
    rec[1] = c;
    rec[2] = 0;
    const uint32_t kw = (L + 5u) / 6u;
    for (uint32_t q = 0; q < kw; q++) rec[3 + q] = key[q];
    __threadfence_system();   // the stores reach the peer before the barrier that follows this kernel
}

// KX6: the received records counted into this rank's (cleared) table; words per length for the placement
__global__ void __launch_bounds__(kXT) k_xchg_absorb(XchgArgs a) {
    const uint32_t n = min(a.recv_n[0], (uint32_t)a.win_cap);
    for (uint32_t i = blockIdx.x * kXT + threadIdx.x; i < n; i += gridDim.x * kXT) {
        const uint32_t *rec = a.win + (size_t)i * a.rec_words;
        const uint32_t L = rec[0], c = rec[1], kw = (L + 5u) / 6u;
        atomicAdd(a.lwords + L, (unsigned long long)c);
        const uint32_t *key = rec + 3;
        if (L <= 24u) {
            const uint32_t slot = hashtab::find_narrow(a.tab, hashtab::narrow_key(key[0], kw > 1 ? key[1] : 0u,
                                                                                  kw > 2 ? key[2] : 0u, kw > 3 ? key[3] : 0u),
                                                       L, true);
            if (slot != hashtab::kUnset) atomicAdd(a.tab.ncnt + slot, c);
        } else {
            auto get = [&](uint32_t q) { return key[q]; };
            const uint64_t fp = hashtab::fingerprint(L, kw, get);
            const uint32_t slot = hashtab::find(a.tab, L, kw, fp, get, true);
            if (slot != hashtab::kUnset) atomicAdd(a.tab.cnt + slot, c);
        }
    }
}

}  // namespace

cudaError_t launch_xchg_sample(const XchgArgs &a, cudaStream_t s) {
    k_xchg_sample<<<(a.nsamples + kXT - 1) / kXT, kXT, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_xchg_split(const XchgArgs &a, cudaStream_t s) {
    if (a.nparts < 2) return cudaSuccess;
    k_xchg_rank<<<(a.nall + kXT - 1) / kXT, kXT, 0, s>>>(a);
    k_xchg_split<<<1, 1024, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_xchg_count(const XchgArgs &a, cudaStream_t s) {
    if (a.D) k_xchg_count<<<(a.D + kXT - 1) / kXT, kXT, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_xchg_write(const XchgArgs &a, cudaStream_t s) {
    k_xchg_offsets<<<1, kMaxRanks, 0, s>>>(a);
    if (a.D) k_xchg_write<<<(a.D + kXT - 1) / kXT, kXT, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_xchg_absorb(const XchgArgs &a, uint32_t grid, cudaStream_t s) {
    k_xchg_absorb<<<grid, kXT, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace wsort
