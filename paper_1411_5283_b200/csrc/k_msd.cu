// k_msd.cu — phase 3 for the staged long words: most-significant-digit radix partitioning of every length
// bucket ("sort each vector ... in the alphabetic order"), finished per
// sub-bucket on one CTA.
//
// Keys only: equal keys are identical words, so no pass has to be stable. A level-l pass splits every
// "big" segment by its l-th 2-letter digit:
//   k_msd_count      per tile: digit histogram in shared memory -> per-segment histogram (atomics)
//   k_msd_plan       per segment: exclusive scan of its histogram -> children's bases / scatter cursors;
//                    every child is queued as a finishing job, or as a segment of the next level
//   k_msd_scatter_p  persistent, TMA double-buffered tiles: a shared-memory atomic gives each key its slot
//                    inside its digit, one global atomic per (tile, digit) reserves the range, keys are
//                    reordered in shared memory and written out coalesced (k_msd_scatter: per-tile form)
// Finishing (AUTO, the streaming finish, stream_fin = 1):
//   k_msd_fin        persistent (job tickets, biggest first): a job (a child of any size, or several small
//                    children) is counted as an exact multiset in a shared-memory table (1-2-word keys: the
//                    key itself; wider keys: a 64-bit fingerprint verified word by word against a
//                    representative), its distinct keys sorted (odd-even transposition = the data-parallel
//                    bubble sort of PAPER.md:23, + merge paths, or rank counting), and each written as text
//                    as often as it occurs (16-byte windows of the repeated "word\n" pattern); a job with
//                    too many distinct keys goes one MSD level deeper
//   k_msd_fin_split  parts of jobs > 128 K keys (32 K keys each, their own CTA, a third stream); the last
//                    part merges the parts' lists; k_msd_fin_emit writes such a job's text by pieces
// Radix finish (msd_radix, and the distinct keys of the COUNT ingest, finish_radix = 1): k_msd_warp_sort
// (<= 32 keys, one warp), k_msd_radix_job / k_msd_cta_sort (one CTA tile), k_msd_copy (finished runs that
// ended in buffer A); every key ends in buffer B at its final index.
#include <type_traits>

#include "k_tma.cuh"
#include "wsort_internal.cuh"

namespace wsort {
namespace {

constexpr int kST = 256;
constexpr uint32_t kFullM = 0xffffffffu;

template <int KW>
__device__ __forceinline__ uint32_t digit_reg(const uint32_t (&k)[KW], uint32_t q) {
    uint32_t w = k[0];
#pragma unroll
    for (int u = 1; u < KW; u++) w = (q / 3) == (uint32_t)u ? k[u] : w;
    return (w >> (20 - 10 * (q % 3))) & 1023u;
}

template <int NT = kST>
__device__ __forceinline__ uint32_t block_excl_scan_m(uint32_t v, uint32_t *wsum, uint32_t *total) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFullM, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NT / 32 ? wsum[lane] : 0u, wi = w;
#pragma unroll
        for (int o = 1; o < NT / 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(kFullM, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < NT / 32) wsum[lane] = wi - w;
        if (lane == NT / 32 - 1) wsum[NT / 32] = wi;
    }
    __syncthreads();
    const uint32_t r = wsum[warp] + incl - v;
    if (total) *total = wsum[NT / 32];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- count
__global__ void __launch_bounds__(kST) k_msd_count(MsdArgs a) {
    __shared__ uint32_t h[kRadixBins];
    const int t = threadIdx.x;
    const MsdTile td = a.tiles[blockIdx.x];
    const MsdSeg sg = a.segs[td.seg];
    const BucketInfo b = a.buckets[sg.L];
    for (int i = t; i < kRadixBins; i += kST) h[i] = 0;
    __syncthreads();
    // only the digit's key word is read; a batch of loads is issued before its atomics
    const uint32_t *keys = ((sg.buf & 1u) ? a.keys_a : a.keys_b) + b.key_off + (uint64_t)(sg.start + td.off) * b.kw + a.level / 3;
    const uint32_t sh = 20 - 10 * (a.level % 3);
    for (uint32_t k0 = t; k0 < td.n; k0 += 8 * kST) {
        uint32_t w[8];
#pragma unroll
        for (int r = 0; r < 8; r++) {
            const uint32_t k = k0 + r * kST;
            w[r] = k < td.n ? __ldg(keys + (uint64_t)k * b.kw) : 0u;
        }
#pragma unroll
        for (int r = 0; r < 8; r++)
            if (k0 + r * kST < td.n) atomicAdd(&h[(w[r] >> sh) & 1023u], 1u);
    }
    __syncthreads();
    uint32_t *gh = a.hist + (size_t)td.seg * kRadixBins;
    for (int i = t; i < kRadixBins; i += kST)
        if (h[i]) atomicAdd(&gh[i], h[i]);
}

// ---------------------------------------------------------------- plan
// One CTA per segment of this level: exclusive scan of its digit histogram gives the children's
// bases (the scatter cursors). The non-empty children are compacted, then thread 0 walks them in
// digit order and classifies each (writing shared memory only):
//   big (> CTA-sort capacity, digits left)  -> next level (segment + its scatter tiles)
//   finished and already in B               -> nothing
//   finished, in A, larger than a CTA tile  -> copy chunks A -> B
//   everything else                         -> packed greedily into CTA / warp sort jobs of at most
//                                              one tile; sorting a run of consecutive children by the
//                                              full key sorts each child (their prefixes differ)
// One atomic per queue then reserves the slots and all threads write the entries.
constexpr int kPlanMax = 2048;
// Jobs of the first queue (q_tiny): <= 32 keys (warp sorts), or in streaming mode the big jobs
// (> kBigJobKeys), which the persistent finish takes before the others (longest first).
constexpr uint32_t kBigJobKeys = 16384;
__device__ __forceinline__ bool first_queue(const MsdArgs &a, uint32_t n) { return a.stream_fin ? n > kBigJobKeys : n <= 32; }   // >= 2 x the non-empty digits of a segment (<= 27*26)
__global__ void __launch_bounds__(kST) k_msd_plan(MsdArgs a) {
    __shared__ uint32_t wsum[kST / 32 + 1];
    __shared__ uint32_t nz_d[kRadixBins];
    __shared__ MsdSeg jobs[kPlanMax];        // sort jobs from the bottom, big/copy children from the top
    __shared__ uint32_t big_t0[kPlanMax];
    __shared__ uint32_t s_n[4], s_q[4];
    const int t = threadIdx.x;
    const uint32_t s = blockIdx.x;
    const MsdSeg sg = a.segs[s];
    const BucketInfo b = a.buckets[sg.L];
    const uint32_t *h = a.hist + (size_t)s * kRadixBins;
    uint32_t c[4];
#pragma unroll
    for (int e = 0; e < 4; e++) c[e] = h[4 * t + e];
    const uint32_t nzc = (c[0] != 0) + (c[1] != 0) + (c[2] != 0) + (c[3] != 0);
    uint32_t ex = block_excl_scan_m(c[0] + c[1] + c[2] + c[3], wsum, nullptr);
    uint32_t nzt = 0;
    uint32_t nzx = block_excl_scan_m(nzc, wsum, &nzt);
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const uint32_t d = 4 * t + e;
        if (a.plan_mode != 2) a.cursor[(size_t)s * kRadixBins + d] = sg.start + ex;   // (mode 2: being consumed)
        if (c[e]) nz_d[nzx++] = sg.start + ex;
        ex += c[e];
    }
    if (a.plan_mode == 1) return;   // the scatter's cursors only; the jobs are planned beside the scatter
    __syncthreads();
    const uint32_t src_a = sg.buf & 1u, dst_a = src_a ^ 1u;   // where the segment is / its children go
    // (chunk mode: the keys are in the staging chunks, every segment is scattered)
    if (t == 0 && nzt == 1 && a.level + 1 < b.ndig && sg.n > 1 && !a.chunk_mode) {
        // every key shares this digit: no data movement; the segment goes to the next level as it is
        a.seg_skip[s] = 1u;
        const uint32_t nt = (sg.n + b.aux - 1) / b.aux;
        const uint32_t q = atomicAdd(a.ctr + kQBig, 1u), t0 = atomicAdd(a.ctr + kQTiles, nt);
        if (q < a.cap_big) a.q_big[q] = MsdSeg{sg.L, sg.start, sg.n, src_a};
        for (uint32_t i = 0; i < nt && t0 + i < a.cap_tiles; i++)
            a.q_tiles[t0 + i] = MsdTile{q, i * b.aux, min(b.aux, sg.n - i * b.aux), 0};
    }
    if (nzt == 1 && a.level + 1 < b.ndig && sg.n > 1 && !a.chunk_mode) return;
    if (t == 0) a.seg_skip[s] = 0u;
    if (t == 0) {
        const bool final_digit = a.level + 1 >= b.ndig;
        const uint32_t cap = b.tile_keys, seg_end = sg.start + sg.n;
        uint32_t nj = 0, ntop = 0, ntiles = 0;
        uint32_t js = 0, jn = 0;
        for (uint32_t k = 0; k < nzt; k++) {
            const uint32_t start = nz_d[k], cnt = (k + 1 < nzt ? nz_d[k + 1] : seg_end) - start;
            const bool fin = final_digit || cnt == 1;
            const bool stream = a.stream_fin;   // every child is a finishing job of k_msd_fin (it writes the text)
            const bool big = !fin && cnt > cap && !stream, skip = fin && !dst_a && !stream,
                       copy = fin && dst_a && cnt > cap && !stream;
            if (big || skip || copy) {
                if (jn) jobs[nj++] = MsdSeg{sg.L, js, jn, dst_a | (a.level << 8)};
                jn = 0;
                if (big) {
                    big_t0[ntop] = ntiles;
                    jobs[kPlanMax - 1 - ntop++] = MsdSeg{sg.L, start, cnt, 1u};
                    ntiles += (cnt + b.aux - 1) / b.aux;
                } else if (copy) {
                    big_t0[ntop] = 0;
                    jobs[kPlanMax - 1 - ntop++] = MsdSeg{sg.L, start, cnt, 2u};
                }
            } else if (cnt > cap) {   // (stream) a child larger than a CTA tile is a job of its own
                if (jn) jobs[nj++] = MsdSeg{sg.L, js, jn, dst_a | (a.level << 8)};
                jn = 0;
                jobs[nj++] = MsdSeg{sg.L, start, cnt, dst_a | (a.level << 8)};
            } else {
                if (jn + cnt > cap) {
                    jobs[nj++] = MsdSeg{sg.L, js, jn, dst_a | (a.level << 8)};
                    jn = 0;
                }
                if (!jn) js = start;
                jn += cnt;
            }
        }
        if (jn) jobs[nj++] = MsdSeg{sg.L, js, jn, dst_a | (a.level << 8)};
        uint32_t ntiny = 0, nbig = 0, nch = 0;
        for (uint32_t k = 0; k < nj; k++) ntiny += first_queue(a, jobs[k].n);
        for (uint32_t k = 0; k < ntop; k++) {
            const MsdSeg &x = jobs[kPlanMax - 1 - k];
            if (x.buf == 1u) nbig++;
            else nch += (x.n * b.kw + kMsdCopyChunk - 1) / kMsdCopyChunk;
        }
        s_n[0] = nj;
        s_n[1] = ntop;
        s_q[0] = ntiny ? atomicAdd(a.ctr + kQTiny, ntiny) : 0u;
        s_q[1] = nj - ntiny ? atomicAdd(a.ctr + kQSmall, nj - ntiny) : 0u;
        s_q[2] = nbig ? atomicAdd(a.ctr + kQBig, nbig) : 0u;
        s_q[3] = ntiles ? atomicAdd(a.ctr + kQTiles, ntiles) : 0u;
        const uint32_t cq = nch ? atomicAdd(a.ctr + kQCopy, nch) : 0u;
        // copies are few: written here; big children get their queue index in buf
        uint32_t ci = 0, bi = 0;
        for (uint32_t k = 0; k < ntop; k++) {
            MsdSeg &x = jobs[kPlanMax - 1 - k];
            if (x.buf == 2u) {
                const uint32_t words = x.n * b.kw;
                for (uint32_t i = 0; i < words; i += kMsdCopyChunk) {
                    const uint64_t w0 = b.key_off + (uint64_t)x.start * b.kw + i;
                    const uint32_t q = cq + ci++;
                    if (q < a.cap_copy) a.q_copy[q] = CopyRange{w0, w0, min(kMsdCopyChunk, words - i), 0};
                }
            } else {
                x.buf = 16u + bi++;   // big: index among this segment's big children
            }
        }
    }
    __syncthreads();
    const uint32_t nj = s_n[0], ntop = s_n[1];
    // sort jobs, order-preserving split into tiny / small: thread t takes a contiguous block of jobs, the
    // tiny ones before it come from a block scan of the blocks' counts
    const uint32_t per = (nj + kST - 1) / kST, k0 = min(nj, per * t), k1 = min(nj, k0 + per);
    uint32_t my_tiny = 0;
    for (uint32_t k = k0; k < k1; k++) my_tiny += first_queue(a, jobs[k].n);
    uint32_t before_tiny = block_excl_scan_m(my_tiny, wsum, nullptr);
    for (uint32_t k = k0; k < k1; k++) {
        const MsdSeg x = jobs[k];
        if (first_queue(a, x.n)) {
            const uint32_t q = s_q[0] + before_tiny;
            if (q < a.cap_local) {
                a.q_tiny[q] = x;
                if (a.stream_fin) {   // a big job is counted by parts: reserve them
                    const uint32_t np = job_parts(x.n);
                    const uint32_t pb = atomicAdd(a.ctr + kQParts, np);
                    a.job_pbase[q] = pb;
                    a.job_done[q] = 0;
                    a.job_ovf[q] = 0;
                    for (uint32_t p = 0; p < np && pb + p < a.cap_parts; p++) a.q_parts[pb + p] = q;
                }
            }
            before_tiny++;
        } else {
            const uint32_t q = s_q[1] + (k - before_tiny);
            if (q < a.cap_local) a.q_small[q] = x;
        }
    }
    for (uint32_t k = t; k < ntop; k += kST) {
        MsdSeg x = jobs[kPlanMax - 1 - k];
        if (x.buf < 16u) continue;
        const uint32_t q = s_q[2] + (x.buf - 16u), t0 = s_q[3] + big_t0[k];
        const uint32_t nt = (x.n + b.aux - 1) / b.aux;
        x.buf = dst_a;   // the children of a scattered segment are in the other buffer
        if (q < a.cap_big) a.q_big[q] = x;
        for (uint32_t i = 0; i < nt && t0 + i < a.cap_tiles; i++)
            a.q_tiles[t0 + i] = MsdTile{q, i * b.aux, min(b.aux, x.n - i * b.aux), 0};
    }
}

// ---------------------------------------------------------------- scatter
template <int KW>
__device__ __forceinline__ void scatter_tile(const MsdArgs &a, const MsdTile &td, const MsdSeg &sg, const BucketInfo &b,
                                             uint32_t *sm, const uint32_t *tile_keys = nullptr) {
    constexpr int KPT = 32 / KW;   // keys per thread (striped)
    const int t = threadIdx.x;
    uint32_t *hist = sm, *toff = sm + kRadixBins, *gbase = sm + 2 * kRadixBins, *kout = sm + 3 * kRadixBins;
    uint32_t *wsum = kout + 8192 + 8192 / 32 + 8;
    for (int i = t; i < kRadixBins; i += kST) hist[i] = 0;
    __syncthreads();
    // the tile's keys: in global memory, or already in shared memory (tile_keys: the persistent kernel's TMA copy)
    const uint32_t *src = tile_keys ? tile_keys : ((sg.buf & 1u) ? a.keys_a : a.keys_b) + b.key_off + (uint64_t)(sg.start + td.off) * KW;
    uint32_t key[KPT][KW], slot[(KPT + 1) / 2];
#pragma unroll
    for (int r = 0; r < (KPT + 1) / 2; r++) slot[r] = 0;
    // all loads first (a shared-memory atomic between them would serialise them)
#pragma unroll
    for (int r = 0; r < KPT; r++) {
        const uint32_t i = t + r * kST;
#pragma unroll
        for (int u = 0; u < KW; u++) key[r][u] = i < td.n ? src[(uint64_t)i * KW + u] : 0u;
    }
#pragma unroll
    for (int r = 0; r < KPT; r++) {
        const uint32_t i = t + r * kST;
        if (i < td.n) slot[r / 2] |= atomicAdd(&hist[digit_reg<KW>(key[r], a.level)], 1u) << (16 * (r & 1));
    }
    __syncthreads();
    uint32_t c[4];
#pragma unroll
    for (int e = 0; e < 4; e++) c[e] = hist[4 * t + e];
    uint32_t ex = block_excl_scan_m(c[0] + c[1] + c[2] + c[3], wsum, nullptr);
    const uint32_t *cur = a.cursor + (size_t)td.seg * kRadixBins;
    // reserve the tile's range of every digit (global atomics), but consume the results only after the
    // shared-memory reorder below: their latency overlaps it
    uint32_t g[4], ex4[4];
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const uint32_t d = 4 * t + e;
        toff[d] = ex;
        ex4[e] = ex;
        g[e] = c[e] ? atomicAdd(const_cast<uint32_t *>(cur + d), c[e]) : 0u;
        ex += c[e];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < KPT; r++) {
        const uint32_t i = t + r * kST;
        if (i < td.n) {
            const uint32_t p = toff[digit_reg<KW>(key[r], a.level)] + ((slot[r / 2] >> (16 * (r & 1))) & 0xffffu);
#pragma unroll
            for (int u = 0; u < KW; u++) kout[p * KW + u + ((p * KW + u) >> 5)] = key[r][u];
        }
    }
#pragma unroll
    for (int e = 0; e < 4; e++) gbase[4 * t + e] = g[e] - ex4[e];
    __syncthreads();
    uint32_t *dst = ((sg.buf & 1u) ? a.keys_b : const_cast<uint32_t *>(a.keys_a)) + b.key_off;
    for (uint32_t i = t; i < td.n * KW; i += kST) {
        const uint32_t p = i / KW, u = i - p * KW;
        const uint32_t w = kout[i + (i >> 5)];
        const uint32_t j = p * KW + a.level / 3;   // the element's digit word
        const uint32_t wd = kout[j + (j >> 5)];
        const uint32_t d = (wd >> (20 - 10 * (a.level % 3))) & 1023u;
        dst[(uint64_t)(gbase[d] + p) * KW + u] = w;
    }
}

__global__ void __launch_bounds__(kST, 2) k_msd_scatter(MsdArgs a) {
    extern __shared__ __align__(16) uint32_t sm[];
    const MsdTile td = a.tiles[blockIdx.x];
    if (a.seg_skip[td.seg]) return;   // all its keys share this digit: the segment moves on in place
    const MsdSeg sg = a.segs[td.seg];
    const BucketInfo b = a.buckets[sg.L];
    switch (b.kw) {
        case 1: scatter_tile<1>(a, td, sg, b, sm); break;
        case 2: scatter_tile<2>(a, td, sg, b, sm); break;
        case 3: scatter_tile<3>(a, td, sg, b, sm); break;
        case 4: scatter_tile<4>(a, td, sg, b, sm); break;
        case 5: scatter_tile<5>(a, td, sg, b, sm); break;
        case 6: scatter_tile<6>(a, td, sg, b, sm); break;
        case 7: scatter_tile<7>(a, td, sg, b, sm); break;
        case 8: scatter_tile<8>(a, td, sg, b, sm); break;
        case 9: scatter_tile<9>(a, td, sg, b, sm); break;
        case 10: scatter_tile<10>(a, td, sg, b, sm); break;
        case 11: scatter_tile<11>(a, td, sg, b, sm); break;
        default: break;   // kw > 11 never reaches the scatter: the host sorts such buckets with LSD
    }
}

// Persistent scatter: CTA b takes tiles b, b + grid, ... (skipping those of skipped segments); the next
// tile's keys are fetched by a TMA bulk copy into the other shared-memory buffer while this one is
// scattered, so the tile's loads no longer stall the scatter (the per-tile kernel waits on them).
constexpr uint32_t kScatBuf = 8192 + 8;   // key words of a tile (<= 8192) + the 16-byte alignment slack
__global__ void __launch_bounds__(kST, 2) k_msd_scatter_p(MsdArgs a, uint32_t ntiles) {
    extern __shared__ __align__(128) uint32_t smp[];
    uint32_t *inb = smp;                                                    // [2][kScatBuf]
    uint64_t *bar = reinterpret_cast<uint64_t *>(smp + 2 * kScatBuf);      // [2]
    uint32_t *sj = reinterpret_cast<uint32_t *>(bar + 2);                   // [0..1] tile, [2..3] word offset
    uint32_t *sm = sj + 8;
    auto fetch = [&](uint32_t j, uint32_t b) {   // thread 0
        while (j < ntiles && a.seg_skip[a.tiles[j].seg]) j += gridDim.x;
        sj[b] = j;
        if (j >= ntiles) return;
        const MsdTile td = a.tiles[j];
        const MsdSeg sg = a.segs[td.seg];
        const BucketInfo bk = a.buckets[sg.L];
        const uint32_t *src = ((sg.buf & 1u) ? a.keys_a : a.keys_b) + bk.key_off + (uint64_t)(sg.start + td.off) * bk.kw;
        const uintptr_t s0 = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
        const uintptr_t s1 = (reinterpret_cast<uintptr_t>(src + (size_t)td.n * bk.kw) + 15) & ~(uintptr_t)15;
        sj[2 + b] = (uint32_t)((reinterpret_cast<uintptr_t>(src) - s0) / 4);
        tma::mbar_expect_tx(&bar[b], (uint32_t)(s1 - s0));
        tma::bulk_g2s(inb + b * kScatBuf, reinterpret_cast<const void *>(s0), (uint32_t)(s1 - s0), &bar[b]);
    };
    if (threadIdx.x == 0) {
        tma::mbar_init(&bar[0], 1);
        tma::mbar_init(&bar[1], 1);
        tma::fence_mbar_init();
        fetch(blockIdx.x, 0);
    }
    __syncthreads();
    for (uint32_t it = 0;; it++) {
        const uint32_t cur = it & 1;
        const uint32_t j = sj[cur];
        if (j >= ntiles) break;
        const uint32_t off = sj[2 + cur];
        if (threadIdx.x == 0) fetch(j + gridDim.x, cur ^ 1);   // (buffer cur^1 was released at the last barrier)
        tma::mbar_wait(&bar[cur], (it >> 1) & 1);
        const MsdTile td = a.tiles[j];
        const MsdSeg sg = a.segs[td.seg];
        const BucketInfo b = a.buckets[sg.L];
        const uint32_t *kin = inb + cur * kScatBuf + off;
        switch (b.kw) {
            case 1: scatter_tile<1>(a, td, sg, b, sm, kin); break;
            case 2: scatter_tile<2>(a, td, sg, b, sm, kin); break;
            case 3: scatter_tile<3>(a, td, sg, b, sm, kin); break;
            case 4: scatter_tile<4>(a, td, sg, b, sm, kin); break;
            case 5: scatter_tile<5>(a, td, sg, b, sm, kin); break;
            case 6: scatter_tile<6>(a, td, sg, b, sm, kin); break;
            case 7: scatter_tile<7>(a, td, sg, b, sm, kin); break;
            case 8: scatter_tile<8>(a, td, sg, b, sm, kin); break;
            case 9: scatter_tile<9>(a, td, sg, b, sm, kin); break;
            case 10: scatter_tile<10>(a, td, sg, b, sm, kin); break;
            default: scatter_tile<11>(a, td, sg, b, sm, kin); break;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- level 0 from the staging chunks
// The ingest (K1) leaves the keys of the words of 6..66 letters in word-major chunks of one key-width class
// K (lengths 6K-5 .. 6K), listed per class. Level 0 partitions them by (length, first 2-letter digit) with
// no regrouping pass: a slice is slice_chunks consecutive chunks of one class's list;
//   k_msd_count0    per slice: histogram of its 6 x 1024 (length, digit) bins (shared memory), added to the
//                   per-length segment histograms for k_msd_plan;
//   k_msd_scatter0  persistent over the chunks (TMA double-buffered): bins -> in-chunk offsets (scan), one
//                   global atomic per non-empty bin reserves the chunk's range of that child, keys
//                   reordered by bin in shared memory and written key-major into buffer B.
__device__ __forceinline__ uint32_t key_len0(uint32_t last, uint32_t K) {   // trailing pad codes (0) of the last word
    return 6u * K - (uint32_t)(__ffs(last) - 1) / 5u;
}
struct Slice0 {
    uint32_t K, j0, j1;   // class, list entries [j0, j1)
};
__device__ __forceinline__ Slice0 slice0_of(const MsdArgs &a, uint32_t sl) {
    uint32_t K = 1;
    while (K < kMaxStageKw && a.slice_pfx[K] <= sl) K++;
    const uint32_t j0 = (sl - a.slice_pfx[K - 1]) * a.slice_chunks;
    return Slice0{K, j0, min(a.cls_cnt[K - 1], j0 + a.slice_chunks)};
}

__global__ void __launch_bounds__(kST) k_msd_count0(MsdArgs a) {
    __shared__ uint32_t h[kC0Bins];
    const uint32_t t = threadIdx.x, sl = blockIdx.x;
    const Slice0 sc = slice0_of(a, sl);
    const uint32_t K = sc.K, cap = 1u << chunk_lg(K), L0 = 6u * K - 5u;
    for (uint32_t i = t; i < kC0Bins; i += kST) h[i] = 0;
    __syncthreads();
    const uint32_t *list = a.cls_list + (size_t)(K - 1) * a.cls_cap;
    for (uint32_t j = sc.j0; j < sc.j1; j++) {
        const uint32_t c = __ldg(list + j), n = __ldg(a.chunk_fill + c);
        const uint32_t *r0 = a.pool + (size_t)c * kChunkWords, *rl = r0 + (K - 1) * cap;   // first / last key words
        for (uint32_t i0 = t; i0 < n; i0 += 4 * kST) {
            uint32_t w0[4], wl[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const uint32_t i = i0 + r * kST;
                w0[r] = i < n ? __ldg(r0 + i) : 0u;
                wl[r] = i < n ? __ldg(rl + i) : 1u;
            }
#pragma unroll
            for (int r = 0; r < 4; r++)
                if (i0 + r * kST < n) atomicAdd(&h[((key_len0(wl[r], K) - L0) << 10) | (w0[r] >> 20)], 1u);
        }
    }
    __syncthreads();
    uint32_t *sh = a.slice_hist ? a.slice_hist + (size_t)sl * kC0Bins : nullptr;
    for (uint32_t b = t; b < kC0Bins; b += kST) {
        const uint32_t v = h[b];
        if (sh) sh[b] = v;
        if (v) atomicAdd(&a.hist[(size_t)(L0 + (b >> 10) - a.seg_l0) * kRadixBins + (b & 1023u)], v);
    }
}

#ifndef WSORT_S0_THREADS
#define WSORT_S0_THREADS 512
#endif
constexpr int kS0T = WSORT_S0_THREADS;   // k_msd_scatter0's threads (2 CTAs / SM: 32 warps hide the chunk phases)
constexpr uint32_t kS0PerThread = kC0Bins / kS0T;   // 12 contiguous bins per thread in the scans
static_assert(kS0PerThread % 4 == 0 && kS0T / 32 + 1 <= 32, "scatter0 scan layout");
constexpr uint32_t kS0Kout = kChunkWords + kChunkWords / 32 + 8;
// [2][kChunkWords] TMA buffers | bar[2] | gb[kC0Bins] | off[kC0Bins] | kout | pbin (u16)[kChunkWords] | wsum
constexpr size_t kScatter0Smem = 2 * kChunkWords * 4 + 16 + 2 * kC0Bins * 4 + kS0Kout * 4 + kChunkWords * 2 + 4 * (kS0T / 32 + 1);

#ifndef WSORT_S0_SLICE
#define WSORT_S0_SLICE 1
#endif
#ifndef WSORT_S0_HINT
#define WSORT_S0_HINT 1
#endif
// One chunk of class K: keys -> (bin, slot), exclusive scan of the bins, keys reordered by bin in shared
// memory and written key-major, coalesced within each bin. The chunk's range of each child comes from
//   SLICE: the slice's range (reserved once per slice from k_msd_count0's slice histogram), advanced in
//          shared memory (gb = the next index of each bin);
//   else:  one global atomic per non-empty bin as the chunk is scattered (gb = its range - in-chunk offset).
template <int K, bool SLICE>
__device__ __forceinline__ void scatter0_chunk(const MsdArgs &a, const uint32_t *kin, uint32_t n, uint32_t *gb,
                                               uint32_t *off, uint32_t *kout, uint16_t *pbin, uint32_t *wsum,
                                               uint64_t *koff, uint64_t wpol) {
    constexpr uint32_t cap = 1u << chunk_lg(K), KPT = (cap + kS0T - 1) / kS0T, L0 = 6u * K - 5u;
    const uint32_t t = threadIdx.x;
    if (t < 6) koff[t] = L0 + t >= a.seg_l0 ? a.buckets[L0 + t].key_off : 0;
    uint32_t key[KPT][K], bin[KPT], slot[KPT];
#pragma unroll
    for (uint32_t r = 0; r < KPT; r++) {
        const uint32_t i = t + r * kS0T;
#pragma unroll
        for (int u = 0; u < K; u++) key[r][u] = i < n ? kin[u * cap + i] : 0u;
    }
#pragma unroll
    for (uint32_t r = 0; r < KPT; r++) {
        const uint32_t i = t + r * kS0T;
        bin[r] = ((key_len0(i < n ? key[r][K - 1] : 1u, K) - L0) << 10) | (key[r][0] >> 20);
        slot[r] = i < n ? atomicAdd(&off[bin[r]], 1u) : 0u;
    }
    __syncthreads();
    // exclusive scan of the counts (thread t: bins [24 t, 24 t + 24))
    uint32_t cnt[kS0PerThread], sum = 0;
    uint4 *o4 = reinterpret_cast<uint4 *>(off + kS0PerThread * t);
#pragma unroll
    for (uint32_t q = 0; q < kS0PerThread / 4; q++) {
        const uint4 v = o4[q];
        cnt[4 * q] = v.x;
        cnt[4 * q + 1] = v.y;
        cnt[4 * q + 2] = v.z;
        cnt[4 * q + 3] = v.w;
        sum += v.x + v.y + v.z + v.w;
    }
    uint32_t ex = block_excl_scan_m<kS0T>(sum, wsum, nullptr);   // (its barriers order the reads above before the writes)
    const uint32_t b0 = kS0PerThread * t;
    uint32_t g[SLICE ? 1 : kS0PerThread];
    if (!SLICE) {
#pragma unroll
        for (uint32_t q = 0; q < kS0PerThread; q++) {   // the chunk's range of each non-empty child (issued together)
            const uint32_t b = b0 + q;
            g[q] = cnt[q] ? atomicAdd(&a.cursor[(size_t)(L0 + (b >> 10) - a.seg_l0) * kRadixBins + (b & 1023u)], cnt[q]) : 0u;
        }
    }
    uint4 *g4 = reinterpret_cast<uint4 *>(gb + b0);
#pragma unroll
    for (uint32_t q = 0; q < kS0PerThread / 4; q++) {
        uint4 v;
        v.x = ex;
        ex += cnt[4 * q];
        v.y = ex;
        ex += cnt[4 * q + 1];
        v.z = ex;
        ex += cnt[4 * q + 2];
        v.w = ex;
        ex += cnt[4 * q + 3];
        o4[q] = v;
        uint4 r = g4[q];   // key p of bin b goes to bucket index gb[b] + p
        if (SLICE) r = make_uint4(r.x - v.x, r.y - v.y, r.z - v.z, r.w - v.w);
        else r = make_uint4(g[4 * q] - v.x, g[4 * q + 1] - v.y, g[4 * q + 2] - v.z, g[4 * q + 3] - v.w);
        g4[q] = r;
    }
    __syncthreads();
    // reorder by bin in shared memory (key-major, padded)
#pragma unroll
    for (uint32_t r = 0; r < KPT; r++) {
        const uint32_t i = t + r * kS0T;
        if (i < n) {
            const uint32_t p = off[bin[r]] + slot[r];
#pragma unroll
            for (int u = 0; u < K; u++) {
                const uint32_t w = p * K + u;
                kout[w + (w >> 5)] = key[r][u];
            }
            pbin[p] = (uint16_t)bin[r];
        }
    }
    __syncthreads();
    for (uint32_t i = t; i < n * K; i += kS0T) {
        const uint32_t p = i / K, u = i - p * K, b = pbin[p];
        uint32_t *dst = a.keys_b + koff[b >> 10] + (uint64_t)(gb[b] + p) * K + u;
#if WSORT_S0_HINT
        tma::st_hint(dst, kout[i + (i >> 5)], wpol);
#else
        (void)wpol;
        *dst = kout[i + (i >> 5)];
#endif
    }
    __syncthreads();
#pragma unroll
    for (uint32_t q = 0; q < kS0PerThread / 4; q++) {
        if (SLICE) {   // the slice's next chunk continues after these keys
            uint4 r = g4[q];
            const uint4 v = o4[q];
            r = make_uint4(r.x + v.x + cnt[4 * q], r.y + v.y + cnt[4 * q + 1], r.z + v.z + cnt[4 * q + 2],
                           r.w + v.w + cnt[4 * q + 3]);
            g4[q] = r;
        }
        o4[q] = make_uint4(0, 0, 0, 0);   // (the next chunk's counts)
    }
}

// SLICE (default): CTA = one slice of k_msd_count0 (its chunks in list order), its ranges reserved first;
// else persistent over the classes' lists concatenated (CTA b: chunks b, b + grid, ...). The next chunk is
// fetched by a TMA bulk copy (evict-first: read once) into the other buffer while this one is scattered;
// the scattered keys are stored evict-last (the sectors a later chunk completes stay in L2).
__global__ void __launch_bounds__(kS0T, 2) k_msd_scatter0(MsdArgs a, uint32_t total) {
    extern __shared__ __align__(128) uint32_t s0m[];
    uint32_t *inb = s0m;                                                      // [2][kChunkWords]
    uint64_t *bar = reinterpret_cast<uint64_t *>(s0m + 2 * kChunkWords);     // [2]
    uint32_t *gb = reinterpret_cast<uint32_t *>(bar + 2);                     // [kC0Bins]
    uint32_t *off = gb + kC0Bins;                                             // [kC0Bins] counts / offsets
    uint32_t *kout = off + kC0Bins;
    uint16_t *pbin = reinterpret_cast<uint16_t *>(kout + kS0Kout);
    uint32_t *wsum = reinterpret_cast<uint32_t *>(pbin + kChunkWords);        // [kS0T / 32 + 1]
    __shared__ uint64_t koff[6];
    __shared__ uint32_t s_n[2], s_k[2];
    const uint32_t t = threadIdx.x;
    const bool slice = WSORT_S0_SLICE;
    const uint64_t rpol = tma::policy_evict_first(), wpol = tma::policy_evict_last();
    uint32_t j0 = blockIdx.x, j1 = total, step = gridDim.x;
    if (slice) {   // this slice's chunks: class K's list entries [j0, j1) -> concatenated indices
        const Slice0 sc = slice0_of(a, blockIdx.x);
        j0 = a.cls_pfx[sc.K - 1] + sc.j0;
        j1 = a.cls_pfx[sc.K - 1] + sc.j1;
        step = 1;
    }
    auto fetch = [&](uint32_t j, uint32_t b) {   // thread 0: chunk j of the concatenated lists -> buffer b
        uint32_t K = 1;
        while (K < kMaxStageKw && a.cls_pfx[K] <= j) K++;
        const uint32_t c = __ldg(a.cls_list + (size_t)(K - 1) * a.cls_cap + (j - a.cls_pfx[K - 1]));
        const uint32_t n = __ldg(a.chunk_fill + c);
        const uint32_t bytes = (((K - 1u) << chunk_lg(K)) * 4u + n * 4u + 15u) & ~15u;   // (word-major: full rows, then the last)
        s_n[b] = n;
        s_k[b] = K;
        tma::mbar_expect_tx(&bar[b], bytes);
#if WSORT_S0_HINT
        tma::bulk_g2s_hint(inb + b * kChunkWords, a.pool + (size_t)c * kChunkWords, bytes, &bar[b], rpol);
#else
        tma::bulk_g2s(inb + b * kChunkWords, a.pool + (size_t)c * kChunkWords, bytes, &bar[b]);
#endif
    };
    if (t == 0) {
        tma::mbar_init(&bar[0], 1);
        tma::mbar_init(&bar[1], 1);
        tma::fence_mbar_init();
        if (j0 < j1) fetch(j0, 0);
    }
    if (slice) {   // the slice's range of every non-empty (length, digit) child: one global atomic per bin
        const Slice0 sc = slice0_of(a, blockIdx.x);
        const uint32_t L0 = 6u * sc.K - 5u;
        const uint32_t *sh = a.slice_hist + (size_t)blockIdx.x * kC0Bins;
        uint32_t v[kS0PerThread], g[kS0PerThread];   // (all loads, then all atomics in flight together)
#pragma unroll
        for (uint32_t r = 0; r < kS0PerThread; r++) v[r] = __ldg(sh + t + r * kS0T);
#pragma unroll
        for (uint32_t r = 0; r < kS0PerThread; r++) {
            const uint32_t b = t + r * kS0T;
            g[r] = v[r] ? atomicAdd(&a.cursor[(size_t)(L0 + (b >> 10) - a.seg_l0) * kRadixBins + (b & 1023u)], v[r]) : 0u;
        }
#pragma unroll
        for (uint32_t r = 0; r < kS0PerThread; r++) gb[t + r * kS0T] = g[r];
    }
    for (uint32_t b = t; b < kC0Bins; b += kS0T) off[b] = 0;
    __syncthreads();
    for (uint32_t j = j0, it = 0; j < j1; j += step, it++) {
        const uint32_t cur = it & 1;
        if (t == 0 && j + step < j1) fetch(j + step, cur ^ 1);   // (buffer cur^1 was released at the last barrier)
        tma::mbar_wait(&bar[cur], (it >> 1) & 1);
        const uint32_t n = s_n[cur], K = s_k[cur];
        const uint32_t *kin = inb + cur * kChunkWords;
#define S0CASE(KK) \
    case KK: \
        if (slice) scatter0_chunk<KK, true>(a, kin, n, gb, off, kout, pbin, wsum, koff, wpol); \
        else scatter0_chunk<KK, false>(a, kin, n, gb, off, kout, pbin, wsum, koff, wpol); \
        break;
        switch (K) {
            S0CASE(1) S0CASE(2) S0CASE(3) S0CASE(4) S0CASE(5) S0CASE(6) S0CASE(7) S0CASE(8) S0CASE(9) S0CASE(10)
            default: if (slice) scatter0_chunk<11, true>(a, kin, n, gb, off, kout, pbin, wsum, koff, wpol);
                     else scatter0_chunk<11, false>(a, kin, n, gb, off, kout, pbin, wsum, koff, wpol);
                     break;
        }
#undef S0CASE
        __syncthreads();   // every bin's count cleared (and its next index advanced) before the next chunk's atomics
    }
}

// ---------------------------------------------------------------- finishing sorts
// One warp per tiny segment (<= 32 keys): odd-even transposition over the lanes, one key per lane,
// compare-exchange with the neighbouring lane through shuffles (32 phases).
template <int KW>
__device__ __forceinline__ void warp_oets(const MsdArgs &a, const MsdSeg &sg, const BucketInfo &b) {
    const int lane = threadIdx.x & 31;
    const uint32_t *src = ((sg.buf & 1u) ? a.keys_a : a.keys_b) + b.key_off + (uint64_t)sg.start * KW;
    uint32_t k[KW];
#pragma unroll
    for (int u = 0; u < KW; u++) k[u] = lane < (int)sg.n ? __ldg(src + lane * KW + u) : 0xffffffffu;
    for (int ph = 0; ph < 32; ph++) {
        const bool lower = (lane & 1) == (ph & 1);
        const int partner = lower ? lane + 1 : lane - 1;
        const bool act = partner >= 0 && partner < 32;
        uint32_t o[KW];
#pragma unroll
        for (int u = 0; u < KW; u++) o[u] = __shfl_sync(kFullM, k[u], act ? partner : lane);
        bool less = false, eq = true;   // o < k ?
#pragma unroll
        for (int u = 0; u < KW; u++) {
            if (eq && o[u] != k[u]) {
                less = o[u] < k[u];
                eq = false;
            }
        }
        const bool take = act && (lower ? less : (!less && !eq));
        if (take) {
#pragma unroll
            for (int u = 0; u < KW; u++) k[u] = o[u];
        }
    }
    uint32_t *dst = a.keys_b + b.key_off + (uint64_t)sg.start * KW;
    if (lane < (int)sg.n) {
#pragma unroll
        for (int u = 0; u < KW; u++) dst[lane * KW + u] = k[u];
    }
}

__global__ void __launch_bounds__(kST) k_msd_warp_sort(MsdArgs a) {
    const uint32_t w = blockIdx.x * (kST / 32) + (threadIdx.x >> 5);
    if (w >= a.n_tiny) return;
    const MsdSeg sg = a.q_tiny[w];
    const BucketInfo b = a.buckets[sg.L];
    switch (b.kw) {
        case 1: warp_oets<1>(a, sg, b); break;
        case 2: warp_oets<2>(a, sg, b); break;
        case 3: warp_oets<3>(a, sg, b); break;
        case 4: warp_oets<4>(a, sg, b); break;
        case 5: warp_oets<5>(a, sg, b); break;
        case 6: warp_oets<6>(a, sg, b); break;
        case 7: warp_oets<7>(a, sg, b); break;
        case 8: warp_oets<8>(a, sg, b); break;
        case 9: warp_oets<9>(a, sg, b); break;
        case 10: warp_oets<10>(a, sg, b); break;
        default: warp_oets<11>(a, sg, b); break;
    }
}

// Keys of KW u32 words held in registers, compared lexicographically.
template <int KW>
struct Key {
    uint32_t w[KW];
};
template <int KW>
__device__ __forceinline__ bool klt(const Key<KW> &x, const Key<KW> &y) {
    if constexpr (KW == 1) {
        return x.w[0] < y.w[0];
    } else if constexpr (KW == 2) {
        return (((uint64_t)x.w[0] << 32) | x.w[1]) < (((uint64_t)y.w[0] << 32) | y.w[1]);
    } else {
#pragma unroll
        for (int u = 0; u < KW; u++)
            if (x.w[u] != y.w[u]) return x.w[u] < y.w[u];
        return false;
    }
}
template <int KW>
__device__ __forceinline__ void kce(Key<KW> &x, Key<KW> &y) {   // compare-exchange: x <= y afterwards
    const bool sw = klt<KW>(y, x);
#pragma unroll
    for (int u = 0; u < KW; u++) {   // branch-free select
        const uint32_t a = x.w[u], b = y.w[u];
        x.w[u] = sw ? b : a;
        y.w[u] = sw ? a : b;
    }
}
template <int KW>
__device__ __forceinline__ Key<KW> kshfl(const Key<KW> &x, int src) {
    Key<KW> r;
#pragma unroll
    for (int u = 0; u < KW; u++) r.w[u] = __shfl_sync(kFullM, x.w[u], src);
    return r;
}
template <int KW>
__device__ __forceinline__ Key<KW> kld(const uint32_t *p) {
    Key<KW> r;
#pragma unroll
    for (int u = 0; u < KW; u++) r.w[u] = p[u];
    return r;
}
template <int KW>
__device__ __forceinline__ void kst(uint32_t *p, const Key<KW> &x) {
#pragma unroll
    for (int u = 0; u < KW; u++) p[u] = x.w[u];
}

// One CTA per small job (<= 256*E keys of one bucket): odd-even transposition inside each thread's
// E keys (the data-parallel bubble sort), odd-even merge-split across groups of 8 lanes through warp
// shuffles (min/max against the reversed partner run + bitonic clean-up), then merge paths in
// shared memory up to the whole tile. Keys stay in registers until the shared-memory merges.
template <int KW, int E = (KW <= 4 ? kFinE : 4)>
__device__ __forceinline__ void cta_sort_job(const MsdArgs &a, const MsdSeg &sg, const BucketInfo &b, uint32_t *sm) {
    constexpr uint32_t TN = kST * E;
    const int t = threadIdx.x, lane = t & 31;
    const uint32_t n = sg.n;
    const uint32_t *src = ((sg.buf & 1u) ? a.keys_a : a.keys_b) + b.key_off + (uint64_t)sg.start * KW;
    Key<KW> v[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t idx = t * E + e;
        if (idx < n) v[e] = kld<KW>(src + (size_t)idx * KW);
        else
#pragma unroll
            for (int u = 0; u < KW; u++) v[e].w[u] = 0xffffffffu;
    }
#pragma unroll
    for (int ph = 0; ph < E; ph++)
#pragma unroll
        for (int i = ph & 1; i + 1 < E; i += 2) kce<KW>(v[i], v[i + 1]);
    const int g = lane & 7;
#pragma unroll 1
    for (int ph = 0; ph < 8; ph++) {
        const bool lower = (g & 1) == (ph & 1);
        const int pg = lower ? g + 1 : g - 1;
        const bool act = pg >= 0 && pg < 8;
        const int srcl = act ? lane - g + pg : lane;
        Key<KW> o[E];
#pragma unroll
        for (int e = 0; e < E; e++) o[e] = kshfl<KW>(v[e], srcl);
        if (act) {
#pragma unroll
            for (int e = 0; e < E; e++) {
                const Key<KW> &y = o[E - 1 - e];
                const bool ylt = klt<KW>(y, v[e]);
                if (lower ? ylt : !ylt) v[e] = y;
            }
#pragma unroll
            for (int d = E / 2; d >= 1; d >>= 1)
#pragma unroll
                for (int i = 0; i < E; i++)
                    if ((i & d) == 0) kce<KW>(v[i], v[i + d]);
        }
    }
    // shared memory: two padded buffers (word w at w + w/32: conflict-free blocked access)
    constexpr uint32_t PW = TN * KW + TN * KW / 32 + 1;
    uint32_t *b0 = sm, *b1 = sm + PW;
    auto lds = [](const uint32_t *base, uint32_t elem) {
        Key<KW> r;
#pragma unroll
        for (int u = 0; u < KW; u++) {
            const uint32_t w = elem * KW + u;
            r.w[u] = base[w + (w >> 5)];
        }
        return r;
    };
    auto sts = [](uint32_t *base, uint32_t elem, const Key<KW> &x) {
#pragma unroll
        for (int u = 0; u < KW; u++) {
            const uint32_t w = elem * KW + u;
            base[w + (w >> 5)] = x.w[u];
        }
    };
#pragma unroll
    for (int e = 0; e < E; e++) sts(b0, t * E + e, v[e]);
    __syncthreads();
    uint32_t *s0 = b0, *s1 = b1;
    for (uint32_t run = 8 * E; run < TN; run *= 2) {
        const uint32_t o = t * E, pair = o / (2 * run), d = o - pair * 2 * run;
        const uint32_t ra = pair * 2 * run, rb = ra + run;   // element indices
        uint32_t lo = d > run ? d - run : 0u, hi = d < run ? d : run;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (!klt<KW>(lds(s0, rb + d - 1 - mid), lds(s0, ra + mid))) lo = mid + 1;
            else hi = mid;
        }
        uint32_t i = lo, j = d - lo;
        Key<KW> x = lds(s0, ra + min(i, run - 1)), y = lds(s0, rb + min(j, run - 1));
#pragma unroll
        for (int k = 0; k < E; k++) {
            const bool take_a = j >= run || (i < run && !klt<KW>(y, x));
            if (take_a) {
                sts(s1, o + k, x);
                i++;
                if (i < run) x = lds(s0, ra + i);
            } else {
                sts(s1, o + k, y);
                j++;
                if (j < run) y = lds(s0, rb + j);
            }
        }
        __syncthreads();
        uint32_t *sw = s0;
        s0 = s1;
        s1 = sw;
    }
    uint32_t *dst = a.keys_b + b.key_off + (uint64_t)sg.start * KW;
    for (uint32_t i = t; i < n * KW; i += kST) dst[i] = s0[i + (i >> 5)];
}

// Local LSD radix finish (optional): a job's keys share the digits above `level` (a job packs
// consecutive children of one segment, which differ first at digit `level`), so sorting it by
// digits ndig-1 .. level (least significant first) sorts it. Each 10-bit digit is two stable 5-bit
// counting sub-passes over the tile in shared memory: thread-private 16-bit counters over 32 bins,
// one block scan, scatter (blocked key ownership keeps the order stable).
__device__ __forceinline__ uint32_t padm(uint32_t i) { return i + (i >> 5); }

template <int KW>
__device__ __forceinline__ void radix_job(const MsdArgs &a, const MsdSeg &sg, const BucketInfo &b, uint32_t *sm) {
    constexpr int KPT = 8;                         // keys per thread (blocked)
    constexpr uint32_t TN = kST * KPT;             // 2048 = CTA-sort capacity for kw <= 4
    const int t = threadIdx.x;
    const uint32_t n = sg.n, level = sg.buf >> 8;
    const uint32_t *src = ((sg.buf & 1u) ? a.keys_a : a.keys_b) + b.key_off + (uint64_t)sg.start * KW;
    constexpr uint32_t PW = TN * KW + TN * KW / 32 + 1;
    uint32_t *A = sm, *B = sm + PW;
    uint32_t *cnt = B + PW;                        // 32 bins x 256 threads, u32, padded
    uint32_t *wsum = cnt + 32 * kST + 32 * kST / 32 + 1;
    for (uint32_t i = t; i < TN * KW; i += kST) A[padm(i)] = i < n * KW ? __ldg(src + i) : 0xffffffffu;
    __syncthreads();
    for (int q = (int)b.ndig - 1; q >= (int)level; q--) {
        const uint32_t wi = q / 3, sh = 20 - 10 * (q % 3);
        for (int half = 0; half < 2; half++) {
            const uint32_t fs = sh + (half ? 5 : 0);   // 5-bit field: low letter first
            uint32_t key[KPT][KW], rk[KPT];
#pragma unroll
            for (int f = 0; f < 32; f++) cnt[padm(f * kST + t)] = 0;
#pragma unroll
            for (int k = 0; k < KPT; k++) {
#pragma unroll
                for (int u = 0; u < KW; u++) key[k][u] = A[padm((t * KPT + k) * KW + u)];
                uint32_t w = key[k][0];
#pragma unroll
                for (int u = 1; u < KW; u++) w = wi == (uint32_t)u ? key[k][u] : w;
                const uint32_t f = (w >> fs) & 31u;
                uint32_t *cp = cnt + padm(f * kST + t);
                rk[k] = *cp;
                *cp = rk[k] + 1;
            }
            __syncthreads();
            {   // exclusive scan in (bin, thread) order; thread t owns linear entries [32t, 32t+32)
                uint32_t sum = 0;
#pragma unroll
                for (int i = 0; i < 32; i++) sum += cnt[padm(32 * t + i)];
                uint32_t run = block_excl_scan_m(sum, wsum, nullptr);
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    const uint32_t x = cnt[padm(32 * t + i)];
                    cnt[padm(32 * t + i)] = run;
                    run += x;
                }
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < KPT; k++) {
                uint32_t w = key[k][0];
#pragma unroll
                for (int u = 1; u < KW; u++) w = wi == (uint32_t)u ? key[k][u] : w;
                const uint32_t pos = cnt[padm(((w >> fs) & 31u) * kST + t)] + rk[k];
#pragma unroll
                for (int u = 0; u < KW; u++) B[padm(pos * KW + u)] = key[k][u];
            }
            __syncthreads();
            uint32_t *sw = A;
            A = B;
            B = sw;
        }
    }
    uint32_t *dst = a.keys_b + b.key_off + (uint64_t)sg.start * KW;
    for (uint32_t i = t; i < n * KW; i += kST) dst[i] = A[padm(i)];
}

__global__ void __launch_bounds__(kST) k_msd_radix_job(MsdArgs a) {
    extern __shared__ __align__(16) uint32_t sm[];
    const MsdSeg sg = a.q_small[blockIdx.x];
    const BucketInfo b = a.buckets[sg.L];
    switch (b.kw) {
        case 1: radix_job<1>(a, sg, b, sm); break;
        case 2: radix_job<2>(a, sg, b, sm); break;
        case 3: radix_job<3>(a, sg, b, sm); break;
        case 4: radix_job<4>(a, sg, b, sm); break;
        default: break;   // wider keys use the odd-even transposition finish
    }
}

__global__ void __launch_bounds__(kST) k_msd_cta_sort(MsdArgs a) {
    extern __shared__ __align__(16) uint32_t sm[];
    const MsdSeg sg = a.q_small[blockIdx.x];
    const BucketInfo b = a.buckets[sg.L];
    if (a.finish_radix && b.kw <= 4) return;   // done by k_msd_radix_job
    switch (b.kw) {
        case 1: cta_sort_job<1>(a, sg, b, sm); break;
        case 2: cta_sort_job<2>(a, sg, b, sm); break;
        case 3: cta_sort_job<3>(a, sg, b, sm); break;
        case 4: cta_sort_job<4>(a, sg, b, sm); break;
        case 5: cta_sort_job<5>(a, sg, b, sm); break;
        case 6: cta_sort_job<6>(a, sg, b, sm); break;
        case 7: cta_sort_job<7>(a, sg, b, sm); break;
        case 8: cta_sort_job<8>(a, sg, b, sm); break;
        case 9: cta_sort_job<9, 1>(a, sg, b, sm); break;    // (tile_keys 256 for > 8 key words)
        case 10: cta_sort_job<10, 1>(a, sg, b, sm); break;
        default: cta_sort_job<11, 1>(a, sg, b, sm); break;
    }
}

// Keys of 1 or 2 words as one native integer (u32 / u64: word 0 is the most significant), so one
// compare decides the order. One CTA per small job (<= 2048 keys): each thread sorts its 8 keys in
// registers by odd-even transposition (the data-parallel bubble sort of PAPER.md:23), then merge-path
// passes in shared memory merge the runs 8 -> 16 -> ... up to the job (the paper's merge).
template <typename T, int KW>
__device__ __forceinline__ T fin_load(const uint32_t *p) {
    if constexpr (KW == 1) return p[0];
    else return ((uint64_t)p[0] << 32) | p[1];
}
template <typename T, int KW>
__device__ __forceinline__ void fin_store(uint32_t *p, T v) {
    if constexpr (KW == 1) {
        p[0] = (uint32_t)v;
    } else {
        p[0] = (uint32_t)(v >> 32);
        p[1] = (uint32_t)v;
    }
}
__device__ __forceinline__ uint32_t fpad(uint32_t i) { return i + (i >> 4); }   // bank spreading

// Sort n <= 2048 keys of type T held in shared memory A (padded layout), using B as scratch: each
// thread sorts its 8 keys in registers by odd-even transposition (the data-parallel bubble sort of
// PAPER.md:23), then merge-path passes merge the runs 8 -> 16 -> ... up to n (the paper's merge,
// PAPER.md:76). Returns the buffer holding the sorted keys. All threads of the CTA must call it.
template <typename T>
__device__ __forceinline__ T *block_sort_smem(T *A, T *B, uint32_t n) {
    constexpr int E = 8;
    const T kMax = ~(T)0;   // above every key (key words are < 2^30)
    const uint32_t t = threadIdx.x;
    uint32_t span = E;
    while (span < n) span *= 2;   // only [0, span) is touched: A and B need fpad(span) entries
    const bool mine = t * E < span;
    T v[E];
    __syncthreads();   // A was filled by other threads
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t idx = t * E + e;
        v[e] = idx < n ? A[fpad(idx)] : kMax;
    }
#pragma unroll
    for (int ph = 0; ph < E; ph++)
#pragma unroll
        for (int i = ph & 1; i + 1 < E; i += 2) {
            const T x = v[i], y = v[i + 1];
            v[i] = x < y ? x : y;
            v[i + 1] = x < y ? y : x;
        }
    __syncthreads();   // (A is read above and rewritten below)
    if (mine)
#pragma unroll
        for (int e = 0; e < E; e++) A[fpad(t * E + e)] = v[e];
    __syncthreads();
    for (uint32_t run = E; run < span; run *= 2) {
        const uint32_t o = t * E;
        if (o < span) {
            const uint32_t ra = (o / (2 * run)) * 2 * run, rb = ra + run, d = o - ra;
            uint32_t lo = d > run ? d - run : 0u, hi = d < run ? d : run;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (A[fpad(ra + mid)] <= A[fpad(rb + d - 1 - mid)]) lo = mid + 1;
                else hi = mid;
            }
            uint32_t i = lo, j = d - lo;
            T x = i < run ? A[fpad(ra + i)] : kMax, y = j < run ? A[fpad(rb + j)] : kMax;
#pragma unroll
            for (int k = 0; k < E; k++) {
                const bool tx = j >= run || (i < run && x <= y);
                B[fpad(o + k)] = tx ? x : y;
                if (tx) {
                    i++;
                    x = i < run ? A[fpad(ra + i)] : kMax;
                } else {
                    j++;
                    y = j < run ? A[fpad(rb + j)] : kMax;
                }
            }
        }
        __syncthreads();
        T *sw = A;
        A = B;
        B = sw;
    }
    return A;
}

// block_sort_smem for u32 indices ordered by a comparator lt(a, b) ("key a < key b"): odd-even
// transposition of each thread's 8 indices in registers, then merge-path passes in shared memory.
template <class Lt>
__device__ __forceinline__ uint32_t *block_sort_idx(uint32_t *A, uint32_t *B, uint32_t n, Lt lt) {
    constexpr int E = 8;
    const uint32_t kPad = 0xffffffffu;   // sorts after every index
    auto less = [&](uint32_t x, uint32_t y) { return y == kPad ? x != kPad : (x == kPad ? false : lt(x, y)); };
    const uint32_t t = threadIdx.x;
    uint32_t span = E;
    while (span < n) span *= 2;
    const bool mine = t * E < span;
    uint32_t v[E];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t idx = t * E + e;
        v[e] = idx < n ? A[fpad(idx)] : kPad;
    }
    if (mine)
#pragma unroll
        for (int ph = 0; ph < E; ph++)
#pragma unroll
            for (int i = ph & 1; i + 1 < E; i += 2) {
                const uint32_t x = v[i], y = v[i + 1];
                const bool sw = less(y, x);
                v[i] = sw ? y : x;
                v[i + 1] = sw ? x : y;
            }
    __syncthreads();
    if (mine)
#pragma unroll
        for (int e = 0; e < E; e++) A[fpad(t * E + e)] = v[e];
    __syncthreads();
    for (uint32_t run = E; run < span; run *= 2) {
        const uint32_t o = t * E;
        if (o < span) {
            const uint32_t ra = (o / (2 * run)) * 2 * run, rb = ra + run, d = o - ra;
            uint32_t lo = d > run ? d - run : 0u, hi = d < run ? d : run;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (!less(A[fpad(rb + d - 1 - mid)], A[fpad(ra + mid)])) lo = mid + 1;
                else hi = mid;
            }
            uint32_t i = lo, j = d - lo;
            uint32_t x = i < run ? A[fpad(ra + i)] : kPad, y = j < run ? A[fpad(rb + j)] : kPad;
#pragma unroll
            for (int k = 0; k < E; k++) {
                const bool tx = j >= run || (i < run && !less(y, x));
                B[fpad(o + k)] = tx ? x : y;
                if (tx) {
                    i++;
                    x = i < run ? A[fpad(ra + i)] : kPad;
                } else {
                    j++;
                    y = j < run ? A[fpad(rb + j)] : kPad;
                }
            }
        }
        __syncthreads();
        uint32_t *sw = A;
        A = B;
        B = sw;
    }
    return A;
}

// K5 fused into the finish (streaming mode): write the text of a finished job — word i of the job
// (bucket L, first word `start`) is `word_of(i)`'s letters + '\n' at byte_off[L] + (start + i)(L + 1)
// (reading A12). Pieces of kFinStage bytes are built in shared memory at the destination's 16-byte
// phase and stored with aligned 16-byte stores.
constexpr uint32_t kFinStage = 8192;   // text bytes staged per piece (+32: the 16-byte phase)
template <int KW, class WordOf>
__device__ __forceinline__ void emit_job_text(const MsdArgs &a, const BucketInfo &b, uint32_t L, uint32_t start, uint32_t n,
                                              uint8_t *stage, WordOf word_of) {
    const uint32_t t = threadIdx.x;
    const uint32_t te = kFinStage / (L + 1);
    for (uint32_t w0 = 0; w0 < n; w0 += te) {
        const uint32_t nk = min(te, n - w0);
        const uint64_t ob = b.byte_off + (uint64_t)(start + w0) * (L + 1);
        const uint32_t head = (uint32_t)(ob & 15u);
        for (uint32_t k = t; k < nk; k += kST) {
            uint32_t key[KW];
            word_of(w0 + k, key);
            uint8_t *o = stage + head + k * (L + 1);
#pragma unroll
            for (int q = 0; q < KW; q++) {
#pragma unroll
                for (int j = 0; j < 6; j++) {
                    const uint32_t li = q * 6 + j;
                    if (li < L) o[li] = (uint8_t)(((key[q] >> (25 - 5 * j)) & 31u) | 0x60u);
                }
            }
            o[L] = '\n';
        }
        __syncthreads();
        const uint64_t end = ob + (uint64_t)nk * (L + 1);
        const uint64_t a0 = (ob + 15) & ~15ull, a1 = end & ~15ull;
        if (a0 >= a1) {
            for (uint64_t x = ob + t; x < end; x += kST) a.words[x] = stage[head + (x - ob)];
        } else {
            for (uint64_t x = ob + t; x < a0; x += kST) a.words[x] = stage[head + (x - ob)];
            for (uint64_t x = a1 + t; x < end; x += kST) a.words[x] = stage[head + (x - ob)];
            const uint64_t base16 = ob & ~15ull;
            uint4 *dst = reinterpret_cast<uint4 *>(a.words);
            for (uint64_t x = a0 + 16ull * t; x < a1; x += 16ull * kST)
                dst[x >> 4] = *reinterpret_cast<const uint4 *>(stage + (x - base16));
        }
        __syncthreads();
    }
}

// index of the run holding output word j: first i with ends[i] > j
__device__ __forceinline__ uint32_t run_of(const uint32_t *ends, uint32_t nd, uint32_t j) {
    uint32_t lo = 0, hi = nd - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ends[mid] > j) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// Text of a job made of runs (the streaming finish): distinct word r (sorted) occupies output words
// [ends[r-1], ends[r]). Its text `letters\n` is laid out repeated in R[r] (W bytes, W >= L+1+16), so
// the 16 output bytes starting at phase f of the pattern are R[r][f .. f+16). Aligned 16-byte chunks
// of the job's byte range are written straight to global memory (one warp takes a contiguous range of
// chunks, so each lane's run index only moves forward); a chunk that crosses run boundaries merges the
// windows of each run's pattern (the next run's word starts at the boundary: its window begins at phase
// -boundary mod L+1) with byte masks; the unaligned head / tail bytes are assembled byte by byte.
__device__ __forceinline__ uint32_t div_by(uint32_t n, uint32_t d, uint32_t m) {   // n / d, m = 2^32/d + 1
    uint32_t q = __umulhi(n, m);
    if ((q + 1) * d <= n) q++;
    if (q * d > n) q--;
    return q;
}
__device__ __forceinline__ uint8_t run_byte(const uint8_t *R, uint32_t W, const uint32_t *ends, uint32_t nd, uint32_t L1,
                                            uint32_t rel, uint32_t m) {
    const uint32_t w = div_by(rel, L1, m);
    const uint32_t r = run_of(ends, nd, w);
    return R[r * W + (rel - w * L1)];
}
__device__ __forceinline__ void emit_runs_text(const MsdArgs &a, const BucketInfo &b, uint32_t L, uint32_t start, uint32_t n,
                                               const uint8_t *R, uint32_t W, const uint32_t *ends, uint32_t nd) {
    const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t L1 = L + 1, m = 0xffffffffu / L1 + 1u;   // (2^32 / L1 or 2^32 / L1 + 1: div_by corrects by 1)
    const uint64_t B0 = b.byte_off + (uint64_t)start * L1, B1 = B0 + (uint64_t)n * L1;
    const uint64_t A0 = (B0 + 15) & ~15ull, A1 = B1 & ~15ull;
    if (A0 >= A1) {
        for (uint64_t x = B0 + t; x < B1; x += kST) a.words[x] = run_byte(R, W, ends, nd, L1, (uint32_t)(x - B0), m);
        return;
    }
    if (t < A0 - B0) a.words[B0 + t] = run_byte(R, W, ends, nd, L1, t, m);
    if (t < B1 - A1) a.words[A1 + t] = run_byte(R, W, ends, nd, L1, (uint32_t)(A1 - B0) + t, m);
    const uint32_t nch = (uint32_t)((A1 - A0) >> 4);
    const uint32_t per = (nch + (kST / 32) - 1) / (kST / 32);   // chunks per warp (contiguous)
    const uint32_t c0 = warp * per, c1 = min(c0 + per, nch);
    uint32_t r = 0;
    bool first = true;
    uint4 *dst = reinterpret_cast<uint4 *>(a.words + A0);
    const uint32_t rel0 = (uint32_t)(A0 - B0);
    for (uint32_t c = c0 + lane; c < c1; c += 32) {
        const uint32_t rel = rel0 + 16 * c;
        const uint32_t w = div_by(rel, L1, m), f = rel - w * L1;
        if (first) {
            r = run_of(ends, nd, w);
            first = false;
        } else {
            while (ends[r] <= w) r++;
        }
        const uint32_t wl = div_by(rel + 15, L1, m);
        // 16 bytes of run r's repeated pattern from phase f
        uint32_t v[4];
        auto window = [&](uint32_t run, uint32_t ph, uint32_t (&o)[4]) {
            const uint8_t *p = R + run * W + ph;
            const uint32_t al = (uint32_t)(reinterpret_cast<uintptr_t>(p) & 3u);
            const uint32_t *p4 = reinterpret_cast<const uint32_t *>(p - al);
            const uint32_t x0 = p4[0], x1 = p4[1], x2 = p4[2], x3 = p4[3], x4 = p4[4];
            o[0] = __funnelshift_r(x0, x1, 8 * al);
            o[1] = __funnelshift_r(x1, x2, 8 * al);
            o[2] = __funnelshift_r(x2, x3, 8 * al);
            o[3] = __funnelshift_r(x3, x4, 8 * al);
        };
        window(r, f, v);
        if (wl >= ends[r]) {   // crosses run boundaries: from byte nb on, the next run's window, whose
            uint32_t rr = r;   // word starts at nb (phase -nb mod L1), merged in by byte masks
            uint32_t nb = (ends[r] - w) * L1 - f;
            while (nb < 16u) {
                const uint32_t wb = ends[rr];
                rr++;
                uint32_t ph = nb;
                while (ph >= L1) ph -= L1;
                ph = ph ? L1 - ph : 0u;
                uint32_t o[4];
                window(rr, ph, o);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const uint32_t lo = 4u * q;
                    const uint32_t keep = nb >= lo + 4u ? 0xffffffffu : nb <= lo ? 0u : (1u << (8u * (nb - lo))) - 1u;
                    v[q] = (v[q] & keep) | (o[q] & ~keep);
                }
                nb += (ends[rr] - wb) * L1;
            }
        }
        dst[c] = make_uint4(v[0], v[1], v[2], v[3]);
    }
}

// Lay out distinct word r's text repeated in R[r] (W bytes): pattern byte i = letter i (i < L) or '\n'.
template <int KW, class KeyOf>
__device__ __forceinline__ void build_run_patterns(uint8_t *R, uint32_t W, uint32_t L, uint32_t nd, KeyOf key_of) {
    for (uint32_t r = threadIdx.x; r < nd; r += kST) {
        uint32_t k[KW];
        key_of(r, k);
        uint8_t pat[6 * KW + 1];
#pragma unroll
        for (int q = 0; q < KW; q++)
#pragma unroll
            for (int j = 0; j < 6; j++) pat[q * 6 + j] = (uint8_t)(((k[q] >> (25 - 5 * j)) & 31u) | 0x60u);
        pat[L] = '\n';
        uint32_t f = 0;
        for (uint32_t i = 0; i < W; i++) {
            R[r * W + i] = pat[f];
            f = f == L ? 0u : f + 1u;
        }
    }
    __syncthreads();
}

// Finishing job of 1- or 2-word keys of any size (a whole MSD child): the keys are streamed from
// global memory into a shared-memory table whose key is the key itself (u32 / u64: exact), the
// distinct keys sorted (block_sort_smem), and each written as often as it occurs. More than
// kStreamDistinct distinct keys: a job of <= 2048 keys is sorted in full; a larger one goes back to
// the MSD as a segment of the next level.
constexpr uint32_t kStreamSlots = 2048, kStreamDistinct = 1024;
// patterns that do not fit shared memory go to global scratch only for runs of >= kPatRunMin words on
// average (measured on c4: shorter runs are cheaper word by word)
constexpr uint32_t kPatRunMin = 8;
__device__ __forceinline__ uint32_t cas_t(uint32_t *p, uint32_t cmp, uint32_t v) { return atomicCAS(p, cmp, v); }
__device__ __forceinline__ uint64_t cas_t(uint64_t *p, uint64_t cmp, uint64_t v) {
    return atomicCAS(reinterpret_cast<unsigned long long *>(p), (unsigned long long)cmp, (unsigned long long)v);
}
template <typename T>
__device__ __forceinline__ uint32_t st_hash(T k) { return (uint32_t)(((uint64_t)k * 0x9E3779B97F4A7C15ull) >> 53); }

// A part of a split job: job q of q_tiny, part p of np, global part id
struct FinPart {
    uint32_t q, p, np, id;
};

// After a part has published its list (or the job's overflow flag): true for the part that arrives
// last (it merges the lists and finishes the job).
__device__ __forceinline__ bool part_arrive(const MsdArgs &a, const FinPart &pr, uint32_t *flag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) *flag = atomicAdd(&a.job_done[pr.q], 1u) == pr.np - 1 ? 1u : 0u;
    __syncthreads();
    const bool last = *flag != 0;
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// A merged split job of more than kEmitSplitMin words: leave its run table in its parts' list space
// ([0] runs, [1..nd] run ends, then the distinct keys in order, KW words each) and queue its text pieces
// for k_msd_fin_emit (many CTAs instead of this one).
template <int KW, class KeyOf>
__device__ __forceinline__ void publish_runs(const MsdArgs &a, const MsdSeg &sg, const FinPart &pr, uint32_t nd,
                                             const uint32_t *ends, KeyOf key_of) {
    uint32_t *tab = reinterpret_cast<uint32_t *>(a.part_list + (size_t)(pr.id - pr.p) * kPartListMax);
    const uint32_t t = threadIdx.x;
    for (uint32_t r = t; r < nd; r += kST) {
        tab[1 + r] = ends[r];
        uint32_t k[KW];
        key_of(r, k);
#pragma unroll
        for (int u = 0; u < KW; u++) tab[1 + nd + r * KW + u] = k[u];
    }
    if (t == 0) tab[0] = nd;
    const uint32_t np = (sg.n + kEmitPieceWords - 1) / kEmitPieceWords;
    __shared__ uint32_t s_e0;
    __threadfence();
    __syncthreads();
    if (t == 0) s_e0 = atomicAdd(a.ctr + kQEmit, np);
    __syncthreads();
    for (uint32_t i = t; i < np; i += kST)
        if (s_e0 + i < a.cap_emit) a.q_emit[s_e0 + i] = make_uint2(pr.q, i);
}

template <typename T, int KW, bool PART>
__device__ __forceinline__ void fin_stream(const MsdArgs &a, const MsdSeg &sg, const BucketInfo &b, uint8_t *smraw,
                                           const FinPart pr) {
    const T kEmpty = ~(T)0;
    const uint32_t t = threadIdx.x, n = sg.n;
    T *slots = reinterpret_cast<T *>(smraw);
    uint32_t *cnt = reinterpret_cast<uint32_t *>(slots + kStreamSlots);
    T *A = reinterpret_cast<T *>(cnt + kStreamSlots);
    T *B = A + fpad(kStreamDistinct);
    uint32_t *pos = reinterpret_cast<uint32_t *>(B + fpad(kStreamDistinct));
    uint32_t *misc = pos + kStreamDistinct;   // [0] distinct keys, [1] overflow, [2..10] scan scratch, [12] flag
    constexpr bool part = PART;
    const uint32_t k0 = part ? pr.p * kPartKeys : 0u;   // the keys this CTA counts: [k0, k0 + nc)
    const uint32_t nc = part ? min(kPartKeys, n - k0) : n;
    // table size adapted to the job (a small job pays for a small table): >= 2n slots, <= kStreamSlots
    // (parts and their merge: the full table)
    uint32_t ns0 = 64;
    while (ns0 < 2 * nc && ns0 < kStreamSlots) ns0 *= 2;
    const uint32_t ns = PART ? kStreamSlots : ns0;
    const uint32_t smask = ns - 1, sshift = 32 - (31 - __clz(ns));
    auto init = [&]() {
        for (uint32_t i = t; i < ns; i += kST) {
            slots[i] = kEmpty;
            cnt[i] = 0;
        }
        if (t < 2) misc[t] = 0;
        __syncthreads();
    };
    auto ins = [&](T k, uint32_t mult) {   // count `mult` occurrences of k (sets the overflow flag if full)
        uint32_t h = (uint32_t)(((uint64_t)k * 0x9E3779B97F4A7C15ull) >> 32) >> sshift;
        for (;;) {
            T cur = slots[h];
            if (cur == kEmpty) {
                if (atomicAdd(misc, 1u) >= kStreamDistinct) {   // table full: give up on this job
                    atomicExch(misc + 1, 1u);
                    return;
                }
                cur = cas_t(&slots[h], kEmpty, k);
                if (cur == kEmpty) cur = k;
                else atomicSub(misc, 1u);   // lost the race for this slot
            }
            if (cur == k) {
                atomicAdd(&cnt[h], mult);
                return;
            }
            h = (h + 1) & smask;
        }
    };
    init();
    if (part && t == 0 && *reinterpret_cast<volatile uint32_t *>(a.job_ovf + pr.q)) misc[1] = 1u;   // (job given up)
    if (part) __syncthreads();
    const uint32_t *src = ((sg.buf & 1u) ? a.keys_a : a.keys_b) + b.key_off + (uint64_t)sg.start * KW;
    for (uint32_t i0 = 0; i0 < nc; i0 += 4 * kST) {
        T k[4];
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const uint32_t i = i0 + r * kST + t;
            k[r] = i < nc ? fin_load<T, KW>(src + (size_t)(k0 + i) * KW) : kEmpty;
        }
        if (*reinterpret_cast<volatile uint32_t *>(misc + 1)) break;
#pragma unroll
        for (int r = 0; r < 4; r++)
            if (k[r] != kEmpty) ins(k[r], 1u);
    }
    __syncthreads();
    if constexpr (PART) {
        if (misc[1]) {
            if (t == 0) atomicExch(a.job_ovf + pr.q, 1u);
        } else {   // publish this part's distinct keys and their counts
            const uint32_t per = (ns + kST - 1) / kST;
            uint32_t occ = 0, nd = 0;
            for (uint32_t e = 0; e < per; e++) occ += (per * t + e < ns) && cnt[per * t + e] != 0;
            uint32_t q = block_excl_scan_m(occ, misc + 2, &nd);
            uint4 *lst = a.part_list + (size_t)pr.id * kPartListMax;
            for (uint32_t e = 0; e < per; e++) {
                const uint32_t h = per * t + e;
                if (h < ns && cnt[h]) {
                    const uint64_t v = (uint64_t)slots[h];
                    lst[q++] = make_uint4((uint32_t)v, (uint32_t)(v >> 32), cnt[h], 0u);
                }
            }
            if (t == 0) a.part_n[pr.id] = nd;
        }
        if (!part_arrive(a, pr, misc + 12)) return;
        // the last part: merge every part's list into a fresh table (the job's distinct keys, counts)
        init();
        if (t == 0 && __ldcg(a.job_ovf + pr.q)) misc[1] = 1u;
        __syncthreads();
        if (!misc[1]) {
            const uint32_t id0 = pr.id - pr.p;
            for (uint32_t p = 0; p < pr.np; p++) {
                const uint32_t m = __ldcg(a.part_n + id0 + p);
                const uint4 *lst = a.part_list + (size_t)(id0 + p) * kPartListMax;
                for (uint32_t e = t; e < m; e += kST) {
                    if (*reinterpret_cast<volatile uint32_t *>(misc + 1)) break;
                    const uint4 v = __ldcg(lst + e);
                    ins((T)(((uint64_t)v.y << 32) | v.x), v.z);
                }
            }
        }
        __syncthreads();
    }
    if (misc[1]) {   // too many distinct keys
        if (n <= b.tile_keys) {   // (possibly several children): sort the job in full
            __syncthreads();
            T *FA = reinterpret_cast<T *>(smraw), *FB = FA + fpad(kST * 8);
            for (uint32_t i = t; i < kST * 8; i += kST) FA[fpad(i)] = i < n ? fin_load<T, KW>(src + (size_t)i * KW) : kEmpty;
            T *S = block_sort_smem<T>(FA, FB, n);
            uint8_t *stage = reinterpret_cast<uint8_t *>(S == FA ? FB : FA);   // (>= kFinStage + 32 bytes)
            emit_job_text<KW>(a, b, sg.L, sg.start, n, stage, [&](uint32_t i, uint32_t (&k)[KW]) {
                const T v = S[fpad(i)];
                if constexpr (KW == 1) k[0] = (uint32_t)v;
                else {
                    k[0] = (uint32_t)((uint64_t)v >> 32);
                    k[1] = (uint32_t)v;
                }
            });
        } else if (t == 0) {   // one child larger than a tile: back to the MSD as a segment of the next
                               // level (a child without digits left holds one key only: this terminates)
            const uint32_t nt = (n + b.aux - 1) / b.aux;
            const uint32_t q = atomicAdd(a.ctr + kQBig, 1u), t0 = atomicAdd(a.ctr + kQTiles, nt);
            if (q < a.cap_big) a.q_big[q] = MsdSeg{sg.L, sg.start, n, sg.buf & 1u};
            for (uint32_t i = 0; i < nt && t0 + i < a.cap_tiles; i++) a.q_tiles[t0 + i] = MsdTile{q, i * b.aux, min(b.aux, n - i * b.aux), 0};
        }
        return;
    }
    // compact the distinct keys (8 slots per thread), sort them, look up their counts, scan
    const uint32_t per = (ns + kST - 1) / kST;   // slots per thread (contiguous)
    uint32_t occ = 0;
    for (uint32_t e = 0; e < per; e++) occ += (per * t + e < ns) && cnt[per * t + e] != 0;
    uint32_t nd = 0;
    uint32_t p = block_excl_scan_m(occ, misc + 2, &nd);
    for (uint32_t e = 0; e < per; e++) {
        const uint32_t h = per * t + e;
        if (h < ns && cnt[h]) A[fpad(p++)] = slots[h];
    }
    T *S = block_sort_smem<T>(A, B, nd);
    uint32_t c4[4], tot = 0;   // nd <= 1024: 4 per thread
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const uint32_t i = 4 * t + e;
        c4[e] = 0;
        if (i < nd) {
            const T k = S[fpad(i)];
            uint32_t h = (uint32_t)(((uint64_t)k * 0x9E3779B97F4A7C15ull) >> 32) >> sshift;
            while (slots[h] != k) h = (h + 1) & smask;
            c4[e] = cnt[h];
        }
        tot += c4[e];
    }
    uint32_t run = block_excl_scan_m(tot, misc + 2, nullptr);
#pragma unroll
    for (int e = 0; e < 4; e++) {
        run += c4[e];
        if (4 * t + e < nd) pos[4 * t + e] = run;   // end (exclusive) of the run of distinct key 4t+e
    }
    __syncthreads();
    // the table is no longer needed: its space holds the runs' repeated patterns (or stages the text)
    auto key_of = [&](uint32_t r, uint32_t (&k)[KW]) {
        const T v = S[fpad(r)];
        if constexpr (KW == 1) k[0] = (uint32_t)v;
        else {
            k[0] = (uint32_t)((uint64_t)v >> 32);
            k[1] = (uint32_t)v;
        }
    };
    if constexpr (PART) {
        if (n > kEmitSplitMin) {
            publish_runs<KW>(a, sg, pr, nd, pos, key_of);
            return;
        }
    }
    const uint32_t W = (sg.L + 1 + 16 + 3) & ~3u;
    uint8_t *R = reinterpret_cast<uint8_t *>(slots);
    if (nd * W + 4 > kStreamSlots * (sizeof(T) + 4)) {   // the patterns do not fit shared memory
        if (n < kPatRunMin * nd) {   // short runs: word by word through a shared-memory stage
            emit_job_text<KW>(a, b, sg.L, sg.start, n, R, [&](uint32_t i, uint32_t (&k)[KW]) { key_of(run_of(pos, nd, i), k); });
            return;
        }
        R = a.pat + (size_t)blockIdx.x * kFinPatBytes;   // long runs: patterns in global scratch
    }
    build_run_patterns<KW>(R, W, sg.L, nd, key_of);
    emit_runs_text(a, b, sg.L, sg.start, n, R, W, pos, nd);
}

// Finishing job of KW >= 3-word keys of any size: as fin_stream, but the table key is a 64-bit
// fingerprint of the key; the first key of each fingerprint is kept as its representative, and a
// second pass compares every key with its representative word by word (exact: any mismatch sorts
// the job in full / sends it to the next MSD level). At most kWideDistinct distinct keys, ranked by
// counting the smaller ones.
constexpr uint32_t kWideSlots = 1024, kWideDistinct = 512;
constexpr uint32_t kRankMax = 256;   // distinct wide keys ordered by rank counting (nd^2 comparisons) up to here
template <int KW>
__device__ __forceinline__ uint64_t fp64(const uint32_t (&k)[KW]) {
    uint64_t h = 0x9E3779B97F4A7C15ull;
#pragma unroll
    for (int u = 0; u < KW; u++) h = (h ^ k[u]) * 0xD6E8FEB86659FD93ull;
    h ^= h >> 29;
    return h == ~0ull ? 0x5555ull : h;   // never ~0 (= empty)
}
// A wide job with too many distinct keys and more keys than one CTA sorts (an MSD child of 13..66-letter
// words, nearly all distinct): instead of going back to the MSD as a segment of the next level (a count /
// plan / scatter pass and a host sync), the CTA that found it partitions it by its next 2-letter digit into
// the other key buffer (same positions) and appends the sub-children, packed greedily into jobs of <= one
// tile, to the sub-job queue; a second k_msd_fin launch (sub_mode, queued right behind, no host sync) runs
// them on every CTA. Sub-jobs are marked (buf bit 4) and never partitioned again.
constexpr uint32_t kSubPartMax = 65536;   // largest job partitioned in a CTA (more: next MSD level)
// the digit a job's keys are partitioned by next: 0 for a whole bucket (the small-text path's jobs), else
// the one after the job's level
__device__ __forceinline__ uint32_t fin_next_digit(const MsdSeg &sg) { return (sg.buf & kSegWhole) ? 0u : (sg.buf >> 8) + 1u; }
template <int KW>
__device__ __forceinline__ bool fin_partition(const MsdArgs &a, const MsdSeg &sg, const BucketInfo &b, uint8_t *smraw) {
    const uint32_t t = threadIdx.x, n = sg.n, q = fin_next_digit(sg);
    uint32_t *hist = reinterpret_cast<uint32_t *>(smraw), *cur = hist + kRadixBins, *wsum = cur + kRadixBins;
    MsdSeg *jobs = reinterpret_cast<MsdSeg *>(wsum + 16);   // [<= 729]
    __shared__ uint32_t s_base, s_ns;
    const uint32_t *src = ((sg.buf & 1u) ? a.keys_a : a.keys_b) + b.key_off + (uint64_t)sg.start * KW;
    uint32_t *dst = ((sg.buf & 1u) ? a.keys_b : const_cast<uint32_t *>(a.keys_a)) + b.key_off + (uint64_t)sg.start * KW;
    for (uint32_t i = t; i < kRadixBins; i += kST) hist[i] = 0;
    __syncthreads();
    for (uint32_t i = t; i < n; i += kST) {
        uint32_t k[KW];
#pragma unroll
        for (int u = 0; u < KW; u++) k[u] = __ldg(src + (size_t)i * KW + u);
        atomicAdd(&hist[digit_reg<KW>(k, q)], 1u);
    }
    __syncthreads();
    uint32_t c[4];
#pragma unroll
    for (int e = 0; e < 4; e++) c[e] = hist[4 * t + e];
    uint32_t ex = block_excl_scan_m(c[0] + c[1] + c[2] + c[3], wsum, nullptr);
#pragma unroll
    for (int e = 0; e < 4; e++) {
        hist[4 * t + e] = ex;   // base of digit 4t+e
        cur[4 * t + e] = ex;
        ex += c[e];
    }
    __syncthreads();
    if (t == 0) {   // the sub-jobs (greedy packing, digit order), then their queue slots (none: next MSD level)
        const uint32_t nbuf = ((sg.buf & 1u) ^ 1u) | 16u | (q << 8);
        uint32_t ns = 0, js = 0, jn = 0;
        for (uint32_t d = 0; d < kRadixBins; d++) {
            const uint32_t st = hist[d], cnt = (d + 1 < kRadixBins ? hist[d + 1] : n) - st;
            if (!cnt) continue;
            if (jn && jn + cnt > b.tile_keys) {
                jobs[ns++] = MsdSeg{sg.L, sg.start + js, jn, nbuf};
                jn = 0;
            }
            if (!jn) js = st;
            jn += cnt;
        }
        if (jn) jobs[ns++] = MsdSeg{sg.L, sg.start + js, jn, nbuf};
        uint32_t base = 0xffffffffu;
        if (*reinterpret_cast<volatile uint32_t *>(a.sub_n) + ns <= a.cap_sub) {
            base = atomicAdd(a.sub_n, ns);
            if (base + ns > a.cap_sub) {   // (lost the race for the last slots: fill ours with empty jobs)
                for (uint32_t k = 0; base + k < a.cap_sub && k < ns; k++) a.sub_stack[base + k] = MsdSeg{sg.L, 0, 0, 0};
                base = 0xffffffffu;
            }
        }
        s_base = base;
        s_ns = ns;
    }
    __syncthreads();
    if (s_base == 0xffffffffu) return false;
    for (uint32_t i = t; i < n; i += kST) {
        uint32_t k[KW];
#pragma unroll
        for (int u = 0; u < KW; u++) k[u] = __ldg(src + (size_t)i * KW + u);
        const uint32_t p = atomicAdd(&cur[digit_reg<KW>(k, q)], 1u);
#pragma unroll
        for (int u = 0; u < KW; u++) dst[(size_t)p * KW + u] = k[u];
    }
    for (uint32_t k = t; k < s_ns; k += kST) a.sub_stack[s_base + k] = jobs[k];
    __syncthreads();
    return true;
}

template <int KW, bool PART>
__device__ __forceinline__ void fin_stream_wide(const MsdArgs &a, const MsdSeg &sg, const BucketInfo &b, uint8_t *smraw,
                                                const FinPart pr) {
    const uint64_t kEmpty = ~0ull;
    const uint32_t t = threadIdx.x, n = sg.n;
    uint64_t *fps = reinterpret_cast<uint64_t *>(smraw);                 // [kWideSlots]
    uint32_t *sid = reinterpret_cast<uint32_t *>(fps + kWideSlots);       // [kWideSlots] distinct id
    uint32_t *cnt = sid + kWideSlots;                                     // [kWideSlots]
    uint32_t *rep = cnt + kWideSlots;                                     // [kWideDistinct][KW]
    uint32_t *dcnt = rep + kWideDistinct * KW;                            // [kWideDistinct] count by id
    uint32_t *order = dcnt + kWideDistinct;                               // [kWideDistinct] id by rank
    uint32_t *pos = order + kWideDistinct;                                // [kWideDistinct] run ends
    uint32_t *misc = pos + kWideDistinct;                                 // [0] nd [1] overflow [2..10] scan [12] flag
    uint32_t *repix = misc + 16;                                          // [kWideDistinct] representative's index
    constexpr bool part = PART;
    const uint32_t k0 = part ? pr.p * kPartKeys : 0u;   // the keys this CTA counts: [k0, k0 + nc)
    const uint32_t nc = part ? min(kPartKeys, n - k0) : n;
    auto init = [&]() {
        for (uint32_t i = t; i < kWideSlots; i += kST) {
            fps[i] = kEmpty;
            sid[i] = 0xffffffffu;
            cnt[i] = 0;
        }
        if (t < 2) misc[t] = 0;
        __syncthreads();
    };
    init();
    if (part && t == 0 && *reinterpret_cast<volatile uint32_t *>(a.job_ovf + pr.q)) misc[1] = 1u;   // (job given up)
    if (part) __syncthreads();
    const uint32_t *src = ((sg.buf & 1u) ? a.keys_a : a.keys_b) + b.key_off + (uint64_t)sg.start * KW;
    // keys are loaded BATCH at a time ahead of their inserts (independent loads in flight)
    constexpr int BATCH = KW <= 2 ? 4 : (KW <= 4 ? 2 : 1);
    auto insert = [&](const uint32_t (&k)[KW], uint32_t mult, uint32_t kidx) {
        const uint64_t f = fp64<KW>(k);
        uint32_t h = (uint32_t)(f >> 40) & (kWideSlots - 1);
        for (;;) {
            uint64_t cur = fps[h];
            if (cur == kEmpty) {
                cur = atomicCAS(reinterpret_cast<unsigned long long *>(&fps[h]), kEmpty, (unsigned long long)f);
                if (cur == kEmpty) {   // new fingerprint: this key is its representative
                    const uint32_t id = atomicAdd(misc, 1u);
                    if (id >= kWideDistinct) {
                        atomicExch(misc + 1, 1u);
                        return;
                    }
#pragma unroll
                    for (int u = 0; u < KW; u++) rep[id * KW + u] = k[u];
                    repix[id] = kidx;
                    atomicExch(&sid[h], id);
                    cur = f;
                }
            }
            if (cur == f) {
                atomicAdd(&cnt[h], mult);
                return;
            }
            h = (h + 1) & (kWideSlots - 1);
        }
    };
    // does key k equal its fingerprint's representative? (a 64-bit fingerprint collision: never expected)
    auto same_as_rep = [&](const uint32_t (&k)[KW]) {
        const uint64_t f = fp64<KW>(k);
        uint32_t h = (uint32_t)(f >> 40) & (kWideSlots - 1);
        while (fps[h] != f) h = (h + 1) & (kWideSlots - 1);
        const uint32_t id = sid[h];
        bool eq = true;
#pragma unroll
        for (int u = 0; u < KW; u++) eq &= rep[id * KW + u] == k[u];
        return eq;
    };
    for (uint32_t i0 = 0; i0 < nc; i0 += BATCH * kST) {
        if (*reinterpret_cast<volatile uint32_t *>(misc + 1)) break;
        uint32_t k[BATCH][KW];
#pragma unroll
        for (int r = 0; r < BATCH; r++) {
            const uint32_t i = i0 + r * kST + t;
#pragma unroll
            for (int u = 0; u < KW; u++) k[r][u] = i < nc ? __ldg(src + (size_t)(k0 + i) * KW + u) : 0u;
        }
#pragma unroll
        for (int r = 0; r < BATCH; r++)
            if (i0 + r * kST + t < nc) insert(k[r], 1u, k0 + i0 + r * kST + t);
    }
    __syncthreads();
    if (!misc[1]) {   // verify: every key equals its fingerprint's representative
        for (uint32_t i0 = 0; i0 < nc; i0 += BATCH * kST) {
            uint32_t k[BATCH][KW];
#pragma unroll
            for (int r = 0; r < BATCH; r++) {
                const uint32_t i = i0 + r * kST + t;
#pragma unroll
                for (int u = 0; u < KW; u++) k[r][u] = i < nc ? __ldg(src + (size_t)(k0 + i) * KW + u) : 0u;
            }
#pragma unroll
            for (int r = 0; r < BATCH; r++)
                if (i0 + r * kST + t < nc && !same_as_rep(k[r])) misc[1] = 1u;
        }
    }
    __syncthreads();
    if constexpr (PART) {
        if (misc[1]) {
            if (t == 0) atomicExch(a.job_ovf + pr.q, 1u);
        } else {   // publish this part's distinct keys: fingerprint, count, representative's index
            const uint32_t per = (kWideSlots + kST - 1) / kST;
            uint32_t occ = 0, nd = 0;
            for (uint32_t e = 0; e < per; e++) occ += cnt[per * t + e] != 0;
            uint32_t q = block_excl_scan_m(occ, misc + 2, &nd);
            uint4 *lst = a.part_list + (size_t)pr.id * kPartListMax;
            for (uint32_t e = 0; e < per; e++) {
                const uint32_t h = per * t + e;
                if (cnt[h]) lst[q++] = make_uint4((uint32_t)fps[h], (uint32_t)(fps[h] >> 32), cnt[h], repix[sid[h]]);
            }
            if (t == 0) a.part_n[pr.id] = nd;
        }
        if (!part_arrive(a, pr, misc + 12)) return;
        // the last part: merge the parts' lists (the representatives come from the keys), then check
        // that equal fingerprints of different parts have equal representatives
        init();
        if (t == 0 && __ldcg(a.job_ovf + pr.q)) misc[1] = 1u;
        __syncthreads();
        const uint32_t id0 = pr.id - pr.p;
        for (int pass = 0; pass < 2; pass++) {
            for (uint32_t p = 0; p < pr.np && !*reinterpret_cast<volatile uint32_t *>(misc + 1); p++) {
                const uint32_t m = __ldcg(a.part_n + id0 + p);
                const uint4 *lst = a.part_list + (size_t)(id0 + p) * kPartListMax;
                for (uint32_t e = t; e < m; e += kST) {
                    const uint4 v = __ldcg(lst + e);
                    uint32_t k[KW];
#pragma unroll
                    for (int u = 0; u < KW; u++) k[u] = __ldg(src + (size_t)v.w * KW + u);
                    if (pass == 0) insert(k, v.z, v.w);
                    else if (!same_as_rep(k)) misc[1] = 1u;
                }
            }
            __syncthreads();
        }
    }
    if (misc[1]) {   // too many distinct keys
        if (n <= b.tile_keys) {   // (possibly several children): sort the job in full
            __syncthreads();
            cta_sort_job<KW, (KW <= 4 ? 4 : (KW <= 8 ? 2 : 1))>(a, sg, b, reinterpret_cast<uint32_t *>(smraw));
            __syncthreads();   // the sorted keys are in buffer B (written by this CTA)
            const uint32_t *kb = a.keys_b + b.key_off + (uint64_t)sg.start * KW;
            emit_job_text<KW>(a, b, sg.L, sg.start, n, smraw, [&](uint32_t i, uint32_t (&k)[KW]) {
#pragma unroll
                for (int u = 0; u < KW; u++) k[u] = kb[(size_t)i * KW + u];
            });
        } else {
            bool done = false;   // partitioned here: the sub-jobs run in the sub_mode launch
            if (!PART && a.sub_stack && !(sg.buf & 16u) && n <= kSubPartMax && fin_next_digit(sg) < b.ndig) {
                __syncthreads();
                done = fin_partition<KW>(a, sg, b, smraw);
            }
            if (!done && t == 0) {   // one child larger than a tile: back to the MSD as a segment of the next
                                     // level (a child without digits left holds one key only: this terminates)
                const uint32_t nt = (n + b.aux - 1) / b.aux;
                const uint32_t q = atomicAdd(a.ctr + kQBig, 1u), t0 = atomicAdd(a.ctr + kQTiles, nt);
                if (q < a.cap_big) a.q_big[q] = MsdSeg{sg.L, sg.start, n, sg.buf & 1u};
                for (uint32_t i = 0; i < nt && t0 + i < a.cap_tiles; i++) a.q_tiles[t0 + i] = MsdTile{q, i * b.aux, min(b.aux, n - i * b.aux), 0};
            }
        }
        return;
    }
    const uint32_t nd = misc[0];
    for (uint32_t i = t; i < kWideSlots; i += kST)
        if (cnt[i]) dcnt[sid[i]] = cnt[i];
    __syncthreads();
    // sort the distinct keys. Few (<= kRankMax): rank = number of smaller keys (full comparison).
    // Else: 64-bit sort key = the 11 letters from the job's first undecided position (its keys share
    // the letters before 2*level) and the key's index, by the odd-even transposition + merge-path block
    // sort; if keys agree on those 11 letters, the indices are sorted again with the full-key
    // comparison (same block sort)
    if (nd <= kRankMax) {
        for (uint32_t me = t; me < nd; me += kST) {
            uint32_t rank = 0;
            for (uint32_t j = 0; j < nd; j++) {
                bool lt = false, decided = false;
#pragma unroll
                for (int u = 0; u < KW; u++) {
                    const uint32_t x = rep[j * KW + u], y = rep[me * KW + u];
                    if (!decided && x != y) {
                        lt = x < y;
                        decided = true;
                    }
                }
                rank += lt;
            }
            order[rank] = me;
        }
        __syncthreads();
    } else {
        uint64_t *SA = reinterpret_cast<uint64_t *>(smraw), *SB = SA + fpad(kWideDistinct);   // (table space: free now)
        const uint32_t p0 = 2u * (sg.buf >> 8);
        for (uint32_t id = t; id < nd; id += kST) {
            uint64_t acc = 0;
#pragma unroll
            for (uint32_t q = 0; q < 11; q++) {
                const uint32_t j = p0 + q;
                const uint32_t code = j < sg.L ? (rep[id * KW + min(j / 6u, (uint32_t)KW - 1)] >> (25 - 5 * (j % 6))) & 31u : 0u;
                acc = (acc << 5) | code;
            }
            SA[fpad(id)] = (acc << 9) | id;
        }
        uint64_t *S = block_sort_smem<uint64_t>(SA, SB, nd);
        uint32_t ties = 0;
        for (uint32_t r = t; r + 1 < nd; r += kST) ties += (S[fpad(r)] >> 9) == (S[fpad(r + 1)] >> 9);
        ties = __syncthreads_count(ties != 0);
        for (uint32_t r = t; r < nd; r += kST) order[r] = (uint32_t)(S[fpad(r)] & 511u);
        __syncthreads();
        if (ties) {
            uint32_t *IA = reinterpret_cast<uint32_t *>(smraw), *IB = IA + fpad(kWideDistinct);
            for (uint32_t r = t; r < nd; r += kST) IA[fpad(r)] = order[r];
            uint32_t *SI = block_sort_idx(IA, IB, nd, [&](uint32_t x, uint32_t y) {
#pragma unroll
                for (int u = 0; u < KW; u++) {
                    const uint32_t a2 = rep[x * KW + u], c2 = rep[y * KW + u];
                    if (a2 != c2) return a2 < c2;
                }
                return false;
            });
            for (uint32_t r = t; r < nd; r += kST) order[r] = SI[fpad(r)];
            __syncthreads();
        }
    }
    constexpr int PT = kWideDistinct / kST;   // ranks per thread (contiguous)
    uint32_t cc[PT], tot = 0;
#pragma unroll
    for (int e = 0; e < PT; e++) {
        const uint32_t r = PT * t + e;
        cc[e] = r < nd ? dcnt[order[r]] : 0u;
        tot += cc[e];
    }
    uint32_t end = block_excl_scan_m(tot, misc + 2, nullptr);
#pragma unroll
    for (int e = 0; e < PT; e++) {
        end += cc[e];
        if (PT * t + e < nd) pos[PT * t + e] = end;
    }
    __syncthreads();
    // the fingerprint table is no longer needed: its space (16 KiB) holds the runs' repeated patterns
    // (or stages the text)
    auto key_of = [&](uint32_t r, uint32_t (&k)[KW]) {
        const uint32_t id = order[r];
#pragma unroll
        for (int u = 0; u < KW; u++) k[u] = rep[id * KW + u];
    };
    if constexpr (PART) {
        if (n > kEmitSplitMin) {
            publish_runs<KW>(a, sg, pr, nd, pos, key_of);
            return;
        }
    }
    const uint32_t W = (sg.L + 1 + 16 + 3) & ~3u;
    uint8_t *R = smraw;
    if (nd * W + 4 > kWideSlots * 16) {   // the patterns do not fit shared memory
        if (n < kPatRunMin * nd) {   // short runs: word by word through a shared-memory stage
            emit_job_text<KW>(a, b, sg.L, sg.start, n, smraw, [&](uint32_t i, uint32_t (&k)[KW]) { key_of(run_of(pos, nd, i), k); });
            return;
        }
        R = a.pat + (size_t)blockIdx.x * kFinPatBytes;   // long runs: patterns in global scratch
    }
    build_run_patterns<KW>(R, W, sg.L, nd, key_of);
    emit_runs_text(a, b, sg.L, sg.start, n, R, W, pos, nd);
}

// Persistent: jobs [small_base, ctr[kQSmall]) — the end is read on the device (this level's plan
// appended them), so the host needs no sync before the launch.
template <bool PART>
__device__ __forceinline__ void fin_job(const MsdArgs &a, const MsdSeg &sg, const BucketInfo &b, uint8_t *fsm, const FinPart &pr) {
    switch (b.kw) {
        case 1: fin_stream<uint32_t, 1, PART>(a, sg, b, fsm, pr); break;
        case 2: fin_stream<uint64_t, 2, PART>(a, sg, b, fsm, pr); break;
        case 3: fin_stream_wide<3, PART>(a, sg, b, fsm, pr); break;
        case 4: fin_stream_wide<4, PART>(a, sg, b, fsm, pr); break;
        case 5: fin_stream_wide<5, PART>(a, sg, b, fsm, pr); break;
        case 6: fin_stream_wide<6, PART>(a, sg, b, fsm, pr); break;
        case 7: fin_stream_wide<7, PART>(a, sg, b, fsm, pr); break;
        case 8: fin_stream_wide<8, PART>(a, sg, b, fsm, pr); break;
        case 9: fin_stream_wide<9, PART>(a, sg, b, fsm, pr); break;
        case 10: fin_stream_wide<10, PART>(a, sg, b, fsm, pr); break;
        default: fin_stream_wide<11, PART>(a, sg, b, fsm, pr); break;
    }
}

// Persistent: tickets [0, parts) are the parts of the big jobs (equal sizes, taken first), then the
// small jobs [small_base, ctr[kQSmall]); both ends are read on the device (this level's plan appended
// them), so the host needs no sync before the launch.
__global__ void __launch_bounds__(kST, 4) k_msd_fin(MsdArgs a) {
    extern __shared__ __align__(16) uint8_t fsm[];
    __shared__ uint32_t s_job;
    // (sub_mode: the jobs are the sub-jobs fin_partition queued during the previous launch)
    const uint32_t np = a.sub_mode ? 0u : min(*reinterpret_cast<volatile uint32_t *>(a.ctr + kQParts), a.cap_parts) - a.parts_base;
    const uint32_t end = a.sub_mode ? min(*reinterpret_cast<volatile uint32_t *>(a.sub_n), a.cap_sub)
                                    : np + min(*reinterpret_cast<volatile uint32_t *>(a.ctr + kQSmall), a.cap_local) - a.small_base;
    for (;;) {
    if (threadIdx.x == 0) s_job = atomicAdd(a.ctr + kQFinTicket, 1u);
    __syncthreads();
    const uint32_t j = s_job;
    if (j >= end) break;
    const MsdSeg sg = a.sub_mode ? a.sub_stack[j] : j < np ? a.q_tiny[a.q_parts[a.parts_base + j]] : a.q_small[a.small_base + j - np];
    if (sg.n == 0) {   // (a sub-job slot left empty)
        __syncthreads();
        continue;
    }
    if (j < np && job_parts(sg.n) > 1) {   // a part of a split job: k_msd_fin_split's
        __syncthreads();
        continue;
    }
    const BucketInfo b = a.buckets[sg.L];
    const long long c0 = a.dbg_jobs ? clock64() : 0;
    fin_job<false>(a, sg, b, fsm, FinPart{0u, 0u, 0u, 0u});
    __syncthreads();   // shared memory is reused by the next job
    if (a.dbg_jobs && threadIdx.x == 0 && j < 65536) {   // (experiments: per-job cycles)
        a.dbg_jobs[4 * j] = sg.n;
        a.dbg_jobs[4 * j + 1] = b.kw | (sg.L << 8);
        a.dbg_jobs[4 * j + 2] = (uint32_t)(clock64() - c0);
        a.dbg_jobs[4 * j + 3] = 0;
    }
    }
}

// The parts of the split jobs (a separate kernel: their code would slow the whole-job kernel down —
// measured 0.95 -> 1.19 ms on c4 when both were one kernel). Runs beside k_msd_fin on its own stream.
__global__ void __launch_bounds__(kST, 4) k_msd_fin_split(MsdArgs a) {
    extern __shared__ __align__(16) uint8_t fsm[];
    __shared__ uint32_t s_job;
    const uint32_t np = min(*reinterpret_cast<volatile uint32_t *>(a.ctr + kQParts), a.cap_parts) - a.parts_base;
    for (;;) {
        if (threadIdx.x == 0) s_job = atomicAdd(a.ctr + kQSplitTicket, 1u);
        __syncthreads();
        const uint32_t j = s_job;
        __syncthreads();
        if (j >= np) break;
        FinPart pr;
        pr.id = a.parts_base + j;
        pr.q = a.q_parts[pr.id];
        const MsdSeg sg = a.q_tiny[pr.q];
        pr.np = job_parts(sg.n);
        if (pr.np == 1) continue;   // a whole job: k_msd_fin's
        pr.p = pr.id - a.job_pbase[pr.q];
        fin_job<true>(a, sg, a.buckets[sg.L], fsm, pr);
        __syncthreads();
    }
}
// The text of one piece [w0, w1) of a merged split job from its run table: the runs overlapping the
// piece get their repeated patterns (shared memory, else this CTA's global scratch) and emit_runs_text
// writes the piece.
template <int KW>
__device__ __forceinline__ void emit_piece(const MsdArgs &a, const MsdSeg &sg, const BucketInfo &b, const uint32_t *tab,
                                           uint32_t w0, uint32_t w1, uint8_t *smraw, size_t smbytes) {
    const uint32_t nd = __ldcg(tab);
    const uint32_t *ends = tab + 1, *keys = tab + 1 + nd;
    uint32_t *e = reinterpret_cast<uint32_t *>(smraw);   // [<= 1024] run ends relative to w0
    uint8_t *R = smraw + 4096;
    __shared__ uint32_t s_r0, s_r1;
    if (threadIdx.x == 0) {
        s_r0 = run_of(ends, nd, w0);
        s_r1 = run_of(ends, nd, w1 - 1);
    }
    __syncthreads();
    const uint32_t r0 = s_r0, nr = s_r1 - r0 + 1;
    for (uint32_t r = threadIdx.x; r < nr; r += kST) e[r] = min(__ldcg(ends + r0 + r), w1) - w0;
    const uint32_t W = (sg.L + 1 + 16 + 3) & ~3u;
    if (nr * W + 4 > smbytes - 4096) R = a.pat + (size_t)blockIdx.x * kFinPatBytes;
    build_run_patterns<KW>(R, W, sg.L, nr, [&](uint32_t r, uint32_t (&k)[KW]) {
#pragma unroll
        for (int u = 0; u < KW; u++) k[u] = __ldcg(keys + (size_t)(r0 + r) * KW + u);
    });
    emit_runs_text(a, b, sg.L, sg.start + w0, w1 - w0, R, W, e, nr);
    __syncthreads();
}

constexpr size_t kEmitSmem = 4096 + 1024 * 32 + 64;   // run ends + patterns of 1-2 word keys (wider: global)
__global__ void __launch_bounds__(kST) k_msd_fin_emit(MsdArgs a) {
    extern __shared__ __align__(16) uint8_t esm[];
    __shared__ uint32_t s_job;
    const uint32_t end = min(*reinterpret_cast<volatile uint32_t *>(a.ctr + kQEmit), a.cap_emit);
    for (;;) {
        if (threadIdx.x == 0) s_job = atomicAdd(a.ctr + kQEmitTicket, 1u);
        __syncthreads();
        const uint32_t j = a.emit_base + s_job;
        __syncthreads();
        if (j >= end) break;
        const uint2 pc = a.q_emit[j];
        const MsdSeg sg = a.q_tiny[pc.x];
        const BucketInfo b = a.buckets[sg.L];
        const uint32_t *tab = reinterpret_cast<const uint32_t *>(a.part_list + (size_t)a.job_pbase[pc.x] * kPartListMax);
        const uint32_t w0 = pc.y * kEmitPieceWords, w1 = min(sg.n, w0 + kEmitPieceWords);
        switch (b.kw) {
            case 1: emit_piece<1>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 2: emit_piece<2>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 3: emit_piece<3>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 4: emit_piece<4>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 5: emit_piece<5>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 6: emit_piece<6>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 7: emit_piece<7>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 8: emit_piece<8>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 9: emit_piece<9>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            case 10: emit_piece<10>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
            default: emit_piece<11>(a, sg, b, tab, w0, w1, esm, kEmitSmem); break;
        }
    }
}

constexpr size_t kFinSmemStream = kStreamSlots * 12 + 2 * (kStreamDistinct + kStreamDistinct / 16) * 8 + (kStreamDistinct + 16) * 4;
constexpr size_t kFinSmemWide = kWideSlots * 16 + (kWideDistinct * 11 + 4 * kWideDistinct + 16) * 4;   // KW <= 11
constexpr size_t kFinSmemSort = 2 * (kST * 4 * 4 + kST * 4 * 4 / 32 + 1) * 4;   // cta_sort_job fallback: TN*KW <= 4096
constexpr size_t kFinSmem0 = kFinSmemStream > kFinSmemWide ? kFinSmemStream : kFinSmemWide;
constexpr size_t kFinSmem = kFinSmem0 > kFinSmemSort ? kFinSmem0 : kFinSmemSort;

__global__ void __launch_bounds__(kST) k_msd_copy(MsdArgs a) {
    const CopyRange r = a.q_copy[blockIdx.x];
    for (uint32_t i = threadIdx.x; i < r.len; i += kST) a.keys_b[r.to + i] = __ldg(a.keys_a + r.from + i);
}

}  // namespace

size_t msd_scatter_smem() { return (size_t)(3 * kRadixBins + 8192 + 8192 / 32 + 8 + kST / 32 + 1) * 4; }

cudaError_t launch_msd_count(const MsdArgs &a, uint32_t ntiles, cudaStream_t s) {
    if (!ntiles) return cudaSuccess;
    k_msd_count<<<ntiles, kST, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_msd_count0(const MsdArgs &a, cudaStream_t s) {
    if (!a.nslices) return cudaSuccess;
    k_msd_count0<<<a.nslices, kST, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_msd_scatter0(const MsdArgs &a, cudaStream_t s) {
    if (!a.cls_pfx[kMaxStageKw]) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_msd_scatter0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kScatter0Smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t total = a.cls_pfx[kMaxStageKw];
    const uint32_t grid = WSORT_S0_SLICE ? a.nslices : std::min<uint32_t>(total, (uint32_t)sms * 2);
    k_msd_scatter0<<<grid, kS0T, kScatter0Smem, s>>>(a, total);
    return cudaGetLastError();
}
cudaError_t launch_msd_plan(const MsdArgs &a, uint32_t nsegs, cudaStream_t s, uint32_t mode) {
    if (!nsegs) return cudaSuccess;
    MsdArgs b = a;
    b.plan_mode = mode;
    k_msd_plan<<<nsegs, kST, 0, s>>>(b);
    return cudaGetLastError();
}
cudaError_t launch_msd_scatter(const MsdArgs &a, uint32_t ntiles, cudaStream_t s) {
    if (!ntiles) return cudaSuccess;
    static const bool persistent = getenv("WSORT_SCATTER_TILES") == nullptr;   // (experiments: the per-tile kernel)
    if (persistent) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const size_t smem = 2 * kScatBuf * 4 + 16 + 32 + msd_scatter_smem();
        cudaError_t e = cudaFuncSetAttribute(k_msd_scatter_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_msd_scatter_p<<<std::min<uint32_t>(ntiles, (uint32_t)sms * 2), kST, smem, s>>>(a, ntiles);
        return cudaGetLastError();
    }
    const size_t smem = msd_scatter_smem();
    cudaError_t e = cudaFuncSetAttribute(k_msd_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_msd_scatter<<<ntiles, kST, smem, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_msd_fin_jobs(const MsdArgs &a, uint32_t first, uint32_t first_part, uint32_t grid, cudaStream_t s) {
    if (!grid) return cudaSuccess;
    MsdArgs b = a;
    b.small_base = first;
    b.parts_base = first_part;
    cudaError_t e = cudaMemsetAsync(a.ctr + kQFinTicket, 0, 4, s);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_msd_fin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFinSmem);
    if (e != cudaSuccess) return e;
    k_msd_fin<<<grid, kST, kFinSmem, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_msd_fin_sub(const MsdArgs &a, uint32_t grid, cudaStream_t s) {
    if (!a.sub_stack || !grid) return cudaSuccess;
    MsdArgs b = a;
    b.sub_mode = 1;
    cudaError_t e = cudaMemsetAsync(a.ctr + kQFinTicket, 0, 4, s);
    if (e != cudaSuccess) return e;
    k_msd_fin<<<grid, kST, kFinSmem, s>>>(b);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return cudaMemsetAsync(a.sub_n, 0, 4, s);   // (the queue is empty again for the next launch)
}

cudaError_t launch_msd_fin_split(const MsdArgs &a, uint32_t first_part, uint32_t grid, cudaStream_t s) {
    MsdArgs b = a;
    b.parts_base = first_part;
    cudaError_t e = cudaMemsetAsync(a.ctr + kQSplitTicket, 0, 4, s);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_msd_fin_split, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFinSmem);
    if (e != cudaSuccess) return e;
    k_msd_fin_split<<<grid, kST, kFinSmem, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_msd_fin_emit(const MsdArgs &a, uint32_t first_piece, uint32_t grid, cudaStream_t s) {
    MsdArgs b = a;
    b.emit_base = first_piece;
    cudaError_t e = cudaMemsetAsync(a.ctr + kQEmitTicket, 0, 4, s);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_msd_fin_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEmitSmem);
    if (e != cudaSuccess) return e;
    k_msd_fin_emit<<<grid, kST, kEmitSmem, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_msd_finish(const MsdArgs &a, uint32_t n_small, uint32_t n_copy, uint32_t max_tile_words,
                              cudaStream_t s) {
    cudaError_t e;
    if (a.n_tiny) {
        k_msd_warp_sort<<<(a.n_tiny + kST / 32 - 1) / (kST / 32), kST, 0, s>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (n_small && a.finish_radix) {
        const size_t smem = ((size_t)2 * (2048 * 4 + 2048 * 4 / 32 + 1) + 32 * kST + 32 * kST / 32 + 1 + kST / 32 + 1) * 4;
        e = cudaFuncSetAttribute(k_msd_radix_job, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_msd_radix_job<<<n_small, kST, smem, s>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        // cta_sort_job's default tile: 256 * E keys of kw words <= 8192 words (jobs are at most tile_keys)
        const size_t tw = 8192;
        (void)max_tile_words;
        const size_t smem2 = (tw + tw / 32 + 1) * 2 * 4;
        e = cudaFuncSetAttribute(k_msd_cta_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        if (e != cudaSuccess) return e;
        k_msd_cta_sort<<<n_small, kST, smem2, s>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (n_copy) {
        k_msd_copy<<<n_copy, kST, 0, s>>>(a);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace wsort
