// k_hash.cu — phase 3 for the long words (6..66 letters) from K1's table of distinct words (k_hash.cuh).
//
// every per-length sub-array is sorted "in the alphabetic order". A sub-array sorted is its
// distinct words in order, each repeated as often as it occurs; K1 counted the occurrences, so only the
// D distinct words are sorted (D << W on text: c4 has ~1 M distinct long words among 57 M):
//   KH1 k_hash_gather   distinct keys -> their length buckets (keys_a), as K3 would pack them
//   (the MSD sort of keys_a -> keys_b, k_msd.cu: the distinct keys in order)
//   KH2 k_hash_runs     per sorted distinct key: its count (exact table lookup) -> run length
//   KH3 scan            run lengths -> run ends (the words before each run's end)
//   KH4 k_run_tiles     per emit tile: the runs holding its first / last word
//   KH5 k_emit_runs     "word\n" written run by run ("prints the results"; reading A12)
#include "k_hash.cuh"

namespace wsort {
namespace {

constexpr int kHT = 256;

// ---------------------------------------------------------------- KH1: gather the distinct keys
// Block b handles 4096 slots (the narrow table's, then the wide table's): per-length counts in shared
// memory, one global atomic per (block, length) reserves the block's range of each bucket, then the keys
// are copied.
constexpr uint32_t kGatherSlots = 4096;
__global__ void __launch_bounds__(kHT) k_hash_gather(HashGatherArgs a) {
    __shared__ uint32_t cnt[256], base[256];
    const uint32_t t = threadIdx.x;
    const uint32_t nblk_narrow = (a.tab.nmask + kGatherSlots) / kGatherSlots;   // (nmask + 1 is a multiple)
    const bool narrow = blockIdx.x < nblk_narrow;
    const uint32_t s0 = (narrow ? blockIdx.x : blockIdx.x - nblk_narrow) * kGatherSlots;
    cnt[t] = 0;
    __syncthreads();
    uint32_t info[kGatherSlots / kHT], rank[kGatherSlots / kHT];   // narrow: L; wide: meta
    hashtab::Key128 nk[kGatherSlots / kHT];
#pragma unroll
    for (int r = 0; r < (int)(kGatherSlots / kHT); r++) {
        const uint32_t i = s0 + t + r * kHT;
        info[r] = hashtab::kUnset;
        rank[r] = 0;
        nk[r] = hashtab::Key128{0ull, 0ull};
        if (narrow) {
            const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2 *>(a.tab.nkey) + i);
            nk[r] = hashtab::Key128{v.x & ~hashtab::kNarrowMark, v.y};
            if (v.x) info[r] = hashtab::narrow_len(nk[r]);
        } else if (i <= a.tab.mask) {
            const uint32_t m = __ldcg(a.tab.meta + i);
            if (m < hashtab::kDead) info[r] = m;
        }
        if (info[r] != hashtab::kUnset) rank[r] = atomicAdd(&cnt[narrow ? info[r] : info[r] >> 24], 1u);
    }
    __syncthreads();
    if (cnt[t]) base[t] = atomicAdd(a.lcursor + t, cnt[t]);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < (int)(kGatherSlots / kHT); r++) {
        if (info[r] == hashtab::kUnset) continue;
        const uint32_t L = narrow ? info[r] : info[r] >> 24, kw = (L + 5u) / 6u;
        uint32_t *dst = a.keys_a + a.buckets[L].key_off + (uint64_t)(base[L] + rank[r]) * kw;
        if (narrow) {
            const uint32_t kk[4] = {(uint32_t)(nk[r].lo >> 32), (uint32_t)nk[r].lo, (uint32_t)(nk[r].hi >> 32), (uint32_t)nk[r].hi};
#pragma unroll
            for (uint32_t q = 0; q < 4; q++)
                if (q < kw) dst[q] = kk[q];
        } else {
            const uint32_t *src = a.tab.keys + (info[r] & 0xffffffu);
            for (uint32_t q = 0; q < kw; q++) dst[q] = __ldcg(src + q);
        }
    }
}

// ---------------------------------------------------------------- KH1b: distinct keys of > 66 letters
// The MSD finish holds keys of <= 11 words (66 letters); longer distinct words are rare (a text's few very
// long words): one CTA per such bucket ranks its keys (rank = how many keys of the bucket are smaller;
// distinct keys, so ranks are a permutation) and writes each to buffer B at its rank. The host takes this
// path only while a bucket's keys fit shared memory (kWideSortWords).
__global__ void __launch_bounds__(kHT) k_sort_wide(const BucketInfo *kb, const uint32_t *lens, const uint32_t *keys_a,
                                                   uint32_t *keys_b) {
    __shared__ uint32_t sk[kWideSortWords];
    const uint32_t L = lens[blockIdx.x], kw = (L + 5u) / 6u;
    const BucketInfo b = kb[L];
    for (uint32_t i = threadIdx.x; i < b.n * kw; i += kHT) sk[i] = keys_a[b.key_off + i];
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < b.n; i += kHT) {
        uint32_t rank = 0;
        for (uint32_t j = 0; j < b.n; j++) {
            uint32_t q = 0;
            while (q < kw && sk[j * kw + q] == sk[i * kw + q]) q++;
            rank += q < kw && sk[j * kw + q] < sk[i * kw + q];
        }
        for (uint32_t q = 0; q < kw; q++) keys_b[b.key_off + (uint64_t)rank * kw + q] = sk[i * kw + q];
    }
}

// ---------------------------------------------------------------- KH2: run lengths of the sorted keys
__global__ void __launch_bounds__(kHT) k_hash_runs(HashRunArgs a) {
    const uint32_t j = blockIdx.x * kHT + threadIdx.x;
    if (j >= a.D) return;
    const TileDesc td = tile_from_prefix(a.dist_pfx, j);   // (L, index inside the bucket)
    const uint32_t L = td.L, kw = (L + 5u) / 6u;
    const uint32_t *key = a.keys + a.kbuckets[L].key_off + (uint64_t)td.tile * kw;
    uint32_t c = 0;   // (never absent: every key came from the table)
    if (L <= 24u) {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (uint32_t q = 0; q < 4; q++)
            if (q < kw) w[q] = __ldg(key + q);
        const uint32_t slot = hashtab::find_narrow(a.tab, hashtab::narrow_key(w[0], w[1], w[2], w[3]), L, false);
        if (slot != hashtab::kUnset) c = __ldcg(a.tab.ncnt + slot);
    } else {
        auto get = [&](uint32_t q) { return __ldg(key + q); };
        const uint64_t fp = hashtab::fingerprint(L, kw, get);
        const uint32_t slot = hashtab::find(a.tab, L, kw, fp, get, false);
        if (slot != hashtab::kUnset) c = __ldcg(a.tab.cnt + slot);
    }
    a.run_end[j] = c;
}

// ---------------------------------------------------------------- KH3: inclusive scan of the run lengths
constexpr uint32_t kScanBlk = 4096;   // elements per block (16 per thread)
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t *ws, uint32_t &total) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kHT / 32 ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < kHT / 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kHT / 32) ws[lane] = w;
    }
    __syncthreads();
    total = ws[kHT / 32 - 1];
    const uint32_t r = x + (warp ? ws[warp - 1] : 0u);
    __syncthreads();
    return r;
}
__global__ void __launch_bounds__(kHT) k_scan_reduce(uint32_t *v, uint32_t n, uint32_t *blk) {
    __shared__ uint32_t ws[kHT / 32];
    const uint32_t e0 = blockIdx.x * kScanBlk + 16u * threadIdx.x;
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < 16; q++) s += e0 + q < n ? v[e0 + q] : 0u;
    uint32_t tot;
    block_incl_scan(s, ws, tot);
    if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(1024) k_scan_blocks(uint32_t *blk, uint32_t nblk) {
    __shared__ uint32_t ws[33];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t run = 0;
    for (uint32_t b0 = 0; b0 < nblk; b0 += 1024) {
        const uint32_t b = b0 + t, v = b < nblk ? blk[b] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            ws[lane] = w;
        }
        __syncthreads();
        if (b < nblk) blk[b] = run + x + (warp ? ws[warp - 1] : 0u) - v;   // exclusive
        run += ws[31];
        __syncthreads();
    }
}
__global__ void __launch_bounds__(kHT) k_scan_apply(uint32_t *v, uint32_t n, const uint32_t *blk) {
    __shared__ uint32_t ws[kHT / 32];
    const uint32_t e0 = blockIdx.x * kScanBlk + 16u * threadIdx.x;
    uint32_t x[16], s = 0;
#pragma unroll
    for (int q = 0; q < 16; q++) {
        x[q] = e0 + q < n ? v[e0 + q] : 0u;
        s += x[q];
    }
    uint32_t tot;
    uint32_t run = block_incl_scan(s, ws, tot) - s + blk[blockIdx.x];
#pragma unroll
    for (int q = 0; q < 16; q++) {
        run += x[q];
        if (e0 + q < n) v[e0 + q] = run;
    }
}

// ---------------------------------------------------------------- KH4: each emit tile's runs
__device__ __forceinline__ uint32_t first_above(const uint32_t *ends, uint32_t lo, uint32_t hi, uint32_t w) {
    while (lo < hi) {   // first e in [lo, hi) with ends[e] > w
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(ends + mid) > w) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}
__global__ void __launch_bounds__(kHT) k_run_tiles(HashRunArgs a) {
    const uint32_t tile = blockIdx.x * kHT + threadIdx.x;
    if (tile >= a.ntiles) return;
    const TileDesc td = tile_from_prefix(a.tile_pfx, tile);
    const BucketInfo b = a.buckets[td.L];
    const uint32_t te = run_tile_words(td.L), k0 = td.tile * te, nk = min(te, b.n - k0);
    const uint32_t g0 = (uint32_t)(b.word_off - a.long_base) + k0;   // long-word index of the tile's first word
    const uint32_t lo = a.dist_pfx[td.L], hi = a.dist_pfx[td.L + 1];
    a.tile_e0[tile] = first_above(a.run_end, lo, hi, g0);
    a.tile_e1[tile] = first_above(a.run_end, lo, hi, g0 + nk - 1u);
}

// ---------------------------------------------------------------- KH5: emit the runs
// A tile = run_tile_words(L) consecutive words of bucket L, processed as segments of <= kRunSeg(L) runs:
// a segment's runs are decoded once into shared memory ("word\n", P = L + 1 bytes each, followed by its
// first 4 bytes again so that any 4 bytes of the periodic run sequence are contiguous); every thread
// assembles consecutive 16-byte chunks of the segment's output: a chunk inside one run is 4 unaligned
// 4-byte reads of that run's pattern (the phase advances by 4 mod P), a chunk crossing runs is assembled
// byte by byte; chunks shared with a neighbouring segment or tile are written byte by byte.
constexpr uint32_t kRunPatBytes = 32768;
__device__ __forceinline__ uint32_t lds_u32_unaligned(const uint8_t *base, uint32_t a) {
    const uint32_t *w = reinterpret_cast<const uint32_t *>(base + (a & ~3u));
    return __funnelshift_r(w[0], w[1], 8u * (a & 3u));
}
__global__ void __launch_bounds__(kHT) k_emit_runs(HashRunArgs a) {
    __shared__ __align__(16) uint8_t s_pat[kRunPatBytes + 16];
    __shared__ uint32_t s_end[2048];
    const uint32_t t = threadIdx.x;
    const TileDesc td = tile_from_prefix_cta(a.tile_pfx, blockIdx.x);
    const uint32_t L = td.L, P = L + 1u, PE = P + 4u, kw = (L + 5u) / 6u;
    const uint32_t rcap = min(2048u, kRunPatBytes / PE);
    const BucketInfo b = a.buckets[L];
    const uint32_t te = run_tile_words(L), k0 = td.tile * te, nk = min(te, b.n - k0);
    const uint32_t g0 = (uint32_t)(b.word_off - a.long_base) + k0;
    const uint32_t e0 = a.tile_e0[blockIdx.x], e1 = a.tile_e1[blockIdx.x];
    const BucketInfo kb = a.kbuckets[L];   // the sorted distinct keys of bucket L
    const uint32_t d0 = a.dist_pfx[L];
    const uint64_t ob = b.byte_off + (uint64_t)k0 * P;
    const uint32_t h = (uint32_t)(ob & 15u);
    uint4 *dst4 = reinterpret_cast<uint4 *>(a.words + (ob - h));
    uint8_t *dst1 = a.words + (ob - h);
    for (uint32_t sf = e0; sf <= e1; sf += rcap) {
        const uint32_t ne = min(e1 - sf + 1u, rcap);
        __syncthreads();   // the previous segment's patterns are no longer read
        for (uint32_t j = t; j < ne; j += kHT) {
            s_end[j] = min(__ldg(a.run_end + sf + j) - g0, nk);
            const uint32_t *key = a.keys + kb.key_off + (uint64_t)(sf + j - d0) * kw;
            uint8_t *p = s_pat + j * PE;
            for (uint32_t q = 0; q < kw; q++) {
                const uint32_t w = __ldg(key + q);
                for (uint32_t c = 0; c < 6u && 6u * q + c < L; c++) p[6u * q + c] = (uint8_t)(((w >> (25u - 5u * c)) & 31u) | 0x60u);
            }
            p[L] = '\n';
            for (uint32_t c = 0; c < 4u; c++) p[P + c] = p[c];
        }
        __syncthreads();
        // this segment's words [wa, wb) of the tile = bytes [wa P, wb P); chunk i covers tile bytes [16 i - h, +16)
        const uint32_t wa = sf == e0 ? 0u : min(__ldg(a.run_end + sf - 1) - g0, nk), wb = s_end[ne - 1];
        const uint32_t ba = wa * P, bb = wb * P;
        const uint32_t c0 = (h + ba) >> 4, c1 = (h + bb + 15) >> 4;
        const uint32_t magic = (uint32_t)((0x100000000ull + P - 1) / P);   // q = umulhi(y, magic) == y / P (y < 2^20)
        // each warp takes a contiguous block of chunks, its lanes interleaved (every store instruction of a
        // warp covers 512 contiguous bytes); a lane's next chunk is 512 bytes on: its run found by walking
        // forward a few runs, else by binary search
        const uint32_t warp = t >> 5, lane = t & 31, nwarp = kHT / 32;
        const uint32_t per = ((c1 - c0 + nwarp - 1) / nwarp + 31) & ~31u;
        const uint32_t wc0 = c0 + warp * per, wc1 = min(c1, wc0 + per);
        uint32_t j = 0;
        for (uint32_t i = wc0 + lane; i < wc1; i += 32) {
            const int32_t x = (int32_t)(16 * i) - (int32_t)h;   // tile-relative start of chunk i
            const uint32_t lo = x > (int32_t)ba ? (uint32_t)x : ba, hb = min((uint32_t)(x + 16), bb);
            const bool full = (int32_t)lo == x && hb == (uint32_t)(x + 16);
            uint32_t q = __umulhi(lo, magic), r = lo - q * P;
            uint32_t step = 0;
            while (s_end[j] <= q && step < 4u) {
                j++;
                step++;
            }
            if (s_end[j] <= q) {
                uint32_t hi = ne - 1;
                while (j < hi) {   // first run ending after word q
                    const uint32_t mid = (j + hi) >> 1;
                    if (s_end[mid] > q) hi = mid;
                    else j = mid + 1;
                }
            }
            uint32_t v[4] = {0u, 0u, 0u, 0u};
            if (full) {   // 4 output words; each spans <= 2 words of the text (P >= 7): branch-free
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const uint32_t rem = P - r;                                  // bytes left in word q
                    const uint32_t jn = q + 1u < s_end[j] ? j : min(j + 1u, ne - 1u);   // word q+1's run
                    const uint32_t a4 = lds_u32_unaligned(s_pat, j * PE + r);
                    const uint32_t b4 = lds_u32_unaligned(s_pat, jn * PE);
                    const uint32_t rs = 4u * min(rem, 3u);   // bytes 0..rem-1 of a4, then b4's first bytes
                    const uint32_t sel = (0x3210u & ((1u << rs) - 1u)) | ((0x7654u << rs) & 0xffffu);
                    v[u] = rem >= 4u ? a4 : __byte_perm(a4, b4, sel);
                    const bool next = rem <= 4u;
                    r = next ? 4u - rem : r + 4u;
                    q += next;
                    j = next ? jn : j;
                }
                dst4[i] = make_uint4(v[0], v[1], v[2], v[3]);
            } else {   // a chunk shared with a neighbouring segment / tile: only this segment's bytes
                for (uint32_t y = lo; y < hb; y++) {
                    dst1[16 * i + (y - (uint32_t)x)] = s_pat[j * PE + r];
                    if (++r == P) {
                        r = 0;
                        if (++q >= s_end[j] && j + 1 < ne) j++;
                    }
                }
            }
        }
    }
}

}  // namespace

cudaError_t launch_hash_gather(const HashGatherArgs &a, cudaStream_t s) {
    const uint32_t nb = (a.tab.nmask + kGatherSlots) / kGatherSlots, wb = (a.tab.mask + kGatherSlots) / kGatherSlots;
    k_hash_gather<<<nb + wb, kHT, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sort_wide(const BucketInfo *kb, const uint32_t *lens, uint32_t nlens, const uint32_t *keys_a,
                             uint32_t *keys_b, cudaStream_t s) {
    if (!nlens) return cudaSuccess;
    k_sort_wide<<<nlens, kHT, 0, s>>>(kb, lens, keys_a, keys_b);
    return cudaGetLastError();
}

cudaError_t launch_hash_runs(const HashRunArgs &a, uint32_t *scan_blk, cudaStream_t s) {
    if (!a.D) return cudaSuccess;
    k_hash_runs<<<(a.D + kHT - 1) / kHT, kHT, 0, s>>>(a);
    const uint32_t nblk = (a.D + kScanBlk - 1) / kScanBlk;
    k_scan_reduce<<<nblk, kHT, 0, s>>>(a.run_end, a.D, scan_blk);
    k_scan_blocks<<<1, 1024, 0, s>>>(scan_blk, nblk);
    k_scan_apply<<<nblk, kHT, 0, s>>>(a.run_end, a.D, scan_blk);
    if (a.ntiles) k_run_tiles<<<(a.ntiles + kHT - 1) / kHT, kHT, 0, s>>>(a);
    return cudaGetLastError();
}
uint32_t hash_scan_blocks(uint32_t D) { return (D + kScanBlk - 1) / kScanBlk; }

cudaError_t launch_hash_counts(const HashRunArgs &a, cudaStream_t s) {
    if (a.D) k_hash_runs<<<(a.D + kHT - 1) / kHT, kHT, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_scan_u32(uint32_t *v, uint32_t n, uint32_t *scan_blk, cudaStream_t s) {
    if (!n) return cudaSuccess;
    const uint32_t nblk = (n + kScanBlk - 1) / kScanBlk;
    k_scan_reduce<<<nblk, kHT, 0, s>>>(v, n, scan_blk);
    k_scan_blocks<<<1, 1024, 0, s>>>(scan_blk, nblk);
    k_scan_apply<<<nblk, kHT, 0, s>>>(v, n, scan_blk);
    return cudaGetLastError();
}

cudaError_t launch_emit_runs(const HashRunArgs &a, cudaStream_t s) {
    if (!a.ntiles) return cudaSuccess;
    k_emit_runs<<<a.ntiles, kHT, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace wsort
