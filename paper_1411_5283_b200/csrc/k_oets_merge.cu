// k_oets_merge.cu — phase 3, variant A: the paper's own sort shape on B200.
//
// PAPER.md:76 (§4): the array is cut into chunks, "each slave will do a bubble sort on own data",
// then "the final step merges all the chunks". Here a chunk is a CTA tile:
//   K4a k_oets_tile_sort   odd-even transposition sort — the data-parallel form of the paper's bubble
//                          sort — first inside each thread (E elements), then across
//                          the 32 lanes of a warp by odd-even merge-split (neighbouring lanes exchange
//                          their sorted runs and keep the lower / upper half), then the 8 warp runs
//                          of the tile are merged in shared memory along merge paths;
//   K4b k_merge_pass       merge-path merging of sorted runs (the paper's merge):
//                          each CTA finds where its output range starts in both input runs by a
//                          binary search along the cross diagonal, stages both pieces in shared
//                          memory, and every thread merges its own diagonal segment.
// Elements are S = kw (+1 with the src_off payload) u32 words, compared lexicographically; with the
// payload appended the order is (key, source offset) = the stable order (reading A6). Padding
// elements are all-ones and sort last. Ties take the left run first (stable merge).
#include "wsort_internal.cuh"

namespace wsort {
namespace {

constexpr int kMT = kMergeThreads;   // 256
constexpr uint32_t kSent = 0xffffffffu;

__device__ __forceinline__ bool le_elem(const uint32_t *x, const uint32_t *y, uint32_t S) {
    for (uint32_t u = 0; u < S; u++) {
        if (x[u] != y[u]) return x[u] < y[u];
    }
    return true;
}

__device__ __forceinline__ void copy_elem(uint32_t *d, const uint32_t *s, uint32_t S) {
    for (uint32_t u = 0; u < S; u++) d[u] = s[u];
}

// Merge path: number of elements taken from a among the first `diag` outputs of merge(a, b),
// a first on ties.
__device__ __forceinline__ uint32_t merge_path(const uint32_t *a, uint32_t na, const uint32_t *b, uint32_t nb,
                                               uint32_t diag, uint32_t S) {
    uint32_t lo = diag > nb ? diag - nb : 0u, hi = diag < na ? diag : na;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (le_elem(a + (size_t)mid * S, b + (size_t)(diag - 1 - mid) * S, S)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Sequential merge of `cnt` outputs starting at (i, j).
__device__ __forceinline__ void serial_merge(const uint32_t *a, uint32_t na, const uint32_t *b, uint32_t nb,
                                             uint32_t i, uint32_t j, uint32_t cnt, uint32_t *out, uint32_t S) {
    for (uint32_t k = 0; k < cnt; k++) {
        const bool take_a = j >= nb || (i < na && le_elem(a + (size_t)i * S, b + (size_t)j * S, S));
        if (take_a) {
            copy_elem(out + (size_t)k * S, a + (size_t)i * S, S);
            i++;
        } else {
            copy_elem(out + (size_t)k * S, b + (size_t)j * S, S);
            j++;
        }
    }
}

__device__ __forceinline__ void cmp_swap(uint32_t *x, uint32_t *y, uint32_t S) {
    if (!le_elem(x, y, S)) {
        for (uint32_t u = 0; u < S; u++) {
            const uint32_t t = x[u];
            x[u] = y[u];
            y[u] = t;
        }
    }
}


// ---------------- typed fast path: elements of S = 1 (u32) or S = 2 (u64, word 0 high) ----------------
template <typename T>
__device__ __forceinline__ T ld_elem(const uint32_t *p) {
    if constexpr (sizeof(T) == 4) return *p;
    else return ((uint64_t)p[0] << 32) | p[1];
}
template <typename T>
__device__ __forceinline__ void st_elem(uint32_t *p, T v) {
    if constexpr (sizeof(T) == 4) {
        *p = v;
    } else {
        p[0] = (uint32_t)(v >> 32);
        p[1] = (uint32_t)v;
    }
}
template <typename T>
__device__ __forceinline__ T shfl_elem(T v, int src) {
    if constexpr (sizeof(T) == 4) {
        return __shfl_sync(0xffffffffu, v, src);
    } else {
        const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
        const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
        return ((uint64_t)hi << 32) | lo;
    }
}
template <typename T>
__device__ __forceinline__ void ce(T &x, T &y) {
    const T lo = x < y ? x : y, hi = x < y ? y : x;
    x = lo;
    y = hi;
}
template <typename T>
__device__ __forceinline__ uint32_t merge_path_t(const T *a, uint32_t na, const T *b, uint32_t nb, uint32_t diag) {
    uint32_t lo = diag > nb ? diag - nb : 0u, hi = diag < na ? diag : na;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] <= b[diag - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
template <typename T>
__device__ __forceinline__ void serial_merge_t(const T *a, uint32_t na, const T *b, uint32_t nb, uint32_t i,
                                               uint32_t j, uint32_t cnt, T *out) {
    for (uint32_t k = 0; k < cnt; k++) {
        const bool take_a = j >= nb || (i < na && a[i] <= b[j]);
        out[k] = take_a ? a[i++] : b[j++];
    }
}

// Tile sort with the 8 elements of each thread in registers: odd-even transposition inside the
// thread, then odd-even merge-split across groups of 8 lanes through warp shuffles (the merge-split
// of two sorted runs is min/max against the reversed partner run + a bitonic clean-up), then merge
// paths in shared memory: 64 -> 128 -> ... -> 2048.
template <typename T>
__device__ __forceinline__ void tile_sort_reg(const OetsArgs &a, const BucketInfo &b, uint32_t tile, uint32_t *smem) {
    constexpr int E = 8;
    constexpr uint32_t TN = kMT * E;
    const int t = threadIdx.x, lane = t & 31;
    const uint32_t kw = b.kw, S = b.estride;
    const uint32_t k0 = tile * TN, nk = min(TN, b.n - k0);
    T v[E];
    const uint32_t *ks = a.keys_in + b.key_off + (uint64_t)k0 * kw;
#pragma unroll
    for (int e = 0; e < E; e++) {
        const uint32_t idx = t * E + e;
        if (idx < nk) {
            if constexpr (sizeof(T) == 8) {
                if (S == kw) v[e] = ld_elem<T>(ks + (size_t)idx * kw);          // two key words
                else v[e] = ((T)__ldg(ks + idx) << 32) | __ldg(a.pay_in + b.word_off + k0 + idx);   // key, payload
            } else {
                v[e] = __ldg(ks + idx);                                          // one key word
            }
        } else {
            v[e] = (T)~(T)0;
        }
    }
    // (1) odd-even transposition within the thread
#pragma unroll
    for (int ph = 0; ph < E; ph++)
#pragma unroll
        for (int i = ph & 1; i + 1 < E; i += 2) ce(v[i], v[i + 1]);
    // (2) odd-even merge-split across the 8 lanes of each lane group
    const int g = lane & 7;
#pragma unroll 1
    for (int ph = 0; ph < 8; ph++) {
        const bool lower = (g & 1) == (ph & 1);
        const int pg = lower ? g + 1 : g - 1;
        const bool active = pg >= 0 && pg < 8;
        const int src = active ? (lane - g + pg) : lane;
        T o[E];
#pragma unroll
        for (int e = 0; e < E; e++) o[e] = shfl_elem(v[e], src);
        if (active) {
#pragma unroll
            for (int e = 0; e < E; e++) {
                const T x = v[e], y = o[E - 1 - e];
                v[e] = lower ? (x < y ? x : y) : (x < y ? y : x);
            }
            // v is bitonic: bitonic merge to ascending
#pragma unroll
            for (int d = E / 2; d >= 1; d >>= 1)
#pragma unroll
                for (int i = 0; i < E; i++)
                    if ((i & d) == 0) ce(v[i], v[i + d]);
        }
    }
    // (3) merge paths in shared memory
    T *buf0 = reinterpret_cast<T *>(smem), *buf1 = buf0 + TN;
#pragma unroll
    for (int e = 0; e < E; e++) buf0[t * E + e] = v[e];
    __syncthreads();
    T *src = buf0, *dst = buf1;
    for (uint32_t run = 8 * E; run < TN; run *= 2) {
        const uint32_t o = t * E;
        const uint32_t pair = o / (2 * run), d = o - pair * 2 * run;
        const T *ra = src + pair * 2 * run, *rb = ra + run;
        const uint32_t i = merge_path_t(ra, run, rb, run, d);
        serial_merge_t(ra, run, rb, run, i, d - i, E, dst + o);
        __syncthreads();
        T *sw = src;
        src = dst;
        dst = sw;
    }
    uint32_t *out = a.out + b.elem_off + (uint64_t)k0 * S;
    for (uint32_t i = t; i < nk; i += kMT) st_elem<T>(out + (size_t)i * S, src[i]);
}

// K4a: sort one tile of E * kMT elements of one bucket (generic element width).
__device__ __forceinline__ void tile_sort_generic(const OetsArgs &a, const TileDesc td, const BucketInfo &b,
                                                  uint32_t *sm) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t kw = b.kw, S = b.estride, E = b.tile_keys / kMT;
    const uint32_t T = b.tile_keys, k0 = td.tile * T, nk = min(T, b.n - k0);
    uint32_t *X = sm, *Y = sm + (size_t)T * S;

    // load (key words from the K3 buckets, payload appended when present), pad with sentinels
    const uint32_t *ks = a.keys_in + b.key_off + (uint64_t)k0 * kw;
    for (uint32_t i = t; i < T * kw; i += kMT) {
        const uint32_t e = i / kw, u = i - e * kw;
        X[(size_t)e * S + u] = e < nk ? __ldg(ks + i) : kSent;
    }
    if (S > kw) {
        const uint32_t *ps = a.pay_in + b.word_off + k0;
        for (uint32_t e = t; e < T; e += kMT) X[(size_t)e * S + kw] = e < nk ? __ldg(ps + e) : kSent;
    }
    __syncthreads();

    // (1) odd-even transposition sort of the thread's own E elements (bubble sort, in parallel)
    uint32_t *mine = X + (size_t)t * E * S;
    for (uint32_t ph = 0; ph < E; ph++)
        for (uint32_t i = ph & 1u; i + 1 < E; i += 2) cmp_swap(mine + i * S, mine + (i + 1) * S, S);
    __syncwarp();

    // (2) odd-even merge-split across the 32 lanes of the warp (32 phases)
    uint32_t *tmp = Y + (size_t)t * E * S;
    for (int ph = 0; ph < 32; ph++) {
        const bool lower = (lane & 1) == (ph & 1);
        const int partner = lower ? lane + 1 : lane - 1;
        if (partner >= 0 && partner < 32) {
            const uint32_t *other = X + (size_t)(warp * 32 + partner) * E * S;
            if (lower) {   // keep the E smallest of mine + other, ascending
                uint32_t i = 0, j = 0;
                for (uint32_t k = 0; k < E; k++) {
                    if (j >= E || (i < E && le_elem(mine + i * S, other + j * S, S))) copy_elem(tmp + k * S, mine + (i++) * S, S);
                    else copy_elem(tmp + k * S, other + (j++) * S, S);
                }
            } else {       // keep the E largest, filled from the back (other first on ties: stable)
                int i = (int)E - 1, j = (int)E - 1;
                for (int k = (int)E - 1; k >= 0; k--) {
                    if (j < 0 || (i >= 0 && !le_elem(mine + i * S, other + j * S, S))) copy_elem(tmp + k * S, mine + (i--) * S, S);
                    else copy_elem(tmp + k * S, other + (j--) * S, S);
                }
            }
        }
        __syncwarp();
        if (partner >= 0 && partner < 32) copy_elem(mine, tmp, E * S);
        __syncwarp();
    }
    __syncthreads();

    // (3) merge the warp runs of the tile along merge paths: 32E -> 64E -> ... -> T
    uint32_t *src = X, *dst = Y;
    for (uint32_t run = 32 * E; run < T; run *= 2) {
        const uint32_t o = t * E;                  // this thread's first output
        const uint32_t pair = o / (2 * run), d = o - pair * 2 * run;
        const uint32_t *ra = src + (size_t)pair * 2 * run * S, *rb = ra + (size_t)run * S;
        const uint32_t i = merge_path(ra, run, rb, run, d, S);
        serial_merge(ra, run, rb, run, i, d - i, E, dst + (size_t)o * S, S);
        __syncthreads();
        uint32_t *sw = src;
        src = dst;
        dst = sw;
    }

    // write the sorted tile (element layout S words)
    uint32_t *out = a.out + b.elem_off + (uint64_t)k0 * S;
    for (uint32_t i = t; i < nk * S; i += kMT) out[i] = src[i];
}

__global__ void __launch_bounds__(kMT) k_oets_tile_sort(OetsArgs a) {
    extern __shared__ __align__(16) uint32_t sm[];
    const TileDesc td = a.tiles[blockIdx.x];
    const BucketInfo b = a.buckets[td.L];
    if (b.estride == 1) tile_sort_reg<uint32_t>(a, b, td.tile, sm);
    else if (b.estride == 2) tile_sort_reg<uint64_t>(a, b, td.tile, sm);
    else tile_sort_generic(a, td, b, sm);
}

// Merge-path split of every merge tile's first output (one thread per tile, all in parallel, so the
// dependent global-memory binary searches overlap instead of stalling each merge CTA).
__global__ void __launch_bounds__(256) k_merge_split(MergeArgs a) {
    const uint32_t j = blockIdx.x * 256 + threadIdx.x;
    if (j >= a.ntiles) return;
    const TileDesc td = a.tiles[j];
    const BucketInfo b = a.buckets[td.L];
    const uint32_t S = b.estride, n = b.n, run = b.tile_keys << a.pass;
    const uint32_t o0 = td.tile * b.tile_keys;
    const uint32_t p0 = (o0 / (2 * run)) * 2 * run;
    const uint32_t na = min(run, n - p0);
    const uint32_t nb = n - p0 > run ? min(run, n - p0 - run) : 0u;
    const uint32_t *ra = a.in + b.elem_off + (uint64_t)p0 * S;
    const uint32_t *rb = ra + (size_t)na * S;
    uint32_t r;
    if (S == 1) r = merge_path_t(ra, na, rb, nb, o0 - p0);
    else r = merge_path(ra, na, rb, nb, o0 - p0, S);
    a.splits[j] = r;
}

// K4b: one merge pass over every bucket with runs left: runs of `run_len(L)` elements are merged
// pairwise; this CTA produces outputs [o0, o0 + TO) of the bucket.
__global__ void __launch_bounds__(kMT) k_merge_pass(MergeArgs a) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int t = threadIdx.x;
    const TileDesc td = a.tiles[blockIdx.x];
    const BucketInfo b = a.buckets[td.L];
    const uint32_t S = b.estride, n = b.n;
    const uint32_t TO = b.tile_keys;                      // output tile = sort tile
    const uint32_t run = b.tile_keys << a.pass;
    const uint32_t o0 = td.tile * TO, o1 = min(o0 + TO, n);
    const uint32_t p0 = (o0 / (2 * run)) * 2 * run;       // pair start (a tile never crosses a pair:
    const uint32_t na = min(run, n - p0);                 //  2*run is a multiple of TO)
    const uint32_t nb = n - p0 > run ? min(run, n - p0 - run) : 0u;
    const uint32_t *base = a.in + b.elem_off + (uint64_t)p0 * S;
    const uint32_t *ra = base, *rb = base + (size_t)na * S;
    const uint32_t d0 = o0 - p0, d1 = o1 - p0;
    const uint32_t i0 = a.splits[blockIdx.x];
    const uint32_t i1 = d1 == na + nb ? na : a.splits[blockIdx.x + 1];   // next tile: same pair
    const uint32_t j0 = d0 - i0, j1 = d1 - i1;
    const uint32_t ca = i1 - i0, cb = j1 - j0;
    // stage both pieces
    uint32_t *sa = sm, *sb = sm + (size_t)ca * S, *so = sm + (size_t)(ca + cb) * S;
    for (uint32_t x = t; x < ca * S; x += kMT) sa[x] = __ldg(ra + (size_t)i0 * S + x);
    for (uint32_t x = t; x < cb * S; x += kMT) sb[x] = __ldg(rb + (size_t)j0 * S + x);
    __syncthreads();
    const uint32_t cnt = ca + cb, per = (cnt + kMT - 1) / kMT;
    const uint32_t d = min(t * per, cnt), e = min(d + per, cnt);
    if (d < e) {
        const uint32_t i = merge_path(sa, ca, sb, cb, d, S);
        serial_merge(sa, ca, sb, cb, i, d - i, e - d, so + (size_t)d * S, S);
    }
    __syncthreads();
    uint32_t *out = a.out + b.elem_off + (uint64_t)o0 * S;
    for (uint32_t x = t; x < cnt * S; x += kMT) out[x] = so[x];
}

}  // namespace

cudaError_t launch_oets_tile_sort(const OetsArgs &a, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    const size_t smem = (size_t)a.max_tile_words * 2 * 4;
    cudaError_t e = cudaFuncSetAttribute(k_oets_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_oets_tile_sort<<<a.ntiles, kMT, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_merge_pass(const MergeArgs &a, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    k_merge_split<<<(a.ntiles + 255) / 256, 256, 0, s>>>(a);
    const size_t smem = (size_t)a.max_tile_words * 2 * 4;
    cudaError_t e = cudaFuncSetAttribute(k_merge_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_merge_pass<<<a.ntiles, kMT, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace wsort
