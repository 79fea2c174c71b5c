// k_tokenize.cu — phase 2 of the method (§3 Methodology, Pre-processing), the path
// used by the stable / legacy sorts (src_off, LSD radix, OETS + merge, multi-GPU packing):
//   K2a k_bucket_offsets  the per-length sub-array sizes "decided depending on a number of elements
//                         with the same number of characters": exclusive prefix off[]
//                         of the length histogram K1 (k_ingest.cu) accumulated;
//   K2b k_cta_bases       per-(CTA, length) scatter bases for K3;
//   K3 k_tokenize<1|2>    re-tokenize, pack each word into its fixed-width key (the paper's
//                         "array char 3D") and scatter it into its length's sub-array
//                         ("all shorter words come before longer words"); mode 2 is stable.
//
// Layout: each CTA owns a contiguous run of 8 KiB steps (the same byte ranges K1 histograms). A step
// is staged in shared memory with 16 bytes before it and a 256-byte halo after it; each thread
// classifies 32 bytes with SWAR arithmetic into a 32-bit letter mask, word starts/ends come from
// mask shifts, and a block scan compacts them into ordered start/end lists. A word belongs to the
// step holding its first letter.
#include "wsort_internal.cuh"
#include "k_text.cuh"

namespace wsort {
namespace {

using namespace text;

struct TkCommon {
    uint4 buf[kTkBuf / 16 + 1];   // +16 B slack: key packing reads whole 32-bit words
    uint16_t sstart[kTkMaxWords];
    uint16_t send[kTkMaxWords + 2];
    uint32_t warp_tot[kTkThreads / 32];
    uint32_t totals;
    uint32_t skip;
    uint32_t qw[2 * (kTkThreads / 32) + 1];
};

struct TkCountSmem {
    TkCommon c;
    uint32_t hist[kHistBins];
};

struct TkScatterSmem {
    TkCommon c;
    uint32_t wl[kTkMaxWords];          // L | warp << 8 | rank << 11
    uint32_t wcnt[kTkThreads / 32][256];
    uint32_t run[256];
    uint64_t key_off[256];
    uint64_t word_off[256];
};

// Stage step `st` and build its ordered word start / end lists. Returns the number of words whose
// first letter lies in the step (S); send[k + skip] is the last letter of word k.
constexpr int kTkPf = (kTkBuf / 16 + kTkThreads - 1) / kTkThreads;   // uint4 per thread per step

// Issue the global loads of step `st` into registers (consumed by the next stage_step).
__device__ __forceinline__ void prefetch_step(uint4 (&pf)[kTkPf], const uint8_t *__restrict__ text, uint64_t s0) {
    const int t = threadIdx.x;
    const uint4 *src = reinterpret_cast<const uint4 *>(text + s0 - kTkPre);
#pragma unroll
    for (int r = 0; r < kTkPf; r++) {
        const int i = t + r * kTkThreads;
        if (i < kTkBuf / 16) pf[r] = __ldg(src + i);
    }
}

// Store a prefetched step into shared memory, then prefetch the next one (in flight while this step
// is processed).
__device__ __forceinline__ uint32_t stage_step(TkCommon &sm, uint4 (&pf)[kTkPf], const uint8_t *__restrict__ text,
                                               uint64_t next_s0, bool has_next) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
    for (int r = 0; r < kTkPf; r++) {
        const int i = t + r * kTkThreads;
        if (i < kTkBuf / 16) sm.buf[i] = pf[r];
    }
    __syncthreads();
    if (has_next) prefetch_step(pf, text, next_s0);

    const uint8_t *sb = reinterpret_cast<const uint8_t *>(sm.buf) + kTkPre;
    uint4 a = sm.buf[1 + 2 * t], b = sm.buf[2 + 2 * t];
    uint32_t M = letter_mask32(a, b);
    uint32_t p = is_letter(sb[32 * t - 1]), nx = is_letter(sb[32 * t + 32]);
    uint32_t starts = M & ~((M << 1) | p);
    uint32_t ends = M & ~((M >> 1) | (nx << 31));
    uint32_t v = __popc(starts) | (__popc(ends) << 16);

    // block exclusive scan of packed (starts, ends) counts
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sm.warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t wt = lane < kTkThreads / 32 ? sm.warp_tot[lane] : 0;
        uint32_t wi = wt;
#pragma unroll
        for (int o = 1; o < kTkThreads / 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(kFull, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kTkThreads / 32) sm.warp_tot[lane] = wi - wt;   // exclusive warp offsets
        if (lane == kTkThreads / 32 - 1) sm.totals = wi;
        if (lane == 0) sm.skip = (is_letter(sb[-1]) && is_letter(sb[0])) ? 1u : 0u;
    }
    __syncthreads();
    uint32_t excl = sm.warp_tot[warp] + incl - v;
    uint32_t ps = excl & 0xffffu, pe = excl >> 16;
    const uint32_t base = 32u * t;
    while (starts) {
        sm.sstart[ps++] = (uint16_t)(base + __ffs(starts) - 1);
        starts &= starts - 1;
    }
    while (ends) {
        sm.send[pe++] = (uint16_t)(base + __ffs(ends) - 1);
        ends &= ends - 1;
    }
    const uint32_t tot = sm.totals;
    const uint32_t S = tot & 0xffffu, E = tot >> 16;
    if (t == kTkThreads - 1 && is_letter(sb[kTkStep - 1]) && is_letter(sb[kTkStep])) {
        // the last word continues past the step: find its end in the halo (reading A7 bounds it)
        int i = kTkStep;
        while (i < kTkStep + kTkHalo && is_letter(sb[i])) i++;
        sm.send[E] = (i < kTkStep + kTkHalo) ? (uint16_t)(i - 1) : (uint16_t)0xffff;
    }
    __syncthreads();
    return S;
}

// kMode: 1 = K3 scatter, any order within a (CTA, length) run (keys only: the sort that follows
// fixes the order of distinct keys, and equal keys are identical words); 2 = K3 scatter, stable (text
// order within each length; needed for the src_off payload).
template <int kMode>
__global__ void __launch_bounds__(kTkThreads) k_tokenize(TkArgs a) {
    extern __shared__ __align__(16) uint8_t tk_smem[];
    auto &sm = *reinterpret_cast<TkScatterSmem *>(tk_smem);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t c = blockIdx.x;
    const uint32_t st0 = c * a.steps_per_cta;
    const uint32_t st1 = min(st0 + a.steps_per_cta, a.nsteps);

    for (int w = 0; w < kTkThreads / 32; w++) sm.wcnt[w][t] = 0;
    sm.run[t] = a.cta_base[(size_t)c * 256 + t];
    sm.key_off[t] = a.buckets[t].key_off;
    sm.word_off[t] = a.buckets[t].word_off;
    // (the first stage_step's __syncthreads orders these initialisations)

    uint4 pf[kTkPf];
    if (st0 < st1) prefetch_step(pf, a.text, (uint64_t)st0 * kTkStep);
    for (uint32_t st = st0; st < st1; st++) {
        const uint64_t s0 = (uint64_t)st * kTkStep;
        // words are dealt round-robin from the ordered lists (even load per thread)
        const uint32_t S = stage_step(sm.c, pf, a.text, s0 + kTkStep, st + 1 < st1);
        const uint32_t skip = sm.c.skip;
        if constexpr (kMode == 1) {
            const uint32_t *buf32 = reinterpret_cast<const uint32_t *>(sm.c.buf);
            for (uint32_t k = t; k < S; k += kTkThreads) {
                const uint32_t start = sm.c.sstart[k];
                const uint32_t L = (uint32_t)sm.c.send[k + skip] - start + 1u;
                const uint32_t idx = atomicAdd(&sm.run[L], 1u);
                const uint32_t kw = (L + 5) / 6;
                uint32_t *dst = a.keys + sm.key_off[L] + (uint64_t)idx * kw;
                if (L <= 192) pack_key(buf32, kTkPre + start, L, kw, dst);   // (its window reads <= 12 bytes past the word)
                else for (uint32_t q = 0; q < kw; q++) dst[q] = pack6(buf32, kTkPre + start + 6 * q, L - 6 * q);
            }
            __syncthreads();
        } else {
            // Phase A: warp w ranks words [kb, ke) by length, in text order (stable).
            const uint32_t kb = (S * warp) / (kTkThreads / 32), ke = (S * (warp + 1)) / (kTkThreads / 32);
            for (uint32_t i = kb; i < ke; i += 32) {
                uint32_t k = i + lane;
                bool v = k < ke;
                uint32_t L = v ? (uint32_t)sm.c.send[k + skip] - sm.c.sstart[k] + 1u : 0u;
                uint32_t peers = __match_any_sync(kFull, L);
                uint32_t before = v ? sm.wcnt[warp][L & 255] : 0u;
                __syncwarp();
                if (v && lane == __ffs(peers) - 1) sm.wcnt[warp][L] = before + __popc(peers);
                __syncwarp();
                if (v) sm.wl[k] = L | ((uint32_t)warp << 8) | ((before + __popc(peers & lanemask_lt())) << 11);
            }
            __syncthreads();
            // Phase B: per length, exclusive scan over warps on top of this CTA's running base.
            {
                uint32_t run = sm.run[t];
#pragma unroll
                for (int w = 0; w < kTkThreads / 32; w++) {
                    uint32_t x = sm.wcnt[w][t];
                    sm.wcnt[w][t] = run;
                    run += x;
                }
                sm.run[t] = run;
            }
            __syncthreads();
            // Phase C: pack keys and scatter them into their buckets.
            for (uint32_t k = t; k < S; k += kTkThreads) {
                uint32_t x = sm.wl[k];
                uint32_t L = x & 255u, w = (x >> 8) & 7u, r = x >> 11;
                uint32_t idx = sm.wcnt[w][L] + r;
                uint32_t start = sm.c.sstart[k];
                const uint32_t kw = (L + 5) / 6;
                uint32_t *dst = a.keys + sm.key_off[L] + (uint64_t)idx * kw;
                const uint32_t *buf32 = reinterpret_cast<const uint32_t *>(sm.c.buf);
                if (L <= 192) pack_key(buf32, kTkPre + start, L, kw, dst);   // (its window reads <= 12 bytes past the word)
                else for (uint32_t q = 0; q < kw; q++) dst[q] = pack6(buf32, kTkPre + start + 6 * q, L - 6 * q);
                if (a.payload) a.payload[sm.word_off[L] + idx] = (uint32_t)(s0 + start);
            }
            __syncthreads();
            for (int w = 0; w < kTkThreads / 32; w++) sm.wcnt[w][t] = 0;
            // the next stage_step's first __syncthreads orders this reset before phase A
        }
    }
}

// K1b (legacy paths only): per-CTA length histograms over K3's byte ranges, for K2b's scatter bases.
// (K1 ingest counts the words of L <= 5 in dense tables instead of a per-CTA histogram.)
__global__ void __launch_bounds__(kTkThreads) k_count_lengths(TkArgs a, uint32_t *ghist) {
    extern __shared__ __align__(16) uint8_t tk_smem[];
    auto &sm = *reinterpret_cast<TkCountSmem *>(tk_smem);
    const int t = threadIdx.x;
    const uint32_t c = blockIdx.x;
    const uint32_t st0 = c * a.steps_per_cta;
    const uint32_t st1 = min(st0 + a.steps_per_cta, a.nsteps);
    for (int i = t; i < kHistBins; i += kTkThreads) sm.hist[i] = 0;
    uint4 pf[kTkPf];
    if (st0 < st1) prefetch_step(pf, a.text, (uint64_t)st0 * kTkStep);
    for (uint32_t st = st0; st < st1; st++) {
        const uint64_t s0 = (uint64_t)st * kTkStep;
        const uint32_t S = stage_step(sm.c, pf, a.text, s0 + kTkStep, st + 1 < st1);
        const uint32_t skip = sm.c.skip;
        for (uint32_t k = t; k < S; k += kTkThreads) {
            const uint32_t e = sm.c.send[k + skip];
            const uint32_t L = e == 0xffffu ? 256u : e - sm.c.sstart[k] + 1u;
            atomicAdd(&sm.hist[min(L, 256u)], 1u);
        }
        __syncthreads();
    }
    __syncthreads();
    for (int i = t; i < kHistBins; i += kTkThreads) {
        const uint32_t h = sm.hist[i];
        a.cta_hist[(size_t)c * kHistBins + i] = h;
        if (h && ghist) atomicAdd(&ghist[i], h);
    }
}

// K2a: the length histogram (accumulated by K1 in ghist) -> off[], key_off[], byte_off[], W, Lmax.
__global__ void __launch_bounds__(256) k_bucket_offsets(const uint32_t *ghist, Summary *sum) {
    __shared__ uint64_t s_hist[256];
    const int L = threadIdx.x;
    s_hist[L] = ghist[L];
    __syncthreads();
    if (L == 0) {
        uint64_t o = 0, ko = 0, bo = 0, letters = 0;
        uint32_t lmax = 0;
        for (int l = 0; l < 256; l++) {
            sum->off[l] = o;
            sum->key_off[l] = ko;
            sum->byte_off[l] = bo;
            uint64_t h = s_hist[l];
            o += h;
            ko += h * (uint64_t)kw_of(l);
            bo += h * (uint64_t)(l + 1);
            letters += h * (uint64_t)l;
            if (h) lmax = l;
        }
        sum->off[256] = o;
        sum->key_off[256] = ko;
        sum->byte_off[256] = bo;
        sum->n_words = o;
        sum->letters = letters;
        sum->max_len = lmax;
        sum->too_long = ghist[256];
    }
}

// K2b (only for K3): per-(CTA, length) scatter bases = exclusive prefix over CTAs of K1's per-CTA
// histograms. One CTA per length; a block scan over the CTAs.
__global__ void __launch_bounds__(256) k_cta_bases(TkArgs a) {
    __shared__ uint32_t wsum[9];
    const uint32_t L = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t run = 0;
    for (uint32_t c0 = 0; c0 < a.grid; c0 += 256) {
        const uint32_t c = c0 + t;
        const uint32_t v = c < a.grid ? a.cta_hist[(size_t)c * kHistBins + L] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = lane < 8 ? wsum[lane] : 0u;
            uint32_t wi = w;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, wi, o);
                if (lane >= o) wi += y;
            }
            if (lane < 8) wsum[lane] = wi - w;
            if (lane == 7) wsum[8] = wi;
        }
        __syncthreads();
        if (c < a.grid) a.cta_base[(size_t)c * 256 + L] = run + wsum[warp] + incl - v;
        run += wsum[8];
        __syncthreads();
    }
}

}  // namespace

cudaError_t launch_bucket_offsets(const uint32_t *ghist, Summary *d_sum, cudaStream_t s) {
    k_bucket_offsets<<<1, 256, 0, s>>>(ghist, d_sum);
    return cudaGetLastError();
}

cudaError_t launch_count_lengths(const TkArgs &a, uint32_t *ghist, cudaStream_t s) {
    if (a.grid == 0) return cudaSuccess;
    k_count_lengths<<<a.grid, kTkThreads, sizeof(TkCountSmem), s>>>(a, ghist);
    return cudaGetLastError();
}

cudaError_t launch_cta_bases(const TkArgs &a, uint32_t max_len, cudaStream_t s) {
    if (a.grid == 0 || max_len == 0) return cudaSuccess;
    k_cta_bases<<<max_len + 1, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pack_scatter(const TkArgs &a, cudaStream_t s) {
    if (a.grid == 0) return cudaSuccess;
    cudaError_t e;
    if (a.payload) {
        e = cudaFuncSetAttribute(k_tokenize<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TkScatterSmem));
        if (e != cudaSuccess) return e;
        k_tokenize<2><<<a.grid, kTkThreads, sizeof(TkScatterSmem), s>>>(a);
    } else {
        e = cudaFuncSetAttribute(k_tokenize<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TkScatterSmem));
        if (e != cudaSuccess) return e;
        k_tokenize<1><<<a.grid, kTkThreads, sizeof(TkScatterSmem), s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace wsort
