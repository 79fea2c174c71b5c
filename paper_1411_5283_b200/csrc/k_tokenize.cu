// k_tokenize.cu — phases 1 and 2 of the method (§3 Methodology, Pre-processing):
//   K1 k_tokenize<0>      "removing / ignoring the special characters": find every maximal run of
//                         ASCII letters (reading A1) and count words per length, per CTA;
//   K2 k_bucket_offsets   the per-length sub-array sizes "decided depending on a number of elements
//                         with the same number of characters": length histogram,
//                         exclusive prefix off[], per-(CTA, length) scatter bases;
//   K3 k_tokenize<1|2>    re-tokenize, pack each word into its fixed-width key (the paper's
//                         "array char 3D") and scatter it, stably, into its length's
//                         sub-array ("all shorter words come before longer words").
//
// Layout: each CTA owns a contiguous run of 8 KiB steps. A step is staged in shared memory with
// 16 bytes before it and a 256-byte halo after it; each thread classifies 32 bytes with SWAR
// arithmetic into a 32-bit letter mask, word starts/ends come from mask shifts, and a block scan
// compacts them into ordered start/end lists. A word belongs to the step holding its first letter.
#include "wsort_internal.cuh"

namespace wsort {
namespace {

constexpr uint32_t kFull = 0xffffffffu;

// 4 bytes -> 4-bit letter mask (bit i = byte i is in [A-Za-z]).
__device__ __forceinline__ uint32_t letter_nibble(uint32_t x) {
    uint32_t w = (x | 0x20202020u) & 0x7f7f7f7fu;   // fold case, drop bit 7
    uint32_t a = w + 0x1f1f1f1fu;                    // bit 7 set iff w >= 'a'
    uint32_t b = w + 0x05050505u;                    // bit 7 set iff w >= '{'
    uint32_t m = a & ~b & ~x & 0x80808080u;          // and the original byte < 0x80
    return ((m >> 7) * 0x10204080u) >> 28;           // gather bits 7,15,23,31
}

__device__ __forceinline__ uint32_t letter_mask32(uint4 a, uint4 b) {
    return letter_nibble(a.x) | (letter_nibble(a.y) << 4) | (letter_nibble(a.z) << 8) |
           (letter_nibble(a.w) << 12) | (letter_nibble(b.x) << 16) | (letter_nibble(b.y) << 20) |
           (letter_nibble(b.z) << 24) | (letter_nibble(b.w) << 28);
}

__device__ __forceinline__ bool is_letter(uint8_t c) { return (uint8_t)((c | 0x20) - 'a') < 26; }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Pack letters [0, min(L,6)) of the word at sb[start] into one key word (letter j -> bits 29-5j..25-5j).
__device__ __forceinline__ uint32_t pack6(const uint32_t *buf32, uint32_t boff, uint32_t L) {
    const uint32_t a = boff >> 2, sh = 8u * (boff & 3u);
    const uint32_t w0 = buf32[a], w1 = buf32[a + 1], w2 = buf32[a + 2];
    const uint32_t lo = __funnelshift_r(w0, w1, sh) & 0x1f1f1f1fu;   // codes of letters 0..3
    const uint32_t hi = __funnelshift_r(w1, w2, sh) & 0x00001f1fu;   // codes of letters 4..5
    const uint32_t r = __byte_perm(lo, 0, 0x0123);                   // letter 0 in the top byte
    const uint32_t t1 = (r & 0x001f001fu) | ((r & 0x1f001f00u) >> 3);
    const uint32_t t2 = (t1 & 0x3ffu) | ((t1 >> 16) << 10);           // 4 letters, 20 bits
    const uint32_t u = ((hi & 0x1fu) << 5) | (hi >> 8);                // letters 4, 5
    uint32_t key = (t2 << 10) | u;
    if (L < 6) key &= ~((1u << (5u * (6u - L))) - 1u);
    return key;
}

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

// kMode: 0 = K1 count; 1 = K3 scatter, any order within a (CTA, length) run (keys only: the sort
// that follows fixes the order of distinct keys, and equal keys are identical words);
// 2 = K3 scatter, stable (text order within each length; needed for the src_off payload).
// List-free variant for K1 and the unordered K3: each thread keeps its own segment's word-start and
// word-end masks; a word that runs past the segment end takes its remaining length from `carry`, the
// length of the letter run that starts at the next segment's first byte (a suffix scan over the
// threads of the run-combining operator (l1,f1)+(l2,f2) = (l1 + f1*l2, f1 & f2), where l is the
// number of leading letters of a segment and f says the segment is all letters).
struct SegRuns {
    uint32_t starts, ends, carry;
};

__device__ __forceinline__ SegRuns stage_step_runs(TkCommon &sm, uint32_t *qw, uint4 (&pf)[kTkPf],
                                                   const uint8_t *__restrict__ text, uint64_t next_s0, bool has_next) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
    for (int r = 0; r < kTkPf; r++) {
        const int i = t + r * kTkThreads;
        if (i < kTkBuf / 16) sm.buf[i] = pf[r];
    }
    __syncthreads();
    if (has_next) prefetch_step(pf, text, next_s0);
    const uint8_t *sb = reinterpret_cast<const uint8_t *>(sm.buf) + kTkPre;
    const uint32_t M = letter_mask32(sm.buf[1 + 2 * t], sm.buf[2 + 2 * t]);
    const uint32_t p = is_letter(sb[32 * t - 1]), nx = is_letter(sb[32 * t + 32]);
    SegRuns r;
    r.starts = M & ~((M << 1) | p);
    r.ends = M & ~((M >> 1) | (nx << 31));
    const uint32_t full = M == 0xffffffffu;
    uint32_t l = full ? 32u : (uint32_t)(__ffs(~M) - 1), f = full;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t l2 = __shfl_down_sync(kFull, l, o), f2 = __shfl_down_sync(kFull, f, o);
        if (lane + o < 32 && f) {
            l += l2;
            f = f2;
        }
    }
    if (lane == 0) qw[warp] = l | (f << 31);
    __syncthreads();
    if (t == 0) {   // chain the warps from the right, starting from the letters at the halo's head
        uint32_t i = kTkStep;
        while (i < kTkStep + kTkHalo && is_letter(sb[i])) i++;
        uint32_t q = i - kTkStep;
        qw[kTkThreads / 32 * 2] = q;
        for (int w = kTkThreads / 32 - 1; w >= 0; w--) {
            const uint32_t x = qw[w];
            q = (x & 0x7fffffffu) + ((x >> 31) ? q : 0u);
            qw[kTkThreads / 32 + w] = q;   // run starting at warp w's first byte
        }
    }
    __syncthreads();
    const uint32_t qnext = warp + 1 < kTkThreads / 32 ? qw[kTkThreads / 32 + warp + 1] : qw[kTkThreads / 32 * 2];
    const uint32_t l1 = __shfl_down_sync(kFull, l, 1), f1 = __shfl_down_sync(kFull, f, 1);
    r.carry = lane < 31 ? l1 + (f1 ? qnext : 0u) : qnext;
    return r;
}

// Visit the words that start in this thread's segment: fn(start byte within the step, length).
template <class F>
__device__ __forceinline__ void for_each_word(const SegRuns &r, F fn) {
    const int t = threadIdx.x;
    uint32_t m = r.starts;
    while (m) {
        const uint32_t s = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t em = r.ends & (0xffffffffu << s);
        const uint32_t L = em ? (uint32_t)(__ffs(em) - 1) - s + 1u : (32u - s) + r.carry;
        fn(32u * t + s, L);
    }
}

template <int kMode>
struct SmemOf { using type = TkScatterSmem; };
template <>
struct SmemOf<0> { using type = TkCountSmem; };

template <int kMode>
__global__ void __launch_bounds__(kTkThreads) k_tokenize(TkArgs a) {
    constexpr bool kScatter = kMode != 0;
    extern __shared__ __align__(16) uint8_t tk_smem[];
    auto &sm = *reinterpret_cast<typename SmemOf<kMode>::type *>(tk_smem);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t c = blockIdx.x;
    const uint32_t st0 = c * a.steps_per_cta;
    const uint32_t st1 = min(st0 + a.steps_per_cta, a.nsteps);

    if constexpr (!kScatter) {
        for (int i = t; i < kHistBins; i += kTkThreads) sm.hist[i] = 0;
    } else {
        for (int w = 0; w < kTkThreads / 32; w++) sm.wcnt[w][t] = 0;
        sm.run[t] = a.cta_base[(size_t)c * 256 + t];
        sm.key_off[t] = a.buckets[t].key_off;
        sm.word_off[t] = a.buckets[t].word_off;
    }
    // (the first stage_step's __syncthreads orders these initialisations)

    uint4 pf[kTkPf];
    if (st0 < st1) prefetch_step(pf, a.text, (uint64_t)st0 * kTkStep);
    for (uint32_t st = st0; st < st1; st++) {
        const uint64_t s0 = (uint64_t)st * kTkStep;
        if constexpr (kMode == 0) {
            const SegRuns r = stage_step_runs(sm.c, sm.c.qw, pf, a.text, s0 + kTkStep, st + 1 < st1);
            for_each_word(r, [&](uint32_t, uint32_t L) { atomicAdd(&sm.hist[min(L, 256u)], 1u); });
            __syncthreads();   // the stage buffer is rewritten by the next step
        } else {
        // K3: words are dealt round-robin from the ordered lists (even load per thread; the per-word
        // work is heavy, so this balances better than the list-free per-segment walk of K1)
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
                for (uint32_t q = 0; q < kw; q++) dst[q] = pack6(buf32, kTkPre + start + 6 * q, L - 6 * q);
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
            const uint8_t *sb = reinterpret_cast<const uint8_t *>(sm.c.buf) + kTkPre;
            for (uint32_t k = t; k < S; k += kTkThreads) {
                uint32_t x = sm.wl[k];
                uint32_t L = x & 255u, w = (x >> 8) & 7u, r = x >> 11;
                uint32_t idx = sm.wcnt[w][L] + r;
                uint32_t start = sm.c.sstart[k];
                const uint32_t kw = (L + 5) / 6;
                uint32_t *dst = a.keys + sm.key_off[L] + (uint64_t)idx * kw;
                const uint32_t *buf32 = reinterpret_cast<const uint32_t *>(sm.c.buf);
                for (uint32_t q = 0; q < kw; q++) dst[q] = pack6(buf32, kTkPre + start + 6 * q, L - 6 * q);
                if (a.payload) a.payload[sm.word_off[L] + idx] = (uint32_t)(s0 + start);
            }
            __syncthreads();
            for (int w = 0; w < kTkThreads / 32; w++) sm.wcnt[w][t] = 0;
            // the next stage_step's first __syncthreads orders this reset before phase A
        }
        }
    }
    if constexpr (!kScatter) {
        __syncthreads();
        for (int i = t; i < kHistBins; i += kTkThreads) a.cta_hist[(size_t)c * kHistBins + i] = sm.hist[i];
    }
}

// K2: one CTA of 256 threads; thread L owns length L.
__global__ void __launch_bounds__(256) k_bucket_offsets(TkArgs a, Summary *sum) {
    __shared__ uint64_t s_hist[256];
    __shared__ uint32_t s_toolong;
    const int L = threadIdx.x;
    uint64_t tot = 0;
    uint32_t G = a.grid;
    uint32_t c = 0;
    for (; c + 4 <= G; c += 4) {
        uint32_t h0 = a.cta_hist[(size_t)(c + 0) * kHistBins + L];
        uint32_t h1 = a.cta_hist[(size_t)(c + 1) * kHistBins + L];
        uint32_t h2 = a.cta_hist[(size_t)(c + 2) * kHistBins + L];
        uint32_t h3 = a.cta_hist[(size_t)(c + 3) * kHistBins + L];
        a.cta_base[(size_t)(c + 0) * 256 + L] = (uint32_t)tot; tot += h0;
        a.cta_base[(size_t)(c + 1) * 256 + L] = (uint32_t)tot; tot += h1;
        a.cta_base[(size_t)(c + 2) * 256 + L] = (uint32_t)tot; tot += h2;
        a.cta_base[(size_t)(c + 3) * 256 + L] = (uint32_t)tot; tot += h3;
    }
    for (; c < G; c++) {
        uint32_t h = a.cta_hist[(size_t)c * kHistBins + L];
        a.cta_base[(size_t)c * 256 + L] = (uint32_t)tot;
        tot += h;
    }
    s_hist[L] = tot;
    if (L == 0) {
        uint32_t tl = 0;
        for (uint32_t k = 0; k < G; k++) tl += a.cta_hist[(size_t)k * kHistBins + 256];
        s_toolong = tl;
    }
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
        sum->too_long = s_toolong;
    }
}

}  // namespace

cudaError_t launch_tokenize_count(const TkArgs &a, cudaStream_t s) {
    if (a.grid == 0) return cudaSuccess;
    k_tokenize<0><<<a.grid, kTkThreads, sizeof(TkCountSmem), s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_bucket_offsets(const TkArgs &a, Summary *d_sum, cudaStream_t s) {
    k_bucket_offsets<<<1, 256, 0, s>>>(a, d_sum);
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
