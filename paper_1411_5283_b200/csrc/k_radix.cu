// k_radix.cu — phase 3, variant B ("sort each vector of string ... in the alphabetic
// order"): a segmented LSD radix sort of every length bucket's fixed-width keys at once.
//
// Digits are 2 letters (10 bits, 1024 bins); bucket L needs ndig(L) = ceil(L/2) passes, least
// significant digit first. One launch per pass processes every bucket that still has a digit left;
// tiles never cross a bucket. Each pass is a single sweep (Onesweep-style): digit totals for all
// passes come from one up-front histogram kernel; each tile
//   1. loads its keys (coalesced) into shared memory,
//   2. counts its 10-bit digits with shared-memory atomics and publishes the counts at once,
//   3. sorts itself stably by the digit in shared memory with two 5-bit counting sub-passes
//      (one per letter of the digit; thread-private counters + a block scan: no warp-match
//      instructions, which measured ~64 SM-cycles each on B200 against ~3 for an smem atomic),
//   4. resolves its global per-digit offsets with a decoupled look-back over the preceding tiles of
//      the same bucket, and
//   5. writes its keys out coalesced (keys with the same digit are contiguous on both sides).
// Every pass is stable, so equal keys (identical words) keep their source order (reading A6) and
// the optional payload (source offsets) comes out in stable order.
#include "wsort_internal.cuh"

namespace wsort {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kNT = kRadixThreads;        // 256
constexpr int kNW = kNT / 32;
constexpr uint32_t kInc = 0x80000000u;    // status: inclusive prefix available (else count + 1)
constexpr uint32_t kSentinel = 0xffffffffu;  // every 5-bit field = 31 > any letter code (<= 26)

__host__ __device__ __forceinline__ uint32_t padw(uint32_t i) { return i + (i >> 5); }   // bank-conflict padding

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t digit_of(uint32_t word, uint32_t sh) { return (word >> sh) & 1023u; }

// Exclusive scan over the block; returns this thread's exclusive prefix, *total = block total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *wsum, uint32_t *total) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kNW ? wsum[lane] : 0u, wi = w;
#pragma unroll
        for (int o = 1; o < kNW; o <<= 1) {
            uint32_t y = __shfl_up_sync(kFull, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kNW) wsum[lane] = wi - w;
        if (lane == kNW - 1) wsum[kNW] = wi;
    }
    __syncthreads();
    uint32_t r = wsum[warp] + incl - v;
    if (total) *total = wsum[kNW];
    return r;
}

// Thread-private 16-bit counters: 32 bins x kNT threads, linear index j = bin * kNT + thread, held
// as u16 pairs with one pad word per 32 words (conflict-free for both access patterns below).
// Bin f of thread t lives at u16 index 264 f + 2 (t/2 + t/64) + (t & 1).
constexpr uint32_t kCntWords = 32 * kNT / 2 + 32 * kNT / 64;
__device__ __forceinline__ uint16_t *cnt_base(uint32_t *cnt, uint32_t t) {
    return reinterpret_cast<uint16_t *>(cnt + (t >> 1) + (t >> 6)) + (t & 1u);
}
constexpr uint32_t kCntRow = 264;   // u16 stride between bins of one thread

// In-place exclusive scan of the counters in (bin, thread) order. Thread t owns linear entries
// [32t, 32t+32) = the 16 words starting at 16t + t/2.
__device__ __forceinline__ void scan_counters(uint32_t *cnt, uint32_t *wsum) {
    const int t = threadIdx.x;
    uint32_t *c = cnt + 16 * t + (t >> 1);
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) {
        const uint32_t x = c[i];
        s += (x & 0xffffu) + (x >> 16);
    }
    uint32_t run = block_excl_scan(s, wsum, nullptr);
#pragma unroll
    for (int i = 0; i < 16; i++) {
        const uint32_t x = c[i];
        const uint32_t lo = run;
        run += x & 0xffffu;
        c[i] = lo | (run << 16);
        run += x >> 16;
    }
}

struct RSmem {
    uint32_t *A, *B;          // padded key buffers (tile words); B == A on the register path
    uint32_t *PA, *PB;        // padded payload buffers (tile keys)
    uint32_t *cnt;            // kCntWords: 32 x kNT u16 counters
    uint32_t *hist;           // [1024] tile digit counts
    uint32_t *gofs;           // [1024] global destination - tile-local position
    uint32_t *wsum;           // [kNW + 1]
};

template <int KW>
__device__ __forceinline__ uint32_t pick(const uint32_t (&k)[KW], uint32_t wi) {
    uint32_t w = k[0];
#pragma unroll
    for (int u = 1; u < KW; u++) w = wi == (uint32_t)u ? k[u] : w;
    return w;
}

// One tile of one bucket. KW in 1..8: keys in registers, one smem key buffer;
// KW == 0: runtime key width, keys stay in two smem buffers.
template <int KW, bool kPay>
__device__ __forceinline__ void radix_tile(const RadixArgs &a, const BucketInfo &b, uint32_t j, uint32_t tile,
                                           const RSmem &s) {
    const int t = threadIdx.x;
    const uint32_t kw = KW ? (uint32_t)KW : b.kw;
    constexpr int RK = KW ? 32 / KW : 1;   // register keys per thread
    const uint32_t KPT = KW ? (uint32_t)RK : b.tile_keys / kNT;
    const uint32_t T = kNT * KPT;
    const uint32_t q = b.ndig - 1 - a.pass, wi = q / 3, sh = 20 - 10 * (q % 3);
    const uint32_t k0 = tile * b.tile_keys;
    const uint32_t nk = min(b.tile_keys, b.n - k0);
    uint32_t *const A = s.A;
    uint32_t *const B = KW ? s.A : s.B;
    uint16_t *const cb = cnt_base(s.cnt, t);

    for (uint32_t i = t; i < kRadixBins; i += kNT) s.hist[i] = 0;
    {
        const uint32_t *src = a.kin + b.key_off + (uint64_t)k0 * kw;
        const uint32_t nw = nk * kw, tw = T * kw;
        for (uint32_t i = t; i < tw; i += kNT) A[padw(i)] = i < nw ? __ldg(src + i) : kSentinel;
        if constexpr (kPay) {
            const uint32_t *ps = a.pin + b.word_off + k0;
            for (uint32_t i = t; i < T; i += kNT) s.PA[padw(i)] = i < nk ? __ldg(ps + i) : 0u;
        }
    }
#pragma unroll
    for (int f = 0; f < 32; f++) cb[kCntRow * f] = 0;
    __syncthreads();

    uint32_t key[RK][KW ? KW : 1];
    uint32_t rk[(RK + 3) / 4];
    uint32_t c4[4];

    // ---- sub-pass 1: low 5 bits (second letter of the pair); also the 10-bit tile histogram ----
#pragma unroll
    for (int i = 0; i < (RK + 3) / 4; i++) rk[i] = 0;
#pragma unroll
    for (uint32_t k = 0; k < KPT; k++) {
        const uint32_t idx = t * KPT + k;
        uint32_t w;
        if constexpr (KW > 0) {
#pragma unroll
            for (int u = 0; u < KW; u++) key[k][u] = A[padw(idx * KW + u)];
            w = pick<KW>(key[k], wi);
        } else {
            w = A[padw(idx * kw + wi)];
        }
        const uint32_t d = digit_of(w, sh);
        uint16_t *cp = cb + kCntRow * (d & 31u);
        const uint32_t c = *cp;
        *cp = (uint16_t)(c + 1);
        if constexpr (KW > 0) rk[k / 4] |= c << (8 * (k % 4));
        atomicAdd(&s.hist[d], 1u);
    }
    __syncthreads();
    // publish this tile's digit counts (aggregate) as early as possible
    uint32_t *st = a.status + (size_t)j * kRadixBins;
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const uint32_t d = 4 * t + e;
        c4[e] = d == 1023u ? 0u : s.hist[d];   // digit 1023 only ever holds sentinels
        st_relaxed(st + d, tile == 0 ? (kInc | c4[e]) : c4[e] + 1u);
    }
    scan_counters(s.cnt, s.wsum);
    __syncthreads();
    // scatter A -> B by the low field (register path: every key is in registers, B == A)
#pragma unroll
    for (uint32_t k = 0; k < KPT; k++) {
        const uint32_t idx = t * KPT + k;
        uint32_t pos;
        if constexpr (KW > 0) {
            pos = cb[kCntRow * (digit_of(pick<KW>(key[k], wi), sh) & 31u)] + ((rk[k / 4] >> (8 * (k % 4))) & 255u);
#pragma unroll
            for (int u = 0; u < KW; u++) B[padw(pos * KW + u)] = key[k][u];
        } else {
            uint16_t *cp = cb + kCntRow * (digit_of(A[padw(idx * kw + wi)], sh) & 31u);   // re-count
            pos = *cp;
            *cp = (uint16_t)(pos + 1);
            for (uint32_t u = 0; u < kw; u++) B[padw(pos * kw + u)] = A[padw(idx * kw + u)];
        }
        if constexpr (kPay) s.PB[padw(pos)] = s.PA[padw(idx)];
    }
    __syncthreads();

    // ---- sub-pass 2: high 5 bits (first letter of the pair) ----
#pragma unroll
    for (int f = 0; f < 32; f++) cb[kCntRow * f] = 0;
#pragma unroll
    for (int i = 0; i < (RK + 3) / 4; i++) rk[i] = 0;
#pragma unroll
    for (uint32_t k = 0; k < KPT; k++) {
        const uint32_t idx = t * KPT + k;
        uint32_t w;
        if constexpr (KW > 0) {
#pragma unroll
            for (int u = 0; u < KW; u++) key[k][u] = B[padw(idx * KW + u)];
            w = pick<KW>(key[k], wi);
        } else {
            w = B[padw(idx * kw + wi)];
        }
        uint16_t *cp = cb + kCntRow * (digit_of(w, sh) >> 5);
        const uint32_t c = *cp;
        *cp = (uint16_t)(c + 1);
        if constexpr (KW > 0) rk[k / 4] |= c << (8 * (k % 4));
    }
    __syncthreads();
    scan_counters(s.cnt, s.wsum);
    // tile-local start of every digit (exclusive scan of the counts over digits)
    uint32_t ex = block_excl_scan(c4[0] + c4[1] + c4[2] + c4[3], s.wsum, nullptr);
    // scatter B -> A by the high field
#pragma unroll
    for (uint32_t k = 0; k < KPT; k++) {
        const uint32_t idx = t * KPT + k;
        uint32_t pos;
        if constexpr (KW > 0) {
            pos = cb[kCntRow * (digit_of(pick<KW>(key[k], wi), sh) >> 5)] + ((rk[k / 4] >> (8 * (k % 4))) & 255u);
#pragma unroll
            for (int u = 0; u < KW; u++) A[padw(pos * KW + u)] = key[k][u];
        } else {
            uint16_t *cp = cb + kCntRow * (digit_of(B[padw(idx * kw + wi)], sh) >> 5);
            pos = *cp;
            *cp = (uint16_t)(pos + 1);
            for (uint32_t u = 0; u < kw; u++) A[padw(pos * kw + u)] = B[padw(idx * kw + u)];
        }
        if constexpr (kPay) s.PA[padw(pos)] = s.PB[padw(idx)];
    }
    // decoupled look-back over the preceding tiles of this bucket (4 digits per thread), as late as
    // possible so that the predecessors have published their inclusive prefixes
    {
        uint32_t pre[4] = {0, 0, 0, 0};
        if (tile != 0) {
            uint32_t done = 0;
            uint32_t jj = j - 1;
            while (done != 0xfu) {
                const uint32_t *sp = a.status + (size_t)jj * kRadixBins + 4 * t;
                uint32_t v[4];
#pragma unroll
                for (int e = 0; e < 4; e++) v[e] = (done >> e) & 1u ? 1u : ld_relaxed(sp + e);
                if (!(v[0] && v[1] && v[2] && v[3])) continue;
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    if ((done >> e) & 1u) continue;
                    if (v[e] & kInc) {
                        pre[e] += v[e] & ~kInc;
                        done |= 1u << e;
                    } else {
                        pre[e] += v[e] - 1u;
                    }
                }
                jj--;
            }
#pragma unroll
            for (int e = 0; e < 4; e++) st_relaxed(st + 4 * t + e, kInc | (pre[e] + c4[e]));
        }
        const uint32_t *dbase = a.dh + (size_t)(b.dh_row + q) * kRadixBins;
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const uint32_t d = 4 * t + e;
            s.gofs[d] = (d == 1023u ? 0u : __ldg(dbase + d)) + pre[e] - ex;
            ex += c4[e];
        }
    }
    __syncthreads();

    // ---- coalesced write-out (the sentinels sort to the end and are dropped) ----
    uint32_t *dst = a.kout + b.key_off;
    if constexpr (KW == 1) {
        for (uint32_t i = t; i < nk; i += kNT) {
            const uint32_t w = A[padw(i)];
            dst[s.gofs[digit_of(w, sh)] + i] = w;
        }
    } else {
        const uint32_t nw = nk * kw;
        for (uint32_t i = t; i < nw; i += kNT) {
            const uint32_t k = i / kw, u = i - k * kw;
            const uint32_t d = digit_of(A[padw(k * kw + wi)], sh);
            dst[(uint64_t)(s.gofs[d] + k) * kw + u] = A[padw(i)];
        }
    }
    if constexpr (kPay) {
        uint32_t *pd = a.pout + b.word_off;
        for (uint32_t i = t; i < nk; i += kNT) {
            const uint32_t d = digit_of(A[padw(i * kw + wi)], sh);
            pd[s.gofs[d] + i] = s.PA[padw(i)];
        }
    }
}

// kGeneric = false: tiles of buckets with kw <= kRadixRegMaxKw (register path, one key buffer);
// kGeneric = true: tiles of buckets with larger keys.
template <bool kGeneric, bool kPay>
__global__ void __launch_bounds__(kNT, kGeneric ? 1 : (kPay ? 1 : 3)) k_radix_pass(RadixArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ uint32_t s_ticket;
    __shared__ uint32_t s_wsum[kNW + 1];
    const int t = threadIdx.x;
    if (t == 0) s_ticket = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint32_t j = s_ticket;
    if (j < a.nzero)
        for (uint32_t i = t; i < kRadixBins; i += kNT) a.status_other[(size_t)j * kRadixBins + i] = 0;
    if (j >= a.ntiles) return;
    const TileDesc td = a.tiles[j];
    const BucketInfo b = a.buckets[td.L];

    RSmem s;
    const uint32_t tw = padw(a.max_tile_words) + 1, tk = padw(a.max_tile_keys) + 1;
    s.A = smem;
    s.B = s.A + (kGeneric ? tw : 0);
    s.cnt = s.B + tw;
    s.hist = s.cnt + kCntWords;
    s.gofs = s.hist + kRadixBins;
    s.PA = s.gofs + kRadixBins;
    s.PB = s.PA + (kPay ? tk : 0);
    s.wsum = s_wsum;
    if constexpr (kGeneric) {
        radix_tile<0, kPay>(a, b, j, td.tile, s);
    } else {
        switch (b.kw) {
            case 1: radix_tile<1, kPay>(a, b, j, td.tile, s); break;
            case 2: radix_tile<2, kPay>(a, b, j, td.tile, s); break;
            case 3: radix_tile<3, kPay>(a, b, j, td.tile, s); break;
            case 4: radix_tile<4, kPay>(a, b, j, td.tile, s); break;
            case 5: radix_tile<5, kPay>(a, b, j, td.tile, s); break;
            case 6: radix_tile<6, kPay>(a, b, j, td.tile, s); break;
            case 7: radix_tile<7, kPay>(a, b, j, td.tile, s); break;
            default: radix_tile<8, kPay>(a, b, j, td.tile, s); break;
        }
    }
}

// Histogram of every digit of every key of one tile (all passes at once), smem atomics.
__global__ void __launch_bounds__(kNT) k_digit_hist(RadixArgs a) {
    extern __shared__ uint32_t h[];
    const int t = threadIdx.x;
    const TileDesc td = a.tiles[blockIdx.x];
    const BucketInfo b = a.buckets[td.L];
    const uint32_t k0 = td.tile * b.tile_keys, k1 = min(k0 + b.tile_keys, b.n);
    const uint32_t nd = b.ndig, ns = min(nd, 12u), kw = b.kw;
    for (uint32_t i = t; i < ns * kRadixBins; i += kNT) h[i] = 0;
    __syncthreads();
    const uint32_t *kin = a.kin + b.key_off;
    if (kw == 1) {
        for (uint32_t kb = k0 + t; kb < k1; kb += 8 * kNT) {   // batch the loads before the atomics
            uint32_t w[8];
#pragma unroll
            for (int r = 0; r < 8; r++) w[r] = kb + r * kNT < k1 ? __ldg(kin + kb + r * kNT) : 0u;
#pragma unroll
            for (int r = 0; r < 8; r++)
                if (kb + r * kNT < k1)
                    for (uint32_t q = 0; q < nd; q++) atomicAdd(&h[q * kRadixBins + digit_of(w[r], 20 - 10 * q)], 1u);
        }
    } else {
        for (uint32_t k = k0 + t; k < k1; k += kNT) {
            for (uint32_t q = 0; q < nd; q++) {
                const uint32_t w = __ldg(kin + (uint64_t)k * kw + q / 3);
                const uint32_t d = digit_of(w, 20 - 10 * (q % 3));
                if (q < 12) atomicAdd(&h[q * kRadixBins + d], 1u);
                else atomicAdd(&a.dh[(size_t)(b.dh_row + q) * kRadixBins + d], 1u);
            }
        }
    }
    __syncthreads();
    for (uint32_t i = t; i < ns * kRadixBins; i += kNT) {
        const uint32_t v = h[i];
        if (v) atomicAdd(&a.dh[(size_t)b.dh_row * kRadixBins + i], v);
    }
}

// Exclusive scan of one 1024-bin histogram row per CTA (in place): digit counts -> digit bases.
__global__ void __launch_bounds__(1024) k_digit_scan(uint32_t *dh) {
    __shared__ uint32_t wsum[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t *row = dh + (size_t)blockIdx.x * kRadixBins;
    const uint32_t x = row[t];
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = wsum[lane], wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(kFull, wi, o);
            if (lane >= o) wi += y;
        }
        wsum[lane] = wi - w;
    }
    __syncthreads();
    row[t] = wsum[warp] + incl - x;
}

}  // namespace

size_t radix_pass_smem(uint32_t tile_keys, uint32_t tile_words, bool payload, bool generic) {
    size_t w = (generic ? 2 : 1) * (size_t)(padw(tile_words) + 1) + kCntWords + 2 * kRadixBins;
    if (payload) w += 2 * (size_t)(padw(tile_keys) + 1);
    return w * 4;
}

cudaError_t launch_digit_hist(const RadixArgs &a, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    k_digit_hist<<<a.ntiles, kNT, 12 * kRadixBins * 4, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_digit_scan(uint32_t *dh, uint32_t rows, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    k_digit_scan<<<rows, 1024, 0, s>>>(dh);
    return cudaGetLastError();
}

template <bool G, bool P>
static cudaError_t launch_pass_t(const RadixArgs &a, uint32_t grid, cudaStream_t s) {
    const size_t smem = radix_pass_smem(a.max_tile_keys, a.max_tile_words, P, G);
    cudaError_t e = cudaFuncSetAttribute(k_radix_pass<G, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_radix_pass<G, P><<<grid, kNT, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_radix_pass(const RadixArgs &a, bool generic, cudaStream_t s) {
    const uint32_t grid = a.ntiles > a.nzero ? a.ntiles : a.nzero;
    if (grid == 0) return cudaSuccess;
    const bool pay = a.pin != nullptr;
    if (generic) return pay ? launch_pass_t<true, true>(a, grid, s) : launch_pass_t<true, false>(a, grid, s);
    return pay ? launch_pass_t<false, true>(a, grid, s) : launch_pass_t<false, false>(a, grid, s);
}

}  // namespace wsort
