// k_radix.cu — phase 3, variant B ("sort each vector of string ... in the alphabetic
// order"): a segmented LSD radix sort of every length bucket's fixed-width keys at once.
//
// Digits are 2 letters (10 bits, 1024 bins); bucket L needs ndig(L) = ceil(L/2) passes, least
// significant digit first. One launch per pass processes every bucket that still has a digit left;
// tiles never cross a bucket. Each pass is a single sweep (Onesweep-style): digit totals for all
// passes come from one up-front histogram kernel; each tile ranks its keys stably in shared memory
// (warp match_any + per-warp counters), publishes its per-digit counts, resolves its global
// per-digit offset with a decoupled look-back over the preceding tiles of the same bucket, reorders
// its keys in shared memory and writes them out coalesced. Because every pass is stable, equal keys
// (identical words) keep their source order (reading A6), so the optional payload (source offsets)
// comes out in the stable order.
#include "wsort_internal.cuh"

namespace wsort {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kRThreads = 512;
constexpr int kRWarps = kRThreads / 32;
constexpr uint32_t kInc = 0x80000000u;   // status: inclusive prefix available (else count + 1)

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t digit_of(uint32_t word, uint32_t sh) { return (word >> sh) & 1023u; }

// Histogram of every digit of every key of one tile (all passes at once).
__global__ void __launch_bounds__(kRThreads) k_digit_hist(RadixArgs a) {
    extern __shared__ uint32_t h[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const TileDesc td = a.tiles[blockIdx.x];
    const BucketInfo b = a.buckets[td.L];
    const uint32_t k0 = td.tile * b.tile_keys, k1 = min(k0 + b.tile_keys, b.n);
    const uint32_t nd = b.ndig, ns = min(nd, 12u), kw = b.kw;
    for (uint32_t i = t; i < ns * kRadixBins; i += kRThreads) h[i] = 0;
    __syncthreads();
    const uint32_t *kin = a.kin + b.key_off;
    for (uint32_t base = k0 + warp * 32; base < k1; base += kRThreads) {
        const uint32_t k = base + lane;
        const bool v = k < k1;
        uint32_t word = 0, cur = 0xffffffffu;
        for (uint32_t q = 0; q < nd; q++) {
            const uint32_t wi = q / 3;
            if (wi != cur) {
                word = v ? __ldg(kin + (uint64_t)k * kw + wi) : 0u;
                cur = wi;
            }
            const uint32_t d = v ? digit_of(word, 20 - 10 * (q % 3)) : 0xffffffffu;
            const uint32_t peers = __match_any_sync(kFull, d);
            if (v && lane == __ffs(peers) - 1) {
                if (q < 12) atomicAdd(&h[q * kRadixBins + d], __popc(peers));
                else atomicAdd(&a.dh[(size_t)(b.dh_row + q) * kRadixBins + d], __popc(peers));
            }
        }
    }
    __syncthreads();
    for (uint32_t i = t; i < ns * kRadixBins; i += kRThreads)
        if (h[i]) atomicAdd(&a.dh[(size_t)b.dh_row * kRadixBins + i], h[i]);
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

// One LSD pass over all active buckets. Shared memory layout (dynamic):
//   wh   u16 [16][1024]  per-warp digit counters, then per-warp exclusive prefixes
//   cnt  u32 [1024]      tile digit counts
//   toff u32 [1024]      tile-local exclusive prefix over digits
//   gofs u32 [1024]      global destination - tile-local position, per digit (mod 2^32)
//   dr   u32 [T]         digit | rank-within-warp << 10, per key
//   kin  u32 [T*KW], kout u32 [T*KW], (payload) pin u32 [T], pout u32 [T]   (T*KW <= max_tile_words)
template <bool kPay>
__global__ void __launch_bounds__(kRThreads) k_radix_pass(RadixArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t s_ticket;
    __shared__ uint32_t s_wsum[kRWarps];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t TK = a.max_tile_keys, TW = a.max_tile_words;
    uint16_t *wh = reinterpret_cast<uint16_t *>(smem);
    uint32_t *cnt = reinterpret_cast<uint32_t *>(smem + kRWarps * kRadixBins * 2);
    uint32_t *toff = cnt + kRadixBins;
    uint32_t *gofs = toff + kRadixBins;
    uint32_t *dr = gofs + kRadixBins;
    uint32_t *kin_s = dr + TK;
    uint32_t *kout_s = kin_s + TW;
    uint32_t *pin_s = kout_s + TW;
    uint32_t *pout_s = pin_s + TK;

    if (t == 0) s_ticket = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint32_t j = s_ticket;
    if (j < a.nzero)
        for (uint32_t i = t; i < kRadixBins; i += kRThreads) a.status_other[(size_t)j * kRadixBins + i] = 0;
    if (j >= a.ntiles) return;

    const TileDesc td = a.tiles[j];
    const BucketInfo b = a.buckets[td.L];
    const uint32_t q = b.ndig - 1 - a.pass;
    const uint32_t wi = q / 3, sh = 20 - 10 * (q % 3);
    const uint32_t T = b.tile_keys, kw = b.kw;
    const uint32_t k0 = td.tile * T;
    const uint32_t nk = min(T, b.n - k0);
    const uint32_t kpw = ((T + kRWarps * 32 - 1) / (kRWarps * 32)) * 32;   // keys per warp

    for (uint32_t i = t; i < kRWarps * kRadixBins / 2; i += kRThreads) reinterpret_cast<uint32_t *>(wh)[i] = 0;
    {
        const uint32_t *src = a.kin + b.key_off + (uint64_t)k0 * kw;
        const uint32_t nw = nk * kw;
        for (uint32_t i = t; i < nw; i += kRThreads) kin_s[i] = __ldg(src + i);
        if constexpr (kPay) {
            const uint32_t *ps = a.pin + b.word_off + k0;
            for (uint32_t i = t; i < nk; i += kRThreads) pin_s[i] = __ldg(ps + i);
        }
    }
    __syncthreads();

    // stable rank within each warp's contiguous key range
    {
        const uint32_t kb = warp * kpw, ke = min(kb + kpw, nk);
        uint16_t *myh = wh + warp * kRadixBins;
        for (uint32_t i = kb; i < kb + kpw; i += 32) {
            const uint32_t k = i + lane;
            const bool v = k < ke;
            const uint32_t d = v ? digit_of(kin_s[k * kw + wi], sh) : 0xffffffffu;
            const uint32_t peers = __match_any_sync(kFull, d);
            const uint32_t before = v ? myh[d] : 0u;
            __syncwarp();
            if (v && lane == __ffs(peers) - 1) myh[d] = (uint16_t)(before + __popc(peers));
            __syncwarp();
            if (v) dr[k] = d | ((before + __popc(peers & lanemask_lt())) << 10);
        }
    }
    __syncthreads();

    // per digit: exclusive prefix over warps; tile counts; block scan over digits
    uint32_t c2[2];
#pragma unroll
    for (int e = 0; e < 2; e++) {
        const uint32_t d = 2 * t + e;
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kRWarps; w++) {
            uint32_t x = wh[w * kRadixBins + d];
            wh[w * kRadixBins + d] = (uint16_t)run;
            run += x;
        }
        c2[e] = run;
    }
    {
        const uint32_t s = c2[0] + c2[1];
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = lane < kRWarps ? s_wsum[lane] : 0u, wi2 = w;
#pragma unroll
            for (int o = 1; o < kRWarps; o <<= 1) {
                uint32_t y = __shfl_up_sync(kFull, wi2, o);
                if (lane >= o) wi2 += y;
            }
            if (lane < kRWarps) s_wsum[lane] = wi2 - w;
        }
        __syncthreads();
        const uint32_t excl = s_wsum[warp] + incl - s;
        toff[2 * t] = excl;
        toff[2 * t + 1] = excl + c2[0];
    }

    // decoupled look-back over the preceding tiles of this bucket
    const uint32_t *dbase = a.dh + (size_t)(b.dh_row + q) * kRadixBins;
#pragma unroll
    for (int e = 0; e < 2; e++) {
        const uint32_t d = 2 * t + e;
        uint32_t *stp = a.status + (size_t)j * kRadixBins + d;
        uint32_t prefix = 0;
        if (td.tile == 0) {
            st_relaxed(stp, kInc | c2[e]);
        } else {
            st_relaxed(stp, c2[e] + 1u);
            uint32_t jj = j - 1;
            for (;;) {
                const uint32_t sv = ld_relaxed(a.status + (size_t)jj * kRadixBins + d);
                if (sv == 0) continue;
                if (sv & kInc) {
                    prefix += sv & ~kInc;
                    break;
                }
                prefix += sv - 1u;
                jj--;
            }
            st_relaxed(stp, kInc | (prefix + c2[e]));
        }
        gofs[d] = dbase[d] + prefix - toff[d];
    }
    __syncthreads();

    // reorder in shared memory by (digit, warp, rank)
    for (uint32_t k = t; k < nk; k += kRThreads) {
        const uint32_t x = dr[k];
        const uint32_t d = x & 1023u, r = x >> 10, w = k / kpw;
        const uint32_t pos = toff[d] + wh[w * kRadixBins + d] + r;
        for (uint32_t u = 0; u < kw; u++) kout_s[pos * kw + u] = kin_s[k * kw + u];
        if constexpr (kPay) pout_s[pos] = pin_s[k];
    }
    __syncthreads();

    // coalesced write-out: keys with the same digit are contiguous in both smem and global
    {
        uint32_t *dst = a.kout + b.key_off;
        const uint32_t nw = nk * kw;
        for (uint32_t i = t; i < nw; i += kRThreads) {
            const uint32_t k = i / kw, u = i - k * kw;
            const uint32_t d = digit_of(kout_s[k * kw + wi], sh);
            dst[(uint64_t)(gofs[d] + k) * kw + u] = kout_s[i];
        }
        if constexpr (kPay) {
            uint32_t *pd = a.pout + b.word_off;
            for (uint32_t k = t; k < nk; k += kRThreads) {
                const uint32_t d = digit_of(kout_s[k * kw + wi], sh);
                pd[gofs[d] + k] = pout_s[k];
            }
        }
    }
}

}  // namespace

size_t radix_pass_smem(uint32_t tile_keys, uint32_t tile_words, bool payload) {
    size_t s = (size_t)kRWarps * kRadixBins * 2 + 3 * kRadixBins * 4 + (size_t)tile_keys * 4 +
               2 * (size_t)tile_words * 4;
    if (payload) s += 2 * (size_t)tile_keys * 4;
    return s;
}

cudaError_t launch_digit_hist(const RadixArgs &a, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    k_digit_hist<<<a.ntiles, kRThreads, 12 * kRadixBins * 4, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_digit_scan(uint32_t *dh, uint32_t rows, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    k_digit_scan<<<rows, 1024, 0, s>>>(dh);
    return cudaGetLastError();
}

cudaError_t launch_radix_pass(const RadixArgs &a, cudaStream_t s) {
    const uint32_t grid = a.ntiles > a.nzero ? a.ntiles : a.nzero;
    if (grid == 0) return cudaSuccess;
    const bool pay = a.pin != nullptr;
    const size_t smem = radix_pass_smem(a.max_tile_keys, a.max_tile_words, pay);
    cudaError_t e;
    if (pay) {
        e = cudaFuncSetAttribute(k_radix_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_radix_pass<true><<<grid, kRThreads, smem, s>>>(a);
    } else {
        e = cudaFuncSetAttribute(k_radix_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_radix_pass<false><<<grid, kRThreads, smem, s>>>(a);
    }
    return cudaGetLastError();
}

}  // namespace wsort
