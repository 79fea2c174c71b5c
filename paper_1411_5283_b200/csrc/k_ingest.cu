// k_ingest.cu — the one-pass text front end of the keys-only path and its two consumers.
//
// K1 k_ingest: phases 1-2 of the method (§3 Methodology, Pre-processing) in ONE read
//   of the text. Every maximal run of ASCII letters is a word (reading A1, "removing / ignoring the
//   special characters"); per word of length L:
//     * the length histogram ("the number of elements with the same number of characters",
//       PAPER.md:13) — per CTA (the byte ranges K3 uses) and global;
//     * L <= 5 (dense-key counting): the word IS its dense index
//       idx = sum c_j 26^(L-1-j) (c_j = letter code 0..25), so its sub-array sorted alphabetically
//       is the counting sort of idx. L <= 2 count in shared memory; L = 3..5 go through a small
//       shared-memory hash cache (hot words) and fall back to global atomics (cold words);
//     * 6 <= L <= 66: the word is packed into its fixed-width key (kw = ceil(L/6) u32, the paper's
//       "array char 3D") and appended to a staging chunk of its key-width class K = kw
//       (lengths 6K-5 .. 6K). Chunks (16 KiB) come from the CTA's own region of the pool (bounded: key
//       bytes <= text bytes) and are word-major (word q of key i at q * cap + i, cap = the chunk's key
//       capacity); order inside a chunk is arbitrary (keys only: equal keys are identical words). Every
//       chunk is listed under its class; the MSD's first level reads the chunks in place, class by class
//       (k_msd.cu: k_msd_count0 / k_msd_scatter0). (One chunk stream per length was measured slower: a
//       warp's keys then go to ~15 chunks, and the stores of the keys cost 0.26 ms more on c4.)
// K2d k_dense_reduce / k_dense_scan / k_dense_compact: exclusive scan of the dense counts (which is
//   the global word index, since buckets 1..5 come first) and compaction of the non-zero entries.
// K3c k_lscatter: the staged keys, chunk by chunk, into their length buckets (buffer A) — for the
//   stage API of the torch.distributed variant (wsort_pack_long); AUTO reads the chunks in the MSD.
// K5d k_emit_dense: "prints the results" for L <= 5: word w of the dense buckets is
//   the entry whose count range holds w; written as "word\n" (reading A12).
#include <algorithm>

#include "k_hash.cuh"
#include "k_text.cuh"
#include "k_tma.cuh"
#include "wsort_internal.cuh"

namespace wsort {
namespace {

using namespace text;

constexpr int kIgWarps = kIgThreads / 32;
#ifndef WSORT_IG_CACHE_LG
#define WSORT_IG_CACHE_LG 13
#endif
constexpr int kCacheLg = WSORT_IG_CACHE_LG, kCacheSlots = 1 << kCacheLg;   // (1024 .. 8192 slots measured: see DESIGN.md)

// entries of the dense tables of lengths < L: (26^L - 26) / 25
__host__ __device__ constexpr uint32_t dense_base(uint32_t L) {
    return L <= 1 ? 0u : L == 2 ? 26u : L == 3 ? 702u : L == 4 ? 18278u : L == 5 ? 475254u : 12356630u;
}

// One CTA of 1024 threads per SM (measured on c4: 1.31 ms against 1.45 ms with two CTAs of 512: one set of
// shared tables, one hash cache of twice the slots and one open chunk per class per SM)
#ifndef WSORT_IG_MINB
#define WSORT_IG_MINB 1
#endif
constexpr int kIgMinBlocks = WSORT_IG_MINB;
#ifndef WSORT_IG_PIECE
#define WSORT_IG_PIECE 0
#endif
// 0 (default): a CTA's range is split into static contiguous warp ranges. > 0 (experiment, measured
// slower: 1.70 vs 1.45 ms on c4 for pieces of 4 .. 32 sub-steps): the range is handed to the warps in pieces
// of kIgPiece sub-steps taken from a shared counter as each warp finishes its piece
constexpr uint32_t kIgPiece = WSORT_IG_PIECE;
#ifndef WSORT_IG_PIECE_MODE
#define WSORT_IG_PIECE_MODE 0
#endif
constexpr int kSub = 1024;                   // bytes per warp sub-step (32 per lane)
constexpr int kSubTail = 128;                // staged bytes past it (a staged word: <= 66 letters + slack)
constexpr int kWBuf = kSub + kSubTail;
constexpr int kWList = kSub / 2;             // at most one word start per two bytes
constexpr uint32_t kTrash16 = 0xfffeu;
// A chunk is published in a ring of kRing slots per class: slot (seq % kRing) = (seq + 1) << 16 | chunk id.
// A lane that ranked key `r` of its class waits for its chunk's entry; an entry of a later sequence
// number means the slot was reused before the lane read it (kRing chunks of that class filled in
// between: never expected); it is reported like an unstaged word (the host then counts the text instead).
constexpr uint32_t kRing = 8;

// keys per chunk of key width k: the largest power of two <= kChunkWords / k (chunk_lg), and the same in
// two instructions for 1 <= k <= 16: 12 - ceil(log2 k) (constexpr twin checked below)
__host__ __device__ constexpr uint32_t cls_lg(uint32_t k) { return chunk_lg(k); }
__host__ __device__ constexpr uint32_t cls_lg_twin(uint32_t k) { return k <= 1 ? 12u : 12u - (32u - (uint32_t)__builtin_clz(k - 1u)); }
__device__ __forceinline__ uint32_t cls_lg_fast(uint32_t k) { return (uint32_t)__clz(k - 1u) - 20u; }
__host__ __device__ constexpr bool cls_lg_agree(uint32_t k) { return k > kMaxStageKw || (cls_lg(k) == cls_lg_twin(k) && cls_lg_agree(k + 1)); }
static_assert(kMaxStageKw <= 16 && kChunkWords == 4096 && cls_lg_agree(1), "cls_lg_fast must equal chunk_lg for every staged width");

struct IgSmem {
    uint4 wbuf[kIgWarps][2][kWBuf / 16 + 1];   // per warp, two slots: a sub-step + tail (+16 B: packing reads
                                               // whole words)
    uint16_t wlist[kIgWarps][kWList];      // per warp: s | (L-3) << 10; L = 3..5 from the front, 6..66 from the back
    uint32_t d12[27 * 27];                 // counts of L = 1, 2: [code of letter 0 (1..26)][code of letter 1, 0 for L = 1]
    uint32_t ctag[kCacheSlots];            // hash cache for L = 3..5: tag = L << 24 | idx, 0 = empty
    uint32_t ccnt[kCacheSlots];
    uint32_t hist[kHistBins];
    uint32_t nchunk;                       // chunks this CTA took from its region
    uint32_t next_piece;                   // next piece of the CTA's range to be taken by a warp (kIgPiece)
    uint32_t cls_fill[kMaxStageKw];        // keys of class i + 1 staged so far
    uint32_t ring[kMaxStageKw][kRing];     // published chunks of each class (see kRing)
};

// dense index of the word of length L <= 5 at byte boff of a staged buffer
__device__ __forceinline__ uint32_t dense_index(const uint32_t *buf32, uint32_t boff, uint32_t L) {
    const uint32_t a = boff >> 2, sh = 8u * (boff & 3u);
    const uint32_t w0 = buf32[a], w1 = buf32[a + 1], w2 = buf32[a + 2];
    const uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);
    uint32_t idx = (lo & 31u) - 1u;
    if (L > 1) idx = idx * 26u + ((lo >> 8) & 31u) - 1u;
    if (L > 2) idx = idx * 26u + ((lo >> 16) & 31u) - 1u;
    if (L > 3) idx = idx * 26u + ((lo >> 24) & 31u) - 1u;
    if (L > 4) idx = idx * 26u + (hi & 31u) - 1u;
    return idx;
}

// one probe of the hash cache: true if the word was counted in slot h
__device__ __forceinline__ bool cache_try(IgSmem &sm, uint32_t h, uint32_t tag) {
    uint32_t cur = *reinterpret_cast<volatile uint32_t *>(&sm.ctag[h]);
    if (cur == 0u) {
        cur = atomicCAS(&sm.ctag[h], 0u, tag);
        if (cur == 0u) cur = tag;
    }
    if (cur != tag) return false;
    atomicAdd(&sm.ccnt[h], 1u);
    return true;
}

// two-choice hash cache (hot words stay in shared memory); a word whose slots are both taken by other
// words is counted in the global table directly (its block of the table marked as touched)
__device__ __forceinline__ void cache_add(IgSmem &sm, uint32_t *dense, uint8_t *touched, uint32_t L, uint32_t idx) {
    const uint32_t tag = (L << 24) | idx;
    const uint32_t hh = tag * 0x9E3779B1u;
    if (cache_try(sm, hh >> (32 - kCacheLg), tag)) return;
    if (cache_try(sm, (hh >> 10) & (kCacheSlots - 1), tag)) return;
    const uint32_t e = dense_base(L) + idx;
    atomicAdd(&dense[e], 1u);
    touched[e / kDenseBlkEntries] = 1;
}

__device__ __forceinline__ uint32_t inclusive_scan_warp(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

#ifndef WSORT_IG_EVICT
#define WSORT_IG_EVICT 1
#endif
// The text is read once: its loads are marked evict-first in L2 so that the staging chunks being filled
// (one open chunk per length and CTA) stay resident until their sectors are complete.
__device__ __forceinline__ uint4 ld_text16(const void *p, uint64_t pol) {
#if WSORT_IG_EVICT
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(reinterpret_cast<const uint4 *>(p));
#endif
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol = 0;
#if WSORT_IG_EVICT
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    return pol;
}

// letters leading a 32-bit letter mask, and whether all 32 are letters
__device__ __forceinline__ uint32_t lead_run(uint32_t M) { return M == 0xffffffffu ? 32u : (uint32_t)(__ffs(~M) - 1); }

// ---- hash mode: long words counted into the global table of distinct words (k_hash.cuh)
// key word of letters [0, n) (n <= 6) of the word at global byte p (words of > 66 letters: not all in the
// shared-memory window)
__device__ __forceinline__ uint32_t pack6_global(const uint8_t *p, uint32_t n) {
    uint32_t key = 0;
    for (uint32_t j = 0; j < 6u && j < n; j++) key |= (uint32_t)(__ldg(p + j) & 31u) << (25u - 5u * j);
    return key;
}

// Words [0, i1) of a warp's long list (from the back), one per lane: histogram, then the word's slot
// (found or inserted) gets one more occurrence. Every length 6..255 is counted (words of > 66 letters,
// listed as 67, are re-measured and packed from the text in global memory).
__device__ __forceinline__ void hash_long(const IngestArgs &a, IgSmem &sm, const uint16_t *lst, uint32_t i1,
                                          const uint32_t *wb32, const uint8_t *gtext, int lane) {
    for (uint32_t b = 0; b < i1; b += 32) {
        const uint32_t i = b + lane;
        if (i >= i1) break;
        const uint32_t x = lst[kWList - 1 - i];
        const uint32_t s = x & 1023u;
        uint32_t L = (x >> 10) + 6u;
        if (L > 6u * kMaxStageKw) {   // (listed as 67: >= 67 letters) the exact length from the text
            L = 6u * kMaxStageKw;
            while (L <= (uint32_t)kMaxLen && is_letter(__ldg(gtext + s + L))) L++;
            if (L > (uint32_t)kMaxLen) continue;   // (> 255: flagged as too long by the list loop)
            atomicAdd(&sm.hist[L], 1u);
            if (a.debug & 2) continue;
            const uint32_t k = (L + 5u) / 6u;
            auto get = [&](uint32_t q) { return pack6_global(gtext + s + 6u * q, L - 6u * q); };
            const uint64_t fp = hashtab::fingerprint(L, k, get);
            const uint32_t slot = hashtab::find(a.tab, L, k, fp, get, true);
            if (slot != hashtab::kUnset) atomicAdd(a.tab.cnt + slot, 1u);
            continue;
        }
        atomicAdd(&sm.hist[L], 1u);
        if (a.debug & 2) continue;
        if (L <= 24u) {
            const uint32_t w0 = pack6(wb32, s, 6u);
            const uint32_t w1 = L > 6u ? pack6(wb32, s + 6u, L - 6u) : 0u;
            const uint32_t w2 = L > 12u ? pack6(wb32, s + 12u, L - 12u) : 0u;
            const uint32_t w3 = L > 18u ? pack6(wb32, s + 18u, L - 18u) : 0u;
            const uint32_t slot = hashtab::find_narrow(a.tab, hashtab::narrow_key(w0, w1, w2, w3), L, true);
            if (slot != hashtab::kUnset) atomicAdd(a.tab.ncnt + slot, 1u);   // (else overflow: staging fallback)
        } else {   // key word q = letters 6q .. 6q+5, recomputed from the text when needed
            const uint32_t k = (L + 5u) / 6u;
            auto get = [&](uint32_t q) { return pack6(wb32, s + 6u * q, L - 6u * q); };
            const uint64_t fp = hashtab::fingerprint(L, k, get);
            const uint32_t slot = hashtab::find(a.tab, L, k, fp, get, true);
            if (slot != hashtab::kUnset) atomicAdd(a.tab.cnt + slot, 1u);
        }
    }
}

// K1. The CTA's byte range is split into contiguous warp ranges (32 warps) of 1 KiB sub-steps; each warp
// streams its sub-steps with no block barrier: every lane classifies 32 bytes (SWAR letter mask, loaded
// one sub-step ahead), word starts / ends come from mask shifts, the letter runs crossing lane
// boundaries from a suffix scan of (l1,f1)+(l2,f2) = (l1 + f1*l2, f1 & f2) (l = letters leading a
// segment, f = all letters). Words of L <= 2 are counted by their owner lane; L = 3..5 and 6..66 are
// listed by category (warp scan) and then taken round-robin by the lanes: hash-cache count / key
// packing into the class's chunk. Chunk (class, seq) is allocated by the lane that receives its
// first rank; the others read its id from shared memory (written once).
template <bool HASH>
__global__ void __launch_bounds__(kIgThreads, kIgMinBlocks) k_ingest(IngestArgs a) {
    extern __shared__ __align__(16) uint8_t ig_smem[];
    IgSmem &sm = *reinterpret_cast<IgSmem *>(ig_smem);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t c = blockIdx.x + a.cta_first;
    const uint64_t b0 = (uint64_t)c * a.steps_per_cta * kTkStep;
    const uint64_t b1 = min((uint64_t)(c + 1) * a.steps_per_cta, (uint64_t)a.nsteps) * kTkStep;
    const uint32_t cbase = c * a.cta_chunks;
    const uint32_t trash = a.grid * a.cta_chunks;

    for (int i = t; i < 27 * 27; i += kIgThreads) sm.d12[i] = 0;
    for (int i = t; i < kCacheSlots; i += kIgThreads) sm.ctag[i] = sm.ccnt[i] = 0;
    for (int i = t; i < kHistBins; i += kIgThreads) sm.hist[i] = 0;
    for (uint32_t i = t; i < kMaxStageKw * kRing; i += kIgThreads) (&sm.ring[0][0])[i] = 0;
    if (t < (int)kMaxStageKw) sm.cls_fill[t] = 0;
    if (t == 0) sm.nchunk = sm.next_piece = 0;
    __syncthreads();

    const uint32_t nsub = b0 < b1 ? (uint32_t)((b1 - b0) / kSub) : 0u;
    uint16_t *wlst = sm.wlist[warp];
    // Two shared-memory slots per warp: the sub-step being processed (+ the next one's first 128 bytes: the
    // tail a word crossing the sub-step continues into) and the next sub-step, written one iteration ahead
    // from the registers that prefetched it. Each sub-step's letter mask is computed once, one iteration
    // ahead, so the tail needs neither its own loads nor its own mask.
    const uint64_t pol = evict_first_policy();
    uint32_t nge[6] = {0, 0, 0, 0, 0, 0};   // this lane's words of >= 1, 2, ..., 6 letters
    for (uint32_t piece = 0;; piece++) {   // (static ranges: one pass)
    uint32_t w0, w1;
    if (kIgPiece) {
#if WSORT_IG_PIECE_MODE == 0      // dynamic
        if (lane == 0) piece = atomicAdd(&sm.next_piece, 1u);
        piece = __shfl_sync(kFull, piece, 0);
        w0 = piece * kIgPiece;
        if (w0 >= nsub) break;
        w1 = min(w0 + kIgPiece, nsub);
#elif WSORT_IG_PIECE_MODE == 1    // static round-robin pieces
        w0 = (piece * kIgWarps + warp) * kIgPiece;
        if (w0 >= nsub) break;
        w1 = min(w0 + kIgPiece, nsub);
#else                             // the static contiguous ranges through the piece loop (run-time trip count)
        const uint32_t np = max(1u, (a.debug >> 8) & 255u);   // (WSORT_INGEST_DEBUG = 256 * pieces per warp range)
        const uint32_t per = (nsub + kIgWarps - 1) / kIgWarps, half = (per + np - 1) / np;
        if (piece >= np) break;
        w0 = min(warp * per + piece * half, nsub);
        w1 = min(min(w0 + half, (warp + 1) * per), nsub);
#endif
    } else {
        if (piece) break;
        w0 = (uint32_t)((uint64_t)nsub * warp / kIgWarps);
        w1 = (uint32_t)((uint64_t)nsub * (warp + 1) / kIgWarps);
    }
    uint4 va = make_uint4(0, 0, 0, 0), vb = va;
    uint32_t prev_last = 0, M = 0;
    if (w0 < w1) {
        const uint8_t *p = a.text + b0 + (uint64_t)w0 * kSub;
        const uint4 ca = ld_text16(reinterpret_cast<const uint4 *>(p) + 2 * lane, pol);
        const uint4 cb = ld_text16(reinterpret_cast<const uint4 *>(p) + 2 * lane + 1, pol);
        va = ld_text16(reinterpret_cast<const uint4 *>(p + kSub) + 2 * lane, pol);   // (the text buffer is padded:
        vb = ld_text16(reinterpret_cast<const uint4 *>(p + kSub) + 2 * lane + 1, pol);   //  reads past a range are safe)
        uint4 *s0 = reinterpret_cast<uint4 *>(sm.wbuf[warp][w0 & 1]);
        s0[2 * lane] = ca;
        s0[2 * lane + 1] = cb;
        M = letter_mask32(ca, cb);
        prev_last = is_letter(p[-1]);
    }
    for (uint32_t sub = w0; sub < w1; sub++) {
        uint8_t *wb = reinterpret_cast<uint8_t *>(sm.wbuf[warp][sub & 1]);
        const uint32_t *wb32 = reinterpret_cast<const uint32_t *>(wb);
        const uint64_t base = b0 + (uint64_t)sub * kSub;
        // the next sub-step (prefetched last iteration): its mask, its slot, and the current slot's tail
        const uint32_t Mn = letter_mask32(va, vb);
        {
            uint4 *sn = reinterpret_cast<uint4 *>(sm.wbuf[warp][(sub + 1) & 1]);
            sn[2 * lane] = va;
            sn[2 * lane + 1] = vb;
            if (lane < kSubTail / 32) {
                reinterpret_cast<uint4 *>(wb + kSub)[2 * lane] = va;
                reinterpret_cast<uint4 *>(wb + kSub)[2 * lane + 1] = vb;
            }
        }
        {   // prefetch the sub-step after the next
            const uint8_t *p = a.text + base + 2 * kSub;
            va = ld_text16(reinterpret_cast<const uint4 *>(p) + 2 * lane, pol);
            vb = ld_text16(reinterpret_cast<const uint4 *>(p) + 2 * lane + 1, pol);
        }
        __syncwarp();
        const uint32_t pm = __shfl_up_sync(kFull, M, 1), nm = __shfl_down_sync(kFull, M, 1);
        const uint32_t pl = lane ? (pm >> 31) : prev_last;
        const uint32_t mt0 = __shfl_sync(kFull, Mn, 0);
        const uint32_t nx = lane < 31 ? (nm & 1u) : (mt0 & 1u);
        prev_last = __shfl_sync(kFull, M, 31) >> 31;
        const uint32_t starts = M & ~((M << 1) | pl);
        const uint32_t ends = M & ~((M >> 1) | (nx << 31));
        // letters continuing past this lane's last byte: the all-letter lanes after it (32 each), then the
        // leading letters of the first lane that is not all letters; past lane 31, the next sub-step's
        // leading letters qh (>= 1024: a run longer than any staged / legal word)
        uint32_t carry;
        {
            const uint32_t fullN = __ballot_sync(kFull, Mn == 0xffffffffu);
            const uint32_t kN = fullN == 0xffffffffu ? 0u : (uint32_t)(__ffs(~fullN) - 1);
            const uint32_t leadN = __shfl_sync(kFull, lead_run(Mn), kN);
            const uint32_t qh = fullN == 0xffffffffu ? 1024u : 32u * kN + leadN;
            const uint32_t fullM = __ballot_sync(kFull, M == 0xffffffffu);
            const uint32_t nf = lane < 31 ? ~fullM & (0xfffffffeu << lane) : 0u;
            const uint32_t k = nf ? (uint32_t)(__ffs(nf) - 1) : 0u;
            const uint32_t lk = __shfl_sync(kFull, lead_run(M), k);
            carry = nf ? 32u * (k - lane - 1u) + lk : 32u * (31u - lane) + qh;
        }
        const uint32_t seg0 = 32u * lane;
        // categories from the masks: a word starting at bit i has L >= j iff bytes i..i+j-1 are letters
        // (X = this lane's letters followed by the next lane's / the tail's); one branch-free loop each
        const uint64_t X = (uint64_t)M | ((uint64_t)(lane < 31 ? nm : mt0) << 32);
        const uint32_t ge2 = starts & (uint32_t)(X >> 1);
        const uint32_t ge3 = ge2 & (uint32_t)(X >> 2);
        const uint32_t ge4 = ge3 & (uint32_t)(X >> 3), ge5 = ge4 & (uint32_t)(X >> 4);
        const uint32_t ge6 = ge5 & (uint32_t)(X >> 5);
        const uint32_t s12 = starts & ~ge3, s345 = ge3 & ~ge6;
        // words of >= 1..6 letters started by this lane (the length histogram of L <= 5 is their differences)
        nge[0] += __popc(starts);
        nge[1] += __popc(ge2);
        nge[2] += __popc(ge3);
        nge[3] += __popc(ge4);
        nge[4] += __popc(ge5);
        nge[5] += __popc(ge6);
        const uint32_t nlong = __popc(ge6), n345 = __popc(s345);
        const uint32_t cnt = n345 | (nlong << 16);
        const uint32_t ci = inclusive_scan_warp(cnt, lane);
        const uint32_t tot = __shfl_sync(kFull, ci, 31);
        uint32_t p3 = (ci - cnt) & 0xffffu, plg = (ci - cnt) >> 16;
        uint32_t *d12 = sm.d12;
        for (uint32_t m = s12; m;) {   // L = 1, 2: count now (shared-memory table [first code][second code or 0])
            const uint32_t low = m & (0u - m), s = seg0 + 31u - (uint32_t)__clz(low);
            m ^= low;
            const uint32_t b0 = wb[s], b1 = wb[s + 1];   // (byte 1024 is the staged tail)
            const uint32_t sel = (ge2 & low) ? (b1 & 31u) : 0u;
            if (!(a.debug & 1)) atomicAdd(&d12[(b0 & 31u) * 27u + sel], 1u);
        }
        for (uint32_t m = s345; m;) {   // L = 3..5: listed for the hash cache (L - 3 = the start is in ge4, in ge5)
            const uint32_t low = m & (0u - m), bit = 31u - (uint32_t)__clz(low);
            m ^= low;
            wlst[p3++] = (uint16_t)(seg0 + bit + ((ge4 & low) ? 1024u : 0u) + ((ge5 & low) ? 1024u : 0u));
        }
        const uint32_t past = 32u + carry;   // (a word with no end in this lane: its letters here + the carry)
        uint32_t ntl = 0;
        for (uint32_t m = ge6; m;) {   // L >= 6: listed for packing (above 66 kept as 67: not staged)
            const uint32_t low = m & (0u - m), bit = 31u - (uint32_t)__clz(low);
            m ^= low;
            const uint32_t em = ends & (0u - low);   // ends at or after the start
            const uint32_t L = (uint32_t)__ffs(em) - bit + (em ? 0u : past);   // (__ffs(0) = 0)
            wlst[kWList - 1 - plg++] = (uint16_t)((seg0 + bit) | ((min(L, 6u * kMaxStageKw + 1u) - 6u) << 10));
            ntl += L > (uint32_t)kMaxLen;
        }
        if (ntl) atomicAdd(&sm.hist[256], ntl);
        __syncwarp();
        const uint32_t n3 = tot & 0xffffu, nlg = tot >> 16;
        for (uint32_t i = lane; i < ((a.debug & 17) ? 0u : n3); i += 32) {   // L = 3..5: hash cache
            const uint32_t x = wlst[i];
            const uint32_t s = x & 1023u, L = (x >> 10) + 3u;
            cache_add(sm, a.dense, a.touched, L, dense_index(wb32, s, L));
        }
        if (HASH) {   // L = 6..66: counted into the global table
            if (!(a.debug & 8)) hash_long(a, sm, wlst, nlg, wb32, a.text + base, lane);
            __syncwarp();
            M = Mn;
            continue;
        }
        for (uint32_t i0 = 0; i0 < ((a.debug & 8) ? 0u : nlg); i0 += 32) {   // L = 6..66: key into its class's chunk
            const uint32_t i = i0 + lane;
            const uint32_t x = i < nlg ? wlst[kWList - 1 - i] : 0u;
            const uint32_t s = x & 1023u, L = (x >> 10) + 6u;
            const bool v = i < nlg && L <= 6u * kMaxStageKw;
            if (i < nlg) {
                if (v) atomicAdd(&sm.hist[L], 1u);
                else atomicAdd(&a.ctr[kIgVeryLong], 1u);   // too long to stage: the host counts the text instead
            }
            const uint32_t k = (L + 5u) / 6u, lg = cls_lg_fast(k), cl = v ? k - 1u : 0u;
            uint32_t r = 0;
            if (v) r = atomicAdd(&sm.cls_fill[cl], 1u);
            const uint32_t seq = r >> lg, pos = r & ((1u << lg) - 1u);
            uint32_t *slot = &sm.ring[cl][seq & (kRing - 1)];
            const uint32_t tag = (seq + 1u) << 16;
            if (v && pos == 0) {   // first key of chunk (k, seq): take a chunk from the region, list and publish it
                uint32_t id = atomicAdd(&sm.nchunk, 1u);
                if (id >= a.cta_chunks) {   // cannot happen (key bytes <= text bytes + 256)
                    atomicExch(&a.ctr[kIgOverflow], 1u);
                    id = kTrash16;
                } else {
                    a.chunk_cls[cbase + id] = k | (seq << 8);
                    a.cls_list[(size_t)cl * a.cls_cap + atomicAdd(&a.ctr[kIgClsCnt + cl], 1u)] = cbase + id;
                }
                *reinterpret_cast<volatile uint32_t *>(slot) = tag | id;
            }
            __syncwarp();   // ids published by this warp are visible; other warps publish right after their atomic
            if (!v || (a.debug & 2)) continue;
            uint32_t e, spins = 0;
            while (((e = *reinterpret_cast<volatile uint32_t *>(slot)) & 0xffff0000u) != tag) {
                if ((e >> 16) > seq + 1u) {   // slot reused (never expected): the host falls back as for
                    atomicAdd(&a.ctr[kIgVeryLong], 1u);   // unstaged words (COUNT ingest, or K3 + LSD)
                    e = kTrash16;
                    break;
                }
                if (++spins > (1u << 22)) {   // never expected: report instead of hanging
                    atomicExch(&a.ctr[kIgOverflow], 2u);
                    e = kTrash16;
                    break;
                }
            }
            const uint32_t id = e & 0xffffu;
            // word-major chunk: word q of key `pos` at q * cap + pos (a warp's keys of one class land on
            // consecutive words of each row)
            uint32_t *dst = a.pool + (size_t)(id == kTrash16 ? trash : cbase + id) * kChunkWords + pos;
            pack_key(wb32, s, L, k, dst, 1u << lg);
        }
        __syncwarp();   // the slot and list are rewritten by the next sub-steps
        M = Mn;
    }
    }
#pragma unroll
    for (int j = 0; j < 6; j++) {   // the warp's counts of L = 1..5 into the histogram (K2 needs no table scan)
#pragma unroll
        for (int o = 16; o; o >>= 1) nge[j] += __shfl_xor_sync(kFull, nge[j], o);
    }
    if (lane < (int)kDenseMaxLen && !(a.debug & 64)) {
        uint32_t v = nge[0] - nge[1];
#pragma unroll
        for (int j = 1; j < (int)kDenseMaxLen; j++) v = lane == j ? nge[j] - nge[j + 1] : v;
        if (v) atomicAdd(&sm.hist[lane + 1], v);
    }
    __syncthreads();
    if (t == 0) atomicMax(&a.ctr[kIgMaxChunks], sm.nchunk);
    if (!HASH) {   // keys in each chunk: full, except the last one of each class
        for (uint32_t id = t; id < min(sm.nchunk, a.cta_chunks); id += kIgThreads) {
            const uint32_t v = a.chunk_cls[cbase + id], K = v & 255u, seq = v >> 8, lg = cls_lg(K);
            a.chunk_fill[cbase + id] = min(1u << lg, sm.cls_fill[K - 1u] - (seq << lg));
        }
    }
    if (a.debug & 32) return;   // (timing experiments: no flush of the shared-memory tables)
    for (int i = t; i < 27 * 27; i += kIgThreads)
        if (sm.d12[i]) {   // (rows / columns of code 0 stay empty) -> dense index: L = 1: c0; L = 2: 26 + 26 c0 + c1
            const uint32_t c0 = (uint32_t)i / 27u - 1u, b1 = (uint32_t)i % 27u;
            atomicAdd(&a.dense[b1 ? 26u + c0 * 26u + b1 - 1u : c0], sm.d12[i]);
            a.touched[0] = 1;   // (702 < one block)
        }
    for (int i = t; i < kCacheSlots; i += kIgThreads) {
        const uint32_t tag = sm.ctag[i];
        if (tag) {
            const uint32_t e = dense_base(tag >> 24) + (tag & 0xffffffu);
            atomicAdd(&a.dense[e], sm.ccnt[i]);
            a.touched[e / kDenseBlkEntries] = 1;
        }
    }
    for (int i = t; i < kHistBins; i += kIgThreads) {   // every length (1..5 from the mask counts above)
        const uint32_t h = sm.hist[i];
        if (h) atomicAdd(&a.ghist[i], h);
    }
}

// Before K1: the blocks the previous text touched are zeroed (instead of the whole 49 MB table)
__global__ void __launch_bounds__(256) k_dense_clear(uint32_t *dense, uint8_t *touched, uint32_t n_entries) {
    const uint32_t b = blockIdx.x;
    if (!touched[b]) return;
    for (uint32_t e = b * kDenseBlkEntries + threadIdx.x; e < min(n_entries, (b + 1) * kDenseBlkEntries); e += 256) dense[e] = 0;
    __syncthreads();
    if (threadIdx.x == 0) touched[b] = 0;
}

// ------------------------------------------------------------------ block scan helper (256 threads)
__device__ __forceinline__ uint32_t excl_scan256(uint32_t v, uint32_t *wsum, uint32_t *total) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
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
    const uint32_t r = wsum[warp] + incl - v;
    if (total) *total = wsum[8];
    __syncthreads();
    return r;
}

// ------------------------------------------------------------------ K2d: dense scan + compaction
constexpr uint32_t kDenseBlk = kDenseBlkEntries;   // entries per block (16 per thread)

// The table's blocks of kDenseBlk entries that no word touched are all zero: skipped (a block-uniform exit)
__global__ void __launch_bounds__(256) k_dense_reduce(DenseArgs a) {
    __shared__ uint32_t wsum[9];
    const uint32_t b = blockIdx.x, t = threadIdx.x;
    if (!a.touched[b]) {
        if (t == 0) a.blk_sum[b] = a.blk_nnz[b] = 0;
        return;
    }
    uint32_t sum = 0, nnz = 0;
    const uint32_t e0 = b * kDenseBlk + 16u * t;
#pragma unroll
    for (int j = 0; j < 16; j++) {
        const uint32_t e = e0 + j;
        const uint32_t v = e < a.n_entries ? a.dense[e] : 0u;
        sum += v;
        nnz += v != 0u;
    }
    uint32_t ts = 0, tn = 0;
    excl_scan256(sum, wsum, &ts);
    excl_scan256(nnz, wsum, &tn);
    if (t == 0) {
        a.blk_sum[b] = ts;
        a.blk_nnz[b] = tn;
    }
}

// words of each length L <= 5 = the sum of its dense table (the length histogram of the dense buckets)
__global__ void __launch_bounds__(256) k_dense_lensum(const uint32_t *dense, const uint8_t *touched, uint32_t *ghist) {
    __shared__ uint32_t h[kDenseMaxLen + 1];
    if (!touched[blockIdx.x]) return;
    const uint32_t t = threadIdx.x, e0 = blockIdx.x * kDenseBlk + 16u * t, ne = dense_base(kDenseMaxLen + 1);
    if (t <= kDenseMaxLen) h[t] = 0;
    __syncthreads();
    uint32_t L = 1;
    while (dense_base(L + 1) <= e0 && L < kDenseMaxLen) L++;
    uint32_t sum = 0;
#pragma unroll
    for (int j = 0; j < 16; j++) {
        const uint32_t e = e0 + j;
        if (e >= ne) break;
        if (e == dense_base(L + 1)) {
            if (sum) atomicAdd(&h[L], sum);
            sum = 0;
            L++;
        }
        sum += dense[e];
    }
    if (sum) atomicAdd(&h[L], sum);
    __syncthreads();
    if (t >= 1 && t <= kDenseMaxLen && h[t]) atomicAdd(&ghist[t], h[t]);
}

__global__ void __launch_bounds__(1024) k_dense_scan(DenseArgs a, uint32_t nblk) {
    __shared__ uint32_t ws[33], wn[33];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    uint32_t run_s = 0, run_n = 0;
    for (uint32_t b0 = 0; b0 < nblk; b0 += 1024) {
        const uint32_t b = b0 + t;
        const uint32_t vs = b < nblk ? a.blk_sum[b] : 0u, vn = b < nblk ? a.blk_nnz[b] : 0u;
        uint32_t is = vs, in = vn;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ys = __shfl_up_sync(kFull, is, o), yn = __shfl_up_sync(kFull, in, o);
            if (lane >= o) {
                is += ys;
                in += yn;
            }
        }
        if (lane == 31) {
            ws[warp] = is;
            wn[warp] = in;
        }
        __syncthreads();
        if (warp == 0) {
            const uint32_t xs = ws[lane], xn = wn[lane];
            uint32_t ps = xs, pn = xn;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t ys = __shfl_up_sync(kFull, ps, o), yn = __shfl_up_sync(kFull, pn, o);
                if (lane >= o) {
                    ps += ys;
                    pn += yn;
                }
            }
            ws[lane] = ps - xs;
            wn[lane] = pn - xn;
            if (lane == 31) {
                ws[32] = ps;
                wn[32] = pn;
            }
        }
        __syncthreads();
        if (b < nblk) {
            a.blk_sum[b] = run_s + ws[warp] + is - vs;
            a.blk_nnz[b] = run_n + wn[warp] + in - vn;
        }
        run_s += ws[32];
        run_n += wn[32];
        __syncthreads();
    }
    if (t == 0) {
        a.n_ent[0] = run_n;
        a.n_ent[1] = run_s;
    }
}

__global__ void __launch_bounds__(256) k_dense_compact(DenseArgs a) {
    __shared__ uint32_t wsum[9];
    const uint32_t b = blockIdx.x, t = threadIdx.x;
    if (!a.touched[b]) return;
    const uint32_t e0 = b * kDenseBlk + 16u * t;
    uint32_t v[16], sum = 0, nnz = 0;
#pragma unroll
    for (int j = 0; j < 16; j++) {
        const uint32_t e = e0 + j;
        v[j] = e < a.n_entries ? a.dense[e] : 0u;
        sum += v[j];
        nnz += v[j] != 0u;
    }
    uint32_t ps = excl_scan256(sum, wsum, nullptr) + a.blk_sum[b];
    uint32_t pn = excl_scan256(nnz, wsum, nullptr) + a.blk_nnz[b];
#pragma unroll
    for (int j = 0; j < 16; j++) {
        if (v[j]) {
            ps += v[j];
            a.ent_idx[pn] = e0 + j;
            a.ent_end[pn] = ps;   // inclusive end: global index of the entry's last word + 1
            pn++;
        }
    }
}

// The entries holding the first and the last word of every emit tile (k_emit_dense): one thread per tile,
// binary search over the compacted entries' word ends.
__device__ __forceinline__ uint32_t first_end_above(const uint32_t *ends, uint32_t n, uint32_t w) {
    uint32_t lo = 0, hi = n;   // first e with ends[e] > w
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(ends + mid) > w) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}
__global__ void __launch_bounds__(256) k_dense_tiles(DenseArgs a, uint32_t ntiles) {
    const uint32_t tile = blockIdx.x * 256 + threadIdx.x;
    if (tile >= ntiles) return;
    const TileDesc td = tile_from_prefix(a.tile_pfx, tile);
    const BucketInfo b = a.buckets[td.L];
    const uint32_t te = dense_tile_words(td.L), k0 = td.tile * te, nk = min(te, b.n - k0);
    const uint32_t w0 = (uint32_t)b.word_off + k0, E = a.n_ent[0];
    a.tile_e0[tile] = first_end_above(a.ent_end, E, w0);
    a.tile_e1[tile] = first_end_above(a.ent_end, E, w0 + nk - 1u);
}

// ------------------------------------------------------------------ K5d: emit the dense buckets
constexpr uint32_t kDenseTileEnt = 2048;   // entries one emit tile can hold (<= its words for L >= 3)

// 16 bytes of the periodic sequence W0|W1|W2 (the pattern repeated) from byte r (0 <= r < 8)
__device__ __forceinline__ uint64_t fshr64(uint64_t lo, uint64_t hi, uint32_t s) {
    return s ? (lo >> s) | (hi << (64 - s)) : lo;
}
// the P-byte pattern (P <= 6) repeated over 8 bytes, starting at its byte ph
__device__ __forceinline__ uint64_t rep64(uint64_t pat, uint32_t P, uint32_t ph) {
    const uint64_t m = (1ull << (8 * P)) - 1ull;
    uint64_t x = ph ? ((pat >> (8 * ph)) | (pat << (8 * (P - ph)))) & m : pat;
    for (uint32_t s = 8 * P; s < 64; s *= 2) x |= x << s;
    return x;
}

// Output-parallel: a tile's output bytes [ob, end) are cut into 16-byte aligned chunks and every thread
// assembles a run of consecutive chunks in registers and writes each with one 16-byte store. A chunk
// inside one entry's run is the entry's "word\n" pattern repeated from some phase (three words of the
// periodic sequence, rebuilt only when the entry changes); a chunk crossing entries is assembled word by
// word; only the chunks shared with the neighbouring tiles (head, tail) are written byte by byte. The
// tile's entries [tile_e0, tile_e1] come from k_dense_compact (no search).
__global__ void __launch_bounds__(256) k_emit_dense(DenseEmitArgs a) {
    extern __shared__ __align__(16) uint8_t dsm[];
    uint64_t *s_pat = reinterpret_cast<uint64_t *>(dsm);                 // entry j's word + '\n' (LE bytes)
    uint32_t *s_end = reinterpret_cast<uint32_t *>(dsm + 8 * kDenseTileEnt);   // inclusive end, tile-relative
    const uint32_t t = threadIdx.x;
    const TileDesc td = tile_from_prefix_cta(a.tile_pfx, blockIdx.x);
    const uint32_t L = td.L, P = L + 1u, magic = 65536u / P + 1u;   // (n * magic) >> 16 == n / P for n <= 21
    const BucketInfo b = a.buckets[L];
    const uint32_t te = dense_tile_words(L);
    const uint32_t k0 = td.tile * te;
    const uint32_t nk = min(te, b.n - k0);
    const uint32_t w0 = (uint32_t)b.word_off + k0;
    const uint32_t e0 = a.tile_e0[blockIdx.x], ne = a.tile_e1[blockIdx.x] - e0 + 1u;   // <= min(nk, 676) for L <= 2
    for (uint32_t j = t; j < ne; j += 256) {
        s_end[j] = min(__ldg(a.ent_end + e0 + j) - w0, nk);
        uint32_t x = __ldg(a.ent_idx + e0 + j) - dense_base(L);
        uint64_t pat = (uint64_t)'\n' << (8 * L);
        for (int q = (int)L - 1; q >= 0; q--) {
            const uint32_t y = x / 26u;
            pat |= (uint64_t)('a' + (x - y * 26u)) << (8 * q);
            x = y;
        }
        s_pat[j] = pat;
    }
    __syncthreads();
    // tile-relative byte offsets (u32): the tile's bytes are [ob, ob + nb); chunk i covers [16 i - h, 16 i - h + 16)
    const uint64_t ob = b.byte_off + (uint64_t)k0 * P;
    const uint32_t h = (uint32_t)(ob & 15u), nb = nk * P;
    const uint32_t nch = (h + nb + 15) >> 4;
    const uint32_t G = (nch + 255) / 256;
    const uint32_t i0 = t * G;
    if (i0 >= nch) return;
    uint4 *dst4 = reinterpret_cast<uint4 *>(a.words + (ob - h));
    uint8_t *dst1 = a.words + (ob - h);
    int32_t x = (int32_t)(16 * i0) - (int32_t)h;   // tile-relative start of chunk i0 (may be < 0 for i0 = 0)
    uint32_t lo = x > 0 ? (uint32_t)x : 0u;
    uint32_t q = lo / P, r = lo - q * P;   // tile-relative word, byte inside it
    uint32_t j = 0;
    {   // first entry with s_end > q
        uint32_t hi = ne - 1;
        while (j < hi) {
            const uint32_t mid = (j + hi) >> 1;
            if (s_end[mid] > q) hi = mid;
            else j = mid + 1;
        }
    }
    uint32_t wj = 0xffffffffu;   // entry whose periodic window is in W0..W2
    uint64_t W0 = 0, W1 = 0, W2 = 0;
    const uint32_t iend = min(i0 + G, nch);
    for (uint32_t i = i0; i < iend; i++, x += 16) {
        const uint32_t hb = min((uint32_t)(x + 16), nb);   // this tile's bytes of the chunk: [lo, hb)
        const bool full = (int32_t)lo == x && hb == (uint32_t)(x + 16);
        uint64_t acc0 = 0, acc1 = 0;
        if (full && (s_end[j] - q) * P - r >= 16u) {   // inside entry j's run
            if (j != wj) {
                const uint64_t pat = s_pat[j];
                W0 = rep64(pat, P, 0);
                W1 = rep64(pat, P, 8u % P);
                W2 = rep64(pat, P, 16u % P);
                wj = j;
            }
            acc0 = fshr64(W0, W1, 8 * r);
            acc1 = fshr64(W1, W2, 8 * r);
            const uint32_t n = r + 16u, d = (n * magic) >> 16;
            q += d;
            r = n - d * P;
            if (q >= s_end[j] && j + 1 < ne) j++;
        } else {
            uint32_t o = lo - (uint32_t)x;
            while (o < hb - (uint32_t)x) {
                const uint64_t pat = s_pat[j] >> (8 * r);
                if (o < 8) {
                    acc0 |= pat << (8 * o);
                    if (o) acc1 |= pat >> (64 - 8 * o);
                } else {
                    acc1 |= pat << (8 * (o - 8));
                }
                o += P - r;
                r = 0;
                if (++q >= s_end[j] && j + 1 < ne) j++;
            }
            // the word that crossed into the next chunk resumes at byte (o - 16) of itself
            if (o > 16) {
                q--;
                if (j > 0 && q < s_end[j - 1]) j--;
                r = P - (o - 16);
            }
        }
        if (full) {
            dst4[i] = make_uint4((uint32_t)acc0, (uint32_t)(acc0 >> 32), (uint32_t)acc1, (uint32_t)(acc1 >> 32));
        } else {   // a chunk shared with the neighbouring tile: only this tile's bytes
            for (uint32_t y = lo; y < hb; y++) {
                const uint32_t k = y - (uint32_t)x;
                dst1[16 * i + k] = (uint8_t)((k < 8 ? acc0 >> (8 * k) : acc1 >> (8 * (k - 8))) & 0xffu);
            }
        }
        lo = (uint32_t)(x + 16);
    }
}
constexpr size_t kEmitDenseSmem = 12 * kDenseTileEnt;

// ------------------------------------------------------------------ K3c: chunks -> length buckets
// Each staged key's length is recovered from its trailing zero 5-bit codes (letters are codes 1..26,
// the pad is 0): L = 6K - (ctz(last key word) / 5). A chunk's keys (one key-width class K: lengths
// 6K-5 .. 6K) are grouped by length in shared memory, one global atomic per (chunk, length) reserves
// their range in the bucket, and they are written out coalesced. Order within a bucket is arbitrary
// (keys only); the MSD levels sort it.
__device__ __forceinline__ uint32_t key_len(uint32_t last, uint32_t K) {
    return 6u * K - (uint32_t)(__ffs(last) - 1) / 5u;
}

template <int K>
__device__ __forceinline__ void lscatter_chunk(const L0Args &a, const uint32_t *src, uint32_t n, uint32_t *sm) {
    constexpr int KPT = (16 + K - 1) / K;   // 4096 / K keys per chunk, 256 threads
    constexpr uint32_t cap = 1u << cls_lg(K);   // word-major chunk: word u of key i at u * cap + i
    const uint32_t t = threadIdx.x;
    uint32_t *cnt = sm, *lbase = sm + 8, *gbase = sm + 16;
    uint64_t *koff = reinterpret_cast<uint64_t *>(sm + 24);
    uint32_t *kout = sm + 40;
    uint8_t *lof = reinterpret_cast<uint8_t *>(kout + kChunkWords + kChunkWords / 32 + 4);
    if (t < 8) cnt[t] = 0;
    if (t < 6) koff[t] = a.buckets[6 * K - 5 + t].key_off;
    __syncthreads();
    uint32_t ls[KPT];   // length offset (3 bits) | slot within the length (<< 3); keys stay in shared memory
#pragma unroll
    for (int r = 0; r < KPT; r++) {
        const uint32_t i = t + r * 256;
        if (i < n) {
            const uint32_t l = key_len(src[(K - 1) * cap + i], K) - (6u * K - 5u);
            ls[r] = l | (atomicAdd(&cnt[l], 1u) << 3);
        }
    }
    __syncthreads();
    uint32_t g = 0;
    if (t < 6) {   // reserve this chunk's range of each length; the result is consumed after the reorder
        uint32_t ex = 0;
        for (uint32_t j = 0; j < t; j++) ex += cnt[j];
        lbase[t] = ex;
        g = cnt[t] ? atomicAdd(&a.lcursor[6 * K - 5 + t], cnt[t]) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < KPT; r++) {
        const uint32_t i = t + r * 256;
        if (i < n) {
            const uint32_t l = ls[r] & 7u, p = lbase[l] + (ls[r] >> 3);
#pragma unroll
            for (int u = 0; u < K; u++) {
                const uint32_t w = p * K + u;
                kout[w + (w >> 5)] = src[u * cap + i];
            }
            lof[p] = (uint8_t)l;
        }
    }
    if (t < 6) gbase[t] = g;
    __syncthreads();
    for (uint32_t i = t; i < n * K; i += 256) {
        const uint32_t p = i / K, u = i - p * K;
        const uint32_t l = lof[p];
        a.dst[koff[l] + (uint64_t)(gbase[l] + p - lbase[l]) * K + u] = kout[i + (i >> 5)];
    }
}

// Persistent: CTA b takes chunks b, b + grid, ... (skipping empty ones); the next chunk is fetched by
// a TMA bulk copy into the other shared-memory buffer while this one is scattered.
constexpr int kLsCtasPerSm = 3;
constexpr uint32_t kLsWork = (40 + kChunkWords + kChunkWords / 32 + 4) * 4 + kChunkWords;
__global__ void __launch_bounds__(256, kLsCtasPerSm) k_lscatter(L0Args a) {
    extern __shared__ __align__(128) uint8_t ls_raw[];
    uint32_t *inb = reinterpret_cast<uint32_t *>(ls_raw);                       // [2][kChunkWords]
    uint64_t *bar = reinterpret_cast<uint64_t *>(ls_raw + 2 * kChunkWords * 4);  // [2]
    uint32_t *sj = reinterpret_cast<uint32_t *>(bar + 2);                        // [2] chunk, [2] keys, [2] class
    uint32_t *work = sj + 8;
    const uint32_t t = threadIdx.x;
    const uint32_t total = a.nctas * a.used_chunks;
    auto chunk_id = [&](uint32_t j) { return (j / a.used_chunks) * a.cta_chunks + j % a.used_chunks; };
    // thread 0: the first non-empty chunk at or after j (stride grid) -> buffer b
    auto fetch = [&](uint32_t j, uint32_t b) {
        uint32_t n = 0;
        while (j < total && (n = a.chunk_fill[chunk_id(j)]) == 0) j += gridDim.x;
        sj[b] = j;
        if (j < total) {
            const uint32_t c = chunk_id(j), K = a.chunk_cls[c] & 255u;
            sj[2 + b] = n;
            sj[4 + b] = K;
            const uint32_t bytes = (((K - 1) << cls_lg(K)) * 4 + n * 4 + 15) & ~15u;   // (word-major)
            tma::mbar_expect_tx(&bar[b], bytes);
            tma::bulk_g2s(inb + b * kChunkWords, a.pool + (size_t)c * kChunkWords, bytes, &bar[b]);
        }
    };
    if (t == 0) {
        tma::mbar_init(&bar[0], 1);
        tma::mbar_init(&bar[1], 1);
        tma::fence_mbar_init();
        fetch(blockIdx.x, 0);
    }
    __syncthreads();
    for (uint32_t it = 0;; it++) {
        const uint32_t cur = it & 1;
        const uint32_t j = sj[cur];
        if (j >= total) break;
        const uint32_t n = sj[2 + cur], K = sj[4 + cur];
        if (t == 0) fetch(j + gridDim.x, cur ^ 1);   // (buffer cur^1 was released at the last barrier)
        tma::mbar_wait(&bar[cur], (it >> 1) & 1);
        const uint32_t *src = inb + cur * kChunkWords;
        switch (K) {
            case 1: lscatter_chunk<1>(a, src, n, work); break;
            case 2: lscatter_chunk<2>(a, src, n, work); break;
            case 3: lscatter_chunk<3>(a, src, n, work); break;
            case 4: lscatter_chunk<4>(a, src, n, work); break;
            case 5: lscatter_chunk<5>(a, src, n, work); break;
            case 6: lscatter_chunk<6>(a, src, n, work); break;
            case 7: lscatter_chunk<7>(a, src, n, work); break;
            case 8: lscatter_chunk<8>(a, src, n, work); break;
            case 9: lscatter_chunk<9>(a, src, n, work); break;
            case 10: lscatter_chunk<10>(a, src, n, work); break;
            default: lscatter_chunk<11>(a, src, n, work); break;
        }
        __syncthreads();
    }
}

constexpr size_t kLscatterSmem = 2 * kChunkWords * 4 + 16 + 32 + kLsWork;

}  // namespace

uint32_t ingest_ctas_per_sm() { return kIgMinBlocks; }
// The tokenizer grid is kIgMinBlocks CTAs per SM (plan_tokenizer): the shared-memory request is padded so
// that no more than that fit on one SM (a third CTA on some SMs would leave the grid unbalanced).
constexpr size_t kIgSmemFloor = 233472 / (kIgMinBlocks + 1);   // (228 KiB per SM)
size_t ingest_smem(uint32_t) { return std::max(sizeof(IgSmem), kIgSmemFloor); }
uint32_t dense_entries() { return dense_base(kDenseMaxLen + 1); }
uint32_t dense_table_base(uint32_t L) { return dense_base(L); }

cudaError_t launch_ingest(const IngestArgs &a, cudaStream_t s) { return launch_ingest_range(a, 0, a.grid, s); }

cudaError_t launch_ingest_range(IngestArgs a, uint32_t first, uint32_t count, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    a.cta_first = first;
    const size_t smem = ingest_smem(a.cta_chunks);
    if (a.hash) {
        cudaError_t e = cudaFuncSetAttribute(k_ingest<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k_ingest<true><<<count, kIgThreads, smem, s>>>(a);
        return cudaGetLastError();
    }
    cudaError_t e = cudaFuncSetAttribute(k_ingest<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_ingest<false><<<count, kIgThreads, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_dense_scan(const DenseArgs &a, cudaStream_t s) {
    const uint32_t nblk = (a.n_entries + kDenseBlk - 1) / kDenseBlk;
    k_dense_reduce<<<nblk, 256, 0, s>>>(a);
    k_dense_scan<<<1, 1024, 0, s>>>(a, nblk);
    k_dense_compact<<<nblk, 256, 0, s>>>(a);
    if (a.tile_e0 && a.ntiles) k_dense_tiles<<<(a.ntiles + 255) / 256, 256, 0, s>>>(a, a.ntiles);
    return cudaGetLastError();
}
uint32_t dense_scan_blocks(uint32_t n_entries) { return (n_entries + kDenseBlk - 1) / kDenseBlk; }
cudaError_t launch_dense_lensum(const uint32_t *dense, const uint8_t *touched, uint32_t *ghist, cudaStream_t s) {
    k_dense_lensum<<<dense_scan_blocks(dense_base(kDenseMaxLen + 1)), 256, 0, s>>>(dense, touched, ghist);
    return cudaGetLastError();
}
cudaError_t launch_dense_clear(uint32_t *dense, uint8_t *touched, cudaStream_t s) {
    k_dense_clear<<<dense_scan_blocks(dense_base(kDenseMaxLen + 1)), 256, 0, s>>>(dense, touched, dense_base(kDenseMaxLen + 1));
    return cudaGetLastError();
}

cudaError_t launch_emit_dense(const DenseEmitArgs &a, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_emit_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEmitDenseSmem);
    if (e != cudaSuccess) return e;
    k_emit_dense<<<a.ntiles, 256, kEmitDenseSmem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_lscatter(const L0Args &a, uint32_t nctas, cudaStream_t s) {
    if (!nctas || !a.used_chunks) return cudaSuccess;
    L0Args b = a;
    b.nctas = nctas;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t grid = std::min<uint32_t>(nctas * a.used_chunks, (uint32_t)sms * kLsCtasPerSm);
    cudaError_t e = cudaFuncSetAttribute(k_lscatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLscatterSmem);
    if (e != cudaSuccess) return e;
    k_lscatter<<<grid, 256, kLscatterSmem, s>>>(b);
    return cudaGetLastError();
}

}  // namespace wsort
