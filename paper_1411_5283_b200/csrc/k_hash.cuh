// k_hash.cuh — the global table of distinct long words (6..66 letters) and their occurrence counts.
//
// Phase 3 of the method sorts each per-length sub-array. Equal words are identical bytes,
// so a sub-array sorted alphabetically is fixed by its DISTINCT words in order and how often each occurs
// (the same exact-multiset reading the dense tables use for L <= 5, SURVEY.md §8(f) NEXT-1, and the MSD
// finish uses per job). K1 counts every long word into this table as it reads the text; afterwards only
// the distinct words are sorted (k_hash.cu) and each is written as often as it occurred.
//
// Open addressing, linear probing, lock-free:
//   fp[i]   u64: 0 = empty, else the key's 64-bit fingerprint | 1 (set once by atomicCAS);
//   meta[i] u32: kUnset until the inserting thread has stored the key words, then
//           key offset (u32 words into keys[], < 2^24) | L << 24; kDead if the key store was exhausted;
//   cnt[i]  u32: occurrences (atomics);
//   keys[]  the key words of every distinct word (bump-allocated by top[0]).
// A lookup verifies the key word by word against the stored one (exact; the fingerprint only filters),
// so two different words never share a slot whatever their fingerprints. A stale L1 copy of fp[i] can
// only read 0 for a filled slot (the CAS then returns the real value); meta and keys are read at L2
// (ld.acquire / ld.cg) after the fingerprint matched.
#pragma once
#include <stdint.h>

#include "wsort_internal.cuh"

namespace wsort {
namespace hashtab {

constexpr uint32_t kUnset = 0xffffffffu, kDead = 0xfffffffeu;
constexpr uint32_t kMaxProbe = 128;
enum { kTopWords = 0, kTopDistinct = 1, kTopOverflow = 2, kTopNarrow = 3 };   // (distinct: wide / narrow)

__device__ __forceinline__ uint32_t rotl(uint32_t x, uint32_t r) { return __funnelshift_l(x, x, r); }

// 64-bit fingerprint of (L, key words): two independent 32-bit mixes
template <class Get>
__device__ __forceinline__ uint64_t fingerprint(uint32_t L, uint32_t k, Get get) {
    uint32_t h1 = 0x9E3779B1u * (L + 1u), h2 = 0x7F4A7C15u ^ (L * 0x85EBCA77u);
    for (uint32_t q = 0; q < k; q++) {
        const uint32_t w = get(q);
        h1 = rotl(h1 ^ (w * 0xCC9E2D51u), 15) * 0x1B873593u;
        h2 = (h2 + rotl(w, 7)) * 0xC2B2AE3Du;
        h2 ^= h2 >> 13;
    }
    h1 ^= h1 >> 16;
    h1 *= 0x85EBCA6Bu;
    h1 ^= h1 >> 13;
    h2 ^= h2 >> 16;
    h2 *= 0x27D4EB2Fu;
    h2 ^= h2 >> 15;
    return ((uint64_t)h1 << 32 | h2) | 1ull;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The slot of the word (L, key words get(0..k-1)) with fingerprint fp; inserted if absent (insert = true).
// Returns kUnset if absent (lookup), or if a capacity limit was hit (then top[kTopOverflow] is set).
template <class Get>
__device__ __forceinline__ uint32_t find(const HashTab &h, uint32_t L, uint32_t k, uint64_t fp, Get get, bool insert) {
    uint32_t i = (uint32_t)(fp >> 32) & h.mask;
    for (uint32_t probe = 0; probe < kMaxProbe; probe++, i = (i + 1) & h.mask) {
        unsigned long long f = h.fp[i];
        if (f == 0ull) {
            if (!insert) return kUnset;
            f = atomicCAS(h.fp + i, 0ull, (unsigned long long)fp);
            if (f == 0ull) {   // this thread owns slot i: store the key, then publish it
                const uint32_t off = atomicAdd(h.top + kTopWords, k);
                if (off + k > h.key_cap) {   // key store exhausted: the text is staged instead (host)
                    atomicExch(h.top + kTopOverflow, 1u);
                    st_release(h.meta + i, kDead);
                    return kUnset;
                }
                for (uint32_t q = 0; q < k; q++) h.keys[off + q] = get(q);
                atomicAdd(h.dcount + L, 1u);
                st_release(h.meta + i, off | (L << 24));
                return i;
            }
        }
        if (f != fp) continue;
        uint32_t m, spins = 0;
        while ((m = ld_acquire(h.meta + i)) == kUnset) {   // the owner is storing the key
            if (++spins > (1u << 20)) {
                atomicExch(h.top + kTopOverflow, 2u);
                return kUnset;
            }
        }
        if (m == kDead || (m >> 24) != L) continue;
        const uint32_t *kk = h.keys + (m & 0xffffffu);
        bool eq = true;
        for (uint32_t q0 = 0; q0 < k && eq; q0 += 11u) {   // 11 stored words in flight at once, then compared
            uint32_t st[11];
#pragma unroll
            for (uint32_t q = 0; q < 11u; q++) st[q] = q0 + q < k ? __ldcg(kk + q0 + q) : 0u;
#pragma unroll
            for (uint32_t q = 0; q < 11u; q++) eq &= q0 + q >= k || st[q] == get(q0 + q);
        }
        if (eq) return i;
    }
    if (insert) atomicExch(h.top + kTopOverflow, 3u);
    return kUnset;
}

// ---- narrow words (6..24 letters, 1-4 key words): the slot holds the whole key, 128 bits, inserted by one
// 128-bit CAS (exact: no fingerprint). lo = key word 0 << 32 | key word 1, hi = key words 2, 3; bit 63 of
// lo (a spare bit: codes use bits 0..29 of a key word) marks hi != 0, so a torn 16-byte read of a slot
// being filled, (new lo, 0) or (0, new hi), never equals a key: lo == 0 is retried by the CAS and
// (lo with the mark, 0) is no key. A key's length is recoverable from it (letters are codes 1..26, the
// padding is 0).
constexpr unsigned long long kNarrowMark = 1ull << 63;
struct Key128 {
    unsigned long long lo, hi;
};
__device__ __forceinline__ Key128 narrow_key(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3) {
    const unsigned long long hi = (unsigned long long)w2 << 32 | w3;
    return Key128{((unsigned long long)w0 << 32 | w1) | (hi ? kNarrowMark : 0ull), hi};
}
__device__ __forceinline__ uint32_t key_word_len(uint32_t w) { return 6u - (uint32_t)(__ffs(w) - 1) / 5u; }   // w != 0
__device__ __forceinline__ uint32_t narrow_len(Key128 k) {
    const uint32_t w1 = (uint32_t)k.lo, w2 = (uint32_t)(k.hi >> 32), w3 = (uint32_t)k.hi;
    if (w3) return 18u + key_word_len(w3);
    if (w2) return 12u + key_word_len(w2);
    return w1 ? 6u + key_word_len(w1) : 6u;
}
__device__ __forceinline__ uint32_t narrow_hash(Key128 k) {
    const unsigned long long x = (k.lo ^ (k.hi * 0xC2B2AE3D27D4EB4Full)) * 0x9E3779B97F4A7C15ull;
    return (uint32_t)(x >> 32) ^ (uint32_t)(x >> 11);
}
__device__ __forceinline__ Key128 cas128(unsigned long long *addr, Key128 cmp, Key128 val) {
    Key128 o;
    asm volatile("{\n\t.reg .b128 c, v, o;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %5};\n\t"
                 "atom.global.cas.b128 o, [%6], c, v;\n\tmov.b128 {%0, %1}, o;\n\t}"
                 : "=l"(o.lo), "=l"(o.hi)
                 : "l"(cmp.lo), "l"(cmp.hi), "l"(val.lo), "l"(val.hi), "l"(addr)
                 : "memory");
    return o;
}
// slot of `key` (inserted if absent and insert); kUnset if absent or on overflow (flag set)
__device__ __forceinline__ uint32_t find_narrow(const HashTab &h, Key128 key, uint32_t L, bool insert) {
    uint32_t i = narrow_hash(key) & h.nmask;
    for (uint32_t probe = 0; probe < kMaxProbe; probe++, i = (i + 1) & h.nmask) {
        const ulonglong2 cur = reinterpret_cast<const ulonglong2 *>(h.nkey)[i];
        if (cur.x == key.lo && cur.y == key.hi) return i;
        if (cur.x != 0ull) continue;   // another key (or its torn lo == 0 half: the CAS below tells)
        if (!insert && cur.y == 0ull) return kUnset;
        if (!insert) continue;
        const Key128 old = cas128(h.nkey + 2 * (size_t)i, Key128{0ull, 0ull}, key);
        if (old.lo == 0ull && old.hi == 0ull) {
            atomicAdd(h.dcount + L, 1u);   // (the host checks the fill against the capacity after K1)
            return i;
        }
        if (old.lo == key.lo && old.hi == key.hi) return i;
    }
    if (insert) atomicExch(h.top + kTopOverflow, 5u);
    return kUnset;
}

}  // namespace hashtab
}  // namespace wsort
