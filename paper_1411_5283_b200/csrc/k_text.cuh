// k_text.cuh — byte-level helpers shared by the text kernels (K1 ingest, K3 pack+scatter).
// Phase 1 of the method ("removing / ignoring the special characters"): a word is a
// maximal run of ASCII letters (reading A1), folded to lower case (A2).
#pragma once
#include <stdint.h>

namespace wsort {
namespace text {

constexpr uint32_t kFull = 0xffffffffu;

// 4 bytes -> 4-bit letter mask (bit i = byte i is in [A-Za-z]).
__device__ __forceinline__ uint32_t letter_nibble(uint32_t x) {
    uint32_t w = (x | 0x20202020u) & 0x7f7f7f7fu;   // fold case, drop bit 7
    uint32_t a = w + 0x1f1f1f1fu;                    // bit 7 set iff w >= 'a'
    uint32_t b = w + 0x05050505u;                    // bit 7 set iff w >= '{'
    uint32_t m = a & ~b & ~x & 0x80808080u;          // and the original byte < 0x80
    return ((m >> 7) * 0x10204080u) >> 28;           // gather bits 7,15,23,31
}

// 32 bytes (two uint4) -> 32-bit letter mask.
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

// Pack letters [0, min(L,6)) of the word at byte offset boff of a 4-byte aligned buffer into one
// key word: letter j -> its 5-bit code c & 0x1F at bits 29-5j .. 25-5j; unused positions are 0.
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

// Letter codes of 6 bytes (bytes 0..3 in lo, 4..5 in the low half of hi) as one key word, as pack6.
__device__ __forceinline__ uint32_t codes6(uint32_t lo, uint32_t hi) {
    lo &= 0x1f1f1f1fu;
    hi &= 0x00001f1fu;
    const uint32_t r = __byte_perm(lo, 0, 0x0123);                   // letter 0 in the top byte
    const uint32_t t1 = (r & 0x001f001fu) | ((r & 0x1f001f00u) >> 3);
    const uint32_t t2 = (t1 & 0x3ffu) | ((t1 >> 16) << 10);           // 4 letters, 20 bits
    return (t2 << 10) | ((hi & 0x1fu) << 5) | (hi >> 8);
}

// All k = ceil(L/6) key words of the word of L letters at byte s (pack6 of each 6-letter slice): two key
// words are 12 bytes = 3 aligned words at one shift, so the window is read once (3 loads per pair);
// only the last key word is masked. Key word q goes to dst[q * stride] (stride 1: contiguous key; the
// staging chunks store word q of every key in a row of its own, stride = the chunk's key capacity).
__device__ __forceinline__ void pack_key(const uint32_t *buf32, uint32_t s, uint32_t L, uint32_t k, uint32_t *dst,
                                         uint32_t stride = 1) {
    const uint32_t sh = 8u * (s & 3u), rem = L - 6u * (k - 1u);   // letters in the last key word: 1..6
    const uint32_t last = rem < 6u ? ~((1u << (5u * (6u - rem))) - 1u) : 0xffffffffu;
    const uint32_t *p = buf32 + (s >> 2);
    uint32_t w0 = p[0];
    for (uint32_t q = 0; q < k; q += 2, p += 3) {
        const uint32_t w1 = p[1], w2 = p[2], w3 = p[3];
        const uint32_t b0 = __funnelshift_r(w0, w1, sh), b1 = __funnelshift_r(w1, w2, sh), b2 = __funnelshift_r(w2, w3, sh);
        dst[q * stride] = codes6(b0, b1) & (q + 1u == k ? last : 0xffffffffu);
        if (q + 1u < k)
            dst[(q + 1u) * stride] = codes6(__funnelshift_r(b1, b2, 16), b2 >> 16) & (q + 2u == k ? last : 0xffffffffu);
        w0 = w3;
    }
}

}  // namespace text
}  // namespace wsort
