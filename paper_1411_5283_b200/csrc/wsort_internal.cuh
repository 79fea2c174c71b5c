// wsort_internal.cuh — shared definitions of the libwsort kernels and host runtime (sm_100a).
// Product code only; nothing here is shared with oracle/ or gen/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace wsort {

constexpr int kMaxLen = 255;          // WSORT_MAX_WORD_LEN (reading A7)
constexpr int kHistBins = 257;        // lengths 0..255 + "too long" bin 256

// ---------------- tokenizer (K1 count, K3 pack+scatter) ----------------
constexpr int kTkThreads = 256;
constexpr int kTkStep = 8192;         // bytes per step = 32 bytes per thread
constexpr int kTkPre = 16;            // bytes kept before the step (previous-byte lookup)
constexpr int kTkHalo = 256;          // bytes kept after the step (tail of a word crossing the step)
constexpr int kTkBuf = kTkPre + kTkStep + kTkHalo;   // 8464 bytes = 529 uint4
constexpr int kTkMaxWords = kTkStep / 2;             // at most one word start per two bytes
constexpr int kTextFrontPad = 256;    // zero bytes before text[0] in the device copy (alignment)

// ---------------- keys ----------------
// A word of length L is packed into KW(L) = ceil(L/6) u32 "key words": letter j (0-based) of the
// word goes to key word j/6, bits [29-5*(j%6) .. 25-5*(j%6)], as its 5-bit code c & 0x1F
// ('a'/'A' -> 1 ... 'z'/'Z' -> 26); unused positions are 0, which orders below 'a'. Within one
// length bucket, unsigned comparison of key words in order == alphabetical order (reading A4).
__host__ __device__ constexpr int kw_of(int L) { return (L + 5) / 6; }
// LSD digits are 2 letters (10 bits): digit q (q = 0 is the most significant) covers letters
// 2q, 2q+1 = key word q/3, bits [29-10*(q%3) .. 20-10*(q%3)].
__host__ __device__ constexpr int ndig_of(int L) { return (L + 1) / 2; }
constexpr int kRadixBins = 1024;

struct Summary {                   // written by K2, copied to pinned host memory
    uint64_t n_words;
    uint64_t letters;
    uint32_t max_len;
    uint32_t too_long;             // number of words longer than kMaxLen
    uint64_t off[kHistBins];       // off[L] = #words shorter than L (L = 0..256); off[256] = W
    uint64_t key_off[kHistBins];   // u32 key-word offset of bucket L
    uint64_t byte_off[kHistBins];  // output byte offset of bucket L
};

struct BucketInfo {                // per-length bucket, built on the host after tokenize
    uint64_t key_off;              // u32 words into the key buffers
    uint64_t word_off;             // off[L]
    uint64_t byte_off;             // output byte offset
    uint32_t n;                    // words in the bucket
    uint32_t kw;                   // key words per word
    uint32_t ndig;                 // LSD digits
    uint32_t tile_keys;            // keys per radix / merge tile
    uint32_t dh_row;               // first row of this bucket's digit histograms (rows of 1024)
    uint32_t final_b;              // sorted keys end in buffer B (1) or A (0)
    uint64_t elem_off;             // u32 words into the final buffer (element layout)
    uint32_t estride;              // u32 words per element in the final buffer (kw, or kw+1 with an
                                   // inline payload word)
    uint32_t aux;                  // msd: keys per scatter tile
};

struct TileDesc {
    uint32_t L;
    uint32_t tile;                 // tile index within the bucket
};

// Tile b of a launch whose tiles are enumerated bucket by bucket: pfx[L] = first tile of bucket L
// (pfx[256] = all tiles). Lets a kernel find its (bucket, tile) without a host-built tile array.
__device__ __forceinline__ TileDesc tile_from_prefix(const uint32_t *pfx, uint32_t b) {
    uint32_t lo = 0, hi = 255;   // largest L with pfx[L] <= b
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(pfx + mid) <= b) lo = mid;
        else hi = mid - 1;
    }
    return TileDesc{lo, b - __ldg(pfx + lo)};
}

// The same for a block-uniform b, called by every thread of the block (full warps): each warp finds it in
// two dependent loads instead of eight (coarse: pfx[8 lane]; fine: pfx[8 k + lane], k the coarse interval)
__device__ __forceinline__ TileDesc tile_from_prefix_cta(const uint32_t *pfx, uint32_t b) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t m = __ballot_sync(0xffffffffu, __ldg(pfx + 8u * lane) <= b);   // (pfx[0] = 0 <= b)
    const uint32_t k = 31u - (uint32_t)__clz(m);
    const uint32_t idx = min(8u * k + (lane & 15u), 256u);
    const uint32_t v = __ldg(pfx + idx);
    const uint32_t m2 = __ballot_sync(0xffffffffu, lane < 16u && v <= b);
    const uint32_t f = 31u - (uint32_t)__clz(m2);
    const uint32_t L = 8u * k + f;
    return TileDesc{L, b - __shfl_sync(0xffffffffu, v, f)};
}

// ---------------- launchers (defined in the .cu files) ----------------
struct TkArgs {
    const uint8_t *text;           // device copy, text[-kTextFrontPad..-1] = 0, zero tail padding
    uint64_t n;
    uint32_t nsteps;
    uint32_t steps_per_cta;
    uint32_t grid;
    uint32_t *cta_hist;            // [grid][257]
    uint32_t *cta_base;            // [grid][256]
    const BucketInfo *buckets;     // [256]
    uint32_t *keys;                // key buffer A
    uint32_t *payload;             // optional u32 local source offsets (bucket order)
};

cudaError_t launch_bucket_offsets(const uint32_t *ghist, Summary *d_sum, cudaStream_t s);
cudaError_t launch_count_lengths(const TkArgs &a, uint32_t *ghist, cudaStream_t s);
cudaError_t launch_cta_bases(const TkArgs &a, uint32_t max_len, cudaStream_t s);
cudaError_t launch_pack_scatter(const TkArgs &a, cudaStream_t s);

// ---------------- K1 ingest: one text pass (k_ingest.cu) ----------------
#ifndef WSORT_IG_THREADS
#define WSORT_IG_THREADS 1024
#endif
constexpr int kIgThreads = WSORT_IG_THREADS;
constexpr int kIgStep = 16384;                       // bytes per ingest step = 32 per thread
constexpr int kIgBuf = kTkPre + kIgStep + kTkHalo;   // 16656 bytes
constexpr uint32_t kDenseMaxLen = 5;                 // words of L <= 5 are counted, not sorted
constexpr uint32_t kDenseBlkEntries = 4096;          // the dense table's blocks (touched flags, scans)
constexpr uint32_t kMaxStageKw = 11;                 // words of 6 <= L <= 66 are staged as keys
constexpr uint32_t kChunkWords = 4096;               // u32 words per staging chunk (16 KiB)
constexpr uint32_t kC0Bins = 6 * 1024;               // level-0 bins of a class: (length - (6K-5)) << 10 | digit
// keys per staging chunk of key width k (log2): the largest power of two <= kChunkWords / k; chunks are
// word-major (word q of key i at q << chunk_lg(k) | i)
__host__ __device__ constexpr uint32_t chunk_lg(uint32_t k) { return k == 1 ? 12u : k == 2 ? 11u : k <= 4 ? 10u : k <= 8 ? 9u : 8u; }
enum { kIgMaxChunks = 0, kIgOverflow = 1, kIgVeryLong = 2, kIgClsCnt = 4, kIgCtrs = 16 };   // [4, 15): chunks per class
// chunks per CTA region: a staged word's key bytes <= its text bytes (+256 for the last word), a full
// chunk holds >= 2304 key words (class 9: 256 keys of 9 words), one partial chunk per class
__host__ __device__ constexpr uint32_t ingest_cta_chunks(uint64_t range_bytes) {
    return (uint32_t)((range_bytes + 256) / 9000 + 2 * kMaxStageKw + 10);
}
// The table of distinct long words (k_hash.cuh): K1 counts every word of 6..66 letters into it.
struct HashTab {
    // narrow words (6..24 letters: 1-4 key words): the 128-bit key itself is the slot's tag (exact)
    unsigned long long *nkey;               // [2 (nmask + 1)] (0, 0) = empty, else the key (k_hash.cuh)
    uint32_t *ncnt;                         // [nmask + 1] occurrences
    uint32_t nmask;
    // wide words (25..255 letters): fingerprint-tagged slots, keys in a side store, verified word by word
    unsigned long long *fp;                 // [mask + 1] 0 = empty, else fingerprint | 1
    uint32_t *meta;                         // [mask + 1] key offset | L << 24 (kUnset / kDead)
    uint32_t *cnt;                          // [mask + 1] occurrences
    uint32_t *keys;                         // [key_cap] key words of the distinct wide words
    uint32_t *top;                          // [4] key words used, distinct words, overflow flag
    uint32_t *dcount;                       // [256] distinct words per length
    uint32_t mask, key_cap, max_distinct;
};
struct HashGatherArgs {
    HashTab tab;
    const BucketInfo *buckets;              // distinct-key buckets (key_off, kw)
    uint32_t *lcursor;                      // [256] zeroed by the host
    uint32_t *keys_a;
};
// words per k_emit_runs tile (its runs are handled in segments that fit shared memory)
__host__ __device__ constexpr uint32_t run_tile_words(uint32_t L) { return L ? 8192u : 8192u; }
struct HashRunArgs {
    HashTab tab;
    const BucketInfo *buckets;              // output buckets: word_off (global word index), byte_off, n words
    const BucketInfo *kbuckets;             // distinct-key buckets: key_off into `keys`, n distinct keys
    const uint32_t *dist_pfx;               // [257] first distinct key of bucket L (tile_from_prefix layout)
    uint32_t D;                             // distinct keys
    const uint32_t *keys;                   // the sorted distinct keys (buffer B)
    uint32_t *run_end;                      // [D] inclusive run ends, long-word index (words of >= 6 letters)
    uint64_t long_base;                     // global word index of the first long word (off[6])
    const uint32_t *tile_pfx;               // [257] first emit tile of bucket L
    uint32_t ntiles;
    uint32_t *tile_e0, *tile_e1;            // [ntiles] runs of the tile's first / last word
    uint8_t *words;
};
cudaError_t launch_hash_gather(const HashGatherArgs &a, cudaStream_t s);
constexpr uint32_t kWideSortWords = 8192;   // k_sort_wide: a bucket's distinct keys (> 66 letters) in shared memory
constexpr uint32_t kMsdMaxLen = 66;         // the MSD radix finish holds keys of <= 11 words
cudaError_t launch_sort_wide(const BucketInfo *kb, const uint32_t *lens, uint32_t nlens, const uint32_t *keys_a,
                             uint32_t *keys_b, cudaStream_t s);
cudaError_t launch_hash_runs(const HashRunArgs &a, uint32_t *scan_blk, cudaStream_t s);   // runs, scan, tiles
uint32_t hash_scan_blocks(uint32_t D);
cudaError_t launch_emit_runs(const HashRunArgs &a, cudaStream_t s);
cudaError_t launch_hash_counts(const HashRunArgs &a, cudaStream_t s);   // run_end[j] = count of key j (no scan)
cudaError_t launch_scan_u32(uint32_t *v, uint32_t n, uint32_t *scan_blk, cudaStream_t s);   // inclusive, in place

// ---------------- ragged backing: references into the text (k_ragged.cu) ----------------
struct RaggedArgs {
    const uint8_t *text;                    // the device text (padded)
    const BucketInfo *buckets;              // word_off (index into in / out), byte_off, n
    const uint32_t *tile_pfx;               // [257] first 1024-reference tile of bucket L
    uint32_t ntiles;
    const uint32_t *in;                     // references (text byte offsets), bucket order
    uint32_t *out;
    uint32_t run;                           // merge pass: sorted run length
    uint8_t *words;
    uint64_t *src_off;                      // nullable
    uint64_t global_base;
};
uint32_t ragged_tile();
cudaError_t launch_ragged_tiles(const RaggedArgs &a, cudaStream_t s);
cudaError_t launch_ragged_merge(const RaggedArgs &a, cudaStream_t s);
cudaError_t launch_ragged_emit(const RaggedArgs &a, cudaStream_t s);

// ---------------- multi-GPU exchange of (distinct word, count) records (k_xchg.cu) ----------------
struct XchgArgs {
    HashTab tab;                            // (absorb) this rank's table, cleared
    const BucketInfo *kbuckets;             // the gathered distinct keys' buckets (keys_a layout)
    const uint32_t *dist_pfx;               // [257] first distinct key of bucket L
    const uint32_t *keys;                   // the gathered distinct keys
    uint32_t D;                             // distinct keys of this rank
    const uint32_t *counts;                 // [D] occurrences of each
    const uint32_t *prefix;                 // [D] inclusive prefix of the counts
    uint32_t rank, nparts, rec_words, nsamples, nall;
    uint32_t *samples;                      // [nsamples][rec_words] this rank's sample records
    const uint32_t *all_samples;            // [nall][rec_words] every rank's (all-gathered)
    uint32_t *order;                        // [nall] samples in (length, word, index) order
    uint32_t *splitters;                    // [nparts - 1][rec_words - 2]: L, key words
    uint8_t *dest;                          // [D] destination rank of each distinct key
    uint32_t *send_counts;                  // [nparts] records to each rank (zeroed)
    const uint32_t *matrix;                 // [nparts][nparts] every rank's send_counts (all-gathered)
    uint32_t *cursor;                       // [nparts]
    uint32_t *recv_n;                       // [1] records this rank receives
    uint32_t *const *peer_win;              // [nparts] every rank's receive window (device pointers)
    uint32_t *win;                          // this rank's receive window
    uint64_t win_cap;                       // records a window holds
    uint32_t *flag;                         // set on a window overflow (never expected)
    unsigned long long *lwords;             // [256] received words per length (zeroed)
};
cudaError_t launch_xchg_sample(const XchgArgs &a, cudaStream_t s);
cudaError_t launch_xchg_split(const XchgArgs &a, cudaStream_t s);
cudaError_t launch_xchg_count(const XchgArgs &a, cudaStream_t s);
cudaError_t launch_xchg_write(const XchgArgs &a, cudaStream_t s);
cudaError_t launch_xchg_absorb(const XchgArgs &a, uint32_t grid, cudaStream_t s);

struct IngestArgs {
    const uint8_t *text;
    uint64_t n;
    uint32_t nsteps, steps_per_cta, grid;   // the K3 geometry (8 KiB steps): same CTA byte ranges
    uint32_t *ghist;                        // [257] histogram of lengths >= 6 and of > 255 (zeroed by the host)
    uint32_t *dense;                        // [dense_entries()] counts (zeroed by the host)
    uint8_t *touched;                       // [dense_scan_blocks()] 1: a word was counted in this block
    uint32_t *pool;                         // [grid * cta_chunks + 1][kChunkWords]; the last is a trash chunk
    uint32_t *chunk_cls, *chunk_fill;       // [grid * cta_chunks] class (key width) | seq << 8, keys of each chunk
    uint32_t *cls_list;                     // [kMaxStageKw][cls_cap] the chunks of each class (ctr[kIgClsCnt + K - 1] each)
    uint32_t cls_cap;
                                            // (fills zeroed by the host: unused chunks stay empty)
    uint32_t cta_chunks;                    // chunks of one CTA's region
    uint32_t *ctr;                          // [kIgCtrs] (zeroed by the host)
    uint32_t debug;                         // timing experiments only (WSORT_INGEST_DEBUG; outputs wrong):
                                            // 1 = skip the L <= 2 counting, 2 = skip key packing, 8 = skip
                                            // the long words, 16 = skip the L = 3..5 cache, 32 = skip the
                                            // end-of-CTA flush, 64 = skip the L <= 5 length counts
    uint32_t hash;                          // 1: count the long words into `tab` instead of staging them
    HashTab tab;
    uint32_t cta_first;                     // this launch's first CTA (streamed ingest launches K1 by CTA ranges)
};
size_t ingest_smem(uint32_t cta_chunks);
uint32_t ingest_ctas_per_sm();   // resident K1 CTAs per SM (the tokenizer grid is one wave of them)
uint32_t dense_entries();
uint32_t dense_table_base(uint32_t L);
cudaError_t launch_ingest(const IngestArgs &a, cudaStream_t s);   // CTAs [a.cta_first, a.cta_first + count)
cudaError_t launch_ingest_range(IngestArgs a, uint32_t first, uint32_t count, cudaStream_t s);

// words per k_emit_dense tile of dense bucket L: L <= 2 has <= 676 entries in all, longer buckets <= one
// entry per word (the tile's entries must fit its shared memory, kDenseTileEnt)
__host__ __device__ constexpr uint32_t dense_tile_words(uint32_t L) { return L <= 2 ? 32768u : 2048u; }
struct DenseArgs {
    const uint32_t *dense;
    uint32_t n_entries;
    uint32_t *blk_sum, *blk_nnz;            // [dense_scan_blocks()]
    uint32_t *ent_idx, *ent_end;            // compacted non-zero entries: table index, inclusive word end
    uint32_t *n_ent;                        // [2]: entries, words
    const uint8_t *touched;                 // [dense_scan_blocks()] blocks with a non-zero entry (others skipped)
    const BucketInfo *buckets;              // (emit tiles) the dense buckets' word ranges
    const uint32_t *tile_pfx;               // [257] first emit tile of each dense bucket
    uint32_t *tile_e0, *tile_e1;            // [emit tiles] entry of the tile's first / last word (nullable)
    uint32_t ntiles;                        // emit tiles
};
uint32_t dense_scan_blocks(uint32_t n_entries);
cudaError_t launch_dense_lensum(const uint32_t *dense, const uint8_t *touched, uint32_t *ghist, cudaStream_t s);   // ghist[1..5] += table sums
cudaError_t launch_dense_clear(uint32_t *dense, uint8_t *touched, cudaStream_t s);   // zero the touched blocks
cudaError_t launch_dense_scan(const DenseArgs &a, cudaStream_t s);

struct DenseEmitArgs {
    const BucketInfo *buckets;
    const uint32_t *tile_pfx;      // [257] first tile of each dense bucket (tile_from_prefix)
    uint32_t ntiles;
    const uint32_t *ent_idx, *ent_end, *n_ent;
    const uint32_t *tile_e0, *tile_e1;   // from k_dense_compact
    uint8_t *words;
};
cudaError_t launch_emit_dense(const DenseEmitArgs &a, cudaStream_t s);

struct L0Args {
    const BucketInfo *buckets;
    const uint32_t *pool, *chunk_cls, *chunk_fill;
    uint32_t *lcursor;                      // [256] keys placed per bucket so far (zeroed by the host)
    uint32_t *dst;                          // buffer A
    uint32_t cta_chunks;                    // chunks per CTA region of the pool
    uint32_t used_chunks;                   // max chunks any CTA used (its first ids)
    uint32_t nctas;                         // K1 CTAs (regions)
};
cudaError_t launch_lscatter(const L0Args &a, uint32_t nctas, cudaStream_t s);

struct RadixArgs {
    const BucketInfo *buckets;
    const TileDesc *tiles;         // tiles of this pass
    uint32_t ntiles;
    uint32_t nzero;                // status slots of the other buffer to clear
    uint32_t pass;
    uint32_t max_tile_keys;        // largest tile (keys) among this launch's buckets
    uint32_t max_tile_words;       // largest tile_keys * kw among this launch's buckets
    const uint32_t *kin;
    uint32_t *kout;
    const uint32_t *pin;           // payload in (nullable)
    uint32_t *pout;
    uint32_t *dh;                  // digit histograms / bases [rows][1024]
    uint32_t *status;              // look-back status of this pass [ntiles][1024]
    uint32_t *status_other;        // the other status buffer (cleared here)
    uint32_t *ticket;              // dynamic tile counter of this pass
};

cudaError_t launch_digit_hist(const RadixArgs &a, cudaStream_t s);
cudaError_t launch_digit_scan(uint32_t *dh, uint32_t rows, cudaStream_t s);
cudaError_t launch_radix_pass(const RadixArgs &a, bool generic, cudaStream_t s);
size_t radix_pass_smem(uint32_t tile_keys, uint32_t tile_words, bool payload, bool generic);
constexpr int kRadixThreads = 256;
constexpr uint32_t kRadixRegMaxKw = 8;   // key widths sorted with keys held in registers
// keys per radix tile: 32 key words per thread (kw = 1: 8192 keys, kw = 2: 4096, ...), >= 1 key/thread
__host__ __device__ constexpr uint32_t radix_tile_keys(uint32_t kw) {
    return kRadixThreads * (kw >= 32 ? 1u : 32u / kw);
}

// ---------------- variant A: odd-even transposition tiles + merge path ----------------
constexpr int kMergeThreads = 256;
// elements per thread of an OETS tile: the largest power of two <= min(8, 32 / S), at least 1
#ifndef WSORT_FIN_E
#define WSORT_FIN_E 8
#endif
constexpr int kFinE = WSORT_FIN_E;   // msd finishing CTA sort: keys per thread for key widths <= 4
__host__ __device__ constexpr uint32_t oets_elems_per_thread(uint32_t S) {
    return S * 8 <= 32 ? 8u : (S * 4 <= 32 ? 4u : (S * 2 <= 32 ? 2u : 1u));
}
struct OetsArgs {
    const BucketInfo *buckets;
    const TileDesc *tiles;
    uint32_t ntiles;
    uint32_t max_tile_words;       // max over buckets of tile_keys * estride
    const uint32_t *keys_in;       // K3 output (key records, kw words)
    const uint32_t *pay_in;        // K3 payload (nullable)
    uint32_t *out;                 // element layout (estride words)
};
struct MergeArgs {
    const BucketInfo *buckets;
    const TileDesc *tiles;
    uint32_t ntiles;
    uint32_t pass;                 // runs of tile_keys << pass are merged pairwise
    uint32_t max_tile_words;
    const uint32_t *in;
    uint32_t *out;
    uint32_t *splits;              // [ntiles] merge-path split of each tile's first output
};
cudaError_t launch_oets_tile_sort(const OetsArgs &a, cudaStream_t s);
cudaError_t launch_merge_pass(const MergeArgs &a, cudaStream_t s);

// ---------------- multi-GPU exchange (sample sort) ----------------
constexpr uint32_t kMaxRanks = 64;
constexpr uint32_t kDistTileKeys = 4096;
struct CopyRange {
    uint64_t from, to;             // u32 words
    uint32_t len, pad_;
};
struct DistArgs {
    const BucketInfo *buckets;
    const uint64_t *off;           // off[0..256] (device)
    const TileDesc *tiles;         // partition tiles (kDistTileKeys keys)
    uint32_t ntiles;
    const uint32_t *keys;          // packed keys (K3 output)
    uint64_t n_words;
    uint32_t rank, nparts, rec_words, nsamples;
    uint32_t *records;             // sample records out [nsamples][rec_words]
    const uint32_t *splitters;     // [nparts-1][rec_words], sorted
    const uint32_t *split_lo;      // [256] #splitters with length < L
    const uint32_t *split_hi;      // [256] #splitters with length <= L
    uint32_t *counts;              // [nparts][256] keys per (dest, L)
    uint32_t *cursor;              // [nparts][256] scatter cursors
    const uint64_t *send_base;     // [nparts][256] u32-word offset of each (dest, L) range
    uint32_t *send;
};
cudaError_t launch_sample(const DistArgs &a, cudaStream_t s);
cudaError_t launch_part_count(const DistArgs &a, cudaStream_t s);
cudaError_t launch_part_scatter(const DistArgs &a, cudaStream_t s);
cudaError_t launch_regroup(const CopyRange *ranges, uint32_t nranges, const uint32_t *recv, uint32_t *keys,
                           cudaStream_t s);

// ---------------- msd_radix: MSD partitioning + CTA-local odd-even transposition finish ----------------
struct MsdSeg {
    uint32_t L, start, n, buf;     // key range [start, start+n) of bucket L; buf bit 0: 1 = in A, 0 = in B
                                   // (segments and jobs alike); buf >> 8: the job's level (sort jobs) = the
                                   // last digit its keys were partitioned by; bit 4: a sub-job of
                                   // fin_partition; bit 5 (kSegWhole): a whole bucket, no digit partitioned
};
constexpr uint32_t kSegWhole = 32u;
struct MsdTile {
    uint32_t seg, off, n, pad_;    // keys [off, off+n) of segment `seg` of this level
};
enum { kQBig = 0, kQTiles = 1, kQTiny = 2, kQSmall = 3, kQCopy = 4, kQFinTicket = 5, kQParts = 6, kQEmit = 7,
       kQSplitTicket = 8, kQEmitTicket = 9, kQCount = 12 };
// Streaming finish, split jobs: a child of more than kBigJobKeys keys is counted by parts of kPartKeys
// keys (one CTA each); each part leaves its distinct keys + counts in a list of <= kPartListMax entries,
// and the part that arrives last merges the lists and finishes the job (sort, emit).
constexpr uint32_t kPartKeys = 32768, kPartListMax = 1024;
// Only jobs of more than kSplitMinKeys keys are split (measured: below that, counting whole jobs in one
// CTA is cheaper — a part cannot stop early when the job has too many distinct keys)
constexpr uint32_t kSplitMinKeys = 4 * kPartKeys;
__host__ __device__ constexpr uint32_t job_parts(uint32_t n) { return n > kSplitMinKeys ? (n + kPartKeys - 1) / kPartKeys : 1u; }
// A merged split job's text is written by pieces of kEmitPieceWords words (k_msd_fin_emit), from its
// run table (distinct keys sorted + run ends) left in its parts' list space.
constexpr uint32_t kEmitPieceWords = 32768;
constexpr uint32_t kEmitSplitMin = kEmitPieceWords;   // (merged jobs are always written by pieces)
constexpr uint32_t kMsdCopyChunk = 65536;   // u32 words per copy job
struct MsdArgs {
    const BucketInfo *buckets;
    uint32_t level, dst_is_a;
    const MsdSeg *segs;            // this level's segments
    const MsdTile *tiles;          // this level's scatter / count tiles
    const uint32_t *src;           // this level's input buffer
    uint32_t *dst;                 // this level's output buffer
    uint32_t *hist;                // [nsegs][1024]
    uint32_t *cursor;              // [nsegs][1024]
    uint32_t *ctr;                 // [kQCount] queue counters
    MsdSeg *q_big;                 // next level's segments
    MsdTile *q_tiles;              // next level's tiles
    MsdSeg *q_tiny, *q_small;      // finishing sort jobs
    CopyRange *q_copy;             // finishing copies A -> B
    uint32_t cap_big, cap_tiles, cap_local, cap_copy;
    const uint32_t *keys_a;        // finishing: buffer A
    uint32_t *keys_b;              // finishing: buffer B (final)
    uint32_t n_tiny;
    uint32_t finish_radix;         // 1: small jobs with kw <= 4 by local LSD radix, else odd-even transposition
    uint32_t stream_fin;           // 1: every child is a finishing job of k_msd_fin, which writes the text
    uint32_t *seg_skip;            // [segments of this level] 1: all keys share the digit (not scattered)
    uint32_t *dbg_jobs;            // (experiments, nullable) per finishing job: n, kw | L << 8, cycles
    uint8_t *words;                // (stream_fin) output text
    uint8_t *pat;                  // (stream_fin) per finishing CTA kFinPatBytes of run patterns that do not
                                   // fit its shared memory (global, L1-resident while the job emits)
    uint32_t small_base;           // k_msd_fin: first job of this launch in q_small
    uint32_t big_base;             // (radix finish) first job of this launch in q_tiny
    // split jobs (streaming): q_tiny holds the big jobs, counted by parts
    uint32_t parts_base;           // k_msd_fin: first part of this launch
    uint32_t cap_parts;
    uint32_t *q_parts;             // [cap_parts] part -> its job (q_tiny index)
    uint32_t *job_pbase;           // [cap_local] big job -> its first part
    uint32_t *job_done;            // [cap_local] parts of the job counted so far
    uint32_t *job_ovf;             // [cap_local] 1: a part overflowed its table (the job re-enters the MSD)
    uint32_t *part_n;              // [cap_parts] entries in the part's list
    uint4 *part_list;              // [cap_parts][kPartListMax] {key lo, key hi | fingerprint, count, key index}
    uint32_t emit_base, cap_emit;  // k_msd_fin_emit: first piece of this launch; capacity of q_emit
    uint2 *q_emit;                 // [cap_emit] text pieces of merged split jobs: {job (q_tiny index), piece}
    // chunk mode (level 0 of AUTO): the ingest's staging chunks are counted and scattered in place, by
    // slices of slice_chunks chunks of one class K (key width; lengths 6K-5 .. 6K, segment L - seg_l0);
    // slices [slice_pfx[K-1], slice_pfx[K]) are class K's
    uint32_t chunk_mode, seg_l0, slice_chunks, nslices, cls_cap;
    uint32_t slice_pfx[kMaxStageKw + 1];
    uint32_t cls_pfx[kMaxStageKw + 1];   // chunks of classes < K: the classes' lists concatenated (scatter0)
    const uint32_t *pool, *chunk_fill, *cls_list, *cls_cnt;
    uint32_t *slice_hist;          // [nslices][kC0Bins] (nullable) each slice's bins, for k_msd_scatter0's ranges
    MsdSeg *sub_stack;             // (nullable) [cap_sub] sub-jobs of the jobs a finishing CTA partitioned
    uint32_t *sub_n;               // [1] sub-jobs queued (reset after the sub_mode launch)
    uint32_t cap_sub, sub_mode;    // sub_mode: this k_msd_fin launch runs the queued sub-jobs
    uint32_t plan_mode;            // k_msd_plan: 0 = cursors + jobs, 1 = cursors only, 2 = jobs only
};
size_t msd_scatter_smem();
constexpr uint32_t kFinPatBytes = 1024 * 48;   // >= max distinct keys x pattern width (1024 x 32, 512 x 88)
cudaError_t launch_msd_count(const MsdArgs &a, uint32_t ntiles, cudaStream_t s);
cudaError_t launch_msd_plan(const MsdArgs &a, uint32_t nsegs, cudaStream_t s, uint32_t mode = 0);
cudaError_t launch_msd_count0(const MsdArgs &a, cudaStream_t s);
cudaError_t launch_msd_fin_sub(const MsdArgs &a, uint32_t grid, cudaStream_t s);   // k_msd_fin over the sub-job queue     // chunk mode, level 0: a.nslices CTAs
cudaError_t launch_msd_scatter0(const MsdArgs &a, cudaStream_t s);
cudaError_t launch_msd_scatter(const MsdArgs &a, uint32_t ntiles, cudaStream_t s);
cudaError_t launch_msd_finish(const MsdArgs &a, uint32_t n_small, uint32_t n_copy, uint32_t max_tile_words,
                              cudaStream_t s);   // tiny jobs, radix-finish jobs, copies (after the last level)
// per level: jobs [first, *ctr[kQSmall]) by `grid` persistent CTAs
cudaError_t launch_msd_fin_jobs(const MsdArgs &a, uint32_t first, uint32_t first_part, uint32_t grid, cudaStream_t s);
cudaError_t launch_msd_fin_emit(const MsdArgs &a, uint32_t first_piece, uint32_t grid, cudaStream_t s);
cudaError_t launch_msd_fin_split(const MsdArgs &a, uint32_t first_part, uint32_t grid, cudaStream_t s);

struct EmitArgs {
    const BucketInfo *buckets;
    const TileDesc *tiles;         // tile list, or (if tile_pfx) none: tiles enumerated bucket by bucket
    const uint32_t *tile_pfx;      // [257] first tile of each bucket (nullable)
    uint32_t ntiles;
    const uint32_t *keys_a;
    const uint32_t *keys_b;
    const uint32_t *pay_a;         // nullable
    const uint32_t *pay_b;
    uint8_t *words;
    uint64_t *src_off;             // nullable
    uint64_t global_base;
};
constexpr int kEmitStage = 16384;  // smem bytes of output staged per emit tile
cudaError_t launch_emit(const EmitArgs &a, cudaStream_t s);
// small (KB) host<->device copy by a kernel through UVA-mapped pinned host memory (no copy engine)
cudaError_t copy_small(void *dst, const void *src, size_t bytes, cudaStream_t s);
// up to kCopyBatch small host tables (pinned) -> device in one kernel launch
constexpr uint32_t kCopyBatch = 16;
struct CopyBatch {
    void *dst[kCopyBatch];
    const void *src[kCopyBatch];
    size_t bytes[kCopyBatch];
    uint32_t n;
};
cudaError_t launch_copy_batch(const CopyBatch &b, cudaStream_t s);

}  // namespace wsort
