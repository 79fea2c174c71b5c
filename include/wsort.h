/*
 * wsort.h — C ABI of libwsort, a B200-native (sm_100a) implementation of the hot path of
 * arXiv 1411.5283, "Parallelize Bubble and Merge Sort Algorithms Using MPI".
 *
 * The method (§3 Methodology, Pre-processing) sorts every word of a text in three
 * phases:
 *   1. remove the special characters                       -> wsort_tokenize  (kernel K1)
 *   2. split the words into per-length sub-arrays, sized by
 *      the number of words of each length,
 *      "all shorter words come before longer words"         -> wsort_tokenize  (K2: histogram,
 *                                                              offsets) and wsort_sort (K3: pack+scatter)
 *   3. sort each sub-array "in the alphabetic order"        -> wsort_sort      (K4: radix or
 *                                                              odd-even transposition + merge path; K5 emit)
 * and returns the sorted word list plus the per-length bucket offsets (wsort_fetch).
 *
 * Readings of the paper fixed by this ABI (A1-A15):
 *   A1/A8  a word is a maximal run of bytes in [A-Za-z]; every other byte value separates words;
 *   A2     letters are folded to lower case; output words are lower case;
 *   A3     duplicates are kept;
 *   A4/A5  order = (length ascending, then unsigned byte order of the folded word);
 *   A6     equal words keep source order (observable only through src_off);
 *   A7     a word longer than WSORT_MAX_WORD_LEN letters is an error (WSORT_E_WORD_TOO_LONG);
 *   A12    output = "word\n" per word, plus off[0..Lmax+1] with off[0]=0 and
 *          off[L+1] = off[L] + (#words of length L); empty input -> no words, off = {0,0};
 *   A13    (P>1) a word belongs to the shard that holds its first byte; the caller cuts shards
 *          so that no word straddles a cut.
 *
 * Conventions.
 *   - Every function returns an int32 status: WSORT_OK (0) or a negative WSORT_E_* code.
 *     No C++ exception crosses the ABI. On failure the context keeps a message for
 *     wsort_last_error().
 *   - "host" pointers are ordinary CPU memory (pageable or pinned); "device" pointers are CUDA
 *     device memory of the context's device (e.g. torch tensors' data_ptr()).
 *   - The caller owns every buffer it passes; the library never keeps a caller pointer after a
 *     call returns. The context owns all device scratch (text copy, keys, output).
 *   - One context per host thread at a time; distinct contexts are independent.
 *   - All GPU work is enqueued on the context's stream (wsort_create / wsort_set_stream).
 */
#ifndef WSORT_H
#define WSORT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
#define WSORT_OK 0
#define WSORT_E_INVALID_ARG (-1)       /* NULL where a pointer is required, bad enum, ... */
#define WSORT_E_STATE (-2)             /* call out of order (see the state machine below) */
#define WSORT_E_NOMEM (-3)             /* device or pinned-host allocation failed */
#define WSORT_E_CUDA (-4)              /* a CUDA runtime error; message in wsort_last_error */
#define WSORT_E_NCCL (-5)              /* an NCCL failure, or (multi-GPU) another rank failed */
#define WSORT_E_TOO_LARGE (-6)         /* a shard of more than WSORT_MAX_SHARD_BYTES bytes */
#define WSORT_E_WORD_TOO_LONG (-7)     /* some word has more than WSORT_MAX_WORD_LEN letters (A7) */
#define WSORT_E_BUFFER_TOO_SMALL (-8)  /* wsort_fetch: a cap is short; sizes are still filled in */
#define WSORT_E_NOFILE (-9)            /* wsort_load_file: path does not exist */
#define WSORT_E_IO (-10)               /* wsort_load_file: exists but cannot be read */

#define WSORT_MAX_WORD_LEN 255
#define WSORT_MAX_SHARD_BYTES 0xFFFFFF00ull /* local byte offsets are 32-bit */

/* where the caller's buffers live */
enum wsort_mem { WSORT_MEM_HOST = 0, WSORT_MEM_DEVICE = 1 };

/* in-bucket sort (phase 3) */
enum wsort_algo {
    WSORT_ALGO_AUTO = 0,       /* library picks: DENSE_MSD for keys-only sorts of a tokenized text with every
                                  word <= 66 letters, else MSD_OETS (keys only, L <= 48), else LSD radix
                                  (measured) */
    WSORT_ALGO_OETS_MERGE = 1, /* odd-even transposition tiles (the data-parallel bubble sort,
                                  PAPER.md:23) + merge-path merging (the paper's merge) */
    WSORT_ALGO_LSD_RADIX = 2,  /* segmented LSD radix over 2-letter (10-bit) digits (stable; src_off) */
    WSORT_ALGO_MSD_RADIX = 3,  /* MSD radix partitioning by 2-letter digits; small sub-buckets finished by
                                  a CTA-local LSD radix in shared memory (keys only, L <= 48; else LSD) */
    WSORT_ALGO_MSD_OETS = 4,   /* as MSD_RADIX, but the small sub-buckets are finished by CTA-local
                                  odd-even transposition (data-parallel bubble sort) + merge paths */
    WSORT_ALGO_DENSE_MSD = 5,  /* words of L <= 5 counted in dense tables during wsort_tokenize (the sorted
                                  sub-array is the counting sort of the word's base-26 value); longer words
                                  staged as keys by the same text pass and sorted by MSD_OETS from there.
                                  Keys only; falls back like AUTO when it does not apply */
    WSORT_ALGO_RAGGED = 6      /* the paper's other data structure, "vectors of strings": every
                                  sub-array element is a reference (text offset) to its word, compared through
                                  the text; bitonic tiles + merge-path merges (stable; src_off). Measured
                                  against the fixed-width keys ("array char 3D") of the others */
};

/* wsort_sort flags */
#define WSORT_FLAG_SRC_OFF 0x1u /* also produce src_off (needed before wsort_fetch asks for it) */

typedef struct wsort_ctx wsort_ctx; /* opaque */

/* Create a context on CUDA device `cuda_device`. `cuda_stream` is a cudaStream_t cast to an
 * integer (e.g. torch.cuda.current_stream().cuda_stream); 0 = the context creates its own
 * non-blocking stream. *out receives the context; on failure *out is NULL. */
int wsort_create(wsort_ctx **out, int cuda_device, uintptr_t cuda_stream);

/* Replace the stream used for subsequent calls (0 = the context's own stream). */
int wsort_set_stream(wsort_ctx *c, uintptr_t cuda_stream);

/* Load a text of n bytes (host or device memory, per `mem`) into context-owned device memory and
 * reset the context to state LOADED. `global_base` is the byte offset of this text inside the
 * whole corpus (0 for a single GPU); it is added to src_off. n may be 0.
 * Errors: INVALID_ARG (bytes NULL with n>0, bad mem), TOO_LARGE (n > WSORT_MAX_SHARD_BYTES),
 * NOMEM, CUDA. The copy is enqueued on the stream; the call returns after it has been enqueued
 * (host source memory must stay valid until the next synchronising call, e.g. wsort_tokenize). */
int wsort_load_text(wsort_ctx *c, const void *bytes, uint64_t n, int mem, uint64_t global_base);

/* wsort_load_text + wsort_tokenize for a text in HOST memory (pinned for the overlap), with the copy
 * streamed: the text is copied to the device in stages on a second stream and K1 runs on each stage as soon
 * as it has arrived, so the host->device copy overlaps phase 1 (SURVEY.md §8(f) NEXT-4 streaming ingest).
 * Same state, results and errors as the two calls. Not while attached to a communicator (STATE). */
int wsort_ingest_host(wsort_ctx *c, const void *bytes, uint64_t n, uint64_t global_base, uint64_t *n_words);

/* Helper: read a whole file and wsort_load_text it (global_base 0). NOFILE if it does not exist,
 * IO if it cannot be read. */
int wsort_load_file(wsort_ctx *c, const char *path);

/* Phases 1-2: tokenize the loaded text on the GPU (kernel K1), build the length
 * histogram and the bucket offsets (K2). Synchronises the stream once (the sizes are needed on
 * the host to plan phase 3) and stores the number of words in *n_words (may be NULL).
 * State: LOADED -> TOKENIZED. Errors: STATE, WORD_TOO_LONG (state stays LOADED), CUDA. */
int wsort_tokenize(wsort_ctx *c, uint64_t *n_words);

/* Phase 3: pack each word into a fixed-width key and scatter it into its length's
 * sub-array (K3), sort every sub-array alphabetically (K4, algorithm `algo`), and decode the
 * keys into the output text (K5). Asynchronous: returns once the work is enqueued.
 * flags: WSORT_FLAG_SRC_OFF to also compute src_off. State: TOKENIZED|SORTED -> SORTED.
 * Errors: STATE, INVALID_ARG (algo), NOMEM, CUDA. */
int wsort_sort(wsort_ctx *c, int algo, unsigned flags);

typedef struct {
    int mem;               /* where the buffers below live: WSORT_MEM_HOST or WSORT_MEM_DEVICE */
    uint8_t *words;        /* out: "w\n" per word, length-major then alphabetical; NULL = skip */
    uint64_t words_cap;    /* in: capacity of words in bytes */
    uint64_t words_len;    /* out: bytes of output = C + W (letters + newlines) */
    uint64_t *bucket_off;  /* out: off[0..max_len+1] (u64); NULL = skip */
    uint32_t bucket_cap;   /* in: capacity of bucket_off in entries (needs max_len + 2) */
    uint32_t max_len;      /* out: longest word (0 if none) */
    uint64_t *src_off;     /* out (optional, needs WSORT_FLAG_SRC_OFF): global byte offset of each
                              word's first letter, in output order (ties in source order, A6) */
    uint64_t src_cap;      /* in: capacity of src_off in entries */
    uint64_t n_words;      /* out: number of words W */
    uint64_t word_base;    /* out: global index of this context's first word (0 for one GPU) */
    uint64_t byte_base;    /* out: global byte position of this context's output (0 for one GPU) */
} wsort_result;

/* Copy results into the caller's buffers (synchronises the stream). Sizes (words_len, max_len,
 * n_words) are always filled in. After wsort_tokenize only bucket_off/max_len/n_words are
 * available (words/src_off must be NULL, else STATE). A cap that is too small returns
 * BUFFER_TOO_SMALL (sizes filled, nothing copied). src_off without WSORT_FLAG_SRC_OFF -> STATE. */
int wsort_fetch(wsort_ctx *c, wsort_result *r);

/* As wsort_fetch, but the copies of words/src_off are only enqueued on the context's stream: the
 * caller's buffers hold the results once wsort_sync(c) returns (or the stream has been synchronised);
 * they must stay valid until then. Sizes and bucket_off are filled in before it returns. Lets a caller
 * overlap one text's device->host copy with the next text's host->device copy and sort (e.g. two
 * contexts in a pipeline). Errors as wsort_fetch. */
int wsort_fetch_async(wsort_ctx *c, wsort_result *r);

/* Wait until all work enqueued by this context has completed. Errors: CUDA. */
int wsort_sync(wsort_ctx *c);

/* Device pointers of the context-owned results (valid until the next load/sort/destroy), for
 * zero-copy consumers. Any out pointer may be NULL. State: SORTED (words, src_off) or
 * TOKENIZED (bucket_off only). */
int wsort_device_results(wsort_ctx *c, const uint8_t **words, const uint64_t **bucket_off,
                         const uint64_t **src_off);

/* Last error message of this context (NUL-terminated, truncated to cap). */
int wsort_last_error(const wsort_ctx *c, char *msg, size_t cap);

/* Static description of a status code. */
const char *wsort_strerror(int status);

/* Release all device and host resources of the context (NULL is a no-op). */
void wsort_destroy(wsort_ctx *c);

/* ---- measurement (bench.py roofline accounting) ---- */
typedef struct {
    char name[32];          /* kernel class, e.g. "k1_tokenize_count" */
    uint64_t launches;      /* launches since the last reset */
    double total_ms;        /* sum of CUDA-event durations of those launches */
    double bytes;           /* sum of ALGORITHMIC bytes (DESIGN.md per-kernel model) */
} wsort_kernel_stat;

/* on != 0: bracket every kernel launch with CUDA events on the stream it is launched on. on == 2 also runs
 * every kernel on the context's stream (no concurrent side streams), so each kernel's events measure it
 * alone and the per-kernel times add up to the serialised step (the bench's kernel table). */
int wsort_set_profiling(wsort_ctx *c, int on);
/* Synchronises; fills up to cap entries and *n with the number of kernel classes seen. */
int wsort_kernel_stats(wsort_ctx *c, wsort_kernel_stat *out, int cap, int *n);
int wsort_reset_kernel_stats(wsort_ctx *c);
/* How wsort_tokenize (K1) treats the words of >= 6 letters (PAPER.md:58 phases 2-3 start there):
 *   STAGE  their fixed-width keys are staged in chunks (the paper's "array char 3D") and AUTO
 *          sorts them by MSD radix with an exact multiset finish (k_msd.cu); words of > 66 letters are not
 *          staged (the sort then packs every word from the text again, K3, and uses LSD radix);
 *   COUNT  every distinct word is counted into a table (k_hash.cuh) and AUTO sorts only the distinct words,
 *          writing each as often as it occurred (k_hash.cu); any length up to 255;
 *   AUTO   (default) STAGE, or COUNT for a text with a word of > 66 letters.
 * Multi-GPU (attached) always counts: the exchange sends (word, count) records. The output never depends
 * on the mode. */
enum wsort_ingest { WSORT_INGEST_AUTO = 0, WSORT_INGEST_STAGE = 1, WSORT_INGEST_COUNT = 2 };
int wsort_set_ingest(wsort_ctx *c, int mode);

/* How the last wsort_tokenize counted the words of >= 6 letters (diagnostics): */
typedef struct {
    int32_t mode;              /* 1: counted into the table of distinct words (k_hash.cuh); 0: staged as keys */
    uint32_t overflow;         /* nonzero: the table overflowed (reason code) and the text was staged instead */
    uint64_t distinct_narrow;  /* distinct words of 6..12 letters seen by the table */
    uint64_t distinct_wide;    /* distinct words of 13..66 letters seen by the table */
    uint64_t narrow_slots, wide_slots;
    uint32_t grow;             /* table size factor the context has reached (x4 per overflow) */
    uint32_t reserved;
} wsort_ingest_info;
int wsort_get_ingest_info(const wsort_ctx *c, wsort_ingest_info *out);

/* Number of kernel launches enqueued by this context since creation. */
uint64_t wsort_launch_count(const wsort_ctx *c);


/* ---- multi-GPU stages (keys only, no src_off) ----
 * One context per rank. The text shard of rank r is [cut_r, cut_{r+1}) with cuts moved forward
 * while both neighbouring bytes are letters (reading A13). Per step:
 *   wsort_load_text(shard, global_base = cut_r); wsort_tokenize; wsort_histogram -> all-reduce;
 *   wsort_pack (K3 only); wsort_sample -> all-gather; wsort_select_splitters (host, identical on
 *   every rank); wsort_partition -> all-to-all of counts and of the send buffer (NCCL, outside the
 *   library); wsort_load_keys(received); wsort_sort; wsort_set_global(global histogram, word_base,
 *   byte_base); wsort_fetch returns this rank's slice of the global output.
 * Global order = (length, key, source rank): the concatenation of the ranks' outputs in rank
 * order equals the one-GPU output.
 *
 * Split variant (the default when every word has <= 66 letters; SURVEY.md §8(f) NEXT-1 with P > 1):
 * the words of <= 5 letters never travel. wsort_pack_long (instead of wsort_pack) packs only the
 * words of >= 6 letters and hands out the context's dense count table; the caller sums the tables of
 * all ranks in place (all-reduce, NCCL) while the long keys go through sample / partition / all-to-all
 * / wsort_load_keys as above; wsort_dense_range then tells each rank which global dense words it emits
 * (rank r: [r*Wd/P, (r+1)*Wd/P), Wd = the words of <= 5 letters), and wsort_sort writes that dense
 * slice followed by the sorted received keys. The global output is then: the ranks' dense slices in
 * rank order, then their key slices in rank order. */

/* Local length histogram hist[0..255] (state >= TOKENIZED). */
int wsort_histogram(wsort_ctx *c, uint64_t *hist);

/* K3 only: pack and scatter the tokenized words into per-length buckets (state TOKENIZED -> PACKED). */
int wsort_pack(wsort_ctx *c);

/* Regular sample of the packed keys: nsamples records of rec_words u32 (device memory, caller
 * owned): [length, rank, key words..., 0 padding]. rec_words >= 2 + ceil(Lmax_global / 6). */
int wsort_sample(wsort_ctx *c, uint32_t nsamples, uint32_t rank, uint32_t rec_words, uint32_t *dev_records);

/* Host only (no context): sort the all-gathered samples by (length, key, rank) and write the
 * nparts-1 splitters (records at quantiles d*n/nparts) into host memory. Deterministic. */
int wsort_select_splitters(const uint32_t *samples, uint64_t nsamples, uint32_t rec_words, uint32_t nparts,
                           uint32_t *splitters);

/* Partition the packed keys by the (host) splitters into dev_send (caller-owned device buffer of at
 * least the local key words), laid out [dest][length][keys]. counts[dest*256 + L] (host, keys) and
 * send_words[dest] (u32 words per destination) are filled. Synchronises once (the counts). */
int wsort_partition(wsort_ctx *c, const uint32_t *splitters, uint32_t nparts, uint32_t rec_words, uint32_t rank,
                    uint32_t *dev_send, uint64_t send_cap_words, uint64_t *counts, uint64_t *send_words);

/* Adopt received keys: dev_recv holds, for src = 0..nparts-1, the ranges [length][keys] whose key
 * counts are counts[src*256 + L] (host). State -> PACKED; wsort_sort then sorts and emits them. */
int wsort_load_keys(wsort_ctx *c, const uint32_t *dev_recv, const uint64_t *counts, uint32_t nparts);

/* Split variant, instead of wsort_pack (state TOKENIZED -> PACKED; keys only). Moves the staged keys of
 * the words of >= 6 letters (K3c) into the packed layout wsort_sample / wsort_partition read; from here
 * on the local histogram and the packed summary count only those words. *dense_table receives the
 * context's device table of dense counts of the words of <= 5 letters (u32[*dense_entries]: entry
 * (26^L - 26)/25 + sum_j c_j 26^(L-1-j) counts the word c_0..c_{L-1}, c_j = letter - 'a'; owned by the
 * context, valid until the next wsort_load_text): the caller may add the other ranks' tables into it
 * (device memory, stream-ordered after this call) before wsort_sort. STATE if a word of > 66 letters
 * was not staged (use wsort_pack). */
int wsort_pack_long(wsort_ctx *c, uint32_t **dense_table, uint64_t *dense_entries);

/* Split variant, after wsort_load_keys: this context's wsort_sort emits the global dense words
 * [lo, hi) (indices into the words of <= 5 letters in their global order, from the summed tables and
 * the global histogram ghist[256], host) in front of the sorted received keys; wsort_fetch then returns
 * n_words = (hi - lo) + received keys and words = dense slice, then key slice. INVALID_ARG if
 * hi > sum ghist[1..5] or lo > hi; STATE if the context did not run wsort_pack_long + wsort_load_keys. */
int wsort_dense_range(wsort_ctx *c, const uint64_t *ghist, uint64_t lo, uint64_t hi);

/* Make wsort_fetch report the GLOBAL bucket offsets (from the all-reduced histogram ghist[256]) and
 * this rank's word_base / byte_base. */
int wsort_set_global(wsort_ctx *c, const uint64_t *ghist, uint64_t word_base, uint64_t byte_base);

/* ---- multi-GPU: the context as one rank of P, the library owning the communicator ----
 * SURVEY.md §8(b), §8(e); the paper's MPI master/slave exchange (§4) replaced by a symmetric
 * one. Attach once (collective), then per text: wsort_load_text(this rank's shard, global_base = its byte
 * offset; reading A13: the caller cuts the text where no word straddles a cut) -> wsort_tokenize ->
 * wsort_sort -> wsort_fetch / wsort_get_slices. While attached, wsort_tokenize and wsort_sort are
 * COLLECTIVE: every rank calls them, and every rank returns the same status (an error flag is all-reduced
 * before any exchange: a word of > 255 letters on any rank makes every rank return WSORT_E_WORD_TOO_LONG;
 * a failure on another rank returns WSORT_E_NCCL). wsort_sort takes WSORT_ALGO_AUTO only, keys only.
 *   wsort_tokenize: K1 (counting ingest) on the shard; all-reduce of the length histogram, the distinct-word
 *     counts and the error flags; *n_words = the GLOBAL number of words.
 *   wsort_sort: the dense tables (words of <= 5 letters) summed over the ranks (all-reduce) and this rank
 *     emits an equal share of the global dense words; the distinct long words of every rank, with their
 *     counts, go to the rank owning their (length, word) range (sample splitters, weighted by count;
 *     records stored straight into the owner's receive window over NVLink, offsets from a device-side scan
 *     of the all-gathered counts), where equal words add their counts; each rank then sorts and writes its
 *     range. This rank's output = its dense slice, then its long slice; wsort_fetch returns it with the
 *     GLOBAL bucket offsets, word_base / byte_base of the first slice; wsort_get_slices gives both places.
 * The concatenation of all ranks' dense slices in rank order, then their long slices in rank order, is
 * the one-GPU output (tests/test_gpu_dist.py). */
#define WSORT_UNIQUE_ID_BYTES 128

/* NCCL unique id for wsort_attach_comm (rank 0 calls it; the caller broadcasts the bytes, e.g. with
 * torch.distributed). NCCL (libnccl.so.2) is loaded at run time. Errors: NCCL. */
int wsort_get_unique_id(uint8_t id[WSORT_UNIQUE_ID_BYTES]);

/* Make the context rank `rank` of `nranks` (one process per GPU): ncclCommInitRank on the context's device
 * (collective; blocks until every rank has called it). Errors: INVALID_ARG, NCCL, NOMEM. */
int wsort_attach_comm(wsort_ctx *c, int rank, int nranks, const uint8_t id[WSORT_UNIQUE_ID_BYTES]);

/* In-process ranks: a group of nranks contexts driven by nranks threads of one process (any device each;
 * the tests put every rank on one GPU: the collectives are host barriers + device copies, so no kernel
 * waits on another rank's). wsort_attach_group is collective over the group's threads. */
typedef struct wsort_group wsort_group;
int wsort_group_create(wsort_group **out, int nranks);
void wsort_group_destroy(wsort_group *g);   /* after every member detached */
int wsort_attach_group(wsort_ctx *c, wsort_group *g, int rank);

/* Back to a single-GPU context (not collective). */
int wsort_detach_comm(wsort_ctx *c);

/* This rank's pieces of the global output after a multi-GPU wsort_sort (single GPU: one slice). */
typedef struct {
    uint64_t local_byte;   /* where the slice starts in this context's words (wsort_fetch) */
    uint64_t bytes, words;
    uint64_t global_byte;  /* its place in the global output */
    uint64_t global_word;
} wsort_slice;
int wsort_get_slices(const wsort_ctx *c, wsort_slice *out, int cap, int *n);

#ifdef __cplusplus
}
#endif
#endif /* WSORT_H */
