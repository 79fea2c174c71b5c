/*
 * wsort_oracle.c — the CPU ORACLE for wsort.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library. The product path (paper_1411_5283_b200/) never
 * imports, links or calls it, and it shares no code, header, table or constant
 * generator with the CUDA path.
 *
 * It is a plain, slow, obviously-correct restatement of the paper's method
 * (arXiv 1411.5283, PAPER.md):
 *   phase 1  remove the special characters           PAPER.md:58 (§3 Methodology, Pre-processing),
 *                                                     PAPER.md:61 (Table 2 row 1)
 *   phase 2  per-length sub-arrays ("array of list
 *            ... based on the length of characters,
 *            all shorter words come before longer")   PAPER.md:58; sizes from the counts PAPER.md:13
 *   phase 3  sort each sub-array alphabetically       PAPER.md:58, with
 *              - the paper's bubble sort              PAPER.md:23 (§2), PAPER.md:29 (§3.1), cost n(n-1)/2 PAPER.md:50
 *              - merge sort (the paper's "merge")     PAPER.md:76 (§4 "merges all the chunks")
 *              - brute force: qsort of all tokens by (len, bytes, pos) — the library-routine special case
 *   paper-mpi: the §4/§5 master/slave shape on host threads: chunk = n/p
 *              (remainder to the lowest chunks) then a k-way merge with run-index
 *              tie-break. CPU baseline only.
 *
 * Readings (A1-A15): a word is a maximal run of bytes in [A-Za-z] (A1, A8);
 * letters are folded to lower case with c|0x20 (A2); duplicates are kept (A3); order is
 * (length, unsigned bytes) (A4, A5); equal words keep source order (A6); a word longer than 255
 * letters is an error, status -7 (A7); output is "word\n" per word plus off[0..Lmax+1] (A12).
 *
 * Build: gcc -O2 -shared -fPIC -pthread -o liboracle.so wsort_oracle.c
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_LEN 255
#define ORACLE_E_INVALID_ARG (-1)
#define ORACLE_E_NOMEM (-3)
#define ORACLE_E_WORD_TOO_LONG (-7)
#define ORACLE_E_BUFFER_TOO_SMALL (-8)

enum { ORACLE_BUBBLE = 0, ORACLE_MERGE = 1, ORACLE_BRUTE = 2 };

typedef struct {
    uint64_t comparisons;
    uint64_t swaps;
    uint64_t passes;
} oracle_stats;

/* ------------------------------------------------------------------ phase 1 */

/* ASCII letter test written out: 'A'..'Z' or 'a'..'z' (never isalpha: locale-dependent). */
static int is_letter(uint8_t c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z'); }

/* Lower-case fold of a letter (PAPER.md silent; reading A2). */
static uint8_t fold(uint8_t c) { return (c >= 'A' && c <= 'Z') ? (uint8_t)(c - 'A' + 'a') : c; }

/* Tokenize: every maximal run of letters is one word; every other byte is a separator
 * ("removing / ignoring the special characters"; reading A1).
 * Writes the byte offset and length of each word, in text order, if pos/len are non-NULL
 * (capacity cap). Returns the number of words, or ORACLE_E_WORD_TOO_LONG. */
int64_t oracle_tokenize(const uint8_t *text, uint64_t n, uint64_t *pos, uint32_t *len, uint64_t cap) {
    int64_t w = 0;
    uint64_t i = 0;
    while (i < n) {
        if (!is_letter(text[i])) { i++; continue; }
        uint64_t s = i;
        while (i < n && is_letter(text[i])) i++;
        uint64_t L = i - s;
        if (L > ORACLE_MAX_LEN) return ORACLE_E_WORD_TOO_LONG;
        if (pos) {
            if ((uint64_t)w >= cap) return ORACLE_E_BUFFER_TOO_SMALL;
            pos[w] = s;
            len[w] = (uint32_t)L;
        }
        w++;
    }
    return w;
}

/* ------------------------------------------------------------------ phase 2 */

/* Length histogram hist[0..256) and exclusive prefix off[0..257):
 * off[0] = 0, off[L+1] = off[L] + hist[L]  (sub-array sizes from the counts).
 * Returns Lmax (0 if no words) or an error. */
int oracle_histogram(const uint8_t *text, uint64_t n, uint64_t *hist, uint64_t *off) {
    for (int L = 0; L < 256; L++) hist[L] = 0;
    int lmax = 0;
    uint64_t i = 0;
    while (i < n) {
        if (!is_letter(text[i])) { i++; continue; }
        uint64_t s = i;
        while (i < n && is_letter(text[i])) i++;
        uint64_t L = i - s;
        if (L > ORACLE_MAX_LEN) return ORACLE_E_WORD_TOO_LONG;
        hist[L]++;
        if ((int)L > lmax) lmax = (int)L;
    }
    off[0] = 0;
    for (int L = 0; L < 256; L++) off[L + 1] = off[L] + hist[L];
    return lmax;
}

/* ------------------------------------------------------------------ phase 3 */

/* A sub-array element: a word is (pos, len) into the folded text. */
typedef struct {
    const uint8_t *folded;
    uint32_t L;
} bucket_ctx;

/* alphabetic order of two equal-length words (reading A4) */
static int cmp_alpha(const bucket_ctx *b, uint64_t pa, uint64_t pb) {
    return memcmp(b->folded + pa, b->folded + pb, b->L);
}

/* The paper's bubble sort: compare each item with the next, swap if out of
 * order, repeat until a pass makes no swap. Reading A9: the range shrinks by one per pass
 * (the largest element has sunk to the end) and the loop stops after a swap-free pass. A swap
 * happens only on strict '>' so equal words keep source order (stable). */
static void bubble_sort(const bucket_ctx *b, uint64_t *a, uint64_t n, oracle_stats *st) {
    uint64_t end = n;
    int swapped = 1;
    while (swapped && end > 1) {
        swapped = 0;
        for (uint64_t i = 1; i < end; i++) {
            st->comparisons++;
            if (cmp_alpha(b, a[i - 1], a[i]) > 0) {
                uint64_t t = a[i - 1];
                a[i - 1] = a[i];
                a[i] = t;
                st->swaps++;
                swapped = 1;
            }
        }
        st->passes++;
        end--;
    }
}

/* Top-down merge sort; on ties the left element is taken (stable). */
static void merge_rec(const bucket_ctx *b, uint64_t *a, uint64_t *tmp, uint64_t n, oracle_stats *st) {
    if (n < 2) return;
    uint64_t h = n / 2;
    merge_rec(b, a, tmp, h, st);
    merge_rec(b, a + h, tmp, n - h, st);
    uint64_t i = 0, j = h, k = 0;
    while (i < h && j < n) {
        st->comparisons++;
        if (cmp_alpha(b, a[j], a[i]) < 0) tmp[k++] = a[j++];
        else tmp[k++] = a[i++];
    }
    while (i < h) tmp[k++] = a[i++];
    while (j < n) tmp[k++] = a[j++];
    memcpy(a, tmp, n * sizeof(uint64_t));
}

/* qsort comparator for the brute-force path over ALL tokens: (len, bytes, pos). */
static const uint8_t *g_brute_folded;
typedef struct { uint64_t pos; uint32_t len; } tokrec;
static int brute_cmp(const void *x, const void *y) {
    const tokrec *a = (const tokrec *)x, *b = (const tokrec *)y;
    if (a->len != b->len) return a->len < b->len ? -1 : 1;
    int c = memcmp(g_brute_folded + a->pos, g_brute_folded + b->pos, a->len);
    if (c) return c;
    return a->pos < b->pos ? -1 : (a->pos > b->pos ? 1 : 0);
}

/* ------------------------------------------------------------------ pipeline */

typedef struct {
    uint64_t n_words;
    uint64_t words_len;   /* C + W */
    uint32_t max_len;
} oracle_result;

static uint8_t *make_folded(const uint8_t *text, uint64_t n) {
    uint8_t *f = (uint8_t *)malloc(n ? n : 1);
    if (!f) return NULL;
    for (uint64_t i = 0; i < n; i++) f[i] = fold(text[i]);
    return f;
}

/* Phase 2 stable scatter: per-length sub-arrays of token positions, text order within each.
 * Returns a malloc'd array of all positions in length-major order (bucket L at [off[L], off[L+1])). */
static uint64_t *bucket_by_length(const uint64_t *pos, const uint32_t *len, uint64_t W, const uint64_t *off) {
    uint64_t *out = (uint64_t *)malloc((W ? W : 1) * sizeof(uint64_t));
    if (!out) return NULL;
    uint64_t cursor[257];
    for (int L = 0; L < 257; L++) cursor[L] = off[L];
    for (uint64_t k = 0; k < W; k++) out[cursor[len[k]]++] = pos[k];
    return out;
}

static void emit(const uint8_t *folded, const uint64_t *order, const uint64_t *off, int lmax,
                 uint8_t *words, uint64_t *src_off) {
    uint64_t b = 0;
    for (int L = 1; L <= lmax; L++) {
        for (uint64_t i = off[L]; i < off[L + 1]; i++) {
            memcpy(words + b, folded + order[i], (size_t)L);
            b += (uint64_t)L;
            words[b++] = '\n';
            if (src_off) src_off[i] = order[i];
        }
    }
}

/* Full oracle: tokenize → bucket → sort each bucket (method) → emit.
 *   words:   C+W bytes "w\n" per word, length-major then alphabetical      (cap words_cap)
 *   off:     off[0..Lmax+1] (caller provides >= 257 entries)
 *   src_off: optional, byte offset of each word's first letter, stable order (cap W)
 * Pass words=NULL to query sizes only (res is filled). */
int oracle_sort(const uint8_t *text, uint64_t n, int method, uint8_t *words, uint64_t words_cap,
                uint64_t *off, uint64_t *src_off, uint64_t src_cap, oracle_result *res, oracle_stats *st) {
    if (!res || !off || (n && !text)) return ORACLE_E_INVALID_ARG;
    oracle_stats dummy = {0, 0, 0};
    if (!st) st = &dummy;
    memset(st, 0, sizeof *st);
    uint64_t hist[256];
    int lmax = oracle_histogram(text, n, hist, off);
    if (lmax < 0) return lmax;
    uint64_t W = off[256];
    uint64_t C = 0;
    for (int L = 1; L < 256; L++) C += hist[L] * (uint64_t)L;
    res->n_words = W;
    res->words_len = C + W;
    res->max_len = (uint32_t)lmax;
    if (!words) return 0;
    if (words_cap < C + W || (src_off && src_cap < W)) return ORACLE_E_BUFFER_TOO_SMALL;

    uint64_t *pos = (uint64_t *)malloc((W ? W : 1) * sizeof(uint64_t));
    uint32_t *len = (uint32_t *)malloc((W ? W : 1) * sizeof(uint32_t));
    uint8_t *folded = make_folded(text, n);
    if (!pos || !len || !folded) { free(pos); free(len); free(folded); return ORACLE_E_NOMEM; }
    int64_t w = oracle_tokenize(text, n, pos, len, W);
    if (w < 0 || (uint64_t)w != W) { free(pos); free(len); free(folded); return (int)(w < 0 ? w : -1); }

    uint64_t *order = NULL;
    int rc = 0;
    if (method == ORACLE_BRUTE) {
        tokrec *t = (tokrec *)malloc((W ? W : 1) * sizeof(tokrec));
        order = (uint64_t *)malloc((W ? W : 1) * sizeof(uint64_t));
        if (!t || !order) { free(t); rc = ORACLE_E_NOMEM; goto done; }
        for (uint64_t k = 0; k < W; k++) { t[k].pos = pos[k]; t[k].len = len[k]; }
        g_brute_folded = folded;
        qsort(t, W, sizeof(tokrec), brute_cmp);
        for (uint64_t k = 0; k < W; k++) order[k] = t[k].pos;
        free(t);
    } else {
        order = bucket_by_length(pos, len, W, off);
        if (!order) { rc = ORACLE_E_NOMEM; goto done; }
        uint64_t *tmp = method == ORACLE_MERGE ? (uint64_t *)malloc((W ? W : 1) * sizeof(uint64_t)) : NULL;
        if (method == ORACLE_MERGE && !tmp) { rc = ORACLE_E_NOMEM; goto done; }
        for (int L = 1; L <= lmax; L++) {
            bucket_ctx b = {folded, (uint32_t)L};
            uint64_t nL = off[L + 1] - off[L];
            if (method == ORACLE_BUBBLE) bubble_sort(&b, order + off[L], nL, st);
            else merge_rec(&b, order + off[L], tmp, nL, st);
        }
        free(tmp);
    }
    emit(folded, order, off, lmax, words, src_off);
done:
    free(order);
    free(pos);
    free(len);
    free(folded);
    return rc;
}

/* ------------------------------------------------------------------ paper-mpi (CPU baseline) */

/* Chunk plan (chunk size = array size / no. of processors; SPEC.md:124-129:
 * the first n mod p chunks get one extra element). bounds[0..p]. */
void oracle_partition(uint64_t n, uint32_t p, uint64_t *bounds) {
    uint64_t q = n / p, r = n % p, b = 0;
    for (uint32_t i = 0; i < p; i++) {
        bounds[i] = b;
        b += q + (i < r ? 1 : 0);
    }
    bounds[p] = b;
}

typedef struct {
    const bucket_ctx *b;
    uint64_t *a;
    uint64_t *tmp;
    uint64_t n;
    int inner;   /* ORACLE_BUBBLE or ORACLE_MERGE */
    oracle_stats st;
} chunk_job;

static void *chunk_worker(void *arg) {
    chunk_job *j = (chunk_job *)arg;
    memset(&j->st, 0, sizeof j->st);
    if (j->inner == ORACLE_BUBBLE) bubble_sort(j->b, j->a, j->n, &j->st);
    else merge_rec(j->b, j->a, j->tmp, j->n, &j->st);
    return NULL;
}

/* paper-mpi: per length bucket, split into p chunks, sort each chunk on its own thread ("each
 * slave will do a bubble sort on own data"), then the master k-way merges the runs
 * (lowest run index wins ties). Output identical to oracle_sort. bubble_comparisons counts only
 * the workers' sort comparisons. */
int oracle_sort_paper_mpi(const uint8_t *text, uint64_t n, uint32_t p, int inner, uint8_t *words,
                          uint64_t words_cap, uint64_t *off, oracle_result *res, oracle_stats *st) {
    if (p < 1 || p > 1024 || !res || !off) return ORACLE_E_INVALID_ARG;
    oracle_stats dummy;
    if (!st) st = &dummy;
    memset(st, 0, sizeof *st);
    uint64_t hist[256];
    int lmax = oracle_histogram(text, n, hist, off);
    if (lmax < 0) return lmax;
    uint64_t W = off[256], C = 0;
    for (int L = 1; L < 256; L++) C += hist[L] * (uint64_t)L;
    res->n_words = W;
    res->words_len = C + W;
    res->max_len = (uint32_t)lmax;
    if (!words) return 0;
    if (words_cap < C + W) return ORACLE_E_BUFFER_TOO_SMALL;
    uint64_t *pos = (uint64_t *)malloc((W ? W : 1) * 8), *tmp = (uint64_t *)malloc((W ? W : 1) * 8);
    uint64_t *merged = (uint64_t *)malloc((W ? W : 1) * 8);
    uint32_t *len = (uint32_t *)malloc((W ? W : 1) * 4);
    uint8_t *folded = make_folded(text, n);
    chunk_job *jobs = (chunk_job *)calloc(p, sizeof(chunk_job));
    pthread_t *th = (pthread_t *)calloc(p, sizeof(pthread_t));
    uint64_t *bounds = (uint64_t *)calloc(p + 1, 8), *head = (uint64_t *)calloc(p, 8);
    int rc = 0;
    uint64_t *order = NULL;
    if (!pos || !tmp || !merged || !len || !folded || !jobs || !th || !bounds || !head) { rc = ORACLE_E_NOMEM; goto done; }
    oracle_tokenize(text, n, pos, len, W);
    order = bucket_by_length(pos, len, W, off);
    if (!order) { rc = ORACLE_E_NOMEM; goto done; }
    for (int L = 1; L <= lmax; L++) {
        bucket_ctx b = {folded, (uint32_t)L};
        uint64_t base = off[L], nL = off[L + 1] - off[L];
        if (!nL) continue;
        oracle_partition(nL, p, bounds);
        for (uint32_t i = 0; i < p; i++) {   /* master sends chunk i to slave i */
            jobs[i].b = &b;
            jobs[i].a = order + base + bounds[i];
            jobs[i].tmp = tmp + base + bounds[i];
            jobs[i].n = bounds[i + 1] - bounds[i];
            jobs[i].inner = inner;
            if (i) pthread_create(&th[i], NULL, chunk_worker, &jobs[i]);
        }
        chunk_worker(&jobs[0]);
        for (uint32_t i = 1; i < p; i++) pthread_join(th[i], NULL);
        for (uint32_t i = 0; i < p; i++) {   /* slaves return results */
            st->comparisons += jobs[i].st.comparisons;
            st->swaps += jobs[i].st.swaps;
            st->passes += jobs[i].st.passes;
            head[i] = bounds[i];
        }
        /* master k-way merge; scanning runs in index order and taking a strictly smaller head
         * keeps the lowest run index on ties */
        for (uint64_t k = 0; k < nL; k++) {
            int best = -1;
            for (uint32_t i = 0; i < p; i++) {
                if (head[i] >= bounds[i + 1]) continue;
                if (best < 0 || cmp_alpha(&b, order[base + head[i]], order[base + head[best]]) < 0) best = (int)i;
            }
            merged[base + k] = order[base + head[best]++];
        }
        memcpy(order + base, merged + base, nL * 8);
    }
    emit(folded, order, off, lmax, words, NULL);
done:
    free(order); free(pos); free(tmp); free(merged); free(len); free(folded);
    free(jobs); free(th); free(bounds); free(head);
    return rc;
}

/* ------------------------------------------------------------------ some sub-arrays (full-size goldens) */

/* Phases 2-3 for the lengths Lmin..Lmax only: the sub-array of the words of each length L (PAPER.md:58
 * "array of list ... based on the length"; the fixed-width "array char 3D" of PAPER.md:29: word i at
 * bytes [i*L, i*L+L) of a compact folded array), sorted alphabetically in the paper-mpi shape (p chunks,
 * each merge-sorted on its own thread, then the k-way merge), emitted as "word\n"
 * per word, shorter lengths first. Because the output is length-major (reading A5), these outputs for
 * consecutive length ranges concatenate to oracle_sort's output (pinned in tests/test_oracle.py); it
 * lets a test-golden script sort texts whose whole token array does not fit in host memory, a few
 * sub-arrays at a time. words = NULL: *n_words (words of lengths Lmin..Lmax) and *words_len only.
 * Returns 0 or an error (a run of > 255 letters anywhere: WORD_TOO_LONG). */
int oracle_sort_lengths(const uint8_t *text, uint64_t n, uint32_t Lmin, uint32_t Lmax, uint32_t p, uint8_t *words,
                        uint64_t words_cap, uint64_t *n_words, uint64_t *words_len) {
    if (Lmin < 1 || Lmax > ORACLE_MAX_LEN || Lmin > Lmax || p < 1 || p > 1024 || !n_words || !words_len ||
        (n && !text))
        return ORACLE_E_INVALID_ARG;
    uint64_t cnt[ORACLE_MAX_LEN + 2] = {0}, i = 0;
    while (i < n) {   /* phase 1: count the words of each length */
        if (!is_letter(text[i])) { i++; continue; }
        uint64_t s = i;
        while (i < n && is_letter(text[i])) i++;
        if (i - s > ORACLE_MAX_LEN) return ORACLE_E_WORD_TOO_LONG;
        cnt[i - s]++;
    }
    uint64_t nw = 0, nb = 0, sub_bytes = 0, nmax = 0;
    uint64_t sub_off[ORACLE_MAX_LEN + 2] = {0}, fill[ORACLE_MAX_LEN + 2] = {0};
    for (uint32_t L = Lmin; L <= Lmax; L++) {
        sub_off[L] = sub_bytes;
        sub_bytes += cnt[L] * L;
        nw += cnt[L];
        nb += cnt[L] * (L + 1);
        if (cnt[L] > nmax) nmax = cnt[L];
    }
    *n_words = nw;
    *words_len = nb;
    if (!words) return 0;
    if (words_cap < nb) return ORACLE_E_BUFFER_TOO_SMALL;
    uint8_t *sub = (uint8_t *)malloc(sub_bytes ? sub_bytes : 1);
    uint64_t *order = (uint64_t *)malloc((nmax ? nmax : 1) * 8), *tmp = (uint64_t *)malloc((nmax ? nmax : 1) * 8);
    uint64_t *merged = (uint64_t *)malloc((nmax ? nmax : 1) * 8);
    chunk_job *jobs = (chunk_job *)calloc(p, sizeof(chunk_job));
    pthread_t *th = (pthread_t *)calloc(p, sizeof(pthread_t));
    uint64_t *bounds = (uint64_t *)calloc(p + 1, 8), *head = (uint64_t *)calloc(p, 8);
    int rc = 0;
    if (!sub || !order || !tmp || !merged || !jobs || !th || !bounds || !head) { rc = ORACLE_E_NOMEM; goto done; }
    /* phase 2: the folded words of each length L in [Lmin, Lmax], text order */
    i = 0;
    while (i < n) {
        if (!is_letter(text[i])) { i++; continue; }
        uint64_t s = i;
        while (i < n && is_letter(text[i])) i++;
        uint64_t L = i - s;
        if (L < Lmin || L > Lmax) continue;
        uint8_t *dst = sub + sub_off[L] + fill[L]++ * L;
        for (uint64_t j = 0; j < L; j++) dst[j] = fold(text[s + j]);
    }
    /* phase 3 per length: p chunks sorted on p threads, then the k-way merge; emit */
    uint64_t out = 0;
    for (uint32_t L = Lmin; L <= Lmax; L++) {
        const uint64_t nL = cnt[L];
        if (!nL) continue;
        bucket_ctx b = {sub + sub_off[L], L};
        for (uint64_t k = 0; k < nL; k++) order[k] = k * L;
        oracle_partition(nL, p, bounds);
        for (uint32_t q = 0; q < p; q++) {
            jobs[q].b = &b;
            jobs[q].a = order + bounds[q];
            jobs[q].tmp = tmp + bounds[q];
            jobs[q].n = bounds[q + 1] - bounds[q];
            jobs[q].inner = ORACLE_MERGE;
            if (q) pthread_create(&th[q], NULL, chunk_worker, &jobs[q]);
        }
        chunk_worker(&jobs[0]);
        for (uint32_t q = 1; q < p; q++) pthread_join(th[q], NULL);
        for (uint32_t q = 0; q < p; q++) head[q] = bounds[q];
        for (uint64_t m = 0; m < nL; m++) {
            int best = -1;
            for (uint32_t q = 0; q < p; q++) {
                if (head[q] >= bounds[q + 1]) continue;
                if (best < 0 || cmp_alpha(&b, order[head[q]], order[head[best]]) < 0) best = (int)q;
            }
            merged[m] = order[head[best]++];
        }
        for (uint64_t m = 0; m < nL; m++) {
            memcpy(words + out, b.folded + merged[m], L);
            words[out + L] = '\n';
            out += L + 1;
        }
    }
done:
    free(sub); free(order); free(tmp); free(merged); free(jobs); free(th); free(bounds); free(head);
    return rc;
}

/* ------------------------------------------------------------------ fingerprint / verify */

/* Order-independent multiset fingerprint of the tokens of `text` (test helper, not part of
 * the method): fp[0] = Σ h1(word) mod 2^64, fp[1] = Σ h2(word) mod 2^64, where
 * h1 = Σ_j c_j·K1^j and h2 = Σ_j c_j·K2^j over the folded letters c_j (wrapping u64). */
#define FP_K1 0x100000001B3ull
#define FP_K2 0x9E3779B97F4A7C15ull
static void word_hash(const uint8_t *w, uint32_t L, uint64_t *h1, uint64_t *h2) {
    uint64_t a = 0, b = 0, p1 = 1, p2 = 1;
    for (uint32_t j = 0; j < L; j++) {
        a += (uint64_t)w[j] * p1;
        b += (uint64_t)w[j] * p2;
        p1 *= FP_K1;
        p2 *= FP_K2;
    }
    *h1 = a;
    *h2 = b;
}

int oracle_fingerprint(const uint8_t *text, uint64_t n, uint64_t *fp) {
    uint8_t buf[ORACLE_MAX_LEN];
    fp[0] = fp[1] = 0;
    uint64_t i = 0;
    while (i < n) {
        if (!is_letter(text[i])) { i++; continue; }
        uint64_t s = i;
        while (i < n && is_letter(text[i])) i++;
        uint64_t L = i - s;
        if (L > ORACLE_MAX_LEN) return ORACLE_E_WORD_TOO_LONG;
        for (uint64_t j = 0; j < L; j++) buf[j] = fold(text[s + j]);
        uint64_t a, b;
        word_hash(buf, (uint32_t)L, &a, &b);
        fp[0] += a;
        fp[1] += b;
    }
    return 0;
}

/* The same fingerprint over a candidate output "w\n"... buffer. */
int oracle_fingerprint_words(const uint8_t *words, uint64_t len, uint64_t *fp) {
    fp[0] = fp[1] = 0;
    uint64_t s = 0;
    for (uint64_t i = 0; i < len; i++) {
        if (words[i] != '\n') continue;
        uint64_t a, b;
        word_hash(words + s, (uint32_t)(i - s), &a, &b);
        fp[0] += a;
        fp[1] += b;
        s = i + 1;
    }
    return s == len ? 0 : -1;
}

/* verify (SPEC.md:398-411 cmd_verify, restated): the candidate is sorted by (len, bytes), every
 * byte is a-z or '\n', its bucket offsets equal the text's histogram prefix sums, and it is a
 * permutation of the text's token multiset (fingerprint). Returns 0, or 1 + index of the first
 * offending word, or a negative code for a structural failure. */
int64_t oracle_verify(const uint8_t *text, uint64_t n, const uint8_t *words, uint64_t words_len,
                      const uint64_t *off, uint32_t n_off) {
    uint64_t hist[256], ref_off[257];
    int lmax = oracle_histogram(text, n, hist, ref_off);
    if (lmax < 0) return lmax;
    if (n_off != (uint32_t)lmax + 2) return -20;
    for (uint32_t L = 0; L < n_off; L++)
        if (off[L] != ref_off[L]) return -21;
    uint64_t s = 0, k = 0, prev_s = 0, prev_L = 0;
    for (uint64_t i = 0; i < words_len; i++) {
        uint8_t c = words[i];
        if (c == '\n') {
            uint64_t L = i - s;
            if (L == 0) return (int64_t)k + 1;
            if (k < ref_off[L] || k >= ref_off[L + 1]) return (int64_t)k + 1;
            if (k > 0 && (L < prev_L || (L == prev_L && memcmp(words + prev_s, words + s, L) > 0)))
                return (int64_t)k + 1;
            prev_s = s;
            prev_L = L;
            s = i + 1;
            k++;
        } else if (c < 'a' || c > 'z') {
            return (int64_t)k + 1;
        }
    }
    if (s != words_len || k != ref_off[lmax + 1]) return -22;
    uint64_t fa[2], fb[2];
    oracle_fingerprint(text, n, fa);
    oracle_fingerprint_words(words, words_len, fb);
    if (fa[0] != fb[0] || fa[1] != fb[1]) return -23;
    return 0;
}
