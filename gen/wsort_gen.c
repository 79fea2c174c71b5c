/*
 * wsort_gen.c — seeded synthetic text generator (INPUT GENERATOR ONLY).
 *
 * Stands in for the paper's two missing English text files (§3
 * Methodology: 190 KB and 1.38 MB of Hamlet) and scales beyond them, following
 * the recipe in DESIGN.md §"Input recipe". It holds NONE of
 * the method's arithmetic (no tokenising, bucketing or sorting): it only emits
 * bytes. Both the oracle (oracle/) and the CUDA path consume its output; neither
 * shares code with the other or with this file beyond the bytes.
 *
 * Determinism: the vocabulary stream is seeded with `seed`; the token stream of
 * 1 MiB block b is seeded with SplitMix64(seed ^ (b+1)*0x9E3779B97F4A7C15), so
 * the output is independent of the thread count.
 *
 * Build: gcc -O2 -shared -fPIC -pthread -o libwsortgen.so wsort_gen.c -lm
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GEN_BLOCK (1u << 20)
#define GEN_MAXL 64

typedef struct {
    uint64_t s[4];
} xrng;

static uint64_t splitmix64(uint64_t *x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static void xrng_seed(xrng *r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; i++) r->s[i] = splitmix64(&x);
}

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static inline uint64_t xrng_next(xrng *r) {
    uint64_t *s = r->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

/* uniform double in [0,1) */
static inline double xrng_unif(xrng *r) { return (double)(xrng_next(r) >> 11) * (1.0 / 9007199254740992.0); }

/* English letter frequencies (percent), public statistics; normalised at use. */
static const double LETTER_FREQ[26] = {
    8.2, 1.5, 2.8, 4.3, 12.7, 2.2, 2.0, 6.1, 7.0, 0.15, 0.8, 4.0, 2.4, /* a..m */
    6.7, 7.5, 1.9, 0.10, 6.0, 6.3, 9.1, 2.8, 1.0, 2.4, 0.15, 2.0, 0.07 /* n..z */
};

static const char PUNCT[] = ",.;:!?'\"()-0123456789";

/* ---------------- vocabulary (one sub-vocabulary = Zipf over its types) ---------------- */
typedef struct {
    uint32_t ntypes;
    double *cdf;        /* cumulative Zipf mass, cdf[ntypes-1] == 1 */
    uint32_t *off;      /* letter offset of type r in `chars` */
    uint8_t *len;       /* length of type r */
    char *chars;
} subvocab;

/* open-addressing string set used only to reject duplicate types */
typedef struct {
    uint64_t *h;
    uint32_t *idx;
    uint64_t cap;
} strset;

static uint64_t str_hash(const char *s, int n) {
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < n; i++) h = (h ^ (uint8_t)s[i]) * 1099511628211ull;
    return h | 1;
}

static int strset_insert(strset *S, const char *chars, const uint32_t *off, const uint8_t *len,
                         const char *s, int n, uint32_t newidx) {
    uint64_t h = str_hash(s, n);
    uint64_t m = S->cap - 1, i = h & m;
    while (S->h[i]) {
        if (S->h[i] == h) {
            uint32_t j = S->idx[i];
            if (len[j] == n && memcmp(chars + off[j], s, n) == 0) return 0; /* duplicate */
        }
        i = (i + 1) & m;
    }
    S->h[i] = h;
    S->idx[i] = newidx;
    return 1;
}

static void draw_letters(xrng *r, const double *lcdf, char *dst, int n) {
    for (int i = 0; i < n; i++) {
        double u = xrng_unif(r);
        int c = 0;
        while (c < 25 && u >= lcdf[c]) c++;
        dst[i] = (char)('a' + c);
    }
}

/* Length assignment modes. */
enum { LEN_GEOM = 0, LEN_FIXED = 1, LEN_PREFIX_FAMILY = 2 };

typedef struct {
    uint32_t V;
    int mode;
    int lmin, lmax;
    int exclude_len;    /* geometric mode: a length never used (0 = none) */
    double p;           /* geometric parameter: P(L) ∝ (1-p)^(L-1) */
    double zipf_s;
    double mix;         /* share of tokens drawn from this sub-vocabulary */
} subvocab_params;

static int build_subvocab(subvocab *v, const subvocab_params *P, xrng *r, const double *lcdf) {
    uint32_t V = P->V;
    v->ntypes = V;
    v->cdf = (double *)malloc(sizeof(double) * V);
    v->off = (uint32_t *)malloc(sizeof(uint32_t) * V);
    v->len = (uint8_t *)malloc(V);
    uint64_t maxchars = (uint64_t)V * (uint64_t)(P->lmax > 12 ? P->lmax : 12);
    v->chars = (char *)malloc(maxchars);
    if (!v->cdf || !v->off || !v->len || !v->chars) return -1;

    double Z = 0;
    for (uint32_t k = 0; k < V; k++) Z += pow((double)(k + 1), -P->zipf_s);
    double acc = 0;
    for (uint32_t k = 0; k < V; k++) {
        acc += pow((double)(k + 1), -P->zipf_s) / Z;
        v->cdf[k] = acc;
    }
    v->cdf[V - 1] = 1.0;

    /* truncated geometric CDF over the allowed lengths */
    double F[GEN_MAXL + 2];
    double cap[GEN_MAXL + 2];
    uint64_t used[GEN_MAXL + 2];
    memset(used, 0, sizeof used);
    {
        double tot = 0;
        for (int L = P->lmin; L <= P->lmax; L++)
            if (L != P->exclude_len) tot += pow(1.0 - P->p, L - 1);
        double a = 0;
        for (int L = 0; L <= GEN_MAXL + 1; L++) F[L] = 0;
        for (int L = P->lmin; L <= P->lmax; L++) {
            if (L != P->exclude_len) a += pow(1.0 - P->p, L - 1) / tot;
            F[L] = a;
        }
        for (int L = 0; L <= GEN_MAXL + 1; L++) cap[L] = (L >= 1 && L <= 13) ? pow(26.0, L) / 2.0 : 1e30;
    }

    strset S;
    S.cap = 1;
    while (S.cap < (uint64_t)V * 2) S.cap <<= 1;
    S.h = (uint64_t *)calloc(S.cap, sizeof(uint64_t));
    S.idx = (uint32_t *)calloc(S.cap, sizeof(uint32_t));
    if (!S.h || !S.idx) return -1;

    /* prefix family: 16 random 12-letter prefixes */
    char prefixes[16][12];
    if (P->mode == LEN_PREFIX_FAMILY)
        for (int i = 0; i < 16; i++) draw_letters(r, lcdf, prefixes[i], 12);

    uint64_t pos = 0;
    double prev = 0;
    for (uint32_t k = 0; k < V; k++) {
        int L;
        if (P->mode == LEN_FIXED) {
            L = P->lmin;
        } else if (P->mode == LEN_PREFIX_FAMILY) {
            L = P->lmin + (int)(xrng_next(r) % (uint64_t)(P->lmax - P->lmin + 1));
        } else {
            /* Zipf-mass midpoint of rank k → geometric quantile (frequent types are short) */
            double mid = 0.5 * (prev + v->cdf[k]);
            L = P->lmin;
            while (L < P->lmax && (F[L] < mid || L == P->exclude_len)) L++;
            while (L < P->lmax && ((double)used[L] >= cap[L] || L == P->exclude_len)) L++;
        }
        prev = v->cdf[k];
        char *dst = v->chars + pos;
        for (int tries = 0;; tries++) {
            if (P->mode == LEN_PREFIX_FAMILY) {
                memcpy(dst, prefixes[xrng_next(r) & 15], 12);
                draw_letters(r, lcdf, dst + 12, L - 12);
            } else {
                draw_letters(r, lcdf, dst, L);
            }
            if (strset_insert(&S, v->chars, v->off, v->len, dst, L, k)) break;
            if (tries > 1000 && P->mode == LEN_GEOM && L < P->lmax) { L++; tries = 0; }
            if (tries > 64 && P->mode == LEN_PREFIX_FAMILY) {   /* short suffixes run out: redraw L */
                L = P->lmin + (int)(xrng_next(r) % (uint64_t)(P->lmax - P->lmin + 1));
                tries = 0;
            }
            if (tries > 100000) return -2;
        }
        v->off[k] = (uint32_t)pos;
        v->len[k] = (uint8_t)L;
        used[L]++;
        pos += (uint64_t)L;
    }
    free(S.h);
    free(S.idx);
    return 0;
}

static void free_subvocab(subvocab *v) {
    free(v->cdf);
    free(v->off);
    free(v->len);
    free(v->chars);
}

/* ---------------- public parameter block ---------------- */
typedef struct {
    int nsub;                       /* 1..3 sub-vocabularies */
    subvocab_params sub[3];
    double cap_prob;                /* first letter upper-cased */
    double punct_prob;              /* token carries attached punctuation/digits */
    double punct_suffix_prob;       /* ... as a suffix (else prefix) */
    double newline_prob;            /* separator is '\n' (else ' ') */
} wsort_gen_params;

typedef struct {
    const wsort_gen_params *P;
    const subvocab *sv;
    uint8_t *out;
    uint64_t n;
    uint64_t seed;
    uint64_t nblocks;
    uint64_t next_block;   /* shared, guarded by mu */
    pthread_mutex_t mu;
    uint64_t tokens;       /* tokens whose first letter lies in [0, n) */
} gen_job;

static uint64_t gen_block(const gen_job *J, uint64_t b) {
    const wsort_gen_params *P = J->P;
    uint64_t bs = b * (uint64_t)GEN_BLOCK;
    uint64_t lim = J->n - bs < GEN_BLOCK ? J->n - bs : GEN_BLOCK;
    uint8_t *dst = J->out + bs;
    uint64_t x = J->seed ^ ((b + 1) * 0x9E3779B97F4A7C15ull);
    xrng r;
    xrng_seed(&r, splitmix64(&x));
    double mixc[3];
    double a = 0;
    for (int i = 0; i < P->nsub; i++) { a += P->sub[i].mix; mixc[i] = a; }
    mixc[P->nsub - 1] = 1e300;
    uint64_t pos = 0, ntok = 0;
    char tok[GEN_MAXL + 8];
    for (;;) {
        double ua = xrng_unif(&r) * a;
        int s = 0;
        while (s < P->nsub - 1 && ua >= mixc[s]) s++;
        const subvocab *v = &J->sv[s];
        double z = xrng_unif(&r);
        uint32_t lo = 0, hi = v->ntypes - 1;
        while (lo < hi) {
            uint32_t mid = (lo + hi) >> 1;
            if (v->cdf[mid] > z) hi = mid; else lo = mid + 1;
        }
        int L = v->len[lo];
        const char *w = v->chars + v->off[lo];
        int t = 0, first_letter = 0;
        double cu = xrng_unif(&r);
        double pu = xrng_unif(&r);
        double su = xrng_unif(&r);
        double nl = xrng_unif(&r);
        int npunct = 0, suffix = 1;
        if (pu < P->punct_prob) {
            npunct = 1 + (int)(xrng_next(&r) & 1);
            suffix = su < P->punct_suffix_prob;
        }
        if (npunct && !suffix)
            for (int i = 0; i < npunct; i++) tok[t++] = PUNCT[xrng_next(&r) % (sizeof(PUNCT) - 1)];
        first_letter = t;
        memcpy(tok + t, w, L);
        if (cu < P->cap_prob) tok[t] = (char)(tok[t] - 'a' + 'A');
        t += L;
        if (npunct && suffix)
            for (int i = 0; i < npunct; i++) tok[t++] = PUNCT[xrng_next(&r) % (sizeof(PUNCT) - 1)];
        tok[t++] = nl < P->newline_prob ? '\n' : ' ';
        if (pos + (uint64_t)t > GEN_BLOCK) break;  /* whole tokens only */
        if (pos < lim) {
            uint64_t c = (uint64_t)t;
            if (pos + c > lim) c = lim - pos;
            memcpy(dst + pos, tok, c);
            if (pos + (uint64_t)first_letter < lim) ntok++;
        }
        pos += (uint64_t)t;
    }
    for (; pos < lim; pos++) dst[pos] = '\n';
    return ntok;
}

static void *gen_worker(void *arg) {
    gen_job *J = (gen_job *)arg;
    uint64_t local = 0;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        uint64_t b = J->next_block++;
        pthread_mutex_unlock(&J->mu);
        if (b >= J->nblocks) break;
        local += gen_block(J, b);
    }
    pthread_mutex_lock(&J->mu);
    J->tokens += local;
    pthread_mutex_unlock(&J->mu);
    return NULL;
}

/* Generate exactly n bytes into out. Returns 0 and the number of generated
 * tokens whose first letter lies in [0,n) in *ntokens, or <0 on failure. */
int wsort_gen_text(uint8_t *out, uint64_t n, uint64_t seed, const wsort_gen_params *P, int nthreads,
                   uint64_t *ntokens) {
    if (!out && n) return -1;
    if (!P || P->nsub < 1 || P->nsub > 3) return -1;
    double lsum = 0, lcdf[26];
    for (int i = 0; i < 26; i++) lsum += LETTER_FREQ[i];
    double acc = 0;
    for (int i = 0; i < 26; i++) { acc += LETTER_FREQ[i] / lsum; lcdf[i] = acc; }
    lcdf[25] = 1.0;

    xrng vr;
    xrng_seed(&vr, seed);
    subvocab sv[3];
    memset(sv, 0, sizeof sv);
    for (int i = 0; i < P->nsub; i++) {
        int rc = build_subvocab(&sv[i], &P->sub[i], &vr, lcdf);
        if (rc) {
            for (int j = 0; j <= i; j++) free_subvocab(&sv[j]);
            return rc;
        }
    }
    gen_job J;
    memset(&J, 0, sizeof J);
    J.P = P;
    J.sv = sv;
    J.out = out;
    J.n = n;
    J.seed = seed;
    J.nblocks = (n + GEN_BLOCK - 1) / GEN_BLOCK;
    pthread_mutex_init(&J.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > J.nblocks) nthreads = (int)(J.nblocks ? J.nblocks : 1);
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int i = 1; i < nthreads; i++) pthread_create(&th[i], NULL, gen_worker, &J);
    gen_worker(&J);
    for (int i = 1; i < nthreads; i++) pthread_join(th[i], NULL);
    pthread_mutex_destroy(&J.mu);
    for (int i = 0; i < P->nsub; i++) free_subvocab(&sv[i]);
    if (ntokens) *ntokens = J.tokens;
    return 0;
}
