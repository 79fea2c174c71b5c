// wsort_api.cu — the libwsort host runtime and C ABI (include/wsort.h).
//
// The context owns every device buffer of the pipeline and enqueues all work on one CUDA stream:
//   wsort_load_text  H2D/D2D copy of the text into a zero-padded device buffer
//   wsort_tokenize   K1 (per-CTA length histograms) + K2 (offsets), one stream sync for the sizes
//   wsort_sort       host planning of buckets and tiles -> one H2D of the plan ->
//                    K3 (pack + scatter) -> K4 (radix: histogram, scan, passes | OETS + merge) -> K5
//   wsort_fetch      copies results into the caller's buffers
// Grow-only allocations: repeated calls on inputs of the same size allocate nothing.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "k_hash.cuh"
#include "wsort.h"
#include "wsort_comm.cuh"
#include "wsort_internal.cuh"

using namespace wsort;

namespace {

enum State { ST_CREATED = 0, ST_LOADED = 1, ST_TOKENIZED = 2, ST_PACKED = 3, ST_SORTED = 4 };

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
};

struct KernelClass {
    std::string name;
    uint64_t launches = 0;
    double ms = 0;
    double bytes = 0;
};

struct PendingEv {
    int cls;
    cudaEvent_t a, b;
    double bytes;
};

}  // namespace

struct wsort_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    cudaStream_t aux = nullptr;                  // second stream: the dense buckets run beside the MSD
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t split = nullptr;                // third stream: parts of split finishing jobs beside k_msd_fin
    cudaStream_t hp = nullptr;                   // high-priority stream: the long words' MSD (the critical path)
    cudaEvent_t ev_hp0 = nullptr, ev_hp1 = nullptr;   // beside the dense branch, which fills the idle SMs
    cudaEvent_t ev_lvl = nullptr, ev_split = nullptr, ev_plan = nullptr;
    int sms = 148;
    State state = ST_CREATED;
    char err[512] = {0};

    // text
    DevBuf text_alloc;
    uint64_t n = 0;
    uint64_t global_base = 0;
    const uint8_t *d_text = nullptr;

    // tokenizer
    TkArgs tk{};
    DevBuf cta_hist, cta_base, d_sum;
    Summary *h_sum = nullptr;   // pinned
    bool cta_bases_ready = false;  // K2b ran for the current tokenize (K3 needs it)
    bool cta_counts_ready = false; // K1b's per-CTA histograms are in cta_hist (K2b needs them)

    // K1 ingest: global histogram, dense counts, staging chunks
    DevBuf ghist, dense, pool, chunk_cls, chunk_fill, ig_ctr, d_touched, cls_list, slice_hist, m_sub, m_subn;
    bool dense_clean = false;                    // the dense table has been zeroed once (then: touched blocks)
    uint32_t *h_ig = nullptr;   // pinned mirror of ig_ctr
    uint32_t cta_chunks = 0, n_chunks = 0;
    DevBuf d_blk_sum, d_blk_nnz, d_ent_idx, d_ent_end, d_n_ent, d_tiles2, d_lcursor, d_tile_e;
    // K1 hash mode: the table of distinct long words (k_hash.cuh) and the run emission after the sort
    bool hashed = false;                         // the last tokenize counted the long words into the table
    int ingest_mode = WSORT_INGEST_AUTO;         // wsort_set_ingest
    uint64_t hash_grow = 1;                      // table size factor (x4 after an overflow, up to 64)
    DevBuf t_wlens, t_nkey, t_ncnt, t_fp, t_meta, t_cnt, t_keys, t_top, t_dcount, t_runend, t_scan, t_tilee, t_kplan, t_dpfx, t_rpfx;
    HashTab tab{};
    uint32_t *h_tab = nullptr;                   // pinned: top[4] + dcount[256]
    wsort_ingest_info ig_info{};                 // what the last tokenize did (wsort_get_ingest_info)

    // sort
    DevBuf keys_a, keys_b, pay_a, pay_b, words, src_off, dh, status0, status1, tickets, plan, va_x, va_y, splits;
    DevBuf m_hist, m_cursor, m_ctr, m_big[2], m_tiles[2], m_tiny, m_small, m_copy, m_skip, m_pat;
    DevBuf m_qparts, m_pbase, m_jdone, m_jovf, m_partn, m_plist, m_qemit;   // split finishing jobs
    uint32_t *h_ctr = nullptr;   // pinned mirror of the msd queue counters
    std::vector<uint8_t> hplan;
    uint8_t *h_plan_pinned = nullptr;
    size_t h_plan_cap = 0;
    // pinned staging arena for the host-built tables of one sort (one region per upload, reused by the
    // next sort once `arena_done` has passed)
    uint8_t *arena = nullptr;
    size_t arena_cap = 0, arena_off = 0;
    struct PendingCopy {
        void *dst;
        const void *src;
        size_t bytes;
    };
    std::vector<PendingCopy> pcopy;   // arena uploads not yet issued (arena_flush)
    cudaGraph_t tk_graph = nullptr;   // the tokenize launch sequence, captured (tokenize_impl)
    cudaGraphExec_t tk_exec = nullptr;
    std::vector<uintptr_t> tk_key;    // what it was captured for (size, mode, buffers)
    uint64_t tk_nlaunch = 0;
    cudaEvent_t arena_done = nullptr;
    bool sorted_with_src = false;
    int last_algo = 0;
    bool packed_pending = false;   // keys_a holds packed, not yet sorted keys (wsort_pack / load_keys)
    bool keys_external = false;    // the keys came from wsort_load_keys (no local text behind them)

    // multi-GPU: global view for wsort_fetch
    bool has_global = false;
    uint64_t goff[kHistBins + 1] = {0};
    uint32_t gmax = 0;
    uint64_t word_base = 0, byte_base = 0;
    // multi-GPU split of the ingest path (wsort_pack_long / wsort_dense_range): the dense table may be
    // summed over the ranks; this context emits the global dense words [dense_lo, dense_hi)
    bool dist_dense = false, dense_range = false;
    // streamed ingest (wsort_ingest_host): the host text copied stage by stage under K1
    const uint8_t *stream_src = nullptr;
    cudaStream_t copy_stream = nullptr;
    std::vector<cudaEvent_t> copy_ev;
    cudaEvent_t ev_ingest = nullptr;
    // multi-GPU with a library-owned communicator (wsort_attach_comm / wsort_attach_group)
    Comm *comm = nullptr;
    uint64_t g_hist[257] = {0};        // global length histogram (all ranks), [256] = words > 255 letters
    uint64_t g_dcount[256] = {0};      // sum over the ranks of the distinct long words per length
    uint32_t g_lmax = 0;
    std::vector<wsort_slice> slices;   // this rank's places in the global output (wsort_get_slices)
    DevBuf x_vec, x_counts, x_prefix, x_samples, x_all, x_order, x_split, x_dest, x_send, x_matrix, x_cursor,
        x_recvn, x_win, x_peers, x_flag, x_lwords, x_lwords_all;
    uint64_t dense_lo = 0, dense_hi = 0;
    uint64_t dslice_off[kDenseMaxLen + 2] = {0};   // global word index of the slice's first word of length L
    uint64_t dslice_n[kDenseMaxLen + 2] = {0};     // its words of length L
    uint64_t slice_words = 0, slice_bytes = 0;     // the dense slice in front of the sorted keys
    DevBuf bk, d_counts, d_cursor, d_sbase, d_split, d_lohi, d_tiles, d_ranges;

    // profiling
    bool prof = false;
    bool prof_serial = false;   // wsort_set_profiling(2): every kernel on the context's stream (exact shares)
    std::vector<KernelClass> classes;
    std::vector<PendingEv> pending;
    std::vector<cudaEvent_t> ev_pool;
    uint64_t launches = 0;
};

namespace {

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}

int set_err(wsort_ctx *c, int code, const char *fmt, ...) {
    if (c) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(c->err, sizeof c->err, fmt, ap);
        va_end(ap);
    }
    return code;
}

int cuda_err(wsort_ctx *c, cudaError_t e, const char *what) {
    return set_err(c, e == cudaErrorMemoryAllocation ? WSORT_E_NOMEM : WSORT_E_CUDA, "%s: %s (%s)", what,
                   cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CK(call, what)                                  \
    do {                                                \
        cudaError_t _e = (call);                        \
        if (_e != cudaSuccess) return cuda_err(c, _e, what); \
    } while (0)

int ensure(wsort_ctx *c, DevBuf &b, size_t bytes, const char *what, bool zero = false) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return WSORT_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    size_t want = bytes + bytes / 16;   // headroom for slightly larger inputs
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(c, WSORT_E_NOMEM, "cudaMalloc(%zu) for %s failed: %s", want, what, cudaGetErrorString(e));
    }
    b.cap = want;
    if (zero) CK(cudaMemsetAsync(b.p, 0, want, c->stream), "memset");
    return WSORT_OK;
}

int upload_small(wsort_ctx *c, DevBuf &dst, const void *src, size_t bytes, const char *what) {
    int rc = ensure(c, dst, bytes, what);   // ensure() allocates at least 16 bytes
    if (rc) return rc;
    if (bytes && src) CK(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyHostToDevice, c->stream), what);
    return WSORT_OK;
}

// Staged uploads: host tables are copied into the pinned arena and sent with one async copy each
// (pageable cudaMemcpyAsync would stage through the driver); regions are not reused within a sort.
int arena_begin(wsort_ctx *c) {
    c->pcopy.clear();
    if (c->arena_done) CK(cudaEventSynchronize(c->arena_done), "arena reuse");
    c->arena_off = 0;
    return WSORT_OK;
}
// The uploads of a sort are batched: one copy kernel launch per batch (arena_flush), issued on the
// context's stream before the next kernel there and before every fork to a side stream.
int arena_flush(wsort_ctx *c) {
    size_t i = 0;
    while (i < c->pcopy.size()) {
        CopyBatch b{};
        for (; i < c->pcopy.size() && b.n < kCopyBatch; i++, b.n++) {
            b.dst[b.n] = c->pcopy[i].dst;
            b.src[b.n] = c->pcopy[i].src;
            b.bytes[b.n] = c->pcopy[i].bytes;
        }
        const cudaError_t e = launch_copy_batch(b, c->stream);
        if (e != cudaSuccess) {
            c->pcopy.clear();
            return cuda_err(c, e, "upload batch");
        }
        c->launches++;
    }
    c->pcopy.clear();
    return WSORT_OK;
}
int arena_upload(wsort_ctx *c, DevBuf &dst, const void *src, size_t bytes, const char *what) {
    int rc = ensure(c, dst, bytes, what);
    if (rc || !bytes) return rc;
    const size_t need = c->arena_off + ((bytes + 255) & ~(size_t)255);
    if (need > c->arena_cap) {   // grow (rare): earlier copies of this sort read the old buffer
        if ((rc = arena_flush(c))) return rc;
        CK(cudaStreamSynchronize(c->stream), "arena grow");
        uint8_t *nb = nullptr;
        const size_t cap = std::max<size_t>(need * 2, 1 << 20);
        if (cudaMallocHost(&nb, cap) != cudaSuccess) {
            cudaGetLastError();
            return set_err(c, WSORT_E_NOMEM, "pinned arena");
        }
        if (c->arena) cudaFreeHost(c->arena);
        c->arena = nb;
        c->arena_cap = cap;
        c->arena_off = 0;
    }
    uint8_t *h = c->arena + c->arena_off;
    memcpy(h, src, bytes);
    c->arena_off += (bytes + 255) & ~(size_t)255;
    c->pcopy.push_back(wsort_ctx::PendingCopy{dst.p, h, bytes});   // (pinned arena, copied by a kernel: no copy-engine queue)
    (void)what;
    return WSORT_OK;
}
int arena_end(wsort_ctx *c) {
    if (int rc = arena_flush(c)) return rc;
    if (!c->arena_done) CK(cudaEventCreateWithFlags(&c->arena_done, cudaEventDisableTiming), "arena event");
    CK(cudaEventRecord(c->arena_done, c->stream), "arena event");
    return WSORT_OK;
}

int class_id(wsort_ctx *c, const char *name) {
    for (size_t i = 0; i < c->classes.size(); i++)
        if (c->classes[i].name == name) return (int)i;
    c->classes.push_back(KernelClass{name});
    return (int)c->classes.size() - 1;
}

cudaEvent_t get_event(wsort_ctx *c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

int arena_flush(wsort_ctx *c);
template <class F>
int launch_on(wsort_ctx *c, cudaStream_t s, const char *name, double bytes, F f) {
    if (s == c->stream && !c->pcopy.empty()) {
        if (int rc = arena_flush(c)) return rc;
    }
    PendingEv pe{};
    if (c->prof) {
        pe.cls = class_id(c, name);
        pe.a = get_event(c);
        pe.b = get_event(c);
        pe.bytes = bytes;
        cudaEventRecord(pe.a, s);
    }
    cudaError_t e = f();
    if (e != cudaSuccess) return cuda_err(c, e, name);
    c->launches++;
    if (c->prof) {
        cudaEventRecord(pe.b, s);
        c->pending.push_back(pe);
    }
    return WSORT_OK;
}
template <class F>
int launch(wsort_ctx *c, const char *name, double bytes, F f) {
    return launch_on(c, c->stream, name, bytes, f);
}

void drain_events(wsort_ctx *c) {
    static const bool timeline = getenv("WSORT_DEBUG_TIMELINE") != nullptr;   // (experiments)
    if (timeline && !c->pending.empty()) {
        cudaEventSynchronize(c->pending.back().b);
        float prev_end = 0;
        for (auto &pe : c->pending) {
            float t0 = 0, t1 = 0;
            cudaEventElapsedTime(&t0, c->pending.front().a, pe.a);
            cudaEventElapsedTime(&t1, c->pending.front().a, pe.b);
            fprintf(stderr, "  %-22s start %8.3f  dur %7.3f  gap %7.3f ms\n", c->classes[pe.cls].name.c_str(), t0, t1 - t0,
                    t0 - prev_end);
            prev_end = t1;
        }
    }
    for (auto &pe : c->pending) {
        float ms = 0;
        cudaEventSynchronize(pe.b);
        cudaEventElapsedTime(&ms, pe.a, pe.b);
        KernelClass &k = c->classes[pe.cls];
        k.launches++;
        k.ms += ms;
        k.bytes += pe.bytes;
        c->ev_pool.push_back(pe.a);
        c->ev_pool.push_back(pe.b);
    }
    c->pending.clear();
}

// K3 (pack + scatter) needs K2b's per-(CTA, length) bases: computed once per tokenize, on demand.
cudaError_t pack_scatter(wsort_ctx *c) {
    if (!c->cta_counts_ready) {
        cudaError_t e = launch_count_lengths(c->tk, nullptr, c->stream);
        if (e != cudaSuccess) return e;
        c->launches++;
        c->cta_counts_ready = true;
    }
    if (!c->cta_bases_ready) {
        cudaError_t e = launch_cta_bases(c->tk, c->h_sum->max_len, c->stream);
        if (e != cudaSuccess) return e;
        c->launches++;
        c->cta_bases_ready = true;
    }
    return launch_pack_scatter(c->tk, c->stream);
}

// Tokenizer geometry: the same CTA -> byte-range mapping for K1 and K3.
void plan_tokenizer(wsort_ctx *c) {
    TkArgs &a = c->tk;
    a.text = c->d_text;
    a.n = c->n;
    a.nsteps = (uint32_t)((c->n + kTkStep - 1) / kTkStep);
    uint32_t want = (uint32_t)c->sms * ingest_ctas_per_sm();   // one wave of K1 ingest
    uint32_t g = std::min<uint32_t>(a.nsteps, want);
    a.steps_per_cta = g ? (a.nsteps + g - 1) / g : 0;
    a.grid = a.steps_per_cta ? (a.nsteps + a.steps_per_cta - 1) / a.steps_per_cta : 0;
}

}  // namespace

extern "C" {

const char *wsort_strerror(int s) {
    switch (s) {
        case WSORT_OK: return "ok";
        case WSORT_E_INVALID_ARG: return "invalid argument";
        case WSORT_E_STATE: return "call out of order";
        case WSORT_E_NOMEM: return "out of memory";
        case WSORT_E_CUDA: return "CUDA error";
        case WSORT_E_NCCL: return "NCCL error";
        case WSORT_E_TOO_LARGE: return "shard too large";
        case WSORT_E_WORD_TOO_LONG: return "word longer than 255 letters";
        case WSORT_E_BUFFER_TOO_SMALL: return "buffer too small";
        case WSORT_E_NOFILE: return "no such file";
        case WSORT_E_IO: return "I/O error";
        default: return "unknown status";
    }
}

int wsort_create(wsort_ctx **out, int cuda_device, uintptr_t cuda_stream) {
    if (!out) return WSORT_E_INVALID_ARG;
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return WSORT_E_CUDA;
    }
    if (cuda_device < 0 || cuda_device >= ndev) return WSORT_E_INVALID_ARG;
    wsort_ctx *c = new (std::nothrow) wsort_ctx();
    if (!c) return WSORT_E_NOMEM;
    c->device = cuda_device;
    if (cudaSetDevice(cuda_device) != cudaSuccess) {
        delete c;
        return WSORT_E_CUDA;
    }
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, cuda_device);
    if (cuda_stream) {
        c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    } else {
        if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete c;
            return WSORT_E_CUDA;
        }
        c->stream = c->own_stream;
    }
    if (cudaMallocHost(&c->h_sum, sizeof(Summary)) != cudaSuccess) {
        cudaGetLastError();
        if (c->own_stream) cudaStreamDestroy(c->own_stream);
        delete c;
        return WSORT_E_NOMEM;
    }
    *out = c;
    return WSORT_OK;
}

int wsort_set_stream(wsort_ctx *c, uintptr_t cuda_stream) {
    if (!c) return WSORT_E_INVALID_ARG;
    cudaSetDevice(c->device);
    if (!cuda_stream && !c->own_stream) {
        if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) return WSORT_E_CUDA;
    }
    c->stream = cuda_stream ? reinterpret_cast<cudaStream_t>(cuda_stream) : c->own_stream;
    return WSORT_OK;
}

void wsort_destroy(wsort_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    delete c->comm;
    cudaStreamSynchronize(c->stream);
    DevBuf *bufs[] = {&c->text_alloc, &c->cta_hist, &c->cta_base, &c->d_sum, &c->keys_a, &c->keys_b,
                      &c->pay_a, &c->pay_b, &c->words, &c->src_off, &c->dh, &c->status0, &c->status1,
                      &c->tickets, &c->plan, &c->va_x, &c->va_y, &c->splits, &c->bk, &c->d_counts,
                      &c->d_cursor, &c->d_sbase, &c->d_split, &c->d_lohi, &c->d_tiles, &c->d_ranges,
                      &c->m_hist, &c->m_cursor, &c->m_ctr, &c->m_big[0], &c->m_big[1], &c->m_tiles[0],
                      &c->m_tiles[1], &c->m_tiny, &c->m_small, &c->m_copy, &c->m_skip, &c->m_pat, &c->m_qparts, &c->m_pbase, &c->m_jdone,
                      &c->m_jovf, &c->m_partn, &c->m_plist, &c->m_qemit, &c->ghist, &c->dense,
                      &c->pool, &c->chunk_cls, &c->chunk_fill, &c->ig_ctr, &c->cls_list, &c->slice_hist, &c->m_sub, &c->m_subn, &c->d_blk_sum, &c->d_blk_nnz,
                      &c->d_ent_idx, &c->d_ent_end, &c->d_n_ent, &c->d_touched, &c->d_tiles2, &c->d_lcursor, &c->d_tile_e,
                      &c->t_wlens, &c->t_nkey, &c->t_ncnt, &c->t_fp, &c->t_meta, &c->t_cnt, &c->t_keys, &c->t_top, &c->t_dcount, &c->t_runend,
                      &c->t_scan, &c->t_tilee, &c->t_kplan, &c->t_dpfx, &c->t_rpfx, &c->x_vec, &c->x_counts,
                      &c->x_prefix, &c->x_samples, &c->x_all, &c->x_order, &c->x_split, &c->x_dest, &c->x_send,
                      &c->x_matrix, &c->x_cursor, &c->x_recvn, &c->x_win, &c->x_peers, &c->x_flag, &c->x_lwords,
                      &c->x_lwords_all};
    for (DevBuf *b : bufs)
        if (b->p) cudaFree(b->p);
    if (c->h_sum) cudaFreeHost(c->h_sum);
    if (c->h_plan_pinned) cudaFreeHost(c->h_plan_pinned);
    if (c->arena) cudaFreeHost(c->arena);
    if (c->arena_done) cudaEventDestroy(c->arena_done);
    if (c->h_ctr) cudaFreeHost(c->h_ctr);
    if (c->h_ig) cudaFreeHost(c->h_ig);
    if (c->h_tab) cudaFreeHost(c->h_tab);
    for (auto &pe : c->pending) {
        cudaEventDestroy(pe.a);
        cudaEventDestroy(pe.b);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->aux && c->aux != c->stream) cudaStreamDestroy(c->aux);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->tk_exec) cudaGraphExecDestroy(c->tk_exec);
    if (c->tk_graph) cudaGraphDestroy(c->tk_graph);
    if (c->hp) cudaStreamDestroy(c->hp);
    if (c->ev_hp0) cudaEventDestroy(c->ev_hp0);
    if (c->ev_hp1) cudaEventDestroy(c->ev_hp1);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->split) cudaStreamDestroy(c->split);
    if (c->ev_lvl) cudaEventDestroy(c->ev_lvl);
    if (c->ev_split) cudaEventDestroy(c->ev_split);
    if (c->ev_plan) cudaEventDestroy(c->ev_plan);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (auto e : c->copy_ev) cudaEventDestroy(e);
    if (c->ev_ingest) cudaEventDestroy(c->ev_ingest);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
}

int wsort_last_error(const wsort_ctx *c, char *msg, size_t cap) {
    if (!c || !msg || cap == 0) return WSORT_E_INVALID_ARG;
    snprintf(msg, cap, "%s", c->err);
    return WSORT_OK;
}

int wsort_ingest_host(wsort_ctx *c, const void *bytes, uint64_t n, uint64_t global_base, uint64_t *n_words) {
    if (!c) return WSORT_E_INVALID_ARG;
    if (c->comm) return set_err(c, WSORT_E_STATE, "wsort_ingest_host: not while attached (use load_text + tokenize)");
    int rc = wsort_load_text(c, nullptr, n ? 0 : 0, WSORT_MEM_HOST, global_base);   // (prepares an empty text)
    if (rc) return rc;
    if (n && !bytes) return set_err(c, WSORT_E_INVALID_ARG, "bytes is NULL with n=%llu", (unsigned long long)n);
    if (n > WSORT_MAX_SHARD_BYTES) return set_err(c, WSORT_E_TOO_LARGE, "shard of %llu bytes", (unsigned long long)n);
    // the buffer for n bytes: zero pads around it, the text itself arrives stage by stage in tokenize
    uint64_t nsteps = (n + kTkStep - 1) / kTkStep;
    size_t need = kTextFrontPad + nsteps * kTkStep + kIgStep + kTkHalo + 64;
    if ((rc = ensure(c, c->text_alloc, need, "text"))) return rc;
    uint8_t *base = static_cast<uint8_t *>(c->text_alloc.p);
    CK(cudaMemsetAsync(base, 0, kTextFrontPad, c->stream), "memset text head");
    CK(cudaMemsetAsync(base + kTextFrontPad + n, 0, need - kTextFrontPad - n, c->stream), "memset text tail");
    c->d_text = base + kTextFrontPad;
    c->n = n;
    plan_tokenizer(c);
    c->state = ST_LOADED;
    c->stream_src = static_cast<const uint8_t *>(bytes);
    rc = wsort_tokenize(c, n_words);
    c->stream_src = nullptr;
    return rc;
}

int wsort_load_text(wsort_ctx *c, const void *bytes, uint64_t n, int mem, uint64_t global_base) {
    if (!c) return WSORT_E_INVALID_ARG;
    if (n && !bytes) return set_err(c, WSORT_E_INVALID_ARG, "bytes is NULL with n=%llu", (unsigned long long)n);
    if (mem != WSORT_MEM_HOST && mem != WSORT_MEM_DEVICE) return set_err(c, WSORT_E_INVALID_ARG, "bad mem %d", mem);
    if (n > WSORT_MAX_SHARD_BYTES)
        return set_err(c, WSORT_E_TOO_LARGE, "shard of %llu bytes exceeds %llu", (unsigned long long)n,
                       (unsigned long long)WSORT_MAX_SHARD_BYTES);
    cudaSetDevice(c->device);
    c->state = ST_CREATED;
    c->packed_pending = false;
    c->keys_external = false;
    c->has_global = false;
    c->word_base = c->byte_base = 0;
    c->dist_dense = c->dense_range = false;
    c->slice_words = c->slice_bytes = 0;
    c->slices.clear();
    uint64_t nsteps = (n + kTkStep - 1) / kTkStep;
    size_t need = kTextFrontPad + nsteps * kTkStep + kIgStep + kTkHalo + 64;   // ingest reads up to 16 KiB + halo past a range
    int rc = ensure(c, c->text_alloc, need, "text");
    if (rc) return rc;
    uint8_t *base = static_cast<uint8_t *>(c->text_alloc.p);
    uint8_t *t = base + kTextFrontPad;
    CK(cudaMemsetAsync(base, 0, kTextFrontPad, c->stream), "memset text head");
    if (n) CK(cudaMemcpyAsync(t, bytes, n, mem == WSORT_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                              c->stream), "copy text");
    CK(cudaMemsetAsync(t + n, 0, need - kTextFrontPad - n, c->stream), "memset text tail");
    c->d_text = t;
    c->n = n;
    c->global_base = global_base;
    plan_tokenizer(c);
    c->state = ST_LOADED;
    return WSORT_OK;
}

int wsort_load_file(wsort_ctx *c, const char *path) {
    if (!c || !path) return WSORT_E_INVALID_ARG;
    FILE *f = fopen(path, "rb");
    if (!f) {
        FILE *probe = fopen(path, "r");
        if (probe) fclose(probe);
        return set_err(c, errno == ENOENT ? WSORT_E_NOFILE : WSORT_E_IO, "cannot open %s", path);
    }
    std::vector<uint8_t> data;
    uint8_t chunk[1 << 16];
    size_t got;
    while ((got = fread(chunk, 1, sizeof chunk, f)) > 0) data.insert(data.end(), chunk, chunk + got);
    bool bad = ferror(f) != 0;
    fclose(f);
    if (bad) return set_err(c, WSORT_E_IO, "read error on %s", path);
    int rc = wsort_load_text(c, data.data(), data.size(), WSORT_MEM_HOST, 0);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->stream), "sync after file load");   // data is a local buffer
    return WSORT_OK;
}

}  // extern "C"
namespace {
int tokenize_impl(wsort_ctx *c, uint64_t *n_words, bool hash);
int tokenize_dist(wsort_ctx *c, uint64_t *n_words);
int sort_dist(wsort_ctx *c);
}
extern "C" {
int wsort_tokenize(wsort_ctx *c, uint64_t *n_words) {
    if (!c) return WSORT_E_INVALID_ARG;
    if (c->state < ST_LOADED) return set_err(c, WSORT_E_STATE, "wsort_tokenize before wsort_load_text");
    cudaSetDevice(c->device);
    if (c->comm) return tokenize_dist(c, n_words);
    // WSORT_INGEST_AUTO: stage the long words' keys (the MSD path); a text with a word of > 66 letters (not
    // staged) is counted into the table of distinct words instead (no fallback to K3 + LSD). COUNT: always
    // the table (it grows x4 per overflow; still overflowing -> staged). STAGE: always staged.
    const bool count_first = c->ingest_mode == WSORT_INGEST_COUNT;
    int rc = tokenize_impl(c, n_words, count_first);
    if (rc == WSORT_OK && !c->hashed && c->ingest_mode == WSORT_INGEST_AUTO && c->h_ig[kIgVeryLong])
        rc = tokenize_impl(c, n_words, true);
    while (rc == WSORT_OK && c->hashed && c->h_tab[hashtab::kTopOverflow] && c->hash_grow < 64) {
        // more distinct long words than the table holds: count again with 4x the slots (kept for later texts)
        c->hash_grow *= 4;
        rc = tokenize_impl(c, n_words, true);
    }
    if (rc == WSORT_OK && c->hashed && c->h_tab[hashtab::kTopOverflow]) {
        // still overflowing (e.g. random letters: nearly every long word distinct): stage the keys instead
        // (one more text pass; the result does not depend on the mode)
        rc = tokenize_impl(c, n_words, false);
    }
    c->ig_info = wsort_ingest_info{};
    c->ig_info.mode = c->hashed ? 1 : 0;
    if (c->hashed) {
        c->ig_info.overflow = c->h_tab[hashtab::kTopOverflow];
        c->ig_info.grow = (uint32_t)c->hash_grow;
        c->ig_info.distinct_narrow = c->h_tab[hashtab::kTopNarrow];
        c->ig_info.distinct_wide = c->h_tab[hashtab::kTopDistinct];
        c->ig_info.narrow_slots = (uint64_t)c->tab.nmask + 1;
        c->ig_info.wide_slots = (uint64_t)c->tab.mask + 1;
    }
    return rc;
}

}  // extern "C"

namespace {

// Hash-mode table sizing: 2^k slots ~ one per 512 (narrow: 6..24 letters) / 4096 (wide: 25..66 letters)
// text bytes, times the context's growth factor (x4 after each overflow, kept for later texts), each
// table at most 70 % filled; key store for 8 words per distinct wide word. c4 (1 GiB): ~1 M distinct
// words of 6..24 letters in 2 M slots.
int hash_alloc(wsort_ctx *c, uint64_t narrow_need = 0, uint64_t wide_need = 0) {
    uint32_t nslots = 4096, slots = 4096;
    while (nslots < (1u << 24) && (uint64_t)nslots * 7 < narrow_need * 10) nslots <<= 1;
    while (slots < (1u << 24) && (uint64_t)slots * 7 < wide_need * 10) slots <<= 1;
    while (nslots < (1u << 24) && ((uint64_t)nslots * 512 < c->n * c->hash_grow || nslots < 4096 * c->hash_grow)) nslots <<= 1;
    while (slots < (1u << 24) && ((uint64_t)slots * 4096 < c->n * c->hash_grow || slots < 4096 * c->hash_grow)) slots <<= 1;
    const uint32_t maxd = (uint32_t)((uint64_t)slots * 7 / 10);
    const uint32_t key_cap = std::min<uint32_t>(maxd * 12 + 1024, (1u << 24) - 64);   // (meta: 24-bit offsets)
    int rc;
    if ((rc = ensure(c, c->t_nkey, (size_t)nslots * 16, "hash narrow keys"))) return rc;
    if ((rc = ensure(c, c->t_ncnt, (size_t)nslots * 4, "hash narrow counts"))) return rc;
    CK(cudaMemsetAsync(c->t_nkey.p, 0, (size_t)nslots * 16, c->stream), "memset hash narrow keys");
    CK(cudaMemsetAsync(c->t_ncnt.p, 0, (size_t)nslots * 4, c->stream), "memset hash narrow counts");
    if ((rc = ensure(c, c->t_fp, (size_t)slots * 8, "hash fingerprints"))) return rc;
    if ((rc = ensure(c, c->t_meta, (size_t)slots * 4, "hash meta"))) return rc;
    if ((rc = ensure(c, c->t_cnt, (size_t)slots * 4, "hash counts"))) return rc;
    if ((rc = ensure(c, c->t_keys, (size_t)key_cap * 4, "hash keys"))) return rc;
    if ((rc = ensure(c, c->t_top, 16, "hash top"))) return rc;
    if ((rc = ensure(c, c->t_dcount, 256 * 4, "hash distinct counts"))) return rc;
    if (!c->h_tab && cudaMallocHost(&c->h_tab, (4 + 256) * 4) != cudaSuccess) {
        cudaGetLastError();
        return set_err(c, WSORT_E_NOMEM, "pinned hash info");
    }
    CK(cudaMemsetAsync(c->t_fp.p, 0, (size_t)slots * 8, c->stream), "memset hash fp");
    CK(cudaMemsetAsync(c->t_meta.p, 0xff, (size_t)slots * 4, c->stream), "memset hash meta");
    CK(cudaMemsetAsync(c->t_cnt.p, 0, (size_t)slots * 4, c->stream), "memset hash counts");
    CK(cudaMemsetAsync(c->t_top.p, 0, 16, c->stream), "memset hash top");
    CK(cudaMemsetAsync(c->t_dcount.p, 0, 256 * 4, c->stream), "memset hash distinct");
    HashTab &t = c->tab;
    t.nkey = static_cast<unsigned long long *>(c->t_nkey.p);
    t.ncnt = static_cast<uint32_t *>(c->t_ncnt.p);
    t.nmask = nslots - 1;
    t.fp = static_cast<unsigned long long *>(c->t_fp.p);
    t.meta = static_cast<uint32_t *>(c->t_meta.p);
    t.cnt = static_cast<uint32_t *>(c->t_cnt.p);
    t.keys = static_cast<uint32_t *>(c->t_keys.p);
    t.top = static_cast<uint32_t *>(c->t_top.p);
    t.dcount = static_cast<uint32_t *>(c->t_dcount.p);
    t.mask = slots - 1;
    t.key_cap = key_cap;
    t.max_distinct = maxd;
    return WSORT_OK;
}

int tokenize_impl(wsort_ctx *c, uint64_t *n_words, bool hash) {
    TkArgs &a = c->tk;
    int rc;
    const uint32_t G = std::max<uint32_t>(a.grid, 1);
    if ((rc = ensure(c, c->cta_hist, (size_t)G * kHistBins * 4, "cta_hist"))) return rc;
    if ((rc = ensure(c, c->cta_base, (size_t)G * 256 * 4, "cta_base"))) return rc;
    if ((rc = ensure(c, c->d_sum, sizeof(Summary), "summary"))) return rc;
    if ((rc = ensure(c, c->ghist, kHistBins * 4, "ghist"))) return rc;
    if ((rc = ensure(c, c->dense, (size_t)dense_entries() * 4, "dense counts"))) return rc;
    if ((rc = ensure(c, c->ig_ctr, kIgCtrs * 4, "ingest counters"))) return rc;
    // staging chunks: each CTA owns a region of the pool; a staged word of kw key words has >= 6kw-4
    // letters plus a separator, so its key bytes <= its text bytes
    c->cta_chunks = hash ? 0u : ingest_cta_chunks((uint64_t)a.steps_per_cta * kTkStep);
    c->n_chunks = G * c->cta_chunks;
    c->hashed = hash;
    if (hash && (rc = hash_alloc(c))) return rc;
    if ((rc = ensure(c, c->pool, ((size_t)c->n_chunks + 1) * kChunkWords * 4, "staging pool"))) return rc;
    if ((rc = ensure(c, c->chunk_cls, (size_t)c->n_chunks * 4, "chunk classes"))) return rc;
    if ((rc = ensure(c, c->chunk_fill, (size_t)c->n_chunks * 4, "chunk fills"))) return rc;
    if ((rc = ensure(c, c->cls_list, (size_t)kMaxStageKw * std::max<uint32_t>(c->n_chunks, 1) * 4, "chunk lists"))) return rc;
    if (!c->h_ig && cudaMallocHost(&c->h_ig, kIgCtrs * 4) != cudaSuccess) {
        cudaGetLastError();
        return set_err(c, WSORT_E_NOMEM, "pinned ingest counters");
    }
    a.cta_hist = static_cast<uint32_t *>(c->cta_hist.p);
    a.cta_base = static_cast<uint32_t *>(c->cta_base.p);
    if ((rc = ensure(c, c->d_touched, dense_scan_blocks(dense_entries()), "dense touched flags", true))) return rc;
    IngestArgs ia{};
    ia.text = a.text;
    ia.n = a.n;
    ia.nsteps = a.nsteps;
    ia.steps_per_cta = a.steps_per_cta;
    ia.grid = a.grid;
    ia.ghist = static_cast<uint32_t *>(c->ghist.p);
    ia.dense = static_cast<uint32_t *>(c->dense.p);
    ia.touched = static_cast<uint8_t *>(c->d_touched.p);
    ia.pool = static_cast<uint32_t *>(c->pool.p);
    ia.chunk_cls = static_cast<uint32_t *>(c->chunk_cls.p);
    ia.chunk_fill = static_cast<uint32_t *>(c->chunk_fill.p);
    ia.cls_list = static_cast<uint32_t *>(c->cls_list.p);
    ia.cls_cap = c->n_chunks;
    ia.cta_chunks = c->cta_chunks;
    ia.ctr = static_cast<uint32_t *>(c->ig_ctr.p);
    ia.hash = hash ? 1u : 0u;
    ia.tab = c->tab;
    if (const char *dbg = getenv("WSORT_INGEST_DEBUG")) ia.debug = (uint32_t)atoi(dbg);
    // Everything from here to the read-back is one launch sequence that depends only on the text size, the
    // mode and the buffers: captured once as a CUDA graph and replayed by later tokenize calls (the
    // launch-bound small texts; not while profiling, streaming the text in, or on the legacy stream)
    auto enqueue = [&]() -> int {
    CK(cudaMemsetAsync(c->ghist.p, 0, kHistBins * 4, c->stream), "memset ghist");
    if (!c->dense_clean) {   // (first use of the table: zero it all; later only the touched blocks)
        CK(cudaMemsetAsync(c->dense.p, 0, (size_t)dense_entries() * 4, c->stream), "memset dense");
        CK(cudaMemsetAsync(c->d_touched.p, 0, dense_scan_blocks(dense_entries()), c->stream), "memset touched");
        c->dense_clean = true;
    } else {
        rc = launch(c, "k0_dense_clear", 0, [&] {
            return launch_dense_clear(static_cast<uint32_t *>(c->dense.p), static_cast<uint8_t *>(c->d_touched.p), c->stream);
        });
        if (rc) return rc;
    }
    CK(cudaMemsetAsync(c->ig_ctr.p, 0, kIgCtrs * 4, c->stream), "memset ingest counters");
    CK(cudaMemsetAsync(c->chunk_fill.p, 0, (size_t)c->n_chunks * 4, c->stream), "memset chunk fills");
    if (c->stream_src) {
        // streamed ingest: S stages of K1 CTAs; stage s's bytes (+32 KiB: the warps' prefetch and words that
        // cross the range end) are copied on the copy stream, and its K1 launch waits for that copy only, so
        // the host->device copy of the later stages overlaps K1 on the earlier ones
        const uint8_t *src = c->stream_src;
        c->stream_src = nullptr;   // (a second pass over the same text reads the device copy)
        if (!c->copy_stream) {
            CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "copy stream");
            CK(cudaEventCreateWithFlags(&c->ev_ingest, cudaEventDisableTiming), "ingest event");
        }
        const uint32_t S = std::min<uint32_t>(8, std::max<uint32_t>(a.grid, 1));
        while (c->copy_ev.size() < S) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "copy event");
            c->copy_ev.push_back(e);
        }
        CK(cudaEventRecord(c->ev_ingest, c->stream), "ingest event");   // (earlier work on the old text is done)
        CK(cudaStreamWaitEvent(c->copy_stream, c->ev_ingest, 0), "ingest wait");
        uint8_t *dst = const_cast<uint8_t *>(c->d_text);
        const uint64_t per_cta = (uint64_t)a.steps_per_cta * kTkStep;
        for (uint32_t st = 0; st < S; st++) {
            const uint32_t g0 = (uint32_t)((uint64_t)a.grid * st / S), g1 = (uint32_t)((uint64_t)a.grid * (st + 1) / S);
            const uint64_t b0 = std::min<uint64_t>(c->n, g0 * per_cta), b1 = std::min<uint64_t>(c->n, g1 * per_cta + 32768);
            if (b1 > b0) CK(cudaMemcpyAsync(dst + b0, src + b0, b1 - b0, cudaMemcpyHostToDevice, c->copy_stream), "copy text stage");
            CK(cudaEventRecord(c->copy_ev[st], c->copy_stream), "copy event");
            CK(cudaStreamWaitEvent(c->stream, c->copy_ev[st], 0), "copy wait");
            rc = launch(c, "k1_ingest", (double)(std::min<uint64_t>(c->n, g1 * per_cta) - b0),
                        [&] { return launch_ingest_range(ia, g0, g1 - g0, c->stream); });
            if (rc) return rc;
        }
    } else {
        rc = launch(c, "k1_ingest", (double)c->n, [&] { return launch_ingest(ia, c->stream); });
        if (rc) return rc;
    }
    // (the histogram of L <= 5 comes from K1's mask counts: no scan of the dense tables here)
    rc = launch(c, "k2_bucket_offsets", (double)kHistBins * 4,
                [&] { return launch_bucket_offsets(ia.ghist, static_cast<Summary *>(c->d_sum.p), c->stream); });
    if (rc) return rc;
    CK(copy_small(c->h_ig, c->ig_ctr.p, kIgCtrs * 4, c->stream), "copy ingest counters");
    CK(copy_small(c->h_sum, c->d_sum.p, sizeof(Summary), c->stream), "copy summary");
    if (hash) {
        CK(copy_small(c->h_tab, c->t_top.p, 16, c->stream), "copy hash top");
        CK(copy_small(c->h_tab + 4, c->t_dcount.p, 256 * 4, c->stream), "copy hash distinct counts");
    }
    return (int)WSORT_OK;
    };
    static const bool no_graph = getenv("WSORT_NO_GRAPH") != nullptr;   // (experiments)
    const char *dbg_env = getenv("WSORT_INGEST_DEBUG");
    const bool graphable = !no_graph && !c->prof && !c->stream_src && c->dense_clean && c->stream != nullptr &&
                           c->stream != cudaStreamLegacy && c->stream != cudaStreamPerThread;
    const uintptr_t key[] = {(uintptr_t)c->n, (uintptr_t)hash, (uintptr_t)a.text, (uintptr_t)c->dense.p,
                             (uintptr_t)c->d_touched.p, (uintptr_t)c->pool.p, (uintptr_t)c->chunk_cls.p,
                             (uintptr_t)c->chunk_fill.p, (uintptr_t)c->cls_list.p, (uintptr_t)c->ig_ctr.p,
                             (uintptr_t)c->ghist.p, (uintptr_t)c->d_sum.p, (uintptr_t)c->h_ig, (uintptr_t)c->h_sum,
                             (uintptr_t)c->h_tab, (uintptr_t)c->tab.nkey, (uintptr_t)c->tab.fp, (uintptr_t)c->tab.keys,
                             (uintptr_t)c->tab.nmask, (uintptr_t)c->tab.mask, (uintptr_t)(dbg_env ? atoi(dbg_env) : 0),
                             (uintptr_t)c->cta_chunks, (uintptr_t)c->t_top.p, (uintptr_t)c->t_dcount.p,
                             (uintptr_t)c->tab.ncnt, (uintptr_t)c->tab.cnt, (uintptr_t)c->tab.meta};
    constexpr size_t nkey = sizeof(key) / sizeof(key[0]);
    if (graphable && c->tk_exec && c->tk_key.size() == nkey && std::equal(key, key + nkey, c->tk_key.begin())) {
        CK(cudaGraphLaunch(c->tk_exec, c->stream), "tokenize graph");
        c->launches += c->tk_nlaunch;
    } else if (graphable) {
        if (c->tk_exec) cudaGraphExecDestroy(c->tk_exec);
        if (c->tk_graph) cudaGraphDestroy(c->tk_graph);
        c->tk_exec = nullptr;
        c->tk_graph = nullptr;
        c->tk_key.clear();
        const uint64_t l0 = c->launches;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "tokenize capture");
        rc = enqueue();
        cudaGraph_t g = nullptr;
        const cudaError_t ee = cudaStreamEndCapture(c->stream, &g);
        if (rc || ee != cudaSuccess) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            return rc ? rc : cuda_err(c, ee, "tokenize capture");
        }
        CK(cudaGraphInstantiate(&c->tk_exec, g, 0), "tokenize graph");
        c->tk_graph = g;
        c->tk_nlaunch = c->launches - l0;
        c->tk_key.assign(key, key + nkey);
        CK(cudaGraphLaunch(c->tk_exec, c->stream), "tokenize graph");
    } else if ((rc = enqueue())) {
        return rc;
    }
    CK(cudaStreamSynchronize(c->stream), "tokenize");
    if (hash) {   // fill of the tables (distinct words per length counted by K1) against their capacity
        uint64_t dn = 0, dw = 0;
        for (uint32_t L = kDenseMaxLen + 1; L < 256; L++) (L <= 24 ? dn : dw) += c->h_tab[4 + L];
        c->h_tab[hashtab::kTopNarrow] = (uint32_t)dn;
        c->h_tab[hashtab::kTopDistinct] = (uint32_t)dw;
        if (dn * 10 > (uint64_t)(c->tab.nmask + 1) * 7 || dw * 10 > (uint64_t)(c->tab.mask + 1) * 7)
            c->h_tab[hashtab::kTopOverflow] |= 8u;
        if (c->h_tab[hashtab::kTopOverflow]) return WSORT_OK;   // (the caller re-tokenizes: bigger table / staging)
    }
    c->cta_bases_ready = c->cta_counts_ready = false;
    if (c->h_ig[kIgVeryLong]) {   // words of 67..255 letters were not staged: histogram them the K3 way
        CK(cudaMemsetAsync(c->ghist.p, 0, kHistBins * 4, c->stream), "memset ghist");
        rc = launch(c, "k1b_count_lengths", (double)c->n,
                    [&] { return launch_count_lengths(a, ia.ghist, c->stream); });
        if (rc) return rc;
        c->cta_counts_ready = true;
        rc = launch(c, "k2_bucket_offsets", (double)kHistBins * 4,
                    [&] { return launch_bucket_offsets(ia.ghist, static_cast<Summary *>(c->d_sum.p), c->stream); });
        if (rc) return rc;
        CK(copy_small(c->h_sum, c->d_sum.p, sizeof(Summary), c->stream), "copy summary");
        CK(cudaStreamSynchronize(c->stream), "tokenize (long words)");
    }
    const Summary &s = *c->h_sum;
    if (c->prof && !c->h_ig[kIgVeryLong] && !hash) {   // K1's algorithmic bytes: the text + the staged keys it wrote
        double staged = 0;
        for (uint32_t L = kDenseMaxLen + 1; L <= s.max_len && L <= 6 * kMaxStageKw; L++)
            staged += 4.0 * kw_of((int)L) * (double)(s.off[L + 1] - s.off[L]);
        const int k1 = class_id(c, "k1_ingest");
        for (auto it = c->pending.rbegin(); it != c->pending.rend(); ++it)
            if (it->cls == k1) {
                it->bytes += staged;
                break;
            }
    }
    if (s.too_long) {
        c->state = ST_LOADED;
        return set_err(c, WSORT_E_WORD_TOO_LONG, "%u word(s) longer than %d letters", s.too_long, kMaxLen);
    }
    if (c->h_ig[kIgOverflow])
        return set_err(c, WSORT_E_CUDA, "ingest: staging %s (internal error)",
                       c->h_ig[kIgOverflow] == 2 ? "chunk id never published" : "pool overflow");
    if (n_words) *n_words = s.n_words;
    c->state = ST_TOKENIZED;
    return WSORT_OK;
}

}  // namespace


namespace {

// Plan layout (one H2D copy): BucketInfo[256] | radix tiles of every pass (class 0 then class 1)
// | emit tiles. Radix tile classes: 0 = buckets with kw <= kRadixRegMaxKw (register path), 1 = wider.
struct SortPlan {
    std::vector<BucketInfo> bk;
    std::vector<std::vector<TileDesc>> tiles[2];            // [class][pass]
    std::vector<uint32_t> tile_keys[2], tile_words[2];      // [class][pass] maxima
    std::vector<double> bytes[2];                           // [class][pass] algorithmic bytes
    std::vector<TileDesc> emit_tiles;
    uint32_t dh_rows = 0;
    uint32_t npasses = 0;
};

int sort_radix(wsort_ctx *c, bool want_src) {
    const Summary &s = *c->h_sum;
    const uint32_t lmax = s.max_len;
    SortPlan P;
    P.bk.assign(256, BucketInfo{});
    for (uint32_t L = 1; L <= lmax; L++) {
        BucketInfo &b = P.bk[L];
        b.key_off = s.key_off[L];
        b.word_off = s.off[L];
        b.byte_off = s.byte_off[L];
        b.n = (uint32_t)(s.off[L + 1] - s.off[L]);
        b.kw = kw_of(L);
        b.ndig = ndig_of(L);
        b.tile_keys = radix_tile_keys(b.kw);
        b.elem_off = b.key_off;
        b.estride = b.kw;
        if (!b.n) continue;
        b.dh_row = P.dh_rows;
        P.dh_rows += b.ndig;
        b.final_b = b.ndig & 1u;
        P.npasses = std::max(P.npasses, b.ndig);
    }
    const uint32_t npasses = P.npasses;
    for (int cl = 0; cl < 2; cl++) {
        P.tiles[cl].resize(npasses);
        P.tile_keys[cl].assign(npasses, 0);
        P.tile_words[cl].assign(npasses, 0);
        P.bytes[cl].assign(npasses, 0.0);
    }
    for (uint32_t p = 0; p < npasses; p++) {
        for (uint32_t L = 1; L <= lmax; L++) {
            const BucketInfo &b = P.bk[L];
            if (!b.n || b.ndig <= p) continue;
            const int cl = b.kw <= kRadixRegMaxKw ? 0 : 1;
            uint32_t nt = (b.n + b.tile_keys - 1) / b.tile_keys;
            for (uint32_t i = 0; i < nt; i++) P.tiles[cl][p].push_back(TileDesc{L, i});
            P.tile_keys[cl][p] = std::max(P.tile_keys[cl][p], b.tile_keys);
            P.tile_words[cl][p] = std::max(P.tile_words[cl][p], b.tile_keys * b.kw);
            P.bytes[cl][p] += 2.0 * (double)b.n * (b.kw * 4 + (want_src ? 4 : 0));
        }
    }
    for (uint32_t L = 1; L <= lmax; L++) {
        const BucketInfo &b = P.bk[L];
        if (!b.n) continue;
        uint32_t te = kEmitStage / (L + 1);
        uint32_t nt = (b.n + te - 1) / te;
        for (uint32_t i = 0; i < nt; i++) P.emit_tiles.push_back(TileDesc{L, i});
    }

    // ---- device buffers ----
    int rc;
    const uint64_t key_words = s.key_off[256];
    const uint64_t W = s.n_words;
    if ((rc = ensure(c, c->keys_a, key_words * 4 + 64, "keys_a"))) return rc;
    if ((rc = ensure(c, c->keys_b, key_words * 4 + 64, "keys_b"))) return rc;
    if (want_src) {
        if ((rc = ensure(c, c->pay_a, W * 4 + 64, "pay_a"))) return rc;
        if ((rc = ensure(c, c->pay_b, W * 4 + 64, "pay_b"))) return rc;
        if ((rc = ensure(c, c->src_off, W * 8 + 64, "src_off"))) return rc;
    }
    if ((rc = ensure(c, c->words, s.byte_off[256] + 64, "words"))) return rc;
    if ((rc = ensure(c, c->dh, (size_t)std::max<uint32_t>(P.dh_rows, 1) * kRadixBins * 4, "dh"))) return rc;
    size_t rows[2] = {0, 0};   // status rows per class: max tiles over passes
    for (int cl = 0; cl < 2; cl++)
        for (auto &v : P.tiles[cl]) rows[cl] = std::max(rows[cl], v.size());
    const size_t status_bytes = std::max<size_t>(rows[0] + rows[1], 1) * kRadixBins * 4;
    if (c->status0.cap < status_bytes || c->status1.cap < status_bytes) {
        if ((rc = ensure(c, c->status0, status_bytes, "status0"))) return rc;
        if ((rc = ensure(c, c->status1, status_bytes, "status1"))) return rc;
        CK(cudaMemsetAsync(c->status0.p, 0, c->status0.cap, c->stream), "memset status0");
        CK(cudaMemsetAsync(c->status1.p, 0, c->status1.cap, c->stream), "memset status1");
    }
    if ((rc = ensure(c, c->tickets, std::max<uint32_t>(2 * npasses, 1) * 4, "tickets"))) return rc;

    // ---- plan upload ----
    const size_t off_tiles = 256 * sizeof(BucketInfo);
    std::vector<size_t> toff[2];
    toff[0].resize(npasses);
    toff[1].resize(npasses);
    size_t cur = off_tiles;
    for (uint32_t p = 0; p < npasses; p++)
        for (int cl = 0; cl < 2; cl++) {
            toff[cl][p] = cur;
            cur += P.tiles[cl][p].size() * sizeof(TileDesc);
        }
    const size_t emit_off = cur;
    cur += P.emit_tiles.size() * sizeof(TileDesc);
    const size_t plan_bytes = cur;
    if (c->h_plan_cap < plan_bytes) {
        if (c->h_plan_pinned) cudaFreeHost(c->h_plan_pinned);
        c->h_plan_pinned = nullptr;
        c->h_plan_cap = 0;
        if (cudaMallocHost(&c->h_plan_pinned, plan_bytes * 2) != cudaSuccess) {
            cudaGetLastError();
            return set_err(c, WSORT_E_NOMEM, "pinned plan buffer");
        }
        c->h_plan_cap = plan_bytes * 2;
    }
    uint8_t *hp = c->h_plan_pinned;
    memcpy(hp, P.bk.data(), off_tiles);
    for (uint32_t p = 0; p < npasses; p++)
        for (int cl = 0; cl < 2; cl++)
            memcpy(hp + toff[cl][p], P.tiles[cl][p].data(), P.tiles[cl][p].size() * sizeof(TileDesc));
    memcpy(hp + emit_off, P.emit_tiles.data(), P.emit_tiles.size() * sizeof(TileDesc));
    if ((rc = ensure(c, c->plan, plan_bytes, "plan"))) return rc;
    CK(cudaMemcpyAsync(c->plan.p, hp, plan_bytes, cudaMemcpyHostToDevice, c->stream), "plan upload");
    uint8_t *dp = static_cast<uint8_t *>(c->plan.p);
    const BucketInfo *d_bk = reinterpret_cast<const BucketInfo *>(dp);

    // ---- K3 ----
    uint32_t *ka = static_cast<uint32_t *>(c->keys_a.p), *kb = static_cast<uint32_t *>(c->keys_b.p);
    uint32_t *pa = want_src ? static_cast<uint32_t *>(c->pay_a.p) : nullptr;
    uint32_t *pb = want_src ? static_cast<uint32_t *>(c->pay_b.p) : nullptr;
    TkArgs &tk = c->tk;
    tk.buckets = d_bk;
    tk.keys = ka;
    tk.payload = pa;
    const double key_bytes = (double)key_words * 4;
    if (!c->packed_pending) {
        rc = launch(c, "k3_pack_scatter", (double)c->n + key_bytes + (want_src ? 4.0 * W : 0.0),
                    [&] { return pack_scatter(c); });
        if (rc) return rc;
    }

    if (npasses) {
        CK(cudaMemsetAsync(c->dh.p, 0, (size_t)P.dh_rows * kRadixBins * 4, c->stream), "memset dh");
        CK(cudaMemsetAsync(c->tickets.p, 0, 2 * npasses * 4, c->stream), "memset tickets");
        uint32_t *dh = static_cast<uint32_t *>(c->dh.p);
        RadixArgs ra{};
        ra.buckets = d_bk;
        ra.tiles = reinterpret_cast<const TileDesc *>(dp + toff[0][0]);   // pass 0, both classes
        ra.ntiles = (uint32_t)(P.tiles[0][0].size() + P.tiles[1][0].size());
        ra.kin = ka;
        ra.dh = dh;
        rc = launch(c, "k4_digit_hist", key_bytes, [&] { return launch_digit_hist(ra, c->stream); });
        if (rc) return rc;
        rc = launch(c, "k4_digit_scan", (double)P.dh_rows * kRadixBins * 8,
                    [&] { return launch_digit_scan(dh, P.dh_rows, c->stream); });
        if (rc) return rc;
        uint32_t *st[2] = {static_cast<uint32_t *>(c->status0.p), static_cast<uint32_t *>(c->status1.p)};
        uint32_t last[2] = {0, 0};   // last pass with tiles, per class
        for (uint32_t p = 0; p < npasses; p++) {
            for (int cl = 0; cl < 2; cl++) {
                const size_t base = cl ? rows[0] * kRadixBins : 0;
                RadixArgs r{};
                r.buckets = d_bk;
                r.tiles = reinterpret_cast<const TileDesc *>(dp + toff[cl][p]);
                r.ntiles = (uint32_t)P.tiles[cl][p].size();
                r.nzero = p ? (uint32_t)P.tiles[cl][p - 1].size() : 0u;
                if (!r.ntiles && !r.nzero) continue;
                if (r.ntiles) last[cl] = p;
                r.pass = p;
                r.max_tile_keys = std::max<uint32_t>(P.tile_keys[cl][p], 32);
                r.max_tile_words = std::max<uint32_t>(P.tile_words[cl][p], 32);
                const bool even = (p & 1u) == 0;
                r.kin = even ? ka : kb;
                r.kout = even ? kb : ka;
                r.pin = want_src ? (even ? pa : pb) : nullptr;
                r.pout = want_src ? (even ? pb : pa) : nullptr;
                r.dh = dh;
                r.status = st[p & 1u] + base;
                r.status_other = st[(p + 1) & 1u] + base;
                r.ticket = static_cast<uint32_t *>(c->tickets.p) + 2 * p + cl;
                rc = launch(c, cl ? "k4_radix_pass_long" : "k4_radix_pass", P.bytes[cl][p],
                            [&] { return launch_radix_pass(r, cl == 1, c->stream); });
                if (rc) return rc;
            }
        }
        // leave both status buffers clean for the next sort
        for (int cl = 0; cl < 2; cl++) {
            const size_t n = P.tiles[cl][last[cl]].size();
            if (n)
                CK(cudaMemsetAsync(st[last[cl] & 1u] + (cl ? rows[0] * kRadixBins : 0), 0, n * kRadixBins * 4,
                                   c->stream), "memset status");
        }
    }

    EmitArgs ea{};
    ea.buckets = d_bk;
    ea.tiles = reinterpret_cast<const TileDesc *>(dp + emit_off);
    ea.ntiles = (uint32_t)P.emit_tiles.size();
    ea.keys_a = ka;
    ea.keys_b = kb;
    ea.pay_a = pa;
    ea.pay_b = pb;
    ea.words = static_cast<uint8_t *>(c->words.p);
    ea.src_off = want_src ? static_cast<uint64_t *>(c->src_off.p) : nullptr;
    ea.global_base = c->global_base;
    rc = launch(c, "k5_emit", key_bytes + (double)s.byte_off[256] + (want_src ? 12.0 * W : 0.0),
                [&] { return launch_emit(ea, c->stream); });
    return rc;
}


// Upload `bytes` of host data through the pinned plan buffer (one H2D copy) into c->plan.
int upload_plan(wsort_ctx *c, const std::vector<uint8_t> &buf) {
    if (c->h_plan_cap < buf.size()) {
        if (c->h_plan_pinned) cudaFreeHost(c->h_plan_pinned);
        c->h_plan_pinned = nullptr;
        c->h_plan_cap = 0;
        if (cudaMallocHost(&c->h_plan_pinned, buf.size() * 2) != cudaSuccess) {
            cudaGetLastError();
            return set_err(c, WSORT_E_NOMEM, "pinned plan buffer");
        }
        c->h_plan_cap = buf.size() * 2;
    }
    memcpy(c->h_plan_pinned, buf.data(), buf.size());
    int rc = ensure(c, c->plan, buf.size(), "plan");
    if (rc) return rc;
    CK(cudaMemcpyAsync(c->plan.p, c->h_plan_pinned, buf.size(), cudaMemcpyHostToDevice, c->stream), "plan upload");
    return WSORT_OK;
}

template <class T>
size_t append(std::vector<uint8_t> &buf, const std::vector<T> &v) {
    size_t off = buf.size();
    buf.resize(off + v.size() * sizeof(T));
    if (!v.empty()) memcpy(buf.data() + off, v.data(), v.size() * sizeof(T));
    return off;
}

// Variant A: OETS tile sort + merge-path passes (PAPER.md:23 bubble sort in chunks, :76 merge).
int sort_oets(wsort_ctx *c, bool want_src) {
    const Summary &s = *c->h_sum;
    const uint32_t lmax = s.max_len;
    std::vector<BucketInfo> bk(256, BucketInfo{});
    uint64_t eoff = 0;
    uint32_t max_passes = 0, max_tw = 32;
    std::vector<uint32_t> npass(256, 0);
    for (uint32_t L = 1; L <= lmax; L++) {
        BucketInfo &b = bk[L];
        b.key_off = s.key_off[L];
        b.word_off = s.off[L];
        b.byte_off = s.byte_off[L];
        b.n = (uint32_t)(s.off[L + 1] - s.off[L]);
        b.kw = kw_of(L);
        b.estride = b.kw + (want_src ? 1 : 0);
        b.tile_keys = kMergeThreads * oets_elems_per_thread(b.estride);
        b.elem_off = want_src ? eoff : b.key_off;
        eoff += (uint64_t)b.n * b.estride;
        if (!b.n) continue;
        uint32_t nt = (b.n + b.tile_keys - 1) / b.tile_keys, m = 0;
        while ((1u << m) < nt) m++;
        npass[L] = m;
        b.final_b = (m & 1u) ? 0u : 1u;   // tile sort writes X (= "b"), each merge pass swaps
        max_passes = std::max(max_passes, m);
        max_tw = std::max(max_tw, b.tile_keys * b.estride);
    }
    std::vector<TileDesc> sort_tiles, emit_tiles;
    std::vector<std::vector<TileDesc>> merge_tiles(max_passes);
    for (uint32_t L = 1; L <= lmax; L++) {
        const BucketInfo &b = bk[L];
        if (!b.n) continue;
        const uint32_t nt = (b.n + b.tile_keys - 1) / b.tile_keys;
        for (uint32_t i = 0; i < nt; i++) sort_tiles.push_back(TileDesc{L, i});
        for (uint32_t m = 0; m < npass[L]; m++)
            for (uint32_t i = 0; i < nt; i++) merge_tiles[m].push_back(TileDesc{L, i});
        const uint32_t te = kEmitStage / (L + 1);
        for (uint32_t i = 0; i < (b.n + te - 1) / te; i++) emit_tiles.push_back(TileDesc{L, i});
    }
    // buffers: keys-only -> X = keys_b, Y = keys_a (K3 output is consumed by the tile sort);
    // with src_off -> interleaved (key words + payload) buffers.
    int rc;
    const uint64_t key_words = s.key_off[256];
    const uint64_t W = s.n_words;
    if ((rc = ensure(c, c->keys_a, key_words * 4 + 64, "keys_a"))) return rc;
    if ((rc = ensure(c, c->keys_b, key_words * 4 + 64, "keys_b"))) return rc;
    if (want_src) {
        if ((rc = ensure(c, c->pay_a, W * 4 + 64, "pay_a"))) return rc;
        if ((rc = ensure(c, c->src_off, W * 8 + 64, "src_off"))) return rc;
        if ((rc = ensure(c, c->va_x, eoff * 4 + 64, "va_x"))) return rc;
        if ((rc = ensure(c, c->va_y, eoff * 4 + 64, "va_y"))) return rc;
    }
    if ((rc = ensure(c, c->words, s.byte_off[256] + 64, "words"))) return rc;
    if ((rc = ensure(c, c->splits, (sort_tiles.size() + 1) * 4, "splits"))) return rc;
    std::vector<uint8_t> plan;
    append(plan, bk);
    const size_t o_sort = append(plan, sort_tiles);
    std::vector<size_t> o_merge(max_passes);
    for (uint32_t m = 0; m < max_passes; m++) o_merge[m] = append(plan, merge_tiles[m]);
    const size_t o_emit = append(plan, emit_tiles);
    if ((rc = upload_plan(c, plan))) return rc;
    uint8_t *dp = static_cast<uint8_t *>(c->plan.p);
    const BucketInfo *d_bk = reinterpret_cast<const BucketInfo *>(dp);

    uint32_t *ka = static_cast<uint32_t *>(c->keys_a.p), *kb = static_cast<uint32_t *>(c->keys_b.p);
    uint32_t *pa = want_src ? static_cast<uint32_t *>(c->pay_a.p) : nullptr;
    uint32_t *X = want_src ? static_cast<uint32_t *>(c->va_x.p) : kb;
    uint32_t *Y = want_src ? static_cast<uint32_t *>(c->va_y.p) : ka;
    TkArgs &tk = c->tk;
    tk.buckets = d_bk;
    tk.keys = ka;
    tk.payload = pa;
    const double key_bytes = (double)key_words * 4, elem_bytes = (double)eoff * 4;
    if (!c->packed_pending) {
        rc = launch(c, "k3_pack_scatter", (double)c->n + key_bytes + (want_src ? 4.0 * W : 0.0),
                    [&] { return pack_scatter(c); });
        if (rc) return rc;
    }
    OetsArgs oa{};
    oa.buckets = d_bk;
    oa.tiles = reinterpret_cast<const TileDesc *>(dp + o_sort);
    oa.ntiles = (uint32_t)sort_tiles.size();
    oa.max_tile_words = max_tw;
    oa.keys_in = ka;
    oa.pay_in = pa;
    oa.out = X;
    rc = launch(c, "k4a_oets_tile_sort", key_bytes + (want_src ? 4.0 * W : 0.0) + (want_src ? elem_bytes : key_bytes),
                [&] { return launch_oets_tile_sort(oa, c->stream); });
    if (rc) return rc;
    for (uint32_t m = 0; m < max_passes; m++) {
        MergeArgs ma{};
        ma.buckets = d_bk;
        ma.tiles = reinterpret_cast<const TileDesc *>(dp + o_merge[m]);
        ma.ntiles = (uint32_t)merge_tiles[m].size();
        ma.pass = m;
        ma.max_tile_words = max_tw;
        ma.in = (m & 1u) ? Y : X;
        ma.out = (m & 1u) ? X : Y;
        ma.splits = static_cast<uint32_t *>(c->splits.p);
        double bytes = 0;
        for (uint32_t L = 1; L <= lmax; L++)
            if (npass[L] > m) bytes += 2.0 * bk[L].n * bk[L].estride * 4.0;
        rc = launch(c, "k4b_merge_pass", bytes, [&] { return launch_merge_pass(ma, c->stream); });
        if (rc) return rc;
    }
    EmitArgs ea{};
    ea.buckets = d_bk;
    ea.tiles = reinterpret_cast<const TileDesc *>(dp + o_emit);
    ea.ntiles = (uint32_t)emit_tiles.size();
    ea.keys_a = Y;
    ea.keys_b = X;
    ea.pay_a = nullptr;
    ea.pay_b = nullptr;
    ea.words = static_cast<uint8_t *>(c->words.p);
    ea.src_off = want_src ? static_cast<uint64_t *>(c->src_off.p) : nullptr;
    ea.global_base = c->global_base;
    return launch(c, "k5_emit", (want_src ? elem_bytes : key_bytes) + (double)s.byte_off[256] + (want_src ? 8.0 * W : 0.0),
                  [&] { return launch_emit(ea, c->stream); });
}


// msd_radix (keys only): MSD partitioning by 2-letter digits, level by level, with device-side
// planning (k_msd_plan queues the next level's segments and the finishing jobs); one small D2H of
// the queue counters per level sizes the next launches.
// MSD queues (segments, scatter tiles, finishing jobs, copies) sized for W words.
int msd_alloc(wsort_ctx *c, MsdArgs &m, uint64_t W, uint64_t key_words) {
    const uint32_t cap_big = (uint32_t)(W / 1024 + 4096), cap_tiles = (uint32_t)(W / 1024 + 2 * cap_big + 4096);
    const uint32_t cap_local = (uint32_t)(W / 256 + 65536), cap_copy = (uint32_t)(W / 1024 + key_words / 65536 + 4096);
    int rc;
    for (int i = 0; i < 2; i++) {
        if ((rc = ensure(c, c->m_big[i], (size_t)cap_big * sizeof(MsdSeg), "msd segs"))) return rc;
        if ((rc = ensure(c, c->m_tiles[i], (size_t)cap_tiles * sizeof(MsdTile), "msd tiles"))) return rc;
    }
    if ((rc = ensure(c, c->m_tiny, (size_t)cap_local * sizeof(MsdSeg), "msd tiny"))) return rc;
    if ((rc = ensure(c, c->m_small, (size_t)cap_local * sizeof(MsdSeg), "msd small"))) return rc;
    if ((rc = ensure(c, c->m_copy, (size_t)cap_copy * sizeof(CopyRange), "msd copy"))) return rc;
    if ((rc = ensure(c, c->m_ctr, kQCount * 4, "msd counters"))) return rc;
    if ((rc = ensure(c, c->m_skip, (size_t)cap_big * 4, "msd skip flags"))) return rc;
    if ((rc = ensure(c, c->m_pat, (size_t)c->sms * 4 * kFinPatBytes, "finish patterns"))) return rc;
    // sub-jobs of the jobs a finishing CTA partitions itself (fin_partition), run by a second k_msd_fin launch
    const uint32_t cap_sub = (uint32_t)(W / 64 + 65536);
    if ((rc = ensure(c, c->m_sub, (size_t)cap_sub * sizeof(MsdSeg), "finish sub-jobs"))) return rc;
    if ((rc = ensure(c, c->m_subn, 16, "finish sub-job count", true))) return rc;
    // finishing tickets of big jobs (> 16384 keys: one each, or one per part of <= kPartKeys keys when
    // split): <= W / 16384 + 2 W / kPartKeys
    const uint32_t cap_parts = (uint32_t)(W / 16384 + 2 * W / kPartKeys + 64);
    if ((rc = ensure(c, c->m_qparts, (size_t)cap_parts * 4, "parts"))) return rc;
    if ((rc = ensure(c, c->m_partn, (size_t)cap_parts * 4, "part sizes"))) return rc;
    if ((rc = ensure(c, c->m_plist, (size_t)cap_parts * kPartListMax * 16, "part lists"))) return rc;
    if ((rc = ensure(c, c->m_pbase, (size_t)cap_local * 4, "job parts"))) return rc;
    if ((rc = ensure(c, c->m_jdone, (size_t)cap_local * 4, "job arrivals"))) return rc;
    if ((rc = ensure(c, c->m_jovf, (size_t)cap_local * 4, "job overflow"))) return rc;
    const uint32_t cap_emit = (uint32_t)(2 * W / kEmitPieceWords + 64);
    if ((rc = ensure(c, c->m_qemit, (size_t)cap_emit * 8, "text pieces"))) return rc;
    if (!c->h_ctr && cudaMallocHost(&c->h_ctr, kQCount * 4) != cudaSuccess) {
        cudaGetLastError();
        return set_err(c, WSORT_E_NOMEM, "pinned counters");
    }
    m = MsdArgs{};
    m.ctr = static_cast<uint32_t *>(c->m_ctr.p);
    m.q_tiny = static_cast<MsdSeg *>(c->m_tiny.p);
    m.q_small = static_cast<MsdSeg *>(c->m_small.p);
    m.q_copy = static_cast<CopyRange *>(c->m_copy.p);
    m.cap_big = cap_big;
    m.cap_tiles = cap_tiles;
    m.cap_local = cap_local;
    m.cap_copy = cap_copy;
    m.keys_a = static_cast<uint32_t *>(c->keys_a.p);
    m.keys_b = static_cast<uint32_t *>(c->keys_b.p);
    m.seg_skip = static_cast<uint32_t *>(c->m_skip.p);
    m.pat = static_cast<uint8_t *>(c->m_pat.p);
    static const bool no_sub = getenv("WSORT_NO_SUBPART") != nullptr;   // (experiments)
    m.sub_stack = no_sub ? nullptr : static_cast<MsdSeg *>(c->m_sub.p);
    m.sub_n = static_cast<uint32_t *>(c->m_subn.p);
    m.cap_sub = cap_sub;
    m.cap_parts = cap_parts;
    m.q_parts = static_cast<uint32_t *>(c->m_qparts.p);
    m.job_pbase = static_cast<uint32_t *>(c->m_pbase.p);
    m.job_done = static_cast<uint32_t *>(c->m_jdone.p);
    m.job_ovf = static_cast<uint32_t *>(c->m_jovf.p);
    m.part_n = static_cast<uint32_t *>(c->m_partn.p);
    m.part_list = static_cast<uint4 *>(c->m_plist.p);
    m.cap_emit = cap_emit;
    m.q_emit = static_cast<uint2 *>(c->m_qemit.p);
    return WSORT_OK;
}

int msd_level_buffers(wsort_ctx *c, MsdArgs &m, uint32_t level, uint32_t nsegs) {
    int rc;
    if ((rc = ensure(c, c->m_hist, (size_t)nsegs * kRadixBins * 4, "msd hist"))) return rc;
    if ((rc = ensure(c, c->m_cursor, (size_t)nsegs * kRadixBins * 4, "msd cursor"))) return rc;
    CK(cudaMemsetAsync(c->m_hist.p, 0, (size_t)nsegs * kRadixBins * 4, c->stream), "memset msd hist");
    CK(cudaMemsetAsync(c->m_ctr.p, 0, 2 * 4, c->stream), "reset big/tiles counters");
    const int cur = level & 1;
    uint32_t *ka = static_cast<uint32_t *>(c->keys_a.p), *kb = static_cast<uint32_t *>(c->keys_b.p);
    m.level = level;
    m.dst_is_a = level & 1u;
    m.segs = static_cast<const MsdSeg *>(c->m_big[cur].p);
    m.tiles = static_cast<const MsdTile *>(c->m_tiles[cur].p);
    m.src = (level & 1u) ? kb : ka;
    m.dst = (level & 1u) ? ka : kb;
    m.hist = static_cast<uint32_t *>(c->m_hist.p);
    m.cursor = static_cast<uint32_t *>(c->m_cursor.p);
    m.q_big = static_cast<MsdSeg *>(c->m_big[cur ^ 1].p);
    m.q_tiles = static_cast<MsdTile *>(c->m_tiles[cur ^ 1].p);
    return WSORT_OK;
}

// After a level's plan + scatter: read the queue counters (one stream sync) for the next level.
int msd_read_counters(wsort_ctx *c, const MsdArgs &m, uint32_t &nsegs, uint32_t &ntiles) {
    CK(copy_small(c->h_ctr, c->m_ctr.p, kQCount * 4, c->stream), "msd counters");
    CK(cudaStreamSynchronize(c->stream), "msd level");
    nsegs = c->h_ctr[kQBig];
    ntiles = c->h_ctr[kQTiles];
    if (nsegs > m.cap_big || ntiles > m.cap_tiles || c->h_ctr[kQTiny] > m.cap_local || c->h_ctr[kQSmall] > m.cap_local ||
        c->h_ctr[kQCopy] > m.cap_copy || c->h_ctr[kQParts] > m.cap_parts || c->h_ctr[kQEmit] > m.cap_emit)
        return set_err(c, WSORT_E_NOMEM, "msd queue overflow (segs %u tiles %u)", nsegs, ntiles);
    return WSORT_OK;
}

// The third stream (high priority): split finishing jobs, and level 0's job planning beside the scatter
int ensure_split_stream(wsort_ctx *c) {
    if (c->split) return WSORT_OK;
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
    CK(cudaStreamCreateWithPriority(&c->split, cudaStreamNonBlocking, greatest), "split stream");
    CK(cudaEventCreateWithFlags(&c->ev_lvl, cudaEventDisableTiming), "level event");
    CK(cudaEventCreateWithFlags(&c->ev_split, cudaEventDisableTiming), "split event");
    CK(cudaEventCreateWithFlags(&c->ev_plan, cudaEventDisableTiming), "plan event");
    return WSORT_OK;
}

// MSD levels from `level` on (its segments / tiles are in m_big[level & 1] / m_tiles[level & 1]) until no
// segment is left, then the finishing sorts: every key ends in buffer B at its final index.
int msd_levels_and_finish(wsort_ctx *c, MsdArgs &m, uint32_t level, uint32_t nsegs, uint32_t ntiles, uint32_t levels,
                          double key_bytes, uint32_t max_tw, bool may_requeue = false) {
    int rc;
    m.stream_fin = m.finish_radix ? 0u : 1u;
    const uint32_t fin_grid = (uint32_t)c->sms * 4;   // k_msd_fin: 4 resident CTAs per SM
    uint32_t small_done = 0, parts_done = 0, emit_done = 0;
    if (!m.finish_radix && (c->h_ctr[kQSmall] || c->h_ctr[kQTiny])) {   // jobs planned before the first level
        if (may_requeue && nsegs == 0) {   // (whole buckets larger than a tile: one with too many distinct keys
                                           // goes back to the MSD as a level-0 segment)
            m.q_big = static_cast<MsdSeg *>(c->m_big[0].p);
            m.q_tiles = static_cast<MsdTile *>(c->m_tiles[0].p);
        }
        rc = launch(c, "k4m_msd_finish", 0, [&] { return launch_msd_fin_jobs(m, 0, 0, fin_grid, c->stream); });
        if (rc) return rc;
        // the sub-jobs of the whole-bucket jobs their finishing CTAs partitioned (fin_partition)
        rc = launch(c, "k4m_msd_fin_sub", 0, [&] { return launch_msd_fin_sub(m, fin_grid, c->stream); });
        if (rc) return rc;
        small_done = c->h_ctr[kQSmall];
        parts_done = c->h_ctr[kQParts];
        if (may_requeue && nsegs == 0) {
            if ((rc = msd_read_counters(c, m, nsegs, ntiles))) return rc;
            small_done = std::min(c->h_ctr[kQSmall], m.cap_local);
        }
    }
    static const bool no_plan_beside = getenv("WSORT_NO_PLAN_BESIDE") != nullptr;   // (experiments)
    for (; nsegs > 0; level++) {
        if (level >= levels) return set_err(c, WSORT_E_CUDA, "msd: segments left after the last digit");
        if ((rc = msd_level_buffers(c, m, level, nsegs))) return rc;
        const double seg_bytes = level == 0 ? key_bytes : 0;   // later levels' sizes are device-side
        if (m.chunk_mode)
            rc = launch(c, "k4m_msd_count0", seg_bytes, [&] { return launch_msd_count0(m, c->stream); });
        else
            rc = launch(c, "k4m_msd_count", seg_bytes, [&] { return launch_msd_count(m, ntiles, c->stream); });
        if (rc) return rc;
        // level 0 of the streaming path: the scatter needs only the children's cursors; the finishing jobs
        // are planned on the split stream beside it (the serial per-segment job packing is off the critical path)
        const bool plan_beside = m.chunk_mode && !m.finish_radix && !c->prof_serial && !no_plan_beside;
        if (plan_beside) {
            if ((rc = ensure_split_stream(c))) return rc;
            rc = launch(c, "k4m_msd_plan", (double)nsegs * kRadixBins * 4, [&] { return launch_msd_plan(m, nsegs, c->stream, 1); });
            if (rc) return rc;
            if ((rc = arena_flush(c))) return rc;
            CK(cudaEventRecord(c->ev_lvl, c->stream), "plan event");
            CK(cudaStreamWaitEvent(c->split, c->ev_lvl, 0), "plan wait");
            rc = launch_on(c, c->split, "k4m_msd_plan_jobs", (double)nsegs * kRadixBins * 4,
                           [&] { return launch_msd_plan(m, nsegs, c->split, 2); });
            if (rc) return rc;
            CK(cudaEventRecord(c->ev_plan, c->split), "plan jobs event");
        } else {
            rc = launch(c, "k4m_msd_plan", (double)nsegs * kRadixBins * 8, [&] { return launch_msd_plan(m, nsegs, c->stream); });
            if (rc) return rc;
        }
        if (m.chunk_mode)
            rc = launch(c, "k4m_msd_scatter0", 2 * seg_bytes, [&] { return launch_msd_scatter0(m, c->stream); });
        else
            rc = launch(c, "k4m_msd_scatter", 2 * seg_bytes, [&] { return launch_msd_scatter(m, ntiles, c->stream); });
        if (rc) return rc;
        if (plan_beside) CK(cudaStreamWaitEvent(c->stream, c->ev_plan, 0), "plan jobs wait");
        m.chunk_mode = 0;   // (only level 0 reads the staging chunks)
        if (!m.finish_radix) {   // this level's finishing jobs (their count is on the device); a job with too
                                 // many distinct keys re-enters the next level
            static const bool dbg = getenv("WSORT_DEBUG_JOBS") != nullptr;   // (experiments: slowest jobs)
            uint32_t *dj = nullptr;
            if (dbg) {
                cudaMalloc(&dj, 65536 * 16);
                cudaMemset(dj, 0, 65536 * 16);
                m.dbg_jobs = dj;
            }
            // the parts of split jobs (if any: their number is on the device) on the third stream, beside
            // the whole jobs; then the text of the split jobs, by pieces
            if ((rc = ensure_split_stream(c))) return rc;
            if ((rc = arena_flush(c))) return rc;
            CK(cudaEventRecord(c->ev_lvl, c->stream), "level event");
            cudaStream_t sp = c->prof_serial ? c->stream : c->split;   // (serial profiling: one stream)
            CK(cudaStreamWaitEvent(sp, c->ev_lvl, 0), "level wait");
            rc = launch_on(c, sp, "k4m_msd_fin_split", 0,
                           [&] { return launch_msd_fin_split(m, parts_done, fin_grid, sp); });
            if (rc) return rc;
            rc = launch_on(c, sp, "k4m_msd_fin_emit", 0,
                           [&] { return launch_msd_fin_emit(m, emit_done, (uint32_t)c->sms * 2, sp); });
            if (rc) return rc;
            CK(cudaEventRecord(c->ev_split, sp), "split event");
            rc = launch(c, "k4m_msd_finish", level == 0 ? 2 * key_bytes : 0,
                        [&] { return launch_msd_fin_jobs(m, small_done, parts_done, fin_grid, c->stream); });
            if (rc) return rc;
            rc = launch(c, "k4m_msd_fin_sub", 0, [&] { return launch_msd_fin_sub(m, fin_grid, c->stream); });
            if (rc) return rc;
            CK(cudaStreamWaitEvent(c->stream, c->ev_split, 0), "split wait");
            if (dbg) {
                cudaStreamSynchronize(c->stream);
                std::vector<uint32_t> h(65536 * 4);
                cudaMemcpy(h.data(), dj, h.size() * 4, cudaMemcpyDeviceToHost);
                std::vector<std::pair<uint32_t, uint32_t>> v;
                uint64_t tot = 0;
                for (uint32_t i = 0; i < 65536; i++)
                    if (h[4 * i]) {
                        v.push_back({h[4 * i + 2], i});
                        tot += h[4 * i + 2];
                    }
                std::sort(v.rbegin(), v.rend());
                fprintf(stderr, "level %u finish: %zu jobs, %.3f Gcycles total; slowest:\n", level, v.size(), tot / 1e9);
                for (size_t q = 0; q < v.size() && q < 12; q++)
                    fprintf(stderr, "   job %u: n %u kw %u L %u  %.1f Mcycles\n", v[q].second, h[4 * v[q].second],
                            h[4 * v[q].second + 1] & 255, h[4 * v[q].second + 1] >> 8, v[q].first / 1e6);
                cudaFree(dj);
                m.dbg_jobs = nullptr;
            }
        }
        if ((rc = msd_read_counters(c, m, nsegs, ntiles))) return rc;   // the level's one host sync
        if (!m.finish_radix) {
            small_done = std::min(c->h_ctr[kQSmall], m.cap_local);
            parts_done = std::min(c->h_ctr[kQParts], m.cap_parts);
            emit_done = std::min(c->h_ctr[kQEmit], m.cap_emit);
        }
        if (getenv("WSORT_DEBUG_MSD")) {
            fprintf(stderr, "msd level %u -> next segs %u tiles %u | tiny %u small %u copy %u parts %u pieces %u\n", level,
                    nsegs, ntiles, c->h_ctr[kQTiny], c->h_ctr[kQSmall], c->h_ctr[kQCopy], c->h_ctr[kQParts], c->h_ctr[kQEmit]);
            std::vector<MsdSeg> jobs(c->h_ctr[kQSmall]);
            cudaMemcpy(jobs.data(), c->m_small.p, jobs.size() * sizeof(MsdSeg), cudaMemcpyDeviceToHost);
            std::vector<uint32_t> sz;
            uint64_t tot = 0;
            for (auto &j : jobs) {
                sz.push_back(j.n);
                tot += j.n;
            }
            std::sort(sz.rbegin(), sz.rend());
            fprintf(stderr, "  jobs so far %zu keys %llu; largest:", sz.size(), (unsigned long long)tot);
            for (size_t i = 0; i < sz.size() && i < 12; i++) fprintf(stderr, " %u", sz[i]);
            uint64_t big = 0;
            for (auto x : sz) big += x > 65536 ? x : 0;
            fprintf(stderr, " | keys in jobs > 64k: %llu\n", (unsigned long long)big);
        }
    }
    m.n_tiny = m.finish_radix ? c->h_ctr[kQTiny] : 0u;   // (streaming: q_tiny held the big jobs, finished)
    const uint32_t n_small = c->h_ctr[kQSmall], n_copy = c->h_ctr[kQCopy];
    return launch(c, "k4m_msd_finish", 0, [&] { return launch_msd_finish(m, n_small, n_copy, max_tw, c->stream); });
}

int emit_keys(wsort_ctx *c, const std::vector<BucketInfo> &bk, const BucketInfo *d_bk, uint32_t lmin, uint32_t lmax,
              double bytes) {
    uint32_t pfx[257], nt = 0;   // tiles of bucket L: [pfx[L], pfx[L+1]); the kernel maps its block to (L, tile)
    for (uint32_t L = 0; L < 256; L++) {
        pfx[L] = nt;
        if (L >= lmin && L <= lmax && bk[L].n) nt += (bk[L].n + kEmitStage / (L + 1) - 1) / (kEmitStage / (L + 1));
    }
    pfx[256] = nt;
    if (!nt) return WSORT_OK;
    int rc;
    if ((rc = arena_upload(c, c->d_tiles, pfx, sizeof pfx, "emit tile prefix"))) return rc;
    EmitArgs ea{};
    ea.buckets = d_bk;
    ea.tile_pfx = static_cast<const uint32_t *>(c->d_tiles.p);
    ea.ntiles = nt;
    ea.keys_a = static_cast<uint32_t *>(c->keys_a.p);
    ea.keys_b = static_cast<uint32_t *>(c->keys_b.p);
    ea.words = static_cast<uint8_t *>(c->words.p);
    ea.global_base = c->global_base;
    return launch(c, "k5_emit", bytes, [&] { return launch_emit(ea, c->stream); });
}

// Buckets of the MSD paths: kw, digits, CTA-sort capacity, scatter tile; the keys of lengths >= lkey
// are laid out contiguously in length order from key word 0.
std::vector<BucketInfo> msd_buckets(const Summary &s, uint32_t lkey, uint32_t &max_tw, uint32_t &levels,
                                    uint64_t &key_words) {
    std::vector<BucketInfo> bk(256, BucketInfo{});
    max_tw = 32;
    levels = 0;
    key_words = 0;
    for (uint32_t L = 1; L <= s.max_len; L++) {
        BucketInfo &b = bk[L];
        b.word_off = s.off[L];
        b.byte_off = s.byte_off[L];
        b.n = (uint32_t)(s.off[L + 1] - s.off[L]);
        b.kw = kw_of(L);
        b.ndig = ndig_of(L);
        // finishing-job capacity: its full-sort fallback holds <= 4096 key words (<= 2048 keys)
        b.tile_keys = b.kw <= 2 ? 2048u : (b.kw <= 4 ? 1024u : (b.kw <= 8 ? 512u : 256u));
        b.aux = kRadixThreads * (32 / b.kw);                          // scatter tile keys
        b.final_b = 1;
        if (L < lkey) continue;
        b.key_off = key_words;
        b.elem_off = b.key_off;
        b.estride = b.kw;
        key_words += (uint64_t)b.n * b.kw;
        max_tw = std::max(max_tw, b.tile_keys * b.kw);
        if (b.n) levels = std::max(levels, b.ndig);
    }
    return bk;
}

// MSD over the key buckets of lengths >= lkey (keys laid out by msd_buckets). `pack` fills buffer A with
// every bucket's keys (K3 from the text, or K3c from the ingest's chunks). Level 0 = whole buckets;
// buckets of at most one CTA tile go straight to the finishing jobs. Ends with the keys emitted.
template <class Pack>
int sort_msd_core(wsort_ctx *c, std::vector<BucketInfo> &bk, uint32_t lkey, uint32_t max_tw, uint32_t levels,
                  uint64_t key_words, uint64_t W, bool finish_radix, Pack pack, const BucketInfo *d_bk_pre = nullptr,
                  bool emit = true, uint32_t lmax_keys = 0, bool from_chunks = false, uint32_t direct_max = 0) {
    const Summary &s = *c->h_sum;
    const uint32_t lmax = lmax_keys ? lmax_keys : s.max_len;
    int rc;
    if ((rc = ensure(c, c->keys_a, key_words * 4 + 64, "keys_a"))) return rc;
    if ((rc = ensure(c, c->keys_b, key_words * 4 + 64, "keys_b"))) return rc;
    MsdArgs m;
    if ((rc = msd_alloc(c, m, W, key_words))) return rc;
    std::vector<MsdSeg> segs, tiny, small;
    std::vector<MsdTile> tiles;
    if (from_chunks) {   // level 0 reads the staging chunks: segment L - lkey = bucket L (every length, in order)
        for (uint32_t L = lkey; L <= lmax; L++) segs.push_back(MsdSeg{L, 0, (uint32_t)bk[L].n, 1});
        // slices of G chunks of one class: about 8 per SM in all (measured 4 / 8 / 16 per SM on c4:
        // count0 0.20 / 0.14 / 0.12 ms, scatter0 0.82 / 0.84 / 0.85 ms)
        uint64_t total = 0;
        for (uint32_t K = 1; K <= kMaxStageKw; K++) total += c->h_ig[kIgClsCnt + K - 1];
        static const uint32_t per_sm = (uint32_t)std::max(1, env_int("WSORT_S0_SLICES_PER_SM", 8));   // (experiments)
        const uint64_t ns = (uint64_t)per_sm * c->sms;
        const uint32_t G = std::max<uint32_t>(2, (uint32_t)((total + ns - 1) / ns));
        m.slice_pfx[0] = m.cls_pfx[0] = 0;
        for (uint32_t K = 1; K <= kMaxStageKw; K++) {
            m.slice_pfx[K] = m.slice_pfx[K - 1] + (c->h_ig[kIgClsCnt + K - 1] + G - 1) / G;
            m.cls_pfx[K] = m.cls_pfx[K - 1] + c->h_ig[kIgClsCnt + K - 1];
        }
        m.chunk_mode = 1;
        m.seg_l0 = lkey;
        m.slice_chunks = G;
        m.nslices = m.slice_pfx[kMaxStageKw];
        m.cls_cap = c->n_chunks;
        m.pool = static_cast<const uint32_t *>(c->pool.p);
        m.chunk_fill = static_cast<const uint32_t *>(c->chunk_fill.p);
        m.cls_list = static_cast<const uint32_t *>(c->cls_list.p);
        m.cls_cnt = static_cast<const uint32_t *>(c->ig_ctr.p) + kIgClsCnt;
        if ((rc = ensure(c, c->slice_hist, (size_t)std::max<uint32_t>(m.nslices, 1) * kC0Bins * 4, "level-0 slice bins")))
            return rc;
        m.slice_hist = static_cast<uint32_t *>(c->slice_hist.p);
    }
    bool may_requeue = false;   // a whole-bucket job larger than a tile (streaming finish: may re-enter the MSD)
    // whole buckets of up to direct_max keys are jobs only if every bucket is (a re-entering job goes to the
    // level-0 segment queue, which must be empty otherwise)
    for (uint32_t L = lkey; L <= lmax && direct_max; L++)
        if (bk[L].n > direct_max) direct_max = 0;
    for (uint32_t L = lkey; L <= lmax && !from_chunks; L++) {
        const BucketInfo &b = bk[L];
        if (!b.n) continue;
        if (b.n <= std::max(b.tile_keys, direct_max)) {
            may_requeue |= b.n > b.tile_keys;
            (finish_radix ? b.n <= 32 : b.n > 16384) ? tiny.push_back(MsdSeg{L, 0, b.n, 1 | kSegWhole}) : small.push_back(MsdSeg{L, 0, b.n, 1 | kSegWhole});
        } else {
            const uint32_t q = (uint32_t)segs.size();
            segs.push_back(MsdSeg{L, 0, b.n, 1});   // packed into buffer A
            for (uint32_t o = 0; o < b.n; o += b.aux) tiles.push_back(MsdTile{q, o, std::min(b.aux, b.n - o), 0});
        }
    }
    const BucketInfo *d_bk = d_bk_pre;
    if (!d_bk) {
        if ((rc = arena_upload(c, c->plan, bk.data(), bk.size() * sizeof(BucketInfo), "plan"))) return rc;
        d_bk = reinterpret_cast<const BucketInfo *>(c->plan.p);
    }
    if ((rc = arena_upload(c, c->m_big[0], segs.data(), segs.size() * sizeof(MsdSeg), "segs0"))) return rc;
    if ((rc = arena_upload(c, c->m_tiles[0], tiles.data(), tiles.size() * sizeof(MsdTile), "tiles0"))) return rc;
    if ((rc = arena_upload(c, c->m_tiny, tiny.data(), tiny.size() * sizeof(MsdSeg), "tiny0"))) return rc;
    if ((rc = arena_upload(c, c->m_small, small.data(), small.size() * sizeof(MsdSeg), "small0"))) return rc;
    uint32_t ctr0[kQCount] = {0, 0, (uint32_t)tiny.size(), (uint32_t)small.size()};
    if ((rc = arena_upload(c, c->m_ctr, ctr0, sizeof ctr0, "counters"))) return rc;
    memcpy(c->h_ctr, ctr0, sizeof ctr0);   // if no level runs, these are the finishing counters
    const double key_bytes = (double)key_words * 4;
    if ((rc = pack(d_bk, key_bytes))) return rc;
    m.buckets = d_bk;
    m.finish_radix = finish_radix ? 1u : 0u;
    m.words = static_cast<uint8_t *>(c->words.p);
    if ((rc = msd_levels_and_finish(c, m, 0, (uint32_t)segs.size(), from_chunks ? m.nslices : (uint32_t)tiles.size(),
                                    levels, key_bytes, max_tw, may_requeue)))
        return rc;
    if (!finish_radix || !emit) return WSORT_OK;   // the streaming finish wrote the text (K5 fused)
    return emit_keys(c, bk, d_bk, lkey, lmax, key_bytes + (double)(s.byte_off[256] - s.byte_off[lkey]));
}

int sort_msd(wsort_ctx *c, bool finish_radix) {
    const Summary &s = *c->h_sum;
    uint32_t max_tw, levels;
    uint64_t key_words;
    std::vector<BucketInfo> bk = msd_buckets(s, 1, max_tw, levels, key_words);
    int rc;
    if ((rc = ensure(c, c->words, s.byte_off[256] + 64, "words"))) return rc;
    return sort_msd_core(c, bk, 1, max_tw, levels, key_words, s.n_words, finish_radix,
                         [&](const BucketInfo *d_bk, double key_bytes) {
                             if (c->packed_pending) return (int)WSORT_OK;
                             TkArgs &tk = c->tk;
                             tk.buckets = d_bk;
                             tk.keys = static_cast<uint32_t *>(c->keys_a.p);
                             tk.payload = nullptr;
                             return launch(c, "k3_pack_scatter", (double)c->n + key_bytes, [&] { return pack_scatter(c); });
                         });
}

// K3c: the ingest's staged keys (chunks) into their length buckets in buffer A (layout of `db`)
int chunk_scatter(wsort_ctx *c, const BucketInfo *db, double key_bytes) {
    int rc;
    if ((rc = ensure(c, c->d_lcursor, 256 * 4, "length cursors"))) return rc;
    CK(cudaMemsetAsync(c->d_lcursor.p, 0, 256 * 4, c->stream), "memset length cursors");
    L0Args la{};
    la.buckets = db;
    la.pool = static_cast<const uint32_t *>(c->pool.p);
    la.chunk_cls = static_cast<const uint32_t *>(c->chunk_cls.p);
    la.chunk_fill = static_cast<const uint32_t *>(c->chunk_fill.p);
    la.lcursor = static_cast<uint32_t *>(c->d_lcursor.p);
    la.dst = static_cast<uint32_t *>(c->keys_a.p);
    la.cta_chunks = c->cta_chunks;
    la.used_chunks = std::min(c->h_ig[kIgMaxChunks], c->cta_chunks);
    return launch(c, "k3c_chunk_scatter", 2 * key_bytes, [&] { return launch_lscatter(la, c->tk.grid, c->stream); });
}

// The dense buckets (L <= 5) on the second stream, beside the MSD of the long ones: scan + compact the
// dense table, then emit bucket L's words bk[L].word_off .. + bk[L].n (global dense word indices) at
// bk[L].byte_off. Records ev_join on the aux stream; the caller joins.
int dense_branch(wsort_ctx *c, const std::vector<BucketInfo> &bk, const BucketInfo *d_bk, double out_bytes) {
    uint32_t dpfx[257], ndt = 0;   // dense emit tiles, bucket by bucket (tile_from_prefix)
    for (uint32_t L = 0; L < 256; L++) {
        dpfx[L] = ndt;
        if (L >= 1 && L <= kDenseMaxLen) ndt += (bk[L].n + dense_tile_words(L) - 1) / dense_tile_words(L);
    }
    dpfx[256] = ndt;
    const uint32_t ne = dense_entries(), nblk = dense_scan_blocks(ne);
    int rc;
    if ((rc = ensure(c, c->d_blk_sum, (size_t)nblk * 4, "dense block sums"))) return rc;
    if ((rc = ensure(c, c->d_blk_nnz, (size_t)nblk * 4, "dense block nnz"))) return rc;
    if ((rc = ensure(c, c->d_ent_idx, (size_t)ne * 4, "dense entries"))) return rc;
    if ((rc = ensure(c, c->d_ent_end, (size_t)ne * 4, "dense entry ends"))) return rc;
    if ((rc = ensure(c, c->d_n_ent, 16, "dense entry count"))) return rc;
    if ((rc = ensure(c, c->d_tile_e, (size_t)2 * (ndt + 1) * 4, "dense tile entries"))) return rc;
    if ((rc = arena_upload(c, c->d_tiles2, dpfx, sizeof dpfx, "dense tile prefix"))) return rc;
    static const bool no_aux = getenv("WSORT_NO_AUX") != nullptr;   // (experiments: serial dense branch)
    if (!c->aux) {
        if (no_aux) c->aux = c->stream;
        else CK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking), "aux stream");
        CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "fork event");
        CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "join event");
    }
    if ((rc = arena_flush(c))) return rc;
    CK(cudaEventRecord(c->ev_fork, c->stream), "fork");
    cudaStream_t aux = c->prof_serial ? c->stream : c->aux;   // (serial profiling: one stream)
    CK(cudaStreamWaitEvent(aux, c->ev_fork, 0), "fork wait");
    DenseArgs da{};
    da.dense = static_cast<const uint32_t *>(c->dense.p);
    da.n_entries = ne;
    da.blk_sum = static_cast<uint32_t *>(c->d_blk_sum.p);
    da.blk_nnz = static_cast<uint32_t *>(c->d_blk_nnz.p);
    da.ent_idx = static_cast<uint32_t *>(c->d_ent_idx.p);
    da.ent_end = static_cast<uint32_t *>(c->d_ent_end.p);
    da.n_ent = static_cast<uint32_t *>(c->d_n_ent.p);
    da.touched = static_cast<const uint8_t *>(c->d_touched.p);
    da.buckets = d_bk;
    da.tile_pfx = static_cast<const uint32_t *>(c->d_tiles2.p);
    da.tile_e0 = static_cast<uint32_t *>(c->d_tile_e.p);
    da.tile_e1 = da.tile_e0 + ndt + 1;
    da.ntiles = ndt;
    rc = launch_on(c, aux, "k2d_dense_scan", 2.0 * ne * 4, [&] { return launch_dense_scan(da, aux); });
    if (rc) return rc;
    DenseEmitArgs ea{};
    ea.buckets = d_bk;
    ea.tile_pfx = static_cast<const uint32_t *>(c->d_tiles2.p);
    ea.ntiles = ndt;
    ea.ent_idx = da.ent_idx;
    ea.ent_end = da.ent_end;
    ea.n_ent = da.n_ent;
    ea.tile_e0 = da.tile_e0;
    ea.tile_e1 = da.tile_e1;
    ea.words = static_cast<uint8_t *>(c->words.p);
    rc = launch_on(c, aux, "k5d_emit_dense", out_bytes, [&] { return launch_emit_dense(ea, aux); });
    if (rc) return rc;
    CK(cudaEventRecord(c->ev_join, aux), "join");
    return WSORT_OK;
}

constexpr uint32_t kSmallJobKeys = 16384, kSmallPathKeys = 1u << 20;
// AUTO (keys only, every word <= 66 letters): the one-pass ingest already counted the words of L <= 5
// (dense tables) and staged the longer ones as keys in per-length chunks. Dense buckets: scan + compact +
// emit. Long buckets: the MSD's first level counts and scatters the chunks in place (chunk mode), then the
// streaming finish.
int sort_dense_msd(wsort_ctx *c) {
    const Summary &s = *c->h_sum;
    uint32_t max_tw, levels;
    uint64_t key_words;
    std::vector<BucketInfo> bk = msd_buckets(s, kDenseMaxLen + 1, max_tw, levels, key_words);
    const uint64_t W = s.n_words, n_dense = s.off[kDenseMaxLen + 1];
    int rc;
    if ((rc = ensure(c, c->words, s.byte_off[256] + 64, "words"))) return rc;
    if ((rc = arena_upload(c, c->plan, bk.data(), bk.size() * sizeof(BucketInfo), "plan"))) return rc;
    const BucketInfo *d_bk = reinterpret_cast<const BucketInfo *>(c->plan.p);
    if (n_dense && (rc = dense_branch(c, bk, d_bk, (double)s.byte_off[kDenseMaxLen + 1]))) return rc;
    if (W > n_dense) {
        // the MSD of the long words is the critical path: it runs on a high-priority stream, so the block
        // scheduler gives the dense branch (default priority) only the SMs the MSD leaves idle
        static const bool no_hp = getenv("WSORT_NO_HP") != nullptr;   // (experiments)
        const bool use_hp = n_dense && !c->prof_serial && !no_hp;
        cudaStream_t user = c->stream;
        if (use_hp) {
            if (!c->hp) {
                int least = 0, greatest = 0;
                CK(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
                CK(cudaStreamCreateWithPriority(&c->hp, cudaStreamNonBlocking, greatest), "high-priority stream");
                CK(cudaEventCreateWithFlags(&c->ev_hp0, cudaEventDisableTiming), "hp event");
                CK(cudaEventCreateWithFlags(&c->ev_hp1, cudaEventDisableTiming), "hp event");
            }
            if ((rc = arena_flush(c))) return rc;
            CK(cudaEventRecord(c->ev_hp0, user), "hp fork");
            CK(cudaStreamWaitEvent(c->hp, c->ev_hp0, 0), "hp fork wait");
            c->stream = c->hp;
        }
        // small texts (every long bucket one finishing job of <= 16 K keys, <= 1 M long words): the staged keys
        // regrouped by length (K3c) and each bucket finished as one job — no level-0 count / plan / scatter
        // launches (latency-bound sizes; with a bucket of more keys the level-0 chunk path is faster: c2
        // 0.27 vs 0.36 ms through the per-bucket MSD)
        uint32_t max_n = 0;
        for (uint32_t L = kDenseMaxLen + 1; L <= s.max_len; L++) max_n = std::max<uint32_t>(max_n, bk[L].n);
        const bool small = max_n <= kSmallJobKeys && W - n_dense <= kSmallPathKeys && !getenv("WSORT_NO_SMALL");
        if (small)
            rc = sort_msd_core(c, bk, kDenseMaxLen + 1, max_tw, levels, key_words, W - n_dense, false,
                               [&](const BucketInfo *db, double kb) { return chunk_scatter(c, db, kb); }, d_bk, true, 0,
                               false, kSmallJobKeys);
        else
            rc = sort_msd_core(c, bk, kDenseMaxLen + 1, max_tw, levels, key_words, W - n_dense, false,
                               [&](const BucketInfo *, double) { return (int)WSORT_OK; }, d_bk, true, 0, true);
        if (use_hp) {
            const int rf = arena_flush(c);   // (on the high-priority stream)
            if (!rc) rc = rf;
            c->stream = user;
            const cudaError_t e0 = cudaEventRecord(c->ev_hp1, c->hp);
            const cudaError_t e1 = e0 == cudaSuccess ? cudaStreamWaitEvent(user, c->ev_hp1, 0) : e0;
            if (!rc && e1 != cudaSuccess) return cuda_err(c, e1, "hp join");
        }
    }
    if (n_dense) {   // join: the sort is complete when both streams are
        const cudaError_t e = cudaStreamWaitEvent(c->stream, c->ev_join, 0);
        if (!rc && e != cudaSuccess) return cuda_err(c, e, "join wait");
    }
    return rc;
}

// The distinct keys of > 66 letters are ranked in shared memory (k_sort_wide): every such bucket must fit.
bool hash_sortable(const wsort_ctx *c) {
    for (uint32_t L = kMsdMaxLen + 1; L <= c->h_sum->max_len; L++)
        if ((uint64_t)c->h_tab[4 + L] * kw_of((int)L) > kWideSortWords) return false;
    return true;
}

// AUTO after a hash-mode tokenize (every word <= 255 letters): dense buckets as in sort_dense_msd; the long
// words from the table of distinct words: gather the D distinct keys into their length buckets, sort them
// (MSD, radix finish: keys end in buffer B), look up each one's count, scan, and write the runs.
void summary_from_counts(Summary &s, const uint64_t *n_per_len);
std::vector<BucketInfo> bucket_table(const Summary &s);

// The long words (>= 6 letters) of the table of distinct words (c->tab, its distinct counts per length in
// c->h_tab + 4) into the output buckets bk / d_bk (bk[L].n words at bk[L].byte_off; the run index of
// bk[L]'s first word is bk[L].word_off - long_base): gather the D distinct keys into their length buckets,
// sort them (MSD, radix finish, keys end in buffer B; > 66 letters: k_sort_wide), look up each one's count,
// scan, and write the runs.
int long_from_table(wsort_ctx *c, const std::vector<BucketInfo> &bk, const BucketInfo *d_bk, uint64_t long_base) {
    const uint32_t *dcount = c->h_tab + 4;
    Summary ks = *c->h_sum;
    std::vector<uint64_t> nd(256, 0);
    uint32_t dpfx[257], rpfx[257], D = 0, ntiles = 0, lmax_d = 0;
    for (uint32_t L = 0; L < 256; L++) {
        dpfx[L] = D;
        rpfx[L] = ntiles;
        if (L > kDenseMaxLen && dcount[L]) {
            nd[L] = dcount[L];
            D += dcount[L];
            lmax_d = L;
            ntiles += (bk[L].n + run_tile_words(L) - 1) / run_tile_words(L);
        }
    }
    dpfx[256] = D;
    rpfx[256] = ntiles;
    if (!D) return WSORT_OK;
    int rc;
    summary_from_counts(ks, nd.data());   // (only the distinct keys' sizes are used)
    uint32_t kmax_tw, klevels;
    uint64_t kkey_words;
    std::vector<BucketInfo> kb = msd_buckets(ks, kDenseMaxLen + 1, kmax_tw, klevels, kkey_words);
    if ((rc = ensure(c, c->t_runend, (size_t)D * 4, "run ends"))) return rc;
    if ((rc = ensure(c, c->t_scan, (size_t)hash_scan_blocks(D) * 4, "run scan"))) return rc;
    if ((rc = ensure(c, c->t_tilee, (size_t)2 * (ntiles + 1) * 4, "run tiles"))) return rc;
    if ((rc = ensure(c, c->d_lcursor, 256 * 4, "length cursors"))) return rc;
    if ((rc = arena_upload(c, c->t_kplan, kb.data(), kb.size() * sizeof(BucketInfo), "key plan"))) return rc;
    if ((rc = arena_upload(c, c->t_dpfx, dpfx, sizeof dpfx, "distinct prefix"))) return rc;
    if ((rc = arena_upload(c, c->t_rpfx, rpfx, sizeof rpfx, "run tile prefix"))) return rc;
    const BucketInfo *d_kb = reinterpret_cast<const BucketInfo *>(c->t_kplan.p);
    std::vector<uint32_t> wide_lens;   // buckets of > 66 letters: k_sort_wide (hash_sortable checked the sizes)
    for (uint32_t L = kMsdMaxLen + 1; L <= lmax_d; L++)
        if (kb[L].n) wide_lens.push_back(L);
    if ((rc = arena_upload(c, c->t_wlens, wide_lens.data(), wide_lens.size() * 4, "wide lengths"))) return rc;
    rc = sort_msd_core(c, kb, kDenseMaxLen + 1, kmax_tw, klevels, kkey_words, D, true,
                       [&](const BucketInfo *db, double kbytes) {
                           CK(cudaMemsetAsync(c->d_lcursor.p, 0, 256 * 4, c->stream), "memset length cursors");
                           HashGatherArgs ga{};
                           ga.tab = c->tab;
                           ga.buckets = db;
                           ga.lcursor = static_cast<uint32_t *>(c->d_lcursor.p);
                           ga.keys_a = static_cast<uint32_t *>(c->keys_a.p);
                           return launch(c, "kh1_hash_gather", kbytes, [&] { return launch_hash_gather(ga, c->stream); });
                       },
                       d_kb, false, std::min<uint32_t>(lmax_d, kMsdMaxLen));
    if (rc) return rc;
    rc = launch(c, "kh1b_sort_wide", 0, [&] {
        return launch_sort_wide(d_kb, static_cast<const uint32_t *>(c->t_wlens.p), (uint32_t)wide_lens.size(),
                                static_cast<const uint32_t *>(c->keys_a.p), static_cast<uint32_t *>(c->keys_b.p), c->stream);
    });
    if (rc) return rc;
    HashRunArgs ra{};
    ra.tab = c->tab;
    ra.buckets = d_bk;
    ra.kbuckets = d_kb;
    ra.dist_pfx = static_cast<const uint32_t *>(c->t_dpfx.p);
    ra.D = D;
    ra.keys = static_cast<const uint32_t *>(c->keys_b.p);
    ra.run_end = static_cast<uint32_t *>(c->t_runend.p);
    ra.long_base = long_base;
    ra.tile_pfx = static_cast<const uint32_t *>(c->t_rpfx.p);
    ra.ntiles = ntiles;
    ra.tile_e0 = static_cast<uint32_t *>(c->t_tilee.p);
    ra.tile_e1 = ra.tile_e0 + ntiles + 1;
    ra.words = static_cast<uint8_t *>(c->words.p);
    rc = launch(c, "kh2_hash_runs", (double)D * 8, [&] { return launch_hash_runs(ra, static_cast<uint32_t *>(c->t_scan.p), c->stream); });
    if (rc) return rc;
    double out_bytes = 0;
    for (uint32_t L = kDenseMaxLen + 1; L < 256; L++) out_bytes += (double)bk[L].n * (L + 1);
    return launch(c, "kh5_emit_runs", out_bytes, [&] { return launch_emit_runs(ra, c->stream); });
}

// AUTO after a hash-mode tokenize: dense buckets as in sort_dense_msd, the long words from the table.
int sort_dense_hash(wsort_ctx *c) {
    const Summary &s = *c->h_sum;
    uint32_t max_tw, levels;
    uint64_t key_words;
    std::vector<BucketInfo> bk = msd_buckets(s, kDenseMaxLen + 1, max_tw, levels, key_words);
    const uint64_t n_dense = s.off[kDenseMaxLen + 1];
    int rc;
    if ((rc = ensure(c, c->words, s.byte_off[256] + 64, "words"))) return rc;
    if ((rc = arena_upload(c, c->plan, bk.data(), bk.size() * sizeof(BucketInfo), "plan"))) return rc;
    const BucketInfo *d_bk = reinterpret_cast<const BucketInfo *>(c->plan.p);
    if (n_dense && (rc = dense_branch(c, bk, d_bk, (double)s.byte_off[kDenseMaxLen + 1]))) return rc;
    rc = long_from_table(c, bk, d_bk, s.off[kDenseMaxLen + 1]);
    if (n_dense) {   // join: the sort is complete when both streams are
        const cudaError_t e = cudaStreamWaitEvent(c->stream, c->ev_join, 0);
        if (!rc && e != cudaSuccess) return cuda_err(c, e, "join wait");
    }
    return rc;
}

// ------------------------------------------------------------------ multi-GPU with an attached communicator
// The host logic between the collectives; the kernels are in k_xchg.cu. Every rank runs the same sequence
// of collectives, errors included (a failing rank still takes part in the error all-reduce).

// wsort_tokenize while attached: K1 on the shard (counting ingest), then one all-reduce of
// [histogram 0..256 | table overflow | error | distinct words per length]; overflow on any rank -> every
// rank counts again with a bigger table.
int tokenize_dist(wsort_ctx *c, uint64_t *n_words) {
    Comm &m = *c->comm;
    constexpr int kV = 257 + 2 + 256;
    int rc;
    if ((rc = ensure(c, c->x_vec, kV * 8, "dist vector"))) return rc;
    std::vector<uint64_t> v(kV);
    for (;;) {
        const int lrc = tokenize_impl(c, nullptr, true);
        std::fill(v.begin(), v.end(), 0ull);
        if (lrc == WSORT_OK || lrc == WSORT_E_WORD_TOO_LONG) {
            const Summary &s = *c->h_sum;
            for (uint32_t L = 0; L < 256; L++) v[L] = s.off[L + 1] - s.off[L];
            v[256] = s.too_long;
            v[257] = c->hashed ? c->h_tab[hashtab::kTopOverflow] != 0 : 1u;
            for (uint32_t L = 0; L < 256 && c->hashed; L++) v[259 + L] = c->h_tab[4 + L];
        } else {
            v[258] = 1;
        }
        CK(cudaMemcpyAsync(c->x_vec.p, v.data(), kV * 8, cudaMemcpyHostToDevice, c->stream), "dist vector");
        if ((rc = m.allreduce_u64(static_cast<uint64_t *>(c->x_vec.p), kV, c->stream)))
            return set_err(c, rc, "tokenize all-reduce: %s", m.err.c_str());
        CK(cudaMemcpyAsync(v.data(), c->x_vec.p, kV * 8, cudaMemcpyDeviceToHost, c->stream), "dist vector");
        CK(cudaStreamSynchronize(c->stream), "dist tokenize");
        if (v[258]) return lrc ? lrc : set_err(c, WSORT_E_NCCL, "tokenize failed on another rank");
        if (v[256]) {
            c->state = ST_LOADED;
            return set_err(c, WSORT_E_WORD_TOO_LONG, "%llu word(s) longer than %d letters (all ranks)",
                           (unsigned long long)v[256], kMaxLen);
        }
        if (!v[257]) break;
        if (c->hash_grow >= 64)
            return set_err(c, WSORT_E_NOMEM, "table of distinct words overflowed on some rank (multi-GPU needs it)");
        c->hash_grow *= 4;
    }
    uint64_t W = 0;
    c->g_lmax = 0;
    for (uint32_t L = 0; L < 256; L++) {
        c->g_hist[L] = v[L];
        c->g_dcount[L] = v[259 + L];
        W += v[L];
        if (v[L]) c->g_lmax = L;
    }
    c->g_hist[256] = 0;
    for (uint32_t L = kMsdMaxLen + 1; L <= c->g_lmax; L++)
        if (c->g_dcount[L] * kw_of((int)L) > kWideSortWords)
            return set_err(c, WSORT_E_NOMEM, "multi-GPU: %llu distinct words of %u letters exceed the wide-key sort",
                           (unsigned long long)c->g_dcount[L], L);
    if (n_words) *n_words = W;
    c->state = ST_TOKENIZED;
    return WSORT_OK;
}

// wsort_sort while attached (AUTO): see include/wsort.h.
int sort_dist(wsort_ctx *c) {
    Comm &m = *c->comm;
    const uint32_t P = (uint32_t)m.size, me = (uint32_t)m.rank;
    int rc;
    auto comm_fail = [&](int code, const char *what) { return set_err(c, code, "%s: %s", what, m.err.c_str()); };
    // (1) dense: the summed tables; this rank's share of the global dense words
    if ((rc = m.allreduce_u32(static_cast<uint32_t *>(c->dense.p), dense_entries(), c->stream)))
        return comm_fail(rc, "dense all-reduce");
    // (other ranks' words: every block may be non-zero now)
    CK(cudaMemsetAsync(c->d_touched.p, 1, dense_scan_blocks(dense_entries()), c->stream), "touched");
    uint64_t Wd = 0;
    for (uint32_t L = 1; L <= kDenseMaxLen; L++) Wd += c->g_hist[L];
    const uint64_t dlo = me * Wd / P, dhi = (me + 1) * Wd / P;
    uint64_t dslice_off[kDenseMaxLen + 1] = {0}, dslice_n[kDenseMaxLen + 1] = {0}, g = 0, dbytes = 0, gdbytes = 0,
             dbyte_base = 0;
    for (uint32_t L = 1; L <= kDenseMaxLen; L++) {
        const uint64_t a = std::max(g, dlo), b = std::min(g + c->g_hist[L], dhi);
        dslice_off[L] = a;
        dslice_n[L] = b > a ? b - a : 0;
        if (dlo > g) dbyte_base += (std::min(dlo, g + c->g_hist[L]) - g) * (L + 1);
        g += c->g_hist[L];
        dbytes += dslice_n[L] * (L + 1);
        gdbytes += c->g_hist[L] * (L + 1);
    }
    // (2) this rank's distinct long words: gathered (keys_a), counted, prefix of the counts
    const uint32_t *dcount = c->h_tab + 4;
    Summary ks = *c->h_sum;
    std::vector<uint64_t> nd(256, 0);
    uint32_t dpfx[257], D = 0;
    for (uint32_t L = 0; L < 256; L++) {
        dpfx[L] = D;
        if (L > kDenseMaxLen) {
            nd[L] = dcount[L];
            D += dcount[L];
        }
    }
    dpfx[256] = D;
    summary_from_counts(ks, nd.data());
    uint32_t kmax_tw, klevels;
    uint64_t kkey_words;
    std::vector<BucketInfo> kb = msd_buckets(ks, kDenseMaxLen + 1, kmax_tw, klevels, kkey_words);
    uint64_t gD = 0;
    for (uint32_t L = 0; L < 256; L++) gD += c->g_dcount[L];
    const uint32_t kwx = kw_of((int)std::max<uint32_t>(c->g_lmax, 1)), rec = 3 + kwx;
    const uint32_t ns = std::max<uint32_t>(1, std::min<uint32_t>(1024, 16384 / P)), nall = ns * P;
    if ((rc = ensure(c, c->keys_a, kkey_words * 4 + 64, "keys_a"))) return rc;
    if ((rc = ensure(c, c->d_lcursor, 256 * 4, "length cursors"))) return rc;
    if ((rc = ensure(c, c->x_counts, (size_t)D * 4 + 16, "xchg counts"))) return rc;
    if ((rc = ensure(c, c->x_prefix, (size_t)D * 4 + 16, "xchg prefix"))) return rc;
    if ((rc = ensure(c, c->t_scan, (size_t)hash_scan_blocks(D + 1) * 4, "scan"))) return rc;
    if ((rc = ensure(c, c->x_samples, (size_t)ns * rec * 4, "xchg samples"))) return rc;
    if ((rc = ensure(c, c->x_all, (size_t)nall * rec * 4, "xchg all samples"))) return rc;
    if ((rc = ensure(c, c->x_order, (size_t)nall * 4, "xchg order"))) return rc;
    if ((rc = ensure(c, c->x_split, (size_t)P * rec * 4, "xchg splitters"))) return rc;
    if ((rc = ensure(c, c->x_dest, (size_t)D + 16, "xchg destinations"))) return rc;
    if ((rc = ensure(c, c->x_send, kMaxRanks * 4, "xchg send counts"))) return rc;
    if ((rc = ensure(c, c->x_matrix, (size_t)P * kMaxRanks * 4, "xchg matrix"))) return rc;
    if ((rc = ensure(c, c->x_cursor, kMaxRanks * 4, "xchg cursors"))) return rc;
    if ((rc = ensure(c, c->x_recvn, 16, "xchg received"))) return rc;
    if ((rc = ensure(c, c->x_win, (size_t)(gD + 1) * rec * 4, "xchg window"))) return rc;
    if ((rc = ensure(c, c->x_peers, kMaxRanks * sizeof(void *), "xchg peers"))) return rc;
    if ((rc = ensure(c, c->x_flag, 16, "xchg flag"))) return rc;
    if ((rc = ensure(c, c->x_lwords, 256 * 8, "xchg length words"))) return rc;
    if ((rc = ensure(c, c->x_lwords_all, (size_t)P * 256 * 8, "xchg all length words"))) return rc;
    if ((rc = arena_upload(c, c->t_kplan, kb.data(), kb.size() * sizeof(BucketInfo), "key plan"))) return rc;
    if ((rc = arena_upload(c, c->t_dpfx, dpfx, sizeof dpfx, "distinct prefix"))) return rc;
    const BucketInfo *d_kb = reinterpret_cast<const BucketInfo *>(c->t_kplan.p);
    CK(cudaMemsetAsync(c->d_lcursor.p, 0, 256 * 4, c->stream), "memset length cursors");
    HashGatherArgs ga{};
    ga.tab = c->tab;
    ga.buckets = d_kb;
    ga.lcursor = static_cast<uint32_t *>(c->d_lcursor.p);
    ga.keys_a = static_cast<uint32_t *>(c->keys_a.p);
    if ((rc = launch(c, "kh1_hash_gather", (double)kkey_words * 4, [&] { return launch_hash_gather(ga, c->stream); })))
        return rc;
    HashRunArgs ra{};
    ra.tab = c->tab;
    ra.kbuckets = d_kb;
    ra.dist_pfx = static_cast<const uint32_t *>(c->t_dpfx.p);
    ra.D = D;
    ra.keys = static_cast<const uint32_t *>(c->keys_a.p);
    ra.run_end = static_cast<uint32_t *>(c->x_counts.p);
    if ((rc = launch(c, "kx0_counts", (double)D * 4, [&] { return launch_hash_counts(ra, c->stream); }))) return rc;
    if (D) CK(cudaMemcpyAsync(c->x_prefix.p, c->x_counts.p, (size_t)D * 4, cudaMemcpyDeviceToDevice, c->stream), "prefix");
    if ((rc = launch(c, "kx0_prefix", (double)D * 8, [&] {
             return launch_scan_u32(static_cast<uint32_t *>(c->x_prefix.p), D, static_cast<uint32_t *>(c->t_scan.p), c->stream);
         })))
        return rc;
    // (3) samples -> all-gather -> identical splitters on every rank
    XchgArgs xa{};
    xa.kbuckets = d_kb;
    xa.dist_pfx = static_cast<const uint32_t *>(c->t_dpfx.p);
    xa.keys = static_cast<const uint32_t *>(c->keys_a.p);
    xa.D = D;
    xa.counts = static_cast<const uint32_t *>(c->x_counts.p);
    xa.prefix = static_cast<const uint32_t *>(c->x_prefix.p);
    xa.rank = me;
    xa.nparts = P;
    xa.rec_words = rec;
    xa.nsamples = ns;
    xa.nall = nall;
    xa.samples = static_cast<uint32_t *>(c->x_samples.p);
    xa.all_samples = static_cast<const uint32_t *>(c->x_all.p);
    xa.order = static_cast<uint32_t *>(c->x_order.p);
    xa.splitters = static_cast<uint32_t *>(c->x_split.p);
    xa.dest = static_cast<uint8_t *>(c->x_dest.p);
    xa.send_counts = static_cast<uint32_t *>(c->x_send.p);
    xa.matrix = static_cast<const uint32_t *>(c->x_matrix.p);
    xa.cursor = static_cast<uint32_t *>(c->x_cursor.p);
    xa.recv_n = static_cast<uint32_t *>(c->x_recvn.p);
    xa.win = static_cast<uint32_t *>(c->x_win.p);
    xa.win_cap = gD + 1;
    xa.flag = static_cast<uint32_t *>(c->x_flag.p);
    xa.lwords = static_cast<unsigned long long *>(c->x_lwords.p);
    if ((rc = launch(c, "kx1_sample", 0, [&] { return launch_xchg_sample(xa, c->stream); }))) return rc;
    if ((rc = m.allgather(c->x_samples.p, c->x_all.p, (size_t)ns * rec * 4, c->stream))) return comm_fail(rc, "sample all-gather");
    CK(cudaMemsetAsync(c->x_split.p, 0, (size_t)P * rec * 4, c->stream), "memset splitters");
    if ((rc = launch(c, "kx2_splitters", 0, [&] { return launch_xchg_split(xa, c->stream); }))) return rc;
    // (4) destinations and the count matrix; the receive windows of every rank
    CK(cudaMemsetAsync(c->x_send.p, 0, kMaxRanks * 4, c->stream), "memset send counts");
    CK(cudaMemsetAsync(c->x_flag.p, 0, 16, c->stream), "memset flag");
    if ((rc = launch(c, "kx4_count", 0, [&] { return launch_xchg_count(xa, c->stream); }))) return rc;
    if ((rc = m.allgather(c->x_send.p, c->x_matrix.p, (size_t)P * 4, c->stream))) return comm_fail(rc, "count all-gather");
    std::vector<void *> peers;
    if ((rc = m.peer_windows(c->x_win.p, c->x_win.cap, peers, c->stream))) return comm_fail(rc, "peer windows");
    CK(cudaMemcpyAsync(c->x_peers.p, peers.data(), P * sizeof(void *), cudaMemcpyHostToDevice, c->stream), "peers");
    CK(cudaStreamSynchronize(c->stream), "peers");   // (the host vector is local)
    xa.peer_win = static_cast<uint32_t *const *>(c->x_peers.p);
    // (5) every record stored into its owner's window (P2P), then a barrier
    if ((rc = launch(c, "kx5_write", (double)D * rec * 4, [&] { return launch_xchg_write(xa, c->stream); }))) return rc;
    if ((rc = m.barrier(c->stream))) return comm_fail(rc, "exchange barrier");
    // (6) the received records counted into this rank's table (cleared, sized for every rank's words)
    uint64_t need_n = 0, need_w = 0;
    for (uint32_t L = kDenseMaxLen + 1; L < 256; L++) (L <= 24 ? need_n : need_w) += c->g_dcount[L];
    if ((rc = hash_alloc(c, need_n, need_w))) return rc;
    xa.tab = c->tab;
    CK(cudaMemsetAsync(c->x_lwords.p, 0, 256 * 8, c->stream), "memset length words");
    if ((rc = launch(c, "kx6_absorb", 0, [&] { return launch_xchg_absorb(xa, (uint32_t)c->sms * 4, c->stream); })))
        return rc;
    if ((rc = m.allgather(c->x_lwords.p, c->x_lwords_all.p, 256 * 8, c->stream))) return comm_fail(rc, "length all-gather");
    std::vector<uint64_t> lw((size_t)P * 256);
    uint32_t xflag = 0;
    CK(copy_small(c->h_tab, c->t_top.p, 16, c->stream), "copy hash top");
    CK(copy_small(c->h_tab + 4, c->t_dcount.p, 256 * 4, c->stream), "copy hash distinct counts");
    CK(cudaMemcpyAsync(lw.data(), c->x_lwords_all.p, lw.size() * 8, cudaMemcpyDeviceToHost, c->stream), "length words");
    CK(cudaMemcpyAsync(&xflag, c->x_flag.p, 4, cudaMemcpyDeviceToHost, c->stream), "flag");
    CK(cudaStreamSynchronize(c->stream), "dist sort");
    if (xflag || c->h_tab[hashtab::kTopOverflow])   // (never expected: the windows and table hold every word)
        return set_err(c, WSORT_E_NOMEM, "multi-GPU exchange overflow (window %u, table %u)", xflag, c->h_tab[hashtab::kTopOverflow]);
    // (7) this rank's output: its dense slice, then its long slice (its (length, word) range)
    std::vector<uint64_t> nl(256, 0);
    uint64_t lbytes_before = 0, lwords_before = 0;
    for (uint32_t r = 0; r < P; r++)
        for (uint32_t L = kDenseMaxLen + 1; L < 256; L++) {
            const uint64_t x = lw[(size_t)r * 256 + L];
            if (r == me) nl[L] = x;
            if (r < me) {
                lbytes_before += x * (L + 1);
                lwords_before += x;
            }
        }
    std::vector<BucketInfo> bk(256, BucketInfo{});
    uint64_t lo = 0, bo = dbytes;
    for (uint32_t L = 1; L < 256; L++) {
        BucketInfo &b = bk[L];
        b.kw = kw_of((int)L);
        if (L <= kDenseMaxLen) {
            b.word_off = dslice_off[L];
            b.n = (uint32_t)dslice_n[L];
        } else {
            b.word_off = lo;
            b.n = (uint32_t)nl[L];
            lo += nl[L];
        }
        b.byte_off = L <= kDenseMaxLen ? 0 : bo;
        if (L > kDenseMaxLen) bo += nl[L] * (L + 1);
    }
    uint64_t db = 0;   // dense byte offsets inside the dense slice
    for (uint32_t L = 1; L <= kDenseMaxLen; L++) {
        bk[L].byte_off = db;
        db += dslice_n[L] * (L + 1);
    }
    if ((rc = ensure(c, c->words, bo + 64, "words"))) return rc;
    if ((rc = arena_upload(c, c->plan, bk.data(), bk.size() * sizeof(BucketInfo), "plan"))) return rc;
    const BucketInfo *d_bk = reinterpret_cast<const BucketInfo *>(c->plan.p);
    const bool dense = dhi > dlo;
    if (dense && (rc = dense_branch(c, bk, d_bk, (double)dbytes))) return rc;
    summary_from_counts(*c->h_sum, nl.data());   // (long_from_table and wsort_fetch: this rank's long slice)
    rc = long_from_table(c, bk, d_bk, 0);
    if (dense) {
        const cudaError_t e = cudaStreamWaitEvent(c->stream, c->ev_join, 0);
        if (!rc && e != cudaSuccess) return cuda_err(c, e, "join wait");
    }
    if (rc) return rc;
    // wsort_fetch: this rank's words = dense slice + long slice; the global bucket offsets
    c->slice_words = dhi - dlo;
    c->slice_bytes = dbytes;
    c->has_global = true;
    uint64_t o = 0;
    c->gmax = c->g_lmax;
    for (int L = 0; L < 256; L++) {
        c->goff[L] = o;
        o += L ? c->g_hist[L] : 0;
    }
    c->goff[256] = o;
    c->goff[c->gmax + 1] = o;
    c->word_base = dlo;
    c->byte_base = dbyte_base;
    c->slices.clear();
    c->slices.push_back(wsort_slice{0, dbytes, dhi - dlo, dbyte_base, dlo});
    c->slices.push_back(wsort_slice{dbytes, bo - dbytes, lo, gdbytes + lbytes_before, Wd + lwords_before});
    return WSORT_OK;
}

// WSORT_ALGO_RAGGED: K3 writes each word's text offset into its bucket (stable), the references are sorted
// through the text (k_ragged.cu), and the words are copied out of the text.
int sort_ragged(wsort_ctx *c, bool want_src) {
    const Summary &s = *c->h_sum;
    const uint64_t W = s.n_words;
    int rc;
    std::vector<BucketInfo> bk = bucket_table(s);
    if ((rc = ensure(c, c->keys_a, s.key_off[256] * 4 + 64, "keys_a"))) return rc;
    if ((rc = ensure(c, c->pay_a, W * 4 + 64, "pay_a"))) return rc;
    if ((rc = ensure(c, c->pay_b, W * 4 + 64, "pay_b"))) return rc;
    if ((rc = ensure(c, c->words, s.byte_off[256] + 64, "words"))) return rc;
    if (want_src && (rc = ensure(c, c->src_off, W * 8 + 64, "src_off"))) return rc;
    uint32_t pfx[257], nt = 0, nmax = 0;
    const uint32_t T = ragged_tile();
    for (uint32_t L = 0; L < 256; L++) {
        pfx[L] = nt;
        if (L >= 1 && bk[L].n) nt += (bk[L].n + T - 1) / T;
        nmax = std::max(nmax, bk[L].n);
    }
    pfx[256] = nt;
    if ((rc = arena_upload(c, c->plan, bk.data(), bk.size() * sizeof(BucketInfo), "plan"))) return rc;
    if ((rc = arena_upload(c, c->d_tiles, pfx, sizeof pfx, "ragged tiles"))) return rc;
    const BucketInfo *d_bk = reinterpret_cast<const BucketInfo *>(c->plan.p);
    TkArgs &tk = c->tk;
    tk.buckets = d_bk;
    tk.keys = static_cast<uint32_t *>(c->keys_a.p);
    tk.payload = static_cast<uint32_t *>(c->pay_a.p);
    if ((rc = launch(c, "k3_pack_scatter", (double)c->n + 4.0 * W, [&] { return pack_scatter(c); }))) return rc;
    RaggedArgs ra{};
    ra.text = c->d_text;
    ra.buckets = d_bk;
    ra.tile_pfx = static_cast<const uint32_t *>(c->d_tiles.p);
    ra.ntiles = nt;
    ra.in = static_cast<const uint32_t *>(c->pay_a.p);
    ra.out = static_cast<uint32_t *>(c->pay_b.p);
    ra.words = static_cast<uint8_t *>(c->words.p);
    ra.src_off = want_src ? static_cast<uint64_t *>(c->src_off.p) : nullptr;
    ra.global_base = c->global_base;
    if ((rc = launch(c, "kr1_ragged_tiles", 8.0 * W, [&] { return launch_ragged_tiles(ra, c->stream); }))) return rc;
    uint32_t *x = static_cast<uint32_t *>(c->pay_b.p), *y = static_cast<uint32_t *>(c->pay_a.p);   // sorted runs in x
    for (uint32_t run = T; run < nmax; run *= 2) {
        ra.in = x;
        ra.out = y;
        ra.run = run;
        if ((rc = launch(c, "kr2_ragged_merge", 8.0 * W, [&] { return launch_ragged_merge(ra, c->stream); }))) return rc;
        std::swap(x, y);
    }
    ra.in = x;
    return launch(c, "kr3_ragged_emit", (double)s.byte_off[256] + 4.0 * W, [&] { return launch_ragged_emit(ra, c->stream); });
}

// Split multi-GPU sort (after wsort_pack_long, the all-reduce of the dense tables, wsort_load_keys and
// wsort_dense_range): this rank's slice of the global dense words, then the keys it received, sorted.
int sort_dist_dense(wsort_ctx *c) {
    const Summary &s = *c->h_sum;   // the received keys (lengths >= 6 only)
    uint32_t max_tw, levels;
    uint64_t key_words;
    std::vector<BucketInfo> bk = msd_buckets(s, kDenseMaxLen + 1, max_tw, levels, key_words);
    uint64_t dbytes = 0;
    for (uint32_t L = 1; L <= kDenseMaxLen; L++) {
        BucketInfo &b = bk[L];
        b = BucketInfo{};
        b.word_off = c->dslice_off[L];
        b.n = (uint32_t)c->dslice_n[L];
        b.byte_off = dbytes;
        b.kw = 1;
        dbytes += c->dslice_n[L] * (L + 1);
    }
    for (uint32_t L = kDenseMaxLen + 1; L < 256; L++) bk[L].byte_off += dbytes;
    int rc;
    if ((rc = ensure(c, c->words, dbytes + s.byte_off[256] + 64, "words"))) return rc;
    if ((rc = arena_upload(c, c->plan, bk.data(), bk.size() * sizeof(BucketInfo), "plan"))) return rc;
    const BucketInfo *d_bk = reinterpret_cast<const BucketInfo *>(c->plan.p);
    const bool dense = c->slice_words != 0;
    if (dense && (rc = dense_branch(c, bk, d_bk, (double)dbytes))) return rc;
    if (s.n_words)
        rc = sort_msd_core(c, bk, kDenseMaxLen + 1, max_tw, levels, key_words, s.n_words, false,
                           [&](const BucketInfo *, double) { return (int)WSORT_OK; },   // keys_a: wsort_load_keys
                           d_bk);
    if (dense) {
        const cudaError_t e = cudaStreamWaitEvent(c->stream, c->ev_join, 0);
        if (!rc && e != cudaSuccess) return cuda_err(c, e, "join wait");
    }
    return rc;
}

}  // namespace

extern "C" {

int wsort_sort(wsort_ctx *c, int algo, unsigned flags) {
    if (!c) return WSORT_E_INVALID_ARG;
    if (c->state < ST_TOKENIZED) return set_err(c, WSORT_E_STATE, "wsort_sort before wsort_tokenize");
    if (algo != WSORT_ALGO_AUTO && algo != WSORT_ALGO_LSD_RADIX && algo != WSORT_ALGO_OETS_MERGE &&
        algo != WSORT_ALGO_MSD_RADIX && algo != WSORT_ALGO_MSD_OETS && algo != WSORT_ALGO_DENSE_MSD &&
        algo != WSORT_ALGO_RAGGED)
        return set_err(c, WSORT_E_INVALID_ARG, "bad algo %d", algo);
    if (flags & ~WSORT_FLAG_SRC_OFF) return set_err(c, WSORT_E_INVALID_ARG, "bad flags 0x%x", flags);
    if (c->keys_external && !c->packed_pending)
        return set_err(c, WSORT_E_STATE, "keys from wsort_load_keys were already sorted; load them again");
    if (c->packed_pending && (flags & WSORT_FLAG_SRC_OFF))
        return set_err(c, WSORT_E_INVALID_ARG, "src_off is not available for packed / exchanged keys");
    cudaSetDevice(c->device);
    const bool want_src = (flags & WSORT_FLAG_SRC_OFF) != 0;
    int rc = arena_begin(c);
    if (rc) return rc;
    if (c->comm) {   // collective (include/wsort.h: multi-GPU)
        if (algo != WSORT_ALGO_AUTO || want_src)
            return set_err(c, WSORT_E_INVALID_ARG, "multi-GPU wsort_sort: AUTO, keys only");
        rc = sort_dist(c);
        if (!rc) rc = arena_end(c);
        if (rc) {
            c->state = ST_TOKENIZED;
            return rc;
        }
        c->sorted_with_src = false;
        c->last_algo = algo;
        c->state = ST_SORTED;
        return WSORT_OK;
    }
    // the dense + MSD path reads what K1 ingest left (dense counts, staged keys): a text this context
    // tokenized, keys only, every word staged (<= 66 letters)
    const bool ingest_ok = !want_src && !c->packed_pending && !c->keys_external && c->h_ig[kIgVeryLong] == 0;
    if (c->keys_external && c->dense_range) {   // split multi-GPU sort: dense slice + received keys
        rc = sort_dist_dense(c);
    } else if (algo == WSORT_ALGO_OETS_MERGE) {
        rc = sort_oets(c, want_src);
    } else if (algo == WSORT_ALGO_RAGGED && !c->packed_pending) {
        rc = sort_ragged(c, want_src);
    } else if (algo == WSORT_ALGO_AUTO && ingest_ok && c->hashed && hash_sortable(c)) {
        rc = sort_dense_hash(c);
    } else if ((algo == WSORT_ALGO_AUTO || algo == WSORT_ALGO_DENSE_MSD) && ingest_ok) {
        if (c->hashed) {   // DENSE_MSD reads the staged keys: tokenize again, staging
            rc = tokenize_impl(c, nullptr, false);
            if (rc) return rc;
        }
        if (!c->h_ig[kIgVeryLong]) rc = sort_dense_msd(c);
        else if (kw_of((int)c->h_sum->max_len) <= (int)kRadixRegMaxKw) rc = sort_msd(c, false);
        else rc = sort_radix(c, false);   // (a word of > 66 letters: not staged)
    } else if ((algo == WSORT_ALGO_MSD_RADIX || algo == WSORT_ALGO_MSD_OETS || algo == WSORT_ALGO_AUTO ||
                algo == WSORT_ALGO_DENSE_MSD) && !want_src &&
               kw_of((int)c->h_sum->max_len) <= (int)kRadixRegMaxKw) {
        rc = sort_msd(c, algo == WSORT_ALGO_MSD_RADIX);   // AUTO: odd-even transposition finish (measured faster)
    } else {
        rc = sort_radix(c, want_src);
    }
    c->packed_pending = false;
    if (!rc) rc = arena_end(c);
    if (rc) {
        c->state = c->keys_external ? ST_CREATED : ST_TOKENIZED;
        return rc;
    }
    c->sorted_with_src = want_src;
    c->last_algo = algo;
    c->state = ST_SORTED;
    return WSORT_OK;
}

int fetch_impl(wsort_ctx *c, wsort_result *r, bool wait);

int wsort_fetch(wsort_ctx *c, wsort_result *r) { return fetch_impl(c, r, true); }
int wsort_fetch_async(wsort_ctx *c, wsort_result *r) { return fetch_impl(c, r, false); }
int wsort_sync(wsort_ctx *c) {
    if (!c) return WSORT_E_INVALID_ARG;
    cudaSetDevice(c->device);
    CK(cudaStreamSynchronize(c->stream), "sync");
    return WSORT_OK;
}

int fetch_impl(wsort_ctx *c, wsort_result *r, bool wait) {
    if (!c || !r) return WSORT_E_INVALID_ARG;
    if (c->state < ST_TOKENIZED) return set_err(c, WSORT_E_STATE, "wsort_fetch before wsort_tokenize");
    if (r->mem != WSORT_MEM_HOST && r->mem != WSORT_MEM_DEVICE) return set_err(c, WSORT_E_INVALID_ARG, "bad mem");
    cudaSetDevice(c->device);
    const Summary &s = *c->h_sum;
    r->n_words = s.n_words + c->slice_words;          // (dense slice of a split multi-GPU sort, if any)
    r->words_len = s.byte_off[256] + c->slice_bytes;
    r->max_len = c->has_global ? c->gmax : s.max_len;
    r->word_base = c->word_base;
    r->byte_base = c->byte_base;
    const bool sorted = c->state == ST_SORTED;
    if (!sorted && (r->words || r->src_off))
        return set_err(c, WSORT_E_STATE, "words/src_off requested before wsort_sort");
    if (r->src_off && !c->sorted_with_src) return set_err(c, WSORT_E_STATE, "src_off needs WSORT_FLAG_SRC_OFF");
    const uint32_t noff = r->max_len + 2;
    const uint64_t *offs = c->has_global ? c->goff : s.off;
    if ((r->bucket_off && r->bucket_cap < noff) || (r->words && r->words_cap < r->words_len) ||
        (r->src_off && r->src_cap < r->n_words))
        return set_err(c, WSORT_E_BUFFER_TOO_SMALL, "fetch: buffer too small");
    const cudaMemcpyKind k = r->mem == WSORT_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (r->words && r->words_len)
        CK(cudaMemcpyAsync(r->words, c->words.p, r->words_len, k, c->stream), "fetch words");
    if (r->src_off && r->n_words)
        CK(cudaMemcpyAsync(r->src_off, c->src_off.p, r->n_words * 8, k, c->stream), "fetch src_off");
    if (wait) CK(cudaStreamSynchronize(c->stream), "fetch");
    if (r->bucket_off) {
        if (r->mem == WSORT_MEM_HOST) {
            memcpy(r->bucket_off, offs, noff * sizeof(uint64_t));
        } else {
            CK(cudaMemcpy(r->bucket_off, offs, noff * sizeof(uint64_t), cudaMemcpyHostToDevice), "fetch off");
        }
    }
    return WSORT_OK;
}

int wsort_device_results(wsort_ctx *c, const uint8_t **words, const uint64_t **bucket_off, const uint64_t **src_off) {
    if (!c) return WSORT_E_INVALID_ARG;
    if (c->state < ST_TOKENIZED) return set_err(c, WSORT_E_STATE, "no results yet");
    if ((words || src_off) && c->state != ST_SORTED) return set_err(c, WSORT_E_STATE, "not sorted yet");
    if (src_off && !c->sorted_with_src) return set_err(c, WSORT_E_STATE, "src_off needs WSORT_FLAG_SRC_OFF");
    if (words) *words = static_cast<const uint8_t *>(c->words.p);
    if (bucket_off) *bucket_off = reinterpret_cast<const uint64_t *>(
                        static_cast<const uint8_t *>(c->d_sum.p) + offsetof(Summary, off));
    if (src_off) *src_off = static_cast<const uint64_t *>(c->src_off.p);
    return WSORT_OK;
}

int wsort_set_profiling(wsort_ctx *c, int on) {
    if (!c) return WSORT_E_INVALID_ARG;
    c->prof = on != 0;
    c->prof_serial = on == 2;
    return WSORT_OK;
}

int wsort_kernel_stats(wsort_ctx *c, wsort_kernel_stat *out, int cap, int *n) {
    if (!c || (!out && cap > 0)) return WSORT_E_INVALID_ARG;
    cudaSetDevice(c->device);
    CK(cudaStreamSynchronize(c->stream), "stats sync");
    drain_events(c);
    int k = (int)c->classes.size();
    if (n) *n = k;
    for (int i = 0; i < k && i < cap; i++) {
        memset(&out[i], 0, sizeof out[i]);
        snprintf(out[i].name, sizeof out[i].name, "%s", c->classes[i].name.c_str());
        out[i].launches = c->classes[i].launches;
        out[i].total_ms = c->classes[i].ms;
        out[i].bytes = c->classes[i].bytes;
    }
    return WSORT_OK;
}

int wsort_reset_kernel_stats(wsort_ctx *c) {
    if (!c) return WSORT_E_INVALID_ARG;
    cudaSetDevice(c->device);
    CK(cudaStreamSynchronize(c->stream), "stats sync");
    drain_events(c);
    for (auto &k : c->classes) {
        k.launches = 0;
        k.ms = 0;
        k.bytes = 0;
    }
    return WSORT_OK;
}

uint64_t wsort_launch_count(const wsort_ctx *c) { return c ? c->launches : 0; }

int wsort_get_unique_id(uint8_t id[WSORT_UNIQUE_ID_BYTES]) {
    if (!id) return WSORT_E_INVALID_ARG;
    std::string err;
    return nccl_unique_id(id, err);
}

int wsort_attach_comm(wsort_ctx *c, int rank, int nranks, const uint8_t id[WSORT_UNIQUE_ID_BYTES]) {
    if (!c || !id || nranks < 1 || nranks > (int)kMaxRanks || rank < 0 || rank >= nranks)
        return c ? set_err(c, WSORT_E_INVALID_ARG, "bad rank %d / nranks %d", rank, nranks) : WSORT_E_INVALID_ARG;
    cudaSetDevice(c->device);
    delete c->comm;
    c->comm = nullptr;
    std::string err;
    const int rc = comm_create_nccl(&c->comm, id, rank, nranks, c->device, c->stream, err);
    if (rc) return set_err(c, rc, "wsort_attach_comm: %s", err.c_str());
    c->state = ST_CREATED;
    return WSORT_OK;
}

int wsort_group_create(wsort_group **out, int nranks) {
    if (!out || nranks < 1 || nranks > (int)kMaxRanks) return WSORT_E_INVALID_ARG;
    *out = reinterpret_cast<wsort_group *>(group_create(nranks));
    return WSORT_OK;
}
void wsort_group_destroy(wsort_group *g) { group_destroy(reinterpret_cast<Group *>(g)); }

int wsort_attach_group(wsort_ctx *c, wsort_group *g, int rank) {
    if (!c || !g || rank < 0 || rank >= group_size(reinterpret_cast<Group *>(g))) return WSORT_E_INVALID_ARG;
    cudaSetDevice(c->device);
    delete c->comm;
    c->comm = nullptr;
    const int rc = comm_create_group(&c->comm, reinterpret_cast<Group *>(g), rank, c->device);
    if (rc) return set_err(c, rc, "wsort_attach_group failed");
    c->state = ST_CREATED;
    return WSORT_OK;
}

int wsort_detach_comm(wsort_ctx *c) {
    if (!c) return WSORT_E_INVALID_ARG;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    delete c->comm;
    c->comm = nullptr;
    c->has_global = false;
    c->slice_words = c->slice_bytes = 0;
    c->word_base = c->byte_base = 0;
    c->state = ST_CREATED;
    return WSORT_OK;
}

int wsort_get_slices(const wsort_ctx *c, wsort_slice *out, int cap, int *n) {
    if (!c || !n || (cap > 0 && !out)) return WSORT_E_INVALID_ARG;
    if (c->state != ST_SORTED) return WSORT_E_STATE;
    std::vector<wsort_slice> sl = c->slices;
    if (!c->comm) sl.assign(1, wsort_slice{0, c->h_sum->byte_off[256] + c->slice_bytes, c->h_sum->n_words + c->slice_words,
                                           c->byte_base, c->word_base});
    *n = (int)sl.size();
    for (int i = 0; i < cap && i < (int)sl.size(); i++) out[i] = sl[i];
    return WSORT_OK;
}

int wsort_set_ingest(wsort_ctx *c, int mode) {
    if (!c) return WSORT_E_INVALID_ARG;
    if (mode != WSORT_INGEST_AUTO && mode != WSORT_INGEST_STAGE && mode != WSORT_INGEST_COUNT)
        return set_err(c, WSORT_E_INVALID_ARG, "bad ingest mode %d", mode);
    c->ingest_mode = mode;
    return WSORT_OK;
}

int wsort_get_ingest_info(const wsort_ctx *c, wsort_ingest_info *out) {
    if (!c || !out) return WSORT_E_INVALID_ARG;
    *out = c->ig_info;
    if (c->ig_info.overflow) out->mode = 0;
    return WSORT_OK;
}

}  // extern "C"

// ====================================================================================
// Multi-GPU stages: pack -> sample -> [all-gather] -> select splitters ->
// partition -> [all-to-all] -> load_keys -> sort -> set_global -> fetch. Keys-only.
// The collectives run outside the library (torch.distributed / NCCL over NVLink); every data step
// between them is a kernel here.
// ====================================================================================
namespace {

std::vector<BucketInfo> bucket_table(const Summary &s) {
    std::vector<BucketInfo> bk(256, BucketInfo{});
    for (uint32_t L = 1; L <= s.max_len && L < 256; L++) {
        BucketInfo &b = bk[L];
        b.key_off = s.key_off[L];
        b.word_off = s.off[L];
        b.byte_off = s.byte_off[L];
        b.n = (uint32_t)(s.off[L + 1] - s.off[L]);
        b.kw = kw_of(L);
        b.elem_off = b.key_off;
        b.estride = b.kw;
    }
    return bk;
}


// Fill the host summary from per-length counts (local bucket layout of packed keys).
void summary_from_counts(Summary &s, const uint64_t *n_per_len) {
    memset(&s, 0, sizeof s);
    uint64_t o = 0, ko = 0, bo = 0, letters = 0;
    uint32_t lmax = 0;
    for (int L = 0; L < 256; L++) {
        s.off[L] = o;
        s.key_off[L] = ko;
        s.byte_off[L] = bo;
        const uint64_t h = L ? n_per_len[L] : 0;
        o += h;
        ko += h * (uint64_t)kw_of(L);
        bo += h * (uint64_t)(L + 1);
        letters += h * (uint64_t)L;
        if (h) lmax = (uint32_t)L;
    }
    s.off[256] = o;
    s.key_off[256] = ko;
    s.byte_off[256] = bo;
    s.n_words = o;
    s.letters = letters;
    s.max_len = lmax;
}

}  // namespace

extern "C" {

int wsort_histogram(wsort_ctx *c, uint64_t *hist) {
    if (!c || !hist) return WSORT_E_INVALID_ARG;
    if (c->state < ST_TOKENIZED) return set_err(c, WSORT_E_STATE, "wsort_histogram before wsort_tokenize");
    const Summary &s = *c->h_sum;
    for (int L = 0; L < 256; L++) hist[L] = s.off[L + 1] - s.off[L];
    return WSORT_OK;
}

int wsort_pack(wsort_ctx *c) {
    if (!c) return WSORT_E_INVALID_ARG;
    if (c->state != ST_TOKENIZED || c->keys_external)
        return set_err(c, WSORT_E_STATE, "wsort_pack needs a freshly tokenized text");
    cudaSetDevice(c->device);
    const Summary &s = *c->h_sum;
    std::vector<BucketInfo> bk = bucket_table(s);
    int rc;
    if ((rc = upload_small(c, c->bk, bk.data(), bk.size() * sizeof(BucketInfo), "bucket table"))) return rc;
    if ((rc = ensure(c, c->keys_a, s.key_off[256] * 4 + 64, "keys_a"))) return rc;
    TkArgs &tk = c->tk;
    tk.buckets = static_cast<const BucketInfo *>(c->bk.p);
    tk.keys = static_cast<uint32_t *>(c->keys_a.p);
    tk.payload = nullptr;
    rc = launch(c, "k3_pack_scatter", (double)c->n + (double)s.key_off[256] * 4,
                [&] { return pack_scatter(c); });
    if (rc) return rc;
    c->packed_pending = true;
    c->state = ST_PACKED;
    return WSORT_OK;
}

int wsort_pack_long(wsort_ctx *c, uint32_t **dense_table, uint64_t *dense_entries_out) {
    if (!c || !dense_table || !dense_entries_out) return WSORT_E_INVALID_ARG;
    if (c->state != ST_TOKENIZED || c->keys_external || c->packed_pending)
        return set_err(c, WSORT_E_STATE, "wsort_pack_long needs a freshly tokenized text");
    if (c->h_ig[kIgVeryLong])
        return set_err(c, WSORT_E_STATE, "wsort_pack_long: words longer than %d letters were not staged", 6 * kMaxStageKw);
    cudaSetDevice(c->device);
    if (c->hashed) {   // the split exchange reads the staged keys: tokenize again, staging
        int rc0 = tokenize_impl(c, nullptr, false);
        if (rc0) return rc0;
    }
    Summary &s = *c->h_sum;
    std::vector<uint64_t> n(256, 0);
    for (uint32_t L = kDenseMaxLen + 1; L < 256; L++) n[L] = s.off[L + 1] - s.off[L];
    summary_from_counts(s, n.data());   // the packed keys: lengths >= 6 only
    int rc;
    if ((rc = upload_small(c, c->d_sum, &s, sizeof(Summary), "long summary"))) return rc;
    std::vector<BucketInfo> bk = bucket_table(s);
    if ((rc = upload_small(c, c->bk, bk.data(), bk.size() * sizeof(BucketInfo), "bucket table"))) return rc;
    if ((rc = ensure(c, c->keys_a, s.key_off[256] * 4 + 64, "keys_a"))) return rc;
    if (s.n_words && (rc = chunk_scatter(c, static_cast<const BucketInfo *>(c->bk.p), (double)s.key_off[256] * 4)))
        return rc;
    c->packed_pending = true;
    c->dist_dense = true;
    c->state = ST_PACKED;
    // the caller adds the other ranks' tables: every block may be non-zero
    CK(cudaMemsetAsync(c->d_touched.p, 1, dense_scan_blocks(dense_entries()), c->stream), "touched");
    *dense_table = static_cast<uint32_t *>(c->dense.p);
    *dense_entries_out = dense_entries();
    return WSORT_OK;
}

int wsort_dense_range(wsort_ctx *c, const uint64_t *ghist, uint64_t lo, uint64_t hi) {
    if (!c || !ghist || lo > hi) return WSORT_E_INVALID_ARG;
    if (!c->dist_dense || !c->keys_external || !c->packed_pending)
        return set_err(c, WSORT_E_STATE, "wsort_dense_range needs wsort_pack_long, then wsort_load_keys");
    uint64_t g = 0;   // global word index of the first word of length L
    for (uint32_t L = 1; L <= kDenseMaxLen; L++) {
        const uint64_t a = std::max(g, lo), b = std::min(g + ghist[L], hi);
        c->dslice_off[L] = a;
        c->dslice_n[L] = b > a ? b - a : 0;
        g += ghist[L];
    }
    if (hi > g) return set_err(c, WSORT_E_INVALID_ARG, "dense range end %llu > %llu dense words",
                               (unsigned long long)hi, (unsigned long long)g);
    if (g > 0xffffffffull) return set_err(c, WSORT_E_TOO_LARGE, "more than 2^32 - 1 dense words");
    c->slice_words = hi - lo;
    c->slice_bytes = 0;
    for (uint32_t L = 1; L <= kDenseMaxLen; L++) c->slice_bytes += c->dslice_n[L] * (L + 1);
    c->dense_lo = lo;
    c->dense_hi = hi;
    c->dense_range = true;
    return WSORT_OK;
}

int wsort_sample(wsort_ctx *c, uint32_t nsamples, uint32_t rank, uint32_t rec_words, uint32_t *dev_records) {
    if (!c || (nsamples && !dev_records) || rec_words < 3) return WSORT_E_INVALID_ARG;
    if (c->state != ST_PACKED || !c->packed_pending) return set_err(c, WSORT_E_STATE, "wsort_sample needs packed keys");
    const Summary &s = *c->h_sum;
    if (rec_words < 2 + (uint32_t)kw_of((int)s.max_len))
        return set_err(c, WSORT_E_INVALID_ARG, "rec_words %u < 2 + kw(%u)", rec_words, s.max_len);
    cudaSetDevice(c->device);
    DistArgs a{};
    a.buckets = static_cast<const BucketInfo *>(c->bk.p);
    a.off = reinterpret_cast<const uint64_t *>(static_cast<const uint8_t *>(c->d_sum.p) + offsetof(Summary, off));
    a.keys = static_cast<const uint32_t *>(c->keys_a.p);
    a.n_words = s.n_words;
    a.rank = rank;
    a.rec_words = rec_words;
    a.nsamples = nsamples;
    a.records = dev_records;
    return launch(c, "k6a_sample", (double)nsamples * rec_words * 8, [&] { return launch_sample(a, c->stream); });
}

static int cmp_records(const uint32_t *x, const uint32_t *y, uint32_t rec_words) {
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;              // length
    for (uint32_t u = 2; u < rec_words; u++)                     // key words
        if (x[u] != y[u]) return x[u] < y[u] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;              // source rank
    return 0;
}

int wsort_select_splitters(const uint32_t *samples, uint64_t nsamples, uint32_t rec_words, uint32_t nparts,
                           uint32_t *splitters) {
    if (!samples || !splitters || nparts < 1 || nparts > kMaxRanks || rec_words < 3 || nsamples < nparts)
        return WSORT_E_INVALID_ARG;
    // (length, first key word) as one u64 decides almost every comparison without touching the records
    struct Ent {
        uint64_t head, i;
    };
    std::vector<Ent> e(nsamples);
    for (uint64_t i = 0; i < nsamples; i++)
        e[i] = Ent{((uint64_t)samples[i * rec_words] << 32) | samples[i * rec_words + 2], i};
    auto less = [&](const Ent &x, const Ent &y) {
        if (x.head != y.head) return x.head < y.head;
        const int r = cmp_records(samples + x.i * rec_words, samples + y.i * rec_words, rec_words);
        return r < 0 || (r == 0 && x.i < y.i);
    };
    // only the nparts-1 order statistics are needed: multi-select (median quantile first, then each
    // side), O(n log nparts) instead of a full sort
    std::vector<uint64_t> ks(nparts - 1);
    for (uint32_t d = 1; d < nparts; d++) ks[d - 1] = (d * nsamples) / nparts;
    std::function<void(uint64_t, uint64_t, size_t, size_t)> select = [&](uint64_t a, uint64_t b, size_t i, size_t j) {
        if (i >= j) return;
        const size_t m = (i + j) / 2;
        const uint64_t k = ks[m];
        std::nth_element(e.begin() + a, e.begin() + k, e.begin() + b, less);
        select(a, k, i, m);
        select(k + 1, b, m + 1, j);
    };
    select(0, nsamples, 0, ks.size());
    for (uint32_t d = 1; d < nparts; d++)
        memcpy(splitters + (size_t)(d - 1) * rec_words, samples + e[ks[d - 1]].i * rec_words, rec_words * 4);
    return WSORT_OK;
}

int wsort_partition(wsort_ctx *c, const uint32_t *splitters, uint32_t nparts, uint32_t rec_words, uint32_t rank,
                    uint32_t *dev_send, uint64_t send_cap_words, uint64_t *counts, uint64_t *send_words) {
    if (!c || !counts || !send_words || nparts < 1 || nparts > kMaxRanks || (nparts > 1 && !splitters) ||
        rank >= nparts)
        return WSORT_E_INVALID_ARG;
    if (c->state != ST_PACKED || !c->packed_pending) return set_err(c, WSORT_E_STATE, "wsort_partition needs packed keys");
    const Summary &s = *c->h_sum;
    if (send_cap_words < s.key_off[256] || (s.key_off[256] && !dev_send))
        return set_err(c, WSORT_E_BUFFER_TOO_SMALL, "send buffer needs %llu words", (unsigned long long)s.key_off[256]);
    cudaSetDevice(c->device);
    int rc;
    // splitter lookup ranges per length
    std::vector<uint32_t> lohi(512, 0);
    for (uint32_t L = 0; L < 256; L++) {
        uint32_t lo = 0, hi = 0;
        for (uint32_t d = 0; d + 1 < nparts; d++) {
            const uint32_t sl = splitters[(size_t)d * rec_words];   // splitter length
            lo += sl < L;
            hi += sl <= L;
        }
        lohi[L] = lo;
        lohi[256 + L] = hi;
    }
    std::vector<TileDesc> tiles;
    for (uint32_t L = 1; L <= s.max_len; L++) {
        const uint64_t n = s.off[L + 1] - s.off[L];
        for (uint64_t i = 0; i * kDistTileKeys < n; i++) tiles.push_back(TileDesc{L, (uint32_t)i});
    }
    if (nparts > 1 && (rc = upload_small(c, c->d_split, splitters, (size_t)(nparts - 1) * rec_words * 4, "splitters")))
        return rc;
    if ((rc = ensure(c, c->d_split, 16, "splitters"))) return rc;
    if ((rc = upload_small(c, c->d_lohi, lohi.data(), lohi.size() * 4, "split ranges"))) return rc;
    if ((rc = upload_small(c, c->d_tiles, tiles.data(), tiles.size() * sizeof(TileDesc), "partition tiles"))) return rc;
    if ((rc = ensure(c, c->d_counts, (size_t)nparts * 256 * 4, "counts"))) return rc;
    if ((rc = ensure(c, c->d_cursor, (size_t)nparts * 256 * 4, "cursor"))) return rc;
    if ((rc = ensure(c, c->d_sbase, (size_t)nparts * 256 * 8, "send base"))) return rc;
    CK(cudaMemsetAsync(c->d_counts.p, 0, (size_t)nparts * 256 * 4, c->stream), "memset counts");
    CK(cudaMemsetAsync(c->d_cursor.p, 0, (size_t)nparts * 256 * 4, c->stream), "memset cursor");
    DistArgs a{};
    a.buckets = static_cast<const BucketInfo *>(c->bk.p);
    a.tiles = static_cast<const TileDesc *>(c->d_tiles.p);
    a.ntiles = (uint32_t)tiles.size();
    a.keys = static_cast<const uint32_t *>(c->keys_a.p);
    a.n_words = s.n_words;
    a.rank = rank;
    a.nparts = nparts;
    a.rec_words = rec_words;
    a.splitters = static_cast<const uint32_t *>(c->d_split.p);
    a.split_lo = static_cast<const uint32_t *>(c->d_lohi.p);
    a.split_hi = a.split_lo + 256;
    a.counts = static_cast<uint32_t *>(c->d_counts.p);
    a.cursor = static_cast<uint32_t *>(c->d_cursor.p);
    a.send_base = static_cast<const uint64_t *>(c->d_sbase.p);
    a.send = dev_send;
    rc = launch(c, "k6b_part_count", (double)s.key_off[256] * 4, [&] { return launch_part_count(a, c->stream); });
    if (rc) return rc;
    std::vector<uint32_t> hc((size_t)nparts * 256);
    CK(cudaMemcpyAsync(hc.data(), c->d_counts.p, hc.size() * 4, cudaMemcpyDeviceToHost, c->stream), "counts D2H");
    CK(cudaStreamSynchronize(c->stream), "partition counts");
    std::vector<uint64_t> base((size_t)nparts * 256);
    uint64_t w = 0;
    for (uint32_t d = 0; d < nparts; d++) {
        const uint64_t w0 = w;
        for (uint32_t L = 0; L < 256; L++) {
            counts[(size_t)d * 256 + L] = hc[(size_t)d * 256 + L];
            base[(size_t)d * 256 + L] = w;
            w += (uint64_t)hc[(size_t)d * 256 + L] * (uint64_t)kw_of((int)L);
        }
        send_words[d] = w - w0;
    }
    if ((rc = upload_small(c, c->d_sbase, base.data(), base.size() * 8, "send base"))) return rc;
    return launch(c, "k6b_part_scatter", (double)s.key_off[256] * 8, [&] { return launch_part_scatter(a, c->stream); });
}

int wsort_load_keys(wsort_ctx *c, const uint32_t *dev_recv, const uint64_t *counts, uint32_t nparts) {
    if (!c || !counts || nparts < 1 || nparts > kMaxRanks) return WSORT_E_INVALID_ARG;
    cudaSetDevice(c->device);
    std::vector<uint64_t> n(256, 0);
    for (uint32_t src = 0; src < nparts; src++)
        for (uint32_t L = 1; L < 256; L++) n[L] += counts[(size_t)src * 256 + L];
    for (uint32_t src = 0; src < nparts; src++)
        if (counts[(size_t)src * 256] != 0) return set_err(c, WSORT_E_INVALID_ARG, "counts of length 0");
    Summary &s = *c->h_sum;
    summary_from_counts(s, n.data());
    if (s.key_off[256] && !dev_recv) return WSORT_E_INVALID_ARG;
    int rc;
    if ((rc = ensure(c, c->keys_a, s.key_off[256] * 4 + 64, "keys_a"))) return rc;
    // received layout: [src][L][keys]; local bucket L = src-ordered concatenation
    std::vector<CopyRange> ranges;
    std::vector<uint64_t> fill(256, 0);
    uint64_t from = 0;
    for (uint32_t src = 0; src < nparts; src++)
        for (uint32_t L = 1; L < 256; L++) {
            const uint64_t cnt = counts[(size_t)src * 256 + L];
            if (!cnt) continue;
            const uint64_t words = cnt * (uint64_t)kw_of((int)L);
            uint64_t to = s.key_off[L] + fill[L];
            for (uint64_t o = 0; o < words; o += 16384) {
                const uint32_t len = (uint32_t)std::min<uint64_t>(16384, words - o);
                ranges.push_back(CopyRange{from + o, to + o, len, 0});
            }
            fill[L] += words;
            from += words;
        }
    if ((rc = upload_small(c, c->d_ranges, ranges.data(), ranges.size() * sizeof(CopyRange), "ranges"))) return rc;
    rc = launch(c, "k6c_regroup", (double)s.key_off[256] * 8, [&] {
        return launch_regroup(static_cast<const CopyRange *>(c->d_ranges.p), (uint32_t)ranges.size(), dev_recv,
                              static_cast<uint32_t *>(c->keys_a.p), c->stream);
    });
    if (rc) return rc;
    c->n = 0;
    c->packed_pending = true;
    c->keys_external = true;
    c->dense_range = false;
    c->slice_words = c->slice_bytes = 0;
    c->has_global = false;
    c->state = ST_PACKED;
    return WSORT_OK;
}

int wsort_set_global(wsort_ctx *c, const uint64_t *ghist, uint64_t word_base, uint64_t byte_base) {
    if (!c || !ghist) return WSORT_E_INVALID_ARG;
    uint64_t o = 0;
    uint32_t lmax = 0;
    for (int L = 0; L < 256; L++) {
        c->goff[L] = o;
        o += L ? ghist[L] : 0;
        if (L && ghist[L]) lmax = (uint32_t)L;
    }
    c->goff[256] = o;
    c->gmax = lmax;
    // off[] has max_len + 2 entries: off[lmax + 1] = W
    c->goff[lmax + 1] = o;
    c->word_base = word_base;
    c->byte_base = byte_base;
    c->has_global = true;
    return WSORT_OK;
}

}  // extern "C"
