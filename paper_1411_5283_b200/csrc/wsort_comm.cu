// wsort_comm.cu — NcclComm (one process per GPU) and GroupComm (ranks as threads of one process); see
// wsort_comm.cuh. NCCL is loaded at run time (dlopen "libnccl.so.2": the copy torch already loaded in this
// process, else the system's), so libwsort has no link-time NCCL dependency and single-GPU use needs none.
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "wsort.h"
#include "wsort_comm.cuh"

namespace wsort {
namespace {

// ---------------------------------------------------------------- NCCL (the few calls used)
typedef int nccl_result;   // ncclResult_t: 0 = ncclSuccess
typedef void *nccl_comm;   // ncclComm_t
struct NcclApi {
    void *lib = nullptr;
    nccl_result (*get_unique_id)(void *id) = nullptr;
    nccl_result (*comm_init_rank)(nccl_comm *comm, int nranks, /* ncclUniqueId by value */ ...) = nullptr;
    nccl_result (*all_reduce)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*all_gather)(const void *, void *, size_t, int, nccl_comm, cudaStream_t) = nullptr;
    nccl_result (*comm_destroy)(nccl_comm) = nullptr;
    const char *(*error_string)(nccl_result) = nullptr;
};
enum { kNcclUint8 = 1, kNcclUint32 = 3, kNcclUint64 = 5, kNcclSum = 0 };
struct UniqueId {
    char internal[128];
};
typedef nccl_result (*init_rank_fn)(nccl_comm *, int, UniqueId, int);

NcclApi *nccl_api(std::string &err) {
    static NcclApi api;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (api.lib) return &api;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        err = std::string("cannot load libnccl.so.2: ") + dlerror();
        return nullptr;
    }
    api.get_unique_id = (nccl_result(*)(void *))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (nccl_result(*)(nccl_comm *, int, ...))dlsym(h, "ncclCommInitRank");
    api.all_reduce = (nccl_result(*)(const void *, void *, size_t, int, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllReduce");
    api.all_gather = (nccl_result(*)(const void *, void *, size_t, int, nccl_comm, cudaStream_t))dlsym(h, "ncclAllGather");
    api.comm_destroy = (nccl_result(*)(nccl_comm))dlsym(h, "ncclCommDestroy");
    api.error_string = (const char *(*)(nccl_result))dlsym(h, "ncclGetErrorString");
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_reduce || !api.all_gather || !api.comm_destroy ||
        !api.error_string) {
        err = "libnccl.so.2 lacks a needed symbol";
        return nullptr;
    }
    api.lib = h;
    return &api;
}

struct NcclComm : Comm {
    NcclApi *api = nullptr;
    nccl_comm comm = nullptr;
    uint32_t *d_tok = nullptr;                 // barrier token
    uint8_t *d_handles = nullptr;              // [size][64] IPC handles (all-gathered)
    std::vector<cudaIpcMemHandle_t> open_h;    // handles currently opened, per peer
    std::vector<void *> open_p;
    const char *kind() const override { return "nccl"; }
    int nccl(nccl_result r, const char *what) {
        if (r == 0) return WSORT_OK;
        err = std::string(what) + ": " + api->error_string(r);
        return WSORT_E_NCCL;
    }
    ~NcclComm() override {
        for (size_t q = 0; q < open_p.size(); q++)
            if (open_p[q] && (int)q != rank) cudaIpcCloseMemHandle(open_p[q]);
        if (comm) api->comm_destroy(comm);
        if (d_tok) cudaFree(d_tok);
        if (d_handles) cudaFree(d_handles);
    }
    int allreduce_u32(uint32_t *buf, size_t n, cudaStream_t s) override {
        return nccl(api->all_reduce(buf, buf, n, kNcclUint32, kNcclSum, comm, s), "ncclAllReduce(u32)");
    }
    int allreduce_u64(uint64_t *buf, size_t n, cudaStream_t s) override {
        return nccl(api->all_reduce(buf, buf, n, kNcclUint64, kNcclSum, comm, s), "ncclAllReduce(u64)");
    }
    int allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override {
        return nccl(api->all_gather(send, recv, bytes, kNcclUint8, comm, s), "ncclAllGather");
    }
    int barrier(cudaStream_t s) override {   // stream-ordered: NCCL's kernel orders every rank's earlier work
        return nccl(api->all_reduce(d_tok, d_tok, 1, kNcclUint32, kNcclSum, comm, s), "ncclAllReduce(barrier)");
    }
    int peer_windows(void *local, size_t, std::vector<void *> &peers, cudaStream_t s) override {
        cudaIpcMemHandle_t h;
        cudaError_t e = cudaIpcGetMemHandle(&h, local);
        if (e != cudaSuccess) {
            err = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
            return WSORT_E_CUDA;
        }
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        std::vector<uint8_t> all((size_t)size * 64);
        if (cudaMemcpyAsync(d_handles + (size_t)rank * 64, &h, 64, cudaMemcpyHostToDevice, s) != cudaSuccess) return WSORT_E_CUDA;
        int rc = allgather(d_handles + (size_t)rank * 64, d_handles, 64, s);
        if (rc) return rc;
        if (cudaMemcpyAsync(all.data(), d_handles, all.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return WSORT_E_CUDA;
        peers.assign(size, nullptr);
        for (int q = 0; q < size; q++) {
            if (q == rank) {
                peers[q] = local;
                continue;
            }
            const cudaIpcMemHandle_t *hq = reinterpret_cast<const cudaIpcMemHandle_t *>(all.data() + (size_t)q * 64);
            if (open_p[q] && memcmp(&open_h[q], hq, 64) == 0) {   // the peer's window did not move
                peers[q] = open_p[q];
                continue;
            }
            if (open_p[q]) cudaIpcCloseMemHandle(open_p[q]);
            open_p[q] = nullptr;
            e = cudaIpcOpenMemHandle(&open_p[q], *hq, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                err = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
                return WSORT_E_CUDA;
            }
            open_h[q] = *hq;
            peers[q] = open_p[q];
        }
        return WSORT_OK;
    }
};

// ---------------------------------------------------------------- in-process group
__global__ void k_sum_u32(uint32_t *dst, const uint32_t *const *src, int n_src, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int q = 0; q < n_src; q++) v += src[q][i];
        dst[i] = v;
    }
}
__global__ void k_sum_u64(uint64_t *dst, const uint64_t *const *src, int n_src, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t v = 0;
        for (int q = 0; q < n_src; q++) v += src[q][i];
        dst[i] = v;
    }
}

}  // namespace

struct Group {
    int n;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const void *> ptr;   // one published pointer per rank
    explicit Group(int nranks) : n(nranks), ptr(nranks, nullptr) {}
    void wait() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == n) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

namespace {

struct GroupComm : Comm {
    Group *g = nullptr;
    void *tmp = nullptr;            // this rank's reduction result before it overwrites its buffer
    size_t tmp_cap = 0;
    const void **d_ptrs = nullptr;  // [size] the published pointers, in device memory
    const char *kind() const override { return "group"; }
    ~GroupComm() override {
        if (tmp) cudaFree(tmp);
        if (d_ptrs) cudaFree(d_ptrs);
    }
    int cuda(cudaError_t e, const char *what) {
        if (e == cudaSuccess) return WSORT_OK;
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return WSORT_E_CUDA;
    }
    // publish p, wait for all; the caller reads g->ptr; a second wait() ends the collective
    int publish(const void *p, cudaStream_t s) {
        int rc = cuda(cudaStreamSynchronize(s), "group: stream sync");
        g->ptr[rank] = p;
        g->wait();
        return rc;
    }
    template <class T, class K>
    int allreduce(T *buf, size_t n, cudaStream_t s, K kernel) {
        int rc = publish(buf, s);
        const size_t bytes = n * sizeof(T);
        if (!rc && tmp_cap < bytes) {
            if (tmp) cudaFree(tmp);
            tmp = nullptr;
            tmp_cap = 0;
            rc = cuda(cudaMalloc(&tmp, bytes), "group: reduction buffer");
            if (!rc) tmp_cap = bytes;
        }
        if (!rc) rc = cuda(cudaMemcpyAsync(d_ptrs, g->ptr.data(), size * sizeof(void *), cudaMemcpyHostToDevice, s), "group: ptrs");
        if (!rc) {
            kernel<<<296, 256, 0, s>>>(static_cast<T *>(tmp), reinterpret_cast<const T *const *>(d_ptrs), size, n);
            rc = cuda(cudaGetLastError(), "group: sum kernel");
        }
        if (!rc) rc = cuda(cudaStreamSynchronize(s), "group: sum");
        g->wait();   // every rank has its sum: the buffers may be overwritten
        if (!rc) rc = cuda(cudaMemcpyAsync(buf, tmp, bytes, cudaMemcpyDeviceToDevice, s), "group: result");
        return rc;
    }
    int allreduce_u32(uint32_t *buf, size_t n, cudaStream_t s) override { return allreduce(buf, n, s, k_sum_u32); }
    int allreduce_u64(uint64_t *buf, size_t n, cudaStream_t s) override { return allreduce(buf, n, s, k_sum_u64); }
    int allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) override {
        int rc = publish(send, s);
        for (int q = 0; q < size && !rc; q++)
            rc = cuda(cudaMemcpyAsync(static_cast<uint8_t *>(recv) + (size_t)q * bytes, g->ptr[q], bytes,
                                      cudaMemcpyDeviceToDevice, s), "group: gather copy");
        if (!rc) rc = cuda(cudaStreamSynchronize(s), "group: gather");
        g->wait();
        return rc;
    }
    int barrier(cudaStream_t s) override {
        int rc = cuda(cudaStreamSynchronize(s), "group: barrier sync");
        g->wait();
        return rc;
    }
    int peer_windows(void *local, size_t, std::vector<void *> &peers, cudaStream_t s) override {
        int rc = publish(local, s);
        peers.assign(size, nullptr);
        for (int q = 0; q < size; q++) peers[q] = const_cast<void *>(g->ptr[q]);
        g->wait();
        return rc;
    }
};

}  // namespace

int nccl_unique_id(uint8_t id[128], std::string &err) {
    NcclApi *api = nccl_api(err);
    if (!api) return WSORT_E_NCCL;
    nccl_result r = api->get_unique_id(id);
    if (r) {
        err = std::string("ncclGetUniqueId: ") + api->error_string(r);
        return WSORT_E_NCCL;
    }
    return WSORT_OK;
}

int comm_create_nccl(Comm **out, const uint8_t id[128], int rank, int nranks, int device, cudaStream_t s,
                     std::string &err) {
    *out = nullptr;
    NcclApi *api = nccl_api(err);
    if (!api) return WSORT_E_NCCL;
    cudaSetDevice(device);
    NcclComm *c = new NcclComm();
    c->api = api;
    c->rank = rank;
    c->size = nranks;
    UniqueId uid;
    memcpy(uid.internal, id, 128);
    nccl_result r = reinterpret_cast<init_rank_fn>(api->comm_init_rank)(&c->comm, nranks, uid, rank);
    if (r) {
        err = std::string("ncclCommInitRank: ") + api->error_string(r);
        c->comm = nullptr;
        delete c;
        return WSORT_E_NCCL;
    }
    if (cudaMalloc(&c->d_tok, 16) != cudaSuccess || cudaMalloc(&c->d_handles, (size_t)nranks * 64) != cudaSuccess ||
        cudaMemsetAsync(c->d_tok, 0, 16, s) != cudaSuccess) {
        err = "NCCL comm scratch allocation failed";
        delete c;
        return WSORT_E_NOMEM;
    }
    c->open_h.assign(nranks, cudaIpcMemHandle_t{});
    c->open_p.assign(nranks, nullptr);
    *out = c;
    return WSORT_OK;
}

Group *group_create(int nranks) { return new Group(nranks); }
void group_destroy(Group *g) { delete g; }
int group_size(const Group *g) { return g ? g->n : 0; }

int comm_create_group(Comm **out, Group *g, int rank, int device) {
    *out = nullptr;
    cudaSetDevice(device);
    GroupComm *c = new GroupComm();
    c->g = g;
    c->rank = rank;
    c->size = g->n;
    if (cudaMalloc(&c->d_ptrs, (size_t)g->n * sizeof(void *)) != cudaSuccess) {
        delete c;
        return WSORT_E_NOMEM;
    }
    *out = c;
    return WSORT_OK;
}

}  // namespace wsort
