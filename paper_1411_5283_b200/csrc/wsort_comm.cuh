// wsort_comm.cuh — the communicator a libwsort context owns when it is one rank of a multi-GPU sort
// (include/wsort.h: wsort_get_unique_id / wsort_attach_comm / wsort_group_*).
//
// Two implementations of the same stream-ordered collectives:
//   NcclComm   one process per GPU: libnccl.so.2 (dlopen'ed: the one torch loaded, or the system's)
//              for all-reduce / all-gather / barrier over NVLink, CUDA IPC handles (exchanged by an
//              all-gather) for the peer windows the exchange kernel stores into;
//   GroupComm  several ranks in ONE process (a thread per rank, any GPUs, e.g. all on one GPU for the
//              tests): collectives by host barriers + device copies / a summing kernel, peer windows =
//              the other ranks' device pointers. No kernel ever waits for another rank's kernel.
// Every call is collective (all ranks call it, in the same order); on return the collective's effect is
// ordered before later work on the caller's stream.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace wsort {

struct Comm {
    int rank = 0, size = 1;
    std::string err;
    virtual ~Comm() {}
    virtual const char *kind() const = 0;
    // in-place sums over the ranks
    virtual int allreduce_u32(uint32_t *buf, size_t n, cudaStream_t s) = 0;
    virtual int allreduce_u64(uint64_t *buf, size_t n, cudaStream_t s) = 0;
    // recv (size * bytes) = every rank's send (bytes), in rank order
    virtual int allgather(const void *send, void *recv, size_t bytes, cudaStream_t s) = 0;
    // every rank's earlier stream work (including stores into peer windows) is complete and visible
    virtual int barrier(cudaStream_t s) = 0;
    // device pointers of every rank's `local` buffer (peers[rank] = local); valid until the next call
    virtual int peer_windows(void *local, size_t bytes, std::vector<void *> &peers, cudaStream_t s) = 0;
};

// returns 0 (WSORT_OK) or a WSORT_E_* code with the message in *err
int nccl_unique_id(uint8_t id[128], std::string &err);
int comm_create_nccl(Comm **out, const uint8_t id[128], int rank, int nranks, int device, cudaStream_t s,
                     std::string &err);

struct Group;   // in-process ranks (wsort_group)
Group *group_create(int nranks);
void group_destroy(Group *g);
int group_size(const Group *g);
int comm_create_group(Comm **out, Group *g, int rank, int device);

}  // namespace wsort
