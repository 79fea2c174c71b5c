// Microbenchmark (experiments): shared-memory atomic throughput on one SM-wide grid, by access pattern.
// Each thread does ITER atomicAdd on a 1024-entry table; patterns: distinct conflict-free addresses, random
// addresses, all lanes one address, only 8 lanes active (distinct), Zipf-like hot addresses.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int PAT>
__global__ void __launch_bounds__(512) k_atom(uint32_t *out, int iters) {
    __shared__ uint32_t h[1024];
    const int t = threadIdx.x, lane = t & 31;
    for (int i = t; i < 1024; i += 512) h[i] = 0;
    __syncthreads();
    uint32_t x = t * 2654435761u + blockIdx.x;
    for (int it = 0; it < iters; it++) {
        x = x * 1664525u + 1013904223u;
        uint32_t a;
        if (PAT == 0) a = (lane + 32 * (it & 31)) & 1023;              // distinct, conflict-free
        else if (PAT == 1) a = x >> 22;                                 // random
        else if (PAT == 2) a = 7;                                       // one address
        else if (PAT == 3) a = (x >> 28) < 3 ? 7 : (x >> 22);           // ~19% hot on one address
        else a = (lane + 32 * (it & 31)) & 1023;
        if (PAT == 4 && lane >= 8) continue;                            // 8 active lanes
        if (PAT == 5) { h[a] += 1; continue; }                          // plain (racy) ld/add/st
        atomicAdd(&h[a], 1u);
    }
    __syncthreads();
    if (t == 0) out[blockIdx.x] = h[0] + h[7];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *out;
    cudaMalloc(&out, 4096 * 4);
    const int iters = 4096, grid = sms * 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[] = {"distinct conflict-free", "random 1024", "one address", "19% hot one address",
                           "8 lanes active distinct", "plain ld/add/st conflict-free"};
    auto run = [&](int p, auto kern) {
        kern<<<grid, 512>>>(out, iters);
        cudaEventRecord(e0);
        kern<<<grid, 512>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double warp_ops = (double)grid * 16 * iters;
        const double cyc = ms * 1e-3 * 1.965e9;
        printf("%-32s %8.3f ms  %6.2f SM-cycles per warp atomic instr (per SM)\n", names[p], ms, cyc / (warp_ops / sms));
    };
    run(0, k_atom<0>);
    run(1, k_atom<1>);
    run(2, k_atom<2>);
    run(3, k_atom<3>);
    run(4, k_atom<4>);
    run(5, k_atom<5>);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
