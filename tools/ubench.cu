// Microbenchmarks of the primitives the wsort kernels rank and count with (B200, sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N_ITER 4096

__global__ void k_match(uint32_t *out, uint32_t seed) {
    uint32_t x = threadIdx.x * 2654435761u ^ seed, acc = 0;
    for (int i = 0; i < N_ITER; i++) {
        x = x * 1664525u + 1013904223u;
        acc += __match_any_sync(0xffffffffu, (x >> 22));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_ballot10(uint32_t *out, uint32_t seed) {
    uint32_t x = threadIdx.x * 2654435761u ^ seed, acc = 0;
    for (int i = 0; i < N_ITER; i++) {
        x = x * 1664525u + 1013904223u;
        uint32_t d = x >> 22, peers = 0xffffffffu;
#pragma unroll
        for (int b = 0; b < 10; b++) {
            uint32_t m = __ballot_sync(0xffffffffu, (d >> b) & 1);
            peers &= ((d >> b) & 1) ? m : ~m;
        }
        acc += peers;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_atoms(uint32_t *out, uint32_t seed, uint32_t mask) {
    __shared__ uint32_t h[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
    __syncthreads();
    uint32_t x = threadIdx.x * 2654435761u ^ seed;
    for (int i = 0; i < N_ITER; i++) {
        x = x * 1664525u + 1013904223u;
        atomicAdd(&h[(x >> 20) & mask], 1u);
    }
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = h[threadIdx.x];
}

__global__ void k_ldssts(uint32_t *out, uint32_t seed) {
    __shared__ uint32_t h[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = i;
    __syncthreads();
    uint32_t x = threadIdx.x * 2654435761u ^ seed, acc = 0;
    for (int i = 0; i < N_ITER; i++) {
        x = x * 1664525u + 1013904223u;
        uint32_t a = (x >> 20) & 4095;
        acc += h[a];
        h[(a + 7) & 4095] = acc;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_divbranch(uint32_t *out, uint32_t seed) {
    uint32_t x = threadIdx.x * 2654435761u ^ seed, acc = 0;
    for (int i = 0; i < N_ITER; i++) {
        x = x * 1664525u + 1013904223u;
        if ((x >> 27) == (threadIdx.x & 31)) acc += x * 3u; // divergent, rarely taken per lane
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_alu(uint32_t *out, uint32_t seed) {
    uint32_t x = threadIdx.x * 2654435761u ^ seed, acc = 0;
    for (int i = 0; i < N_ITER; i++) {
        x = x * 1664525u + 1013904223u;
        acc += (x >> 3) ^ (x << 5);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * 8, threads = 256;
    uint32_t *out;
    cudaMalloc(&out, blocks * threads * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double warps = (double)blocks * threads / 32 * N_ITER;
    auto run = [&](const char *name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 5; r++) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        int clk = 0;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        double cyc = ms * 1e-3 * clk * 1e3;
        printf("%-28s %8.3f ms  %.3f SM-cycles per warp-iteration (per SM)\n", name, ms, cyc * sms / warps);
    };
    run("alu baseline (2 ops)", [&] { k_alu<<<blocks, threads>>>(out, 1); });
    run("match_any 10-bit", [&] { k_match<<<blocks, threads>>>(out, 1); });
    run("ballot x10 peers", [&] { k_ballot10<<<blocks, threads>>>(out, 1); });
    run("atoms 4096 bins", [&] { k_atoms<<<blocks, threads>>>(out, 1, 4095); });
    run("atoms 1024 bins", [&] { k_atoms<<<blocks, threads>>>(out, 1, 1023); });
    run("atoms 4 bins (conflict)", [&] { k_atoms<<<blocks, threads>>>(out, 1, 3); });
    run("atoms 1 bin", [&] { k_atoms<<<blocks, threads>>>(out, 1, 0); });
    run("lds+sts random", [&] { k_ldssts<<<blocks, threads>>>(out, 1); });
    run("divergent branch", [&] { k_divbranch<<<blocks, threads>>>(out, 1); });
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
