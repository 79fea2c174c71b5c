// Microbenchmark: global / shared-memory counting atomics under skewed (Zipf-like) key streams —
// the primitive of dense-key counting for short words.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_atom tools/ubench_atom.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_red_global(const uint32_t *__restrict__ keys, size_t n, uint32_t *table) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += s) atomicAdd(&table[keys[i]], 1u);
}

// warp pre-aggregation: lanes with equal keys add once
__global__ void k_red_global_match(const uint32_t *__restrict__ keys, size_t n, uint32_t *table) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    for (; i - threadIdx.x % 32 < n; i += s) {
        bool v = i < n;
        uint32_t k = v ? keys[i] : 0xffffffffu;
        uint32_t peers = __match_any_sync(0xffffffffu, k);
        if (v && (threadIdx.x % 32) == __ffs(peers) - 1) atomicAdd(&table[k], __popc(peers));
    }
}

// per-CTA shared-memory table of T entries, flushed (non-zero only) at the end
template <int T>
__global__ void k_smem_count(const uint32_t *__restrict__ keys, size_t n, uint32_t *table) {
    extern __shared__ uint32_t h[];
    for (int j = threadIdx.x; j < T; j += blockDim.x) h[j] = 0;
    __syncthreads();
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += s) atomicAdd(&h[keys[i] % T], 1u);
    __syncthreads();
    for (int j = threadIdx.x; j < T; j += blockDim.x)
        if (h[j]) atomicAdd(&table[j], h[j]);
}

__global__ void k_read(const uint32_t *__restrict__ keys, size_t n, uint32_t *table) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (; i < n; i += s) acc += keys[i];
    if (acc == 0x12345678u) table[0] = acc;
}

static std::vector<uint32_t> zipf_keys(size_t n, int types, double s, uint32_t space, uint32_t seed) {
    std::mt19937_64 g(seed);
    std::vector<double> cdf(types);
    double acc = 0;
    for (int r = 0; r < types; r++) cdf[r] = (acc += std::pow(r + 1.0, -s));
    std::vector<uint32_t> ids(types);
    for (int r = 0; r < types; r++) ids[r] = (uint32_t)(g() % space);
    std::vector<uint32_t> k(n);
    std::uniform_real_distribution<double> u(0, acc);
    for (size_t i = 0; i < n; i++) {
        size_t r = std::lower_bound(cdf.begin(), cdf.end(), u(g)) - cdf.begin();
        k[i] = ids[r < (size_t)types ? r : types - 1];
    }
    return k;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t n = 32u << 20;
    uint32_t *d_keys, *d_table;
    cudaMalloc(&d_keys, n * 4);
    cudaMalloc(&d_table, (size_t)12u << 22);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Dist {
        const char *name;
        int types;
        double s;
        uint32_t space;
    } dists[] = {{"uniform 457k", 0, 0, 456976},      {"zipf 167 types (L=4)", 167, 0.9, 456976},
                 {"zipf 45 types (L=3)", 45, 1.1, 17576}, {"zipf 12 types (L=2)", 12, 1.1, 676},
                 {"2 types (L=1)", 2, 1.1, 26},        {"uniform 11.9M (L=5)", 0, 0, 11881376},
                 {"zipf 531 types in 11.9M", 531, 0.9, 11881376}};
    for (auto &d : dists) {
        std::vector<uint32_t> k;
        if (d.types == 0) {
            std::mt19937 g(7);
            k.resize(n);
            for (auto &x : k) x = g() % d.space;
        } else {
            k = zipf_keys(n, d.types, d.s, d.space, 11);
        }
        cudaMemcpy(d_keys, k.data(), n * 4, cudaMemcpyHostToDevice);
        auto run = [&](const char *what, auto launch) {
            cudaMemset(d_table, 0, (size_t)d.space * 4);
            launch();
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int r = 0; r < 5; r++) launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 5;
            printf("%-26s %-22s %8.3f ms  %7.2f G ops/s\n", d.name, what, ms, n / (ms * 1e6));
        };
        const int grid = sms * 8;
        run("read only", [&] { k_read<<<grid, 256>>>(d_keys, n, d_table); });
        run("global red", [&] { k_red_global<<<grid, 256>>>(d_keys, n, d_table); });
        run("global red + match", [&] { k_red_global_match<<<grid, 256>>>(d_keys, n, d_table); });
        if (d.space <= 17576) {
            cudaFuncSetAttribute(k_smem_count<17576>, cudaFuncAttributeMaxDynamicSharedMemorySize, 17576 * 4);
            run("smem 17576 (1 CTA/SM)", [&] { k_smem_count<17576><<<sms, 1024, 17576 * 4>>>(d_keys, n, d_table); });
            run("smem 17576 (2 CTA/SM)", [&] { k_smem_count<17576><<<2 * sms, 512, 17576 * 4>>>(d_keys, n, d_table); });
        }
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
