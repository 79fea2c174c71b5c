// k_emit.cu — K5: decode the sorted keys of every length bucket into the output text
// ("The final step merges all the chunks and prints the results"; reading A12:
// one word per line). Word i of bucket L lands at byte byte_off[L] + (i - off[L]) * (L + 1), so no
// scan is needed. A tile decodes its keys into a shared-memory stage placed at the same 16-byte
// phase as its global destination and writes it out with aligned 16-byte stores.
#include <algorithm>

#include "wsort_internal.cuh"

namespace wsort {
namespace {

constexpr int kEThreads = 256;

__global__ void __launch_bounds__(kEThreads) k_emit(EmitArgs a) {
    __shared__ __align__(16) uint8_t stage[kEmitStage + 32];
    const int t = threadIdx.x;
    const TileDesc td = a.tile_pfx ? tile_from_prefix_cta(a.tile_pfx, blockIdx.x) : a.tiles[blockIdx.x];
    const uint32_t L = td.L;
    const BucketInfo b = a.buckets[L];
    const uint32_t te = kEmitStage / (L + 1);
    const uint32_t k0 = td.tile * te;
    const uint32_t nk = min(te, b.n - k0);
    const uint32_t kw = b.kw, es = b.estride;
    const uint32_t *keys = (b.final_b ? a.keys_b : a.keys_a) + b.elem_off;
    const uint64_t ob = b.byte_off + (uint64_t)k0 * (L + 1);
    const uint32_t head = (uint32_t)(ob & 15u);

    for (uint32_t k = t; k < nk; k += kEThreads) {
        uint8_t *o = stage + head + k * (L + 1);
        const uint32_t *kp = keys + (uint64_t)(k0 + k) * es;
        for (uint32_t q = 0; q < kw; q++) {
            const uint32_t word = __ldg(kp + q);
#pragma unroll
            for (int j = 0; j < 6; j++) {
                const uint32_t li = q * 6 + j;
                if (li < L) o[li] = (uint8_t)(((word >> (25 - 5 * j)) & 31u) | 0x60u);
            }
        }
        o[L] = '\n';
    }
    if (a.src_off) {
        uint64_t *so = a.src_off + b.word_off + k0;
        if (es > kw) {   // payload stored inline as the element's last word (variant A)
            for (uint32_t k = t; k < nk; k += kEThreads) so[k] = a.global_base + __ldg(keys + (uint64_t)(k0 + k) * es + kw);
        } else {
            const uint32_t *pay = (b.final_b ? a.pay_b : a.pay_a) + b.word_off + k0;
            for (uint32_t k = t; k < nk; k += kEThreads) so[k] = a.global_base + __ldg(pay + k);
        }
    }
    __syncthreads();

    const uint64_t total = (uint64_t)nk * (L + 1);
    const uint64_t end = ob + total;
    const uint64_t a0 = (ob + 15) & ~15ull, a1 = end & ~15ull;
    if (a0 >= a1) {  // no full aligned chunk
        for (uint64_t x = ob + t; x < end; x += kEThreads) a.words[x] = stage[head + (x - ob)];
        return;
    }
    for (uint64_t x = ob + t; x < a0; x += kEThreads) a.words[x] = stage[head + (x - ob)];
    for (uint64_t x = a1 + t; x < end; x += kEThreads) a.words[x] = stage[head + (x - ob)];
    const uint64_t base16 = ob & ~15ull;   // stage offset of global address x is x - base16
    uint4 *dst = reinterpret_cast<uint4 *>(a.words);
    for (uint64_t x = a0 + 16ull * t; x < a1; x += 16ull * kEThreads)
        dst[x >> 4] = *reinterpret_cast<const uint4 *>(stage + (x - base16));
}

}  // namespace

// Small host<->device copies done by SM loads/stores through UVA-mapped pinned host memory instead of
// a copy engine: the copy engines stay free for the bulk text / output transfers (whose queue a
// few-KB table would otherwise wait behind).
__global__ void k_copy_small(uint8_t *dst, const uint8_t *src, size_t n) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)dst | (uintptr_t)src | n) & 15u) == 0) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (size_t i = t; i < n / 16; i += stride) d4[i] = s4[i];
    } else {
        for (size_t i = t; i < n; i += stride) dst[i] = src[i];
    }
}

// Several small host tables (pinned arena) -> device in one launch: block (x, y) copies part x of table y.
__global__ void k_copy_batch(CopyBatch b) {
    const uint32_t y = blockIdx.y;
    const uint8_t *src = static_cast<const uint8_t *>(b.src[y]);
    uint8_t *dst = static_cast<uint8_t *>(b.dst[y]);
    const size_t n = b.bytes[y], t = (size_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)dst | (uintptr_t)src) & 15u) == 0) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (size_t i = t; i < n / 16; i += stride) d4[i] = s4[i];
        for (size_t i = (n & ~(size_t)15) + t; i < n; i += stride) dst[i] = src[i];
    } else {
        for (size_t i = t; i < n; i += stride) dst[i] = src[i];
    }
}
cudaError_t launch_copy_batch(const CopyBatch &b, cudaStream_t s) {
    if (!b.n) return cudaSuccess;
    size_t mx = 0;
    for (uint32_t i = 0; i < b.n; i++) mx = b.bytes[i] > mx ? b.bytes[i] : mx;
    const uint32_t gx = (uint32_t)std::min<size_t>(64, (mx + 4095) / 4096);
    k_copy_batch<<<dim3(gx ? gx : 1, b.n), 256, 0, s>>>(b);
    return cudaGetLastError();
}

cudaError_t launch_emit(const EmitArgs &a, cudaStream_t s) {
    if (a.ntiles == 0) return cudaSuccess;
    k_emit<<<a.ntiles, kEThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t copy_small(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (!bytes) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<size_t>((bytes + 4095) / 4096, 64);
    k_copy_small<<<grid, 256, 0, s>>>(static_cast<uint8_t *>(dst), static_cast<const uint8_t *>(src), bytes);
    return cudaGetLastError();
}

}  // namespace wsort
