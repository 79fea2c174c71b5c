// probe: operand order of mov.b128 {a, b} (which half is a?) for atom.global.cas.b128
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long *p, unsigned long long *o) {
    unsigned long long lo = 0x1111, hi = 0x2222, olo, ohi;
    asm volatile("{\n\t.reg .b128 c, v, r;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %5};\n\t"
                 "atom.global.cas.b128 r, [%6], c, v;\n\tmov.b128 {%0, %1}, r;\n\t}"
                 : "=l"(olo), "=l"(ohi) : "l"(0ull), "l"(0ull), "l"(lo), "l"(hi), "l"(p) : "memory");
    o[0] = p[0]; o[1] = p[1];
}
int main() {
    unsigned long long *p, *o, h[2];
    cudaMalloc(&p, 16); cudaMalloc(&o, 16); cudaMemset(p, 0, 16);
    k<<<1, 1>>>(p, o);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("mem[0]=%llx mem[1]=%llx (lo operand 0x1111 first in {a,b})\n", h[0], h[1]);
}
