// Probe: k1_accumulate_1<FIRST, DETECT=false, STATS=true> over [lo, hi) with an INF at one element; prints the stat.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1806_00187_b200/csrc/kernels.cuh"
using namespace smpu;
int main() {
    const int n = 32;
    uint16_t h[n];
    for (int i = 0; i < n; ++i) h[i] = 0x3c00;   // 1.0
    h[1] = 0x7c00;
    uint16_t *g, *acc; int* flag; uint32_t* stat;
    cudaMalloc(&g, 4096); cudaMalloc(&acc, 4096); cudaMalloc(&flag, 4); cudaMalloc(&stat, 4);
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    struct { int lo, hi; } cases[] = {{0, 1}, {1, 32}, {0, 32}, {1, 16}, {0, 16}, {16, 32}};
    for (auto c : cases) {
        cudaMemset(stat, 0, 4);
        cudaMemset(acc, 0, 4096);
        k1_accumulate_1<true, false, true><<<1, 256>>>(acc, g + c.lo, c.lo, c.hi, flag, stat);
        k1_accumulate<true, false, true><<<1, 256>>>(acc, g + c.lo, c.lo, c.hi, flag, stat);
        uint32_t s = 0; uint16_t a[n];
        cudaMemcpy(&s, stat, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(a, acc, sizeof a, cudaMemcpyDeviceToHost);
        printf("[%d,%d): stat %#x acc[1] %#x err %s\n", c.lo, c.hi, s, a[1], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
