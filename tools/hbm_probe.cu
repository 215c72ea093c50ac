// hbm_probe.cu -- HBM ceilings for the access mixes of the update-step kernels, and K1/K2 design variants.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/hbm_probe.cu -o tools/hbm_probe
//   ./tools/hbm_probe            (on a B200; prints one line per variant: GB/s of algorithmic bytes)
//
// Mixes: read-only (sum), copy (1R1W), K1 add (2R1W fp16), K2-like (4R4W: 2+12 B in, 12+2 B out).
// Knobs: vector width (128/256-bit), units in flight per thread (U), CTAs per SM, cache hints.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

struct __align__(32) V8 { uint32_t w[8]; };

template <int HINT> __device__ __forceinline__ V8 ld(const void* p) {
    V8 r;
    if (HINT == 0)
        asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]) : "l"(p));
    else if (HINT == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]) : "l"(p));
    else
        asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]) : "l"(p));
    return r;
}
template <int HINT> __device__ __forceinline__ void st(void* p, const V8& v) {
    if (HINT == 2)
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7]) : "memory");
    else
        asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7]) : "memory");
}

// NR input streams, NW output streams of 32-byte units; out = xor of inputs (cheap ALU)
template <int NR, int NW, int U, int HINT>
__global__ void __launch_bounds__(256) mix(const V8* __restrict__ a, const V8* __restrict__ b, const V8* __restrict__ c,
                                           const V8* __restrict__ d, V8* o0, V8* o1, V8* o2, V8* o3, int64_t units,
                                           uint32_t* sink) {
    const V8* in[4] = {a, b, c, d};
    V8* out[4] = {o0, o1, o2, o3};
    int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < units; base += U * nthr) {
        V8 v[U][NR];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int r = 0; r < NR; ++r)
                if (base + u * nthr < units) v[u][r] = ld<HINT>(in[r] + base + u * nthr);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (base + u * nthr >= units) break;
            V8 x = v[u][0];
#pragma unroll
            for (int r = 1; r < NR; ++r)
#pragma unroll
                for (int j = 0; j < 8; ++j) x.w[j] ^= v[u][r].w[j];
            if (NW == 0) {
#pragma unroll
                for (int j = 0; j < 8; ++j) acc ^= x.w[j];
            }
#pragma unroll
            for (int w = 0; w < NW; ++w) st<HINT>(out[w] + base + u * nthr, x);
        }
    }
    if (NW == 0 && acc == 0x12345678u) *sink = acc;
}

template <int NR, int NW, int U, int HINT>
int run(const char* name, std::vector<V8*>& bufs, int64_t units, int ctas_per_sm, int sms, uint32_t* sink) {
    auto k = mix<NR, NW, U, HINT>;
    int grid = sms * ctas_per_sm;
    if (ctas_per_sm == 0) grid = (int)((units + 255) / 256);  // one unit per thread, non-persistent
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k<<<grid, 256>>>(bufs[0], bufs[1], bufs[2], bufs[3], bufs[4], bufs[5], bufs[6], bufs[7], units, sink);
    cudaEventRecord(e0);
    const int it = 20;
    for (int i = 0; i < it; ++i) k<<<grid, 256>>>(bufs[0], bufs[1], bufs[2], bufs[3], bufs[4], bufs[5], bufs[6], bufs[7], units, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)units * 32 * (NR + NW);
    printf("%-28s NR=%d NW=%d U=%d hint=%d ctas/sm=%d : %8.1f GB/s  (%.1f us)\n", name, NR, NW, U, HINT, ctas_per_sm,
           bytes * it / (ms * 1e-3) / 1e9, ms * 1e3 / it);
    return 0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t units = (int64_t)420 << 20 >> 5;   // 420 MiB per stream
    std::vector<V8*> bufs(8);
    for (auto& b : bufs) {
        CK(cudaMalloc(&b, units * 32));
        CK(cudaMemset(b, 1, units * 32));
    }
    uint32_t* sink;
    CK(cudaMalloc(&sink, 4));
    printf("SMs %d, %lld MiB per stream\n", sms, (long long)(units * 32 >> 20));
    for (int cps : {2, 4, 8, 0}) {
        run<1, 0, 2, 0>("read", bufs, units, cps, sms, sink);
        run<1, 1, 2, 0>("copy", bufs, units, cps, sms, sink);
        run<2, 1, 2, 0>("k1-like 2R1W", bufs, units, cps, sms, sink);
        run<4, 4, 1, 0>("k2-like 4R4W", bufs, units, cps, sms, sink);
    }
    for (int cps : {4, 8}) {
        run<1, 1, 4, 0>("copy U4", bufs, units, cps, sms, sink);
        run<2, 1, 4, 0>("k1-like U4", bufs, units, cps, sms, sink);
        run<2, 1, 2, 1>("k1-like L2::256B", bufs, units, cps, sms, sink);
        run<2, 1, 2, 2>("k1-like .cs", bufs, units, cps, sms, sink);
        run<4, 4, 2, 0>("k2-like U2", bufs, units, cps, sms, sink);
        run<4, 4, 1, 2>("k2-like .cs", bufs, units, cps, sms, sink);
    }
    return 0;
}
