// tma_probe.cu -- is a 1-D bulk-copy (cp.async.bulk, "TMA") pipeline faster than one-shot LDG.256 for the
// K2 access mix (4 input streams: 2+12 B, 4 output streams: 12+2 B per element)?  Same arithmetic-free mix as
// hbm_probe's "k2-like": out = xor of inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_probe.cu -o tools/tma_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(b)),
                 "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// chunk = E elements; per stage: R (2E B), theta/m/v (4E B each)
template <int E, int STAGES>
__global__ void __launch_bounds__(256, 1) k2_tma(const uint16_t* R, float* th, float* m, float* v, uint16_t* w16,
                                                 int64_t n) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
    uint8_t* data = sm + 128;
    constexpr int STAGE_BYTES = E * 14;
    const int64_t nchunks = n / E;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t c, int s) {
        uint8_t* st = data + s * STAGE_BYTES;
        mbar_expect_tx(&bars[s], STAGE_BYTES);
        bulk_g2s(st, R + c * E, E * 2, &bars[s]);
        bulk_g2s(st + E * 2, th + c * E, E * 4, &bars[s]);
        bulk_g2s(st + E * 6, m + c * E, E * 4, &bars[s]);
        bulk_g2s(st + E * 10, v + c * E, E * 4, &bars[s]);
    };
    int64_t first = blockIdx.x;
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s)
            if (first + (int64_t)s * gridDim.x < nchunks) issue(first + (int64_t)s * gridDim.x, s);
    uint32_t phase = 0;
    int s = 0;
    for (int64_t c = first; c < nchunks; c += gridDim.x) {
        mbar_wait(&bars[s], phase);
        uint8_t* st = data + s * STAGE_BYTES;
        const uint16_t* r = reinterpret_cast<const uint16_t*>(st);
        const float* t = reinterpret_cast<const float*>(st + E * 2);
        const float* mm = reinterpret_cast<const float*>(st + E * 6);
        const float* vv = reinterpret_cast<const float*>(st + E * 10);
        for (int i = threadIdx.x * 4; i < E; i += blockDim.x * 4) {
            float4 a = *reinterpret_cast<const float4*>(t + i);
            float4 b = *reinterpret_cast<const float4*>(mm + i);
            float4 d = *reinterpret_cast<const float4*>(vv + i);
            uint2 rr = *reinterpret_cast<const uint2*>(r + i);
            int64_t g = c * E + i;
            *reinterpret_cast<float4*>(th + g) = make_float4(a.x + 1, a.y + 1, a.z + 1, a.w + 1);
            *reinterpret_cast<float4*>(m + g) = b;
            *reinterpret_cast<float4*>(v + g) = d;
            *reinterpret_cast<uint2*>(w16 + g) = rr;
        }
        __syncthreads();   // everyone done with stage s
        if (threadIdx.x == 0) {
            int64_t nc = c + (int64_t)STAGES * gridDim.x;
            if (nc < nchunks) issue(nc, s);
        }
        if (++s == STAGES) { s = 0; phase ^= 1; }
    }
}

// reference: one-shot LDG.128 version of the same mix
__global__ void __launch_bounds__(256) k2_ldg(const uint16_t* R, float* th, float* m, float* v, uint16_t* w16, int64_t n) {
    int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i >= n) return;
    float4 a = *reinterpret_cast<const float4*>(th + i);
    float4 b = *reinterpret_cast<const float4*>(m + i);
    float4 d = *reinterpret_cast<const float4*>(v + i);
    uint2 rr = *reinterpret_cast<const uint2*>(R + i);
    *reinterpret_cast<float4*>(th + i) = make_float4(a.x + 1, a.y + 1, a.z + 1, a.w + 1);
    *reinterpret_cast<float4*>(m + i) = b;
    *reinterpret_cast<float4*>(v + i) = d;
    *reinterpret_cast<uint2*>(w16 + i) = rr;
}

template <typename F>
float time_it(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 20;
}

template <int E, int ST>
int run_tma(int ctas_per_sm, int sms, const uint16_t* R, float* th, float* m, float* v, uint16_t* w, int64_t n) {
    size_t smem = 128 + (size_t)ST * E * 14;
    CK(cudaFuncSetAttribute(k2_tma<E, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    float ms = time_it([&] { k2_tma<E, ST><<<sms * ctas_per_sm, 256, smem>>>(R, th, m, v, w, n); });
    CK(cudaGetLastError());
    printf("tma E=%d stages=%d ctas/sm=%d smem=%zu: %.1f GB/s (%.1f us)\n", E, ST, ctas_per_sm, smem,
           28.0 * n / (ms * 1e-3) / 1e9, ms * 1e3);
    return 0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t n = 209911808 / 8192 * 8192;
    uint16_t *R, *w;
    float *th, *m, *v;
    CK(cudaMalloc(&R, n * 2));
    CK(cudaMalloc(&w, n * 2));
    CK(cudaMalloc(&th, n * 4));
    CK(cudaMalloc(&m, n * 4));
    CK(cudaMalloc(&v, n * 4));
    cudaMemset(R, 0, n * 2);
    cudaMemset(th, 0, n * 4);
    cudaMemset(m, 0, n * 4);
    cudaMemset(v, 0, n * 4);
    float ms = time_it([&] { k2_ldg<<<(unsigned)((n / 4 + 255) / 256), 256>>>(R, th, m, v, w, n); });
    printf("ldg one-shot 128-bit: %.1f GB/s (%.1f us)\n", 28.0 * n / (ms * 1e-3) / 1e9, ms * 1e3);
    run_tma<2048, 3>(2, sms, R, th, m, v, w, n);
    run_tma<2048, 4>(1, sms, R, th, m, v, w, n);
    run_tma<4096, 3>(1, sms, R, th, m, v, w, n);
    run_tma<1024, 4>(3, sms, R, th, m, v, w, n);
    run_tma<1024, 6>(2, sms, R, th, m, v, w, n);
    return 0;
}
