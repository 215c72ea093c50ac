// nvlink_probe.cu -- the NVLink roofline for the bucket all-reduce: what SM loads / stores to a peer GPU move on
// this box (one process, cudaDeviceEnablePeerAccess, every GPU running the same kernel at once).
//
//   pull   each GPU reads its peer's buffer (256-bit loads, one unit per thread per iteration) and writes it locally
//   push   each GPU reads its own buffer and stores it into the peer's (256-bit stores)
//   pullpush  both at once, half the data each way: the all-reduce's traffic shape (k_ar32 at W = 2)
// GPU g's peer is g ^ 1 (pairs), so at W = 2 both directions of the one link are busy.  CUDA events, best of 5.
// Output: one JSON object per line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            fprintf(stderr, "%s: %s (%s:%d)\n", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

struct V8 {
    unsigned w[8];
};
__device__ __forceinline__ V8 ld256(const void* p) {
    V8 r;
    asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                   "=r"(r.w[6]), "=r"(r.w[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st256(void* p, const V8& v) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]),
                 "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}

// copy units [0, n) of 32 B from src to dst, U units in flight per thread
template <int U>
__global__ void copy32(const char* __restrict__ src, char* __restrict__ dst, long n) {
    const long tid = (long)blockIdx.x * blockDim.x + threadIdx.x, nthr = (long)gridDim.x * blockDim.x;
    for (long u = tid; u < n; u += U * nthr) {
        V8 a[U];
#pragma unroll
        for (int q = 0; q < U; ++q)
            if (u + q * nthr < n) a[q] = ld256(src + (u + q * nthr) * 32);
#pragma unroll
        for (int q = 0; q < U; ++q)
            if (u + q * nthr < n) st256(dst + (u + q * nthr) * 32, a[q]);
    }
}

int main(int argc, char** argv) {
    int ng = 0;
    CK(cudaGetDeviceCount(&ng));
    if (ng < 2) {
        printf("{\"error\": \"needs 2 GPUs\"}\n");
        return 0;
    }
    ng &= ~1;
    const size_t bytes = (size_t)(argc > 1 ? atol(argv[1]) : 512) << 20;
    std::vector<char*> own(ng), tmp(ng);
    std::vector<cudaStream_t> st(ng), st2(ng);
    std::vector<cudaEvent_t> f0(ng), f1(ng);
    std::vector<cudaEvent_t> e0(ng), e1(ng);
    int sms = 0;
    for (int g = 0; g < ng; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceEnablePeerAccess(g ^ 1, 0));
        CK(cudaMalloc(&own[g], bytes));
        CK(cudaMalloc(&tmp[g], bytes));
        CK(cudaMemset(own[g], g + 1, bytes));
        CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&st2[g], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&f0[g], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&f1[g], cudaEventDisableTiming));
        CK(cudaEventCreate(&e0[g]));
        CK(cudaEventCreate(&e1[g]));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g));
    }
    const long units = (long)(bytes / 32);
    auto run = [&](const char* mode, int ctas_per_sm, int threads, int unroll) {
        float best = 1e30f;
        for (int rep = 0; rep < 6; ++rep) {
            for (int g = 0; g < ng; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaDeviceSynchronize());
            }
            for (int g = 0; g < ng; ++g) {
                CK(cudaSetDevice(g));
                const int p = g ^ 1;
                CK(cudaEventRecord(e0[g], st[g]));
                const int grid = sms * ctas_per_sm;
                auto launch = [&](const char* s, char* d, long n, cudaStream_t q) {
                    if (unroll == 1) copy32<1><<<grid, threads, 0, q>>>(s, d, n);
                    else if (unroll == 2) copy32<2><<<grid, threads, 0, q>>>(s, d, n);
                    else copy32<4><<<grid, threads, 0, q>>>(s, d, n);
                };
                if (!strcmp(mode, "pull")) launch(own[p], tmp[g], units, st[g]);
                else if (!strcmp(mode, "push")) launch(own[g], tmp[p], units, st[g]);
                else {   // pullpush: the two halves concurrently, on two streams
                    CK(cudaEventRecord(f0[g], st[g]));
                    CK(cudaStreamWaitEvent(st2[g], f0[g], 0));
                    launch(own[p], tmp[g], units / 2, st[g]);
                    launch(own[g] + bytes / 2, tmp[p] + bytes / 2, units / 2, st2[g]);
                    CK(cudaEventRecord(f1[g], st2[g]));
                    CK(cudaStreamWaitEvent(st[g], f1[g], 0));
                }
                CK(cudaGetLastError());
                CK(cudaEventRecord(e1[g], st[g]));
            }
            float worst = 0;
            for (int g = 0; g < ng; ++g) {
                CK(cudaSetDevice(g));
                CK(cudaEventSynchronize(e1[g]));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
                if (ms > worst) worst = ms;
            }
            if (rep > 0 && worst < best) best = worst;
        }
        // bytes crossing the link in EACH direction per GPU pair: pull / push move `bytes` one way per GPU, i.e.
        // `bytes` per direction; pullpush moves bytes / 2 in, bytes / 2 out per GPU, again `bytes` per direction
        printf("{\"probe\": \"%s\", \"gpus\": %d, \"mib\": %zu, \"ctas_per_sm\": %d, \"threads\": %d, \"unroll\": %d, "
               "\"ms\": %.4f, \"per_direction_gbs\": %.1f}\n",
               mode, ng, bytes >> 20, ctas_per_sm, threads, unroll, best, bytes / (best * 1e-3) / 1e9);
        fflush(stdout);
    };
    for (const char* mode : {"pull", "push", "pullpush"})
        for (int cps : {1, 2, 4})
            for (int u : {1, 2, 4}) run(mode, cps, 256, u);
    return 0;
}
