// synth_gpu.cu -- seeded synthetic INPUT generator (GPU twin of synth.c).
//
// Harness code, not the product: it fills micro-gradient / theta0 buffers on
// the device so that full-size (GB-scale) inputs need not cross PCIe.  Same
// counter-based recipe as synth.c (see its header); the two are checked
// bit-for-bit against each other in tests/test_gpu_synth.py.  Holds none of
// the method's arithmetic.
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    uint64_t z = x + 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ int lanes_q(uint64_t h) {
    int s = (int)(h & 0xFFFF) + (int)((h >> 16) & 0xFFFF) + (int)((h >> 32) & 0xFFFF) +
            (int)((h >> 48) & 0xFFFF);
    return s - 131070;
}

__constant__ int c_log2_sigma[3] = {-5, -3, -7};
__constant__ int c_qt[3] = {-6, -4, -8};

// family: 0 real, 1 exact, 2 zero
__global__ void fill_kernel(uint16_t* __restrict__ out, int64_t begin, int64_t end, int family, int cls,
                            uint64_t key, int e, int K) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < end; i += stride) {
        uint16_t bits = 0;
        if (family != 2) {
            uint64_t h = mix(key ^ (uint64_t)i);
            float v;
            if (family == 0) {
                v = ldexpf((float)lanes_q(h), c_log2_sigma[cls] + e - 17);
            } else {
                int64_t kk = (int64_t)(h % (uint64_t)(2 * K + 1)) - K;
                int q = c_qt[cls] + e - 7;
                q = q < -24 ? -24 : (q > 4 ? 4 : q);
                v = ldexpf((float)kk, q);
            }
            bits = __half_as_ushort(__float2half_rn(v));
        }
        out[i] = bits;
    }
}

// one launch over the whole packed vector: each thread finds its tensor by binary search in a shared-memory
// copy of the tensor table (begin[0..nt], cls[0..nt-1])
__global__ void fill_all_kernel(uint16_t* __restrict__ out, int64_t n, const int64_t* __restrict__ tbegin,
                                const int32_t* __restrict__ tcls, int nt, int family, uint64_t key, int e, int K) {
    extern __shared__ int64_t sh[];
    int64_t* sb = sh;
    int32_t* sc = reinterpret_cast<int32_t*>(sh + nt + 1);
    for (int j = threadIdx.x; j <= nt; j += blockDim.x) sb[j] = tbegin[j];
    for (int j = threadIdx.x; j < nt; j += blockDim.x) sc[j] = tcls[j];
    __syncthreads();
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int lo = 0, hi = nt - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (sb[mid] <= i) lo = mid; else hi = mid - 1;
        }
        int cls = sc[lo];
        uint16_t bits = 0;
        if (family != 2) {
            uint64_t h = mix(key ^ (uint64_t)i);
            float v;
            if (family == 0) {
                v = ldexpf((float)lanes_q(h), c_log2_sigma[cls] + e - 17);
            } else {
                int64_t kk = (int64_t)(h % (uint64_t)(2 * K + 1)) - K;
                int q = c_qt[cls] + e - 7;
                q = q < -24 ? -24 : (q > 4 ? 4 : q);
                v = ldexpf((float)kk, q);
            }
            bits = __half_as_ushort(__float2half_rn(v));
        }
        out[i] = bits;
    }
}

__global__ void theta0_kernel(float* __restrict__ out, int64_t n, uint64_t key) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = ldexpf((float)lanes_q(mix(key ^ (uint64_t)i)), -21);
}

}  // namespace

extern "C" {

// Fill a packed device vector, one launch per tensor.  tensor_begin/cls are HOST arrays.
int synth_gpu_fill(uint16_t* dev_out, int n_tensors, const int64_t* tensor_begin, const int32_t* cls,
                   int family, uint64_t key, int e, int K, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    for (int j = 0; j < n_tensors; ++j) {
        int64_t b = tensor_begin[j], end = tensor_begin[j + 1];
        if (end <= b) continue;
        int64_t blocks = (end - b + 255) / 256;
        if (blocks > 148 * 32) blocks = 148 * 32;
        fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(dev_out, b, end, family, cls[j], key, e, K);
    }
    return (int)cudaGetLastError();
}

// Same values as synth_gpu_fill in one launch; tensor_begin (nt+1) / cls (nt) are DEVICE arrays.
int synth_gpu_fill_all(uint16_t* dev_out, int64_t n, const int64_t* dev_begin, const int32_t* dev_cls, int n_tensors,
                       int family, uint64_t key, int e, int K, void* stream) {
    size_t shmem = (size_t)(n_tensors + 1) * 8 + (size_t)n_tensors * 4;
    if (shmem > 48 * 1024) return -1;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    fill_all_kernel<<<(unsigned)blocks, 256, shmem, (cudaStream_t)stream>>>(dev_out, n, dev_begin, dev_cls, n_tensors,
                                                                          family, key, e, K);
    return (int)cudaGetLastError();
}

int synth_gpu_theta0(float* dev_out, int64_t n, uint64_t key, void* stream) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks < 1) blocks = 1;
    theta0_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dev_out, n, key);
    return (int)cudaGetLastError();
}

}  // extern "C"
