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

// h mod m for a modulus m < 2^16 with 32-bit operations only: the same value as the CPU's 64-bit `h % m`
// (h = hi 2^32 + lo, so h mod m = ((hi mod m) (2^32 mod m) + lo mod m) mod m; the product is < m^2 < 2^32)
__device__ __forceinline__ uint32_t mod_small(uint64_t h, uint32_t m, uint32_t two32_mod_m) {
    const uint32_t hi = (uint32_t)(h >> 32) % m, lo = (uint32_t)h % m;
    return ((hi * two32_mod_m) % m + lo) % m;
}

// 2^s exactly, for the normal range -126 <= s <= 127 (built from its exponent bits)
__device__ __forceinline__ float pow2f(int s) { return __int_as_float((s + 127) << 23); }

__device__ __forceinline__ uint16_t gen_bits(uint64_t key, int64_t i, int family, int cls, int e, int K,
                                             uint32_t two32_mod_m) {
    if (family == 2) return 0;
    const uint64_t h = mix(key ^ (uint64_t)i);
    float v;
    if (family == 0) {
        // q * 2^s with s = log2(sigma) + e - 17: a power-of-two scale, exact (same value as ldexpf)
        v = (float)lanes_q(h) * pow2f(c_log2_sigma[cls] + e - 17);
    } else {
        const int64_t kk = (int64_t)mod_small(h, (uint32_t)(2 * K + 1), two32_mod_m) - K;
        int q = c_qt[cls] + e - 7;
        q = q < -24 ? -24 : (q > 4 ? 4 : q);
        v = (float)kk * pow2f(q);
    }
    return __half_as_ushort(__float2half_rn(v));
}

// one launch over the whole packed vector: each thread makes 8 consecutive elements (one 16-byte store), finding
// its tensor once by binary search in a shared-memory copy of the tensor table (begin[0..nt], cls[0..nt-1])
__global__ void fill_all_kernel(uint16_t* __restrict__ out, int64_t n, const int64_t* __restrict__ tbegin,
                                const int32_t* __restrict__ tcls, int nt, int family, uint64_t key, int e, int K) {
    extern __shared__ int64_t sh[];
    int64_t* sb = sh;
    int32_t* sc = reinterpret_cast<int32_t*>(sh + nt + 1);
    for (int j = threadIdx.x; j <= nt; j += blockDim.x) sb[j] = tbegin[j];
    for (int j = threadIdx.x; j < nt; j += blockDim.x) sc[j] = tcls[j];
    __syncthreads();
    const uint32_t m = (uint32_t)(2 * K + 1);
    const uint32_t two32_mod_m = (uint32_t)((((uint64_t)1) << 32) % m);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i0 < n; i0 += stride) {
        int lo = 0, hi = nt - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (sb[mid] <= i0) lo = mid; else hi = mid - 1;
        }
        uint16_t b[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int64_t i = i0 + t;
            while (lo + 1 < nt && sb[lo + 1] <= i) ++lo;
            b[t] = i < n ? gen_bits(key, i, family, sc[lo], e, K, two32_mod_m) : 0;
        }
        if (i0 + 8 <= n && ((reinterpret_cast<uintptr_t>(out + i0) & 15) == 0)) {
            uint4 w;
            w.x = b[0] | ((uint32_t)b[1] << 16);
            w.y = b[2] | ((uint32_t)b[3] << 16);
            w.z = b[4] | ((uint32_t)b[5] << 16);
            w.w = b[6] | ((uint32_t)b[7] << 16);
            *reinterpret_cast<uint4*>(out + i0) = w;
        } else {
            for (int t = 0; t < 8 && i0 + t < n; ++t) out[i0 + t] = b[t];
        }
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
    if (family == 1 && (K < 0 || 2 * (int64_t)K + 1 >= 65536)) return -2;   // mod_small's range
    size_t shmem = (size_t)(n_tensors + 1) * 8 + (size_t)n_tensors * 4;
    if (shmem > 48 * 1024) return -1;
    int64_t blocks = (n + 8 * 256 - 1) / (8 * 256);
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
