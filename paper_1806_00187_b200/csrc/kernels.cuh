// kernels.cuh -- the sm_100a kernels of the update step (private to libsmpu.so).
//
//   K1   accumulate   A = g (first micro-batch) | A = rn16(A + g) (later ones), optional overflow test of
//                     the OUTPUT A (finite + finite can overflow: 65504 + 16 -> inf).
//   K1s  sweep        overflow test of the reduced R, W > 1, only when the early decision was undecided.  P:158, R4
//   K0   decide       one thread: overflow -> skip/apply, dynamic loss scaler, t, lr(t), Adam scalars, result
//                     record, next loss scale.  W = 1: from K1's flag.  W > 1: EARLY from an all-reduced
//                     (N, sum_r max|A_r|) pair before the gradient all-reduces finish (exact, see k0_early),
//                     LATE from the K1s sweep in the rare undecided case.
//   K2   adam         fused unscale + normalise by N + Adam (fp32 master) + fp16 re-cast, per bucket right
//                     behind that bucket's all-reduce (W > 1) or whole (W = 1); every CTA exits before any
//                     store when K0 decided to skip.
//   K12  fused        W = 1 (fuse_final): the last micro-batch's K1 add fused into K2, computed speculatively into
//                     a second bank of theta/m/v (k12_fused, k12_fused_many); kc_restore re-casts w16 on a skip.
//   K1 fp32           accum_fp32 (SURVEY Z1 knob): fp32 sums, rn16 of the last one into the fp16 accumulator.
//   Kc   cast         w16 = rn16(theta) (init / set_state only).
//
// All of them are HBM-streaming: 256-bit (v8.b32) global accesses (sm_100a LDG/STG.256), L1 no-allocate,
// grid-stride over 32-byte vector units with two units in flight per thread.  Overflow test on packed
// fp16 words: ((w & 0x7C007C00) + 0x04000400) & 0x80008000 is non-zero iff a half has exponent 0x1F.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "smpu.h"

#ifndef SMPU_K1_MINB
#define SMPU_K1_MINB 6   // min resident CTAs/SM for the one-shot K1 (register cap 40); 8 forces 32 registers
#endif

namespace smpu {

struct __align__(32) V8 { uint32_t w[8]; };   // 32 B: 16 halves or 8 floats
struct __align__(16) V4 { uint32_t w[4]; };   // 16 B: 8 halves

// ---------------------------------------------------------------------------------------------- memory ops
// L2 cache-hint experiments (tools/experiments/l2_hints.sh): SMPU_L2_HINT=1 adds the 256-B L2 prefetch-size
// hint to every 256-bit load, =2 marks every 256-bit load and store L2::evict_first.  Default: no hint.
#ifndef SMPU_L2_HINT
#define SMPU_L2_HINT 0
#endif
#if SMPU_L2_HINT == 1
#define SMPU_LDH ".L2::256B"
#define SMPU_STH ""
#elif SMPU_L2_HINT == 2
#define SMPU_LDH ".L2::evict_first"
#define SMPU_STH ".L2::evict_first"
#else
#define SMPU_LDH ""
#define SMPU_STH ""
#endif
__device__ __forceinline__ V8 ld256_ro(const void* p) {          // read-only for the whole kernel
    V8 r;
    asm volatile("ld.global.nc.L1::no_allocate" SMPU_LDH ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                   "=r"(r.w[6]), "=r"(r.w[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ V8 ld256(const void* p) {             // read then written by the same thread
    V8 r;
    asm volatile("ld.global.L1::no_allocate" SMPU_LDH ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                   "=r"(r.w[6]), "=r"(r.w[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st256(void* p, const V8& v) {
    asm volatile("st.global.L1::no_allocate" SMPU_STH ".v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]),
                 "r"(v.w[1]), "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}
__device__ __forceinline__ V4 ld128_ro(const void* p) {
    V4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st128(void* p, const V4& v) {
    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
                 "r"(v.w[2]), "r"(v.w[3])
                 : "memory");
}

// Programmatic dependent launch (sm_90+): `pdl_trigger` lets the next kernel of the stream start its CTAs while
// this one finishes its last wave; `pdl_wait` blocks until the previous kernel has completed and its memory is
// visible.  Every kernel below waits before its first global load or store -- the caller's micro-gradient
// included, since the kernel that wrote it may itself trigger early.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// fp16x2 add, round-to-nearest-even, never contracted (reading R1)
__device__ __forceinline__ uint32_t hadd2_rn(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t nonfinite_bits(uint32_t w) {
    return ((w & 0x7C007C00u) + 0x04000400u) & 0x80008000u;
}
__device__ __forceinline__ bool h_nonfinite(uint16_t h) { return (h & 0x7C00u) == 0x7C00u; }

__device__ __forceinline__ void raise_flag(bool bad, int* flag) {
    // one store per warp that saw a non-finite value; every writer stores 1, so no atomics are needed
    unsigned any = __ballot_sync(0xffffffffu, bad);
    if (any && (threadIdx.x & 31) == (unsigned)(__ffs(any) - 1)) *(volatile int*)flag = 1;
}

// max of the fp16 magnitudes (bits & 0x7FFF, monotone in |x|; >= 0x7C00 iff non-finite) of a packed word
__device__ __forceinline__ uint32_t mag_max2(uint32_t m, uint32_t w) { return __vmaxu2(m, w & 0x7FFF7FFFu); }

// CTA-wide max, then at most one atomicMax per CTA and only when it raises the running maximum (a read of
// the L2-resident value first): one atomic per warp on a single address serialises at its L2 slice (measured
// 2.5x slower final-micro K1 at W = 2).  Every thread of the CTA must call it.
__device__ __forceinline__ void publish_max(uint32_t m2, uint32_t* stat) {
    __shared__ uint32_t s_m[32];
    uint32_t m = max(m2 & 0xFFFFu, m2 >> 16);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, s_m[w]);
        if (m > *(volatile uint32_t*)stat) atomicMax(stat, m);
    }
}

// ---------------------------------------------------------------------------------------------- K1
// acc[lo, hi) (absolute indices) <- g[0, hi-lo) (+ acc).  Vector path when acc+i and g+(i-lo) are
// both 32-B aligned at the first 16-element boundary i >= lo, else an element path (correct, slower).
// DETECT: flag |= any non-finite output (W = 1 last micro-batch).  STATS: *stat = max(*stat, max fp16
// magnitude bits of the output) (W > 1 last micro-batch: input of the early overflow decision, K0 EARLY).
template <bool FIRST, bool DETECT, bool STATS = false>
__global__ void __launch_bounds__(256) k1_accumulate(uint16_t* __restrict__ acc, const uint16_t* __restrict__ g,
                                                     int64_t lo, int64_t hi, int* __restrict__ flag,
                                                     uint32_t* __restrict__ stat = nullptr) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const uint16_t* gb = g - lo;                       // gb[i] is the gradient of element i
    int64_t vbeg = (lo + 15) & ~(int64_t)15;
    if (vbeg > hi) vbeg = hi;
    bool vec_ok = ((reinterpret_cast<uintptr_t>(gb + vbeg) & 31) == 0);
    int64_t nvec = vec_ok ? (hi - vbeg) / 16 : 0;
    int64_t vend = vbeg + nvec * 16;
    uint32_t bad = 0, mx = 0;
    if (vec_ok) {
        // body: 16 halves per unit, two units per thread in flight
        int64_t u = tid;
        for (; u + nthr < nvec; u += 2 * nthr) {
            const int64_t i0 = vbeg + u * 16, i1 = vbeg + (u + nthr) * 16;
            V8 g0 = ld256_ro(gb + i0), g1 = ld256_ro(gb + i1);
            if (!FIRST) {
                V8 a0 = ld256(acc + i0), a1 = ld256(acc + i1);
#pragma unroll
                for (int j = 0; j < 8; ++j) { g0.w[j] = hadd2_rn(a0.w[j], g0.w[j]); g1.w[j] = hadd2_rn(a1.w[j], g1.w[j]); }
            }
            if (DETECT) {
#pragma unroll
                for (int j = 0; j < 8; ++j) bad |= nonfinite_bits(g0.w[j]) | nonfinite_bits(g1.w[j]);
            }
            if (STATS) {
#pragma unroll
                for (int j = 0; j < 8; ++j) mx = mag_max2(mag_max2(mx, g0.w[j]), g1.w[j]);
            }
            st256(acc + i0, g0);
            st256(acc + i1, g1);
        }
        if (u < nvec) {
            const int64_t i0 = vbeg + u * 16;
            V8 g0 = ld256_ro(gb + i0);
            if (!FIRST) {
                V8 a0 = ld256(acc + i0);
#pragma unroll
                for (int j = 0; j < 8; ++j) g0.w[j] = hadd2_rn(a0.w[j], g0.w[j]);
            }
            if (DETECT) {
#pragma unroll
                for (int j = 0; j < 8; ++j) bad |= nonfinite_bits(g0.w[j]);
            }
            if (STATS) {
#pragma unroll
                for (int j = 0; j < 8; ++j) mx = mag_max2(mx, g0.w[j]);
            }
            st256(acc + i0, g0);
        }
    }
    // element path: head [lo, vbeg) and tail [vend, hi) -- or everything when not co-aligned
    auto elem = [&](int64_t i) {
        uint16_t x = gb[i];
        if (!FIRST) {
            uint32_t s = hadd2_rn((uint32_t)acc[i], (uint32_t)x);
            x = (uint16_t)(s & 0xFFFFu);
        }
        if (DETECT && h_nonfinite(x)) bad |= 1u;
        if (STATS) mx = mag_max2(mx, (uint32_t)x);   // per lane: mx holds two packed magnitudes
        acc[i] = x;
    };
    if (vec_ok) {
        for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
        for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
    } else {
        for (int64_t i = lo + tid; i < hi; i += nthr) elem(i);
    }
    if (DETECT) raise_flag(bad != 0, flag);
    if (STATS) publish_max(mx, stat);
}

// One-shot K1: exactly one 16-half unit per thread, grid = ceil(units / 256), no loop, registers capped for
// 6+ resident CTAs per SM.  Maximum thread-level parallelism is what saturates HBM on this access mix
// (tools/hbm_probe.cu: 2R1W one-shot 6.3-6.8 TB/s vs 6.2 for the 4-CTA/SM persistent loop).  The element
// path (unaligned head / tail / not co-aligned) is taken by the first threads of the grid.
template <bool FIRST, bool DETECT, bool STATS>
__global__ void __launch_bounds__(256, SMPU_K1_MINB) k1_accumulate_1(uint16_t* __restrict__ acc, const uint16_t* __restrict__ g,
                                                          int64_t lo, int64_t hi, int* __restrict__ flag,
                                                          uint32_t* __restrict__ stat) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const uint16_t* gb = g - lo;
    int64_t vbeg = (lo + 15) & ~(int64_t)15;
    if (vbeg > hi) vbeg = hi;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(gb + vbeg) & 31) == 0);
    const int64_t nvec = vec_ok ? (hi - vbeg) / 16 : 0;
    const int64_t vend = vbeg + nvec * 16;
    uint32_t bad = 0, mx = 0;
    pdl_trigger();
    // Nothing is loaded before the wait, not even the caller's gradient: its writer may be a PDL-aware kernel
    // (a CUTLASS / cuBLASLt GEMM) that lets this kernel start before its epilogue stores land.
    pdl_wait();
    if (tid < nvec) {
        const int64_t i0 = vbeg + tid * 16;
        V8 g0 = ld256_ro(gb + i0);
        if (!FIRST) {
            V8 a0 = ld256(acc + i0);
#pragma unroll
            for (int j = 0; j < 8; ++j) g0.w[j] = hadd2_rn(a0.w[j], g0.w[j]);
        }
        if (DETECT) {
#pragma unroll
            for (int j = 0; j < 8; ++j) bad |= nonfinite_bits(g0.w[j]);
        }
        if (STATS) {
#pragma unroll
            for (int j = 0; j < 8; ++j) mx = mag_max2(mx, g0.w[j]);
        }
        st256(acc + i0, g0);
    }
    auto elem = [&](int64_t i) {
        uint16_t x = gb[i];
        if (!FIRST) x = (uint16_t)(hadd2_rn((uint32_t)acc[i], (uint32_t)x) & 0xFFFFu);
        if (DETECT && h_nonfinite(x)) bad |= 1u;
        if (STATS) mx = mag_max2(mx, (uint32_t)x);   // per lane: mx holds two packed magnitudes
        acc[i] = x;
    };
    if (vec_ok) {
        for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
        for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
    } else {
        for (int64_t i = lo + tid; i < hi; i += nthr) elem(i);
    }
    if (DETECT) raise_flag(bad != 0, flag);
    if (STATS) publish_max(mx, stat);
}

// K1 over several resident micro-batches in one pass (smpu_accumulate_many): per element
// x = [first ? g_0 : rn16(A + g_0)], then x = rn16(x + g_k) for k = 1..count-1 in order, one store -- the
// same additions in the same order as `count` K1 launches, bitwise, but each gradient is read once and the
// accumulator is read/written once: 2 count + 2 (or + 4) bytes per element instead of 6 count (-2).
constexpr int kMaxMany = 32;
struct ManyPtrs {
    const uint16_t* g[kMaxMany];   // g[k][i - lo] is micro-batch k's gradient of element i
};

template <bool FIRST, bool DETECT, bool STATS>
__global__ void __launch_bounds__(256, 4) k1_accumulate_many(uint16_t* __restrict__ acc, ManyPtrs P, int count,
                                                             int64_t lo, int64_t hi, int* __restrict__ flag,
                                                             uint32_t* __restrict__ stat) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t vbeg = (lo + 15) & ~(int64_t)15;
    if (vbeg > hi) vbeg = hi;
    bool vec_ok = true;
    for (int k = 0; k < count; ++k) vec_ok &= ((reinterpret_cast<uintptr_t>(P.g[k] + (vbeg - lo)) & 31) == 0);
    const int64_t nvec = vec_ok ? (hi - vbeg) / 16 : 0;
    const int64_t vend = vbeg + nvec * 16;
    uint32_t bad = 0, mx = 0;
    pdl_trigger();
    pdl_wait();
    if (tid < nvec) {
        const int64_t i0 = vbeg + tid * 16, r0 = i0 - lo;
        V8 x;
        int k = 0;
        if (FIRST) {
            x = ld256_ro(P.g[0] + r0);
            k = 1;
        } else {
            x = ld256(acc + i0);
        }
        // four gradients in flight at a time, added strictly in micro-batch order
        for (; k < count; k += 4) {
            V8 y[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < count) y[j] = ld256_ro(P.g[k + j] + r0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < count) {
#pragma unroll
                    for (int w = 0; w < 8; ++w) x.w[w] = hadd2_rn(x.w[w], y[j].w[w]);
                }
        }
        if (DETECT) {
#pragma unroll
            for (int w = 0; w < 8; ++w) bad |= nonfinite_bits(x.w[w]);
        }
        if (STATS) {
#pragma unroll
            for (int w = 0; w < 8; ++w) mx = mag_max2(mx, x.w[w]);
        }
        st256(acc + i0, x);
    }
    auto elem = [&](int64_t i) {
        uint32_t x = FIRST ? (uint32_t)P.g[0][i - lo] : (uint32_t)acc[i];
        for (int k = FIRST ? 1 : 0; k < count; ++k) x = hadd2_rn(x, (uint32_t)P.g[k][i - lo]) & 0xFFFFu;
        if (DETECT && h_nonfinite((uint16_t)x)) bad |= 1u;
        if (STATS) mx = mag_max2(mx, (uint32_t)x);   // per lane: mx holds two packed magnitudes
        acc[i] = (uint16_t)x;
    };
    if (vec_ok) {
        for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
        for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
    } else {
        for (int64_t i = lo + tid; i < hi; i += nthr) elem(i);
    }
    if (DETECT) raise_flag(bad != 0, flag);
    if (STATS) publish_max(mx, stat);
}

// Scan of the accumulator itself, for micro-batches the producer accumulated in place (a weight-
// gradient GEMM adding its output into smpu_accumulator with beta = 1): the overflow test (W = 1) or the max
// |A| statistic (W > 1) that K1 would have fused, 2 bytes per element, one-shot.
template <bool DETECT, bool STATS>
__global__ void __launch_bounds__(256) k1_scan(const uint16_t* __restrict__ acc, int64_t lo, int64_t hi,
                                               int* __restrict__ flag, uint32_t* __restrict__ stat) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t vbeg = (lo + 15) & ~(int64_t)15;
    if (vbeg > hi) vbeg = hi;
    const int64_t nvec = (hi - vbeg) / 16, vend = vbeg + nvec * 16;
    uint32_t bad = 0, mx = 0;
    if (tid < nvec) {
        V8 a = ld256_ro(acc + vbeg + tid * 16);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (DETECT) bad |= nonfinite_bits(a.w[j]);
            if (STATS) mx = mag_max2(mx, a.w[j]);
        }
    }
    auto elem = [&](int64_t i) {
        uint16_t x = acc[i];
        if (DETECT && h_nonfinite(x)) bad |= 1u;
        if (STATS) mx = mag_max2(mx, (uint32_t)x);   // per lane: mx holds two packed magnitudes
    };
    for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
    for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
    if (DETECT) raise_flag(bad != 0, flag);
    if (STATS) publish_max(mx, stat);
}

// ---------------------------------------------------------------------------------------------- K1 (fp32 acc.)
// smpu_config.accum_fp32 (SURVEY Z1 knob; oracle.c orc_accumulate32): an fp32 accumulator A32 instead of fp16.
//   MODE 0  A32 = fp32(g)                       first micro-batch                         6 B/element
//   MODE 1  A32 = fl32(A32 + fp32(g))           later ones                               10 B/element
//   MODE 2  acc16 = rn16(fl32(A32 + fp32(g)))   the last one: the rank's fp16 gradient    8 B/element
//   MODE 3  acc16 = rn16(A32)                   the last one, accumulated in place        6 B/element
// The fp16 output of modes 2/3 is what K1's last micro-batch would have written (overflow test / max |A| on it);
// everything downstream (all-reduce, decision, Adam) is unchanged.  16 elements per thread, one-shot grid.
template <int MODE, bool DETECT, bool STATS>
__global__ void __launch_bounds__(256, SMPU_K1_MINB) k1_acc32(float* __restrict__ A32, uint16_t* __restrict__ acc16,
                                                              const uint16_t* __restrict__ g, int64_t lo, int64_t hi,
                                                              int* __restrict__ flag, uint32_t* __restrict__ stat) {
    constexpr bool HAS_G = MODE != 3;
    constexpr bool OUT16 = MODE >= 2;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const uint16_t* gb = g - lo;
    int64_t vbeg = (lo + 15) & ~(int64_t)15;
    if (vbeg > hi) vbeg = hi;
    const bool vec_ok = !HAS_G || ((reinterpret_cast<uintptr_t>(gb + vbeg) & 31) == 0);
    const int64_t nvec = vec_ok ? (hi - vbeg) / 16 : 0;
    const int64_t vend = vbeg + nvec * 16;
    uint32_t bad = 0, mx = 0;
    if (tid < nvec) {
        const int64_t i0 = vbeg + tid * 16;
        V8 gv, a0, a1;
        if (HAS_G) gv = ld256_ro(gb + i0);
        if (MODE != 0) {
            a0 = ld256(A32 + i0);
            a1 = ld256(A32 + i0 + 8);
        }
        if (MODE == 0 || MODE == 1 || MODE == 2) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float2 gf = __half22float2(*reinterpret_cast<const __half2*>(&gv.w[j]));
                V8& a = j < 4 ? a0 : a1;
                const int w = 2 * (j & 3);
                if (MODE == 0) {
                    a.w[w] = __float_as_uint(gf.x);
                    a.w[w + 1] = __float_as_uint(gf.y);
                } else {
                    a.w[w] = __float_as_uint(__fadd_rn(__uint_as_float(a.w[w]), gf.x));
                    a.w[w + 1] = __float_as_uint(__fadd_rn(__uint_as_float(a.w[w + 1]), gf.y));
                }
            }
        }
        if (OUT16) {
            V8 h;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const V8& a = j < 4 ? a0 : a1;
                const int w = 2 * (j & 3);
                __half2 hh = __floats2half2_rn(__uint_as_float(a.w[w]), __uint_as_float(a.w[w + 1]));
                h.w[j] = *reinterpret_cast<uint32_t*>(&hh);
                if (DETECT) bad |= nonfinite_bits(h.w[j]);
                if (STATS) mx = mag_max2(mx, h.w[j]);
            }
            st256(acc16 + i0, h);
        } else {
            st256(A32 + i0, a0);
            st256(A32 + i0 + 8, a1);
        }
    }
    auto elem = [&](int64_t i) {
        float a = MODE == 0 ? 0.0f : A32[i];
        if (HAS_G) {
            const float gf = __half2float(__ushort_as_half(gb[i]));
            a = MODE == 0 ? gf : __fadd_rn(a, gf);
        }
        if (OUT16) {
            const uint16_t x = __half_as_ushort(__float2half_rn(a));
            if (DETECT && h_nonfinite(x)) bad |= 1u;
            if (STATS) mx = mag_max2(mx, (uint32_t)x);   // per lane: mx holds two packed magnitudes
            acc16[i] = x;
        } else {
            A32[i] = a;
        }
    };
    if (vec_ok) {
        for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
        for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
    } else {
        for (int64_t i = lo + tid; i < hi; i += nthr) elem(i);
    }
    if (DETECT) raise_flag(bad != 0, flag);
    if (STATS) publish_max(mx, stat);
}

// ---------------------------------------------------------------------------------------------- K1s
struct Scalars;
__device__ __forceinline__ int32_t decision_of(const Scalars* sc);

// only when the early decision could not decide (K0 EARLY wrote UNDECIDED); otherwise returns at once
__global__ void __launch_bounds__(256) k1s_sweep(const uint16_t* __restrict__ R, int64_t lo, int64_t hi,
                                                 int* __restrict__ flag, const Scalars* __restrict__ sc) {
    if (decision_of(sc) != 2) return;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t vbeg = (lo + 15) & ~(int64_t)15;
    if (vbeg > hi) vbeg = hi;
    int64_t nvec = (hi - vbeg) / 16, vend = vbeg + nvec * 16;
    uint32_t bad = 0;
    int64_t u = tid;
    for (; u + nthr < nvec; u += 2 * nthr) {
        V8 a = ld256_ro(R + vbeg + u * 16), b = ld256_ro(R + vbeg + (u + nthr) * 16);
#pragma unroll
        for (int j = 0; j < 8; ++j) bad |= nonfinite_bits(a.w[j]) | nonfinite_bits(b.w[j]);
    }
    if (u < nvec) {
        V8 a = ld256_ro(R + vbeg + u * 16);
#pragma unroll
        for (int j = 0; j < 8; ++j) bad |= nonfinite_bits(a.w[j]);
    }
    for (int64_t i = lo + tid; i < vbeg; i += nthr) bad |= h_nonfinite(R[i]);
    for (int64_t i = vend + tid; i < hi; i += nthr) bad |= h_nonfinite(R[i]);
    raise_flag(bad != 0, flag);
}

// ---------------------------------------------------------------------------------------------- K0
struct DevState {          // device-resident scaler / optimizer counters
    int64_t e;             // scale exponent (scale = 2^e)
    int64_t clean;         // consecutive clean updates
    int64_t t;             // applied updates
    int64_t attempts;      // update attempts
    int64_t bank;          // fused final micro-batch (W = 1): which copy of theta/m/v is current (0 / 1)
};

// decision states (Scalars::state)
enum : int32_t { DEC_APPLY = 0, DEC_SKIP = 1, DEC_UNDECIDED = 2, DEC_APPLY_LATE = 3 };

struct Scalars {           // written by K0, read by every K2 CTA
    int32_t state;         // DEC_*
    float inv_sN;          // fp32(1 / (2^e * N))
    float step;            // fp32(lr / bc1)
    float inv_sqrt_bc2;    // fp32(1 / sqrt(bc2))
    float b1, omb1, b2, omb2, eps;
};

__device__ __forceinline__ int32_t decision_of(const Scalars* sc) { return *(volatile const int32_t*)&sc->state; }

struct DevCfg {
    double peak_lr;
    int64_t warmup;
    double beta1, beta2, eps;
    int32_t emin, emax;
    int64_t growth;
};

// lr(t) = peak * min(t / warmup, sqrt(warmup / t)) in fp64 (IEEE div/sqrt/mul, no contraction), one
// rounding to fp32 (reading R14).
__device__ __forceinline__ float lr_at(int64_t t, const DevCfg& c) {
    double tt = (double)t, w = (double)c.warmup;
    double lin = __ddiv_rn(tt, w);
    double isq = __dsqrt_rn(__ddiv_rn(w, tt));
    double f = lin < isq ? lin : isq;
    return __double2float_rn(__dmul_rn(c.peak_lr, f));
}

// Adam scalars of applied update t, from the exponent e the gradients carry (before growth) and N.
__device__ void adam_scalars(int64_t t, int32_t e, int64_t N, float lr, const DevCfg& cfg, Scalars* sc) {
    double sN = ldexp((double)N, (int)e);
    double bc1 = 1.0 - pow(cfg.beta1, (double)t);
    double bc2 = 1.0 - pow(cfg.beta2, (double)t);
    sc->inv_sN = __double2float_rn(1.0 / sN);
    sc->step = __double2float_rn((double)lr / bc1);
    sc->inv_sqrt_bc2 = __double2float_rn(1.0 / sqrt(bc2));
    sc->b1 = (float)cfg.beta1;
    sc->omb1 = (float)(1.0 - cfg.beta1);
    sc->b2 = (float)cfg.beta2;
    sc->omb2 = (float)(1.0 - cfg.beta2);
    sc->eps = (float)cfg.eps;
}

// The scaler step + Adam scalars + result record, once per update attempt.
// Returns the decision state written (DEC_APPLY / DEC_SKIP; apply_state for a late decision).
__device__ void decide(int overflow, int64_t N, DevState* st, Scalars* sc, float* loss_scale,
                       smpu_step_result* ring, int ring_mask, const DevCfg& cfg, int32_t apply_state) {
    DevState s = *st;
    smpu_step_result r;
    r.attempt = ++s.attempts;
    r.overflow = overflow;
    r.scale_log2_used = (int32_t)s.e;
    r.ntokens_total = N;
    r.discarded = 0;
    int32_t state;
    if (N <= 0) {                                      // reading R19: nothing changes
        state = DEC_SKIP;
        r.discarded = 1;
        r.applied = 0;
        r.lr = lr_at(s.t + 1, cfg);
    } else if (overflow) {                             // P:158 "scales down the loss when overflow is detected"
        state = DEC_SKIP;
        s.e = s.e - 1 < cfg.emin ? cfg.emin : s.e - 1;
        s.clean = 0;
        r.applied = 0;
        r.lr = lr_at(s.t + 1, cfg);                    // reading R15
    } else {
        state = apply_state;
        s.t += 1;
        s.clean += 1;
        r.applied = 1;
        r.lr = lr_at(s.t, cfg);
        adam_scalars(s.t, r.scale_log2_used, N, r.lr, cfg, sc);
        if (s.clean >= cfg.growth) {                   // P:158 "scales the loss up if no overflows ... 2,000"
            s.e = s.e + 1 > cfg.emax ? cfg.emax : s.e + 1;
            s.clean = 0;
        }
    }
    sc->state = state;
    r.scale_log2_next = (int32_t)s.e;
    r.num_updates = s.t;
    r.clean_streak = s.clean;
    *st = s;
    *loss_scale = ldexpf(1.0f, (int)s.e);
    ring[(r.attempt - 1) & ring_mask] = r;             // mapped pinned host memory
    __threadfence_system();
}

// W = 1: the last K1 tested the reduced (= local) gradient exactly.
// tok_ptr != nullptr (CUDA-graph replays): the token count is read from the device at run time
// fused: the update ran speculatively (k12_fused wrote the other bank); applying = making that bank current.
__global__ void k0_decide(int* __restrict__ flag, int64_t tokens, const int64_t* __restrict__ tok_ptr,
                          DevState* __restrict__ st, Scalars* __restrict__ sc, float* __restrict__ loss_scale,
                          smpu_step_result* __restrict__ ring, int ring_mask, DevCfg cfg, int fused = 0) {
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (tok_ptr) tokens = *tok_ptr;
    const int overflow = *(volatile int*)flag != 0;
    *(volatile int*)flag = 0;                          // re-armed for the next update
    decide(overflow, tokens, st, sc, loss_scale, ring, ring_mask, cfg, DEC_APPLY);
    if (fused && sc->state == DEC_APPLY) st->bank ^= 1;
}

// W = 1 with the fused final micro-batch: before it, the Adam scalars of update t+1 as if it will apply (the
// same fp64 arithmetic as decide()); N = 0 (discarded) turns k12_fused off.
__global__ void k0_fused_prep(int64_t tokens, const int64_t* __restrict__ tok_ptr, const DevState* __restrict__ st,
                              Scalars* __restrict__ sc, DevCfg cfg) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (tok_ptr) tokens = *tok_ptr;
    const DevState s = *st;
    if (tokens <= 0) {
        sc->state = DEC_SKIP;
        return;
    }
    adam_scalars(s.t + 1, (int32_t)s.e, tokens, lr_at(s.t + 1, cfg), cfg, sc);
    sc->state = DEC_APPLY;
}

// W > 1, before the gradient all-reduces finish.  xs = {N, sum_r M_r} summed over ranks by one int64
// all-reduce, M_r = rank r's max |A_r| in units of 2^-24 (or kNonFinite if A_r holds inf/NaN).
//   some A_r non-finite            => R non-finite in every order            => overflow (exact)
//   sum_r M_r <= 2^15 (all finite) => every partial sum of any order and width stays < 65520 (W-1 roundings
//                                     add at most 16 each) => R finite       => clean (exact)
//   otherwise                      => UNDECIDED: the sweep of R (K1s) and K0 LATE decide after the reduce.
// Overflow <=> "R holds a non-finite element" (reading R4) holds in all three cases.
constexpr int64_t kNonFinite = int64_t(1) << 50;   // > 1024 ranks x 2^40 (65504 in units of 2^-24)
__device__ __forceinline__ int64_t mag_units(uint32_t bits) {
    if (bits >= 0x7C00u) return kNonFinite;
    int ex = (int)(bits >> 10), man = (int)(bits & 0x3FF);
    return ex == 0 ? (int64_t)man : ((int64_t)(1024 + man)) << (ex - 1);   // |x| / 2^-24
}

__global__ void k_stats_prep(uint32_t* __restrict__ stat, int64_t local_tokens, const int64_t* __restrict__ tok_ptr,
                             int64_t* __restrict__ xs) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    xs[0] = tok_ptr ? *tok_ptr : local_tokens;
    xs[1] = mag_units(*stat);
    *stat = 0;                                         // re-armed for the next update
}

__global__ void k0_early(const int64_t* __restrict__ xs, DevState* __restrict__ st, Scalars* __restrict__ sc,
                         float* __restrict__ loss_scale, smpu_step_result* __restrict__ ring, int ring_mask,
                         DevCfg cfg) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t N = xs[0], M = xs[1];
    if (M >= kNonFinite) decide(1, N, st, sc, loss_scale, ring, ring_mask, cfg, DEC_APPLY);
    else if (M <= (int64_t(1) << 39)) decide(0, N, st, sc, loss_scale, ring, ring_mask, cfg, DEC_APPLY);
    else sc->state = DEC_UNDECIDED;                    // 2^39 units = 2^15
}

// W > 1, after every all-reduce and (if undecided) the K1s sweeps.
__global__ void k0_late(int* __restrict__ flag, const int64_t* __restrict__ xs, DevState* __restrict__ st,
                        Scalars* __restrict__ sc, float* __restrict__ loss_scale, smpu_step_result* __restrict__ ring,
                        int ring_mask, DevCfg cfg) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (sc->state == DEC_UNDECIDED) {
        const int overflow = *(volatile int*)flag != 0;
        decide(overflow, xs[0], st, sc, loss_scale, ring, ring_mask, cfg, DEC_APPLY_LATE);
    }
    *(volatile int*)flag = 0;
}

// ---------------------------------------------------------------------------------------------- K2
// Per element (Kingma & Ba Alg. 1 in torch's arrangement, reading R13):
//   g = fp32(R) * inv_sN;  m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2
//   theta -= step * m / (sqrt(v) * inv_sqrt_bc2 + eps);  w16 = rn16(theta)
// Every rounding spelled out with _rn intrinsics: left to the compiler, `a * b + c` is contracted into an FMA
// differently in the vector and the element paths (seen on hardware as 1-ulp differences of m and v between
// a bucket's aligned body and its unaligned head), and every path must give the same bits for an element.
__device__ __forceinline__ void adam_elem(float R, float& th, float& m, float& v, const Scalars& s) {
    const float g = __fmul_rn(R, s.inv_sN);
    m = __fmaf_rn(s.b1, m, __fmul_rn(s.omb1, g));
    v = __fmaf_rn(s.b2, v, __fmul_rn(s.omb2, __fmul_rn(g, g)));
    const float denom = __fmaf_rn(__fsqrt_rn(v), s.inv_sqrt_bc2, s.eps);
    th = __fmaf_rn(-s.step, __fdiv_rn(m, denom), th);
}

__device__ __forceinline__ void adam_unit(const V4& r16, V8& th, V8& m, V8& v, V4& w16, const Scalars& s) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        __half2 rh = *reinterpret_cast<const __half2*>(&r16.w[j]);
        float2 rf = __half22float2(rh);
        float t0 = __uint_as_float(th.w[2 * j]), t1 = __uint_as_float(th.w[2 * j + 1]);
        float m0 = __uint_as_float(m.w[2 * j]), m1 = __uint_as_float(m.w[2 * j + 1]);
        float v0 = __uint_as_float(v.w[2 * j]), v1 = __uint_as_float(v.w[2 * j + 1]);
        adam_elem(rf.x, t0, m0, v0, s);
        adam_elem(rf.y, t1, m1, v1, s);
        th.w[2 * j] = __float_as_uint(t0);
        th.w[2 * j + 1] = __float_as_uint(t1);
        m.w[2 * j] = __float_as_uint(m0);
        m.w[2 * j + 1] = __float_as_uint(m1);
        v.w[2 * j] = __float_as_uint(v0);
        v.w[2 * j + 1] = __float_as_uint(v1);
        __half2 wh = __floats2half2_rn(t0, t1);
        w16.w[j] = *reinterpret_cast<uint32_t*>(&wh);
    }
}

// Elements [lo, hi) of the ctx arrays (a bucket, or everything).  Runs only when K0 wrote `need`
// (DEC_APPLY for the exact early / W = 1 decision, DEC_APPLY_LATE for the fallback); on a skip every CTA
// returns before any store (R6).  Vector units of 8 elements start at the first multiple of 8 >= lo
// (the arrays are 256-B aligned), head and tail take the element path.
__global__ void __launch_bounds__(256) k2_adam(float* __restrict__ theta, float* __restrict__ m,
                                               float* __restrict__ v, uint16_t* __restrict__ w16,
                                               const uint16_t* __restrict__ R, int64_t lo, int64_t hi,
                                               const Scalars* __restrict__ scp, int32_t need) {
    if (decision_of(scp) != need) return;
    const Scalars s = *scp;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t vbeg = (lo + 7) & ~(int64_t)7;
    if (vbeg > hi) vbeg = hi;
    const int64_t nvec = (hi - vbeg) / 8, vend = vbeg + nvec * 8;
    int64_t u = tid;
    for (; u + nthr < nvec; u += 2 * nthr) {
        const int64_t i0 = vbeg + u * 8, i1 = vbeg + (u + nthr) * 8;
        V4 r0 = ld128_ro(R + i0), r1 = ld128_ro(R + i1);
        V8 t0 = ld256(theta + i0), t1 = ld256(theta + i1);
        V8 m0 = ld256(m + i0), m1 = ld256(m + i1);
        V8 v0 = ld256(v + i0), v1 = ld256(v + i1);
        V4 w0, w1;
        adam_unit(r0, t0, m0, v0, w0, s);
        adam_unit(r1, t1, m1, v1, w1, s);
        st256(theta + i0, t0);
        st256(m + i0, m0);
        st256(v + i0, v0);
        st128(w16 + i0, w0);
        st256(theta + i1, t1);
        st256(m + i1, m1);
        st256(v + i1, v1);
        st128(w16 + i1, w1);
    }
    if (u < nvec) {
        const int64_t i0 = vbeg + u * 8;
        V4 r0 = ld128_ro(R + i0);
        V8 t0 = ld256(theta + i0), m0 = ld256(m + i0), v0 = ld256(v + i0);
        V4 w0;
        adam_unit(r0, t0, m0, v0, w0, s);
        st256(theta + i0, t0);
        st256(m + i0, m0);
        st256(v + i0, v0);
        st128(w16 + i0, w0);
    }
    auto elem = [&](int64_t i) {
        float th = theta[i], mm = m[i], vv = v[i];
        adam_elem(__half2float(__ushort_as_half(R[i])), th, mm, vv, s);
        theta[i] = th;
        m[i] = mm;
        v[i] = vv;
        w16[i] = __half_as_ushort(__float2half_rn(th));
    };
    for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
    for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
}

// One-shot K2: exactly one 8-element unit per thread (112 B in flight), registers capped for 4 resident CTAs
// per SM; same arithmetic as k2_adam (adam_unit / adam_elem).
__global__ void __launch_bounds__(256, 4) k2_adam_1(float* __restrict__ theta, float* __restrict__ m,
                                                    float* __restrict__ v, uint16_t* __restrict__ w16,
                                                    const uint16_t* __restrict__ R, int64_t lo, int64_t hi,
                                                    const Scalars* __restrict__ scp, int32_t need) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t vbeg = (lo + 7) & ~(int64_t)7;
    if (vbeg > hi) vbeg = hi;
    const int64_t nvec = (hi - vbeg) / 8, vend = vbeg + nvec * 8;
    pdl_trigger();
    // No load before the wait: with small grids every kernel of the chain triggers its dependent at once, so
    // the previous update's Adam (the last writer of theta/m/v) may still be running here.
    pdl_wait();
    if (decision_of(scp) != need) return;
    const Scalars s = *scp;
    if (tid < nvec) {
        const int64_t i0 = vbeg + tid * 8;
        V8 t0 = ld256(theta + i0), m0 = ld256(m + i0), v0 = ld256(v + i0);
        V4 r0 = ld128_ro(R + i0);
        V4 w0;
        adam_unit(r0, t0, m0, v0, w0, s);
        st256(theta + i0, t0);
        st256(m + i0, m0);
        st256(v + i0, v0);
        st128(w16 + i0, w0);
    }
    auto elem = [&](int64_t i) {
        float th = theta[i], mm = m[i], vv = v[i];
        adam_elem(__half2float(__ushort_as_half(R[i])), th, mm, vv, s);
        theta[i] = th;
        m[i] = mm;
        v[i] = vv;
        w16[i] = __half_as_ushort(__float2half_rn(th));
    };
    for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
    for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
}

// ---------------------------------------------------------------------------------------------- K12
// W = 1: the last micro-batch's accumulation fused into Adam (30 instead of 6 + 28 bytes per element; 28 at
// c = 1).  Per element R = [HAS_ACC ? A : g_0] (+ g_k for the rest, in order, fp16 RNE: K1's additions), then
// exactly K2's arithmetic (adam_unit / adam_elem).  Speculative: the overflow decision needs all of R, so the
// update is computed from bank b of theta/m/v into bank 1-b and K0 makes it current only if R was finite; w16
// is written in place and re-cast from the current bank on a skip (kc_restore).  R itself is never stored.
// one element of K12 (heads, tails, misaligned buffers); returns the non-finite bit of R
template <bool HAS_ACC>
__device__ __forceinline__ uint32_t k12_elem(int64_t i, const uint16_t* __restrict__ acc, const ManyPtrs& P, int count,
                                             int64_t lo, const float* ti, const float* mi, const float* vi, float* to,
                                             float* mo, float* vo, uint16_t* __restrict__ w16, const Scalars& s) {
    uint32_t x = HAS_ACC ? (uint32_t)acc[i] : (uint32_t)P.g[0][i - lo];
    for (int k = HAS_ACC ? 0 : 1; k < count; ++k) x = hadd2_rn(x, (uint32_t)P.g[k][i - lo]) & 0xFFFFu;
    float th = ti[i], mm = mi[i], vv = vi[i];
    adam_elem(__half2float(__ushort_as_half((uint16_t)x)), th, mm, vv, s);
    to[i] = th;
    mo[i] = mm;
    vo[i] = vv;
    w16[i] = __half_as_ushort(__float2half_rn(th));
    return h_nonfinite((uint16_t)x) ? 1u : 0u;
}

template <bool HAS_ACC>
__global__ void __launch_bounds__(256, 4) k12_fused(const uint16_t* __restrict__ acc, ManyPtrs P, int count,
                                                    int64_t lo, int64_t hi, float* th0, float* m0, float* v0,
                                                    float* th1, float* m1, float* v1, uint16_t* __restrict__ w16,
                                                    const DevState* __restrict__ st, const Scalars* __restrict__ scp,
                                                    int* __restrict__ flag) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t vbeg = (lo + 7) & ~(int64_t)7;
    if (vbeg > hi) vbeg = hi;
    bool vec_ok = true;
    for (int k = 0; k < count; ++k) vec_ok &= ((reinterpret_cast<uintptr_t>(P.g[k] + (vbeg - lo)) & 15) == 0);
    const int64_t nvec = vec_ok ? (hi - vbeg) / 8 : 0, vend = vbeg + nvec * 8;
    // Issue order matters (the asm loads are volatile, so they stay in program order): the accumulator and the
    // first gradients do not depend on the decision state or the bank, so they go first and are in flight
    // while those are read; theta/m/v follow before any add, so one thread never waits for two latencies.
    const int k0 = HAS_ACC ? 0 : 1;
    const int64_t i0 = vbeg + tid * 8, r0 = i0 - lo;
    V4 x, y[4];
    if (tid < nvec) {
        x = HAS_ACC ? ld128_ro(acc + i0) : ld128_ro(P.g[0] + r0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (k0 + j < count) y[j] = ld128_ro(P.g[k0 + j] + r0);
    }
    if (decision_of(scp) != DEC_APPLY) return;         // N = 0: the update is discarded
    const Scalars s = *scp;
    const bool b = st->bank != 0;
    const float* __restrict__ ti = b ? th1 : th0;
    const float* __restrict__ mi = b ? m1 : m0;
    const float* __restrict__ vi = b ? v1 : v0;
    float* __restrict__ to = b ? th0 : th1;
    float* __restrict__ mo = b ? m0 : m1;
    float* __restrict__ vo = b ? v0 : v1;
    uint32_t bad = 0;
    if (tid < nvec) {
        V8 t = ld256_ro(ti + i0), m = ld256_ro(mi + i0), v = ld256_ro(vi + i0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (k0 + j < count) {
#pragma unroll
                for (int w = 0; w < 4; ++w) x.w[w] = hadd2_rn(x.w[w], y[j].w[w]);
            }
        for (int k = k0 + 4; k < count; k += 4) {     // resident micro-batches beyond the first four
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < count) y[j] = ld128_ro(P.g[k + j] + r0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < count) {
#pragma unroll
                    for (int w = 0; w < 4; ++w) x.w[w] = hadd2_rn(x.w[w], y[j].w[w]);
                }
        }
#pragma unroll
        for (int w = 0; w < 4; ++w) bad |= nonfinite_bits(x.w[w]);
        V4 w16v;
        adam_unit(x, t, m, v, w16v, s);
        st256(to + i0, t);
        st256(mo + i0, m);
        st256(vo + i0, v);
        st128(w16 + i0, w16v);
    }
    auto elem = [&](int64_t i) { bad |= k12_elem<HAS_ACC>(i, acc, P, count, lo, ti, mi, vi, to, mo, vo, w16, s); };
    if (vec_ok) {
        for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
        for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
    } else {
        for (int64_t i = lo + tid; i < hi; i += nthr) elem(i);
    }
    raise_flag(bad != 0, flag);
}

// K12 over several resident micro-batches (smpu_accumulate_many's last call, count >= 4): 16-element units so
// that every gradient load is 32 B and four of them are in flight per round, as in k1_accumulate_many; the sum
// is then consumed by two 8-element Adam halves (theta/m/v are loaded only after the gradients, which keeps
// the registers under the 4-CTA cap).  Same additions in the same order and the same Adam arithmetic.
template <bool HAS_ACC>
__global__ void __launch_bounds__(256, 4) k12_fused_many(const uint16_t* __restrict__ acc, ManyPtrs P, int count,
                                                         int64_t lo, int64_t hi, float* th0, float* m0, float* v0,
                                                         float* th1, float* m1, float* v1,
                                                         uint16_t* __restrict__ w16, const DevState* __restrict__ st,
                                                         const Scalars* __restrict__ scp, int* __restrict__ flag) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t vbeg = (lo + 15) & ~(int64_t)15;
    if (vbeg > hi) vbeg = hi;
    bool vec_ok = true;
    for (int k = 0; k < count; ++k) vec_ok &= ((reinterpret_cast<uintptr_t>(P.g[k] + (vbeg - lo)) & 31) == 0);
    const int64_t nvec = vec_ok ? (hi - vbeg) / 16 : 0, vend = vbeg + nvec * 16;
    const int k0 = HAS_ACC ? 0 : 1;
    const int64_t i0 = vbeg + tid * 16, r0 = i0 - lo;
    V8 x, y[4];
    if (tid < nvec) {      // independent of the decision state and the bank: in flight while those are read
        x = HAS_ACC ? ld256_ro(acc + i0) : ld256_ro(P.g[0] + r0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (k0 + j < count) y[j] = ld256_ro(P.g[k0 + j] + r0);
    }
    if (decision_of(scp) != DEC_APPLY) return;         // N = 0: the update is discarded
    const Scalars s = *scp;
    const bool b = st->bank != 0;
    const float* __restrict__ ti = b ? th1 : th0;
    const float* __restrict__ mi = b ? m1 : m0;
    const float* __restrict__ vi = b ? v1 : v0;
    float* __restrict__ to = b ? th0 : th1;
    float* __restrict__ mo = b ? m0 : m1;
    float* __restrict__ vo = b ? v0 : v1;
    uint32_t bad = 0;
    if (tid < nvec) {
        for (int k = k0;; ) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < count) {
#pragma unroll
                    for (int w = 0; w < 8; ++w) x.w[w] = hadd2_rn(x.w[w], y[j].w[w]);
                }
            k += 4;
            if (k >= count) break;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < count) y[j] = ld256_ro(P.g[k + j] + r0);
        }
#pragma unroll
        for (int w = 0; w < 8; ++w) bad |= nonfinite_bits(x.w[w]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t j0 = i0 + 8 * h;
            V8 t = ld256_ro(ti + j0), m = ld256_ro(mi + j0), v = ld256_ro(vi + j0);
            V4 xr, w16v;
#pragma unroll
            for (int w = 0; w < 4; ++w) xr.w[w] = x.w[4 * h + w];
            adam_unit(xr, t, m, v, w16v, s);
            st256(to + j0, t);
            st256(mo + j0, m);
            st256(vo + j0, v);
            st128(w16 + j0, w16v);
        }
    }
    auto elem = [&](int64_t i) { bad |= k12_elem<HAS_ACC>(i, acc, P, count, lo, ti, mi, vi, to, mo, vo, w16, s); };
    if (vec_ok) {
        for (int64_t i = lo + tid; i < vbeg; i += nthr) elem(i);
        for (int64_t i = vend + tid; i < hi; i += nthr) elem(i);
    } else {
        for (int64_t i = lo + tid; i < hi; i += nthr) elem(i);
    }
    raise_flag(bad != 0, flag);
}

// After a skipped fused update: w16 = rn16(current theta) again (k12_fused wrote it speculatively).  Returns at
// once unless K0 decided to skip.
__global__ void __launch_bounds__(256) kc_restore(const float* __restrict__ th0, const float* __restrict__ th1,
                                                  const DevState* __restrict__ st, const Scalars* __restrict__ scp,
                                                  uint16_t* __restrict__ w16, int64_t n) {
    if (decision_of(scp) != DEC_SKIP) return;
    const float* __restrict__ th = st->bank ? th1 : th0;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nthr)
        w16[i] = __half_as_ushort(__float2half_rn(th[i]));
}

// ---------------------------------------------------------------------------------------------- Kc
__global__ void kc_cast(const float* __restrict__ theta, uint16_t* __restrict__ w16, int64_t n) {
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nthr)
        w16[i] = __half_as_ushort(__float2half_rn(theta[i]));
}

}  // namespace smpu
