/*
 * synth.c -- seeded synthetic INPUT generator (CPU side).
 *
 * This module is neither the oracle nor the product: it only produces the
 * inputs both of them consume (micro-gradients, token counts, initial
 * weights).  It holds none of the method's arithmetic (no accumulation, no
 * reduction, no scaler, no Adam).  The GPU twin is synth_gpu.cu; both
 * implement the same counter-based generator and are checked against each
 * other bit-for-bit and against the published SplitMix64 vectors
 * (tests/test_synth.py).  Recipe: DESIGN.md "Input recipe".
 *
 *   f(x)   = SplitMix64 output function applied to x + 0x9e3779b97f4a7c15
 *   key    = f(f(f(f(seed) ^ u) ^ r) ^ k)            (update u, rank r, micro k)
 *   h_i    = f(key ^ i)                              (packed element index i)
 *   G_real : q = sum of the four 16-bit lanes of h_i - 131070  (Irwin-Hall(4))
 *            g = rn16(q * 2^(log2sigma_t + e - 17))  (exact in fp32, one rounding)
 *   G_exact: K = floor(2048/(W*c)), kk = (h_i mod (2K+1)) - K
 *            g = kk * 2^clamp(q_t + e - 7, -24, 4)   (exact in fp16)
 *   theta0 : q * 2^-21 from key(seed, 0, 0xFFFF, 0)  (exact in fp32)
 *   ntokens: 2780 + (f(key ^ 0x5A5A5A5A) mod 721)    (uniform on [2780, 3500])
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC synth.c -o libsynth.so
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>

#define SYNTH_GOLDEN 0x9e3779b97f4a7c15ULL

enum { SYNTH_REAL = 0, SYNTH_EXACT = 1, SYNTH_ZERO = 2 };
/* tensor classes: 0 = weight matrix, 1 = bias / LayerNorm, 2 = embedding */
static const int k_log2_sigma[3] = {-5, -3, -7};
static const int k_qt[3] = {-6, -4, -8};

uint64_t synth_mix(uint64_t x) {
    uint64_t z = x + SYNTH_GOLDEN;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t synth_key(uint64_t seed, uint64_t u, uint64_t r, uint64_t k) {
    uint64_t c0 = synth_mix(seed);
    uint64_t c1 = synth_mix(c0 ^ u);
    uint64_t c2 = synth_mix(c1 ^ r);
    return synth_mix(c2 ^ k);
}

int64_t synth_ntokens(uint64_t key) {
    return 2780 + (int64_t)(synth_mix(key ^ 0x5A5A5A5AULL) % 721ULL);
}

static inline int32_t lanes_q(uint64_t h) {
    int32_t s = (int32_t)(h & 0xFFFF) + (int32_t)((h >> 16) & 0xFFFF) +
                (int32_t)((h >> 32) & 0xFFFF) + (int32_t)((h >> 48) & 0xFFFF);
    return s - 131070;
}

static inline uint16_t to_half_bits(float v) {
    _Float16 h = (_Float16)v;  /* libgcc round-to-nearest-even */
    uint16_t b;
    memcpy(&b, &h, 2);
    return b;
}

static inline uint16_t gen_elem(uint64_t key, int64_t i, int family, int cls, int e, int K) {
    if (family == SYNTH_ZERO) return 0;
    uint64_t h = synth_mix(key ^ (uint64_t)i);
    if (family == SYNTH_REAL) {
        float v = ldexpf((float)lanes_q(h), k_log2_sigma[cls] + e - 17);
        return to_half_bits(v);
    }
    int64_t kk = (int64_t)(h % (uint64_t)(2 * K + 1)) - K;
    int q = k_qt[cls] + e - 7;
    if (q < -24) q = -24;
    if (q > 4) q = 4;
    return to_half_bits(ldexpf((float)kk, q));
}

/* Fill the whole packed vector: tensors j = 0..n_tensors-1 occupy
 * [tensor_begin[j], tensor_begin[j+1]); cls[j] is the tensor class. */
void synth_fill(uint16_t* out, int n_tensors, const int64_t* tensor_begin, const int32_t* cls,
                int family, uint64_t key, int e, int K) {
    for (int j = 0; j < n_tensors; ++j) {
        int64_t b = tensor_begin[j], end = tensor_begin[j + 1];
        int c = cls[j];
#pragma omp parallel for schedule(static)
        for (int64_t i = b; i < end; ++i) out[i] = gen_elem(key, i, family, c, e, K);
    }
}

static int find_tensor(int n_tensors, const int64_t* tensor_begin, int64_t i) {
    int lo = 0, hi = n_tensors - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) / 2;
        if (tensor_begin[mid] <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
}

/* Elements [lo, hi) of the packed vector into out[0 .. hi-lo). */
void synth_fill_range(uint16_t* out, int64_t lo, int64_t hi, int n_tensors, const int64_t* tensor_begin,
                      const int32_t* cls, int family, uint64_t key, int e, int K) {
    for (int j = 0; j < n_tensors; ++j) {
        int64_t b = tensor_begin[j] > lo ? tensor_begin[j] : lo;
        int64_t end = tensor_begin[j + 1] < hi ? tensor_begin[j + 1] : hi;
        int c = cls[j];
#pragma omp parallel for schedule(static)
        for (int64_t i = b; i < end; ++i) out[i - lo] = gen_elem(key, i, family, c, e, K);
    }
}

/* Values at arbitrary packed indices idx[0..m). */
void synth_sample(uint16_t* out, const int64_t* idx, int64_t m, int n_tensors,
                  const int64_t* tensor_begin, const int32_t* cls, int family, uint64_t key, int e, int K) {
    for (int64_t j = 0; j < m; ++j) {
        int t = find_tensor(n_tensors, tensor_begin, idx[j]);
        out[j] = gen_elem(key, idx[j], family, cls[t], e, K);
    }
}

void synth_theta0(float* out, int64_t n, uint64_t key) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = ldexpf((float)lanes_q(synth_mix(key ^ (uint64_t)i)), -21);
}

void synth_theta0_sample(float* out, const int64_t* idx, int64_t m, uint64_t key) {
    for (int64_t j = 0; j < m; ++j) out[j] = ldexpf((float)lanes_q(synth_mix(key ^ (uint64_t)idx[j])), -21);
}

/* Row-sparse embedding gradient: only the rows of the micro-batch's token ids carry gradient.
 * mask[v] = 1 iff row v is among T token ids drawn i.i.d. from Zipf(s) over the V rows -- p(v) proportional to
 * (v + 1)^-s, row 0 the most frequent -- by inverse CDF with the uniform (f(key ^ (0xE3B0 << 32) ^ t) >> 11) * 2^-53
 * for draw t.  The mask is an input: the CPU and GPU fills both apply this one array.  Returns the distinct rows. */
int64_t synth_embed_rows(uint8_t* mask, int64_t V, uint64_t key, int64_t T, double s) {
    double* cdf = (double*)malloc((size_t)V * sizeof(double));
    if (!cdf) return -1;
    double acc = 0.0;
    for (int64_t v = 0; v < V; ++v) {
        acc += pow((double)(v + 1), -s);
        cdf[v] = acc;
    }
    memset(mask, 0, (size_t)V);
    int64_t distinct = 0;
    for (int64_t t = 0; t < T; ++t) {
        const double x = (double)(synth_mix(key ^ (0xE3B0ULL << 32) ^ (uint64_t)t) >> 11) * 0x1.0p-53 * acc;
        int64_t lo = 0, hi = V - 1;            /* first v with cdf[v] > x */
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (cdf[mid] > x) hi = mid;
            else lo = mid + 1;
        }
        distinct += !mask[lo];
        mask[lo] = 1;
    }
    free(cdf);
    return distinct;
}
