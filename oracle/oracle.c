/*
 * oracle.c -- CPU ORACLE for the synchronous mixed-precision large-batch update
 * step of Ott et al., "Scaling Neural Machine Translation" (arXiv 1806.00187).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product (paper_1806_00187_b200/, libsmpu.so) never includes, links or calls
 * anything here, and this file includes nothing from it.
 *
 * Plain, slow, obviously correct: everything the GPU keeps in fp32 is kept
 * here in fp64; everything the GPU keeps in fp16 goes through the hand-written
 * binary16 codec below.  Loops follow the paper's order with no blocking,
 * fusion or reordering.  OpenMP only splits independent elements (results do
 * not depend on the thread count: every stage is elementwise and the overflow
 * test is an OR).
 *
 * Passages (PAPER.md line numbers, "P:n"; SPEC.md "S:n"; readings "Rn" are
 * listed in DESIGN.md):
 *   fp16 fwd/bwd + fp16 all-reduce, fp32 master + optimizer ... P:151-152 (4.1)
 *   loss scaled right after forward ............................ P:153 (4.1)
 *   convert to fp32 and restore the scale after the all-reduce . P:154 (4.1)
 *   dynamic loss scaling: down on overflow, up after 2,000 ..... P:156-158 (4.1)
 *   accumulate gradients over sub-batches (cumul) .............. P:139, P:178 (4.2, Table 1)
 *   Adam beta1=0.9 beta2=0.98 eps=1e-8 ......................... P:104 (3.2)
 *   linear warmup 4,000 steps to 5e-4, then inverse sqrt ....... P:105-106 (3.2)
 *   batch size counted in target tokens excluding padding ..... P:45 (Fig. 1)
 *   buckets change timing, never values ........................ P:209-212 (4.3)
 *
 * Pins (tests/test_oracle.py): exhaustive codec round trip + numpy.float16 on
 * random fp32 + SPEC S:51-64 printed examples; fp16 add worked examples;
 * scaler S:91-94 examples + torch._amp_update_scale_ + closed-form traces;
 * LR S:196-199 + fp32 bit patterns; Adam S:206-208 + constant-gradient closed
 * form + torch.optim.Adam in fp64; reduce S:390-393; large-batch equivalence
 * on a brute-force softmax-regression model; the fp32-accumulator variant
 * (SURVEY Z1 knob) against numpy's binary32 adds + hand-worked special cases.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#if FLT_EVAL_METHOD != 0
#error "orc_accumulate32 needs binary32 evaluation of float expressions (FLT_EVAL_METHOD 0)"
#endif

/* OpenMP thread count of the element loops (results do not depend on it); returns the count now in effect */
int orc_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
    return omp_get_max_threads();
#else
    (void)t;
    return 1;
#endif
}

/* ------------------------------------------------------------------ binary16 codec
 * IEEE 754 binary16: 1 sign bit, 5 exponent bits (bias 15), 10 mantissa bits.
 * (SPEC S:30-36 HalfValue; S:46-64 fp16_round / fp16_to_fp32.)              */

/* exact widening of a binary16 pattern */
double orc_h2d(uint16_t h) {
    int sign = (h >> 15) & 1;
    int expo = (h >> 10) & 0x1F;
    int mant = h & 0x3FF;
    double mag;
    if (expo == 0x1F) {
        mag = mant ? NAN : INFINITY;
    } else if (expo == 0) {
        mag = ldexp((double)mant, -24);                 /* subnormal: mant * 2^-24 */
    } else {
        mag = ldexp((double)(1024 + mant), expo - 25);  /* (1 + mant/1024) * 2^(expo-15) */
    }
    return sign ? -mag : mag;
}

/* round-to-nearest-even from fp64 (one rounding); NaN -> canonical 0x7E00 */
uint16_t orc_d2h(double x) {
    if (isnan(x)) return 0x7E00;
    uint16_t sign = signbit(x) ? 0x8000 : 0;
    double a = fabs(x);
    if (isinf(a)) return sign | 0x7C00;
    if (a < ldexp(1.0, -14)) {
        /* subnormal range: units of 2^-24; nearbyint rounds half to even */
        double q = nearbyint(a / ldexp(1.0, -24));
        return sign | (uint16_t)q;                      /* q == 1024 gives 0x0400, the least normal */
    }
    int E;
    frexp(a, &E);            /* a = f * 2^E, f in [0.5, 1) => a in [2^(E-1), 2^E) */
    E -= 1;                  /* a in [2^E, 2^(E+1)) */
    double q = nearbyint(a / ldexp(1.0, E - 10));       /* significand in units of 2^(E-10): [1024, 2048] */
    if (q == 2048.0) { q = 1024.0; E += 1; }
    if (E > 15) return sign | 0x7C00;                   /* beyond 65504 after rounding -> inf */
    return sign | (uint16_t)((E + 15) << 10) | (uint16_t)(q - 1024.0);
}

int orc_h_nonfinite(uint16_t h) { return (h & 0x7C00) == 0x7C00; }   /* +-inf or NaN */

/* fp16 addition as the accumulation performs it: exact sum (fp64 holds any sum
 * of two binary16 values exactly), one rounding to binary16. */
uint16_t orc_hadd(uint16_t a, uint16_t b) { return orc_d2h(orc_h2d(a) + orc_h2d(b)); }

/* bulk codec helpers (tests) */
void orc_h2d_array(const uint16_t* h, double* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_h2d(h[i]);
}
void orc_d2h_array(const double* x, uint16_t* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_d2h(x[i]);
}

/* ------------------------------------------------------------------ accumulation
 * A = G_1 (copy, reading R2); A = rn16(A + G_k) for k = 2..c (reading R1).  */
void orc_accumulate(uint16_t* A, const uint16_t* G, int64_t n, int first) {
    if (first) { memcpy(A, G, (size_t)n * 2); return; }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) A[i] = orc_hadd(A[i], G[i]);
}

/* ------------------------------------------------------------------ fp32 accumulator variant (SURVEY Z1 knob)
 * P:151 puts fwd/bwd and the all-reduce in FP16 but never names the accumulator (reading Z1 takes fp16, above).
 * Variant: A32 = fp32(G_1); A32 = fl32(A32 + fp32(G_k)) for k = 2..c, binary32 round-to-nearest-even.  This is
 * kept in binary32 (C float arithmetic: FLT_EVAL_METHOD 0, no contraction), not fp64, because the fp16 result
 * depends on every binary32 rounding.  The rank's fp16 gradient is then rn16(A32), which enters the fp16 all-reduce
 * unchanged.  Overflow stays "R holds a non-finite" (R4): a finite sum >= 65520 rounds to inf there. */
void orc_accumulate32(float* A, const uint16_t* G, int64_t n, int first) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        float g = (float)orc_h2d(G[i]);   /* exact: binary16 is a subset of binary32 */
        A[i] = first ? g : A[i] + g;
    }
}

void orc_round16(uint16_t* out, const float* A, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = orc_d2h((double)A[i]);   /* one rounding: binary32 is exact in fp64 */
}

/* ------------------------------------------------------------------ all-reduce
 * R = A_0; R = rn16(R + A_r) for r = 1..W-1: fixed ascending-rank order (reading R3). */
void orc_reduce(uint16_t* R, const uint16_t* const* A, int W, int64_t n) {
    memcpy(R, A[0], (size_t)n * 2);
    for (int r = 1; r < W; ++r) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) R[i] = orc_hadd(R[i], A[r][i]);
    }
}

/* overflow <=> some element of the reduced gradient is non-finite (reading R4/R5) */
int64_t orc_count_nonfinite(const uint16_t* R, int64_t n) {
    int64_t cnt = 0;
#pragma omp parallel for schedule(static) reduction(+ : cnt)
    for (int64_t i = 0; i < n; ++i) cnt += orc_h_nonfinite(R[i]);
    return cnt;
}

/* ------------------------------------------------------------------ LR schedule
 * lr(t) = peak * min(t / warmup, sqrt(warmup / t)) in fp64, one rounding to fp32 (reading R14). */
float orc_lr(int64_t t, double peak, int64_t warmup) {
    double tt = (double)t, w = (double)warmup;
    double lin = tt / w;
    double isq = sqrt(w / tt);
    double f = lin < isq ? lin : isq;
    return (float)(peak * f);
}

/* ------------------------------------------------------------------ dynamic loss scaler
 * scale = 2^e.  overflow: skip, e = max(e-1, emin), clean = 0.
 * clean:   t += 1, clean += 1; clean == growth -> e = min(e+1, emax), clean = 0.
 * (readings R6-R10.)                                                 */
typedef struct {
    int32_t e;          /* current scale exponent */
    int64_t clean;      /* consecutive overflow-free updates since last change */
    int64_t t;          /* applied updates */
} orc_scaler;

typedef struct {
    int32_t overflow, applied, e_used, e_next;
    float lr;
    int64_t t, N, clean;
} orc_result;

typedef struct {
    double peak_lr;
    int64_t warmup;
    double beta1, beta2, eps;
    int32_t emin, emax;
    int64_t growth;
} orc_cfg;

/* decision half of the step (no data): returns 1 if the update is applied */
int orc_scaler_step(orc_scaler* s, const orc_cfg* cfg, int overflow, orc_result* res) {
    res->e_used = s->e;
    if (overflow) {
        s->e = s->e - 1 < cfg->emin ? cfg->emin : s->e - 1;
        s->clean = 0;
        res->overflow = 1;
        res->applied = 0;
        res->lr = orc_lr(s->t + 1, cfg->peak_lr, cfg->warmup);   /* reading R15 */
    } else {
        s->t += 1;
        s->clean += 1;
        res->overflow = 0;
        res->applied = 1;
        res->lr = orc_lr(s->t, cfg->peak_lr, cfg->warmup);
        if (s->clean >= cfg->growth) {
            s->e = s->e + 1 > cfg->emax ? cfg->emax : s->e + 1;
            s->clean = 0;
        }
    }
    res->e_next = s->e;
    res->t = s->t;
    res->clean = s->clean;
    return res->applied;
}

/* ------------------------------------------------------------------ Adam (Kingma & Ba Alg. 1, reading R13)
 * g = R / (2^e * N)                 (P:154 unscale; P:45 normalise by target tokens, reading R11)
 * m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2
 * theta = theta - lr * (m / bc1) / (sqrt(v / bc2) + eps),  bc_j = 1 - b_j^t
 * w16 = rn16(theta)                 (P:152 fp16 copy of the fp32 master, reading R16)     */
void orc_adam(double* theta, double* m, double* v, uint16_t* w16, const uint16_t* R, int64_t n,
              int32_t e, int64_t N, float lr, int64_t t, const orc_cfg* cfg) {
    double sN = ldexp((double)N, e);
    double b1 = cfg->beta1, b2 = cfg->beta2, eps = cfg->eps;
    double bc1 = 1.0 - pow(b1, (double)t);
    double bc2 = 1.0 - pow(b2, (double)t);
    double lrd = (double)lr;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double g = orc_h2d(R[i]) / sN;
        m[i] = b1 * m[i] + (1.0 - b1) * g;
        v[i] = b2 * v[i] + (1.0 - b2) * g * g;
        theta[i] = theta[i] - lrd * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
        w16[i] = orc_d2h(theta[i]);
    }
}

/* ------------------------------------------------------------------ one whole update
 * G[r*c + k] (k = 0..c-1) are the micro-gradients of rank r; A is W*n scratch, R n scratch.
 * N = sum of the W*c token counts.  On overflow theta/m/v/w16/t are untouched (reading R6). */
int orc_update(double* theta, double* m, double* v, uint16_t* w16, int64_t n,
               const uint16_t* const* G, int W, int c, int64_t N,
               uint16_t* A, uint16_t* R, orc_scaler* s, const orc_cfg* cfg, orc_result* res) {
    const uint16_t* Ar[256];
    if (W > 256) return -1;
    for (int r = 0; r < W; ++r) {
        uint16_t* a = A + (int64_t)r * n;
        for (int k = 0; k < c; ++k) orc_accumulate(a, G[r * c + k], n, k == 0);
        Ar[r] = a;
    }
    orc_reduce(R, Ar, W, n);
    int overflow = orc_count_nonfinite(R, n) > 0;
    int32_t e_used = s->e;
    res->N = N;
    if (orc_scaler_step(s, cfg, overflow, res))
        orc_adam(theta, m, v, w16, R, n, e_used, N, res->lr, s->t, cfg);
    return 0;
}
