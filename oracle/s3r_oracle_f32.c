/*
 * s3r_oracle_f32.c — fp32 CONTRACT instance of the CPU oracle, plus the
 * precision-independent pieces (time normalisation, instance-camera
 * composition, the LOD random generator, point-life update, commit, reset).
 * TEST INFRASTRUCTURE ONLY (see s3r_oracle.h).  Build: gcc -O2
 * -ffp-contract=off (no fast-math): every line is one IEEE-754 operation.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "s3r_oracle.h"

/* ------------------------------------------------------------------------
 * s3r_exp2 (DESIGN.md R-ARITH, exp2 form of Eq.2's exponential): 2^x for
 * x <= 0, written so that any IEEE-754 machine evaluates it bit-identically.
 *   x < -24             -> 0        (flush: a contribution alpha T < 2^-24,
 *                                    below fp32 resolution of the pixel, is
 *                                    dropped; reading R14)
 *   t = x + 1.5*2^23;  n = t - 1.5*2^23   (exact rint, ties to even)
 *   r = x - n           (exact, |r| <= 1/2)
 *   y = 1 + r P(r)      P: degree-4 relative-minimax fit of (2^r - 1)/r on
 *                       [-1/2, 1/2] (Lawson iteration, fp32 coefficients
 *                       tuned by +-2 ulp), Horner with fma: <= 2.02 ulp
 *   return y * 2^n      (exact: 2^-24 is normal)
 * ---------------------------------------------------------------------- */
float so_exp2_f32(float x)
{
    if (!(x >= -24.0f)) return 0.0f;
    float t = x + 12582912.0f;
    float n = t - 12582912.0f;
    float r = x - n;
    float p = 1.3264695880934596e-3f;
    p = fmaf(p, r, 9.671507403254509e-3f);
    p = fmaf(p, r, 5.550733208656311e-2f);
    p = fmaf(p, r, 2.4022243916988373e-1f);
    p = fmaf(p, r, 6.931470036506653e-1f);
    float y = fmaf(p, r, 1.0f);
    return ldexpf(y, (int)n);
}

/* SplitMix64 (reading R9): the counter-based generator behind the Bernoulli
 * draw of Eq.7 row 2.  Keyed by (per-view seed, global Gaussian
 * index) so the draw is independent of compaction, batching and GPU count. */
uint64_t so_splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* u = top 24 bits of splitmix64(seed ^ splitmix64(g)) times 2^-24: exact in
 * fp32, uniform on {0, 2^-24, ..., 1 - 2^-24}. */
float so_lod_uniform(uint64_t seed, int64_t g)
{
    uint64_t h = so_splitmix64(seed ^ so_splitmix64((uint64_t)g));
    return (float)(uint32_t)(h >> 40) * 5.9604644775390625e-8f;
}

/* ------------------------------------------------------------------------
 * NEXT-3 noise for the LOD noisy offset (Eq.7 row 4, "N(0,1)"): three
 * standard normals per (view seed, Gaussian), by Box-Muller on counter-based
 * uniforms, every step an R-ARITH fp32 operation so that any IEEE-754 machine
 * draws the same numbers.
 *   u_k = top 24 bits of splitmix64((seed ^ splitmix64(g)) + (k+1) C) * 2^-24,
 *         C = 0xD1B54A32D192ED03, k = 0..3 (streams distinct from the
 *         Bernoulli draw of so_lod_uniform)
 *   (n0, n1) = sqrt(-2 ln(1 - u_0)) (cos, sin)(2 pi u_1),
 *   (n2, -)  = sqrt(-2 ln(1 - u_2)) (cos, sin)(2 pi u_3).
 * ---------------------------------------------------------------------- */
float so_lod_uniform_k(uint64_t seed, int64_t g, int k)
{
    uint64_t base = seed ^ so_splitmix64((uint64_t)g);
    uint64_t h = so_splitmix64(base + (uint64_t)(k + 1) * 0xD1B54A32D192ED03ull);
    return (float)(uint32_t)(h >> 40) * 5.9604644775390625e-8f;
}

/* log2(x), x > 0 normal: x = m 2^e with m in [sqrt(2)/2, sqrt(2)) (exact bit
 * split), s = (m - 1) / (m + 1), log2(m) = s (c1 + s^2 (c3 + s^2 (c5 + s^2 (c7
 * + s^2 c9)))), c_k = 2 / (k ln 2) (the atanh series; |s| <= 0.1716, so the
 * first omitted term is < 1e-9). */
float so_log2_f32(float x)
{
    union { float f; uint32_t u; } b = {x};
    int e = (int)((b.u >> 23) & 0xffu) - 127;
    b.u = (b.u & 0x007fffffu) | 0x3f800000u;          /* m in [1, 2) */
    float m = b.f;
    if (m > 1.41421356f) {
        m = m * 0.5f;
        e = e + 1;
    }
    float s = (m - 1.0f) / (m + 1.0f);
    float s2 = s * s;
    float p = 0.320598898f;                        /* 2 / (9 ln 2) */
    p = fmaf(p, s2, 0.412198583f);                 /* 2 / (7 ln 2) */
    p = fmaf(p, s2, 0.577078016f);                 /* 2 / (5 ln 2) */
    p = fmaf(p, s2, 0.961796694f);                 /* 2 / (3 ln 2) */
    p = fmaf(p, s2, 2.885390082f);                 /* 2 / ln 2     */
    return fmaf(s, p, (float)e);
}

/* (sin, cos)(2 pi u) for u in [0, 1) a multiple of 2^-24: quadrant q =
 * floor(4u), f = 4u - q (both exact), phi = f pi/2, Taylor polynomials of sin
 * (to phi^11) and cos (to phi^12) on [0, pi/2) in Horner form in phi^2, then
 * the quadrant rotation. */
void so_sincos_turn_f32(float u, float* sn, float* cs)
{
    float x4 = u * 4.0f;
    float q = floorf(x4);
    float f = x4 - q;
    float ph = f * 1.57079637f;
    float p2 = ph * ph;
    float sp = -2.50521084e-8f;                    /* -1/11! */
    sp = fmaf(sp, p2, 2.75573192e-6f);             /*  1/9!  */
    sp = fmaf(sp, p2, -1.98412698e-4f);            /* -1/7!  */
    sp = fmaf(sp, p2, 8.33333333e-3f);             /*  1/5!  */
    sp = fmaf(sp, p2, -1.66666667e-1f);            /* -1/3!  */
    sp = fmaf(sp, p2, 1.0f);
    float s = ph * sp;
    float cp = 2.08767570e-9f;                     /*  1/12! */
    cp = fmaf(cp, p2, -2.75573192e-7f);            /* -1/10! */
    cp = fmaf(cp, p2, 2.48015873e-5f);             /*  1/8!  */
    cp = fmaf(cp, p2, -1.38888889e-3f);            /* -1/6!  */
    cp = fmaf(cp, p2, 4.16666667e-2f);             /*  1/4!  */
    cp = fmaf(cp, p2, -0.5f);                      /* -1/2!  */
    float c = fmaf(cp, p2, 1.0f);
    int qi = (int)q;
    if (qi == 0) { *sn = s; *cs = c; }
    else if (qi == 1) { *sn = c; *cs = -s; }
    else if (qi == 2) { *sn = -s; *cs = -c; }
    else { *sn = -c; *cs = s; }
}

void so_lod_normal3(uint64_t seed, int64_t g, float out[3])
{
    float sn, cs;
    float r0 = sqrtf(so_log2_f32(1.0f - so_lod_uniform_k(seed, g, 0)) * -1.38629436f);
    so_sincos_turn_f32(so_lod_uniform_k(seed, g, 1), &sn, &cs);
    out[0] = r0 * cs;
    out[1] = r0 * sn;
    float r1 = sqrtf(so_log2_f32(1.0f - so_lod_uniform_k(seed, g, 2)) * -1.38629436f);
    so_sincos_turn_f32(so_lod_uniform_k(seed, g, 3), &sn, &cs);
    out[2] = r1 * cs;
}

/* Time normalisation ("we first normalize the rendering time of the
 * whole scene to [-1,1]"): frame i of F -> -1 + 2 i / (F - 1); F = 1 -> 0. */
double so_normalize_time(int64_t frame, int64_t frame_count)
{
    if (frame_count <= 1) return 0.0;
    return -1.0 + (2.0 * (double)frame) / (double)(frame_count - 1);
}

/* Instance cameras: W_{t,i} = W_t W_{t,i2g}; slot 0 = W_t
 * (reading R17).  3x4 row-major [R|t] operands; computed in fp64 with the
 * dot3 order of R-ARITH, then rounded once to fp32.
 *   w2c: [12], i2g: [K][12], out: [(K+1)][12]. */
void so_compose_instance_cameras(const float* w2c, const float* i2g, int32_t K, float* out)
{
    for (int k = 0; k < 12; ++k) out[k] = w2c[k];
    for (int32_t i = 0; i < K; ++i) {
        const float* B = i2g + 12 * (int64_t)i;
        float* O = out + 12 * (int64_t)(i + 1);
        for (int r = 0; r < 3; ++r) {
            double a0 = w2c[4 * r + 0], a1 = w2c[4 * r + 1], a2 = w2c[4 * r + 2], a3 = w2c[4 * r + 3];
            for (int c = 0; c < 3; ++c) {
                double acc = a0 * (double)B[0 * 4 + c];
                acc = fma(a1, (double)B[1 * 4 + c], acc);
                acc = fma(a2, (double)B[2 * 4 + c], acc);
                O[4 * r + c] = (float)acc;
            }
            double acc = fma(a0, (double)B[0 * 4 + 3], a3);
            acc = fma(a1, (double)B[1 * 4 + 3], acc);
            acc = fma(a2, (double)B[2 * 4 + 3], acc);
            O[4 * r + 3] = (float)acc;
        }
    }
}

/* O7 point-life update (Eq.5): for M_t[i]: l_s = min(l_s, t),
 * l_e = max(l_e, t).  t is canonicalised (-0 -> +0). */
void so_update_life_f32(so_scene* s, const uint8_t* visible, float t)
{
    t = t + 0.0f;
    for (int64_t g = 0; g < s->n; ++g) {
        if (!visible[g]) continue;
        if (t < s->life[2 * g + 0]) s->life[2 * g + 0] = t;
        if (t > s->life[2 * g + 1]) s->life[2 * g + 1] = t;
    }
}

/* O8 commit (Eq.6): t_s = l_s - 0.1, t_e = l_e + 0.1, clamped to
 * [-1,1]; a never-observed Gaussian (l_s > l_e, the initial (1,-1)) becomes
 * visible at all times (reading R18); life is reset to (1,-1). */
void so_commit_visibility(so_scene* s, float margin)
{
    for (int64_t g = 0; g < s->n; ++g) {
        float ls = s->life[2 * g + 0], le = s->life[2 * g + 1];
        if (ls > le) {
            s->visibility[2 * g + 0] = -1.0f;
            s->visibility[2 * g + 1] = 1.0f;
        } else {
            s->visibility[2 * g + 0] = fmaxf(-1.0f, ls - margin);
            s->visibility[2 * g + 1] = fminf(1.0f, le + margin);
        }
        s->life[2 * g + 0] = 1.0f;
        s->life[2 * g + 1] = -1.0f;
    }
}

/* P:183 "we periodically reset the temporal visibility ... to be visible". */
void so_reset_visibility(so_scene* s)
{
    for (int64_t g = 0; g < s->n; ++g) {
        s->visibility[2 * g + 0] = -1.0f;
        s->visibility[2 * g + 1] = 1.0f;
    }
}

#define REAL float
#define SO(x) x##_f32
#define R(x) x##f
#define FMA fmaf
#define SQRT sqrtf
#define CEIL ceilf
#define FLOOR floorf
#define FMIN fminf
#define FMAX fmaxf
#define ISFIN isfinite
#define EXPF so_exp2_f32   /* unused: SO_CONTRACT_EXP2 selects the exp2 form */
#define SO_CONTRACT_EXP2 1
#include "s3r_oracle_impl.inc"
