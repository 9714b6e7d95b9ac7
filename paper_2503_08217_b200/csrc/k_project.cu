// k_project.cu — K2: instance-specific projection + EWA covariance + frustum
// mask M_t + Adaptive-LOD cull + point-life update, with compaction of the
// rendered splats of every view; plus the instance-camera composition and the
// K9 commit / reset / life-flip kernels.
//
// PAPER.md P:158-159 (instance-specific projection: W_{t,i} = W_t W_{t,i2g},
// "we simply select the corresponding cameras based on the Gaussian's instance
// ID"), Eq.1 P:107-112 (mu' = K W mu, Sigma' = J W Sigma W^T J^T)
// (frustum mask M_t), Eq.7 rows 1-3 P:189-193 (LOD: p = p_max + (p_max - 1e-2)
// min(0,(d-D)/D), M_LOD = Bernoulli(p) <= 0), Eq.5 P:173-178 (l_s = min(l_s,t),
// l_e = max(l_e,t) where M_t).  Readings R2-R9 of DESIGN.md.
//
// Arithmetic: the fp32 R-ARITH contract of DESIGN.md, op for op (this file is
// compiled with -fmad=false; FMAs are the explicit __fmaf_rn below).
//
// Layout: grid (CTA, view); one CTA walks 4 x 256 consecutive entries of its
// view's temporal index list (coalesced 4-byte index loads, then 16-byte
// gathers of the SoA float4 streams).  The view's (K+1) x 3x4 camera table is
// staged in shared memory once per CTA.  A conservative frustum pre-test
// queues the entries it cannot reject, and the exact path runs on those in
// dense warps.  Rendered splats are compacted with ballot/popc and ONE atomic
// per warp-round on the view's counter, into 48-byte records
// {mx,my,z,o}{qa,qb,qc,rect.x}{r,g,b,rect.y} and a 64-bit depth key (depth
// bits << gbits | Gaussian index).  The record order is therefore not
// deterministic; the depth sort (K5a) on those keys restores the unique
// (depth, index) order, so everything downstream is deterministic.  (Equal
// depths are common: a car face seen along a camera axis has thousands of
// Gaussians at one fp32 depth, so the index bits cannot be left to a fix-up.)
#include <algorithm>

#include "s3r_internal.cuh"

namespace s3r {

namespace {
#ifndef S3R_K2_WARP_COMPACT
#define S3R_K2_WARP_COMPACT 1
#endif
constexpr int PT = 256;
#ifndef S3R_K2_PR
#define S3R_K2_PR 4
#endif
constexpr int PR_BIG = S3R_K2_PR;     // rounds of PT entries per CTA
constexpr int PTILE = PT * PR_BIG;
// batches whose K2 grid would not fill the GPU (small scenes: C1) take chunks of
// one round, 4x more CTAs on the same entries (shorter serial chains)

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Exact float min / max through integer atomics (valid for non-NaN values;
// times are canonicalised so -0 never occurs).
__device__ __forceinline__ void atomic_min_f(float* addr, float v)
{
    if (v >= 0.f) atomicMin(reinterpret_cast<int*>(addr), __float_as_int(v));
    else atomicMax(reinterpret_cast<unsigned*>(addr), __float_as_uint(v));
}
__device__ __forceinline__ void atomic_max_f(float* addr, float v)
{
    if (v >= 0.f) atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
    else atomicMin(reinterpret_cast<unsigned*>(addr), __float_as_uint(v));
}

struct Splat {
    float k[6];          // mx, my, z, a, b, c of the projection (dump keys)
    float rm[3];         // mx, my, z of the splat (the jittered mean's, if moved)
    float mu[3];         // own-frame mean of the splat (moved by the noisy offset)
    float A, B, C;
    int tx0, tx1, ty0, ty1;
    uint8_t flags;
};

// O2: keys of a Gaussian with mean (x, y, z) in the frame of camera M (the 12
// floats of its instance camera).  Returns false behind the near plane.
__device__ __forceinline__ bool project_keys(const float* __restrict__ M, float x, float y,
                                             float z, float4 sc, float4 q, const DevView& V,
                                             float lox, float hix, float loy, float hiy,
                                             float* k)
{
    float p[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        float acc = __fmaf_rn(M[4 * r + 0], x, M[4 * r + 3]);
        acc = __fmaf_rn(M[4 * r + 1], y, acc);
        acc = __fmaf_rn(M[4 * r + 2], z, acc);
        p[r] = acc;
    }
    const float pz = p[2];
    if (!(pz > V.near_plane)) return false;
    float n2 = q.x * q.x;
    n2 = __fmaf_rn(q.y, q.y, n2);
    n2 = __fmaf_rn(q.z, q.z, n2);
    n2 = __fmaf_rn(q.w, q.w, n2);
    const float nrm = sqrtf(n2);
    const float w = q.x / nrm, a1 = q.y / nrm, a2 = q.z / nrm, a3 = q.w / nrm;
    const float xx = a1 * a1, yy = a2 * a2, zz = a3 * a3;
    const float xy = a1 * a2, xz = a1 * a3, yz = a2 * a3;
    const float wx = w * a1, wy = w * a2, wz = w * a3;
    float Rq[9];
    Rq[0] = 1.0f - 2.0f * (yy + zz);
    Rq[1] = 2.0f * (xy - wz);
    Rq[2] = 2.0f * (xz + wy);
    Rq[3] = 2.0f * (xy + wz);
    Rq[4] = 1.0f - 2.0f * (xx + zz);
    Rq[5] = 2.0f * (yz - wx);
    Rq[6] = 2.0f * (xz - wy);
    Rq[7] = 2.0f * (yz + wx);
    Rq[8] = 1.0f - 2.0f * (xx + yy);
    const float sg[3] = {sc.x, sc.y, sc.z};
    float T[9];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float acc = M[4 * r + 0] * Rq[c];
            acc = __fmaf_rn(M[4 * r + 1], Rq[3 + c], acc);
            acc = __fmaf_rn(M[4 * r + 2], Rq[6 + c], acc);
            T[3 * r + c] = acc * sg[c];
        }
    }
    const float u = p[0] / pz;
    const float vv = p[1] / pz;
    const float uc = fminf(fmaxf(u, lox), hix);
    const float vc = fminf(fmaxf(vv, loy), hiy);
    const float j00 = V.fx / pz;
    const float j02 = -((V.fx * uc) / pz);
    const float j11 = V.fy / pz;
    const float j12 = -((V.fy * vc) / pz);
    float U0[3], U1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        U0[c] = __fmaf_rn(j02, T[6 + c], j00 * T[c]);
        U1[c] = __fmaf_rn(j12, T[6 + c], j11 * T[3 + c]);
    }
    float ka = U0[0] * U0[0];
    ka = __fmaf_rn(U0[1], U0[1], ka);
    ka = __fmaf_rn(U0[2], U0[2], ka);
    float kb = U0[0] * U1[0];
    kb = __fmaf_rn(U0[1], U1[1], kb);
    kb = __fmaf_rn(U0[2], U1[2], kb);
    float kc = U1[0] * U1[0];
    kc = __fmaf_rn(U1[1], U1[1], kc);
    kc = __fmaf_rn(U1[2], U1[2], kc);
    k[0] = __fmaf_rn(V.fx, u, V.cx);
    k[1] = __fmaf_rn(V.fy, vv, V.cy);
    k[2] = pz;
    k[3] = ka;
    k[4] = kb;
    k[5] = kc;
    return true;
}

struct Dec {
    float A, B, C, disc;
    int tx0, tx1, ty0, ty1;
};

// O3: dilation, conic, radius, pixel box, frustum membership, tile rectangle.
__device__ __forceinline__ bool decide(const float* k, const DevView& V, Dec& d)
{
    const float mx = k[0], my = k[1], pz = k[2], ka = k[3], kb = k[4], kc = k[5];
    if (!(isfinite(mx) && isfinite(my) && isfinite(pz) && isfinite(ka) && isfinite(kb) &&
          isfinite(kc)))
        return false;
    const float ad = ka + 0.3f;
    const float cd = kc + 0.3f;
    const float d1 = ad * cd;
    const float d2 = kb * kb;
    const float det = d1 - d2;
    if (!(det > 0.0f)) return false;
    d.A = cd / det;
    d.B = (-kb) / det;
    d.C = ad / det;
    const float h = 0.5f * (ka - kc);
    const float e1 = h * h;
    const float e2 = kb * kb;
    d.disc = sqrtf(e1 + e2);
    const float lamd = (0.5f * (ad + cd)) + d.disc;
    const float rf = ceilf(3.0f * sqrtf(lamd));
    if (!isfinite(rf)) return false;
    const float xlo = ceilf(mx - rf), xhi = floorf(mx + rf);
    const float ylo = ceilf(my - rf), yhi = floorf(my + rf);
    const float Wm1 = (float)(V.W - 1), Hm1 = (float)(V.H - 1);
    if (!(xlo <= Wm1 && xhi >= 0.0f && ylo <= Hm1 && yhi >= 0.0f)) return false;
    const int x0 = (int)fmaxf(xlo, 0.0f), x1 = (int)fminf(xhi, Wm1);
    const int y0 = (int)fmaxf(ylo, 0.0f), y1 = (int)fminf(yhi, Hm1);
    d.tx0 = x0 >> 4; d.tx1 = x1 >> 4; d.ty0 = y0 >> 4; d.ty1 = y1 >> 4;
    return true;
}

// ---- NEXT-3 noise (Eq.7 row 4, "N(0,1)"; reading R10): three standard
// normals per (view seed, Gaussian) by Box-Muller on counter-based uniforms,
// each step an R-ARITH fp32 operation (DESIGN.md §4 "LOD noisy offset").
__device__ __forceinline__ float lod_uniform_k(unsigned long long base, int k)
{
    const unsigned long long h = splitmix64(base + (unsigned long long)(k + 1) * 0xD1B54A32D192ED03ull);
    return (float)(uint32_t)(h >> 40) * 5.9604644775390625e-8f;
}

__device__ __forceinline__ float log2_rarith(float x)
{
    uint32_t u = __float_as_uint(x);
    int e = (int)((u >> 23) & 0xffu) - 127;
    float m = __uint_as_float((u & 0x007fffffu) | 0x3f800000u);
    if (m > 1.41421356f) {
        m = m * 0.5f;
        e = e + 1;
    }
    const float s = (m - 1.0f) / (m + 1.0f);
    const float s2 = s * s;
    float p = 0.320598898f;
    p = __fmaf_rn(p, s2, 0.412198583f);
    p = __fmaf_rn(p, s2, 0.577078016f);
    p = __fmaf_rn(p, s2, 0.961796694f);
    p = __fmaf_rn(p, s2, 2.885390082f);
    return __fmaf_rn(s, p, (float)e);
}

__device__ __forceinline__ void sincos_turn(float u, float& sn, float& cs)
{
    const float x4 = u * 4.0f;
    const float q = floorf(x4);
    const float f = x4 - q;
    const float ph = f * 1.57079637f;
    const float p2 = ph * ph;
    float sp = -2.50521084e-8f;
    sp = __fmaf_rn(sp, p2, 2.75573192e-6f);
    sp = __fmaf_rn(sp, p2, -1.98412698e-4f);
    sp = __fmaf_rn(sp, p2, 8.33333333e-3f);
    sp = __fmaf_rn(sp, p2, -1.66666667e-1f);
    sp = __fmaf_rn(sp, p2, 1.0f);
    const float s = ph * sp;
    float cp = 2.08767570e-9f;
    cp = __fmaf_rn(cp, p2, -2.75573192e-7f);
    cp = __fmaf_rn(cp, p2, 2.48015873e-5f);
    cp = __fmaf_rn(cp, p2, -1.38888889e-3f);
    cp = __fmaf_rn(cp, p2, 4.16666667e-2f);
    cp = __fmaf_rn(cp, p2, -0.5f);
    const float c = __fmaf_rn(cp, p2, 1.0f);
    const int qi = (int)q;
    if (qi == 0) { sn = s; cs = c; }
    else if (qi == 1) { sn = c; cs = -s; }
    else if (qi == 2) { sn = -s; cs = -c; }
    else { sn = -c; cs = s; }
}

__device__ __noinline__ void lod_normal3(unsigned long long seed, long long g, float* out)
{
    const unsigned long long base = seed ^ splitmix64((unsigned long long)g);
    float sn, cs;
    const float r0 = sqrtf(log2_rarith(1.0f - lod_uniform_k(base, 0)) * -1.38629436f);
    sincos_turn(lod_uniform_k(base, 1), sn, cs);
    out[0] = r0 * cs;
    out[1] = r0 * sn;
    const float r1 = sqrtf(log2_rarith(1.0f - lod_uniform_k(base, 2)) * -1.38629436f);
    sincos_turn(lod_uniform_k(base, 3), sn, cs);
    out[2] = r1 * cs;
}

// NEXT-3 (rare path, kept out of line): move the mean of a kept small Gaussian
// by the noisy offset, project it again, and take the splat, depth and tile
// rectangle from the moved mean.  False if the moved mean is not visible.
__device__ __noinline__ bool jitter_reproject(const float* __restrict__ M, float4 mo, float4 sc,
                                              float4 q, const DevView& V, float lox, float hix,
                                              float loy, float hiy, long long g, float pz,
                                              Splat& s)
{
    float nz[3];
    lod_normal3(V.seed, g, nz);
    const float nd = fminf(1.0f, pz / V.lod_D);
    const float mu[3] = {mo.x, mo.y, mo.z};
    float mj[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) mj[ax] = __fmaf_rn(V.jit[ax] * nd, nz[ax], mu[ax]);
    float kj[6];
    if (!project_keys(M, mj[0], mj[1], mj[2], sc, q, V, lox, hix, loy, hiy, kj)) return false;
    Dec dj;
    if (!decide(kj, V, dj)) return false;
    s.A = dj.A; s.B = dj.B; s.C = dj.C;
    s.tx0 = dj.tx0; s.tx1 = dj.tx1; s.ty0 = dj.ty0; s.ty1 = dj.ty1;
    s.rm[0] = kj[0]; s.rm[1] = kj[1]; s.rm[2] = kj[2];
    s.mu[0] = mj[0]; s.mu[1] = mj[1]; s.mu[2] = mj[2];
    return true;
}

// O2 + O3 + O4 (+ the NEXT-3 noisy offset) of DESIGN.md for Gaussian g in
// view V; M = the 12 floats of its instance camera.  Sets s.flags.
template <bool JIT>
__device__ __forceinline__ void project_one(const float* __restrict__ M, float4 mo, float4 sc,
                                            float4 q, const DevView& V, float lox, float hix,
                                            float loy, float hiy, long long g, Splat& s)
{
    s.flags = F_TEMPORAL;
    if (!project_keys(M, mo.x, mo.y, mo.z, sc, q, V, lox, hix, loy, hiy, s.k)) {
#pragma unroll
        for (int j = 0; j < 6; ++j) s.k[j] = __int_as_float(0x7fc00000);
        return;
    }
    Dec d;
    if (!decide(s.k, V, d)) return;
    s.A = d.A; s.B = d.B; s.C = d.C;
    s.tx0 = d.tx0; s.tx1 = d.tx1; s.ty0 = d.ty0; s.ty1 = d.ty1;
    s.rm[0] = s.k[0]; s.rm[1] = s.k[1]; s.rm[2] = s.k[2];
    s.mu[0] = mo.x; s.mu[1] = mo.y; s.mu[2] = mo.z;
    s.flags |= F_VISIBLE;

    // ---- O4 adaptive LOD ----
    const float ka = s.k[3], kc = s.k[5], pz = s.k[2];
    const float lam = (0.5f * (ka + kc)) + d.disc;
    const float sc2 = 3.0f * sqrtf(fmaxf(lam, 0.0f));
    if (V.lod_r > 0.0f && sc2 <= V.lod_r) {
        s.flags |= F_SMALL;
        const float m = fminf(0.0f, (pz - V.lod_D) / V.lod_D);
        float pd = __fmaf_rn(V.lod_pmax - 0.01f, m, V.lod_pmax);
        pd = fminf(fmaxf(pd, 0.0f), 1.0f);
        const unsigned long long hsh = splitmix64(V.seed ^ splitmix64((unsigned long long)g));
        const float uu = (float)(uint32_t)(hsh >> 40) * 5.9604644775390625e-8f;
        if (uu < pd) {
            s.flags |= F_DROPPED;
            return;
        }
        // ---- NEXT-3 noisy offset (Eq.7 row 4): mu += jit normalize(d) N(0,1),
        // normalize(d) = min(1, d / D) (reading R10), then project again
        if constexpr (JIT) {
            if (V.jit[0] != 0.0f || V.jit[1] != 0.0f || V.jit[2] != 0.0f) {
                s.flags |= F_JITTERED;
                if (!jitter_reproject(M, mo, sc, q, V, lox, hix, loy, hiy, g, pz, s)) return;
            }
        }
    }
    s.flags |= F_RENDERED;
}

// Conservative frustum pre-test (changes no result): true only when the
// Gaussian is certainly invisible, so the exact path (quaternion
// normalisation, ~10 IEEE divisions, 3 square roots) is skipped for the
// in-front Gaussians outside the view.  Bound (exact arithmetic):
//   lambda'_max <= a + c + 0.3,  a + c = |J T|_F^2 <= |J|_F^2 |M3|_F^2 (sx^2+sy^2+sz^2)
// (R_q orthonormal; Cauchy-Schwarz per entry also bounds the fp32-computed a, c
// to within a few ulps), |J|_F^2 = (fx/z)^2 (1 + uc^2) + (fy/z)^2 (1 + vc^2), so
// r_f = ceil(3 sqrt(lambda')) <= 3 sqrt(bound) + 1.  Approximate reciprocal /
// sqrt are used here; the 1 % + 2 px + 1e-4 |m| slack covers their error and
// the rounding of mx = fx u + cx.  Non-finite values never cull (every compare
// is false), so such Gaussians take the exact path.  With debug dumps on, the
// exact path still runs and a visible Gaussian the pre-test had culled sets
// ERR_PRECULL (a self-check the parity tests read through s3r_check).
__device__ __forceinline__ float rcp_apx(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt_apx(float x)
{
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ bool surely_outside(const float* __restrict__ M, float4 mo, float4 sc,
                                               const DevView& V, float lox, float hix,
                                               float loy, float hiy)
{
    float p[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        float acc = __fmaf_rn(M[4 * r + 0], mo.x, M[4 * r + 3]);
        acc = __fmaf_rn(M[4 * r + 1], mo.y, acc);
        acc = __fmaf_rn(M[4 * r + 2], mo.z, acc);
        p[r] = acc;
    }
    const float z = p[2];
    if (!(z > V.near_plane)) return false;       // the exact path rejects it cheaply
    const float iz = rcp_apx(z);
    const float u = p[0] * iz, v = p[1] * iz;
    const float uc = fminf(fmaxf(u, lox), hix), vc = fminf(fmaxf(v, loy), hiy);
    const float fz = V.fx * iz, gz = V.fy * iz;
    const float j2 = __fmaf_rn(fz * fz, __fmaf_rn(uc, uc, 1.0f), (gz * gz) * __fmaf_rn(vc, vc, 1.0f));
    float m2 = 0.0f;
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) m2 = __fmaf_rn(M[4 * r + c], M[4 * r + c], m2);
    const float s2 = __fmaf_rn(sc.x, sc.x, __fmaf_rn(sc.y, sc.y, sc.z * sc.z));
    const float lam = __fmaf_rn((j2 * m2) * s2, 1.01f, 0.31f);
    const float mx = __fmaf_rn(V.fx, u, V.cx), my = __fmaf_rn(V.fy, v, V.cy);
    const float rb = __fmaf_rn(3.03f, sqrt_apx(lam), 3.0f) +
                     1e-4f * (fabsf(mx) + fabsf(my));
    return mx - rb > (float)(V.W - 1) || mx + rb < 0.0f || my - rb > (float)(V.H - 1) ||
           my + rb < 0.0f;
}

// Pass A of K2 over one CTA chunk of (PT * PR) temporal-list entries: all PR
// rounds' loads are issued before any test (two dependent load latencies per
// chunk instead of two per round); the conservative pre-test (surely_outside)
// runs on each valid entry, and the entries it cannot reject (and, with debug
// dumps, all valid ones; tag bit 15 = "the pre-test would have culled it") are
// appended to the shared-memory queue (qt, qg) through the counter *qn.  Bad
// instance ids are counted into c_bad (and dumped) here.
template <int PR, bool LEAN>
__device__ __forceinline__ void precull_chunk(const ProjectArgs& a, const DevView& V, int vi,
                                              long long i0, long long n_t,
                                              const int32_t* __restrict__ tl,
                                              const float* __restrict__ s_tab, float lox,
                                              float hix, float loy, float hiy, uint16_t* qt,
                                              uint32_t* qg, int* qn, unsigned long long& c_bad)
{
    const int tid = threadIdx.x, lane = tid & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int K1 = a.num_instances;
    long long gA[PR];
    int idA[PR];
    float4 scA[PR], moA[PR];
#pragma unroll
    for (int rd = 0; rd < PR; ++rd) {
        const long long i = i0 + rd * PT + tid;
        gA[rd] = i < n_t ? (long long)tl[i] : -1ll;
    }
#pragma unroll
    for (int rd = 0; rd < PR; ++rd) idA[rd] = gA[rd] >= 0 ? __ldg(a.ids + gA[rd]) : 0;
#pragma unroll
    for (int rd = 0; rd < PR; ++rd) {
        const long long g = max(gA[rd], 0ll);
        scA[rd] = __ldg(a.scales + g);
        moA[rd] = (!LEAN && a.world_mo) ? __ldg(a.world_mo + (long long)vi * a.n + g)
                                        : __ldg(a.means_opacity + g);
    }
#pragma unroll
    for (int rd = 0; rd < PR; ++rd) {
        const int li = rd * PT + tid;
        const long long i = i0 + li;
        bool keep = false;
        uint16_t tag = (uint16_t)li;
        if (i < n_t) {
            const int id = idA[rd];
            if (id < 0 || id >= K1) {
                c_bad++;
                if (!LEAN && a.dbg_flags) {
                    const long long di = V.dbg_off + i;
                    a.dbg_flags[di] = F_TEMPORAL | F_BADID;
#pragma unroll
                    for (int j = 0; j < 6; ++j) a.dbg_keys[6 * di + j] = __int_as_float(0x7fc00000);
#pragma unroll
                    for (int j = 0; j < 4; ++j) a.dbg_rect[4 * di + j] = 0;
                }
            } else {
                const bool out = surely_outside(s_tab + 12 * ((!LEAN && a.world_mo) ? 0 : id), moA[rd],
                                                scA[rd], V, lox, hix, loy, hiy);
                keep = !out || (!LEAN && a.dbg_flags);
                if (out) tag |= 0x8000u;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        int qb = 0;
        if (lane == 0 && bal) qb = atomicAdd(qn, __popc(bal));
        qb = __shfl_sync(0xffffffffu, qb, 0);
        if (keep) {
            qt[qb + __popc(bal & lt)] = tag;
            qg[qb + __popc(bal & lt)] = (uint32_t)gA[rd];
        }
    }
}

// K2 prologue: the view's camera table into
// shared memory and the tangent-plane clamp bounds (reading R5, R-ARITH order)
__device__ __forceinline__ void stage_view(const ProjectArgs& a, const DevView& V, float* s_tab,
                                           float* s_bounds)
{
    const int tid = threadIdx.x;
    for (int i = tid; i < a.num_instances * 12; i += PT) s_tab[i] = V.table[i];
    if (tid == 0) {
        const float Wf = (float)V.W, Hf = (float)V.H;
        s_bounds[0] = (-(0.15f * Wf) - V.cx) / V.fx;
        s_bounds[1] = ((1.15f * Wf) - V.cx) / V.fx;
        s_bounds[2] = (-(0.15f * Hf) - V.cy) / V.fy;
        s_bounds[3] = ((1.15f * Hf) - V.cy) / V.fy;
    }
}

#ifndef S3R_K2_MINB
#define S3R_K2_MINB 4     // 64 registers (A/B: K2 0.91 ms vs 1.03 at 3, 1.40 at 2)
#endif
// LEAN: no debug dumps, no NeurF record means, not the conventional pipeline,
// no LOD noisy offset (ProjectArgs::lean) — those paths compiled out, which
// keeps the splat in registers (the noisy offset's out-of-line call otherwise
// puts it on the stack)
template <int PR, bool LEAN>
__global__ void __launch_bounds__(PT, S3R_K2_MINB) k_project(ProjectArgs a)
{
    extern __shared__ float s_tab[];          // [K1][12]
    __shared__ float s_bounds[4];
#if !S3R_K2_WARP_COMPACT
    __shared__ uint32_t s_wcnt[PT / 32];
    __shared__ uint32_t s_base;
#endif
    __shared__ unsigned long long s_red[6][PT / 32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int vi = blockIdx.y;
    const DevView& V = a.views[vi];
    const long long n_t = V.n_temporal;
    // one chunk of PT * PR list entries per CTA (the capacity mode bounds
    // n_temporal by the reserved temporal_view, which sizes grid.x)
    const long long i0 = (long long)blockIdx.x * (PT * PR);
    if (i0 >= n_t) return;                    // uniform for the CTA
    [[maybe_unused]] const int K1 = a.num_instances;
    stage_view(a, V, s_tab, s_bounds);
    __syncthreads();
    const float lox = s_bounds[0], hix = s_bounds[1], loy = s_bounds[2], hiy = s_bounds[3];
    const int32_t* tl = a.tidx + (long long)V.tslot * a.idx_stride;
    const long long cap_off = V.cap_off;
    const float t = V.t;
    uint8_t* vis_out = V.visible;
    ViewCounters* ctr = a.counters + vi;
    const unsigned lt = (1u << lane) - 1u;

    unsigned long long c_vis = 0, c_small = 0, c_drop = 0, c_pairs = 0, c_bad = 0, c_spairs = 0;
    // ---- pass A (precull_chunk) queues the entries the conservative pre-test
    // cannot reject, so that pass B runs the exact path on dense warps (the
    // visible Gaussians are scattered through the index list: without the queue
    // nearly every warp holds one and pays the full path for all 32 lanes).
    __shared__ int s_qn;
    __shared__ uint16_t s_q[(PT * PR)];
    __shared__ uint32_t s_g[(PT * PR)];
    const uint16_t* qt = s_q;
    const uint32_t* qg = s_g;
    if (tid == 0) s_qn = 0;
    __syncthreads();
    precull_chunk<PR, LEAN>(a, V, vi, i0, n_t, tl, s_tab, lox, hix, loy, hiy, s_q, s_g, &s_qn, c_bad);
    __syncthreads();
    const int qn = s_qn;
    for (int qbase = 0; qbase < qn; qbase += PT) {
        const int qi = qbase + tid;
        const uint16_t tag = qi < qn ? qt[qi] : (uint16_t)0;
        const long long i = qi < qn ? i0 + (tag & 0x7fff) : n_t;
        const bool culled = tag & 0x8000u;
        Splat sp;
        sp.flags = 0;
        long long g = -1;
        int gid_id = 0;
        float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < n_t) {
            g = qg[qi];
            const int id = __ldg(a.ids + g);
            gid_id = id;
            {
                const float4 sc = __ldg(a.scales + g);
                float4 mo, q;
                int slot = id;
                if (!LEAN && a.world_mo) {      // conventional: the view's world copy, camera W_t
                    const long long wg = (long long)vi * a.n + g;
                    mo = __ldg(a.world_mo + wg);
                    q = __ldg(a.world_rot + wg);
                    slot = 0;
                } else {
                    mo = __ldg(a.means_opacity + g);
                    q = __ldg(a.rotations + g);
                }
                project_one<!LEAN>(s_tab + 12 * slot, mo, sc, q, V, lox, hix, loy, hiy, g, sp);
                if (culled && (sp.flags & F_VISIBLE)) atomicOr(a.err, ERR_PRECULL);
                if (sp.flags & F_VISIBLE) {
                    c_vis++;
                    if (vis_out) vis_out[g] = 1;
                    if (a.life) {
                        const float2 l = a.life[g];
                        float* lp = reinterpret_cast<float*>(a.life + g);
                        if (t < l.x) atomic_min_f(lp, t);
                        if (t > l.y) atomic_max_f(lp + 1, t);
                    }
                }
                if (sp.flags & F_SMALL) c_small++;
                if (sp.flags & F_DROPPED) c_drop++;
                if (sp.flags & F_RENDERED) {
                    col = __ldg(a.colors + g);
                    col.w = mo.w;    // opacity travels in the record
                    c_pairs += (unsigned long long)(sp.tx1 - sp.tx0 + 1) *
                               (unsigned long long)(sp.ty1 - sp.ty0 + 1);
                    const int sh = V.sshift;
                    c_spairs += (unsigned long long)((sp.tx1 >> sh) - (sp.tx0 >> sh) + 1) *
                                (unsigned long long)((sp.ty1 >> sh) - (sp.ty0 >> sh) + 1);
                }
            }
            if (!LEAN && a.dbg_flags) {
                const long long di = V.dbg_off + i;
                a.dbg_flags[di] = sp.flags;
#pragma unroll
                for (int j = 0; j < 6; ++j) a.dbg_keys[6 * di + j] = sp.k[j];
                const bool vis = sp.flags & F_VISIBLE;
                a.dbg_rect[4 * di + 0] = (int16_t)(vis ? sp.tx0 : 0);
                a.dbg_rect[4 * di + 1] = (int16_t)(vis ? sp.tx1 : 0);
                a.dbg_rect[4 * di + 2] = (int16_t)(vis ? sp.ty0 : 0);
                a.dbg_rect[4 * di + 3] = (int16_t)(vis ? sp.ty1 : 0);
            }
        }
#if S3R_K2_WARP_COMPACT
        // ---- compaction: ballot/popc per warp, one atomic per warp-round (the
        // record order is not needed: the depth sort restores (depth, index)) ----
        const bool rend = (sp.flags & F_RENDERED) != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, rend);
        unsigned long long wbase = 0;
        if (bal) {
            if (lane == 0) wbase = atomicAdd(&ctr->n_rendered, (unsigned long long)__popc(bal));
            wbase = __shfl_sync(0xffffffffu, wbase, 0);
        }
#else
        // ---- compaction: ballot/popc in the CTA, one atomic per CTA-round ----
        const bool rend = (sp.flags & F_RENDERED) != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, rend);
        if (lane == 0) s_wcnt[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
            const uint32_t c = lane < PT / 32 ? s_wcnt[lane] : 0u;
            uint32_t x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane < PT / 32) s_wcnt[lane] = x - c;
            const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
            if (lane == 0)
                s_base = tot ? (uint32_t)atomicAdd(&ctr->n_rendered, (unsigned long long)tot) : 0u;
        }
        __syncthreads();
        const unsigned long long wbase = (unsigned long long)s_base + s_wcnt[warp];
#endif
        if (rend) {
            const long long o = cap_off + (long long)wbase + __popc(bal & lt);
            const uint32_t rx = (uint32_t)sp.tx0 | ((uint32_t)sp.tx1 << 16);
            const uint32_t ry = (uint32_t)sp.ty0 | ((uint32_t)sp.ty1 << 16);
            float4* r = a.rec + 3 * o;
            r[0] = make_float4(sp.rm[0], sp.rm[1], sp.rm[2], col.w);
            // exp2-form blend coefficients (R-ARITH): qa = A (-log2e/2), qb = B (-log2e),
            // qc = C (-log2e/2)
            r[1] = make_float4(sp.A * -0x1.715476p-1f, sp.B * -0x1.715476p+0f,
                               sp.C * -0x1.715476p-1f, __uint_as_float(rx));
            r[2] = make_float4(col.x, col.y, col.z, __uint_as_float(ry));
            // depth-sort key (reading R11): depth bits above the Gaussian index,
            // so the order is (depth, index) whatever the compaction order was
            a.dkey[o] = ((unsigned long long)__float_as_uint(sp.rm[2]) << a.gbits) |
                        (unsigned long long)g;
            if (!LEAN && a.gidx) a.gidx[o] = (int32_t)g;
            if (!LEAN && a.rec_mu) a.rec_mu[o] = make_float4(sp.mu[0], sp.mu[1], sp.mu[2], __int_as_float(gid_id));
        }
    }
    // ---- per-view counters: one set of atomics per CTA ----
    unsigned long long cv[6] = {c_vis, c_small, c_drop, c_pairs, c_bad, c_spairs};
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        unsigned long long x = cv[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) s_red[j][warp] = x;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long t5[6] = {0, 0, 0, 0, 0, 0};
        for (int w = 0; w < PT / 32; ++w)
            for (int j = 0; j < 6; ++j) t5[j] += s_red[j][w];
        if (t5[5]) atomicAdd(&ctr->n_spairs, t5[5]);
        if (t5[0]) atomicAdd(&ctr->n_visible, t5[0]);
        if (t5[1]) atomicAdd(&ctr->n_small, t5[1]);
        if (t5[2]) atomicAdd(&ctr->n_dropped, t5[2]);
        if (t5[3]) atomicAdd(&ctr->n_pairs, t5[3]);
        if (t5[4]) {
            atomicAdd(&ctr->n_bad, t5[4]);
            atomicOr(a.err, ERR_BADID);
        }
    }
}

// W_{t,i} = W_t W_{t,i2g} in fp64 (R-ARITH dot3 order), rounded once.
__global__ void k_compose(const float* __restrict__ w2c, const float* __restrict__ i2g,
                          int n_views, int K, float* __restrict__ out)
{
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int K1 = K + 1;
    if (idx >= n_views * K1) return;
    const int v = idx / K1, i = idx % K1;
    const float* A = w2c + 12ll * v;
    float* O = out + 12ll * idx;
    if (i == 0) {
        for (int k = 0; k < 12; ++k) O[k] = A[k];
        return;
    }
    const float* B = i2g + 12ll * ((long long)v * K + (i - 1));
    for (int r = 0; r < 3; ++r) {
        const double a0 = A[4 * r + 0], a1 = A[4 * r + 1], a2 = A[4 * r + 2], a3 = A[4 * r + 3];
        for (int c = 0; c < 3; ++c) {
            double acc = a0 * (double)B[c];
            acc = __fma_rn(a1, (double)B[4 + c], acc);
            acc = __fma_rn(a2, (double)B[8 + c], acc);
            O[4 * r + c] = (float)acc;
        }
        double acc = __fma_rn(a0, (double)B[3], a3);
        acc = __fma_rn(a1, (double)B[7], acc);
        acc = __fma_rn(a2, (double)B[11], acc);
        O[4 * r + 3] = (float)acc;
    }
}

// K9: Eq.6 commit and P:183 reset.
__global__ void k_commit(float2* __restrict__ vis, float2* __restrict__ life, long long n,
                         float margin)
{
    const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (g >= n) return;
    const float2 l = life[g];
    float2 v;
    if (l.x > l.y) {
        v = make_float2(-1.0f, 1.0f);
    } else {
        v = make_float2(fmaxf(-1.0f, l.x - margin), fminf(1.0f, l.y + margin));
    }
    vis[g] = v;
    life[g] = make_float2(1.0f, -1.0f);
}

__global__ void k_reset(float2* __restrict__ vis, long long n)
{
    const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (g < n) vis[g] = make_float2(-1.0f, 1.0f);
}

// l_s -> -l_s (exact) so that one all-reduce MAX merges (min l_s, max l_e).
__global__ void k_life_flip(float2* __restrict__ life, long long n)
{
    const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (g < n) life[g].x = -life[g].x;
}

// ---- conventional pipeline C0 (NEXT-2; Fig.1a): the
// local-to-global transformation of every dynamic Gaussian, per view, that the
// streamlined stage removes.  mu_w = R mu + t, q_w = quat(R) (x) q, in the
// R-ARITH op order written out in DESIGN.md §4 (conventional pipeline C0).
__device__ void quat_from_rot(const float* M, float* q)   // M: 3x4 row-major pose
{
    const float r00 = M[0], r01 = M[1], r02 = M[2];
    const float r10 = M[4], r11 = M[5], r12 = M[6];
    const float r20 = M[8], r21 = M[9], r22 = M[10];
    const float tr = (r00 + r11) + r22;
    if (tr > 0.0f) {
        const float s = sqrtf(tr + 1.0f) * 2.0f;
        q[0] = 0.25f * s;
        q[1] = (r21 - r12) / s;
        q[2] = (r02 - r20) / s;
        q[3] = (r10 - r01) / s;
    } else if (r00 > r11 && r00 > r22) {
        const float s = sqrtf(((1.0f + r00) - r11) - r22) * 2.0f;
        q[0] = (r21 - r12) / s;
        q[1] = 0.25f * s;
        q[2] = (r01 + r10) / s;
        q[3] = (r02 + r20) / s;
    } else if (r11 > r22) {
        const float s = sqrtf(((1.0f + r11) - r00) - r22) * 2.0f;
        q[0] = (r02 - r20) / s;
        q[1] = (r01 + r10) / s;
        q[2] = 0.25f * s;
        q[3] = (r12 + r21) / s;
    } else {
        const float s = sqrtf(((1.0f + r22) - r00) - r11) * 2.0f;
        q[0] = (r10 - r01) / s;
        q[1] = (r02 + r20) / s;
        q[2] = (r12 + r21) / s;
        q[3] = 0.25f * s;
    }
}

constexpr int WT = 256;

__global__ void __launch_bounds__(WT) k_to_world(const float4* __restrict__ mo,
                                                 const float4* __restrict__ rot,
                                                 const int32_t* __restrict__ ids, int K1,
                                                 long long n, const DevView* __restrict__ views,
                                                 float4* __restrict__ wmo, float4* __restrict__ wrot)
{
    extern __shared__ float s_w[];          // [K1][12] poses, then [K1][4] quat(R)
    const int vi = blockIdx.y;
    const DevView& V = views[vi];
    float* s_q = s_w + 12 * K1;
    for (int i = threadIdx.x; i < 12 * K1; i += WT) s_w[i] = V.table[i];
    __syncthreads();
    for (int i = 1 + threadIdx.x; i < K1; i += WT) quat_from_rot(s_w + 12 * i, s_q + 4 * i);
    __syncthreads();
    const long long stride = (long long)gridDim.x * WT;
    for (long long g = blockIdx.x * (long long)WT + threadIdx.x; g < n; g += stride) {
        const int id = __ldg(ids + g);
        float4 m = __ldg(mo + g), q = __ldg(rot + g);
        if (id > 0 && id < K1) {
            const float* M = s_w + 12 * id;
            float p[3];
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                float acc = __fmaf_rn(M[4 * r + 0], m.x, M[4 * r + 3]);
                acc = __fmaf_rn(M[4 * r + 1], m.y, acc);
                acc = __fmaf_rn(M[4 * r + 2], m.z, acc);
                p[r] = acc;
            }
            m = make_float4(p[0], p[1], p[2], m.w);
            const float* a = s_q + 4 * id;
            float w = a[0] * q.x;
            w = __fmaf_rn(-a[1], q.y, w);
            w = __fmaf_rn(-a[2], q.z, w);
            w = __fmaf_rn(-a[3], q.w, w);
            float x = a[0] * q.y;
            x = __fmaf_rn(a[1], q.x, x);
            x = __fmaf_rn(a[2], q.w, x);
            x = __fmaf_rn(-a[3], q.z, x);
            float y = a[0] * q.z;
            y = __fmaf_rn(-a[1], q.w, y);
            y = __fmaf_rn(a[2], q.x, y);
            y = __fmaf_rn(a[3], q.y, y);
            float z = a[0] * q.w;
            z = __fmaf_rn(a[1], q.z, z);
            z = __fmaf_rn(-a[2], q.y, z);
            z = __fmaf_rn(a[3], q.x, z);
            q = make_float4(w, x, y, z);
        }
        const long long o = (long long)vi * n + g;
        wmo[o] = m;
        wrot[o] = q;
    }
}

__global__ void k_iota(int32_t* __restrict__ idx, long long n)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) idx[i] = (int32_t)i;
}

// small device -> host readback by stores into mapped page-locked memory: it
// does not queue on the copy engines, so it never waits behind bulk copies
// that other streams have in flight
__global__ void k_readback(const uint32_t* __restrict__ src, volatile uint32_t* dst, int words)
{
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = src[i];
}
}  // namespace

void launch_world(const float4* mo, const float4* rot, const int32_t* ids, int num_instances,
                  long long n, const DevView* views, int n_views, float4* wmo, float4* wrot,
                  cudaStream_t st)
{
    if (n == 0 || n_views == 0) return;
    const size_t smem = (size_t)num_instances * 16 * sizeof(float);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_to_world, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long blocks = std::min<long long>((n + WT - 1) / WT, 148ll * 8);
    k_to_world<<<dim3((unsigned)blocks, n_views), WT, smem, st>>>(mo, rot, ids, num_instances, n,
                                                                   views, wmo, wrot);
}

void launch_iota(int32_t* idx, long long n, cudaStream_t st)
{
    if (n == 0) return;
    k_iota<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(idx, n);
}

void launch_readback(void* host_mapped, const void* dev, size_t bytes, cudaStream_t st)
{
    if (bytes == 0) return;
    k_readback<<<1, 256, 0, st>>>(static_cast<const uint32_t*>(dev),
                                  static_cast<uint32_t*>(host_mapped), (int)(bytes / 4));
}

void launch_project(const ProjectArgs& a, cudaStream_t st)
{
    if (a.max_tiles == 0 || a.n_views == 0) return;
    const size_t smem = (size_t)a.num_instances * 12 * sizeof(float);
    const bool small_grid = (long long)a.max_tiles * a.n_views < 2 * 148;
    const dim3 grid = small_grid ? dim3(a.max_tiles * PR_BIG, a.n_views) : dim3(a.max_tiles, a.n_views);
    auto go = [&](auto kern) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, PT, smem, st>>>(a);
    };
#ifndef S3R_K2_LEAN
#define S3R_K2_LEAN 1
#endif
    const bool lean = S3R_K2_LEAN && a.lean;
    if (small_grid) {
        if (lean) go(k_project<1, true>);
        else go(k_project<1, false>);
    } else {
        if (lean) go(k_project<PR_BIG, true>);
        else go(k_project<PR_BIG, false>);
    }
}

int project_tile() { return PTILE; }

void launch_compose(const float* w2c, const float* i2g, int n_views, int K, float* out,
                    cudaStream_t st)
{
    const int total = n_views * (K + 1);
    if (total == 0) return;
    k_compose<<<(total + 127) / 128, 128, 0, st>>>(w2c, i2g, n_views, K, out);
}

void launch_commit(float2* vis, float2* life, long long n, float margin, cudaStream_t st)
{
    if (n == 0) return;
    k_commit<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vis, life, n, margin);
}

void launch_reset(float2* vis, long long n, cudaStream_t st)
{
    if (n == 0) return;
    k_reset<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vis, n);
}

void launch_life_flip(float2* life, long long n, cudaStream_t st)
{
    if (n == 0) return;
    k_life_flip<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(life, n);
}

}  // namespace s3r
