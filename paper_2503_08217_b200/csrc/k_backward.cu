// k_backward.cu — config 5: adjoint of the alpha blend (Eq.2) and
// of the instance-specific projection (Eq.1 P:107-112 through W_{t,i} of
// P:158-159), for the views of the last forward batch; plus the MSE helper.
//
// K7b k_raster_bwd: one warp per (view, tile), 8 pixels per thread (one column,
// every other row) as 4 packed fp32 pairs, so the per-splat warp reduction
// below is shared by 256 pixels (A/B: 37.1 ms vs 40.7 ms with the forward's
// 64-thread, 4-pixel layout).
// Every pixel knows from the forward its final transmittance and how many list
// entries it blended; the warp walks its tile list BACK TO FRONT in batches of
// 256 staged records (only those whose flush ellipse reaches the tile, from a
// compacted list built while staging), recomputes alpha with the forward's
// R-ARITH ops on packed pairs (so the flush / clamps / skips are the
// forward's), recovers T before each splat as T / (1 - alpha), and forms
//     dL/dc = w gC,  dL/dz = w gD,
//     dL/dalpha = T (c.gC + z gD) - (R + gT T_final) / (1 - alpha),
//     R += (c.gC + z gD) w,
// then dL/do = dL/dalpha exp(power) (unless alpha hit 0.99) and dL/dpower =
// dL/dalpha alpha (unless power was clamped at 0), and the conic / mean
// gradients of power = -1/2 (A dx^2 + C dy^2) - B dx dy.  The 10 per-splat
// sums are reduced over the warp with shuffles and added with one atomic per
// value per warp into the splat's accumulator (by depth rank).
//
// K2b k_project_bwd: per (view, rank): the chain rule from (mx, my, z, A, B,
// C, o, rgb) to the Gaussian's raw parameters (mean in its instance frame,
// linear scales, unnormalised quaternion, opacity, colour), atomically added
// into the caller's gradient arrays.
#include <algorithm>
#include <type_traits>

#include "s3r_internal.cuh"

namespace s3r {

namespace {

#ifndef S3R_BWD_RPIX
#define S3R_BWD_RPIX 8
#endif
#ifndef S3R_BWD_MINB
#define S3R_BWD_MINB 14     // 128 registers with NOBR (A/B: 31.7 ms; 16: 33.0, 12: 34.3, 18: 34.9)
#endif
#ifndef S3R_BWD_ADJ
#define S3R_BWD_ADJ 0   // adjacent-row pairs: neutral here (A/B 34.17 vs 34.15 ms)
#endif
#ifndef S3R_BWD_RPR
#define S3R_BWD_RPR 1   // records per warp reduction (1 or 2)
#endif
#ifndef S3R_POSE_GROUPS
#define S3R_POSE_GROUPS 4   // instances per warp reduced in registers in k_project_bwd
#endif
#ifndef S3R_BWD_ROWSKIP
#define S3R_BWD_ROWSKIP 0   // 1: skip a pair whose 4-row band is beyond the flush extent (A/B: 33.7 vs 31.7 ms: the branches stop the pairs interleaving; off)
#endif
#ifndef S3R_BWD_NOBR
#define S3R_BWD_NOBR 1  // no per-pair skip branch (A/B with MINB 14: 31.7 vs 34.1 ms)
#endif
#ifndef S3R_BWD_VRED
#define S3R_BWD_VRED 0  // 1: the 10 reduced values gathered into 3 lanes, added with vector REDs (v4, v4, v2)
#endif
#ifndef S3R_BWD_ULAST
#define S3R_BWD_ULAST 0 // 1: no per-pixel "entry before the pixel's stop" test in a batch every pixel of the warp reaches
#endif
#ifndef S3R_BWD_SMEMCOT
#define S3R_BWD_SMEMCOT 0 // 1: the per-pixel RGB cotangents and stops in shared memory (fewer registers)
#endif
#ifndef S3R_BWD_EX2
#define S3R_BWD_EX2 0   // 0: exact R-ARITH exp2 on pairs (A/B 35.9 ms); 1, 2: ex2.approx + re-decision (37.0, 36.6)
#endif
// pixels per thread; a tile is 256 pixels, so RT = 256 / RPIX threads, each
// warp covering BW columns of the tile and 32 / BW rows per k step
constexpr int RPIX = S3R_BWD_RPIX;
constexpr int RT = TILE * TILE / RPIX;
constexpr int BW = TILE / (RT / 32);
#ifndef S3R_BWD_RB
#define S3R_BWD_RB 256
#endif
constexpr int RB = S3R_BWD_RB;   // records staged per batch
constexpr int NW = RT / 32;        // warps (= pixel blocks) per tile CTA
}  // namespace
// per-splat accumulator stride in floats (16-byte rows for the vector REDs)
constexpr int ACC_STRIDE = S3R_BWD_VRED ? 12 : 10;
int splat_grad_stride() { return ACC_STRIDE; }
namespace {

#if S3R_BWD_EX2
__device__ __forceinline__ float s3r_exp2_b(float x)
{
    const float t = x + 12582912.0f;
    const float n = t - 12582912.0f;
    const float r = x - n;
    float p = 1.3264695880934596e-3f;
    p = __fmaf_rn(p, r, 9.671507403254509e-3f);
    p = __fmaf_rn(p, r, 5.550733208656311e-2f);
    p = __fmaf_rn(p, r, 2.4022243916988373e-1f);
    p = __fmaf_rn(p, r, 6.931470036506653e-1f);
    const float y = __fmaf_rn(p, r, 1.0f);
    return y * __uint_as_float((__float_as_uint(t) << 23) + 0x3F800000u);
}
#endif

__device__ __forceinline__ float rcp_approx(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

#if S3R_BWD_EX2
__device__ __forceinline__ float ex2_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
#endif

__device__ __forceinline__ float warp_sum(float x)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 neg2(float2 x) { return make_float2(-x.x, -x.y); }

// s3r_exp2_b on a pair (component-wise the same operations; -24 <= x <= 0)
__device__ __forceinline__ float2 s3r_exp2_pair(float2 x)
{
    const float2 t = __fadd2_rn(x, f2(12582912.0f));
    const float2 n = __fadd2_rn(t, f2(-12582912.0f));
    const float2 r = __fadd2_rn(x, neg2(n));
    float2 p = __ffma2_rn(f2(1.3264695880934596e-3f), r, f2(9.671507403254509e-3f));
    p = __ffma2_rn(p, r, f2(5.550733208656311e-2f));
    p = __ffma2_rn(p, r, f2(2.4022243916988373e-1f));
    p = __ffma2_rn(p, r, f2(6.931470036506653e-1f));
    const float2 y = __ffma2_rn(p, r, f2(1.0f));
    const float2 sc = make_float2(__uint_as_float((__float_as_uint(t.x) << 23) + 0x3F800000u),
                                  __uint_as_float((__float_as_uint(t.y) << 23) + 0x3F800000u));
    return __fmul2_rn(y, sc);
}

// HAS_D / HAS_T: some view has a depth / final-T cotangent (otherwise those
// terms are zero and compiled out)
template <bool HAS_D, bool HAS_T>
__global__ void __launch_bounds__(RT, S3R_BWD_MINB) k_raster_bwd(BackwardArgs a)
{
    __shared__ float4 s_rec[3 * RB];
    __shared__ uint8_t s_cl[NW][RB];   // per warp block: staged records reaching it
    __shared__ int s_wc[NW][NW];       // [staging warp][warp block] kept counts
    __shared__ int s_max;
#if S3R_BWD_SMEMCOT
    // per thread (column) and pair: the RGB cotangent pairs and the stops,
    // [P][tid] so that a warp's loads of one pair are contiguous
    __shared__ float2 s_gr[RPIX / 2][RT], s_gg[RPIX / 2][RT], s_gb[RPIX / 2][RT];
    __shared__ int2 s_last[RPIX / 2][RT];
#endif
    const int v = blockIdx.y;
    const DevView& V = a.views[v];
    const int tile = blockIdx.x;
    if (tile >= V.ntiles) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tile % V.TX, ty = tile / V.TX;
    const int px = tx * TILE + (tid >> 5) * BW + (lane % BW);
    const int py0 = ty * TILE + (lane / BW);
    const float fpx = (float)px;
    // centre of the warp's BW x TILE pixel block (flush-ellipse culling; the
    // stored extents include the 8 x 16 block's half size, so a wider block
    // adds the difference)
    static_assert(TILE == 16 && BW >= 8, "cull extents assume >= 8 x 16 warp blocks");
    constexpr float XPAD = 0.5f * (BW - 1) - CULL_HALF_BX;
    const float bcx0 = (float)(tx * TILE) + 0.5f * (BW - 1);     // warp block 0
    const float bcy = (float)(ty * TILE) + CULL_HALF_BY;
#if S3R_BWD_ROWSKIP
    static_assert(!S3R_BWD_ADJ && RPIX == 8 && BW == 16, "row bands assume rows py0 + 2k");
    const float band_c0 = (float)(ty * TILE) + 1.5f;     // centre of pair 0's row band
#endif
    const s3r_cot C = a.cots[v];
    // the thread's RPIX pixels of one column as RPIX / 2 packed pairs: pair P holds
    // k = 2P (.x) and 2P + 1 (.y); sm_100a FADD2/FMUL2/FFMA2 work on both
    float Tk[RPIX], gtTk[RPIX], grk[RPIX], ggk[RPIX], gbk[RPIX], gdk[RPIX], nfk[RPIX];
    int last[RPIX];
    int mymax = 0;
#pragma unroll
    for (int k = 0; k < RPIX; ++k) {
#if S3R_BWD_ADJ
        // the two pixels of a packed pair are vertically adjacent (as in K7)
        const int py = ty * TILE + 2 * (32 / BW) * (k >> 1) + 2 * (lane / BW) + (k & 1);
#else
        const int py = py0 + (32 / BW) * k;
#endif
        nfk[k] = -(float)py;
        last[k] = 0;
        Tk[k] = 1.0f;
        grk[k] = ggk[k] = gbk[k] = gdk[k] = gtTk[k] = 0.0f;
        if (px < V.W && py < V.H) {
            const long long pix = (long long)py * V.W + px;
            last[k] = a.train_n[V.pix_off + pix];
            Tk[k] = a.train_T[V.pix_off + pix];
            grk[k] = C.rgb[3 * pix];
            ggk[k] = C.rgb[3 * pix + 1];
            gbk[k] = C.rgb[3 * pix + 2];
            if (HAS_D && C.depth) gdk[k] = C.depth[pix];
            if (HAS_T && C.final_T) gtTk[k] = C.final_T[pix] * Tk[k];
            mymax = max(mymax, last[k]);
        }
    }
    constexpr int NP = RPIX / 2;
    float2 Tc[NP], gtTf[NP], Rr[NP], gr[NP], gg[NP], gb[NP], gd[NP], nfpy[NP];
#pragma unroll
    for (int P = 0; P < NP; ++P) {
        Tc[P] = make_float2(Tk[2 * P], Tk[2 * P + 1]);
        gtTf[P] = make_float2(gtTk[2 * P], gtTk[2 * P + 1]);
#if S3R_BWD_SMEMCOT
        s_gr[P][tid] = make_float2(grk[2 * P], grk[2 * P + 1]);
        s_gg[P][tid] = make_float2(ggk[2 * P], ggk[2 * P + 1]);
        s_gb[P][tid] = make_float2(gbk[2 * P], gbk[2 * P + 1]);
        s_last[P][tid] = make_int2(last[2 * P], last[2 * P + 1]);
#else
        gr[P] = make_float2(grk[2 * P], grk[2 * P + 1]);
        gg[P] = make_float2(ggk[2 * P], ggk[2 * P + 1]);
        gb[P] = make_float2(gbk[2 * P], gbk[2 * P + 1]);
#endif
        gd[P] = make_float2(gdk[2 * P], gdk[2 * P + 1]);
        nfpy[P] = make_float2(nfk[2 * P], nfk[2 * P + 1]);
        Rr[P] = f2(0.0f);
    }
    if (tid == 0) s_max = 0;
    __syncthreads();
    atomicMax(&s_max, mymax);
    __syncthreads();
    // the smallest stop over the thread's pixels (pixels outside the image have
    // last = 0 and never differentiate anything)
    int minlast = last[0];
#pragma unroll
    for (int k = 1; k < RPIX; ++k) minlast = min(minlast, last[k]);
    const int2 rg = a.tranges[V.trange_off + tile];
    const uint32_t* lst = a.tlists + V.tlist_off;
    const float4* recs = a.rec_sorted + 3 * V.cap_off;
    float* acc = a.splat_grads + (long long)ACC_STRIDE * V.cap_off;
    // conic from the exp2-form coefficients: qa = A (-log2e/2), qb = B (-log2e),
    // qc = C (-log2e/2)  =>  A = qa (-2 ln2), B = qb (-ln2), C = qc (-2 ln2)
    const float k2 = -1.3862943611198906f, k1 = -0.6931471805599453f;
    for (int hi = s_max; hi > 0;) {
        const int lo = max(0, hi - RB);
        const int nb = hi - lo;
        __syncthreads();
        // stage the batch and, per warp block, the order-preserving list of the
        // records whose flush ellipse reaches it (the others were flushed on
        // every pixel of the block in the forward: nothing to differentiate)
        int run[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) run[w] = 0;
        for (int base = 0; base < nb; base += RT) {
            const int i = base + tid;
            bool keep[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) keep[w] = false;
            if (i < nb) {
                const uint32_t e = lst[rg.x + lo + i];
                const float4* src = recs + 3ll * e;
                const float4 r0 = src[0];
                float4 r1 = src[1];
                const float4 r2 = src[2];
                const float hx = XPAD != 0.0f ? r1.w + XPAD : r1.w;
                const bool yok = !S3R_CULL || !(fabsf(r0.y - bcy) > r2.w);
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    keep[w] = yok && (!S3R_CULL || !(fabsf(r0.x - (bcx0 + (float)(w * BW))) > hx));
                r1.w = __uint_as_float(e);            // list entry, for the atomics
                s_rec[3 * i + 0] = r0;
                s_rec[3 * i + 1] = r1;
                s_rec[3 * i + 2] = r2;
            }
            unsigned bal[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                bal[w] = __ballot_sync(0xffffffffu, keep[w]);
                if (lane == 0) s_wc[warp][w] = __popc(bal[w]);
            }
            __syncthreads();
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                int off = run[w], tot = 0;
#pragma unroll
                for (int sw = 0; sw < NW; ++sw) {
                    const int c = s_wc[sw][w];
                    if (sw < warp) off += c;
                    tot += c;
                }
                if (keep[w]) s_cl[w][off + __popc(bal[w] & ((1u << lane) - 1u))] = (uint8_t)i;
                run[w] += tot;
            }
            __syncthreads();
        }
        // one record (by staged index jj): per-pixel recurrences (T, R) and the
        // thread's partial sums -> v10 (the splat's 10 gradient values before the
        // warp reduction); returns whether any pixel of the thread contributed
        auto eval_record = [&](int jj, float* v10, auto chk_tag) -> bool {
            constexpr bool CHK = decltype(chk_tag)::value;   // test j < last per pixel
            const int j = lo + jj;
            const float4 q0 = s_rec[3 * jj], q1 = s_rec[3 * jj + 1], q2 = s_rec[3 * jj + 2];
            const float dx = q0.x - fpx;
            const float a1 = q1.x * dx;
            const float a2 = a1 * dx;
            const float b1 = q1.y * dx;
            const float A = q1.x * k2, B = q1.y * k1, Cc = q1.z * k2;
            // per-thread partial sums (pairs, summed before the warp reduction);
            // the conic / mean terms factor through the thread's shared column
            // offset dx: with gP the power gradient,
            //   sum gP dx^2 = dx^2 S0, sum gP dx dy = dx S1, sum gP dy^2 = S2
            float2 S0 = f2(0.f), S1 = f2(0.f), S2 = f2(0.f), s_z = f2(0.f), s_o = f2(0.f),
                   s_r = f2(0.f), s_g = f2(0.f), s_b = f2(0.f);
            bool any = false;
#if S3R_BWD_ROWSKIP
            // pair P of every lane covers the 4-row band [4P, 4P + 3] of the tile:
            // a band beyond the record's flush-ellipse y extent (q2.w minus the
            // 16-row block half size, s3r_internal.cuh flush_extent) is flushed
            // for all its pixels — skipped warp-uniformly
            const float thr = q2.w - (CULL_HALF_BY - 1.5f);
            const float dyc = q0.y - band_c0;
#endif
#pragma unroll
            for (int P = 0; P < NP; ++P) {
#if S3R_BWD_ROWSKIP
                if (fabsf(dyc - 4.0f * P) > thr) continue;
#endif
                const float2 dy = __fadd2_rn(f2(q0.y), nfpy[P]);
                const float2 c1 = __ffma2_rn(f2(q1.z), dy, f2(b1));
                const float2 e2raw = __ffma2_rn(dy, c1, f2(a2));
                const float2 e2 = make_float2(fminf(0.0f, e2raw.x), fminf(0.0f, e2raw.y));
                // entries after the pixel's termination, or flushed in the forward
                // (alpha = 0): nothing to differentiate
#if S3R_BWD_SMEMCOT
                const int2 lst2 = CHK ? s_last[P][tid] : make_int2(0, 0);
                const bool okx = (!CHK || j < lst2.x) && e2.x >= -24.0f;
                const bool oky = (!CHK || j < lst2.y) && e2.y >= -24.0f;
                const float2 grP = s_gr[P][tid], ggP = s_gg[P][tid], gbP = s_gb[P][tid];
#else
                const bool okx = (!CHK || j < last[2 * P]) && e2.x >= -24.0f;
                const bool oky = (!CHK || j < last[2 * P + 1]) && e2.y >= -24.0f;
                const float2 grP = gr[P], ggP = gg[P], gbP = gb[P];
#endif
#if S3R_BWD_NOBR
                // branch-free: a pair with neither pixel ok gets G = 0 below, which
                // leaves T, R and every sum bit-identical; the pairs' dependency
                // chains can then interleave
                any = any || okx || oky;
#else
                if (!(okx || oky)) continue;
#endif
#if S3R_BWD_EX2 == 1
                // hardware exp2 (rel. error ~2^-22); the forward's clamp decision
                // (o G < 0.99) is re-taken with the exact R-ARITH exp2 whenever
                // the approximate product lies within 1e-5 of the threshold
                float2 G = make_float2(ex2_approx(e2.x), ex2_approx(e2.y));
                float2 og = __fmul2_rn(f2(q0.w), G);
                if (fabsf(og.x - 0.99f) < 1e-5f) {
                    G.x = s3r_exp2_b(e2.x);
                    og.x = q0.w * G.x;
                }
                if (fabsf(og.y - 0.99f) < 1e-5f) {
                    G.y = s3r_exp2_b(e2.y);
                    og.y = q0.w * G.y;
                }
#elif S3R_BWD_EX2 == 2
                // as 1, one branch for the pair
                float2 G = make_float2(ex2_approx(e2.x), ex2_approx(e2.y));
                float2 og = __fmul2_rn(f2(q0.w), G);
                const float2 dd = __fadd2_rn(og, f2(-0.99f));
                if (fminf(fabsf(dd.x), fabsf(dd.y)) < 1e-5f) {
                    G = s3r_exp2_pair(e2);
                    og = __fmul2_rn(f2(q0.w), G);
                }
#else
                // the exact R-ARITH exp2 on the pair (the forward's values)
                const float2 G = s3r_exp2_pair(e2);
#endif
                // a pixel of the pair that is not ok gets G = 0, hence o G = 0,
                // alpha = 0: T, R and the sums are unchanged, and its o / power
                // gradients (go G, go alpha) vanish — one select per pixel
                const float2 Gm = make_float2(okx ? G.x : 0.0f, oky ? G.y : 0.0f);
                const float2 ogm = __fmul2_rn(f2(q0.w), Gm);
                const float2 alpha = make_float2(fminf(0.99f, ogm.x), fminf(0.99f, ogm.y));
                const float2 om = __fadd2_rn(f2(1.0f), neg2(alpha));
                const float2 inv = make_float2(rcp_approx(om.x), rcp_approx(om.y));
                const float2 Tb = __fmul2_rn(Tc[P], inv);        // T before this splat
                const float2 w = __fmul2_rn(alpha, Tb);
                float2 cdot = __fmul2_rn(f2(q2.x), grP);
                cdot = __ffma2_rn(f2(q2.y), ggP, cdot);
                cdot = __ffma2_rn(f2(q2.z), gbP, cdot);
                if (HAS_D) cdot = __ffma2_rn(f2(q0.z), gd[P], cdot);
                // dL/dalpha = T (c.gC + z gD) - (R + gT T_final) / (1 - alpha)
                const float2 rest = __fmul2_rn(HAS_T ? __fadd2_rn(Rr[P], gtTf[P]) : Rr[P], inv);
                const float2 galpha = __ffma2_rn(Tb, cdot, neg2(rest));
                Rr[P] = __ffma2_rn(cdot, w, Rr[P]);
                Tc[P] = Tb;
#if !S3R_BWD_NOBR
                any = true;
#endif
                s_r = __ffma2_rn(w, grP, s_r);
                s_g = __ffma2_rn(w, ggP, s_g);
                s_b = __ffma2_rn(w, gbP, s_b);
                if (HAS_D) s_z = __ffma2_rn(w, gd[P], s_z);
                // alpha clamped at 0.99: no gradient to o or the power;
                // power clamped at 0 (e2raw > 0): no gradient to the power
                const float2 go = make_float2(ogm.x < 0.99f ? galpha.x : 0.0f,
                                              ogm.y < 0.99f ? galpha.y : 0.0f);
                s_o = __ffma2_rn(go, Gm, s_o);
                float2 gP = __fmul2_rn(go, alpha);
                gP.x = e2raw.x <= 0.0f ? gP.x : 0.0f;
                gP.y = e2raw.y <= 0.0f ? gP.y : 0.0f;
                const float2 t = __fmul2_rn(gP, dy);
                S0 = __fadd2_rn(S0, gP);
                S1 = __fadd2_rn(S1, t);
                S2 = __ffma2_rn(t, dy, S2);
            }
                const float S0s = S0.x + S0.y, S1s = S1.x + S1.y, S2s = S2.x + S2.y;
                const float dS0 = dx * S0s;
                const float vv[10] = {-(A * dS0 + B * S1s), -(B * dS0 + Cc * S1s), s_z.x + s_z.y,
                                       -0.5f * dx * dS0, -dx * S1s, -0.5f * S2s,
                                       s_o.x + s_o.y, s_r.x + s_r.y, s_g.x + s_g.y, s_b.x + s_b.y};
#pragma unroll
            for (int i = 0; i < 10; ++i) v10[i] = vv[i];
            return any;
        };
#if S3R_BWD_RPR == 2
        // two records per warp reduction: 20 values, 21 shuffles (10 at distance
        // 16 separate the records, then the 10-value scheme below per record)
        for (int kk = run[warp] - 1; kk >= 0; kk -= 2) {
            const int jjA = s_cl[warp][kk];
            float vA[10], vB[10];
            const bool anyA = eval_record(jjA, vA, std::true_type{});
            const bool hasB = kk >= 1;                      // warp-uniform
            int jjB = 0;
            bool anyB = false;
            if (hasB) {
                jjB = s_cl[warp][kk - 1];
                anyB = eval_record(jjB, vB, std::true_type{});
            } else {
#pragma unroll
                for (int i = 0; i < 10; ++i) vB[i] = 0.0f;
            }
            if (__any_sync(0xffffffffu, anyA || anyB)) {
                const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4, u2 = lane & 2, u1 = lane & 1;
                float v10[10], v5[5], v3[3], v2[2];
#pragma unroll
                for (int i = 0; i < 10; ++i)
                    v10[i] = (u16 ? vB[i] : vA[i]) +
                             __shfl_xor_sync(0xffffffffu, u16 ? vA[i] : vB[i], 16);
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    v5[i] = (u8 ? v10[5 + i] : v10[i]) +
                            __shfl_xor_sync(0xffffffffu, u8 ? v10[i] : v10[5 + i], 8);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const float hiv = i < 2 ? v5[3 + i] : 0.0f;
                    v3[i] = (u4 ? hiv : v5[i]) + __shfl_xor_sync(0xffffffffu, u4 ? v5[i] : hiv, 4);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float hiv = i < 1 ? v3[2 + i] : 0.0f;
                    v2[i] = (u2 ? hiv : v3[i]) + __shfl_xor_sync(0xffffffffu, u2 ? v3[i] : hiv, 2);
                }
                const float v1 = (u1 ? v2[1] : v2[0]) + __shfl_xor_sync(0xffffffffu, u1 ? v2[0] : v2[1], 1);
                const int inner = 5 * u8 + 3 * u4 + 2 * u2 + u1;
                if (2 * u2 + u1 <= 2 && 3 * u4 + 2 * u2 + u1 <= 4 && (!u16 || hasB)) {
                    const int jjR = u16 ? jjB : jjA;
                    const uint32_t g = __float_as_uint(s_rec[3 * jjR + 1].w);   // list entry
                    atomicAdd(acc + (long long)ACC_STRIDE * g + inner, v1);
                }
            }
        }
#else
        // every pixel of the warp differentiates every entry of this batch
        // (its stop lies at or beyond the batch's end): no per-pixel test
        const bool full = S3R_BWD_ULAST && __all_sync(0xffffffffu, minlast >= hi);
        for (int kk = run[warp] - 1; kk >= 0; --kk) {
            const int jj = s_cl[warp][kk];
            const float4 q1 = s_rec[3 * jj + 1];
            float v10[10];
            const bool any = full ? eval_record(jj, v10, std::false_type{})
                                  : eval_record(jj, v10, std::true_type{});
            if (__any_sync(0xffffffffu, any)) {
                const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4, u2 = lane & 2;
                float v5[5], v3[3], v2[2];
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    v5[i] = (u16 ? v10[5 + i] : v10[i]) +
                            __shfl_xor_sync(0xffffffffu, u16 ? v10[i] : v10[5 + i], 16);
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    const float hiv = i < 2 ? v5[3 + i] : 0.0f;
                    v3[i] = (u8 ? hiv : v5[i]) + __shfl_xor_sync(0xffffffffu, u8 ? v5[i] : hiv, 8);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float hiv = i < 1 ? v3[2 + i] : 0.0f;
                    v2[i] = (u4 ? hiv : v3[i]) + __shfl_xor_sync(0xffffffffu, u4 ? v3[i] : hiv, 4);
                }
                float v1 = (u2 ? v2[1] : v2[0]) + __shfl_xor_sync(0xffffffffu, u2 ? v2[0] : v2[1], 2);
                v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
                const uint32_t g = __float_as_uint(q1.w);        // list entry staged in .w
#if S3R_BWD_VRED
                // value i now sits in lane L(i) = {0, 2, 4, 8, 10, 16, 18, 20, 24, 26}[i];
                // lanes 0, 1, 2 gather values 0-3, 4-7, 8-9 (slot s of lane l reads
                // byte l of SRC[s]) and add them with one vector RED each
                constexpr uint32_t SRC0 = 0x00180a00u, SRC1 = 0x001a1002u, SRC2 = 0x00001204u,
                                   SRC3 = 0x00001408u;
                const int sh = 8 * (lane & 3);
                const float w0 = __shfl_sync(0xffffffffu, v1, (SRC0 >> sh) & 31);
                const float w1 = __shfl_sync(0xffffffffu, v1, (SRC1 >> sh) & 31);
                const float w2 = __shfl_sync(0xffffffffu, v1, (SRC2 >> sh) & 31);
                const float w3 = __shfl_sync(0xffffffffu, v1, (SRC3 >> sh) & 31);
                float* dst = acc + (long long)ACC_STRIDE * g + 4 * lane;
                if (lane < 2)
                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};"
                                 ::"l"(dst), "f"(w0), "f"(w1), "f"(w2), "f"(w3) : "memory");
                else if (lane == 2)
                    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};"
                                 ::"l"(dst), "f"(w0), "f"(w1) : "memory");
#else
                const int inner = 3 * u8 + 2 * u4 + u2;
                if (!(lane & 1) && 2 * u4 + u2 <= 2 && inner <= 4)
                    atomicAdd(acc + (long long)ACC_STRIDE * g + 5 * u16 + inner, v1);
#endif
            }
        }
#endif
        hi = lo;
    }
}

// chain rule of one splat (view V, depth rank r): atomics into the caller's
// per-Gaussian gradients; gm12 = its dL/d(instance camera) when requested.
// Returns the instance id, or -1 when the splat has no gradient.
__device__ __forceinline__ int project_bwd_one(const BackwardArgs& a, const DevView& V,
                                               long long r, float* gm12)
{
    const float* acc = a.splat_grads + (long long)ACC_STRIDE * (V.cap_off + r);
    const float gmx = acc[0], gmy = acc[1], gz = acc[2], gA = acc[3], gB = acc[4], gC = acc[5],
                go = acc[6], gcr = acc[7], gcg = acc[8], gcb = acc[9];
    if (gmx == 0.f && gmy == 0.f && gz == 0.f && gA == 0.f && gB == 0.f && gC == 0.f &&
        go == 0.f && gcr == 0.f && gcg == 0.f && gcb == 0.f)
        return -1;
    const long long g = (long long)(a.dkey_sorted[V.cap_off + r] & a.gmask);
    const int id = a.ids[g];
    const float* M = V.table + 12 * id;
    float4 mo = a.means_opacity[g];
    const float4 sc = a.scales[g], qq = a.rotations[g];
    if (a.rec_mu) {
        // rendered from the mean moved by the LOD noisy offset (NEXT-3): the
        // adjoint runs there; the offset is a constant (reading R23), so the
        // mean gradient is the moved mean's
        const float4 m = a.rec_mu[V.cap_off + a.order[V.cap_off + r]];
        mo.x = m.x; mo.y = m.y; mo.z = m.z;
    }
    float p[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) p[i] = M[4 * i] * mo.x + M[4 * i + 1] * mo.y + M[4 * i + 2] * mo.z + M[4 * i + 3];
    const float qn = sqrtf(qq.x * qq.x + qq.y * qq.y + qq.z * qq.z + qq.w * qq.w);
    const float w = qq.x / qn, x = qq.y / qn, y = qq.z / qn, zq = qq.w / qn;
    float Rq[9];
    Rq[0] = 1.f - 2.f * (y * y + zq * zq); Rq[1] = 2.f * (x * y - w * zq); Rq[2] = 2.f * (x * zq + w * y);
    Rq[3] = 2.f * (x * y + w * zq); Rq[4] = 1.f - 2.f * (x * x + zq * zq); Rq[5] = 2.f * (y * zq - w * x);
    Rq[6] = 2.f * (x * zq - w * y); Rq[7] = 2.f * (y * zq + w * x); Rq[8] = 1.f - 2.f * (x * x + y * y);
    const float sg[3] = {sc.x, sc.y, sc.z};
    float WR[9], T[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            WR[3 * i + c] = M[4 * i] * Rq[c] + M[4 * i + 1] * Rq[3 + c] + M[4 * i + 2] * Rq[6 + c];
            T[3 * i + c] = WR[3 * i + c] * sg[c];
        }
    const float fx = V.fx, fy = V.fy;
    const float Wf = (float)V.W, Hf = (float)V.H;
    const float lox = (-(0.15f * Wf) - V.cx) / fx, hix = ((1.15f * Wf) - V.cx) / fx;
    const float loy = (-(0.15f * Hf) - V.cy) / fy, hiy = ((1.15f * Hf) - V.cy) / fy;
    const float pz = p[2];
    const float u = p[0] / pz, vv = p[1] / pz;
    const bool uclamp = (u < lox || u > hix), vclamp = (vv < loy || vv > hiy);
    const float uc = fminf(fmaxf(u, lox), hix), vc = fminf(fmaxf(vv, loy), hiy);
    const float J[6] = {fx / pz, 0.f, -fx * uc / pz, 0.f, fy / pz, -fy * vc / pz};
    float U[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) U[3 * i + c] = J[3 * i] * T[c] + J[3 * i + 1] * T[3 + c] + J[3 * i + 2] * T[6 + c];
    const float ka = U[0] * U[0] + U[1] * U[1] + U[2] * U[2];
    const float kb = U[0] * U[3] + U[1] * U[4] + U[2] * U[5];
    const float kc = U[3] * U[3] + U[4] * U[4] + U[5] * U[5];
    const float ad = ka + 0.3f, cd = kc + 0.3f, det = ad * cd - kb * kb;
    const float Q[4] = {cd / det, -kb / det, -kb / det, ad / det};
    // conic -> Sigma'_dil: G_S = -Q G_Q Q, G_Q = [[gA, gB/2], [gB/2, gC]]
    const float GQ[4] = {gA, 0.5f * gB, 0.5f * gB, gC};
    float QG[4], GS[4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) QG[2 * i + j] = Q[2 * i] * GQ[j] + Q[2 * i + 1] * GQ[2 + j];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) GS[2 * i + j] = -(QG[2 * i] * Q[j] + QG[2 * i + 1] * Q[2 + j]);
    float gU[6];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) gU[3 * i + k] = 2.f * (GS[2 * i] * U[k] + GS[2 * i + 1] * U[3 + k]);
    float gJ[6], gT[9];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) gJ[3 * i + k] = gU[3 * i] * T[3 * k] + gU[3 * i + 1] * T[3 * k + 1] + gU[3 * i + 2] * T[3 * k + 2];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int c = 0; c < 3; ++c) gT[3 * k + c] = J[k] * gU[c] + J[3 + k] * gU[3 + c];
    float gs[3] = {0.f, 0.f, 0.f}, gWR[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            gs[c] += gT[3 * i + c] * WR[3 * i + c];
            gWR[3 * i + c] = gT[3 * i + c] * sg[c];
        }
    float gR[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) gR[3 * i + c] = M[i] * gWR[c] + M[4 + i] * gWR[3 + c] + M[8 + i] * gWR[6 + c];
    const float dRw[9] = {0.f, -2.f * zq, 2.f * y, 2.f * zq, 0.f, -2.f * x, -2.f * y, 2.f * x, 0.f};
    const float dRx[9] = {0.f, 2.f * y, 2.f * zq, 2.f * y, -4.f * x, -2.f * w, 2.f * zq, 2.f * w, -4.f * x};
    const float dRy[9] = {-4.f * y, 2.f * x, 2.f * w, 2.f * x, 0.f, 2.f * zq, -2.f * w, 2.f * zq, -4.f * y};
    const float dRz[9] = {-4.f * zq, -2.f * w, 2.f * x, 2.f * w, -4.f * zq, 2.f * y, 2.f * x, 2.f * y, 0.f};
    float gq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        gq[0] += gR[k] * dRw[k];
        gq[1] += gR[k] * dRx[k];
        gq[2] += gR[k] * dRy[k];
        gq[3] += gR[k] * dRz[k];
    }
    const float qh[4] = {w, x, y, zq};
    const float dotq = qh[0] * gq[0] + qh[1] * gq[1] + qh[2] * gq[2] + qh[3] * gq[3];
    float gp0 = 0.f, gp1 = 0.f, gp2 = 0.f;
    const float iz2 = 1.f / (pz * pz);
    gp2 += gJ[0] * (-fx * iz2) + gJ[4] * (-fy * iz2);
    if (uclamp) {
        gp2 += gJ[2] * (fx * uc * iz2);
    } else {
        gp0 += gJ[2] * (-fx * iz2);
        gp2 += gJ[2] * (2.f * fx * p[0] * iz2 / pz);
    }
    if (vclamp) {
        gp2 += gJ[5] * (fy * vc * iz2);
    } else {
        gp1 += gJ[5] * (-fy * iz2);
        gp2 += gJ[5] * (2.f * fy * p[1] * iz2 / pz);
    }
    gp0 += gmx * fx / pz;
    gp2 += gmx * (-fx * p[0] * iz2);
    gp1 += gmy * fy / pz;
    gp2 += gmy * (-fy * p[1] * iz2);
    gp2 += gz;
    if (a.g_table) {
        // NEXT-1 pose gradient: M = [Wr | t], p = Wr mu + t, WR = Wr R_q:
        // dL/dWr = gp mu^T + gWR R_q^T, dL/dt = gp
        const float gpv[3] = {gp0, gp1, gp2}, muv[3] = {mo.x, mo.y, mo.z};
#pragma unroll
        for (int i = 0; i < 3; ++i) {
#pragma unroll
            for (int k = 0; k < 3; ++k)
                gm12[4 * i + k] = gpv[i] * muv[k] + gWR[3 * i] * Rq[3 * k] +
                                  gWR[3 * i + 1] * Rq[3 * k + 1] + gWR[3 * i + 2] * Rq[3 * k + 2];
            gm12[4 * i + 3] = gpv[i];
        }
    }
    float* gm = a.g_means + 4 * g;
    atomicAdd(gm + 0, M[0] * gp0 + M[4] * gp1 + M[8] * gp2);
    atomicAdd(gm + 1, M[1] * gp0 + M[5] * gp1 + M[9] * gp2);
    atomicAdd(gm + 2, M[2] * gp0 + M[6] * gp1 + M[10] * gp2);
    atomicAdd(gm + 3, go);
    float* gsc = a.g_scales + 4 * g;
    atomicAdd(gsc + 0, gs[0]);
    atomicAdd(gsc + 1, gs[1]);
    atomicAdd(gsc + 2, gs[2]);
    float* gro = a.g_rot + 4 * g;
#pragma unroll
    for (int k = 0; k < 4; ++k) atomicAdd(gro + k, (gq[k] - qh[k] * dotq) / qn);
    float* gco = a.g_colors + 4 * g;
    atomicAdd(gco + 0, gcr);
    atomicAdd(gco + 1, gcg);
    atomicAdd(gco + 2, gcb);
    return id;
}

__global__ void __launch_bounds__(256) k_project_bwd(BackwardArgs a)
{
    extern __shared__ float s_gt[];          // [K1][12] pose-gradient partials (if requested)
    const int vi = blockIdx.y;
    const DevView& V = a.views[vi];
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool use_smem = a.g_table && a.smem_table;
    if (use_smem)
        for (int i = threadIdx.x; i < 12 * a.num_instances; i += blockDim.x) s_gt[i] = 0.0f;
    if (use_smem) __syncthreads();
    if ((long long)blockIdx.x * blockDim.x >= V.n_rendered) return;     // uniform for the CTA
    float gm12[12];
#pragma unroll
    for (int j = 0; j < 12; ++j) gm12[j] = 0.0f;
    const int id = r < V.n_rendered ? project_bwd_one(a, V, r, gm12) : -1;
    if (!a.g_table) return;
    float* gt_view = a.g_table + (long long)vi * a.num_instances * 12;
    // a warp whose active splats share one instance (the common case: static)
    // reduces in registers first; otherwise per-splat shared atomics
    const int lane = threadIdx.x & 31;
    const bool act = id >= 0;
    const unsigned am = __ballot_sync(0xffffffffu, act);
    if (am) {
        float* dst = use_smem ? s_gt : gt_view;
        // segmented by instance: up to S3R_POSE_GROUPS instances of the warp are
        // reduced in registers (one warp sum per value, one atomic by the group's
        // first lane); splats of further instances add their own values (depth
        // order mixes instances, but a warp rarely holds more than a few)
        unsigned rem = am;
        for (int it = 0; it < S3R_POSE_GROUPS && rem; ++it) {
            const int leader = __ffs(rem) - 1;
            const int idl = __shfl_sync(0xffffffffu, id, leader);
            const bool mine = act && id == idl;
            rem &= ~__ballot_sync(0xffffffffu, mine);
#pragma unroll
            for (int j = 0; j < 12; ++j) {
                const float v = warp_sum(mine ? gm12[j] : 0.0f);
                if (lane == leader) atomicAdd(dst + 12 * idl + j, v);
            }
        }
        if ((rem >> lane) & 1u) {
#pragma unroll
            for (int j = 0; j < 12; ++j) atomicAdd(dst + 12 * id + j, gm12[j]);
        }
    }
    if (use_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < 12 * a.num_instances; i += blockDim.x)
            if (s_gt[i] != 0.0f) atomicAdd(gt_view + i, s_gt[i]);
    }
}

__global__ void __launch_bounds__(256) k_mse(const float* __restrict__ x,
                                             const float* __restrict__ y, long long n,
                                             float scale, float* __restrict__ grad,
                                             float* __restrict__ loss)
{
    // float4 body over the 16-byte-aligned prefix (all three pointers share the
    // alignment when n4 > 0), scalar tail
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                       reinterpret_cast<uintptr_t>(grad)) & 15) == 0;
    const long long n4 = vec ? n / 4 : 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const float s2 = 2.f * scale;
    float s = 0.f;
    for (long long i = t0; i < n4; i += stride) {
        const float4 a = reinterpret_cast<const float4*>(x)[i];
        const float4 b = reinterpret_cast<const float4*>(y)[i];
        const float4 d = make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
        reinterpret_cast<float4*>(grad)[i] = make_float4(s2 * d.x, s2 * d.y, s2 * d.z, s2 * d.w);
        s += d.x * d.x + d.y * d.y + d.z * d.z + d.w * d.w;
    }
    for (long long i = 4 * n4 + t0; i < n; i += stride) {
        const float d = x[i] - y[i];
        grad[i] = s2 * d;
        s += d * d;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0 && s != 0.f) atomicAdd(loss, scale * s);
}
}  // namespace

void launch_backward(const BackwardArgs& a, int max_tiles, long long max_rendered, cudaStream_t st)
{
    if (a.n_views == 0) return;
    if (max_tiles) {
        const dim3 grid(max_tiles, a.n_views);
        if (a.has_depth_cot && a.has_T_cot) k_raster_bwd<true, true><<<grid, RT, 0, st>>>(a);
        else if (a.has_depth_cot) k_raster_bwd<true, false><<<grid, RT, 0, st>>>(a);
        else if (a.has_T_cot) k_raster_bwd<false, true><<<grid, RT, 0, st>>>(a);
        else k_raster_bwd<false, false><<<grid, RT, 0, st>>>(a);
    }
    if (max_rendered) {
        const size_t smem = a.g_table && a.smem_table ? (size_t)a.num_instances * 48 : 0;
        k_project_bwd<<<dim3((unsigned)((max_rendered + 255) / 256), a.n_views), 256, smem, st>>>(a);
    }
}

void launch_mse(const float* x, const float* y, long long n, float scale, float* grad,
                float* loss, cudaStream_t st)
{
    if (n == 0) return;
    const long long blocks = std::min<long long>((n / 4 + 255) / 256 + 1, 148ll * 8);
    k_mse<<<(unsigned)blocks, 256, 0, st>>>(x, y, n, scale, grad, loss);
}

}  // namespace s3r
