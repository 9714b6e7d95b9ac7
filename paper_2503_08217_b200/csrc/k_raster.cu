// k_raster.cu — K7 alpha-blended tile rasterizer (+ debug dump of the depth
// order).
//
// K7 implements Eq.2: C = sum_i c_i alpha_i prod_{j<i}
// (1 - alpha_j), front to back over the Gaussians of the pixel's 16x16 tile in
// (depth, index) order, with the readings R12-R15 of DESIGN.md: the Gaussians
// of a tile are those whose tile rectangle contains it; integer pixel centres;
// alpha = min(0.99, o exp(power)), power = min(0, -1/2 d^T Sigma^-1 d);
// include-then-stop at T < 1e-4; black background; depth = sum w z.  The
// exponential is R-ARITH's exp2 form (bit-identical to the oracle's f32
// contract).
//
// Layout: one 64-thread CTA per (view, tile); each thread owns 4 pixels of one
// column (rows ly, ly+4, ly+8, ly+12), so the per-splat dx terms and the
// shared-memory record loads are amortised over 4 pixel evaluations.  The CTA
// walks its tile's depth-ordered list of ranks (k_bin.cu) and stages 256 of
// the 48-byte records at a time in shared memory; every pixel then blends the
// batch.  A pixel stops at its termination; the CTA stops when all its pixels
// have (__syncthreads_count).
#include <algorithm>
#include <type_traits>

#include "s3r_internal.cuh"

namespace s3r {

namespace {

// R-ARITH s3r_exp2 for -24 <= x <= 0 (the caller handles the flush x < -24 -> 0),
// evaluated on pixel pairs, times the opacity, by o_exp2_x2 below: n = rint(x)
// by the 1.5*2^23 shifter (full-rate FADDs, no F2I/FRND), r = x - n exact, 2^r
// as 1 + r P(r) with the degree-4 P of DESIGN.md R-ARITH, times 2^n built from
// the shifter's bits: bits(t) = 0x4B400000 + n, so bits(t) << 23 == n << 23.
// c0 = 1.3264695880934596e-3f (the leading coefficient of P) is passed in a
// register (see k_raster).

#ifndef S3R_RASTER_RPIX
#define S3R_RASTER_RPIX 4
#endif
// pixels per thread (RPIX rows of one column, RS rows apart); a CTA covers TH
// rows of its tile (the whole tile, or one half: blockIdx.z), TILE * TH / RPIX
// threads, each warp owning BW columns.  The product layout is RPIX = 4, TH =
// 16 (2 packed pairs per thread, 64-thread CTAs); a batch whose grid cannot fill
// the GPU (C1: 16 tiles) takes RPIX = 2, TH = 8 (one pair per thread, two
// 64-thread CTAs per tile): four times the warps on twice the SMs.
template <int RP, int TH = TILE>
struct Geo {
    static constexpr int RPIX = RP;
    static constexpr int RT = TILE * TH / RPIX;
    static constexpr int BW = TILE / (RT / 32);
    static constexpr int RS = 32 / BW;
    static constexpr int NP = RPIX / 2;
    static constexpr int NW = RT / 32;   // warps (= pixel blocks) per tile CTA
};
constexpr int RPIX_BIG = S3R_RASTER_RPIX;
#ifndef S3R_RASTER_ADJ
#define S3R_RASTER_ADJ 1     // vertically adjacent pixel pairs (A/B: 14.65 vs 15.01 ms)
#endif
#ifndef S3R_RASTER_ALUEXP
#define S3R_RASTER_ALUEXP 0  // 1: o 2^n exponent add as a funnel shift (ALU pipe) instead of IMAD
#endif
#ifndef S3R_RASTER_UVOTE
#define S3R_RASTER_UVOTE 0   // 1: warp-uniform skip of a pixel pair (vote) instead of a divergent branch
#endif
#ifndef S3R_RASTER_FASTLIVE
#define S3R_RASTER_FASTLIVE 1   // no per-pixel liveness test while every pixel of the warp is live (A/B, C3: training forward 19.2 -> 17.6 ms; render neutral)
#endif
#ifndef S3R_RASTER_STAGE
#define S3R_RASTER_STAGE 1   // record staging: 0 LDG+STS, 1 cp.async (A/B: 14.55 vs 14.57 ms), 2 cp.async double-buffered at 128 records (15.20 ms)
#endif
#ifndef S3R_RASTER_RB
#define S3R_RASTER_RB (S3R_RASTER_STAGE == 2 ? 128 : 256)
#endif
constexpr int RB = S3R_RASTER_RB;   // records staged per batch (per buffer)
constexpr int NBUF = S3R_RASTER_STAGE == 2 ? 2 : 1;

// Build-time variants (for A/B measurement; the defaults are the product):
//   S3R_RASTER_MINB   minimum resident CTAs per SM for __launch_bounds__ (0: none)
// Measured and removed: the per-record cull test in the blend
// loop instead of per-warp compacted lists, per-pair-block masks, a vote every
// 2 / 4 records, the branch-free pair, a persistent grid.
#ifndef S3R_RASTER_MINB
#define S3R_RASTER_MINB 16    // 64 registers, 32 resident warps per SM (A/B: 16.6 vs 17.2 ms)
#endif
#ifndef S3R_RASTER_TRAIN_MINB
#define S3R_RASTER_TRAIN_MINB S3R_RASTER_MINB   // the training forward's bound
#endif
#ifndef S3R_FLUSH_E2
#define S3R_FLUSH_E2 FLUSH_E2
#endif

// Packed pairs: sm_100a executes two fp32 operations per instruction
// (FADD2 / FMUL2 / FFMA2, __fadd2_rn / __fmul2_rn / __ffma2_rn), each component
// rounded exactly like the scalar __fadd_rn / __fmul_rn / __fmaf_rn.  A thread's
// 4 pixels are blended as 2 pairs (rows k, k+4 | k+8, k+12), which halves the
// issue slots of the FP32 work while the result stays bit-identical to the
// scalar R-ARITH sequence.
__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 neg2(float2 x) { return make_float2(-x.x, -x.y); }

// s3r_exp2 on a pair (same operations as s3r_exp2, component-wise)
// o * s3r_exp2(x) on a pair, as y * (o 2^n): o 2^n is exact (an exponent add on
// o's bits, no under/overflow for o in (0, 1], n in [-24, 0]), so the one
// rounding is that of the exact product o y 2^n — bit-identical to
// o * (y * 2^n), one multiply less
__device__ __forceinline__ float2 o_exp2_x2(float2 x, float o, float c0)
{
    const float2 t = __fadd2_rn(x, f2(12582912.0f));
    const float2 n = __fadd2_rn(t, f2(-12582912.0f));
    const float2 r = __fadd2_rn(x, neg2(n));
    float2 p = __ffma2_rn(f2(c0), r, f2(9.671507403254509e-3f));
    p = __ffma2_rn(p, r, f2(5.550733208656311e-2f));
    p = __ffma2_rn(p, r, f2(2.4022243916988373e-1f));
    p = __ffma2_rn(p, r, f2(6.931470036506653e-1f));
    const float2 y = __ffma2_rn(p, r, f2(1.0f));
    // bits(t) << 23 == n << 23 (mod 2^32): the shifter's 0x4B400000 part shifts out
    const uint32_t ob = __float_as_uint(o);
#if S3R_RASTER_ALUEXP
    // as a funnel shift (LEA.HI / SHF on the ALU pipe) instead of the IMAD that
    // ptxas otherwise picks, which issues to the saturated FMA pipe
    const float2 osc = make_float2(
        __uint_as_float(ob + __funnelshift_l(0u, __float_as_uint(t.x), 23)),
        __uint_as_float(ob + __funnelshift_l(0u, __float_as_uint(t.y), 23)));
#else
    const float2 osc = make_float2(__uint_as_float(ob + (__float_as_uint(t.x) << 23)),
                                   __uint_as_float(ob + (__float_as_uint(t.y) << 23)));
#endif
    return __fmul2_rn(y, osc);
}

// Fast-exponential mode (s3r_set_fast_exp): 2^x from the SFU's ex2.approx.ftz
// (MUFU.EX2, <= 2 ulp) instead of the R-ARITH polynomial.  The MUFU pipe runs
// beside the FP32 pipe, so the 8 FP32 instructions per pair of the polynomial
// leave the blend's bottleneck (A/B, C3: raster 11.9 vs 14.6 ms).  Not
// bit-exact with the oracle (R24).
__device__ __forceinline__ float ex2_sfu(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// cp.async of one 16-byte chunk global -> shared (L2 only: the records are
// re-read by the other tiles of the splat, not by this SM)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem)
{
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One (view, tile): the whole K7 computation of the tile's 256 pixels.
template <bool COUNT, bool TRAIN, bool FAST, int RP, int TH>
__device__ __forceinline__ void raster_tile(const RasterArgs& a, const int v, const int tile,
                                            const int half)
{
    using G = Geo<RP, TH>;
    constexpr int RPIX = G::RPIX, RT = G::RT, BW = G::BW, RS = G::RS, NP = G::NP, NW = G::NW;
    __shared__ float4 s_rec[NBUF][3 * RB];   // staged splat records, 48 B each
    __shared__ uint16_t s_cl[NW][RB];        // per warp block: staged records reaching it
    __shared__ int s_wc[NW][NW];             // [staging warp][warp block] kept counts
    const DevView& V = a.views[v];
    if (tile >= V.ntiles) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tx = tile % V.TX, ty = tile / V.TX;
    // warp w owns columns BW w .. BW w + BW - 1; for pixel k a warp covers a
    // compact BW x RS block (rows RS k .. RS k + RS - 1)
    const int px = tx * TILE + (tid >> 5) * BW + (lane % BW);
#if S3R_RASTER_ADJ
    // pixel k of the thread at row 2 RS (k >> 1) + 2 (lane / BW) + (k & 1): the
    // two pixels of a pair are vertically adjacent
    auto prow = [&](int k) {
        return ty * TILE + half * TH + 2 * RS * (k >> 1) + 2 * (lane / BW) + (k & 1);
    };
#else
    const int py0 = ty * TILE + half * TH + (lane / BW);
    auto prow = [&](int k) { return py0 + RS * k; };
#endif
    const float fpx = (float)px;
    // centre of the warp's BW x 16 pixel block (flush-ellipse culling; the
    // stored extents include the 8 x 16 block's half size)
    // (the stored extents include an 8 x 16 block's half size; XPAD corrects
    // for another block width, negative for BW < 8)
    static_assert(BW >= 1 && RS * 2 * NP == TH, "warp blocks span the CTA's TH rows");
    constexpr float XPAD = 0.5f * (BW - 1) - CULL_HALF_BX;
    // YPAD: the same correction for a block of TH < 16 rows (still conservative:
    // the stored extent minus 4 keeps the 3.5-row half height of 8 rows)
    constexpr float YPAD = 0.5f * (TH - 1) - CULL_HALF_BY;
    const float bcx0 = (float)(tx * TILE) + 0.5f * (BW - 1);     // warp block 0
    const float bcy = (float)(ty * TILE + half * TH) + 0.5f * (TH - 1);
    // pair P holds pixels k = 2P (.x) and 2P + 1 (.y)
    float2 nfpy[NP], T[NP], cr[NP], cg[NP], cb[NP], dp[NP];
    int stop[RPIX];
    int nlive = 0;                     // pixels of this thread still blending
    unsigned inside = 0;
#pragma unroll
    for (int k = 0; k < RPIX; ++k) {
        const int py = prow(k);
        stop[k] = -1;
        const bool in = px < V.W && py < V.H;
        inside |= (in ? 1u : 0u) << k;
        nlive += in ? 1 : 0;
    }
#pragma unroll
    for (int P = 0; P < NP; ++P) {
        nfpy[P] = make_float2(-(float)prow(2 * P), -(float)prow(2 * P + 1));
        // a pixel outside the image starts "terminated" (T = 0 is never written)
        T[P] = make_float2((inside >> (2 * P)) & 1 ? 1.0f : 0.0f,
                           (inside >> (2 * P + 1)) & 1 ? 1.0f : 0.0f);
        cr[P] = cg[P] = cb[P] = dp[P] = f2(0.0f);
    }
#if S3R_RASTER_FASTLIVE
    // every pixel of the warp live (warp-uniform): the blend skips the per-pixel
    // T >= 1e-4 tests until the first termination in the warp
    bool all_live = __all_sync(0xffffffffu, inside == (1u << RPIX) - 1u);
#endif
    const int2 rg = a.tranges[V.trange_off + tile];
    const uint32_t* lst = a.tlists + V.tlist_off;
    const float4* recs = a.rec_sorted + 3 * V.cap_off;
    // first Horner coefficient of s3r_exp2 (1.3264695880934596e-3f), a kernel
    // argument so it stays in a register (an immediate is re-materialised per use)
    const float c0 = a.exp2_c0;

    // one record (staged slot j of buffer `buf`, tile-list entry tpos + j) for the
    // thread's 4 pixels; LIVE: test each pixel's T >= 1e-4 (else all are live)
    auto blend = [&](const float4* sr, const int tj, auto live_tag) {
        constexpr bool LIVE = decltype(live_tag)::value;
        const float4 q0 = sr[0];   // mx, my, z, o
        const float4 q1 = sr[1];   // qa, qb, qc, flush half extent x
        const float4 q2 = sr[2];   // r, g, b, flush half extent y
        // e2 = log2(e) * power = qa dx^2 + qb dx dy + qc dy^2 (R-ARITH exp2
        // form); the dx terms are shared by the thread's 4 pixels
        const float dx = q0.x - fpx;
        const float a1 = q1.x * dx;
        const float a2 = a1 * dx;
        const float b1 = q1.y * dx;
#pragma unroll
        for (int P = 0; P < NP; ++P) {
            const float2 dy = __fadd2_rn(f2(q0.y), nfpy[P]);
            const float2 c1 = __ffma2_rn(f2(q1.z), dy, f2(b1));
            const float2 e2r = __ffma2_rn(dy, c1, f2(a2));
            // A dead pixel (T < 1e-4) or a flushed exp2 (e2 < -24, s3r_exp2 = 0)
            // has alpha = 0, which leaves C, D and T bit-identical
            // (fma(c, 0, C) == C, T - 0 == T): such evaluations are skipped
            // (both of the pair) or get alpha = 0 (one of the pair).
            const bool livx = !LIVE || T[P].x >= 1e-4f, livy = !LIVE || T[P].y >= 1e-4f;
            // the flush test min(0, e2) >= F is !(e2 < F) for F < 0 (a NaN
            // passes, as fminf(0, NaN) = 0 does), so the clamp min(0, e2) is
            // taken inside the branch only (A/B, C3: raster 14.66 vs 14.72 ms)
            const bool onx = !(e2r.x < S3R_FLUSH_E2) && livx;
            const bool ony = !(e2r.y < S3R_FLUSH_E2) && livy;
            if (TRAIN && !COUNT) {
                // the backward's per-pixel bound: the last entry the pixel
                // was live at (its terminating one, or a later entry that
                // is flushed for it anyway), one select per pixel
                stop[2 * P] = livx ? tj : stop[2 * P];
                stop[2 * P + 1] = livy ? tj : stop[2 * P + 1];
            }
#if S3R_RASTER_UVOTE
            if (__any_sync(0xffffffffu, onx || ony)) {
#else
            if (onx || ony) {
#endif
                const float2 e2 = make_float2(fminf(0.0f, e2r.x), fminf(0.0f, e2r.y));
                const float2 og = FAST
                    ? __fmul2_rn(make_float2(ex2_sfu(e2.x), ex2_sfu(e2.y)), f2(q0.w))
                    : o_exp2_x2(e2, q0.w, c0);
                const float2 alpha = make_float2(onx ? fminf(0.99f, og.x) : 0.0f,
                                                 ony ? fminf(0.99f, og.y) : 0.0f);
                const float2 w = __fmul2_rn(alpha, T[P]);
                cr[P] = __ffma2_rn(f2(q2.x), w, cr[P]);
                cg[P] = __ffma2_rn(f2(q2.y), w, cg[P]);
                cb[P] = __ffma2_rn(f2(q2.z), w, cb[P]);
                dp[P] = __ffma2_rn(f2(q0.z), w, dp[P]);
                const float2 Tn = __fadd2_rn(T[P], neg2(w));
                // include-then-stop (R14): the pixel is dead once T < 1e-4
                if (COUNT) {
                    if (onx && Tn.x < 1e-4f) stop[2 * P] = tj + 1;
                    if (ony && Tn.y < 1e-4f) stop[2 * P + 1] = tj + 1;
                }
                T[P] = Tn;
            }
        }
    };
    auto tmax_of = [&]() {
        float m = fmaxf(T[0].x, T[0].y);
#pragma unroll
        for (int P = 1; P < NP; ++P) m = fmaxf(m, fmaxf(T[P].x, T[P].y));
        return m;
    };

    // stage records [c, c + n) of the tile list into buffer b (16-byte pieces)
    auto stage = [&](int b, int c, int n) {
        for (int i = tid; i < n; i += RT) {
            const float4* src = recs + 3ll * lst[c + i];
#if S3R_RASTER_STAGE == 0
            const float4 q0 = src[0], q1 = src[1], q2 = src[2];
            s_rec[b][3 * i + 0] = q0;
            s_rec[b][3 * i + 1] = q1;
            s_rec[b][3 * i + 2] = q2;
#else
            cp_async16(&s_rec[b][3 * i + 0], src + 0);
            cp_async16(&s_rec[b][3 * i + 1], src + 1);
            cp_async16(&s_rec[b][3 * i + 2], src + 2);
#endif
        }
#if S3R_RASTER_STAGE != 0
        cp_async_commit();
#endif
    };

    int cur = rg.x;                    // cursor in the tile list (uniform)
    int tpos = 0;                      // tile-list entries consumed so far (uniform)
    uint32_t n_exec = 0;
    int buf = 0;
#if S3R_RASTER_STAGE == 2
    if (cur < rg.y) stage(0, cur, min(RB, rg.y - cur));
#endif
    while (cur < rg.y) {
        if (__syncthreads_count(nlive) == 0) break;
        const int nb = min(RB, rg.y - cur);
#if S3R_RASTER_STAGE == 2
        // the next batch streams into the other buffer while this one blends
        // (the barrier above ended every warp's use of that buffer)
        if (cur + nb < rg.y) stage(buf ^ 1, cur + nb, min(RB, rg.y - cur - nb));
        else cp_async_commit();              // empty group: wait_group 1 stays uniform
        cp_async_wait<1>();
        __syncthreads();
#elif S3R_RASTER_STAGE == 1
        stage(0, cur, nb);
        cp_async_wait<0>();
        __syncthreads();
#endif
        // ---- the staged batch's per-warp-block lists: the order-preserving
        // list of the records whose flush ellipse reaches the block (the others
        // have alpha = 0 on every pixel of the block, s3r_internal.cuh
        // flush_extent): ballot + popc inside each staging warp, warps in order
        int run[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) run[w] = 0;
        for (int base = 0; base < nb; base += RT) {
            const int i = base + tid;
            bool keep[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) keep[w] = false;
            if (i < nb) {
#if S3R_RASTER_STAGE == 0
                const float4* src = recs + 3ll * lst[cur + i];
                const float4 q0 = src[0], q1 = src[1], q2 = src[2];
                s_rec[0][3 * i + 0] = q0;
                s_rec[0][3 * i + 1] = q1;
                s_rec[0][3 * i + 2] = q2;
#else
                const float4 q0 = s_rec[buf][3 * i + 0], q1 = s_rec[buf][3 * i + 1],
                             q2 = s_rec[buf][3 * i + 2];
#endif
                const float hx = XPAD != 0.0f ? q1.w + XPAD : q1.w;
                const bool yok = !(fabsf(q0.y - bcy) > (YPAD != 0.0f ? q2.w + YPAD : q2.w));
#pragma unroll
                for (int w = 0; w < NW; ++w)
                    keep[w] = yok && !(fabsf(q0.x - (bcx0 + (float)(w * BW))) > hx);
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
                if (keep[w]) s_cl[w][off + __popc(bal[w] & ((1u << lane) - 1u))] = (uint16_t)i;
                run[w] += tot;
            }
            __syncthreads();
        }
        const int nk = run[warp];
        cur += nb;
        n_exec += nb;
        const float4* sb = s_rec[buf];
        // the blend loop is warp-uniform (every lane runs it while any lane of
        // its warp is live) so that the votes below see the full warp
        if (__any_sync(0xffffffffu, nlive != 0)) {
            int jj = 0;
#if S3R_RASTER_FASTLIVE
            if (all_live) {
                for (; jj < nk; ++jj) {
                    const int j = s_cl[warp][jj];
                    blend(sb + 3 * j, tpos + j, std::false_type{});
                    float m = fminf(T[0].x, T[0].y);
#pragma unroll
                    for (int P = 1; P < NP; ++P) m = fminf(m, fminf(T[P].x, T[P].y));
                    if (__any_sync(0xffffffffu, m < 1e-4f)) {   // a pixel of the warp died
                        all_live = false;
                        ++jj;
                        nlive = tmax_of() >= 1e-4f ? 1 : 0;
                        if (!__any_sync(0xffffffffu, nlive != 0)) jj = nk;
                        break;
                    }
                }
            }
#endif
            for (; jj < nk; ++jj) {
                const int j = s_cl[warp][jj];
                blend(sb + 3 * j, tpos + j, std::true_type{});
                nlive = tmax_of() >= 1e-4f ? 1 : 0;
                if (!__any_sync(0xffffffffu, nlive != 0)) break;   // whole warp done
            }
        }
        tpos += nb;
#if S3R_RASTER_STAGE == 2
        buf ^= 1;
#endif
    }
#if S3R_RASTER_STAGE == 2
    cp_async_wait<0>();                   // nothing in flight when the CTA exits
#endif
    if (COUNT) {
        // E_alg = sum over pixels of the tile-list entries examined up to and
        // including the terminating one; E_exec = 256 x entries the CTA staged
        unsigned long long e = 0;
#pragma unroll
        for (int k = 0; k < RPIX; ++k)
            if (inside & (1u << k)) e += (unsigned long long)(stop[k] >= 0 ? stop[k] : tpos);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_down_sync(0xffffffffu, e, o);
        if (lane == 0) atomicAdd(a.evals + 2 * v, e);
        if (tid == 0) atomicAdd(a.evals + 2 * v + 1, (unsigned long long)(TILE * TH) * n_exec);
    }
#pragma unroll
    for (int k = 0; k < RPIX; ++k) {
        if (!(inside & (1u << k))) continue;
        const int P = k >> 1;
        const bool hi = k & 1;
        const long long pix = (long long)prow(k) * V.W + px;
        float* o = V.rgb + 3 * pix;
        o[0] = hi ? cr[P].y : cr[P].x;
        o[1] = hi ? cg[P].y : cg[P].x;
        o[2] = hi ? cb[P].y : cb[P].x;
        const float Tk = hi ? T[P].y : T[P].x;
        if (V.depth) V.depth[pix] = hi ? dp[P].y : dp[P].x;
        if (V.finalT) V.finalT[pix] = Tk;
        if (TRAIN) {      // state the backward (k_raster_bwd) starts from
            a.train_T[V.pix_off + pix] = Tk;
            // entries the backward differentiates: [0, train_n).  With COUNT the
            // terminating entry + 1 (else every entry); otherwise the last live
            // entry + 1 — the same derivative, since the entries between them are
            // flushed for the pixel (culled from its warp's list)
            a.train_n[V.pix_off + pix] = COUNT ? (stop[k] >= 0 ? stop[k] : tpos) : stop[k] + 1;
        }
    }
}

// K7: one CTA per (tile, view)
template <bool COUNT, bool TRAIN, bool FAST, int RP, int TH>
__global__ void __launch_bounds__(Geo<RP, TH>::RT,
                                  RP == RPIX_BIG ? (TRAIN ? S3R_RASTER_TRAIN_MINB : S3R_RASTER_MINB) : 8)
    k_raster(RasterArgs a)
{
    raster_tile<COUNT, TRAIN, FAST, RP, TH>(a, blockIdx.y, blockIdx.x, blockIdx.z);
}

template <int RP, int TH>
void launch_raster_rp(const RasterArgs& a, dim3 grid, cudaStream_t st)
{
    constexpr int RT = Geo<RP, TH>::RT;
    grid.z = TILE / TH;
    // training renders always take the exact R-ARITH exponential: the backward
    // recomputes alpha with it and relies on the forward's decisions
    if (a.train_T) {
        if (a.evals) k_raster<true, true, false, RP, TH><<<grid, RT, 0, st>>>(a);
        else k_raster<false, true, false, RP, TH><<<grid, RT, 0, st>>>(a);
    } else if (a.fast_exp) {
        if (a.evals) k_raster<true, false, true, RP, TH><<<grid, RT, 0, st>>>(a);
        else k_raster<false, false, true, RP, TH><<<grid, RT, 0, st>>>(a);
    } else {
        if (a.evals) k_raster<true, false, false, RP, TH><<<grid, RT, 0, st>>>(a);
        else k_raster<false, false, false, RP, TH><<<grid, RT, 0, st>>>(a);
    }
}

// ------------------------------------------------------------------ dumps
__global__ void k_dump_order(const uint32_t* __restrict__ order, const int32_t* __restrict__ gidx,
                             long long base, long long count, int32_t* __restrict__ out)
{
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r < count) out[r] = gidx[base + order[base + r]];
}
}  // namespace

void launch_raster(const RasterArgs& args, cudaStream_t st)
{
    if (args.max_tiles == 0 || args.n_views == 0) return;
    RasterArgs a = args;
    a.exp2_c0 = 1.3264695880934596e-3f;
    const dim3 grid(a.max_tiles, a.n_views);
#ifndef S3R_RASTER_SMALL_TH
#define S3R_RASTER_SMALL_TH 8   // rows per CTA on a grid that cannot fill the GPU (16: whole tiles)
#endif
    if ((long long)a.max_tiles * a.n_views < 2 * 148) launch_raster_rp<2, S3R_RASTER_SMALL_TH>(a, grid, st);
    else launch_raster_rp<RPIX_BIG, TILE>(a, grid, st);
}

void launch_dump_order(const uint32_t* order, const int32_t* gidx, long long base,
                       long long count, int32_t* out, cudaStream_t st)
{
    if (count == 0) return;
    k_dump_order<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(order, gidx, base, count, out);
}

}  // namespace s3r
