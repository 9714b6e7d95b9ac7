// k_raster.cu — K3/K4 depth-ordered permute + tile-count scan + key emission,
// K6 tile ranges, K7 alpha-blended tile rasterizer, debug dumps.
//
// K7 implements Eq.2: C = sum_i c_i alpha_i prod_{j<i}
// (1 - alpha_j), front to back over the Gaussians of the pixel's 16x16 tile in
// (depth, index) order, with the readings R13-R15 of DESIGN.md: integer pixel
// centres, alpha = min(0.99, o exp(power)), power = min(0, -1/2 d^T Sigma^-1 d),
// include-then-stop at T < 1e-4, black background, depth = sum w z.  exp is the
// s3r_exp of R-ARITH (bit-identical to the oracle's).
//
// K7 layout: one 64-thread CTA per (view, tile); each thread owns 4 pixels of
// one column (rows ly, ly+4, ly+8, ly+12), so the per-splat dx terms and the
// shared-memory record loads are amortised over 4 pixel evaluations.  The
// tile's sorted pair list is consumed in batches of 256 records (48 B each,
// 16-byte loads from the depth-sorted record array) staged in shared memory.
// A pixel stops at its termination; the CTA stops when all its pixels have
// (__syncthreads_count).
#include "s3r_internal.cuh"

namespace s3r {

namespace {
constexpr int ET = 256;
constexpr int EITEMS = 4;
constexpr int ETILE = ET * EITEMS;


__device__ __forceinline__ int find_seg(const int* seg_tile0, int nsegs, int gt)
{
    int lo = 0, hi = nsegs - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (seg_tile0[mid] <= gt) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ------------------------------------------------------------------ K3/K4
__global__ void __launch_bounds__(ET) k_emit(EmitArgs a)
{
    __shared__ int s_gt, s_sg;
    __shared__ uint32_t s_off[ETILE + 1];
    __shared__ uint32_t s_rx[ETILE], s_ry[ETILE];
    __shared__ uint32_t s_warp[ET / 32];
    __shared__ uint32_t s_base;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        const int gt = atomicAdd(a.ticket, 1);
        s_gt = gt;
        s_sg = find_seg(a.seg_tile0, a.nsegs, gt);
    }
    __syncthreads();
    const int gt = s_gt, sg = s_sg;
    const Seg S = a.segs[sg];
    const DevView& V = a.views[sg];
    const int ltile = gt - a.seg_tile0[sg];
    const long long r0 = (long long)ltile * ETILE + tid * EITEMS;

    uint32_t n[EITEMS];
    uint32_t tot = 0;
#pragma unroll
    for (int k = 0; k < EITEMS; ++k) {
        const long long r = r0 + k;
        n[k] = 0;
        s_rx[tid * EITEMS + k] = 0;
        s_ry[tid * EITEMS + k] = 0;
        if (r < S.count) {
            const uint32_t j = a.order[S.base + r];
            const float4* src = a.rec + 3 * (S.base + j);
            const float4 q0 = src[0], q1 = src[1], q2 = src[2];
            float4* dst = a.rec_sorted + 3 * (S.base + r);
            dst[0] = q0; dst[1] = q1; dst[2] = q2;
            const uint32_t rx = __float_as_uint(q1.w), ry = __float_as_uint(q2.w);
            s_rx[tid * EITEMS + k] = rx;
            s_ry[tid * EITEMS + k] = ry;
            n[k] = ((rx >> 16) - (rx & 0xffff) + 1) * ((ry >> 16) - (ry & 0xffff) + 1);
        }
        tot += n[k];
    }
    // block exclusive scan of the per-thread totals
    uint32_t v = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_warp[warp] = v;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < ET / 32 ? s_warp[lane] : 0;
        uint32_t ww = w;
#pragma unroll
        for (int o = 1; o < ET / 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, ww, o);
            if (lane >= o) ww += y;
        }
        if (lane < ET / 32) s_warp[lane] = ww - w;
        const uint32_t agg = __shfl_sync(0xffffffffu, ww, ET / 32 - 1);
        // decoupled look-back over the view's preceding CTAs (warp-cooperative)
        uint32_t* lb = a.lookback;
        if (lane == 0) lb_publish(lb + gt, (ltile == 0 ? LB_PRE : LB_AGG) | agg);
        const uint32_t excl = (ltile == 0) ? 0u : warp_lookback(lb, 1, gt, gt - ltile);
        if (lane == 0) {
            if (ltile != 0) lb_publish(lb + gt, LB_PRE | (excl + agg));
            s_base = excl;
            s_off[ETILE] = agg;
        }
    }
    __syncthreads();
    uint32_t off = v - tot + s_warp[warp];
#pragma unroll
    for (int k = 0; k < EITEMS; ++k) {
        s_off[tid * EITEMS + k] = off;
        off += n[k];
    }
    __syncthreads();
    const uint32_t total = s_off[ETILE];
    unsigned long long* out = a.pairs + V.pair_off + s_base;
    const int TX = V.TX;
    // load-balanced emission: pair p of this CTA belongs to the last item whose
    // exclusive offset is <= p; tiles of an item in row-major order
    for (uint32_t p = tid; p < total; p += ET) {
        int lo = 0, hi = ETILE - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_off[mid] <= p) lo = mid; else hi = mid - 1;
        }
        const uint32_t m = p - s_off[lo];
        const uint32_t rx = s_rx[lo], ry = s_ry[lo];
        const uint32_t w = (rx >> 16) - (rx & 0xffff) + 1;
        const uint32_t ty = (ry & 0xffff) + m / w, tx = (rx & 0xffff) + m % w;
        const uint32_t tile = ty * (uint32_t)TX + tx;
        const uint32_t r = (uint32_t)(ltile * ETILE + lo);
        out[p] = ((unsigned long long)tile << 32) | r;
    }
}

// ------------------------------------------------------------------ K6
__global__ void k_ranges(const unsigned long long* __restrict__ pairs, long long total,
                         const long long* __restrict__ view_pair_off, int n_views,
                         const int* __restrict__ range_off, int2* __restrict__ ranges)
{
    const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= total) return;
    int lo = 0, hi = n_views - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (view_pair_off[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const long long b = view_pair_off[lo], e = view_pair_off[lo + 1];
    const uint32_t tile = (uint32_t)(pairs[p] >> 32);
    int2* R = ranges + range_off[lo];
    const int lp = (int)(p - b);
    if (p == b || (uint32_t)(pairs[p - 1] >> 32) != tile) R[tile].x = lp;
    if (p == e - 1 || (uint32_t)(pairs[p + 1] >> 32) != tile) R[tile].y = lp + 1;
}

// ------------------------------------------------------------------ K7
// R-ARITH s3r_exp2 for -44 <= x <= 0 (the caller handles x < -44 -> 0):
// n = rint(x) by the 1.5*2^23 shifter (all full-rate FADDs, no F2I/FRND),
// r = x - n exact, 2^r by the Cephes exp2f polynomial, times 2^n built from
// the shifter's bits: bits(t) = 0x4B400000 + n, so (bits(t) << 23) +
// 0x3F800000 = bits(2^n).
// c0 = 1.535336188319500e-4f is passed in a register (see k_raster).
__device__ __forceinline__ float s3r_exp2(float x, float c0)
{
    const float t = x + 12582912.0f;
    const float n = t - 12582912.0f;
    const float r = x - n;
    float p = __fmaf_rn(c0, r, 1.339887440266574e-3f);
    p = __fmaf_rn(p, r, 9.618437357674640e-3f);
    p = __fmaf_rn(p, r, 5.550332471162809e-2f);
    p = __fmaf_rn(p, r, 2.402264791363012e-1f);
    p = __fmaf_rn(p, r, 6.931472028550421e-1f);
    const float y = __fmaf_rn(p, r, 1.0f);
    return y * __uint_as_float((__float_as_uint(t) << 23) + 0x3F800000u);
}

constexpr int RT = 64;      // threads per tile CTA: 16 columns x 4 row groups
constexpr int RPIX = 4;     // pixels per thread: rows ly, ly+4, ly+8, ly+12 of one column
constexpr int RB = 256;     // splat records staged in shared memory per batch

template <bool COUNT>
__global__ void __launch_bounds__(RT) k_raster(RasterArgs a)
{
    __shared__ float4 s_rec[3 * RB];   // RB splat records, 48 B each
    const int v = blockIdx.y;
    const DevView& V = a.views[v];
    const int tile = blockIdx.x;
    if (tile >= V.ntiles) return;
    const int tid = threadIdx.x;
    const int tx = tile % V.TX, ty = tile / V.TX;
    const int px = tx * TILE + (tid & 15);
    const int py0 = ty * TILE + (tid >> 4);
    const float fpx = (float)px;
    float fpy[RPIX], T[RPIX], cr[RPIX], cg[RPIX], cb[RPIX], dp[RPIX];
    int stop[RPIX];
    int nlive = 0;                     // pixels of this thread still blending
    unsigned inside = 0;
#pragma unroll
    for (int k = 0; k < RPIX; ++k) {
        const int py = py0 + 4 * k;
        fpy[k] = (float)py;
        cr[k] = cg[k] = cb[k] = dp[k] = 0.0f;
        stop[k] = -1;
        const bool in = px < V.W && py < V.H;
        // a pixel outside the image starts "terminated" (T = 0 is never written)
        T[k] = in ? 1.0f : 0.0f;
        inside |= (in ? 1u : 0u) << k;
        nlive += in ? 1 : 0;
    }
    const int2 rg = a.ranges[a.range_off[v] + tile];
    const unsigned long long* pw = a.pairs + V.pair_off;
    const float4* recs = a.rec_sorted + 3 * V.cap_off;
    // first Horner coefficient of s3r_exp2 (1.535336188319500e-4f), a kernel
    // argument so it stays in a register (an immediate is re-materialised per use)
    const float c0 = a.exp2_c0;

    uint32_t n_exec = 0;
    for (int b = rg.x; b < rg.y; b += RB) {
        if (__syncthreads_count(nlive) == 0) break;
        const int nb = min(RB, rg.y - b);
        n_exec += nb;
        for (int i = tid; i < nb; i += RT) {
            const uint32_t r = (uint32_t)pw[b + i];
            const float4* src = recs + 3ll * r;
            s_rec[3 * i + 0] = src[0];
            s_rec[3 * i + 1] = src[1];
            s_rec[3 * i + 2] = src[2];
        }
        __syncthreads();
        if (nlive) {
            for (int j = 0; j < nb; ++j) {
                const float4* sr = s_rec + 3 * j;
                const float4 q0 = sr[0];   // mx, my, z, o
                const float4 q1 = sr[1];   // qa, qb, qc, rect
                const float4 q2 = sr[2];   // r, g, b, rect
                // e2 = log2(e) * power = qa dx^2 + qb dx dy + qc dy^2 (R-ARITH exp2
                // form); the dx terms are shared by the thread's 4 pixels
                const float dx = q0.x - fpx;
                const float a1 = q1.x * dx;
                const float a2 = a1 * dx;
                const float b1 = q1.y * dx;
#pragma unroll
                for (int k = 0; k < RPIX; ++k) {
                    const float dy = q0.y - fpy[k];
                    const float c1 = __fmaf_rn(q1.z, dy, b1);
                    const float e2 = fminf(0.0f, __fmaf_rn(dy, c1, a2));
                    // live pixel (T >= 1e-4) and a non-zero exp2 (s3r_exp2 flushes
                    // below -44: alpha = 0 would leave C, D and T bit-identical)
                    if (e2 >= -44.0f && T[k] >= 1e-4f) {
                        const float alpha = fminf(0.99f, q0.w * s3r_exp2(e2, c0));
                        const float w = alpha * T[k];
                        cr[k] = __fmaf_rn(q2.x, w, cr[k]);
                        cg[k] = __fmaf_rn(q2.y, w, cg[k]);
                        cb[k] = __fmaf_rn(q2.z, w, cb[k]);
                        dp[k] = __fmaf_rn(q0.z, w, dp[k]);
                        T[k] = T[k] - w;
                        // include-then-stop (R14): the pixel is dead once T < 1e-4
                        if (COUNT && T[k] < 1e-4f) stop[k] = b + j + 1;
                    }
                }
                const float tmax = fmaxf(fmaxf(T[0], T[1]), fmaxf(T[2], T[3]));
                if (tmax < 1e-4f) {
                    nlive = 0;
                    break;
                }
            }
        }
    }
    if (COUNT) {
        // E_alg = sum over pixels of the splats examined up to and including the
        // terminating one; E_exec = 256 x splats the CTA walked
        unsigned long long e = 0;
#pragma unroll
        for (int k = 0; k < RPIX; ++k)
            if (inside & (1u << k)) e += (unsigned long long)((stop[k] >= 0 ? stop[k] : rg.y) - rg.x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_down_sync(0xffffffffu, e, o);
        if ((tid & 31) == 0) atomicAdd(a.evals + 2 * v, e);
        if (tid == 0) atomicAdd(a.evals + 2 * v + 1, 256ull * n_exec);
    }
#pragma unroll
    for (int k = 0; k < RPIX; ++k) {
        if (!(inside & (1u << k))) continue;
        const long long pix = (long long)(py0 + 4 * k) * V.W + px;
        float* o = V.rgb + 3 * pix;
        o[0] = cr[k];
        o[1] = cg[k];
        o[2] = cb[k];
        if (V.depth) V.depth[pix] = dp[k];
        if (V.finalT) V.finalT[pix] = T[k];
    }
}

// ------------------------------------------------------------------ dumps
__global__ void k_dump_order(const uint32_t* __restrict__ order, const int32_t* __restrict__ gidx,
                             long long base, long long count, int32_t* __restrict__ out)
{
    const long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r < count) out[r] = gidx[base + order[base + r]];
}

__global__ void k_dump_pairs(const unsigned long long* __restrict__ pairs, long long count,
                             const uint32_t* __restrict__ order, const int32_t* __restrict__ gidx,
                             long long base, int32_t* __restrict__ tile_out,
                             int32_t* __restrict__ gauss_out)
{
    const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= count) return;
    const unsigned long long w = pairs[p];
    if (tile_out) tile_out[p] = (int32_t)(w >> 32);
    if (gauss_out) gauss_out[p] = gidx[base + order[base + (uint32_t)w]];
}
}  // namespace

int emit_tile() { return ETILE; }

void launch_emit(const EmitArgs& a, cudaStream_t st)
{
    if (a.total_tiles == 0) return;
    k_emit<<<a.total_tiles, ET, 0, st>>>(a);
}

void launch_ranges(const unsigned long long* pairs, long long total_pairs, const DevView* views,
                   int n_views, const long long* view_pair_off, const int* range_off, int2* ranges,
                   cudaStream_t st)
{
    (void)views;
    if (total_pairs == 0) return;
    k_ranges<<<(unsigned)((total_pairs + 255) / 256), 256, 0, st>>>(pairs, total_pairs,
                                                                     view_pair_off, n_views,
                                                                     range_off, ranges);
}

void launch_raster(const RasterArgs& args, cudaStream_t st)
{
    if (args.max_tiles == 0 || args.n_views == 0) return;
    RasterArgs a = args;
    a.exp2_c0 = 1.535336188319500e-4f;
    dim3 grid(a.max_tiles, a.n_views);
    if (a.evals) k_raster<true><<<grid, RT, 0, st>>>(a);
    else k_raster<false><<<grid, RT, 0, st>>>(a);
}

void launch_dump_order(const uint32_t* order, const int32_t* gidx, long long base,
                       long long count, int32_t* out, cudaStream_t st)
{
    if (count == 0) return;
    k_dump_order<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(order, gidx, base, count, out);
}

void launch_dump_pairs(const unsigned long long* pairs, long long count, const uint32_t* order,
                       const int32_t* gidx, long long base, int32_t* tile_out, int32_t* gauss_out,
                       cudaStream_t st)
{
    if (count == 0) return;
    k_dump_pairs<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(pairs, count, order, gidx, base,
                                                                   tile_out, gauss_out);
}

}  // namespace s3r
