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
// K7 layout: one CTA per (view, tile), one pixel per thread.  The tile's
// sorted pair list is consumed in batches of 256: each thread fetches one
// 48-byte splat record (3 x 16-byte loads from the depth-sorted record array)
// into shared memory; every pixel then walks the batch.  A pixel stops at its
// termination; the CTA stops when all 256 pixels have (__syncthreads_count).
#include "s3r_internal.cuh"

namespace s3r {

namespace {
constexpr int ET = 256;
constexpr int EITEMS = 4;
constexpr int ETILE = ET * EITEMS;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p)
{
    return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v)
{
    *reinterpret_cast<volatile uint32_t*>(p) = v;
}

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
        if (lane == 0) {
            uint32_t excl = 0;
            uint32_t* lb = a.lookback;
            if (ltile == 0) {
                st_volatile(lb + gt, LB_PRE | agg);
            } else {
                st_volatile(lb + gt, LB_AGG | agg);
                int j = gt - 1;
                while (true) {
                    const uint32_t w2 = ld_volatile(lb + j);
                    if ((w2 >> 30) == 0) continue;
                    excl += w2 & LB_MASK;
                    if (w2 & LB_PRE) break;
                    --j;
                }
                st_volatile(lb + gt, LB_PRE | (excl + agg));
            }
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
__device__ __forceinline__ float s3r_exp(float x)
{
    // R-ARITH software exponential (Cephes expf), x <= 0
    if (!(x >= -30.0f)) return 0.0f;
    const float n = rintf(x * 1.44269504f);
    float r = __fmaf_rn(-n, 0.693359375f, x);
    r = __fmaf_rn(-n, -2.12194440e-4f, r);
    float p = 1.9875691500e-4f;
    p = __fmaf_rn(p, r, 1.3981999507e-3f);
    p = __fmaf_rn(p, r, 8.3334519073e-3f);
    p = __fmaf_rn(p, r, 4.1665795894e-2f);
    p = __fmaf_rn(p, r, 1.6666665459e-1f);
    p = __fmaf_rn(p, r, 5.0000001201e-1f);
    const float r2 = r * r;
    float y = __fmaf_rn(p, r2, r);
    y = y + 1.0f;
    return y * __int_as_float((127 + (int)n) << 23);
}

__global__ void __launch_bounds__(256) k_raster(RasterArgs a)
{
    __shared__ float4 s0[256], s1[256], s2[256];
    const int v = blockIdx.y;
    const DevView& V = a.views[v];
    const int tile = blockIdx.x;
    if (tile >= V.ntiles) return;
    const int tid = threadIdx.x;
    const int tx = tile % V.TX, ty = tile / V.TX;
    const int px = tx * TILE + (tid & 15), py = ty * TILE + (tid >> 4);
    const bool inside = px < V.W && py < V.H;
    const float fpx = (float)px, fpy = (float)py;
    const int2 rg = a.ranges[a.range_off[v] + tile];
    const unsigned long long* pw = a.pairs + V.pair_off;
    const float4* recs = a.rec_sorted + 3 * V.cap_off;

    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f, dp = 0.0f;
    bool done = !inside;
    uint32_t n_eval = 0, n_exec = 0;    // work counters (only stored when a.evals)
    for (int b = rg.x; b < rg.y; b += 256) {
        if (__syncthreads_count(done) == 256) break;
        n_exec += min(256, rg.y - b);
        const int i = b + tid;
        if (i < rg.y) {
            const uint32_t r = (uint32_t)pw[i];
            const float4* src = recs + 3ll * r;
            s0[tid] = src[0];
            s1[tid] = src[1];
            s2[tid] = src[2];
        }
        __syncthreads();
        const int nb = min(256, rg.y - b);
        if (!done) {
            int j = 0;
            for (; j < nb; ++j) {
                const float4 q0 = s0[j];
                const float4 q1 = s1[j];
                const float dx = q0.x - fpx;
                const float dy = q0.y - fpy;
                const float t1 = dx * dx;
                const float t2 = dy * dy;
                const float t3 = dx * dy;
                const float sq = __fmaf_rn(q1.x, t1, q1.z * t2);
                const float power = fminf(0.0f, __fmaf_rn(-0.5f, sq, -(q1.y * t3)));
                // exp(power) == 0 below -30: alpha = 0 leaves C, D and T bit-identical
                if (!(power >= -30.0f)) continue;
                const float alpha = fminf(0.99f, q0.w * s3r_exp(power));
                const float w = alpha * T;
                const float4 q2 = s2[j];
                cr = __fmaf_rn(q2.x, w, cr);
                cg = __fmaf_rn(q2.y, w, cg);
                cb = __fmaf_rn(q2.z, w, cb);
                dp = __fmaf_rn(q0.z, w, dp);
                T = T * (1.0f - alpha);
                if (T < 1e-4f) {
                    done = true;
                    ++j;
                    break;
                }
            }
            n_eval += j;
        }
    }
    if (a.evals) {
        // E_alg = sum of per-pixel examined splats; E_exec = 256 x splats walked
        unsigned long long e = n_eval;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_down_sync(0xffffffffu, e, o);
        if ((tid & 31) == 0) atomicAdd(a.evals + 2 * v, e);
        if (tid == 0) atomicAdd(a.evals + 2 * v + 1, 256ull * n_exec);
    }
    if (inside) {
        const long long pix = (long long)py * V.W + px;
        float* o = V.rgb + 3 * pix;
        o[0] = cr;
        o[1] = cg;
        o[2] = cb;
        if (V.depth) V.depth[pix] = dp;
        if (V.finalT) V.finalT[pix] = T;
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

void launch_raster(const RasterArgs& a, cudaStream_t st)
{
    if (a.max_tiles == 0 || a.n_views == 0) return;
    dim3 grid(a.max_tiles, a.n_views);
    k_raster<<<grid, 256, 0, st>>>(a);
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
