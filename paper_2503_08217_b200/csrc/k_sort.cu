// k_sort.cu — K5: the depth sort of a batch: a segmented, stable LSD radix
// sort (onesweep with decoupled look-back) of 64-bit keys
// (bits(z) << gbits | Gaussian index) with the compacted slot as the value.
// z > near > 0, so the IEEE bit order of z is its numeric order, and the
// index bits make every key unique: the result is the (depth, index) order of
// reading R11 whatever order K2 compacted the records in.  8-bit digits,
// ceil((32 + gbits) / 8) passes (7 at C3's 2 M Gaussians).
// Segments are views: every view has its own digit histograms (k_hist, one
// read of the keys for all passes) and its own look-back chain, so one launch
// per pass sorts the whole batch.  seg_tile0[nsegs] = the batch's tiles; a grid
// larger than that (sized from a capacity, no host readback) is allowed.  Tile binning does not sort (k_bin.cu).
//
// Per pass each CTA takes a tile of 256*ITEMS keys (warp-striped, coalesced),
// ranks them with __match_any_sync per warp (stable: lane order within a
// round, rounds in order), scans the 256 digit counts across warps, publishes
// them to the look-back array, resolves its global digit offsets, stages the
// tile in shared memory in digit order and writes it out in coalesced runs.
// Algorithmic bytes per pass: (key + value) read + written once.
#include "s3r_internal.cuh"

namespace s3r {

namespace {
constexpr int ST = 256;
constexpr int SW = ST / 32;
#ifndef S3R_SORT_ITEMS
#define S3R_SORT_ITEMS 8
#endif
#ifndef S3R_SORT_MINB
#define S3R_SORT_MINB 4   // 64 registers, 4 CTAs/SM (A/B: depth sort 0.446 ms; 3 (80 regs): 0.481, none (96): 0.564)
#endif
constexpr int ITEMS64 = S3R_SORT_ITEMS;
constexpr int HITEMS = S3R_SORT_ITEMS;   // histogram tiles == onesweep tiles (ST * ITEMS keys)

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

// Block-wide exclusive scan of one value per thread (256 threads).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_warp)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_warp[warp] = v;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < SW ? s_warp[lane] : 0;
        uint32_t ww = w;
#pragma unroll
        for (int o = 1; o < SW; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, ww, o);
            if (lane >= o) ww += y;
        }
        if (lane < SW) s_warp[lane] = ww - w;
    }
    __syncthreads();
    return v - x + s_warp[warp];
}

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K key, int shift)
{
    return (uint32_t)(key >> shift) & (RADIX - 1);
}

// ------------------------------------------------------------------ hist
template <typename K>
__global__ void __launch_bounds__(ST) k_hist(const K* __restrict__ keys, const Seg* __restrict__ segs,
                                             int nsegs, const int* __restrict__ seg_tile0,
                                             int shift0, int npasses, uint32_t* __restrict__ hist)
{
    __shared__ uint32_t s_h[8][RADIX];
    const int gt = blockIdx.x;
    if (gt >= seg_tile0[nsegs]) return;       // capacity-sized grid: beyond the batch's tiles
    const int sg = find_seg(seg_tile0, nsegs, gt);
    const Seg S = segs[sg];
    const long long lbase = (long long)(gt - seg_tile0[sg]) * (ST * HITEMS);
    for (int i = threadIdx.x; i < npasses * RADIX; i += ST) (&s_h[0][0])[i] = 0;
    __syncthreads();
    for (int k = 0; k < HITEMS; ++k) {
        const long long li = lbase + k * ST + threadIdx.x;
        if (li < S.count) {
            const K key = keys[S.base + li];
            for (int p = 0; p < npasses; ++p) atomicAdd(&s_h[p][digit_of(key, shift0 + 8 * p)], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npasses * RADIX; i += ST) {
        const uint32_t c = (&s_h[0][0])[i];
        if (c) atomicAdd(hist + (long long)sg * npasses * RADIX + i, c);
    }
}

// exclusive scan of every (segment, pass) histogram, in place
__global__ void __launch_bounds__(ST) k_hist_scan(uint32_t* __restrict__ hist)
{
    __shared__ uint32_t s_warp[SW];
    uint32_t* h = hist + (long long)blockIdx.x * RADIX;
    const uint32_t x = h[threadIdx.x];
    const uint32_t e = block_excl_scan(x, s_warp);
    h[threadIdx.x] = e;
}

// ------------------------------------------------------------------ onesweep
template <typename K, bool KV, int ITEMS>
__global__ void __launch_bounds__(ST, S3R_SORT_MINB) k_onesweep(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                 K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                 const Seg* __restrict__ segs, int nsegs,
                                                 const int* __restrict__ seg_tile0,
                                                 const uint32_t* __restrict__ digit_base,
                                                 int pass, int npasses,
                                                 uint32_t* __restrict__ lookback,
                                                 int* __restrict__ ticket, int shift)
{
    constexpr int TI = ST * ITEMS;
    __shared__ int s_gt, s_sg;
    __shared__ uint32_t s_whist[SW][RADIX];
    __shared__ uint32_t s_local[RADIX];
    __shared__ uint32_t s_global[RADIX];
    __shared__ uint32_t s_warp[SW];
    __shared__ K s_keys[TI];
    __shared__ uint32_t s_vals[KV ? TI : 1];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        const int gt = atomicAdd(ticket, 1);
        s_gt = gt;
        s_sg = find_seg(seg_tile0, nsegs, gt);
    }
    for (int i = tid; i < SW * RADIX; i += ST) (&s_whist[0][0])[i] = 0;
    __syncthreads();
    const int gt = s_gt, sg = s_sg;
    // capacity-sized grid: tickets past the batch's tiles have nothing to sort
    // (they come after every real tile, so no look-back chain waits on them)
    if (gt >= seg_tile0[nsegs]) return;
    const Seg S = segs[sg];
    const int ltile = gt - seg_tile0[sg];
    const long long tbase = (long long)ltile * TI;
    const int cnt = (int)min((long long)TI, S.count - tbase);

    K key[ITEMS];
    uint32_t val[ITEMS];
    uint32_t rnk[ITEMS];
    const unsigned ltmask = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int li = warp * 32 * ITEMS + k * 32 + lane;
        const bool valid = li < cnt;
        key[k] = valid ? kin[S.base + tbase + li] : (K)0;
        if (KV) val[k] = valid ? (vin ? vin[S.base + tbase + li] : (uint32_t)(tbase + li)) : 0u;
        const uint32_t d = valid ? digit_of(key[k], shift) : (uint32_t)RADIX;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        uint32_t cur = 0;
        if (valid) cur = s_whist[warp][d];
        rnk[k] = cur + __popc(peers & ltmask);
        __syncwarp();
        if (valid && (peers & ltmask) == 0) s_whist[warp][d] = cur + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // per digit: exclusive over warps, block count
    const int d = tid;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < SW; ++w) {
        const uint32_t c = s_whist[w][d];
        s_whist[w][d] = run;
        run += c;
    }
    const uint32_t cnt_d = run;
    s_local[d] = block_excl_scan(cnt_d, s_warp);

    // decoupled look-back for digit d within the segment
    uint32_t* lb = lookback + (long long)gt * RADIX + d;
    uint32_t excl = 0;
    if (ltile == 0) {
        st_volatile(lb, LB_PRE | cnt_d);
    } else {
        st_volatile(lb, LB_AGG | cnt_d);
        long long j = gt - 1;
        while (true) {
            const uint32_t w = ld_volatile(lookback + j * RADIX + d);
            if ((w >> 30) == 0) continue;
            excl += w & LB_MASK;
            if (w & LB_PRE) break;
            --j;
        }
        st_volatile(lb, LB_PRE | (excl + cnt_d));
    }
    s_global[d] = digit_base[((long long)sg * npasses + pass) * RADIX + d] + excl;
    __syncthreads();

#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const int li = warp * 32 * ITEMS + k * 32 + lane;
        if (li < cnt) {
            const uint32_t dd = digit_of(key[k], shift);
            const uint32_t pos = s_local[dd] + s_whist[warp][dd] + rnk[k];
            s_keys[pos] = key[k];
            if (KV) s_vals[pos] = val[k];
        }
    }
    __syncthreads();
    for (int i = tid; i < cnt; i += ST) {
        const K kk = s_keys[i];
        const uint32_t dd = digit_of(kk, shift);
        const long long gp = (long long)s_global[dd] + (i - (long long)s_local[dd]);
        kout[S.base + gp] = kk;
        if (KV) vout[S.base + gp] = s_vals[i];
    }
}
}  // namespace

int onesweep64_tile() { return ST * ITEMS64; }
int hist_tile() { return ST * HITEMS; }

void launch_hist64(const unsigned long long* keys, const Seg* segs, int nsegs,
                   const int* seg_tile0, int total_tiles, int shift0, int npasses, uint32_t* hist,
                   cudaStream_t st)
{
    if (total_tiles == 0) return;
    k_hist<unsigned long long><<<total_tiles, ST, 0, st>>>(keys, segs, nsegs, seg_tile0, shift0,
                                                           npasses, hist);
}

void launch_hist_scan(uint32_t* hist, int nsegs, int npasses, cudaStream_t st)
{
    if (nsegs * npasses == 0) return;
    k_hist_scan<<<nsegs * npasses, ST, 0, st>>>(hist);
}

void launch_onesweep64kv(const unsigned long long* kin, const uint32_t* vin,
                         unsigned long long* kout, uint32_t* vout, const Seg* segs, int nsegs,
                         const int* seg_tile0, int total_tiles, const uint32_t* digit_base,
                         int pass, int npasses, uint32_t* lookback, int* ticket, int shift,
                         cudaStream_t st)
{
    if (total_tiles == 0) return;
    k_onesweep<unsigned long long, true, ITEMS64><<<total_tiles, ST, 0, st>>>(
        kin, vin, kout, vout, segs, nsegs, seg_tile0, digit_base, pass, npasses, lookback, ticket,
        shift);
}

}  // namespace s3r
