// k_small.cu — the a4 step (depth order + tile binning) of a SMALL view in one
// CTA: when a view renders at most SMALL_MAX splats over at most SMALL_TILES
// tiles, the depth sort (K5: hist, scan, ~6 onesweep passes), the permute (K3)
// and the supertile binning (K4: count, scan, scatter, expand) — a dozen
// launches that each do almost nothing at this size — are replaced by one CTA
// that keeps the view on chip (SURVEY.md §7 hard part 7: C1 is
// launch-bound).  The outputs are the big path's, bit for bit: the sorted
// (depth << gbits | index) keys and slot order, the records and rectangles by
// rank (with the flush-ellipse extents), and per-tile lists of ranks in rank
// order with their ranges — only packed without the supertile area's gaps.
//
// Order (reading R11): the keys are unique (the Gaussian index is in the low
// bits), so sorting (key, slot) by key (warp bitonic runs + pairwise merges)
// gives the same order as the stable radix sort.  Tile lists (R12): a warp takes one contiguous part of the ranks
// of tile t (a view with few tiles splits each tile's ranks over the idle
// warps), walks it 32 ranks at a time and keeps those whose rectangle contains
// t (ballot + popc keep rank order); one pass counts per (tile, part), a block
// scan in (tile, part) order places the parts, a second pass writes.
#include "s3r_internal.cuh"

namespace s3r {

namespace {

constexpr int SMT = 1024;
#ifndef S3R_SMALL_MASK
#define S3R_SMALL_MASK 1   // views of <= 32 tiles: tile lists from per-rank tile masks + ballots
#endif
constexpr int SMW = SMT / 32;

__device__ __forceinline__ bool rect_has(uint2 rr, int tx, int ty)
{
    return tx >= (int)(rr.x & 0xffff) && tx <= (int)(rr.x >> 16) && ty >= (int)(rr.y & 0xffff) &&
           ty <= (int)(rr.y >> 16);
}

// Sort of (key, slot) over E * SMT positions (thread t holds positions t and
// t + SMT), padding keys (~0) last.  Each warp first sorts its 32 consecutive
// positions with a bitonic network on shuffles; then sorted runs of L = 32, 64,
// ... are merged pairwise in shared memory: an element's place in the merged run
// is its rank in its own run plus the number of keys of the partner run below
// it (a branch-free binary search; a right-run element also counts equal keys,
// which keeps the padding duplicates apart).  The result is left in
// s_key / s_idx by position.
template <int E>
__device__ __forceinline__ void merge_sort(const unsigned long long* __restrict__ dkey,
                                           long long base, int n,
                                           unsigned long long* s_key, uint16_t* s_idx)
{
    const int tid = threadIdx.x;
    unsigned long long key[E];
    uint32_t idx[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int p = tid + e * SMT;
        key[e] = p < n ? dkey[base + p] : ~0ull;
        idx[e] = (uint32_t)p;
    }
    // ---- 32-element runs, ascending, in registers
    for (int k = 2; k <= 32; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const unsigned long long pk = __shfl_xor_sync(0xffffffffu, key[e], j);
                const uint32_t pi = __shfl_xor_sync(0xffffffffu, idx[e], j);
                const int p = tid + e * SMT;
                const bool up = k == 32 || (p & k) == 0;
                const bool keep_min = ((p & j) == 0) == up;
                if (keep_min ? pk < key[e] : pk > key[e]) {
                    key[e] = pk;
                    idx[e] = pi;
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
        s_key[tid + e * SMT] = key[e];
        s_idx[tid + e * SMT] = (uint16_t)idx[e];
    }
    __syncthreads();
    // ---- pairwise merges of sorted runs of length L
    for (int L = 32; L < E * SMT; L <<= 1) {
        int outp[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int p = tid + e * SMT;
            const int r = p / L;
            const int q0 = (r ^ 1) * L;
            const bool right = r & 1;
            int c = 0;
            for (int st = L >> 1; st > 0; st >>= 1) {
                const unsigned long long a = s_key[q0 + c + st - 1];
                if (right ? a <= key[e] : a < key[e]) c += st;
            }
            const unsigned long long a = s_key[q0 + c];
            if (right ? a <= key[e] : a < key[e]) c += 1;
            outp[e] = (r & ~1) * L + (p % L) + c;
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            s_key[outp[e]] = key[e];
            s_idx[outp[e]] = (uint16_t)idx[e];
        }
        __syncthreads();
        // the element now at position tid (+ SMT) for the next round
#pragma unroll
        for (int e = 0; e < E; ++e) {
            key[e] = s_key[tid + e * SMT];
            idx[e] = s_idx[tid + e * SMT];
        }
    }
}

__global__ void __launch_bounds__(SMT) k_small_sortbin(DevView* __restrict__ views,
                                                       const unsigned long long* __restrict__ dkey,
                                                       const float4* __restrict__ rec,
                                                       unsigned long long* __restrict__ keys_out,
                                                       uint32_t* __restrict__ order_out,
                                                       float4* __restrict__ rec_sorted,
                                                       uint2* __restrict__ rect_sorted,
                                                       uint32_t* __restrict__ tlists,
                                                       int2* __restrict__ tranges,
                                                       SmallPlan sp)
{
    static_assert(SMALL_MAX == 2 * SMT, "two elements per thread");
    __shared__ unsigned long long s_key[SMALL_MAX];
    __shared__ uint16_t s_idx[SMALL_MAX];
    __shared__ uint2 s_rect[SMALL_MAX];
    __shared__ int s_cnt[SMALL_TILES];
    __shared__ int s_w[SMW];
    DevView& V = views[blockIdx.x];
    if (!V.small) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int n;
    if (sp.ctr) {
        // self-planned view (k_plan_bins' job for this view): its splat count,
        // the capacity check, the stats copy
        const ViewCounters k = sp.ctr[blockIdx.x];
        long long nr = (long long)k.n_rendered;
        if (nr > sp.cap_rendered || !small_view(nr, V.ntiles)) {
            nr = 0;
            if (tid == 0) atomicOr(sp.err, ERR_CAPACITY);
        }
        n = (int)nr;
        if (tid == 0) {
            sp.h_ctr[blockIdx.x] = k;
            V.n_rendered = nr;
            V.n_pairs = nr ? (long long)k.n_pairs : 0;
        }
    } else {
        n = (int)V.n_rendered;
    }
    const long long base = V.cap_off;
    // ---- depth order: (key, slot) sorted in registers / shared memory
    if (n <= SMT) merge_sort<1>(dkey, base, n, s_key, s_idx);
    else merge_sort<2>(dkey, base, n, s_key, s_idx);
    // ---- permute (K3): records and rectangles by rank
    for (int r = tid; r < n; r += SMT) {
        const uint32_t j = s_idx[r];
        keys_out[base + r] = s_key[r];
        order_out[base + r] = j;
        const float4* src = rec + 3 * (base + j);
        const float4 q0 = src[0];
        float4 q1 = src[1], q2 = src[2];
        const uint2 rr = make_uint2(__float_as_uint(q1.w), __float_as_uint(q2.w));
        rect_sorted[base + r] = rr;
        s_rect[r] = rr;
        flush_extent(q1.x, q1.y, q1.z, q1.w, q2.w);
        float4* dst = rec_sorted + 3 * (base + r);
        dst[0] = q0;
        dst[1] = q1;
        dst[2] = q2;
    }
    __syncthreads();
    const int nt = V.ntiles;
#if S3R_SMALL_MASK
    if (nt <= 32) {
        // ---- a view of <= 32 tiles (C1: 16): a warp takes 32 ranks a round,
        // each lane its rank's tile mask (bit t = tile t of the view), one
        // ballot per tile; per-(round, tile) counts scanned over the rounds
        // give each round's place in the tile's list (rank order), the tile
        // totals scanned over the tiles give the lists' starts.  s_key (free
        // after the permute) holds the counts and ballots.
        const int nr = (n + 31) >> 5;                                  // <= 64 rounds
        uint32_t* s_c2 = reinterpret_cast<uint32_t*>(s_key);           // [64][32] counts
        uint32_t* s_b2 = s_c2 + 64 * 32;                                // [64][32] ballots
        const int TX = V.TX;
        auto mask_of = [&](int r) -> uint32_t {
            if (r >= n) return 0u;
            const uint2 rr = s_rect[r];
            const int tx0 = rr.x & 0xffff, tx1 = rr.x >> 16, ty0 = rr.y & 0xffff, ty1 = rr.y >> 16;
            const int wdt = tx1 - tx0 + 1;
            const uint32_t row = (wdt >= 32 ? ~0u : ((1u << wdt) - 1u)) << tx0;
            uint32_t m = 0;
            for (int ty = ty0; ty <= ty1; ++ty) m |= row << (ty * TX);
            return m;
        };
        for (int rd = warp; rd < nr; rd += SMW) {
            const uint32_t m = mask_of(rd * 32 + lane);
            for (int t = 0; t < nt; ++t) {
                const uint32_t b = __ballot_sync(0xffffffffu, (m >> t) & 1u);
                if (lane == t) {
                    s_b2[rd * 32 + t] = b;
                    s_c2[rd * 32 + t] = __popc(b);
                }
            }
        }
        __syncthreads();
        // per tile (warp t): exclusive scan over the rounds, in place; total
        if (warp < nt) {
            const int t = warp;
            uint32_t run = 0;
            for (int h = 0; h < 2; ++h) {                 // rounds 0-31, then 32-63
                const int rd = h * 32 + lane;
                const uint32_t c = rd < nr ? s_c2[rd * 32 + t] : 0u;
                uint32_t y = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
                    if (lane >= o) y += z;
                }
                if (rd < nr) s_c2[rd * 32 + t] = run + y - c;
                run += __shfl_sync(0xffffffffu, y, 31);
            }
            if (lane == 0) s_cnt[t] = (int)run;
        }
        __syncthreads();
        // tile starts: exclusive scan over the tiles (one warp)
        if (warp == 0) {
            const int c = lane < nt ? s_cnt[lane] : 0;
            int y = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int z = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += z;
            }
            if (lane < nt) {
                s_w[lane] = y - c;
                tranges[V.trange_off + lane] = make_int2(y - c, y);
            }
        }
        __syncthreads();
        uint32_t* out = tlists + V.tlist_off;
        const unsigned lt = (1u << lane) - 1u;
        for (int rd = warp; rd < nr; rd += SMW) {
            const int r = rd * 32 + lane;
            const uint32_t m = mask_of(r);
            for (int t = 0; t < nt; ++t)
                if ((m >> t) & 1u)
                    out[s_w[t] + s_c2[rd * 32 + t] + __popc(s_b2[rd * 32 + t] & lt)] = (uint32_t)r;
        }
        return;
    }
#endif
    // ---- per-tile list lengths: a tile's ranks are split into PP parts (all
    // 32 warps busy when the view has few tiles); slot t PP + part
    int PP = 1;
    while (PP * 2 * nt <= SMW) PP *= 2;
    const int ns = nt * PP;                 // <= SMT slots
    const int plen = (n + PP - 1) / PP;
    for (int sl = warp; sl < ns; sl += SMW) {
        const int t = sl / PP, part = sl % PP;
        const int tx = t % V.TX, ty = t / V.TX;
        const int r0 = part * plen, r1 = min(n, r0 + plen);
        int c = 0;
        for (int b = r0; b < r1; b += 32) {
            const int r = b + lane;
            c += __popc(__ballot_sync(0xffffffffu, r < r1 && rect_has(s_rect[r], tx, ty)));
        }
        if (lane == 0) s_cnt[sl] = c;
    }
    __syncthreads();
    // ---- exclusive scan of the slot lengths
    const int x = tid < ns ? s_cnt[tid] : 0;
    int v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_w[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const int w = s_w[lane];
        int ww = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ww, o);
            if (lane >= o) ww += y;
        }
        s_w[lane] = ww - w;
    }
    __syncthreads();
    const int start = s_w[warp] + v - x;
    __syncthreads();
    if (tid < ns) s_cnt[tid] = start;
    if (tid == ns - 1) s_w[0] = start + x;          // the view's total (P)
    __syncthreads();
    // tile ranges: [its first slot's start, the next tile's first slot's start)
    if (tid < nt)
        tranges[V.trange_off + tid] =
            make_int2(s_cnt[tid * PP], tid + 1 < nt ? s_cnt[(tid + 1) * PP] : s_w[0]);
    // ---- the lists: ranks in rank order
    uint32_t* out = tlists + V.tlist_off;
    const unsigned lt = (1u << lane) - 1u;
    for (int sl = warp; sl < ns; sl += SMW) {
        const int t = sl / PP, part = sl % PP;
        const int tx = t % V.TX, ty = t / V.TX;
        const int r0 = part * plen, r1 = min(n, r0 + plen);
        int c = s_cnt[sl];
        for (int b = r0; b < r1; b += 32) {
            const int r = b + lane;
            const bool in = r < r1 && rect_has(s_rect[r], tx, ty);
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            if (in) out[c + __popc(bal & lt)] = (uint32_t)r;
            c += __popc(bal);
        }
    }
}

}  // namespace

void launch_small_sortbin(DevView* views, int n_views, const unsigned long long* dkey,
                          const float4* rec, unsigned long long* keys_out, uint32_t* order_out,
                          float4* rec_sorted, uint2* rect_sorted, uint32_t* tlists,
                          int2* tranges, const SmallPlan& sp, cudaStream_t st)
{
    if (n_views == 0) return;
    k_small_sortbin<<<n_views, SMT, 0, st>>>(views, dkey, rec, keys_out, order_out, rec_sorted,
                                             rect_sorted, tlists, tranges, sp);
}

}  // namespace s3r
