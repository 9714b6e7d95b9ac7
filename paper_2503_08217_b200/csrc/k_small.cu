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
// bits), so a bitonic sort of (key, slot) gives the same order as the stable
// radix sort.  Tile lists (R12): warp w takes tile t, walks the ranks 32 at a
// time and keeps those whose rectangle contains t (ballot + popc keep rank
// order); one pass counts, a block scan places the lists, a second pass writes.
#include "s3r_internal.cuh"

namespace s3r {

namespace {

constexpr int SMT = 1024;
constexpr int SMW = SMT / 32;

__device__ __forceinline__ bool rect_has(uint2 rr, int tx, int ty)
{
    return tx >= (int)(rr.x & 0xffff) && tx <= (int)(rr.x >> 16) && ty >= (int)(rr.y & 0xffff) &&
           ty <= (int)(rr.y >> 16);
}

// Bitonic sort of (key, slot) over E * SMT elements in registers (thread t
// holds positions t and t + SMT): partners within a warp by shuffles, farther
// ones through shared memory, SMT apart inside the thread; padding keys (~0)
// sort last.  The result is left in s_key / s_idx by position.
template <int E>
__device__ __forceinline__ void bitonic_sort(const unsigned long long* __restrict__ dkey,
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
    for (int k = 2; k <= E * SMT; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (E == 2 && j == SMT) {   // k = 2 SMT: ascending, partner in the thread
                if (key[E - 1] < key[0]) {
                    const unsigned long long tk = key[0];
                    key[0] = key[E - 1];
                    key[E - 1] = tk;
                    const uint32_t ti = idx[0];
                    idx[0] = idx[E - 1];
                    idx[E - 1] = ti;
                }
                continue;
            }
            unsigned long long pk[E];
            uint32_t pi[E];
            if (j >= 32) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    s_key[tid + e * SMT] = key[e];
                    s_idx[tid + e * SMT] = (uint16_t)idx[e];
                }
                __syncthreads();
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    pk[e] = s_key[(tid ^ j) + e * SMT];
                    pi[e] = s_idx[(tid ^ j) + e * SMT];
                }
                __syncthreads();
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    pk[e] = __shfl_xor_sync(0xffffffffu, key[e], j);
                    pi[e] = __shfl_xor_sync(0xffffffffu, idx[e], j);
                }
            }
#pragma unroll
            for (int e = 0; e < E; ++e) {
                // the pair's lower position keeps the min in an ascending block
                // (the max in a descending one), the upper position the other
                const int p = tid + e * SMT;
                const bool keep_min = ((p & j) == 0) == ((p & k) == 0);
                if (keep_min ? pk[e] < key[e] : pk[e] > key[e]) {
                    key[e] = pk[e];
                    idx[e] = pi[e];
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
}

__global__ void __launch_bounds__(SMT) k_small_sortbin(const DevView* __restrict__ views,
                                                       const unsigned long long* __restrict__ dkey,
                                                       const float4* __restrict__ rec,
                                                       unsigned long long* __restrict__ keys_out,
                                                       uint32_t* __restrict__ order_out,
                                                       float4* __restrict__ rec_sorted,
                                                       uint2* __restrict__ rect_sorted,
                                                       uint32_t* __restrict__ tlists,
                                                       int2* __restrict__ tranges)
{
    static_assert(SMALL_MAX == 2 * SMT, "two elements per thread");
    __shared__ unsigned long long s_key[SMALL_MAX];
    __shared__ uint16_t s_idx[SMALL_MAX];
    __shared__ uint2 s_rect[SMALL_MAX];
    __shared__ int s_cnt[SMALL_TILES];
    __shared__ int s_w[SMW];
    const DevView& V = views[blockIdx.x];
    if (!V.small) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = (int)V.n_rendered;
    const long long base = V.cap_off;
    // ---- depth order: (key, slot) sorted in registers / shared memory
    if (n <= SMT) bitonic_sort<1>(dkey, base, n, s_key, s_idx);
    else bitonic_sort<2>(dkey, base, n, s_key, s_idx);
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
    // ---- per-tile list lengths
    const int nt = V.ntiles;
    for (int t = warp; t < nt; t += SMW) {
        const int tx = t % V.TX, ty = t / V.TX;
        int c = 0;
        for (int b = 0; b < n; b += 32) {
            const int r = b + lane;
            c += __popc(__ballot_sync(0xffffffffu, r < n && rect_has(s_rect[r], tx, ty)));
        }
        if (lane == 0) s_cnt[t] = c;
    }
    __syncthreads();
    // ---- exclusive scan of the lengths (nt <= SMALL_TILES = SMT)
    const int x = tid < nt ? s_cnt[tid] : 0;
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
    if (tid < nt) {
        s_cnt[tid] = start;
        tranges[V.trange_off + tid] = make_int2(start, start + x);
    }
    __syncthreads();
    // ---- the lists: ranks in rank order
    uint32_t* out = tlists + V.tlist_off;
    const unsigned lt = (1u << lane) - 1u;
    for (int t = warp; t < nt; t += SMW) {
        const int tx = t % V.TX, ty = t / V.TX;
        int c = s_cnt[t];
        for (int b = 0; b < n; b += 32) {
            const int r = b + lane;
            const bool in = r < n && rect_has(s_rect[r], tx, ty);
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            if (in) out[c + __popc(bal & lt)] = (uint32_t)r;
            c += __popc(bal);
        }
    }
}

}  // namespace

void launch_small_sortbin(const DevView* views, int n_views, const unsigned long long* dkey,
                          const float4* rec, unsigned long long* keys_out, uint32_t* order_out,
                          float4* rec_sorted, uint2* rect_sorted, uint32_t* tlists,
                          int2* tranges, cudaStream_t st)
{
    if (n_views == 0) return;
    k_small_sortbin<<<n_views, SMT, 0, st>>>(views, dkey, rec, keys_out, order_out, rec_sorted,
                                             rect_sorted, tlists, tranges);
}

}  // namespace s3r
