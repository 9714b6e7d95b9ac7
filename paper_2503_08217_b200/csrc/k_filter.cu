// k_filter.cu — K1: temporal-visibility filter + ordered stream compaction.
//
// PAPER.md P:171-172 (§3.3 "Temporal separation"): "we directly select the
// visible Gaussians G' whose visibility intervals encompass t, denoted as
// t_s <= t <= t_e".  Reading R1: t_s == v_s, t_e == v_e, inclusive; NaN -> out.
//
// One CTA serves a group of up to MAX_TSLOTS distinct view times: it reads its
// 4096-Gaussian slice of v = (v_s, v_e) ONCE (16-byte vector loads, 8 per
// thread) and produces, for every time slot of its group, the ascending list
// of kept indices.  A large scene takes one group per launch; a small one
// (C2: 49 slices) splits its times into smaller groups launched together as
// grid.y (filter_groups), so that the grid fills the GPU.  Within a CTA the order is fixed by warp ballots + popc (per
// (round, warp) counts, one warp scan per slot); across CTAs by a decoupled
// look-back per slot (CTA order from an atomic ticket, so a CTA only waits on
// CTAs that are already resident).  On large scenes (RANGE) a (round, warp)
// group tests only the slots whose time lies in its 64 Gaussians' interval
// hull — a contiguous run of the sorted slot times, ~1/5 of them because the
// scene's index order is spatially coherent.  Algorithmic bytes: 8 N read +
// 4 sum_s N_t(s) written.
#include <algorithm>

#include "s3r_internal.cuh"

namespace s3r {

namespace {
constexpr int FT = 256;          // threads
constexpr int FV = 8;            // float4 (2 Gaussians) per thread
constexpr int FTILE = FT * FV * 2;
constexpr int FGROUPS = FV * (FT / 32);   // (round, warp) groups = 64
// RANGE: per (round, warp) only the slots inside the warp's interval hull are
// tested.  Chosen per launch (launch_filter): it pays on large scenes (C3
// 0.129 -> 0.099 ms, C4 0.474 -> 0.261 ms) but not on a grid of a few dozen
// CTAs, where its serial binary searches are exposed (C2: 0.100 vs 0.137 ms).
#ifndef S3R_FILTER_WANT_BIG
#define S3R_FILTER_WANT_BIG 0   // CTAs a large scene's K1 grid aims at by grouping slots (0: MAX_TSLOTS per launch)
#endif
#ifndef S3R_FILTER_RANGE_MIN_TILES
#define S3R_FILTER_RANGE_MIN_TILES 296   // 2 CTAs per SM
#endif


// blockIdx.y = slot group: slots [gs y, gs y + gs) of the launch's Tall, each
// group with its own ticket, look-back chains, counts and output lists
template <bool RANGE>
__global__ void __launch_bounds__(FT) k_filter(const float2* __restrict__ vis, long long n,
                                               const float* __restrict__ times, int Tall, int gs,
                                               int32_t* __restrict__ idx_out, long long stride,
                                               unsigned long long* __restrict__ counts,
                                               uint32_t* __restrict__ lookback,
                                               int* __restrict__ ticket, int ntiles)
{
    const int s0 = blockIdx.y * gs;
    const int T = min(gs, Tall - s0);
    times += s0;
    idx_out += (long long)s0 * stride;
    counts += s0;
    lookback += (long long)s0 * ntiles;
    ticket += blockIdx.y;
    __shared__ int s_tile;
    __shared__ float s_t[MAX_TSLOTS];
    __shared__ float s_st[MAX_TSLOTS];       // the slot times in ascending order
    __shared__ int s_sid[MAX_TSLOTS];        // ... and their slot ids
    __shared__ uint8_t s_rng[FV][FT / 32][2];  // per (round, warp): sorted positions [lo, hi]
    __shared__ uint16_t s_cnt[MAX_TSLOTS][FGROUPS];
    __shared__ uint32_t s_agg[MAX_TSLOTS];
    __shared__ uint32_t s_base[MAX_TSLOTS];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ticket, 1);
    if (tid < T) s_t[tid] = times[tid];
    __syncthreads();
    if constexpr (RANGE) {
        if (tid < T) {          // rank sort of the (distinct) slot times
            const float ti = s_t[tid];
            int r = 0;
            for (int j = 0; j < T; ++j) r += (s_t[j] < ti || (s_t[j] == ti && j < tid)) ? 1 : 0;
            s_st[r] = ti;
            s_sid[r] = tid;
        }
        for (int i = tid; i < T * FGROUPS; i += FT) (&s_cnt[0][0])[i] = 0;
        __syncthreads();
    }
    const int tile = s_tile;
    const long long g0 = (long long)tile * FTILE;

    // v for Gaussians g0 + 2*(k*FT + tid) + {0,1}
    float4 v[FV];
    const float4* vis4 = reinterpret_cast<const float4*>(vis);
#pragma unroll
    for (int k = 0; k < FV; ++k) {
        long long g = g0 + 2ll * (k * FT + tid);
        if (g + 1 < n) {
            v[k] = __ldg(vis4 + (g >> 1));
        } else if (g < n) {
            float2 a = __ldg(vis + g);
            v[k] = make_float4(a.x, a.y, __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
        } else {
            v[k] = make_float4(__int_as_float(0x7fc00000), 0.f, __int_as_float(0x7fc00000), 0.f);
        }
    }

    if constexpr (RANGE) {
        // per (round, warp): only the slots whose time lies in [min v_s, max v_e] of
        // the warp's 64 Gaussians can keep any of them (the scene's index order is
        // spatially coherent, so that is ~1/5 of the slots); those are a contiguous
        // run [lo, hi] of the sorted times.  NaN bounds never pass (fminf / fmaxf
        // drop them from the run; the exact test below still applies).
#pragma unroll
        for (int k = 0; k < FV; ++k) {
            float vmin = fminf(v[k].x, v[k].z), vmax = fmaxf(v[k].y, v[k].w);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
                vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
            }
            int lo = 0, hi = T;                  // first sorted position with t >= vmin
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (s_st[mid] < vmin) lo = mid + 1; else hi = mid;
            }
            int lo2 = lo, hi2 = T;               // first sorted position with t > vmax
            while (lo2 < hi2) {
                const int mid = (lo2 + hi2) >> 1;
                if (s_st[mid] <= vmax) lo2 = mid + 1; else hi2 = mid;
            }
            if (lane == 0) {
                s_rng[k][warp][0] = (uint8_t)lo;
                s_rng[k][warp][1] = (uint8_t)lo2;
            }
            for (int q = lo; q < lo2; ++q) {
                const float t = s_st[q];
                const bool f0 = (v[k].x <= t) && (t <= v[k].y);
                const bool f1 = (v[k].z <= t) && (t <= v[k].w);
                const unsigned b0 = __ballot_sync(0xffffffffu, f0);
                const unsigned b1 = __ballot_sync(0xffffffffu, f1);
                if (lane == 0) s_cnt[s_sid[q]][k * (FT / 32) + warp] = (uint16_t)(__popc(b0) + __popc(b1));
            }
        }
        __syncthreads();
    } else {
        // per (slot, round, warp) counts
        for (int s = 0; s < T; ++s) {
            const float t = s_t[s];
#pragma unroll
            for (int k = 0; k < FV; ++k) {
                bool f0 = (v[k].x <= t) && (t <= v[k].y);
                bool f1 = (v[k].z <= t) && (t <= v[k].w);
                unsigned b0 = __ballot_sync(0xffffffffu, f0);
                unsigned b1 = __ballot_sync(0xffffffffu, f1);
                if (lane == 0) s_cnt[s][k * (FT / 32) + warp] = (uint16_t)(__popc(b0) + __popc(b1));
            }
        }
        __syncthreads();
    }

    // exclusive scan of the 64 groups of each slot (one warp per slot)
    for (int s = warp; s < T; s += FT / 32) {
        uint32_t c0 = s_cnt[s][2 * lane], c1 = s_cnt[s][2 * lane + 1];
        uint32_t x = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        uint32_t ex = x - (c0 + c1);
        s_cnt[s][2 * lane] = (uint16_t)ex;
        s_cnt[s][2 * lane + 1] = (uint16_t)(ex + c0);
        if (lane == 31) s_agg[s] = x;
    }
    __syncthreads();

    // decoupled look-back per slot: publish every slot's aggregate first, then
    // one warp per slot walks its chain 32 predecessors at a time
    if (tid < T) lb_publish(lookback + (long long)tid * ntiles + tile,
                            (tile == 0 ? LB_PRE : LB_AGG) | s_agg[tid]);
    for (int s = warp; s < T; s += FT / 32) {
        uint32_t* lb = lookback + (long long)s * ntiles;
        const uint32_t agg = s_agg[s];
        const uint32_t excl = (tile == 0) ? 0u : warp_lookback(lb, 1, tile, 0);
        if (lane == 0) {
            if (tile != 0) lb_publish(lb + tile, LB_PRE | (excl + agg));
            s_base[s] = excl;
            if (tile == ntiles - 1) counts[s] = (unsigned long long)(excl + agg);
        }
    }
    __syncthreads();

    const unsigned lt = (1u << lane) - 1u;
    if constexpr (RANGE) {
#pragma unroll
        for (int k = 0; k < FV; ++k) {
            const int lo = s_rng[k][warp][0], hi = s_rng[k][warp][1];
            const long long g = g0 + 2ll * (k * FT + tid);
            for (int q = lo; q < hi; ++q) {
                const float t = s_st[q];
                const int s = s_sid[q];
                const bool f0 = (v[k].x <= t) && (t <= v[k].y);
                const bool f1 = (v[k].z <= t) && (t <= v[k].w);
                const unsigned b0 = __ballot_sync(0xffffffffu, f0);
                const unsigned b1 = __ballot_sync(0xffffffffu, f1);
                const uint32_t o = s_base[s] + s_cnt[s][k * (FT / 32) + warp] + __popc(b0 & lt) +
                                   __popc(b1 & lt);
                int32_t* out = idx_out + (long long)s * stride;
                if (f0) out[o] = (int32_t)g;
                if (f1) out[o + (f0 ? 1 : 0)] = (int32_t)(g + 1);
            }
        }
    } else {
        for (int s = 0; s < T; ++s) {
            const float t = s_t[s];
            const uint32_t base = s_base[s];
            int32_t* out = idx_out + (long long)s * stride;
#pragma unroll
            for (int k = 0; k < FV; ++k) {
                bool f0 = (v[k].x <= t) && (t <= v[k].y);
                bool f1 = (v[k].z <= t) && (t <= v[k].w);
                unsigned b0 = __ballot_sync(0xffffffffu, f0);
                unsigned b1 = __ballot_sync(0xffffffffu, f1);
                uint32_t o = base + s_cnt[s][k * (FT / 32) + warp] + __popc(b0 & lt) + __popc(b1 & lt);
                long long g = g0 + 2ll * (k * FT + tid);
                if (f0) out[o] = (int32_t)g;
                if (f1) out[o + (f0 ? 1 : 0)] = (int32_t)(g + 1);
            }
        }
    }
}
}  // namespace

void launch_filter(const float2* vis, long long n, const float* d_times, int T, int gs,
                   int32_t* idx_out, long long idx_stride, unsigned long long* counts,
                   uint32_t* lookback, int* ticket, cudaStream_t st)
{
    int ntiles = (int)((n + FTILE - 1) / FTILE);
    if (ntiles == 0 || T == 0) return;
    const dim3 grid(ntiles, (T + gs - 1) / gs);
    if (ntiles >= S3R_FILTER_RANGE_MIN_TILES)
        k_filter<true><<<grid, FT, 0, st>>>(vis, n, d_times, T, gs, idx_out, idx_stride, counts,
                                            lookback, ticket, ntiles);
    else
        k_filter<false><<<grid, FT, 0, st>>>(vis, n, d_times, T, gs, idx_out, idx_stride, counts,
                                             lookback, ticket, ntiles);
}

int filter_groups(long long n, int T)
{
    // slots per group: a scene of few 4096-Gaussian tiles (C2: 49) splits its
    // distinct times into groups launched together, so that the grid fills the
    // GPU (~4 CTAs per SM); a large scene keeps MAX_TSLOTS per launch
    const long long ntiles = (n + FTILE - 1) / FTILE;
    if (ntiles == 0 || T == 0) return MAX_TSLOTS;
    if (ntiles >= S3R_FILTER_RANGE_MIN_TILES && S3R_FILTER_WANT_BIG == 0) return MAX_TSLOTS;
    const long long want = ntiles >= S3R_FILTER_RANGE_MIN_TILES ? S3R_FILTER_WANT_BIG : 4 * 148;
    const long long gs = (T * ntiles + want - 1) / want;
    return (int)std::max(1ll, std::min((long long)MAX_TSLOTS, gs));
}

int filter_tile() { return FTILE; }

}  // namespace s3r
