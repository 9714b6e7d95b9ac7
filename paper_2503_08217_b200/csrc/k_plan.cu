// k_plan.cu — device-side sizing of a batch for the capacity mode
// (s3r_set_capacity): the per-view offsets that the synchronous path computes
// on the host after reading back K1's and K2's counters are computed here, so
// that a batch is enqueued without a host synchronisation (and can be
// captured in a CUDA graph).  Each kernel is one CTA of 1024 threads that
// walks the views in blocks of 1024 with block-wide exclusive scans.
//
// Capacity rule (both kernels): offsets are exclusive prefix sums of the
// views' sizes in view order; a view whose segment does not end within the
// reserved capacity is dropped (size 0: it renders an empty image) and
// ERR_CAPACITY is raised in the device error word (s3r_check reports
// S3R_ECAPACITY).  Offsets grow with the view index, so once one view is
// dropped every later one is too: the kept views' layout is exactly the
// synchronous path's.
#include "s3r_internal.cuh"

namespace s3r {

namespace {

constexpr int PLT = 1024;

// block-wide inclusive scan of one 64-bit value per thread (blockDim.x = 32 k)
__device__ __forceinline__ unsigned long long block_incl_scan(unsigned long long x,
                                                              unsigned long long* s_w)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (nw == 1) {           // one warp (batches of <= 32 views): shuffles only
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        return x;
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < nw ? s_w[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        s_w[lane] = w;
    }
    __syncthreads();
    const unsigned long long r = x + (warp ? s_w[warp - 1] : 0ull);
    __syncthreads();
    return r;
}

// After K1: n_temporal per view (from its distinct time's count) and the
// view's record segment [cap_off, cap_off + n_temporal); a view above the
// per-view capacity (which sized K2's grid) is dropped as well.
__global__ void __launch_bounds__(PLT) k_plan_records(DevView* __restrict__ views, int nv,
                                                      const unsigned long long* __restrict__ counts,
                                                      long long cap_records, long long cap_view,
                                                      long long* __restrict__ h_ntemp,
                                                      uint32_t* __restrict__ err)
{
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int T = blockDim.x;
    for (int base = 0; base < nv; base += T) {
        const int v = base + threadIdx.x;
        const unsigned long long n = v < nv ? counts[views[v].tslot] : 0ull;
        const unsigned long long incl = block_incl_scan(n, s_w);
        const unsigned long long off = s_carry + incl - n;
        if (v < nv) {
            DevView& V = views[v];
            const bool fits = (long long)(off + n) <= cap_records && (long long)n <= cap_view;
            V.cap_off = (long long)off;
            V.dbg_off = (long long)off;
            V.n_temporal = fits ? (long long)n : 0;
            if (h_ntemp) h_ntemp[v] = (long long)n;
            if (!fits) atomicOr(err, ERR_CAPACITY);
        }
        __syncthreads();
        if (threadIdx.x == T - 1) s_carry += incl;
        __syncthreads();
    }
}

// After K2: n_rendered / n_pairs per view, the sort segments, the binning
// layout (chunks, count offsets, supertile-list and tile-list offsets).
__global__ void __launch_bounds__(PLT) k_plan_bins(DevView* __restrict__ views, int nv,
                                                   const ViewCounters* __restrict__ ctr,
                                                   Seg* __restrict__ segs, int* __restrict__ dt0,
                                                   PlanCaps caps, ViewCounters* __restrict__ h_ctr,
                                                   uint32_t* __restrict__ err)
{
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_c[4];
    if (threadIdx.x < 4) s_c[threadIdx.x] = 0;
    __syncthreads();
    const int T = blockDim.x;
    for (int base = 0; base < nv; base += T) {
        const int v = base + threadIdx.x;
        ViewCounters k{};
        long long nr = 0, ns = 0;
        int nb = 0, SS = 0;
        if (v < nv) {
            k = ctr[v];
            const DevView& V = views[v];
            nb = V.nbins;
            SS = 1 << (2 * V.sshift);
            nr = (long long)k.n_rendered;
            ns = (long long)k.n_spairs;
            // per-view limits: the rendered capacity (count / scatter grids) and
            // the 32-bit list positions
            if (nr > caps.rendered_view || (long long)k.n_pairs >= (1ll << 31) ||
                (long long)SS * ns >= (1ll << 31)) {
                nr = 0;
                ns = 0;
                atomicOr(err, ERR_CAPACITY);
            }
            if (h_ctr) h_ctr[v] = k;
        }
        const unsigned long long q_sp = (unsigned long long)ns;
        const unsigned long long q_tl = (unsigned long long)SS * (unsigned long long)ns;
        const bool sm = v < nv && small_view(nr, views[v].ntiles);
        const long long nch = sm ? 0 : (nr + caps.bin_chunk - 1) / caps.bin_chunk;
        const unsigned long long q_cnt = (unsigned long long)nb * (unsigned long long)nch;
        const unsigned long long q_dt =
            sm ? 0ull : (unsigned long long)((nr + caps.sort_tile - 1) / caps.sort_tile);
        const unsigned long long i_sp = block_incl_scan(q_sp, s_w);
        const unsigned long long i_tl = block_incl_scan(q_tl, s_w);
        const unsigned long long i_cnt = block_incl_scan(q_cnt, s_w);
        const unsigned long long o_sp = s_c[0] + i_sp - q_sp, o_tl = s_c[1] + i_tl - q_tl,
                                 o_cnt = s_c[2] + i_cnt - q_cnt;
        const bool fits = (long long)(o_sp + q_sp) <= caps.bin_pairs &&
                          (long long)(o_tl + q_tl) <= caps.tile_entries &&
                          (long long)(o_cnt + q_cnt) <= caps.counts;
        // a dropped view sorts nothing: its tiles are taken out of the sort grid
        const unsigned long long q_dt2 = fits ? q_dt : 0ull;
        const unsigned long long i_dt = block_incl_scan(q_dt2, s_w);
        const unsigned long long o_dt = s_c[3] + i_dt - q_dt2;
        if (v < nv) {
            DevView& V = views[v];
            if (!fits) {
                nr = 0;
                atomicOr(err, ERR_CAPACITY);
            }
            V.n_rendered = nr;
            V.n_pairs = fits ? (long long)k.n_pairs : 0;
            // (a dropped view renders nothing: small if its tiles fit, so that
            // its empty tile ranges are written when the big path is not run)
            V.small = (fits ? sm : small_view(0, V.ntiles)) ? 1 : 0;
            V.nchunks = V.small ? 0 : (int)((nr + caps.bin_chunk - 1) / caps.bin_chunk);
            V.cnt_off = (long long)o_cnt;
            V.pair_off = (long long)o_sp;
            V.tlist_off = (long long)o_tl;
            segs[v] = Seg{V.cap_off, V.small ? 0 : nr, (int)o_dt, (int)q_dt2};
            dt0[v] = (int)o_dt;
        }
        __syncthreads();
        if (threadIdx.x == T - 1) {
            s_c[0] += i_sp;
            s_c[1] += i_tl;
            s_c[2] += i_cnt;
            s_c[3] += i_dt;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) dt0[nv] = (int)s_c[3];
}

}  // namespace

void launch_plan_records(DevView* views, int nv, const unsigned long long* counts,
                         long long cap_records, long long cap_view, long long* h_ntemp,
                         uint32_t* err, cudaStream_t st)
{
    if (nv == 0) return;
    // one warp for a batch of <= 32 views (no block barriers), else 1024 threads
    k_plan_records<<<1, nv <= 32 ? 32 : PLT, 0, st>>>(views, nv, counts, cap_records, cap_view,
                                                      h_ntemp, err);
}

void launch_plan_bins(DevView* views, int nv, const ViewCounters* ctr, Seg* segs, int* dt0,
                      const PlanCaps& caps, ViewCounters* h_ctr, uint32_t* err, cudaStream_t st)
{
    if (nv == 0) return;
    k_plan_bins<<<1, nv <= 32 ? 32 : PLT, 0, st>>>(views, nv, ctr, segs, dt0, caps, h_ctr, err);
}

}  // namespace s3r
