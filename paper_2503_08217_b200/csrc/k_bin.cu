// k_bin.cu — a4 tile binning: depth-ordered permute (K3) and a stable
// counting sort of (supertile, depth rank) pairs (K4 count / scan / scatter),
// plus the debug expansion of supertile lists into per-tile lists.
//
// Reading R11/R12: every pixel of a 16x16 tile blends, in (depth,
// index) order, the rendered Gaussians whose tile rectangle contains the tile.
// After the depth sort (K5a) the splats of a view sit in rank order r.  Instead
// of materialising one (tile, r) pair per covered tile and radix-sorting them
// (3DGS practice; ~28 pairs per splat here), the splats are binned by SUPERTILE
// (S x S tiles, S = 4 unless the image needs more): each splat emits one pair
// per supertile its rectangle touches (~5x fewer pairs), written directly to its
// final position by a stable counting sort whose single digit is the supertile
// id (one pass: count per (chunk, bin), exclusive scan in (bin, chunk) order,
// scatter in rank order).  The rasterizer (K7) walks its supertile's list in
// order and keeps the entries whose rectangle contains its tile, which yields
// exactly the per-tile list of R11/R12 — the debug dump below materialises it.
#include "s3r_internal.cuh"

namespace s3r {

namespace {

constexpr int KT = 256;          // threads of the bin kernels
constexpr int KCHUNK = 1024;     // splats (ranks) per chunk / CTA
constexpr int KWARPS = KT / 32;
constexpr int KWCHUNK = KCHUNK / KWARPS;   // 128 ranks per warp in the scatter

__device__ __forceinline__ void rect_of(uint2 rr, int& tx0, int& tx1, int& ty0, int& ty1)
{
    tx0 = rr.x & 0xffff; tx1 = rr.x >> 16; ty0 = rr.y & 0xffff; ty1 = rr.y >> 16;
}

// 16-bit mask of the tiles of 4 x 4 supertile (sbx, sby) that the tile
// rectangle [tx0, tx1] x [ty0, ty1] contains (bit 4 ly + lx)
__device__ __forceinline__ uint32_t tile_mask4(int tx0, int tx1, int ty0, int ty1, int sbx, int sby)
{
    const int lx0 = max(tx0 - 4 * sbx, 0), lx1 = min(tx1 - 4 * sbx, 3);
    const int ly0 = max(ty0 - 4 * sby, 0), ly1 = min(ty1 - 4 * sby, 3);
    const uint32_t xm = (2u << lx1) - (1u << lx0);                    // bits lx0..lx1
    const uint32_t ym = ((1u << (4 * ly1 + 4)) - (1u << (4 * ly0))) & 0x1111u;
    return xm * ym;                                                   // no carries: xm < 16
}

// ------------------------------------------------------------------ K3 permute
// rec_sorted[r] = rec[order[r]] and rect_sorted[r] = its tile rectangle.
__global__ void __launch_bounds__(256) k_permute(const DevView* __restrict__ views,
                                                 const uint32_t* __restrict__ order,
                                                 const float4* __restrict__ rec,
                                                 float4* __restrict__ rec_sorted,
                                                 uint2* __restrict__ rect_sorted)
{
    const DevView& V = views[blockIdx.y];
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (V.small || r >= V.n_rendered) return;      // small views: k_small.cu
    const long long base = V.cap_off;
    const uint32_t j = order[base + r];
    const float4* src = rec + 3 * (base + j);
    const float4 q0 = src[0];
    float4 q1 = src[1], q2 = src[2];
    rect_sorted[base + r] = make_uint2(__float_as_uint(q1.w), __float_as_uint(q2.w));
    // the rasterizers read the flush-ellipse half extents where the rectangle was
    flush_extent(q1.x, q1.y, q1.z, q1.w, q2.w);
    float4* dst = rec_sorted + 3 * (base + r);
    dst[0] = q0;
    dst[1] = q1;
    dst[2] = q2;
}

// ------------------------------------------------------------------ K4 count
// cnt[view][bin][chunk] = number of (bin, r) pairs of chunk `chunk`.
__global__ void __launch_bounds__(KT) k_bin_count(const DevView* __restrict__ views,
                                                  const uint2* __restrict__ rect_sorted,
                                                  uint32_t* __restrict__ cnt)
{
    extern __shared__ uint32_t s_cnt[];        // [nbins]
    const DevView& V = views[blockIdx.y];
    const int c = blockIdx.x;
    const long long r0 = (long long)c * KCHUNK;
    if (V.small || r0 >= V.n_rendered || V.nbins == 0) return;
    const int nb = V.nbins, sh = V.sshift, sx = V.STX;
    for (int b = threadIdx.x; b < nb; b += KT) s_cnt[b] = 0;
    __syncthreads();
    const long long r1 = min((long long)KCHUNK, V.n_rendered - r0);
    for (int i = threadIdx.x; i < r1; i += KT) {
        int tx0, tx1, ty0, ty1;
        rect_of(rect_sorted[V.cap_off + r0 + i], tx0, tx1, ty0, ty1);
        for (int by = ty0 >> sh; by <= (ty1 >> sh); ++by)
            for (int bx = tx0 >> sh; bx <= (tx1 >> sh); ++bx) atomicAdd(&s_cnt[by * sx + bx], 1u);
    }
    __syncthreads();
    uint32_t* out = cnt + V.cnt_off;
    for (int b = threadIdx.x; b < nb; b += KT) out[(long long)b * V.nchunks + c] = s_cnt[b];
}

// ------------------------------------------------------------------ K4 scan
// One CTA per view: exclusive scan of cnt in (bin, chunk) order; bin ranges.
// Tiles of 1024 x SCAN_SB elements go through shared memory: coalesced loads,
// each thread scans SCAN_SB contiguous elements (padded index: no bank
// conflicts), one block scan of the 1024 partial sums, coalesced stores.
// (A per-thread contiguous run over global memory was L1-sector bound: 122 us
// on C3; one barrier round per 1024 elements: 310 us.)
constexpr int SCAN_SB = 8;
__device__ __forceinline__ int scan_pad(int p) { return p + (p >> 5); }
__global__ void __launch_bounds__(1024) k_bin_scan(const DevView* __restrict__ views,
                                                   uint32_t* __restrict__ cnt,
                                                   int2* __restrict__ ranges)
{
    __shared__ uint32_t s_tile[1024 * SCAN_SB + 1024 * SCAN_SB / 32];
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_carry;
    const DevView& V = views[blockIdx.x];
    if (V.small) return;
    const long long n = (long long)V.nbins * V.nchunks;
    uint32_t* a = cnt + V.cnt_off;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_carry = 0;
    for (long long base = 0; base < n; base += 1024 * SCAN_SB) {
#pragma unroll
        for (int k = 0; k < SCAN_SB; ++k) {
            const long long i = base + k * 1024 + tid;
            s_tile[scan_pad(k * 1024 + tid)] = i < n ? a[i] : 0u;
        }
        __syncthreads();
        uint32_t x[SCAN_SB], sum = 0;
#pragma unroll
        for (int k = 0; k < SCAN_SB; ++k) {
            x[k] = s_tile[scan_pad(tid * SCAN_SB + k)];
            sum += x[k];
        }
        uint32_t v = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane == 31) s_warp[warp] = v;
        __syncthreads();
        if (warp == 0) {
            const uint32_t w = s_warp[lane];
            uint32_t ww = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, ww, o);
                if (lane >= o) ww += y;
            }
            s_warp[lane] = ww - w;
        }
        __syncthreads();
        uint32_t run = s_carry + s_warp[warp] + v - sum;
#pragma unroll
        for (int k = 0; k < SCAN_SB; ++k) {
            s_tile[scan_pad(tid * SCAN_SB + k)] = run;
            run += x[k];
        }
        __syncthreads();
        if (tid == 1023) s_carry = run;          // carry into the next tile
#pragma unroll
        for (int k = 0; k < SCAN_SB; ++k) {
            const long long i = base + k * 1024 + tid;
            if (i < n) a[i] = s_tile[scan_pad(k * 1024 + tid)];
        }
        __syncthreads();
    }
    // bin ranges: [first of bin b, first of bin b+1)
    const uint32_t total = s_carry;
    int2* R = ranges + V.range_off;
    for (int b = tid; b < V.nbins; b += 1024) {
        if (V.nchunks == 0) {           // nothing rendered in this view
            R[b] = make_int2(0, 0);
            continue;
        }
        const uint32_t s = a[(long long)b * V.nchunks];
        const uint32_t e = (b + 1 < V.nbins) ? a[(long long)(b + 1) * V.nchunks] : total;
        R[b] = make_int2((int)s, (int)e);
    }
}

// ------------------------------------------------------------------ K4 expand
// One CTA per (supertile, view) walks the supertile's list XT entries at a
// time and appends each entry to the lists of the supertile's tiles its
// rectangle contains, in list order (ballot + popc).  Tile t (local index in
// the supertile, S*S of them) owns [S*S*start + t*len, +len) of the view's
// tile-list area, len = supertile list length, so no count pass is needed.
// 4 x 4 supertiles (the product case) use per-entry tile masks (below); a
// larger S (huge images) stages the entries in shared memory and gives each
// warp a set of tiles.
#ifndef S3R_XMASK
#define S3R_XMASK 1    // 4 x 4 supertiles: per-entry tile masks + 16 ballots (A/B, bin stage with the
                       // ballots staged through shared memory and predicated stores: C3 0.957 -> 0.880 ms,
                       // C2 0.390 -> 0.352 ms against per-tile lane-select counts and branches)
#endif
#ifndef S3R_XPREF
#define S3R_XPREF 1    // expansion: next round's entry + rectangle loaded one round ahead
#endif
#ifndef S3R_XT
#define S3R_XT 128     // A/B (mask expansion): bin 1.025 ms vs 1.059 at 256
#endif
constexpr int XT = S3R_XT;
__global__ void __launch_bounds__(XT) k_bin_expand(const DevView* __restrict__ views,
                                                   const uint2* __restrict__ rect_sorted,
                                                   const uint32_t* __restrict__ lists,
                                                   const int2* __restrict__ ranges,
                                                   uint32_t* __restrict__ tlists,
                                                   int2* __restrict__ tranges)
{
    __shared__ uint32_t s_r[XT];
    __shared__ uint2 s_rect[XT];
    const DevView& V = views[blockIdx.y];
    const int b = blockIdx.x;
    if (V.small || b >= V.nbins) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = 1 << V.sshift, SS = S * S;
    const int bx = b % V.STX, by = b / V.STX;
    const int2 rg = ranges[V.range_off + b];
    const int len = rg.y - rg.x;
    const uint32_t* lst = lists + V.pair_off;
    const uint2* rects = rect_sorted + V.cap_off;
    uint32_t* out = tlists + V.tlist_off + (long long)SS * rg.x;
    // running count of each tile's list (tile t is owned by warp t % 16)
    __shared__ int s_tcnt[MAX_BINS];              // S*S <= MAX_BINS tiles per supertile
    for (int t = tid; t < SS; t += XT) s_tcnt[t] = 0;
    __syncthreads();
#if S3R_XMASK
    if (V.sshift == 2) {
        // 4 x 4 supertile: each thread takes one entry and forms the 16-bit mask
        // of the supertile's tiles its rectangle contains (tile t = 4 ty + tx
        // local); per tile one ballot gives the warp's members in list order.
        // The warp's 16 ballots go to shared memory once (lane t then counts
        // tile t), per-warp counts order the warps, and each tile's members are
        // stored with a predicated store at base + rank within the warp.
        __shared__ int s_wc[XT / 32][16];
        __shared__ __align__(16) unsigned s_bal[XT / 32][16];
        const unsigned lt = (1u << lane) - 1u;
#if S3R_XPREF
        // the next round's entry and rectangle are loaded while this round's
        // are expanded (two dependent loads per round otherwise exposed)
        uint32_t r_nx = 0;
        uint2 rr_nx = make_uint2(0u, 0u);
        if (rg.x + tid < rg.y) {
            r_nx = lst[rg.x + tid];
            rr_nx = rects[r_nx];
        }
#endif
        for (int base = rg.x; base < rg.y; base += XT) {
            const int e = base + tid;
            uint32_t r = 0, m = 0;
#if S3R_XPREF
            const uint2 rr = rr_nx;
            r = r_nx;
            if (e + XT < rg.y) {
                r_nx = lst[e + XT];
                rr_nx = rects[r_nx];
            }
            if (e < rg.y) {
                int tx0, tx1, ty0, ty1;
                rect_of(rr, tx0, tx1, ty0, ty1);
                m = tile_mask4(tx0, tx1, ty0, ty1, bx, by);
            }
#else
            if (e < rg.y) {
                r = lst[e];
                int tx0, tx1, ty0, ty1;
                rect_of(rects[r], tx0, tx1, ty0, ty1);
                m = tile_mask4(tx0, tx1, ty0, ty1, bx, by);
            }
#endif
            unsigned bal[16];
#pragma unroll
            for (int t = 0; t < 16; ++t)     // one bit test + one vote per tile
                asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 x;\n\tand.b32 x, %1, %2;\n\t"
                             "setp.ne.b32 p, x, 0;\n\tvote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
                             : "=r"(bal[t]) : "r"(m), "r"(1u << t));
            if (lane == 0) {
#pragma unroll
                for (int t = 0; t < 16; t += 4)
                    *reinterpret_cast<uint4*>(&s_bal[warp][t]) =
                        make_uint4(bal[t], bal[t + 1], bal[t + 2], bal[t + 3]);
            }
            __syncwarp();
            if (lane < 16) s_wc[warp][lane] = __popc(s_bal[warp][lane]);
            __syncthreads();
            // lane t < 16: tile t's list position for this warp's members
            uint32_t myoff = 0;
            int mytot = 0;
            if (lane < 16) {
                int o = s_tcnt[lane];
#pragma unroll
                for (int w = 0; w < XT / 32; ++w) {
                    const int c = s_wc[w][lane];
                    if (w < warp) o += c;
                    mytot += c;
                }
                myoff = (uint32_t)(lane * len + o);
            }
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const uint32_t off = __shfl_sync(0xffffffffu, myoff, t);
                const uint32_t pos = off + __popc(bal[t] & lt);
                // out[pos] = r if the entry has tile t (one wide multiply-add for
                // the address, one predicated store)
                asm volatile("{\n\t.reg .pred q;\n\t.reg .b32 x;\n\t.reg .b64 a;\n\t"
                             "and.b32 x, %3, %4;\n\tsetp.ne.b32 q, x, 0;\n\t"
                             "mad.wide.u32 a, %1, 4, %0;\n\t@q st.global.b32 [a], %2;\n\t}"
                             ::"l"(out), "r"(pos), "r"(r), "r"(m), "r"(1u << t) : "memory");
            }
            __syncthreads();
            if (warp == 0 && lane < 16) s_tcnt[lane] += mytot;
            __syncthreads();
        }
    } else
#endif
    {
    for (int base = rg.x; base < rg.y; base += XT) {
        const int n = min(XT, rg.y - base);
        if (tid < n) {
            const uint32_t r = lst[base + tid];
            s_r[tid] = r;
            s_rect[tid] = rects[r];
        }
        __syncthreads();
        for (int t = warp; t < SS; t += XT / 32) {
            const int tx = bx * S + (t % S), ty = by * S + (t / S);
            if (tx >= V.TX || ty >= V.TY) continue;
            int c = s_tcnt[t];
            for (int k = 0; k < n; k += 32) {
                const int e = k + lane;
                bool pass = false;
                if (e < n) {
                    const uint2 rr = s_rect[e];
                    pass = tx >= (int)(rr.x & 0xffff) && tx <= (int)(rr.x >> 16) &&
                           ty >= (int)(rr.y & 0xffff) && ty <= (int)(rr.y >> 16);
                }
                const unsigned bal = __ballot_sync(0xffffffffu, pass);
                if (pass) out[(long long)t * len + c + __popc(bal & ((1u << lane) - 1u))] = s_r[e];
                c += __popc(bal);
            }
            __syncwarp();
            if (lane == 0) s_tcnt[t] = c;
        }
        __syncthreads();
    }
    }
    for (int t = tid; t < SS; t += XT) {
        const int tx = bx * S + (t % S), ty = by * S + (t / S);
        if (tx >= V.TX || ty >= V.TY) continue;
        const long long s0 = (long long)SS * rg.x + (long long)t * len;
        tranges[V.trange_off + ty * V.TX + tx] = make_int2((int)s0, (int)(s0 + s_tcnt[t]));
    }
}

// ------------------------------------------------------------------ K4 scatter
#ifndef S3R_SCAT_SMALL
#define S3R_SCAT_SMALL 16   // a splat with more bins is taken by the whole warp
#endif
constexpr int SCAT_SMALL = S3R_SCAT_SMALL;
// Writes every (bin, r) pair's rank r at its final position.  Stability: a
// chunk's pairs for one bin follow the chunk's scanned base; inside the chunk
// warp w's pairs follow warps < w (per-warp counts, scanned in shared memory);
// inside a warp the splats are taken 32 at a time, one per lane (lane order =
// rank order).  Each (splat, bin) ORs the splat's lane bit into the warp's
// mask of the bin; a pair's position is the bin's running count + the number
// of lower lanes in the mask; the highest lane of a mask then advances the
// running count and clears the mask.  A splat with at most SCAT_SMALL bins
// walks its own bins (<= SCAT_SMALL iterations per lane); a larger one is taken
// by the whole warp, lanes over its bins, so the few big splats of a view (C3:
// 3.9 supertiles per splat on average, tails of 100+) do not serialise the warp.
// (A/B, bin stage, against a per-view choice between this lane-per-splat form
// without the big-splat path and a warp-per-splat form: C3 0.877 -> 0.822 ms,
// C4 5.18 -> 4.21 ms, C2 0.352 -> 0.299 ms; SCAT_SMALL 8 / 24 / 32 within 1 %.)
__global__ void __launch_bounds__(KT) k_bin_scatter(const DevView* __restrict__ views,
                                                    const uint2* __restrict__ rect_sorted,
                                                    const uint32_t* __restrict__ cnt,
                                                    uint32_t* __restrict__ lists)
{
    extern __shared__ uint32_t s_dyn[];
    const DevView& V = views[blockIdx.y];
    const int c = blockIdx.x;
    const long long r0 = (long long)c * KCHUNK;
    if (V.small || r0 >= V.n_rendered || V.nbins == 0) return;
    const int nb = V.nbins, sh = V.sshift, sx = V.STX;
    uint32_t* s_base = s_dyn;                                    // [nb] chunk base per bin
    uint32_t* s_w = s_dyn + nb;                                  // [KWARPS][nb] counts, then [KWARPS][nb] masks
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 2 * KWARPS * nb; i += KT) s_w[i] = 0;
    for (int b = tid; b < nb; b += KT) s_base[b] = cnt[V.cnt_off + (long long)b * V.nchunks + c];
    __syncthreads();
    const long long n_r = V.n_rendered;
    const long long wr0 = r0 + (long long)warp * KWCHUNK;
    const int wn = (int)max(0ll, min((long long)KWCHUNK, n_r - wr0));
    // per-warp counts
    uint32_t* mine = s_w + warp * nb;
    for (int i = lane; i < wn; i += 32) {
        int tx0, tx1, ty0, ty1;
        rect_of(rect_sorted[V.cap_off + wr0 + i], tx0, tx1, ty0, ty1);
        for (int by = ty0 >> sh; by <= (ty1 >> sh); ++by)
            for (int bx = tx0 >> sh; bx <= (tx1 >> sh); ++bx)
                atomicAdd(&mine[by * sx + bx], 1u);
    }
    __syncthreads();
    // exclusive scan across warps, per bin
    for (int b = tid; b < nb; b += KT) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < KWARPS; ++w) {
            const uint32_t t = s_w[w * nb + b];
            s_w[w * nb + b] = run;
            run += t;
        }
    }
    __syncthreads();
    uint32_t* out = lists + V.pair_off;
    uint32_t* wmask = s_w + KWARPS * nb + warp * nb;          // zeroed above
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < wn; base += 32) {
        const int i = base + lane;
        int bx0 = 0, bx1 = -1, by0 = 0, by1 = -1;
        if (i < wn) {
            int tx0, tx1, ty0, ty1;
            rect_of(rect_sorted[V.cap_off + wr0 + i], tx0, tx1, ty0, ty1);
            bx0 = tx0 >> sh; bx1 = tx1 >> sh; by0 = ty0 >> sh; by1 = ty1 >> sh;
        }
        const int bw = bx1 - bx0 + 1, nbin = bw * (by1 - by0 + 1);
        const bool big = nbin > SCAT_SMALL;
        const unsigned bigm = __ballot_sync(0xffffffffu, big);
        const int n_own = big ? 0 : nbin;
        const uint32_t rr = (uint32_t)(wr0 + i);
        // the bins of each big splat L of the warp, lanes over them
        auto big_bins = [&](auto&& f) {
            for (unsigned m = bigm; m; m &= m - 1) {
                const int L = __ffs(m) - 1;
                const int Lbx0 = __shfl_sync(0xffffffffu, bx0, L), Lby0 = __shfl_sync(0xffffffffu, by0, L);
                const int Lbw = __shfl_sync(0xffffffffu, bw, L), Ln = __shfl_sync(0xffffffffu, nbin, L);
                const uint32_t Lr = __shfl_sync(0xffffffffu, rr, L);
                for (int k = lane; k < Ln; k += 32) {
                    const int yy = k / Lbw, xx = k - yy * Lbw;
                    f(L, (Lby0 + yy) * sx + Lbx0 + xx, Lr);
                }
            }
        };
        // the lane's own bins (a small splat), row-major in its rectangle
        auto own_bins = [&](auto&& f) {
            int xx = 0, yy = 0;
            for (int k = 0; k < n_own; ++k) {
                f((by0 + yy) * sx + bx0 + xx);
                if (++xx == bw) { xx = 0; ++yy; }
            }
        };
        own_bins([&](int b) { atomicOr(&wmask[b], 1u << lane); });
        big_bins([&](int L, int b, uint32_t) { atomicOr(&wmask[b], 1u << L); });
        __syncwarp();
        own_bins([&](int b) { out[s_base[b] + mine[b] + __popc(wmask[b] & lt)] = rr; });
        big_bins([&](int L, int b, uint32_t Lr) {
            out[s_base[b] + mine[b] + __popc(wmask[b] & ((1u << L) - 1u))] = Lr;
        });
        __syncwarp();
        // the highest member of a mask advances the bin's count (a lower member
        // that reads the mask after it was cleared sees 0: not the highest)
        own_bins([&](int b) {
            const uint32_t m = wmask[b];
            if (lane == 31 - __clz(m)) {
                mine[b] += __popc(m);
                wmask[b] = 0u;
            }
        });
        big_bins([&](int L, int b, uint32_t) {
            const uint32_t m = wmask[b];
            if (L == 31 - __clz(m)) {
                mine[b] += __popc(m);
                wmask[b] = 0u;
            }
        });
        __syncwarp();
    }
}

// ------------------------------------------------------------------ debug
// The per-tile lists of view vi packed in tile order as (tile, Gaussian) pairs
// ((tile, depth, index) order) with [start, end) ranges; toff = exclusive scan
// of the tile list lengths.
__global__ void k_dbg_tile_pairs(const DevView* __restrict__ views, int vi,
                                 const uint32_t* __restrict__ tlists,
                                 const int2* __restrict__ tranges, const uint32_t* __restrict__ toff,
                                 const uint32_t* __restrict__ order, const int32_t* __restrict__ gidx,
                                 int32_t* __restrict__ tile_out, int32_t* __restrict__ gauss_out,
                                 int32_t* __restrict__ ranges_out)
{
    const DevView& V = views[vi];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= V.ntiles) return;
    const int2 rg = tranges[V.trange_off + t];
    const uint32_t o0 = toff[t];
    for (int i = rg.x; i < rg.y; ++i) {
        const uint32_t r = tlists[V.tlist_off + i];
        const uint32_t o = o0 + (uint32_t)(i - rg.x);
        if (tile_out) tile_out[o] = t;
        if (gauss_out) gauss_out[o] = gidx[V.cap_off + order[V.cap_off + r]];
    }
    if (ranges_out) {
        ranges_out[2 * t] = (int32_t)o0;
        ranges_out[2 * t + 1] = (int32_t)(o0 + (uint32_t)(rg.y - rg.x));
    }
}

}  // namespace

int bin_chunk() { return KCHUNK; }

void launch_permute(const DevView* views, int n_views, long long max_rendered,
                    const uint32_t* order, const float4* rec, float4* rec_sorted,
                    uint2* rect_sorted, cudaStream_t st)
{
    if (n_views == 0 || max_rendered == 0) return;
    dim3 grid((unsigned)((max_rendered + 255) / 256), n_views);
    k_permute<<<grid, 256, 0, st>>>(views, order, rec, rec_sorted, rect_sorted);
}

void launch_bin(const DevView* views, int n_views, int max_chunks, int max_bins,
                const uint2* rect_sorted, uint32_t* cnt, int2* ranges, uint32_t* lists,
                uint32_t* tlists, int2* tranges, cudaStream_t st)
{
    if (n_views == 0) return;
    dim3 grid(max_chunks, n_views);
    if (max_chunks) k_bin_count<<<grid, KT, (size_t)max_bins * 4, st>>>(views, rect_sorted, cnt);
    k_bin_scan<<<n_views, 1024, 0, st>>>(views, cnt, ranges);
    if (max_chunks) {
        const size_t smem = (size_t)max_bins * 4 * (1 + 2 * KWARPS);
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_bin_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_bin_scatter<<<grid, KT, smem, st>>>(views, rect_sorted, cnt, lists);
    }
    k_bin_expand<<<dim3(max_bins, n_views), XT, 0, st>>>(views, rect_sorted, lists, ranges, tlists,
                                                       tranges);
}

void launch_dbg_tile_pairs(const DevView* views, int vi, int ntiles, const uint32_t* tlists,
                           const int2* tranges, const uint32_t* toff, const uint32_t* order,
                           const int32_t* gidx, int32_t* tile_out, int32_t* gauss_out,
                           int32_t* ranges_out, cudaStream_t st)
{
    if (ntiles == 0) return;
    k_dbg_tile_pairs<<<(unsigned)((ntiles + 127) / 128), 128, 0, st>>>(
        views, vi, tlists, tranges, toff, order, gidx, tile_out, gauss_out, ranges_out);
}

}  // namespace s3r
