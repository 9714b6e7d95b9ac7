// s3r_internal.cuh — device-side types and launch declarations of libs3r.
//
// sm_100a only.  Compiled with -fmad=false: every multiply-add that the
// R-ARITH contract writes as an FMA is an explicit __fmaf_rn; no
// other contraction happens, so the fp32 keys are reproducible bit for bit.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef __CUDACC__
#error "s3r kernels need nvcc"
#endif

namespace s3r {

constexpr int TILE = 16;                 // tile edge (reading R12)
constexpr float FLUSH_E2 = -24.0f;       // s3r_exp2(x) = 0 for x < -24 (R-ARITH flush, R14)

// Flush-ellipse culling (exact).  For a splat with exp2-form
// coefficients (qa, qb, qc), every pixel offset d = (dx, dy) with
// -(qa dx^2 + qb dx dy + qc dy^2) > CULL_TAU evaluates, in R-ARITH fp32, to
// e2 < FLUSH_E2, i.e. alpha = 0: the relative rounding error of that evaluation
// is below 6 * 2^-24 * kappa, kappa = (|qa| + |qb| + |qc|) / lambda_min, and the
// extent is only used (finite) when kappa <= CULL_KAPPA, where that error is
// <= 3.6e-3 << CULL_TAU / 24 - 1 = 5 %.  The half extents of the CULL_TAU
// ellipse (inflated by 0.1 % + 0.01 px for their own rounding) are stored in
// the sorted splat record's two .w slots; +inf disables culling for the splat.
#ifndef S3R_CULL
#define S3R_CULL 1       // build-time switch (A/B measurement); 1 is the product
#endif
constexpr float CULL_TAU = 25.2f;
constexpr float CULL_KAPPA = 1.0e4f;
// the rasterizers' warp pixel block is 8 columns x 16 rows (k_raster,
// k_raster_bwd): the stored extents include its half size, so the per-record
// test is |mean - block centre| > extent
constexpr float CULL_HALF_BX = 3.5f, CULL_HALF_BY = 7.5f;

__device__ __forceinline__ void flush_extent(float qa, float qb, float qc, float& hx, float& hy)
{
    const float a = -qa, b = -qb, c = -qc;
    const float det4 = a * c - 0.25f * b * b;
    const float h = 0.5f * (a + c);
    const float g = sqrtf(0.25f * (a - c) * (a - c) + 0.25f * b * b);
    const float lmin = det4 / (h + g);
    hx = hy = __int_as_float(0x7f800000);
    if (a > 0.0f && c > 0.0f && det4 > 0.0f && lmin > 0.0f &&
        a + fabsf(b) + c <= CULL_KAPPA * lmin) {
        hx = sqrtf(CULL_TAU * c / det4) * 1.001f + (0.01f + CULL_HALF_BX);
        hy = sqrtf(CULL_TAU * a / det4) * 1.001f + (0.01f + CULL_HALF_BY);
    }
}
constexpr int MAX_TSLOTS = 64;           // distinct times per K1 launch
constexpr int RADIX_BITS = 8;
constexpr int RADIX = 1 << RADIX_BITS;   // 256 bins per onesweep pass

// Decoupled look-back word: 2 flag bits + 30-bit count.
constexpr uint32_t LB_AGG = 1u << 30;
constexpr uint32_t LB_PRE = 2u << 30;
constexpr uint32_t LB_MASK = (1u << 30) - 1;

__device__ __forceinline__ void lb_publish(uint32_t* p, uint32_t w)
{
    *reinterpret_cast<volatile uint32_t*>(p) = w;
}

// Warp-cooperative decoupled look-back (all 32 lanes of one warp call it).
// Tiles [first, tile) precede `tile` in its chain; tile j's flag word is at
// lb[j * stride].  Each step inspects 32 predecessors at once and stops at the
// nearest inclusive prefix (LB_PRE); tiles before `first` count as a prefix of
// 0.  Returns the exclusive prefix of `tile` (identical in every lane).
__device__ __forceinline__ uint32_t warp_lookback(const uint32_t* lb, long long stride, int tile,
                                                  int first)
{
    const int lane = threadIdx.x & 31;
    uint32_t excl = 0;
    int j = tile - 1;
    while (j >= first) {
        const int jj = j - lane;
        uint32_t w = LB_PRE;
        if (jj >= first) {
            const volatile uint32_t* p = lb + (long long)jj * stride;
            do {
                w = *p;
            } while ((w >> 30) == 0);
        }
        const unsigned pre = __ballot_sync(0xffffffffu, (w & LB_PRE) != 0);
        const int last = pre ? (__ffs(pre) - 1) : 31;
        uint32_t c = (lane <= last) ? (w & LB_MASK) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        excl += c;
        if (pre) break;
        j -= 32;
    }
    return excl;
}

// Per-Gaussian flag bits (debug dump; same meaning as the header)
constexpr uint8_t F_TEMPORAL = 1, F_VISIBLE = 2, F_SMALL = 4, F_DROPPED = 8,
                  F_RENDERED = 16, F_BADID = 32, F_JITTERED = 64;

// Device error bits
constexpr uint32_t ERR_BADID = 1;
constexpr uint32_t ERR_PRECULL = 2;   // K2 pre-test culled a visible Gaussian (debug self-check)
constexpr uint32_t ERR_CAPACITY = 4;  // capacity mode: a view did not fit the reserved scratch

// Per-view descriptor in device memory (one per view of a batch).
struct DevView {
    float t;
    int W, H;
    float fx, fy, cx, cy, near_plane;
    const float* table;      // [K1][12]
    float lod_r, lod_pmax, lod_D;
    unsigned long long seed;
    float jit[3];            // NEXT-3 LOD noisy offset scale [dx, dy, dz] (0: off)
    int tslot;               // index of the view's distinct time
    int TX, TY, ntiles;
    float* rgb;
    float* depth;
    float* finalT;
    uint8_t* visible;
    // filled per phase by the host
    long long cap_off;       // offset of the view's segment in per-rendered arrays
    long long n_temporal;
    long long pair_off;      // offset of the view's supertile lists
    long long n_rendered;
    long long n_pairs;       // (tile, splat) pairs P (K2 count); capacity of the lists
    long long dbg_off;       // offset in the debug arrays (keys/flags/rect)
    // supertile binning (k_bin.cu): S = 2^sshift tiles per supertile edge
    int sshift, STX, STY, nbins, nchunks;
    int range_off;           // offset of the view's supertile ranges
    long long cnt_off;       // offset of the view's (bin, chunk) counts
    long long tlist_off;     // offset of the view's tile-list area (S*S * supertile pairs)
    int trange_off;          // offset of the view's tile ranges (ntiles entries)
    long long pix_off;       // offset of the view's pixels in the training buffers
    int small;               // a4 in one CTA (k_small.cu) instead of the sort + binning kernels
};

// Views small enough for the one-CTA depth order + tile binning (k_small.cu):
// at most SMALL_MAX rendered splats, SMALL_TILES tiles, and SMALL_WORK
// (splat, tile) containment tests.
constexpr int SMALL_MAX = 2048;
constexpr int SMALL_TILES = 1024;
constexpr long long SMALL_WORK = 1ll << 18;
__host__ __device__ inline bool small_view(long long n_rendered, int ntiles)
{
    return n_rendered <= SMALL_MAX && ntiles <= SMALL_TILES && n_rendered * ntiles <= SMALL_WORK;
}

// Per-view counters written by K2 (device, zeroed per batch)
struct ViewCounters {
    unsigned long long n_visible, n_small, n_dropped, n_rendered, n_pairs, n_bad, n_spairs;
};

// Segment of a segmented onesweep sort / scan (one per view)
struct Seg {
    long long base;          // element offset of the segment
    long long count;         // elements
    int tile0;               // first global tile of the segment
    int ntiles;              // tiles of the segment
};

// Capacity-mode limits for the device-side planner (k_plan.cu)
struct PlanCaps {
    long long rendered_view;   // splats rendered per view (count / scatter / permute grids)
    long long bin_pairs;       // supertile pairs over the batch (list buffer)
    long long tile_entries;    // tile-list area over the batch (S*S x supertile pairs)
    long long counts;          // (bin, chunk) counters over the batch
    long long bin_chunk;       // k_bin.cu KCHUNK
    long long sort_tile;       // onesweep keys per CTA
};

// ---------------- launchers (each enqueues on `st`) ----------------------

// capacity mode: device-side sizing after K1 (record segments) and after K2
// (sort segments, binning layout); see k_plan.cu
void launch_plan_records(DevView* views, int nv, const unsigned long long* counts,
                         long long cap_records, long long cap_view, long long* h_ntemp,
                         uint32_t* err, cudaStream_t st);
void launch_plan_bins(DevView* views, int nv, const ViewCounters* ctr, Seg* segs, int* dt0,
                      const PlanCaps& caps, ViewCounters* h_ctr, uint32_t* err, cudaStream_t st);

// K1: temporal filter + ordered compaction of T distinct times in groups of gs
// (<= MAX_TSLOTS) slots, one ticket per group (ticket[0 .. ceil(T / gs))) and
// look-back words lookback[slot][tile].
void launch_filter(const float2* vis, long long n, const float* d_times, int T, int gs,
                   int32_t* idx_out, long long idx_stride, unsigned long long* counts,
                   uint32_t* lookback, int* ticket, cudaStream_t st);
// slots per K1 group for a scene of n Gaussians and T distinct times: all T in
// one launch when the scene has few filter tiles, else MAX_TSLOTS per launch
int filter_groups(long long n, int T);

// Compose instance cameras (fp64, rounded once).
void launch_compose(const float* w2c, const float* i2g, int n_views, int K, float* out,
                    cudaStream_t st);

// K2: instance-specific projection + EWA + decisions + LOD + life update,
// ordered compaction of rendered splats per view.
struct ProjectArgs {
    const float4* means_opacity;
    const float4* scales;
    const float4* rotations;
    const float4* colors;
    const int32_t* ids;
    float2* life;
    int num_instances;
    long long n;
    const DevView* views;
    int n_views;
    const int32_t* tidx;         // [T][idx_stride]
    long long idx_stride;
    int max_tiles;               // grid.x: max over views of ceil(n_temporal / project_tile)
    // conventional pipeline: world-frame means / rotations per view (NULL:
    // streamlined, instance-specific cameras); every valid id uses slot 0
    const float4* world_mo;
    const float4* world_rot;
    // NeurF colour query on: per record the own-frame mean of the splat (the
    // moved one under the LOD noisy offset) and the instance id bits (NULL: off)
    float4* rec_mu;
    // outputs
    float4* rec;                 // [cap][3] splat records (compacted, unordered)
    unsigned long long* dkey;    // [cap] (depth bits << gbits) | Gaussian index
    int gbits;                   // bits of the Gaussian index in dkey
    int32_t* gidx;               // [cap] Gaussian index (debug dumps) or NULL
    ViewCounters* counters;      // [n_views]; n_rendered is the compaction cursor
    uint32_t* err;
    // debug (NULL when off)
    float* dbg_keys;
    uint8_t* dbg_flags;
    int16_t* dbg_rect;
    // no debug dumps, no rec_mu, no world copy and no LOD noisy offset in this
    // batch: the specialised K2 without those paths
    int lean;
};
void launch_project(const ProjectArgs& a, cudaStream_t st);
int project_tile();

// Conventional pipeline (NEXT-2): K0 moves every Gaussian to the world frame
// of each view's time (views[v].table slot i >= 1 = local->world pose of
// instance i), writing wmo / wrot [n_views][n]; K1 is replaced by the identity
// index list (no temporal filter).
void launch_world(const float4* mo, const float4* rot, const int32_t* ids, int num_instances,
                  long long n, const DevView* views, int n_views, float4* wmo, float4* wrot,
                  cudaStream_t st);
void launch_iota(int32_t* idx, long long n, cudaStream_t st);

// K6 NeurF colour query on the tensor cores (NEXT-4, k_neurf.cu): colours of
// the compacted records of every view, written into rec[3 o + 2].xyz.
struct NeurfArgs {
    const DevView* views;
    int n_views;
    const int* tile_off;         // [n_views] first 128-record tile of each view
    int total_tiles;
    const float4* rec_mu;        // [cap] own-frame mean + instance id bits
    float4* rec;                 // [cap][3] splat records
    const void* wpack;           // bf16 core-matrix weight tiles (neurf_pack_bytes)
    const float* bias;           // [neurf_bias_count] fp32
    const float* time_emb;       // [n_time][8]
    int n_time;
    const float* class_emb;      // [num_instances][4]
    float pos_scale;
};
size_t neurf_pack_bytes();
int neurf_bias_count();
void launch_neurf_pack(const float* w1, const float* b1, const float* w2, const float* b2,
                       const float* w3, const float* b3, void* wpack, float* bias,
                       cudaStream_t st);
void launch_neurf(const NeurfArgs& a, cudaStream_t st);

// K5 depth sort: segmented LSD radix sort of 64-bit keys (onesweep with
// decoupled look-back), digit = (key >> shift) & 255.
void launch_hist64(const unsigned long long* keys, const Seg* segs, int nsegs,
                   const int* seg_tile0, int total_tiles, int shift0, int npasses,
                   uint32_t* hist, cudaStream_t st);
void launch_hist_scan(uint32_t* hist, int nsegs, int npasses, cudaStream_t st);
// 32-bit values (vin == NULL: value = index in the segment).
void launch_onesweep64kv(const unsigned long long* kin, const uint32_t* vin,
                         unsigned long long* kout, uint32_t* vout, const Seg* segs, int nsegs,
                         const int* seg_tile0, int total_tiles, const uint32_t* digit_base,
                         int pass, int npasses, uint32_t* lookback, int* ticket, int shift,
                         cudaStream_t st);
int onesweep64_tile();
int hist_tile();

// K3: depth-ordered permute of the records (+ compact rectangles by rank).
void launch_permute(const DevView* views, int n_views, long long max_rendered,
                    const uint32_t* order, const float4* rec, float4* rec_sorted,
                    uint2* rect_sorted, cudaStream_t st);
// K4: stable counting sort of (supertile, rank) pairs: count, scan, scatter.
int bin_chunk();
constexpr int MAX_BINS = 1024;   // supertiles per view (S grows for huge images)
// ... then K4 expand: per-tile lists (ranks) + tile ranges from the supertile lists.
void launch_bin(const DevView* views, int n_views, int max_chunks, int max_bins,
                const uint2* rect_sorted, uint32_t* cnt, int2* ranges, uint32_t* lists,
                uint32_t* tlists, int2* tranges, cudaStream_t st);
// Debug: the per-tile lists of view vi as (tile, Gaussian) pairs + [start,end) ranges.
// a4 of the small views of a batch in one CTA each (k_small.cu).  With
// sp.ctr set (capacity mode, every view small by reservation) each CTA also
// plans its view from K2's counters, in place of k_plan_bins.
struct SmallPlan {
    const ViewCounters* ctr = nullptr;
    ViewCounters* h_ctr = nullptr;          // mapped copy for s3r_get_stats
    uint32_t* err = nullptr;
    long long cap_rendered = 0;
};
void launch_small_sortbin(DevView* views, int n_views, const unsigned long long* dkey,
                          const float4* rec, unsigned long long* keys_out, uint32_t* order_out,
                          float4* rec_sorted, uint2* rect_sorted, uint32_t* tlists,
                          int2* tranges, const SmallPlan& sp, cudaStream_t st);
void launch_dbg_tile_pairs(const DevView* views, int vi, int ntiles, const uint32_t* tlists,
                           const int2* tranges, const uint32_t* toff, const uint32_t* order,
                           const int32_t* gidx, int32_t* tile_out, int32_t* gauss_out,
                           int32_t* ranges_out, cudaStream_t st);

// K7: rasterizer.
struct RasterArgs {
    const DevView* views;
    int n_views;
    int max_tiles;
    const int2* tranges;         // tile ranges, per view at V.trange_off
    const uint32_t* tlists;      // tile lists of depth ranks, per view at V.tlist_off
    const float4* rec_sorted;    // splat records by rank, per view at V.cap_off
    unsigned long long* evals;   // [n_views][2] (E_alg, E_exec) or NULL
    float* train_T;              // per pixel final T (training) or NULL, at V.pix_off
    int* train_n;                // per pixel blended list entries (training), at V.pix_off
    float exp2_c0;               // 1.3264695880934596e-3f (set by launch_raster)
    int fast_exp;                // 1: SFU ex2.approx instead of R-ARITH (not for training)
};
void launch_raster(const RasterArgs& a, cudaStream_t st);

// Config 5: backward of K7 and K2.
struct s3r_cot {
    const float* rgb;
    const float* depth;
    const float* final_T;
};
struct BackwardArgs {
    const DevView* views;
    int n_views;
    const s3r_cot* cots;                 // [n_views]
    const int2* tranges;
    const uint32_t* tlists;
    const float4* rec_sorted;
    const float* train_T;
    const int* train_n;
    float* splat_grads;                  // [cap][splat_grad_stride()] per depth rank (10 used)
    const unsigned long long* dkey_sorted;
    unsigned long long gmask;            // (1 << gbits) - 1
    const int32_t* ids;
    const float4* means_opacity;
    const float4* scales;
    const float4* rotations;
    float* g_means;
    float* g_scales;
    float* g_rot;
    float* g_colors;
    float* g_table;                      // [n_views][num_instances][12] or NULL (pose gradient)
    int num_instances;
    int smem_table;                      // accumulate g_table per CTA in shared memory
    int has_depth_cot, has_T_cot;        // some view has a depth / final_T cotangent
    const float4* rec_mu;                // [cap] moved own-frame means (noisy offset) or NULL
    const uint32_t* order;               // [cap] depth rank -> compacted slot
};
void launch_backward(const BackwardArgs& a, int max_tiles, long long max_rendered, cudaStream_t st);
void launch_mse(const float* x, const float* y, long long n, float scale, float* grad,
                float* loss, cudaStream_t st);

// K9: commit / reset.
void launch_commit(float2* vis, float2* life, long long n, float margin, cudaStream_t st);

// bytes (a multiple of 4) from device memory into mapped page-locked host
// memory (cudaHostAlloc under unified addressing), by a kernel
void launch_readback(void* host_mapped, const void* dev, size_t bytes, cudaStream_t st);
void launch_reset(float2* vis, long long n, cudaStream_t st);
void launch_life_flip(float2* life, long long n, cudaStream_t st);

// Debug helpers.
void launch_dump_order(const uint32_t* order, const int32_t* gidx, long long base,
                       long long count, int32_t* out, cudaStream_t st);

}  // namespace s3r
