/*
 * s3r.h — C ABI of the B200-native S3R-GS streamlined per-view splatting path.
 *
 * The library (paper_2503_08217_b200/libs3r.so, CUDA for sm_100a) renders
 * batches of camera views of one Gaussian scene through the pipeline of
 * PAPER.md §3.3 (arxiv 2503.08217, "Streamlined Reconstruction Stage",
 * P:148-199; Fig.1b):
 *
 *   temporal-visibility filter          -> s3r_render_batch, stage K1
 *   instance-specific projection (Eq.1)  -> stage K2
 *   Adaptive-LOD cull (Eq.7 rows 1-3)    -> stage K2
 *   tile binning + depth sort                       -> stages K3-K6
 *   alpha-blended tile rasterization (Eq.2)  -> stage K7
 *   point-life update with M_t (Eq.5)    -> stage K2 (atomics)
 *   visibility commit / reset (Eq.6)     -> s3r_commit_visibility,
 *                                                      s3r_reset_visibility
 * and the rows SURVEY.md §8(f) marks next:
 *   backward of blend + projection, pose gradient   -> s3r_render_backward,
 *     (config 5)                            s3r_mse, s3r_set_training
 *   conventional pipeline (Fig.1a)             -> s3r_set_pipeline
 *   LOD noisy offset (Eq.7 row 4)            -> s3r_set_lod_jitter
 *   NeurF colour query (Eq.7 rows 5-6)       -> s3r_set_neural_colors
 *
 * "P:n" = line n of /root/reference/PAPER.md.  The arithmetic is the fp32
 * contract "R-ARITH" of DESIGN.md; readings of the paper (R1-R23) are listed
 * there.
 *
 * Conventions for every call:
 *  - Plain C types only.  "device" pointers are CUDA device (or managed)
 *    memory of the context's device; "host" pointers are CPU memory.
 *  - All scene, view and output memory is CALLER-OWNED.  The context owns only
 *    scratch, grown on demand and reused; no caller pointer is retained after a
 *    call returns.
 *  - Calls enqueue work on `stream` (a cudaStream_t, NULL = legacy default
 *    stream) and return.  By default s3r_render / s3r_render_batch synchronise
 *    the stream twice internally to size scratch exactly (after K1 and after
 *    K2); in the capacity mode (s3r_set_capacity) they do not synchronise at
 *    all and can be captured in a CUDA graph.  s3r_check,
 *    s3r_get_stage_times and s3r_render_batch_host synchronise it fully.
 *  - Return value: S3R_OK (0) or a negative S3R_E* code; the message is in
 *    s3r_last_error(ctx).  Nothing throws or aborts across the ABI.
 *  - A context is bound to one device and must not be used from two threads
 *    at once.
 */
#ifndef S3R_H
#define S3R_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define S3R_VERSION 10100 /* 1.1.0 */
#define S3R_TILE 16       /* tile edge in pixels (reading R12) */

enum {
    S3R_OK = 0,
    S3R_EINVAL = -1,    /* bad argument: NULL required pointer, misaligned
                           pointer, n < 0, width/height outside [1,16384],
                           fx/fy <= 0 or non-finite, t outside [-1,1] or NaN,
                           num_instances < 1, non-finite LOD parameters,
                           lod_pmax outside [0,1], lod_D <= 0, near_plane <= 0,
                           n_views < 0                                        */
    S3R_EINSTANCE = -2, /* a Gaussian carried an instance id outside
                           [0, num_instances-1]; it was treated as invisible
                           ("ID in Z"); reported by s3r_check          */
    S3R_ENOMEM = -3,    /* scratch allocation failed                          */
    S3R_ECUDA = -4,     /* a CUDA runtime error; see s3r_last_error           */
    S3R_ESTATE = -5,    /* call out of order (e.g. dump without a render, or
                           debug data requested without s3r_set_debug)        */
    S3R_EINTERNAL = -6, /* an internal self-check failed (with s3r_set_debug
                           on: K2's conservative frustum pre-test culled a
                           Gaussian the exact test found visible); reported
                           by s3r_check; a library bug, never expected        */
    S3R_ECAPACITY = -7  /* capacity mode (s3r_set_capacity): a view of a batch
                           did not fit the reserved scratch and was rendered
                           empty (black, final T = 1); reported by s3r_check */
};

typedef struct s3r_ctx s3r_ctx;

/* The Gaussian scene ("each Gaussian is assigned a 3D position mu, a 3D
 * covariance Sigma, an opacity alpha, a temporal visibility v and a point life
 * l ... dynamic Gaussian is associated with an instance ID").  Structure of
 * arrays, one element per Gaussian, all DEVICE pointers, 16-byte aligned.   */
typedef struct {
    int64_t n;                   /* number of Gaussians, 0 <= n < 2^30          */
    int32_t num_instances;       /* K+1: id 0 = static background, 1..K objects */
    const float* means_opacity;  /* float4[n]: mu (x,y,z) in the local frame of
                                    its instance (world frame for id 0), opacity
                                    in (0,1)                                    */
    const float* scales;         /* float4[n]: sigma_x, sigma_y, sigma_z (> 0,
                                    linear metres; activation is the caller's),
                                    .w ignored                                  */
    const float* rotations;      /* float4[n]: quaternion (w,x,y,z), non-zero,
                                    normalised inside the kernel                */
    const float* colors;         /* float4[n]: r,g,b (constant per Gaussian,
                                    reading R16), .w ignored                    */
    const int32_t* instance_ids; /* int32[n]                                    */
    float* visibility;           /* float2[n]: (v_s, v_e) temporal visibility;
                                    read by render, written by commit/reset     */
    float* life;                 /* float2[n]: (l_s, l_e) point life; updated by
                                    render with atomics (Eq.5); NULL = no update */
} s3r_scene;

/* One camera view at time t ("at each time t rendering").            */
typedef struct {
    float t;                     /* normalised time in [-1,1]; -0 is
                                    treated as +0                               */
    int32_t width, height;       /* image size in pixels, [1, 16384]            */
    float fx, fy, cx, cy;        /* pinhole intrinsics K_t (pixels)             */
    float near_plane;            /* camera-z near plane, > 0 (0.01 m, R5)       */
    const float* instance_w2c;   /* DEVICE float[num_instances][12]: row-major
                                    3x4 [R|t] local->camera, slot 0 = W_t, slot
                                    i = W_t W_{t,i2g}.  Build it with
                                    s3r_compose_instance_cameras.               */
    float lod_r;                 /* LOD threshold r in pixels ("such as 4
                                    pixels"); <= 0 disables LOD                 */
    float lod_pmax;              /* p_max in [0,1] (Eq.7)                       */
    float lod_D;                 /* D > 0 in metres (Eq.7)                      */
    uint64_t lod_seed;           /* per-view seed of the Bernoulli draw (R9)    */
} s3r_view;

/* Per-view outputs, DEVICE pointers, caller-allocated.  rgb is required.    */
typedef struct {
    float* rgb;                  /* float[height][width][3], Eq.2 colour       */
    float* depth;                /* float[height][width] sum_i w_i z_i, or NULL */
    float* final_T;              /* float[height][width] final transmittance,
                                    or NULL                                     */
    uint8_t* visible;            /* uint8[n] M_t (1 = in the view frustum after
                                    projection, before LOD; reading R2), or NULL */
} s3r_outputs;

/* Per-view counts (rendered <= visible <= temporal <= scene).               */
typedef struct {
    int64_t n_scene;             /* N                                           */
    int64_t n_temporal;          /* passed the temporal filter (projected)      */
    int64_t n_visible;           /* |M_t|                                       */
    int64_t n_lod_small;         /* 2D scale <= r                               */
    int64_t n_lod_dropped;       /* culled by the Bernoulli draw                */
    int64_t n_rendered;          /* blended                                     */
    int64_t n_pairs;             /* (tile, Gaussian) pairs                      */
    int64_t n_bad_instance;      /* ids outside [0,K]                           */
    int64_t n_bin_pairs;         /* (supertile, Gaussian) pairs of the binning  */
    int64_t n_blend_evals;       /* E_alg: sum over pixels of the splats the
                                    pixel examines up to and including its
                                    terminating one (0 unless counters are on) */
    int64_t n_blend_exec;        /* E_exec: 256 x splats each tile CTA walked
                                    (0 unless counters are on)                  */
} s3r_stats;

/* Debug dump of one view's intermediates (DEVICE pointers, caller-allocated
 * with the sizes of s3r_get_stats; any may be NULL).  keys/flags/rect need
 * s3r_set_debug(ctx, 1) before the render.                                 */
typedef struct {
    int32_t* temporal_idx;       /* [n_temporal] ascending Gaussian indices     */
    float* keys;                 /* [n_temporal][6] mx,my,z,a,b,c (fp32 keys)   */
    uint8_t* flags;              /* [n_temporal] bit 1 visible, 2 small,
                                    3 dropped, 4 rendered, 5 bad id, 6 mean moved
                                    by the LOD noisy offset (bit 0 set)          */
    int16_t* rect;               /* [n_temporal][4] tile rect tx0,tx1,ty0,ty1   */
    int32_t* depth_order;        /* [n_rendered] Gaussian indices by (z, index) */
    int32_t* pair_tile;          /* [n_pairs] sorted pairs: tile id (row-major) */
    int32_t* pair_gauss;         /* [n_pairs] sorted pairs: Gaussian index      */
    int32_t* ranges;             /* [tiles][2] [start,end) per tile             */
    float* splat_rgb;            /* [n_rendered][3] splat colour by depth rank
                                    (the NeurF query's output when enabled)     */
} s3r_debug;

/* Stage timers (milliseconds, summed over renders since the last reset).    */
enum {
    S3R_STAGE_FILTER = 0,        /* K1 temporal filter + compaction            */
    S3R_STAGE_PROJECT,           /* K2 projection + LOD + life update          */
    S3R_STAGE_DEPTH_SORT,        /* K5 (depth, index) radix sort                */
    S3R_STAGE_BIN,               /* K3 depth-order permute + K4 supertile
                                    counting sort (count, scan, scatter) and
                                    the per-tile list expansion with ranges     */
    S3R_STAGE_RASTER,            /* K7 tile filter + alpha-blend rasterizer     */
    S3R_STAGE_COLOR,             /* K6 NeurF colour query (0 unless enabled)    */
    S3R_NUM_STAGES
};

int s3r_version(void);

/* Create a context on CUDA device `device`.  *out receives the handle.      */
int s3r_create(int device, s3r_ctx** out);
void s3r_destroy(s3r_ctx* ctx);
/* Message of the last failed call (never NULL; empty when none).            */
const char* s3r_last_error(const s3r_ctx* ctx);

/* Enable (1) / disable (0) the per-Gaussian debug intermediates
 * (keys/flags/rect) of s3r_dump_intermediates.  Costs one extra write of
 * 34 B per projected Gaussian when on.                                      */
int s3r_set_debug(s3r_ctx* ctx, int enable);
/* Enable (1) / disable (0) the rasterizer work counters n_blend_evals /
 * n_blend_exec of s3r_stats (one block reduction + atomic per tile CTA).   */
int s3r_set_counters(s3r_ctx* ctx, int enable);
/* Enable (1) / disable (0) CUDA-event stage timers; resets the sums.        */
int s3r_set_timing(s3r_ctx* ctx, int enable);
/* out_ms[S3R_NUM_STAGES]: summed stage times; out_count: renders timed.
 * Synchronises the context's last stream.                                   */
int s3r_get_stage_times(s3r_ctx* ctx, double* out_ms, int64_t* out_count);

/* Instance-specific cameras: for each view v, out[v][0] = w2c[v]
 * and out[v][i] = w2c[v] * i2g[v][i-1] (3x4 [R|t] as 4x4 homogeneous), i in
 * 1..K, computed in fp64 and rounded once to fp32 (R-ARITH).
 *   w2c: DEVICE float[n_views][12]; i2g: DEVICE float[n_views][K][12] (NULL if
 *   K == 0); out: DEVICE float[n_views][K+1][12].                           */
int s3r_compose_instance_cameras(s3r_ctx* ctx, const float* w2c, const float* i2g,
                                 int32_t n_views, int32_t K, float* out, void* stream);

/* Render one view: s3r_render_batch with n_views = 1.                       */
int s3r_render(s3r_ctx* ctx, const s3r_scene* scene, const s3r_view* view,
               const s3r_outputs* out, void* stream);

/* Render n_views views of one scene (views/outs: HOST arrays of structs whose
 * pointer members are DEVICE pointers).  Views sharing a time t share one
 * temporal compaction.  If scene->life is non-NULL it is updated with every
 * view's M_t (Eq.5; order-independent, so the result does not depend on the
 * batch split).  Returns S3R_EINSTANCE (after completing the render) if a
 * Gaussian had an out-of-range instance id.                                 */
int s3r_render_batch(s3r_ctx* ctx, const s3r_scene* scene, const s3r_view* views,
                     int32_t n_views, const s3r_outputs* outs, void* stream);

/* Overlapped batches (default off): s3r_render_batch with >= 16 views renders
 * the second half of the batch in an internal twin context (its own scratch)
 * on an internal stream forked from and joined back into `stream`, so that
 * half's filter / projection / sort / binning (and their host syncs) run while
 * the first half rasterizes.  Results are identical to one piece;
 * s3r_get_stats covers every view; s3r_dump_intermediates returns S3R_ESTATE
 * after such a batch.  Debug, counters, training and NeurF renders are never
 * split.  enable = 0 (the default; S3R_OVERLAP=1 at s3r_create turns it on)
 * renders every batch in one piece.  Measured neutral on the C3 workload
 * (the rasterizer already fills every SM), kept as an option
 * for workloads whose front stages dominate.                               */
int s3r_set_overlap(s3r_ctx* ctx, int enable);

/* Fast exponential (default off): the rasterizer (K7, Eq.2's exp) evaluates
 * 2^x with the SFU's ex2.approx.ftz (<= 2 ulp) instead of the R-ARITH
 * polynomial of DESIGN.md §4; the SFU runs beside the FP32 pipe that bounds
 * the blend.  Images are then NOT bit-identical to the oracle: RGB and final T
 * stay within 1e-4 (include-then-stop bounds a flipped termination by the
 * remaining T < 1e-4), depth within 1e-4 * (the largest splat depth of the
 * pixel's list) at such flips (reading R24).  Everything before K7
 * (decisions, order, life, stats) is unaffected.  Training renders
 * (s3r_set_training) always use the exact exponential, since the backward
 * recomputes alpha with it.  Returns S3R_EINVAL for a NULL ctx.             */
int s3r_set_fast_exp(s3r_ctx* ctx, int enable);

/* Capacity mode (PAPER.md P:155 runs the per-view pipeline once per training
 * view; SURVEY.md §7 "hard parts" 4 and 7: a per-view host readback of the
 * splat / pair counts serialises small views).  With a reservation in place,
 * s3r_render / s3r_render_batch size every step of a batch on the device
 * (k_plan.cu) from the reserved capacities instead of reading counts back:
 * the call enqueues the whole batch without a host synchronisation and may be
 * captured in a CUDA graph (cudaStreamBeginCapture on `stream`; replaying the
 * graph re-renders the same views and outputs).  Results are bit-identical to
 * the default mode.  Scratch is allocated at reservation size on the next
 * render.  A view whose counts exceed a capacity is rendered empty and
 * s3r_check then returns S3R_ECAPACITY: check it (once per many batches is
 * enough, it accumulates) or reserve from s3r_capacity_from_last with a
 * margin.  Debug dumps, training, NeurF and the conventional pipeline keep the
 * synchronous sizing (their renders ignore the reservation); s3r_get_stats
 * synchronises on the batch.
 *   records        rendered-candidate records over a batch: the sum over views
 *                  of n_temporal (Gaussians passing the temporal filter)
 *   rendered_view  splats rendered (after LOD) in any one view
 *   bin_pairs      supertile pairs over a batch (s3r_stats.n_bin_pairs summed)
 *   tile_entries   tile-list entries over a batch: sum of S*S x bin pairs
 *                  (S = 4, or 8 above 4096 supertiles of 4 x 4 tiles)
 *   temporal_view  n_temporal of any one view (sizes the projection grid)
 * cap == NULL switches the mode off.  S3R_EINVAL for a NULL ctx or a
 * negative / zero capacity.                                                */
typedef struct s3r_capacity {
    int64_t records, rendered_view, bin_pairs, tile_entries, temporal_view;
} s3r_capacity;
int s3r_set_capacity(s3r_ctx* ctx, const s3r_capacity* cap);

/* The capacities the last batch needed, each multiplied by `margin` (>= 1),
 * for s3r_set_capacity.  Synchronises on the last batch.  S3R_ESTATE
 * without a previous render.                                               */
int s3r_capacity_from_last(s3r_ctx* ctx, float margin, s3r_capacity* out);

/* Same as s3r_render_batch, but every pointer of scene, views (including
 * instance_w2c) and outs is a HOST pointer (page-locked memory recommended).
 * The library copies the inputs to device scratch, renders, copies the
 * outputs (and the updated life) back and synchronises the stream.  Batches of
 * more than 8 views are rendered 8 views at a time while finished views are
 * copied back on an internal second stream (results identical to one batch);
 * s3r_get_stats then covers every view, s3r_dump_intermediates returns
 * S3R_ESTATE.  With debug, counters, timing or training enabled the batch is
 * rendered in one piece.                                                    */
int s3r_render_batch_host(s3r_ctx* ctx, const s3r_scene* scene, const s3r_view* views,
                          int32_t n_views, const s3r_outputs* outs, void* stream);

/* Counts of view `view_index` of the last render (host struct).            */
int s3r_get_stats(const s3r_ctx* ctx, int32_t view_index, s3r_stats* out);

/* Copy intermediates of view `view_index` of the last render into `dbg`.   */
int s3r_dump_intermediates(s3r_ctx* ctx, int32_t view_index, const s3r_debug* dbg,
                           void* stream);

/* Visibility commit after a sweep (Eq.6): for every Gaussian,
 * l_s > l_e (never observed) -> v = (-1, 1); else v = (max(-1, l_s - margin),
 * min(1, l_e + margin)); then l = (1, -1).  margin = 0.1 in the paper.      */
int s3r_commit_visibility(s3r_ctx* ctx, const s3r_scene* scene, float margin, void* stream);

/* Periodic reset: v = (-1, 1) for every Gaussian.                   */
int s3r_reset_visibility(s3r_ctx* ctx, const s3r_scene* scene, void* stream);

/* ---------------------------------------------------------------- training
 * Backward pass (config 5): the adjoint of the alpha blend (Eq.2) and of the
 * instance-specific projection (Eq.1) for the views of the LAST
 * s3r_render_batch, which must have run with s3r_set_training(ctx, 1) (the
 * forward then keeps, per pixel, the final transmittance and the number of
 * list entries it blended).  Piecewise decisions (LOD drops, the 0.99 and
 * power clamps, the 2^-24 flush, termination, tile membership, the tangent
 * clamp) are held fixed.  The per-Gaussian gradients of all views are
 * ACCUMULATED (+=) with atomics into `grads` (order of the float additions is
 * not fixed, so results agree to rounding, not bit for bit).              */
int s3r_set_training(s3r_ctx* ctx, int enable);

/* Pipeline of the following renders (NEXT-2 of SURVEY.md §8(f)):
 *   S3R_PIPELINE_STREAMLINED (default) — the paper's streamlined stage
 *     (P:148-199): temporal filter, instance-specific cameras, adaptive LOD.
 *   S3R_PIPELINE_CONVENTIONAL — the baseline it replaces (Fig.1a; P:20,
 *     P:45): per view, every dynamic Gaussian is moved to the world
 *     frame (mu_w = R mu + t, q_w = quat(R) (x) q, R-ARITH op order of
 *     DESIGN.md §4), then ALL Gaussians are projected through
 *     W_t; no temporal filter, no LOD.  In this mode views[v].instance_w2c
 *     slot 0 is W_t (world->camera) and slot i >= 1 the instance's
 *     local->WORLD pose W_{t,i2g} (not the composed local->camera table).
 *     Scratch: 32 B per Gaussian per view of the batch.  The backward
 *     (s3r_render_backward) supports the streamlined pipeline only.
 * Returns S3R_EINVAL for an unknown value.                                  */
enum { S3R_PIPELINE_STREAMLINED = 0, S3R_PIPELINE_CONVENTIONAL = 1 };
int s3r_set_pipeline(s3r_ctx* ctx, int pipeline);

/* Adaptive-LOD noisy offset (Eq.7 row 4; NEXT-3) for the following
 * streamlined renders: every small Gaussian that survives the Bernoulli cull
 * has its mean moved, in the frame of its instance, by
 *   mu_a <- fma(d_a * min(1, z / D), n_a, mu_a),   a = x, y, z
 * (reading R10: normalize(d) = min(1, d / D) with z the projected depth and D
 * the view's lod_D), n = three standard normals drawn per (view lod_seed,
 * Gaussian) by the R-ARITH Box-Muller sampler of DESIGN.md §4, and is
 * projected again: its splat, depth key and tile rectangle come from the moved
 * mean (it is not rendered if that leaves the frustum); M_t, the small set and
 * the drop set come from the original one.  (0, 0, 0) = off (the default).
 * Ignored by the conventional pipeline (no LOD).  s3r_render_backward of a
 * training render made with it differentiates at the moved means, the offset
 * being a constant (reading R23).  S3R_EINVAL if non-finite.                */
int s3r_set_lod_jitter(s3r_ctx* ctx, float dx, float dy, float dz);

/* NeurF colour query (Eq.7 rows 5-6; NEXT-4): with it enabled the
 * colour of every rendered Gaussian is c = NeurF_sta(mu, d, dir, emb(t)) for
 * static and NeurF_dyn(mu, d, dir, emb(t), class) for dynamic ones instead of
 * scene->colors, computed on the tensor cores (tcgen05, bf16 operands, fp32
 * accumulation) between projection and depth sort.  Architecture (DESIGN.md
 * reading R22): 64 features in the Gaussian's own frame — mu / S, sin / cos of
 * 2^l pi mu / S for l = 0..3 (index 3 + 6 l + 2 axis + {0 sin, 1 cos}),
 * min(1, d / lod_D), the viewing direction R^T p / |p| (p = W_{t,i} mu),
 * emb(t) (8, linear interpolation of time_emb on t_j = -1 + 2 j / (n_time-1)),
 * the class embedding (4; 0 for static), zero padding — then per network
 * h1 = relu(W1 f + b1), h2 = relu(W2 h1 + b2), c = sigmoid(W3 h2 + b3).
 * All pointers DEVICE fp32, copied (weights converted to bf16) by this call:
 *   w1 [2][64][64], b1 [2][64], w2 [2][64][64], b2 [2][64], w3 [2][3][64],
 *   b3 [2][3]  (index 0 = NeurF_sta, 1 = NeurF_dyn; weight rows = outputs);
 *   time_emb [n_time][8] (n_time >= 1); class_emb [num_instances][4] (row 0
 *   unused).  pos_scale = S > 0.
 * Applies to streamlined renders whose scene has num_instances <=
 * num_instances given here (S3R_EINVAL otherwise); the conventional pipeline
 * keeps scene->colors.  params = NULL disables it.  s3r_render_backward
 * refuses (S3R_ESTATE) a render made with it.                               */
typedef struct {
    const float* w1;
    const float* b1;
    const float* w2;
    const float* b2;
    const float* w3;
    const float* b3;
    const float* time_emb;
    int32_t n_time;
    const float* class_emb;
    int32_t num_instances;
    float pos_scale;
} s3r_neurf;
int s3r_set_neural_colors(s3r_ctx* ctx, const s3r_neurf* params, void* stream);

/* Cotangents of one view: DEVICE pointers, dL/d(output) in the output layout;
 * rgb required, depth / final_T may be NULL (= 0).                         */
typedef struct {
    const float* rgb;            /* float[height][width][3]                     */
    const float* depth;          /* float[height][width] or NULL                */
    const float* final_T;        /* float[height][width] or NULL                */
} s3r_cotangents;

/* Gradient accumulators, DEVICE float4[n] each, scene-row layout:
 * means_opacity = dL/d(mu_x, mu_y, mu_z, opacity); scales = dL/d(sigma), .w
 * untouched; rotations = dL/dq (w,x,y,z) of the unnormalised quaternion;
 * colors = dL/d(r,g,b), .w untouched.  table (optional, NULL = not wanted):
 * DEVICE float[n_views][num_instances][12] += dL/d(instance camera table)
 * (NEXT-1 pose gradient: slot 0 = dL/dW_t, slot i = dL/dW_{t,i}, row-major
 * 3x4 [R | t]; the caller chains it through W_{t,i} = W_t W_{t,i2g} to the
 * object poses, e.g. dL/dR_i2g = R_t^T dL/dR_{t,i}, dL/dt_i2g = R_t^T dL/dt_{t,i}). */
typedef struct {
    float* means_opacity;
    float* scales;
    float* rotations;
    float* colors;
    float* table;
} s3r_grads;

/* scene and views must be the ones of the last render; cots: HOST array of
 * n_views structs (device pointers inside).                                */
int s3r_render_backward(s3r_ctx* ctx, const s3r_scene* scene, const s3r_view* views,
                        int32_t n_views, const s3r_cotangents* cots, const s3r_grads* grads,
                        void* stream);

/* Mean-squared-error helper for a training step: over n floats,
 * grad[i] = 2 scale (x[i] - y[i]) and *loss += scale sum (x - y)^2 (loss is a
 * DEVICE float, accumulated with atomics).  x, y, grad: DEVICE float[n].    */
int s3r_mse(s3r_ctx* ctx, const float* x, const float* y, int64_t n, float scale, float* grad,
            float* loss, void* stream);

/* Multi-GPU point-life merge helper (Eq.5 is a min/max, so replicas merge
 * exactly): negates l_s of every Gaussian in place (an involution).  Between
 * two calls an all-reduce MAX over the float[2n] life array (NCCL) yields
 * (min l_s, max l_e) over ranks.  life: DEVICE float2[n].                  */
int s3r_life_flip(s3r_ctx* ctx, float* life, int64_t n, void* stream);

/* Synchronise `stream` and return the device error state accumulated since
 * the last check: S3R_EINTERNAL (a failed self-check, see the enum),
 * S3R_ECAPACITY, S3R_EINSTANCE, S3R_ECUDA or S3R_OK.                       */
int s3r_check(s3r_ctx* ctx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* S3R_H */
