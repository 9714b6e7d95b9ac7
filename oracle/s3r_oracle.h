/*
 * s3r_oracle.h — CPU ORACLE of the S3R-GS streamlined per-view splatting path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2503_08217_b200/, include/s3r.h) never links, includes or calls it, and
 * it shares no code with the CUDA path: every formula here is restated from
 * PAPER.md (arxiv 2503.08217) and the DESIGN.md readings.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation named
 * beside it).  Eq.1 projection P:107-112, Eq.2 alpha-blend P:114-118, Eq.5
 * point-life P:173-178, Eq.6 commit P:180-182, Eq.7 adaptive LOD P:189-198.
 *
 * The library is compiled twice from one source (s3r_oracle_impl.inc):
 *   *_f32 — the fp32 CONTRACT arithmetic: single IEEE ops
 *           in the written order, explicit fmaf, -ffp-contract=off, the software
 *           exponential s3r_exp.  Integer decisions (visible set, LOD set,
 *           tiles, order) are taken in fp32, the precision of the kernel.
 *   *_f64 — an fp64 SHADOW of the same algorithm with libm exp; used by the
 *           pin tests to bound the fp32 rounding error.
 * Single-threaded, slow, no blocking/fusion: one view at a time, one Gaussian
 * at a time, one pixel at a time.
 */
#ifndef S3R_ORACLE_H
#define S3R_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scene: host arrays of n Gaussians ("each Gaussian is assigned a 3D
 * position mu, a 3D covariance Sigma, an opacity alpha, a temporal visibility v
 * and a point life l ... dynamic Gaussian is associated with an instance ID"). */
typedef struct {
    int64_t n;
    int32_t num_instances;        /* K+1; id 0 = static (reading R17)          */
    const float* means_opacity;   /* [n][4]: x,y,z (local frame of its id), o  */
    const float* scales;          /* [n][4]: sigma_x, sigma_y, sigma_z, pad    */
    const float* rotations;       /* [n][4]: w,x,y,z (normalised here)         */
    const float* colors;          /* [n][4]: r,g,b, pad                         */
    const int32_t* instance_ids;  /* [n]                                        */
    float* visibility;            /* [n][2]: v_s, v_e                           */
    float* life;                  /* [n][2]: l_s, l_e  (NULL = no update)       */
} so_scene;

/* One view at time t: intrinsics K_t and the per-instance extrinsics
 * W_{t,i} = W_t W_{t,i2g}, slot 0 = W_t. */
typedef struct {
    float t;
    int32_t width, height;
    float fx, fy, cx, cy;
    float near_plane;
    const float* instance_w2c;    /* [num_instances][12] row-major 3x4          */
    float lod_r, lod_pmax, lod_D; /* Eq.7 r, p_max, D                           */
    uint64_t lod_seed;
    float lod_jitter[3];          /* Eq.7 row 4 [dx, dy, dz]; 0 = no offset     */
} so_view;

/* Per-view statistics. */
typedef struct {
    int64_t n_scene, n_temporal, n_visible, n_lod_small, n_lod_dropped,
            n_rendered, n_pairs, n_bad_instance;
} so_stats;

/* Per-Gaussian flag bits written to so_out.flags */
#define SO_F_TEMPORAL 1u   /* passed the temporal filter            */
#define SO_F_VISIBLE  2u   /* M_t: in the view frustum              */
#define SO_F_SMALL    4u   /* 2D scale <= r (Eq.7 set G'_{t,Sigma'<=r})    */
#define SO_F_DROPPED  8u   /* culled by the Bernoulli draw (Eq.7 row 2)     */
#define SO_F_RENDERED 16u  /* blended (visible and not dropped)             */
#define SO_F_BADID    32u  /* instance id outside [0, K]                    */
#define SO_F_JITTERED 64u  /* small, kept, mean moved by the LOD noisy offset */

#define SO_TILE 16

/* Optional outputs (any pointer may be NULL).  Arrays are caller-owned. */
#define SO_DECLARE_OUT(SUF, REAL)                                               \
    typedef struct {                                                            \
        REAL* rgb;            /* [H][W][3] */                                   \
        REAL* depth;          /* [H][W]    */                                   \
        REAL* final_T;        /* [H][W]    */                                   \
        uint8_t* visible;     /* [n]  M_t  */                                   \
        int32_t* temporal_idx;/* [n]  ascending indices passing the filter */   \
        REAL* keys;           /* [n][6] mx,my,z,a,b,c (only temporal ones) */   \
        REAL* splat_keys;     /* [n][6] keys of the rendered splat (moved) */   \
        uint8_t* flags;       /* [n]  SO_F_* */                                 \
        int16_t* rect;        /* [n][4] tx0,tx1,ty0,ty1 (visible ones) */       \
        int32_t* pair_tile;   /* [pair_capacity] sorted pairs: tile id */       \
        int32_t* pair_gauss;  /* [pair_capacity] sorted pairs: Gaussian */      \
        int64_t pair_capacity;                                                  \
        int32_t* ranges;      /* [tiles][2] start,end into the pair list */     \
        so_stats stats;                                                         \
    } so_out_##SUF;
SO_DECLARE_OUT(f32, float)
SO_DECLARE_OUT(f64, double)

/* ---- f32 contract ---------------------------------------------------- */
double   so_normalize_time(int64_t frame, int64_t frame_count);
float    so_exp2_f32(float x);
uint64_t so_splitmix64(uint64_t x);
float    so_lod_uniform(uint64_t seed, int64_t g);
/* NEXT-3 noise: three standard normals for Gaussian g of a view (R-ARITH
 * Box-Muller, so_log2_f32 / so_sincos_turn_f32), and its building blocks */
void     so_lod_normal3(uint64_t seed, int64_t g, float out[3]);
float    so_lod_uniform_k(uint64_t seed, int64_t g, int k);
float    so_log2_f32(float x);
void     so_sincos_turn_f32(float u, float* s, float* c);
void     so_compose_instance_cameras(const float* w2c, const float* i2g,
                                     int32_t K, float* out);
int64_t  so_temporal_filter_f32(const so_scene* s, float t, int32_t* idx);
int      so_project_f32(const so_scene* s, const so_view* v, int64_t g, float keys[6]);
float    so_drop_probability_f32(float d, float pmax, float D);
int      so_render_view_f32(const so_scene* s, const so_view* v, so_out_f32* o);
int      so_blend_bruteforce_f32(const so_scene* s, const so_view* v, const uint8_t* flags,
                                 const float* keys, const int16_t* rect,
                                 float* rgb, float* depth, float* final_T);
void     so_update_life_f32(so_scene* s, const uint8_t* visible, float t);
/* conventional pipeline C0 (NEXT-2): local -> world copy of the scene */
void     so_quat_from_rot_f32(const float R[9], float q[4]);
void     so_quat_mul_f32(const float a[4], const float b[4], float o[4]);
int64_t  so_world_transform_f32(const so_scene* s, const float* i2g, float* mo_out,
                                float* rot_out);
void     so_commit_visibility(so_scene* s, float margin);
void     so_reset_visibility(so_scene* s);

/* ---- f64 adjoint (config 5; s3r_oracle_bwd.c) ------------------------ */
/* grads += dL/d(raw params) of view v, double[n][16] in scene-row layout
 * {mu xyz, opacity, sigma xyz, 0, q wxyz, rgb, 0}; g_rgb [H][W][3] required,
 * g_depth [H][W] and g_T [H][W] optional (NULL = 0); g_table (optional)
 * += dL/d(instance camera table) double[num_instances][12] (NEXT-1 pose
 * gradient, row-major 3x4 [R | t] per slot). */
int      so_backward_f64(const so_scene* s, const so_view* v, const double* g_rgb,
                         const double* g_depth, const double* g_T, double* grads,
                         double* g_table);

/* ---- f64 shadow ------------------------------------------------------ */
double   so_exp_f64(double x);
int64_t  so_temporal_filter_f64(const so_scene* s, double t, int32_t* idx);
int      so_project_f64(const so_scene* s, const so_view* v, int64_t g, double keys[6]);
double   so_drop_probability_f64(double d, double pmax, double D);
int      so_render_view_f64(const so_scene* s, const so_view* v, so_out_f64* o);
void     so_quat_from_rot_f64(const double R[9], double q[4]);
void     so_quat_mul_f64(const double a[4], const double b[4], double o[4]);
int64_t  so_world_transform_f64(const so_scene* s, const float* i2g, float* mo_out,
                                float* rot_out);
int      so_blend_bruteforce_f64(const so_scene* s, const so_view* v, const uint8_t* flags,
                                 const double* keys, const int16_t* rect,
                                 double* rgb, double* depth, double* final_T);

#ifdef __cplusplus
}
#endif
#endif
