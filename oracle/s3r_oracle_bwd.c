/*
 * s3r_oracle_bwd.c — fp64 ADJOINT of the oracle's forward (config 5).
 * TEST INFRASTRUCTURE ONLY (see s3r_oracle.h).
 *
 * The gradient of a scalar loss L with respect to every Gaussian's raw
 * parameters (mean in its instance frame, linear scales, unnormalised
 * quaternion, opacity, colour), given dL/d(rgb, depth, final_T) of one view.
 * It differentiates the fp64 shadow forward (Eq.1 projection P:107-112 through
 * the instance camera of P:158-159, Eq.2 blending P:114-118, readings R5, R12-R15
 * of DESIGN.md) exactly as written: piecewise (clamps, LOD drops, termination,
 * tile membership) are held fixed, as autograd does.  Plain loops, no fusion:
 *   1. forward: filter -> project -> decide -> LOD -> per-pixel ordered list
 *      with every alpha_k and T_k recorded;
 *   2. blend adjoint per pixel, back to front:
 *        dL/dc_k = w_k gC, dL/dz_k = w_k gD,
 *        dL/dalpha_k = T_k (c_k.gC + z_k gD) - (R_k + gT T_final)/(1 - alpha_k),
 *        R_k = sum_{j>k} (c_j.gC + z_j gD) w_j,
 *      then alpha = o exp(power) (unless clamped at 0.99) and power =
 *      -1/2 (A dx^2 + C dy^2) - B dx dy (unless clamped at 0);
 *   3. projection adjoint per Gaussian: conic = inverse(Sigma' + 0.3 I),
 *      Sigma' = U U^T, U = J T, T = W R(q/|q|) diag(sigma), J(p) with the
 *      tangent clamp, mean = pinhole(p), p = W mu + t.
 * grads (accumulated, +=): double[n][16] laid out like the scene rows:
 *   {mu_x, mu_y, mu_z, opacity, s_x, s_y, s_z, 0, q_w, q_x, q_y, q_z, r, g, b, 0}.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "s3r_oracle.h"

typedef struct {
    double mx, my, z, o, A, B, C, r, g, b;
    /* accumulated per-splat gradients */
    double gmx, gmy, gz, gA, gB, gC, go, gr, gg, gb;
} bw_splat;

typedef struct {
    int32_t tile;
    int32_t g;
    double z;
} bw_pair;

static int bw_pair_cmp(const void* pa, const void* pb)
{
    const bw_pair* a = (const bw_pair*)pa;
    const bw_pair* b = (const bw_pair*)pb;
    if (a->tile != b->tile) return a->tile < b->tile ? -1 : 1;
    if (a->z != b->z) return a->z < b->z ? -1 : 1;
    if (a->g != b->g) return a->g < b->g ? -1 : 1;
    return 0;
}

/* rotation matrix of a unit quaternion (w,x,y,z), row-major */
static void rotmat(double w, double x, double y, double z, double R[9])
{
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

/* Projection adjoint of Gaussian g in view v: from the splat's accumulated
 * (gmx, gmy, gz, gA, gB, gC) to mean, scales and quaternion. */
static void project_adjoint(const so_scene* s, const so_view* v, int64_t g, const bw_splat* sp,
                            const double* key, int jittered, double* out, double* gtab)
{
    const int32_t id = s->instance_ids[g];
    const float* Mf = v->instance_w2c + 12 * (int64_t)id;
    double Wr[9], t[3];
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) Wr[3 * r + c] = Mf[4 * r + c];
        t[r] = Mf[4 * r + 3];
    }
    double mu[3] = {s->means_opacity[4 * g], s->means_opacity[4 * g + 1],
                    s->means_opacity[4 * g + 2]};
    if (jittered) {
        /* the splat was rendered from the mean moved by the LOD noisy offset
         * (NEXT-3, as in the forward); reading R23: the offset is a constant of
         * the backward (stop-gradient through the noise and its depth scale), so
         * dL/dmu = dL/dmu_moved and the projection adjoint runs at mu_moved */
        float nz[3];
        so_lod_normal3(v->lod_seed, g, nz);
        const double nd = fmin(1.0, key[2] / (double)v->lod_D);
        for (int a = 0; a < 3; ++a) mu[a] = fma((double)v->lod_jitter[a] * nd, (double)nz[a], mu[a]);
    }
    double p[3];
    for (int r = 0; r < 3; ++r) p[r] = Wr[3 * r] * mu[0] + Wr[3 * r + 1] * mu[1] + Wr[3 * r + 2] * mu[2] + t[r];
    const double qr[4] = {s->rotations[4 * g], s->rotations[4 * g + 1], s->rotations[4 * g + 2],
                          s->rotations[4 * g + 3]};
    const double qn = sqrt(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
    const double w = qr[0] / qn, x = qr[1] / qn, y = qr[2] / qn, zq = qr[3] / qn;
    double Rq[9];
    rotmat(w, x, y, zq, Rq);
    const double sg[3] = {s->scales[4 * g], s->scales[4 * g + 1], s->scales[4 * g + 2]};
    double WR[9], T[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            WR[3 * r + c] = Wr[3 * r] * Rq[c] + Wr[3 * r + 1] * Rq[3 + c] + Wr[3 * r + 2] * Rq[6 + c];
            T[3 * r + c] = WR[3 * r + c] * sg[c];
        }
    const double fx = v->fx, fy = v->fy;
    const double Wf = v->width, Hf = v->height;
    const double lox = (-(0.15 * Wf) - v->cx) / fx, hix = ((1.15 * Wf) - v->cx) / fx;
    const double loy = (-(0.15 * Hf) - v->cy) / fy, hiy = ((1.15 * Hf) - v->cy) / fy;
    const double pz = p[2];
    const double u = p[0] / pz, vv = p[1] / pz;
    const int uclamp = (u < lox || u > hix), vclamp = (vv < loy || vv > hiy);
    const double uc = fmin(fmax(u, lox), hix), vc = fmin(fmax(vv, loy), hiy);
    double J[6] = {fx / pz, 0, -fx * uc / pz, 0, fy / pz, -fy * vc / pz};
    double U[6];
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) U[3 * r + c] = J[3 * r] * T[c] + J[3 * r + 1] * T[3 + c] + J[3 * r + 2] * T[6 + c];
    const double a = U[0] * U[0] + U[1] * U[1] + U[2] * U[2];
    const double b = U[0] * U[3] + U[1] * U[4] + U[2] * U[5];
    const double c = U[3] * U[3] + U[4] * U[4] + U[5] * U[5];
    const double ad = a + 0.3, cd = c + 0.3, det = ad * cd - b * b;
    const double Q[4] = {cd / det, -b / det, -b / det, ad / det};

    /* conic -> Sigma'_dil:  G_S = -Q G_Q Q with G_Q = [[gA, gB/2],[gB/2, gC]] */
    const double GQ[4] = {sp->gA, 0.5 * sp->gB, 0.5 * sp->gB, sp->gC};
    double QG[4], GS[4];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) QG[2 * i + j] = Q[2 * i] * GQ[j] + Q[2 * i + 1] * GQ[2 + j];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) GS[2 * i + j] = -(QG[2 * i] * Q[j] + QG[2 * i + 1] * Q[2 + j]);
    /* Sigma' = U U^T:  dL/dU = 2 G_S U  (G_S symmetric) */
    double gU[6];
    for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k) gU[3 * r + k] = 2.0 * (GS[2 * r] * U[k] + GS[2 * r + 1] * U[3 + k]);
    /* U = J T:  dL/dJ = gU T^T,  dL/dT = J^T gU */
    double gJ[6], gT[9];
    for (int r = 0; r < 2; ++r)
        for (int k = 0; k < 3; ++k) gJ[3 * r + k] = gU[3 * r] * T[3 * k] + gU[3 * r + 1] * T[3 * k + 1] + gU[3 * r + 2] * T[3 * k + 2];
    for (int k = 0; k < 3; ++k)
        for (int c2 = 0; c2 < 3; ++c2) gT[3 * k + c2] = J[k] * gU[c2] + J[3 + k] * gU[3 + c2];
    /* T = (W R_q) diag(sigma) */
    double gWR[9];
    for (int r = 0; r < 3; ++r)
        for (int c2 = 0; c2 < 3; ++c2) {
            out[4 + c2] += gT[3 * r + c2] * WR[3 * r + c2];
            gWR[3 * r + c2] = gT[3 * r + c2] * sg[c2];
        }
    double gR[9];   /* dL/dR_q = W^T gWR */
    for (int r = 0; r < 3; ++r)
        for (int c2 = 0; c2 < 3; ++c2) gR[3 * r + c2] = Wr[r] * gWR[c2] + Wr[3 + r] * gWR[3 + c2] + Wr[6 + r] * gWR[6 + c2];
    const double dRw[9] = {0, -2 * zq, 2 * y, 2 * zq, 0, -2 * x, -2 * y, 2 * x, 0};
    const double dRx[9] = {0, 2 * y, 2 * zq, 2 * y, -4 * x, -2 * w, 2 * zq, 2 * w, -4 * x};
    const double dRy[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * zq, -2 * w, 2 * zq, -4 * y};
    const double dRz[9] = {-4 * zq, -2 * w, 2 * x, 2 * w, -4 * zq, 2 * y, 2 * x, 2 * y, 0};
    double gqn[4] = {0, 0, 0, 0};
    for (int k = 0; k < 9; ++k) {
        gqn[0] += gR[k] * dRw[k];
        gqn[1] += gR[k] * dRx[k];
        gqn[2] += gR[k] * dRy[k];
        gqn[3] += gR[k] * dRz[k];
    }
    const double qh[4] = {w, x, y, zq};
    const double dotq = qh[0] * gqn[0] + qh[1] * gqn[1] + qh[2] * gqn[2] + qh[3] * gqn[3];
    for (int k = 0; k < 4; ++k) out[8 + k] += (gqn[k] - qh[k] * dotq) / qn;

    /* J(p) and the mean (mx, my, z) -> p */
    double gp[3] = {0, 0, 0};
    gp[2] += gJ[0] * (-fx / (pz * pz)) + gJ[4] * (-fy / (pz * pz));
    if (uclamp) {
        gp[2] += gJ[2] * (fx * uc / (pz * pz));
    } else {
        gp[0] += gJ[2] * (-fx / (pz * pz));
        gp[2] += gJ[2] * (2.0 * fx * p[0] / (pz * pz * pz));
    }
    if (vclamp) {
        gp[2] += gJ[5] * (fy * vc / (pz * pz));
    } else {
        gp[1] += gJ[5] * (-fy / (pz * pz));
        gp[2] += gJ[5] * (2.0 * fy * p[1] / (pz * pz * pz));
    }
    gp[0] += sp->gmx * fx / pz;
    gp[2] += sp->gmx * (-fx * p[0] / (pz * pz));
    gp[1] += sp->gmy * fy / pz;
    gp[2] += sp->gmy * (-fy * p[1] / (pz * pz));
    gp[2] += sp->gz;
    for (int k = 0; k < 3; ++k) out[k] += Wr[k] * gp[0] + Wr[3 + k] * gp[1] + Wr[6 + k] * gp[2];
    /* the instance camera M = [Wr | t] (NEXT-1 pose gradient): p = Wr mu + t and
     * WR = Wr R_q give dL/dWr = gp mu^T + gWR R_q^T, dL/dt = gp */
    if (gtab) {
        double* G = gtab + 12 * (int64_t)id;
        for (int r = 0; r < 3; ++r) {
            for (int k = 0; k < 3; ++k)
                G[4 * r + k] += gp[r] * mu[k] + gWR[3 * r] * Rq[3 * k] + gWR[3 * r + 1] * Rq[3 * k + 1] +
                                gWR[3 * r + 2] * Rq[3 * k + 2];
            G[4 * r + 3] += gp[r];
        }
    }
    out[3] += sp->go;
    out[12] += sp->gr;
    out[13] += sp->gg;
    out[14] += sp->gb;
}

int so_backward_f64(const so_scene* s, const so_view* v, const double* g_rgb,
                    const double* g_depth, const double* g_T, double* grads, double* g_table)
{
    if (!s || !v || !g_rgb || !grads) return -1;
    const int32_t W = v->width, H = v->height;
    const int32_t TX = (W + SO_TILE - 1) / SO_TILE, TY = (H + SO_TILE - 1) / SO_TILE;
    const int64_t n = s->n;
    so_out_f64 o;
    memset(&o, 0, sizeof(o));
    double* keys = (double*)malloc((size_t)(n > 0 ? n : 1) * 6 * sizeof(double));
    double* skeys = (double*)malloc((size_t)(n > 0 ? n : 1) * 6 * sizeof(double));
    uint8_t* flags = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
    int16_t* rect = (int16_t*)calloc((size_t)(n > 0 ? n : 1) * 4, sizeof(int16_t));
    o.keys = keys;
    o.splat_keys = skeys;
    o.flags = flags;
    o.rect = rect;
    so_render_view_f64(s, v, &o);            /* forward decisions (f64 shadow) */

    bw_splat* sp = (bw_splat*)calloc((size_t)(n > 0 ? n : 1), sizeof(bw_splat));
    int64_t npairs = 0;
    for (int64_t g = 0; g < n; ++g) {
        if (!(flags[g] & SO_F_RENDERED)) continue;
        const double* k = skeys + 6 * g;            /* the rendered splat (moved mean) */
        const double ad = k[3] + 0.3, cd = k[5] + 0.3, det = ad * cd - k[4] * k[4];
        bw_splat* q = &sp[g];
        q->mx = k[0]; q->my = k[1]; q->z = k[2];
        q->A = cd / det; q->B = -k[4] / det; q->C = ad / det;
        q->o = s->means_opacity[4 * g + 3];
        q->r = s->colors[4 * g]; q->g = s->colors[4 * g + 1]; q->b = s->colors[4 * g + 2];
        npairs += (int64_t)(rect[4 * g + 1] - rect[4 * g] + 1) * (rect[4 * g + 3] - rect[4 * g + 2] + 1);
    }
    bw_pair* pairs = (bw_pair*)malloc((size_t)(npairs > 0 ? npairs : 1) * sizeof(bw_pair));
    int64_t m = 0;
    for (int64_t g = 0; g < n; ++g) {
        if (!(flags[g] & SO_F_RENDERED)) continue;
        for (int ty = rect[4 * g + 2]; ty <= rect[4 * g + 3]; ++ty)
            for (int tx = rect[4 * g]; tx <= rect[4 * g + 1]; ++tx) {
                pairs[m].tile = ty * TX + tx;
                pairs[m].g = (int32_t)g;
                pairs[m].z = sp[g].z;
                ++m;
            }
    }
    qsort(pairs, (size_t)m, sizeof(bw_pair), bw_pair_cmp);
    int64_t* start = (int64_t*)calloc((size_t)TX * TY + 1, sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) start[pairs[i].tile + 1]++;
    for (int64_t tt = 0; tt < (int64_t)TX * TY; ++tt) start[tt + 1] += start[tt];

    double* al = (double*)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    double* Tk = (double*)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    double* pw = (double*)malloc((size_t)(m > 0 ? m : 1) * sizeof(double));
    for (int32_t py = 0; py < H; ++py) {
        for (int32_t px = 0; px < W; ++px) {
            const int64_t tt = (int64_t)(py / SO_TILE) * TX + (px / SO_TILE);
            const int64_t b0 = start[tt], e0 = start[tt + 1];
            /* forward, recording alpha_k, T_k and the raw power */
            double T = 1.0;
            int64_t last = b0;
            for (int64_t i = b0; i < e0; ++i) {
                const bw_splat* q = &sp[pairs[i].g];
                const double dx = q->mx - px, dy = q->my - py;
                const double power = -0.5 * (q->A * dx * dx + q->C * dy * dy) - q->B * dx * dy;
                const double a = fmin(0.99, q->o * exp(fmin(0.0, power)));
                al[i] = a;
                Tk[i] = T;
                pw[i] = power;
                T = T * (1.0 - a);
                last = i + 1;
                if (T < 1e-4) break;
            }
            const int64_t pix = (int64_t)py * W + px;
            const double gC[3] = {g_rgb[3 * pix], g_rgb[3 * pix + 1], g_rgb[3 * pix + 2]};
            const double gD = g_depth ? g_depth[pix] : 0.0;
            const double gTf = g_T ? g_T[pix] : 0.0;
            double Rsum = 0.0;
            for (int64_t i = last - 1; i >= b0; --i) {
                bw_splat* q = &sp[pairs[i].g];
                const double a = al[i], Ti = Tk[i], w = a * Ti;
                q->gr += w * gC[0];
                q->gg += w * gC[1];
                q->gb += w * gC[2];
                q->gz += w * gD;
                const double cdot = q->r * gC[0] + q->g * gC[1] + q->b * gC[2] + q->z * gD;
                const double ga = Ti * cdot - (Rsum + gTf * T) / (1.0 - a);
                Rsum += cdot * w;
                const double G = exp(fmin(0.0, pw[i]));
                if (q->o * G >= 0.99) continue;         /* alpha clamped at 0.99 */
                q->go += ga * G;
                if (pw[i] > 0.0) continue;              /* power clamped at 0 */
                const double gP = ga * a;
                const double dx = q->mx - px, dy = q->my - py;
                q->gA += -0.5 * dx * dx * gP;
                q->gC += -0.5 * dy * dy * gP;
                q->gB += -dx * dy * gP;
                q->gmx += -(q->A * dx + q->B * dy) * gP;
                q->gmy += -(q->B * dx + q->C * dy) * gP;
            }
        }
    }
    for (int64_t g = 0; g < n; ++g)
        if (flags[g] & SO_F_RENDERED)
            project_adjoint(s, v, g, &sp[g], keys + 6 * g, (flags[g] & SO_F_JITTERED) != 0,
                            grads + 16 * g, g_table);

    free(pw); free(Tk); free(al); free(start); free(pairs); free(sp);
    free(rect); free(flags); free(keys); free(skeys);
    return 0;
}
