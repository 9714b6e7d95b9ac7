// k_neurf.cu — K6 NeurF colour query on the 5th-generation tensor cores
// (NEXT-4; Eq.7 rows 5-6: c = NeurF_sta(mu, d, dir, emb(t)),
// c = NeurF_dyn(mu, d, dir, emb(t), class), queried for the rendered Gaussians
// after the LOD cull).  Architecture: reading R22 of DESIGN.md —
// 64 own-frame features (mu / S, 4 octaves of sin / cos of pi mu / S, min(1,
// d / D), the viewing direction in the Gaussian's frame, an 8-wide time
// embedding, a 4-wide class embedding), then per network 64 -> 64 -> 64 -> 3
// with ReLU, ReLU, sigmoid; bf16 operands, fp32 accumulation.
//
// Layout: a persistent CTA of 128 threads walks 128-record tiles of the
// compacted splat records (all views, flattened).  Thread r builds row r's
// features and writes them as bf16 into the A tile in shared memory in the
// canonical no-swizzle K-major core-matrix layout (8 rows x 16 bytes per core
// matrix; K-adjacent core matrices 128 B apart = LBO, 8-row groups 1024 B
// apart = SBO).  One elected thread issues tcgen05.mma.cta_group::1.kind::f16
// (M = 128, K = 16 per instruction, 4 per layer) with the accumulator in TMEM
// (128 lanes x 128 fp32 columns); tcgen05.commit arrives on an mbarrier; each
// warp reads its 32 TMEM lanes back with tcgen05.ld.32x32b, adds the bias,
// applies the activation, rounds to bf16 and writes the next layer's A tile in
// place.  Both networks run on every tile (layer 1 and 2 as one N = 128 MMA:
// rows 0-63 of B = NeurF_sta, 64-127 = NeurF_dyn; layer 3 as N = 32) and each
// row keeps its own network's half.  Weights (36 KB bf16, pre-packed in the
// same layout by k_neurf_pack) are loaded once per CTA.
#include <cuda_bf16.h>

#include "s3r_internal.cuh"

namespace s3r {

namespace {

constexpr int NT = 128;              // threads = rows per tile = MMA M
constexpr int KF = 64;               // features = hidden width = MMA K per layer
constexpr int A_BYTES = NT * KF * 2;             // 16 KB
constexpr int W12_BYTES = 128 * KF * 2;          // 16 KB each (sta | dyn)
constexpr int W3_BYTES = 32 * KF * 2;            // 4 KB
constexpr int NB = 128 + 128 + 32;               // fp32 biases b1 | b2 | b3
constexpr int MAXV = 256;      // views whose tile offsets fit in smem (keeps 4 CTAs per SM)
constexpr size_t SMEM = (size_t)A_BYTES + 2 * W12_BYTES + W3_BYTES + NB * 4 + 64 + MAXV * 4;

// byte offset of element (row, k) in a K-major no-swizzle core-matrix tile
// with 64 columns: core matrix (row / 8, k / 8) at ((row/8) * 8 + k/8) * 128
__host__ __device__ __forceinline__ uint32_t cm_off(int row, int k)
{
    return (uint32_t)((((row >> 3) * 8 + (k >> 3)) << 7) + ((row & 7) << 4) + ((k & 7) << 1));
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr)
{
    // start >> 4 [0,14) | LBO 128 B >> 4 [16,30) | SBO 1024 B >> 4 [32,46) |
    // version 1 [46,48) | base offset 0 | layout SWIZZLE_NONE (0) [61,64)
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 16) |
           ((uint64_t)(1024 >> 4) << 32) | (1ull << 46);
}

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N)
{
    // D f32 [4,6) = 1, A bf16 [7,10) = 1, B bf16 [10,13) = 1, both K-major,
    // N >> 3 at [17,23), M >> 4 at [24,29)
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     mbar)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}\n" ::"r"(mbar),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* r)
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// the sta and dyn halves of 16 columns, one wait for both loads
__device__ __forceinline__ void tmem_ld16x2(uint32_t ta, uint32_t tb, float* va, float* vb)
{
    uint32_t ra[16], rb[16];
    tmem_ld16_nowait(ta, ra);
    tmem_ld16_nowait(tb, rb);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        va[i] = __uint_as_float(ra[i]);
        vb[i] = __uint_as_float(rb[i]);
    }
}

__device__ __forceinline__ void fence_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b)
{
    const __nv_bfloat16 x = __float2bfloat16_rn(a), y = __float2bfloat16_rn(b);
    return (uint32_t)__bfloat16_as_ushort(x) | ((uint32_t)__bfloat16_as_ushort(y) << 16);
}

// 8 consecutive k of row r (k0 multiple of 8): one 16-byte store
__device__ __forceinline__ void st_row8(uint8_t* tile, int r, int k0, const float* v)
{
    uint4 u;
    u.x = pack_bf16(v[0], v[1]);
    u.y = pack_bf16(v[2], v[3]);
    u.z = pack_bf16(v[4], v[5]);
    u.w = pack_bf16(v[6], v[7]);
    *reinterpret_cast<uint4*>(tile + cm_off(r, k0)) = u;
}

// one layer: 4 MMAs over K = 64 into TMEM columns [0, N), then commit
__device__ __forceinline__ void issue_layer(uint32_t tmem, uint32_t sa, uint32_t sb, int N,
                                            uint32_t mbar)
{
    const uint32_t id = idesc_bf16(NT, N);
#pragma unroll
    for (int j = 0; j < KF / 16; ++j)
        mma_bf16(tmem, smem_desc(sa + 256u * j), smem_desc(sb + 256u * j), id, j > 0 ? 1u : 0u);
    mma_commit(mbar);
}

__global__ void __launch_bounds__(NT) k_neurf(NeurfArgs a)
{
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sW1 = sA + A_BYTES;
    uint8_t* sW2 = sW1 + W12_BYTES;
    uint8_t* sW3 = sW2 + W12_BYTES;
    float* sB = reinterpret_cast<float*>(sW3 + W3_BYTES);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sB + NB);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 1);
    int* s_toff = reinterpret_cast<int*>(smem + A_BYTES + 2 * W12_BYTES + W3_BYTES + NB * 4 + 64);
    const int tid = threadIdx.x, warp = tid >> 5;

    // ---- weights and biases (pre-packed bf16 core-matrix layout) ----
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.wpack);
        uint4* dst = reinterpret_cast<uint4*>(sW1);
        for (int i = tid; i < (2 * W12_BYTES + W3_BYTES) / 16; i += NT) dst[i] = src[i];
        for (int i = tid; i < NB; i += NT) sB[i] = a.bias[i];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(mbar)));
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar);
    const uint32_t saA = (uint32_t)__cvta_generic_to_shared(sA);
    const uint32_t saW1 = (uint32_t)__cvta_generic_to_shared(sW1);
    const uint32_t saW2 = (uint32_t)__cvta_generic_to_shared(sW2);
    const uint32_t saW3 = (uint32_t)__cvta_generic_to_shared(sW3);
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);   // this warp's TMEM lanes
    uint32_t phase = 0;
    const float inv_s = 1.0f / a.pos_scale;

    // first tile of each view in shared memory (the per-tile view lookup is a
    // binary search there), and the next tile's per-row mean prefetched into a
    // register while the current tile is in the MMA / epilogue phases
    const int nv = a.n_views;
    const bool toff_smem = nv <= MAXV;
    if (toff_smem)
        for (int i = tid; i < nv; i += NT) s_toff[i] = a.tile_off[i];
    __syncthreads();
    auto view_of = [&](int T) -> int {
        int lo = 0, hi = nv - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((toff_smem ? s_toff[mid] : a.tile_off[mid]) <= T) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    auto row_of = [&](int T, int v, long long& o) -> bool {
        const DevView& W = a.views[v];
        const long long rr = (long long)(T - (toff_smem ? s_toff[v] : a.tile_off[v])) * NT + tid;
        o = W.cap_off + rr;
        return rr < W.n_rendered;
    };
    int Tn = blockIdx.x, vn = 0;
    long long on = 0;
    bool validn = false;
    float4 m4n = make_float4(0.f, 0.f, 0.f, 0.f);
    if (Tn < a.total_tiles) {
        vn = view_of(Tn);
        validn = row_of(Tn, vn, on);
        if (validn) m4n = a.rec_mu[on];
    }
    for (int T = blockIdx.x; T < a.total_tiles; T += gridDim.x) {
        const int lo = vn;
        const DevView& V = a.views[lo];
        const int r = tid;
        const bool valid = validn;
        const long long o = on;
        const float4 m4c = m4n;
        bool dyn = false;
        // ---- features of row r (zero rows past the view's records) ----
        float f[KF];
#pragma unroll
        for (int k = 0; k < KF; ++k) f[k] = 0.0f;
        if (valid) {
            const float4 m4 = m4c;
            const int id = __float_as_int(m4.w);
            dyn = id > 0;
            const float* M = V.table + 12 * id;
            float p[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                float acc = __fmaf_rn(M[4 * i + 0], m4.x, M[4 * i + 3]);
                acc = __fmaf_rn(M[4 * i + 1], m4.y, acc);
                acc = __fmaf_rn(M[4 * i + 2], m4.z, acc);
                p[i] = acc;
            }
            const float mu[3] = {m4.x * inv_s, m4.y * inv_s, m4.z * inv_s};
            f[0] = mu[0]; f[1] = mu[1]; f[2] = mu[2];
            // octave 0 by sincospif, octaves 1-3 by the double-angle identities
            // sin 2a = 2 sin a cos a, cos 2a = 1 - 2 sin^2 a (absolute error grows
            // ~2x per octave, ~1e-6 at octave 3, far below the features' bf16 step)
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {
                float sn, cs;
                sincospif(mu[ax], &sn, &cs);
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    f[3 + 6 * l + 2 * ax] = sn;
                    f[4 + 6 * l + 2 * ax] = cs;
                    const float s2 = 2.0f * sn * cs;
                    cs = fmaf(-2.0f * sn, sn, 1.0f);
                    sn = s2;
                }
            }
            f[27] = fminf(1.0f, p[2] / V.lod_D);
            const float rn = rsqrtf(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
            const float ph[3] = {p[0] * rn, p[1] * rn, p[2] * rn};
#pragma unroll
            for (int i = 0; i < 3; ++i) f[28 + i] = M[i] * ph[0] + M[4 + i] * ph[1] + M[8 + i] * ph[2];
            // emb(t): linear interpolation on the uniform grid of t in [-1, 1]
            const int nt = a.n_time;
            if (nt == 1) {
#pragma unroll
                for (int e = 0; e < 8; ++e) f[31 + e] = a.time_emb[e];
            } else {
                const float x = (V.t + 1.0f) * 0.5f * (float)(nt - 1);
                const int j = min(max((int)floorf(x), 0), nt - 2);
                const float w = fminf(fmaxf(x - (float)j, 0.0f), 1.0f);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    f[31 + e] = (1.0f - w) * a.time_emb[8 * j + e] + w * a.time_emb[8 * (j + 1) + e];
            }
            if (dyn) {
#pragma unroll
                for (int e = 0; e < 4; ++e) f[39 + e] = a.class_emb[4 * id + e];
            }
        }
#pragma unroll
        for (int k0 = 0; k0 < KF; k0 += 8) st_row8(sA, r, k0, f + k0);
        fence_async_smem();
        __syncthreads();
        // prefetch the next tile's row (lands during this tile's three layers)
        Tn = T + gridDim.x;
        validn = false;
        if (Tn < a.total_tiles) {
            vn = view_of(Tn);
            validn = row_of(Tn, vn, on);
            if (validn) m4n = a.rec_mu[on];
        }

        // ---- layers 1 and 2 (N = 128: sta | dyn), layer 3 (N = 32) ----
#pragma unroll 1
        for (int layer = 0; layer < 3; ++layer) {
            if (tid == 0) {
                tc_fence_after();
                issue_layer(tmem, saA, layer == 0 ? saW1 : layer == 1 ? saW2 : saW3,
                            layer == 2 ? 32 : 128, mb);
            }
            mbar_wait(mb, phase);
            phase ^= 1u;
            tc_fence_after();
            if (layer < 2) {
                const float* bias = sB + (layer == 0 ? 0 : 128) + (dyn ? 64 : 0);
#pragma unroll
                for (int c0 = 0; c0 < 64; c0 += 16) {
                    float vs[16], vd[16];
                    tmem_ld16x2(trow + c0, trow + 64 + c0, vs, vd);   // NeurF_sta | NeurF_dyn
                    float h[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) h[i] = fmaxf((dyn ? vd[i] : vs[i]) + bias[c0 + i], 0.0f);
                    st_row8(sA, r, c0, h);
                    st_row8(sA, r, c0 + 8, h + 8);
                }
            } else {
                float v[16], w[16];
                tmem_ld16x2(trow, trow + 16, v, w);       // sta outputs in columns 0-2, dyn 16-18
                if (valid) {
                    const float* b3 = sB + 256 + (dyn ? 16 : 0);
                    float c[3];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const float z = (dyn ? w[i] : v[i]) + b3[i];
                        c[i] = 1.0f / (1.0f + expf(-z));
                    }
                    float4* rec = a.rec + 3 * o + 2;
                    const float4 old = *rec;
                    *rec = make_float4(c[0], c[1], c[2], old.w);
                }
            }
            // TMEM reads and A-tile writes done before the next MMA
            tc_fence_before();
            fence_async_smem();
            __syncthreads();
        }
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// f32 weights -> bf16 core-matrix tiles:  W1 (sta rows 0-63 | dyn 64-127),
// W2 (same), W3 (sta rows 0-2, dyn rows 16-18, rest 0); biases b1 | b2 | b3
__global__ void k_neurf_pack(const float* __restrict__ w1, const float* __restrict__ b1,
                             const float* __restrict__ w2, const float* __restrict__ b2,
                             const float* __restrict__ w3, const float* __restrict__ b3,
                             uint8_t* __restrict__ wpack, float* __restrict__ bias)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    // W1, W2: 128 rows x 64 k each
    if (i < 2 * 128 * 64) {
        const int m = i / (128 * 64), rem = i % (128 * 64), row = rem / 64, k = rem % 64;
        const float* w = m == 0 ? w1 : w2;
        const float x = w[row * 64 + k];                 // [2][64][64] = row-major 128 x 64
        *reinterpret_cast<__nv_bfloat16*>(wpack + m * W12_BYTES + cm_off(row, k)) =
            __float2bfloat16_rn(x);
    }
    if (i < 32 * 64) {
        const int row = i / 64, k = i % 64;
        const int net = row >> 4, j = row & 15;
        const float x = j < 3 ? w3[(net * 3 + j) * 64 + k] : 0.0f;
        *reinterpret_cast<__nv_bfloat16*>(wpack + 2 * W12_BYTES + cm_off(row, k)) =
            __float2bfloat16_rn(x);
    }
    if (i < NB) {
        float x;
        if (i < 128) x = b1[i];
        else if (i < 256) x = b2[i - 128];
        else {
            const int row = i - 256, net = row >> 4, j = row & 15;
            x = j < 3 ? b3[net * 3 + j] : 0.0f;
        }
        bias[i] = x;
    }
}

}  // namespace

size_t neurf_pack_bytes() { return (size_t)2 * W12_BYTES + W3_BYTES; }
int neurf_bias_count() { return NB; }

void launch_neurf_pack(const float* w1, const float* b1, const float* w2, const float* b2,
                       const float* w3, const float* b3, void* wpack, float* bias,
                       cudaStream_t st)
{
    k_neurf_pack<<<(2 * 128 * 64 + 255) / 256, 256, 0, st>>>(w1, b1, w2, b2, w3, b3,
                                                             static_cast<uint8_t*>(wpack), bias);
}

void launch_neurf(const NeurfArgs& a, cudaStream_t st)
{
    if (a.total_tiles == 0) return;
    cudaFuncSetAttribute(k_neurf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    const int grid = a.total_tiles < 148 * 4 ? a.total_tiles : 148 * 4;
    k_neurf<<<grid, NT, SMEM, st>>>(a);
}

}  // namespace s3r
