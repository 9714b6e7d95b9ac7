// s3r_api.cu — the C ABI of include/s3r.h: validation, scratch management and
// the launch sequence of one batch (K1 -> K2 -> depth sort -> emit -> tile
// sort -> ranges -> raster).  Host code only orchestrates; every step of the
// path runs in the kernels of k_*.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/s3r.h"
#include "s3r_internal.cuh"

using namespace s3r;

namespace s3r {
int filter_tile();
int project_tile();
int splat_grad_stride();
}

namespace {

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
};

struct StageEvent {
    int stage;
    cudaEvent_t a, b;
};

}  // namespace

struct s3r_ctx {
    int device = 0;
    std::string err;
    bool debug = false, timing = false, counters = false, training = false;
    int pipeline = S3R_PIPELINE_STREAMLINED, last_pipeline = S3R_PIPELINE_STREAMLINED;
    float lod_jitter[3] = {0.0f, 0.0f, 0.0f};   // NEXT-3 noisy offset scale
    bool last_jitter = false, last_recmu = false;
    // NEXT-4 NeurF colour query
    bool neurf = false, last_neurf = false;
    Buf d_nw, d_nb, d_temb, d_cemb, d_recmu, d_toff;
    int neurf_ntime = 0, neurf_ninst = 0;
    float neurf_scale = 1.0f;
    Buf d_wmo, d_wrot;                       // conventional pipeline: world copies
    bool last_training = false;
    int last_nviews = 0, last_max_tiles = 0;
    long long last_max_r = 0, last_N = -1;
    Buf d_train_T, d_train_n, d_sgrads, d_cots;
    bool last_counters = false, evals_fetched = false;
    Buf d_evals;
    bool last_debug = false;
    // pinned (mapped) staging: a ring of NSTAGE areas, so that a call waits only
    // for the call that used its area NSTAGE calls earlier; a call captured in
    // a CUDA graph gets an area of its own (kept until s3r_destroy)
    struct Stage {
        char* h = nullptr;
        char* d = nullptr;
        size_t cap = 0;
        cudaEvent_t ev = nullptr;
        bool rec = false;
    };
    static constexpr int NSTAGE = 3;
    Stage ring[NSTAGE];
    int ring_i = 0, cur_slot = -1;
    std::vector<char*> graph_blocks;
    char* graph_spare = nullptr;             // pinned area for the next captured call
    size_t graph_spare_cap = 0;
    char* h_stage = nullptr;                 // the current call's area
    char* h_stage_dev = nullptr;             // its device address (mapped)
    size_t h_stage_cap = 0;
    size_t h_stage_top = 0;
    bool capture_now = false;                // the current call is being graph-captured
    // capacity mode (s3r_set_capacity)
    bool cap_on = false;
    s3r_capacity cap{};
    bool cap_pending = false;                // stats of the last batch still on the device side
    bool cap_suspend = false;                // s3r_render_batch_host: per-chunk stats on the host
    bool last_capm = false;                  // the last render was planned on the device
    long long* cap_h_ntemp = nullptr;        // mapped per-view n_temporal of that batch
    ViewCounters* cap_h_ctr = nullptr;       // mapped per-view K2 counters of that batch
    // the last batch's needs (for s3r_capacity_from_last)
    s3r_capacity last_need{};
    bool last_need_valid = false;
    cudaStream_t last_stream = nullptr;
    // device scratch
    // per-batch small state: one zeroed arena (work tickets, K1 counts, K1
    // look-back words, K2 counters: ONE memset per batch) and one upload arena
    // (distinct times, device views: one copy in the capacity mode)
    Buf d_zero, d_up;
    int* p_ticket = nullptr;
    unsigned long long* p_counts = nullptr;
    uint32_t* p_lb1 = nullptr;
    ViewCounters* p_ctr = nullptr;
    float* p_times = nullptr;
    DevView* p_views = nullptr;
    Buf d_tidx, d_lb, d_rec, d_dkey, d_gidx,
        d_sortk[2], d_sortv[2], d_recs, d_rects, d_lists, d_tlists, d_tranges, d_cnt, d_hist,
        d_dsegs, d_dtile0,
        d_ranges, d_err, d_dbg_keys, d_dbg_flags, d_dbg_rect, d_dbg_tcnt;
    int ticket_slot = 0, ticket_cap = 0;
    bool ticket_overflow = false;
    int gbits = 1;
    // mirrors for s3r_render_batch_host
    Buf m_scene[7];
    cudaStream_t copy_stream = nullptr;      // D2H of finished chunks (host path)
    // overlapped batches: the second half of a batch renders in a twin context
    // (own scratch) on its own stream, so its filter / projection / sort /
    // binning run while the first half rasterizes
    s3r_ctx* twin = nullptr;
    cudaStream_t twin_stream = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    bool overlap = false;
    bool fast_exp = false;                   // s3r_set_fast_exp: SFU ex2 in K7
    std::vector<cudaEvent_t> chunk_done;
    bool host_chunked = false;               // last render was a chunked host batch
    std::vector<Buf> m_tab, m_rgb, m_depth, m_T, m_vis;
    // last batch
    std::vector<DevView> hv;
    std::vector<s3r_stats> stats;
    long long N_last = 0;
    int final_order = 1;
    bool have_render = false;
    // timers
    std::vector<StageEvent> ev;
    double stage_ms[S3R_NUM_STAGES] = {0};
    long long timed_renders = 0;
};

namespace {

int fail(s3r_ctx* c, int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

#define CU(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess)                                                              \
            return fail(c, S3R_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x,              \
                        cudaGetErrorString(e_));                                            \
    } while (0)

int ensure(s3r_ctx* c, Buf& b, size_t bytes)
{
    if (bytes <= b.cap && b.p) return S3R_OK;
    if (b.p) {
        cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
    }
    size_t want = std::max<size_t>(bytes + bytes / 4, 256);
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        if (cudaMalloc(&b.p, std::max<size_t>(bytes, 256)) != cudaSuccess) {
            cudaGetLastError();
            b.p = nullptr;
            return fail(c, S3R_ENOMEM, "cudaMalloc of %zu bytes failed", bytes);
        }
        want = std::max<size_t>(bytes, 256);
    }
    b.cap = want;
    return S3R_OK;
}

template <typename T>
T* P(const Buf& b) { return reinterpret_cast<T*>(b.p); }

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// pinned staging: the next area of the ring (or, while the stream is being
// captured, a fresh area owned by the graph), at least `bytes` large; a bump
// allocator over it (stage_alloc) for the call
int stage_begin(s3r_ctx* c, size_t bytes, cudaStream_t st)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        cudaGetLastError();
        cs = cudaStreamCaptureStatusNone;
    }
    c->capture_now = cs != cudaStreamCaptureStatusNone;
    const size_t want = std::max<size_t>(bytes * 2, 1 << 16);
    char *h = nullptr, *d = nullptr;
    if (c->capture_now) {
        // no allocation or synchronisation may happen while capturing: the spare
        // area (made outside the capture) becomes the graph's, for good
        if (!c->graph_spare || c->graph_spare_cap < bytes)
            return fail(c, S3R_ESTATE, "graph capture: no staging area of %zu bytes reserved "
                                       "(render once outside the capture first)", bytes);
        h = c->graph_spare;
        if (cudaHostGetDevicePointer((void**)&d, h, 0) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, S3R_ECUDA, "cudaHostGetDevicePointer failed");
        }
        c->graph_blocks.push_back(h);
        c->graph_spare = nullptr;
        c->cur_slot = -1;
        c->h_stage = h;
        c->h_stage_dev = d;
        c->h_stage_cap = want;
        c->h_stage_top = 0;
        return S3R_OK;
    }
    if (c->cap_on && (!c->graph_spare || c->graph_spare_cap < want)) {
        // capacity mode: keep a spare area for a later captured call
        if (c->graph_spare) cudaFreeHost(c->graph_spare);
        c->graph_spare = nullptr;
        c->graph_spare_cap = 0;
        const size_t gw = std::max<size_t>(want * 2, 1 << 20);
        if (cudaHostAlloc((void**)&c->graph_spare, gw, cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            c->graph_spare = nullptr;
            return fail(c, S3R_ENOMEM, "cudaHostAlloc (mapped) of %zu bytes failed", gw);
        }
        c->graph_spare_cap = gw;
    }
    c->ring_i = (c->ring_i + 1) % s3r_ctx::NSTAGE;
    s3r_ctx::Stage& S = c->ring[c->ring_i];
    if (!S.ev && cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, S3R_ECUDA, "cudaEventCreate failed");
    }
    if (S.rec) {            // the call that used this area NSTAGE calls ago
        if (cudaEventSynchronize(S.ev) != cudaSuccess)
            return fail(c, S3R_ECUDA, "staging: %s", cudaGetErrorString(cudaGetLastError()));
        S.rec = false;
    }
    if (bytes > S.cap) {
        if (S.h) cudaFreeHost(S.h);
        S.h = S.d = nullptr;
        S.cap = 0;
        if (cudaHostAlloc((void**)&S.h, want, cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer((void**)&S.d, S.h, 0) != cudaSuccess) {
            cudaGetLastError();
            if (S.h) cudaFreeHost(S.h);
            S.h = nullptr;
            return fail(c, S3R_ENOMEM, "cudaHostAlloc (mapped) of %zu bytes failed", want);
        }
        S.cap = want;
    }
    c->cur_slot = c->ring_i;
    c->h_stage = S.h;
    c->h_stage_dev = S.d;
    c->h_stage_cap = S.cap;
    c->h_stage_top = 0;
    return S3R_OK;
}

// the current call's staging area is free again once `st` reaches this point
int stage_end(s3r_ctx* c, cudaStream_t st)
{
    if (c->cur_slot < 0) return S3R_OK;
    s3r_ctx::Stage& S = c->ring[c->cur_slot];
    CU(cudaEventRecord(S.ev, st));
    S.rec = true;
    return S3R_OK;
}

// device address of a pointer into the (mapped) staging buffer
void* mapped(s3r_ctx* c, void* host) { return c->h_stage_dev + ((char*)host - c->h_stage); }

void* stage_alloc(s3r_ctx* c, size_t bytes)
{
    size_t off = (c->h_stage_top + 255) & ~size_t(255);
    c->h_stage_top = off + bytes;
    return c->h_stage + off;
}

int* next_ticket(s3r_ctx* c)
{
    // sized per batch by construction; running out is an internal error that
    // render_impl reports (S3R_EINTERNAL) instead of writing past the buffer
    if (c->ticket_slot >= c->ticket_cap) {
        c->ticket_overflow = true;
        return c->p_ticket;
    }
    return c->p_ticket + (c->ticket_slot++);
}

// NVTX range per stage (host-side enqueue span; free without a tool attached)
const char* const kStageName[S3R_NUM_STAGES] = {"s3r.filter", "s3r.project", "s3r.depth_sort",
                                                "s3r.bin", "s3r.raster", "s3r.color"};

void ev_begin(s3r_ctx* c, int stage, cudaStream_t st, StageEvent& e)
{
    nvtxRangePushA(kStageName[stage]);
    e.stage = -1;
    if (!c->timing || c->capture_now) return;
    if (c->ev.size() > 200000) return;
    e.stage = stage;
    cudaEventCreate(&e.a);
    cudaEventCreate(&e.b);
    cudaEventRecord(e.a, st);
}
void ev_end(s3r_ctx* c, cudaStream_t st, StageEvent& e)
{
    nvtxRangePop();
    if (e.stage < 0) return;
    cudaEventRecord(e.b, st);
    c->ev.push_back(e);
}

int validate(s3r_ctx* c, const s3r_scene* s, const s3r_view* views, int nv,
             const s3r_outputs* outs)
{
    if (!s) return fail(c, S3R_EINVAL, "scene is NULL");
    if (s->n < 0 || s->n >= (1ll << 30)) return fail(c, S3R_EINVAL, "n = %lld out of [0, 2^30)", (long long)s->n);
    if (s->num_instances < 1 || s->num_instances > 4096)
        return fail(c, S3R_EINVAL, "num_instances = %d out of [1, 4096]", s->num_instances);
    if (s->n > 0) {
        const void* req[] = {s->means_opacity, s->scales, s->rotations, s->colors, s->visibility};
        const char* nm[] = {"means_opacity", "scales", "rotations", "colors", "visibility"};
        for (int i = 0; i < 5; ++i) {
            if (!req[i]) return fail(c, S3R_EINVAL, "scene.%s is NULL", nm[i]);
            if (!aligned(req[i], 16)) return fail(c, S3R_EINVAL, "scene.%s is not 16-byte aligned", nm[i]);
        }
        if (!s->instance_ids || !aligned(s->instance_ids, 4))
            return fail(c, S3R_EINVAL, "scene.instance_ids is NULL or misaligned");
        if (s->life && !aligned(s->life, 8)) return fail(c, S3R_EINVAL, "scene.life is not 8-byte aligned");
    }
    if (nv < 0) return fail(c, S3R_EINVAL, "n_views < 0");
    if (nv > 0 && (!views || !outs)) return fail(c, S3R_EINVAL, "views/outs is NULL");
    for (int v = 0; v < nv; ++v) {
        const s3r_view& V = views[v];
        if (V.width < 1 || V.width > 16384 || V.height < 1 || V.height > 16384)
            return fail(c, S3R_EINVAL, "view %d: size %dx%d out of [1,16384]", v, V.width, V.height);
        if (!(std::isfinite(V.fx) && V.fx > 0 && std::isfinite(V.fy) && V.fy > 0))
            return fail(c, S3R_EINVAL, "view %d: fx/fy must be finite and > 0", v);
        if (!(std::isfinite(V.cx) && std::isfinite(V.cy)))
            return fail(c, S3R_EINVAL, "view %d: cx/cy must be finite", v);
        if (!(V.t >= -1.0f && V.t <= 1.0f)) return fail(c, S3R_EINVAL, "view %d: t outside [-1,1]", v);
        if (!(std::isfinite(V.near_plane) && V.near_plane > 0))
            return fail(c, S3R_EINVAL, "view %d: near_plane must be finite and > 0", v);
        if (!V.instance_w2c || !aligned(V.instance_w2c, 4))
            return fail(c, S3R_EINVAL, "view %d: instance_w2c is NULL or misaligned", v);
        if (!std::isfinite(V.lod_r)) return fail(c, S3R_EINVAL, "view %d: lod_r not finite", v);
        if (!(V.lod_pmax >= 0.0f && V.lod_pmax <= 1.0f))
            return fail(c, S3R_EINVAL, "view %d: lod_pmax outside [0,1]", v);
        if (!(std::isfinite(V.lod_D) && V.lod_D > 0))
            return fail(c, S3R_EINVAL, "view %d: lod_D must be finite and > 0", v);
        const s3r_outputs& O = outs[v];
        if (!O.rgb || !aligned(O.rgb, 4)) return fail(c, S3R_EINVAL, "outs[%d].rgb is NULL or misaligned", v);
        if (O.depth && !aligned(O.depth, 4)) return fail(c, S3R_EINVAL, "outs[%d].depth misaligned", v);
        if (O.final_T && !aligned(O.final_T, 4)) return fail(c, S3R_EINVAL, "outs[%d].final_T misaligned", v);
    }
    return S3R_OK;
}

int bits_for(long long x)   // bits needed to hold values in [0, x)
{
    int b = 0;
    while ((1ll << b) < x) ++b;
    return std::max(b, 1);
}

int render_impl(s3r_ctx* c, const s3r_scene* sc, const s3r_view* views, int nv,
                const s3r_outputs* outs, cudaStream_t st)
{
    int rc = validate(c, sc, views, nv, outs);
    if (rc) return rc;
    CU(cudaSetDevice(c->device));
    c->last_stream = st;
    c->have_render = false;
    c->host_chunked = false;
    c->cap_pending = false;
    const long long N = sc->n;
    c->N_last = N;
    c->ticket_slot = 0;
    c->ticket_overflow = false;
    c->last_debug = c->debug;
    c->gbits = bits_for(std::max<long long>(N, 2));   // Gaussian-index bits of the depth key
    const bool conv = c->pipeline == S3R_PIPELINE_CONVENTIONAL;
    c->last_pipeline = c->pipeline;
    c->last_jitter = !conv && (c->lod_jitter[0] != 0.0f || c->lod_jitter[1] != 0.0f ||
                               c->lod_jitter[2] != 0.0f);
    const bool neurf = c->neurf && !conv;
    c->last_neurf = neurf;
    if (neurf && sc->num_instances > c->neurf_ninst)
        return fail(c, S3R_EINVAL, "NeurF: class table has %d rows, scene has %d instances",
                    c->neurf_ninst, sc->num_instances);
    // capacity mode: every size below comes from the reservation and the device
    // plans the batch (k_plan.cu); the modes that need the per-view layout on
    // the host (dumps, training, NeurF, the conventional world copies) keep the
    // synchronous sizing
    const bool capm = c->cap_on && !c->cap_suspend && !c->debug && !c->training && !neurf && !conv;
    c->last_capm = capm;

    // ---- distinct times (views sharing t share K1's compaction); the
    // conventional pipeline has no temporal filter: one identity list
    std::vector<float> tk;
    std::vector<int> slot(nv);
    for (int v = 0; v < nv; ++v) {
        const float t = conv ? 0.0f : views[v].t + 0.0f;
        int s = -1;
        for (size_t i = 0; i < tk.size(); ++i)
            if (tk[i] == t) { s = (int)i; break; }
        if (s < 0) { s = (int)tk.size(); tk.push_back(t); }
        slot[v] = s;
    }
    const int T = (int)tk.size();

    c->hv.assign(nv, DevView{});
    long long total_px = 0;
    int total_bins = 0, total_tiles = 0, max_bins = 0, max_tiles = 0;
    for (int v = 0; v < nv; ++v) {
        const s3r_view& V = views[v];
        DevView& d = c->hv[v];
        d.t = V.t + 0.0f;
        d.W = V.width; d.H = V.height;
        d.fx = V.fx; d.fy = V.fy; d.cx = V.cx; d.cy = V.cy; d.near_plane = V.near_plane;
        d.table = V.instance_w2c;
        d.lod_r = conv ? 0.0f : V.lod_r;          // no LOD in the conventional pipeline
        d.lod_pmax = V.lod_pmax; d.lod_D = V.lod_D;
        for (int a = 0; a < 3; ++a) d.jit[a] = conv ? 0.0f : c->lod_jitter[a];
        d.seed = (unsigned long long)V.lod_seed;
        d.tslot = slot[v];
        d.TX = (V.width + TILE - 1) / TILE;
        d.TY = (V.height + TILE - 1) / TILE;
        d.ntiles = d.TX * d.TY;
        // supertile edge S = 2^sshift tiles: the smallest S >= 4 with <= MAX_BINS bins
        d.sshift = 2;
        while (((d.TX + (1 << d.sshift) - 1) >> d.sshift) *
                   ((d.TY + (1 << d.sshift) - 1) >> d.sshift) > MAX_BINS)
            ++d.sshift;
        d.STX = (d.TX + (1 << d.sshift) - 1) >> d.sshift;
        d.STY = (d.TY + (1 << d.sshift) - 1) >> d.sshift;
        d.nbins = d.STX * d.STY;
        d.range_off = total_bins;             // supertile ranges / tile ranges: image sizes only
        d.trange_off = total_tiles;
        total_bins += d.nbins;
        total_tiles += d.ntiles;
        max_bins = std::max(max_bins, d.nbins);
        max_tiles = std::max(max_tiles, d.ntiles);
        d.rgb = outs[v].rgb; d.depth = outs[v].depth; d.finalT = outs[v].final_T;
        d.visible = outs[v].visible;
        d.pix_off = total_px;
        total_px += (long long)d.W * d.H;
    }
    // capacity mode with every view small by reservation: k_small_sortbin plans
    // its own view from K2's counters (no k_plan_bins launch); each view gets a
    // fixed tile-list area of SMALL_WORK entries
    const bool self_plan = capm && small_view(c->cap.rendered_view, max_tiles);
    if (self_plan)
        for (int v = 0; v < nv; ++v) {
            c->hv[v].small = 1;
            c->hv[v].tlist_off = (long long)v * SMALL_WORK;
        }
    if (c->training) {
        if ((rc = ensure(c, c->d_train_T, (size_t)std::max(total_px, 1ll) * 4))) return rc;
        if ((rc = ensure(c, c->d_train_n, (size_t)std::max(total_px, 1ll) * 4))) return rc;
    }

    // staging layout for this batch
    const size_t stage_bytes = 8192 + (size_t)T * 16 + (size_t)nv * (3 * sizeof(DevView) + 256) +
                               (size_t)(nv + 1) * 64;
    if ((rc = stage_begin(c, stage_bytes + (capm ? (size_t)nv * (sizeof(ViewCounters) + 8) + 512 : 0),
                          st)))
        return rc;
    if (c->capture_now && !capm)
        return fail(c, S3R_ESTATE, "graph capture of a render needs the capacity mode "
                                   "(s3r_set_capacity) and no debug / training / NeurF / "
                                   "conventional pipeline");
    // one zeroed work counter per launch that takes tickets: the filter chunks
    // and the depth-sort passes
    // K1 groups: a small scene takes all T distinct times in one launch of
    // ceil(T / fgs) groups (one ticket each, all look-back words zeroed with the
    // arena); a large one ceil(T / MAX_TSLOTS) launches of one group
    const int fgs = conv ? MAX_TSLOTS : filter_groups(N, T);
    const bool f_grouped = fgs < MAX_TSLOTS;
    const int n_tickets = (T + fgs - 1) / fgs +
                          (32 + c->gbits + RADIX_BITS - 1) / RADIX_BITS;
    c->ticket_cap = n_tickets;
    if ((rc = ensure(c, c->d_err, sizeof(uint32_t)))) return rc;
    // the zeroed arena and the upload arena (16-byte aligned parts)
    const long long ntf_all = conv ? 0 : (N + filter_tile() - 1) / filter_tile();
    auto al16 = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t z_ticket = 0;
    const size_t z_counts = al16(z_ticket + (size_t)n_tickets * 4);
    const size_t z_lb1 = al16(z_counts + (size_t)std::max(T, 1) * 8);
    const size_t z_ctr = al16(z_lb1 + (size_t)(f_grouped ? std::max(T, 1)
                                                           : std::min(std::max(T, 1), MAX_TSLOTS)) *
                                          ntf_all * 4);
    const size_t z_end = al16(z_ctr + (size_t)std::max(nv, 1) * sizeof(ViewCounters));
    if ((rc = ensure(c, c->d_zero, z_end))) return rc;
    c->p_ticket = reinterpret_cast<int*>(P<char>(c->d_zero) + z_ticket);
    c->p_counts = reinterpret_cast<unsigned long long*>(P<char>(c->d_zero) + z_counts);
    c->p_lb1 = reinterpret_cast<uint32_t*>(P<char>(c->d_zero) + z_lb1);
    c->p_ctr = reinterpret_cast<ViewCounters*>(P<char>(c->d_zero) + z_ctr);
    CU(cudaMemsetAsync(c->d_zero.p, 0, z_end, st));
    const size_t u_views = al16((size_t)std::max(T, 1) * 4);
    const size_t u_end = u_views + (size_t)std::max(nv, 1) * sizeof(DevView);
    if ((rc = ensure(c, c->d_up, u_end))) return rc;
    c->p_times = P<float>(c->d_up);
    c->p_views = reinterpret_cast<DevView*>(P<char>(c->d_up) + u_views);

    // ================= K1: temporal filter + compaction
    const long long Ns = std::max<long long>(N, 1);
    if ((rc = ensure(c, c->d_tidx, (size_t)std::max(T, 1) * Ns * sizeof(int32_t)))) return rc;
    // the upload arena's image in staging: [times | views]; the capacity mode
    // sends it whole now (the device fills in the per-view sizes), the
    // synchronous mode sends the times now and the sized views after K1
    char* h_up = (char*)stage_alloc(c, u_end);
    float* h_times = reinterpret_cast<float*>(h_up);
    for (int i = 0; i < T; ++i) h_times[i] = tk[i];
    if (capm) {
        std::memcpy(h_up + u_views, c->hv.data(), (size_t)nv * sizeof(DevView));
        CU(cudaMemcpyAsync(c->d_up.p, h_up, u_end, cudaMemcpyHostToDevice, st));
    } else if (T) {
        CU(cudaMemcpyAsync(c->p_times, h_times, T * sizeof(float), cudaMemcpyHostToDevice, st));
    }
    unsigned long long* h_counts =
        (unsigned long long*)stage_alloc(c, (size_t)std::max(T, 1) * sizeof(unsigned long long));
    if (conv) {
        // no temporal filter: every Gaussian is projected (identity list)
        StageEvent e;
        ev_begin(c, S3R_STAGE_FILTER, st, e);
        launch_iota(P<int32_t>(c->d_tidx), N, st);
        ev_end(c, st, e);
        h_counts[0] = (unsigned long long)N;
    } else {
        StageEvent e;
        ev_begin(c, S3R_STAGE_FILTER, st, e);
        const long long ntf = (N + filter_tile() - 1) / filter_tile();
        if (f_grouped && N > 0) {
            const int ng = (T + fgs - 1) / fgs;
            int* tk0 = next_ticket(c);
            for (int g = 1; g < ng; ++g) next_ticket(c);      // consecutive tickets
            launch_filter(reinterpret_cast<const float2*>(sc->visibility), N, c->p_times, T, fgs,
                          P<int32_t>(c->d_tidx), Ns, c->p_counts, c->p_lb1, tk0, st);
        }
        for (int c0 = 0; !f_grouped && c0 < T && N > 0; c0 += MAX_TSLOTS) {
            const int Tc = std::min(MAX_TSLOTS, T - c0);
            // look-back words: zeroed with the arena for the first chunk of
            // distinct times, re-zeroed for later ones
            if (c0) CU(cudaMemsetAsync(c->p_lb1, 0, (size_t)Tc * ntf * sizeof(uint32_t), st));
            launch_filter(reinterpret_cast<const float2*>(sc->visibility), N,
                          c->p_times + c0, Tc, Tc, P<int32_t>(c->d_tidx) + (long long)c0 * Ns,
                          Ns, c->p_counts + c0, c->p_lb1, next_ticket(c), st);
        }
        ev_end(c, st, e);
        CU(cudaGetLastError());
        if (!capm) {
            if (T) launch_readback(mapped(c, h_counts), c->p_counts, T * sizeof(unsigned long long), st);
            CU(cudaStreamSynchronize(st));
        }
    }

    // ================= K2: projection + LOD + life + compaction
    long long cap = 0;
    int k2_tiles = 0;          // grid.x of K2 (grid.y = views)
    if (capm) {
        cap = c->cap.records;
        k2_tiles = (int)std::max<long long>(1, (c->cap.temporal_view + project_tile() - 1) / project_tile());
    } else {
        for (int v = 0; v < nv; ++v) {
            DevView& d = c->hv[v];
            d.n_temporal = (long long)h_counts[d.tslot];
            d.cap_off = cap;
            d.dbg_off = cap;
            cap += d.n_temporal;
            k2_tiles = std::max(k2_tiles, (int)((d.n_temporal + project_tile() - 1) / project_tile()));
        }
    }
    const long long capS = std::max<long long>(cap, 1);
    if ((rc = ensure(c, c->d_rec, (size_t)capS * 48))) return rc;
    if ((rc = ensure(c, c->d_dkey, (size_t)capS * 8))) return rc;
    if (c->debug && (rc = ensure(c, c->d_gidx, (size_t)capS * 4))) return rc;
    // per-record own-frame means: the NeurF query, and the backward of a
    // training render under the noisy offset (the projection adjoint runs at the
    // moved mean)
    const bool want_mu = neurf || (c->training && c->last_jitter);
    c->last_recmu = want_mu;
    if (want_mu && (rc = ensure(c, c->d_recmu, (size_t)capS * 16))) return rc;
    if (c->debug) {
        if ((rc = ensure(c, c->d_dbg_keys, (size_t)capS * 24))) return rc;
        if ((rc = ensure(c, c->d_dbg_flags, (size_t)capS))) return rc;
        if ((rc = ensure(c, c->d_dbg_rect, (size_t)capS * 8))) return rc;
    }
    if (!capm && nv) {
        // the sized views (the K2 counters were zeroed with the arena); the
        // capacity mode uploaded them with the times and plans them on the device
        DevView* h_views = (DevView*)stage_alloc(c, (size_t)std::max(nv, 1) * sizeof(DevView));
        std::memcpy(h_views, c->hv.data(), (size_t)nv * sizeof(DevView));
        CU(cudaMemcpyAsync(c->p_views, h_views, nv * sizeof(DevView), cudaMemcpyHostToDevice, st));
    }
    for (int v = 0; v < nv; ++v)
        if (outs[v].visible && N > 0) CU(cudaMemsetAsync(outs[v].visible, 0, (size_t)N, st));
    if (capm) {
        // record segments on the device from K1's counts
        c->cap_h_ntemp = (long long*)stage_alloc(c, (size_t)std::max(nv, 1) * 8);
        launch_plan_records(c->p_views, nv, c->p_counts,
                            c->cap.records, c->cap.temporal_view,
                            (long long*)mapped(c, c->cap_h_ntemp),
                            P<uint32_t>(c->d_err), st);
    }
    if (conv && N > 0 && nv > 0) {
        // ---- C0: local-to-world transformation of every view's Gaussians
        if ((rc = ensure(c, c->d_wmo, (size_t)nv * N * 16))) return rc;
        if ((rc = ensure(c, c->d_wrot, (size_t)nv * N * 16))) return rc;
        StageEvent e;
        ev_begin(c, S3R_STAGE_PROJECT, st, e);
        launch_world(reinterpret_cast<const float4*>(sc->means_opacity),
                     reinterpret_cast<const float4*>(sc->rotations), sc->instance_ids,
                     sc->num_instances, N, c->p_views, nv, P<float4>(c->d_wmo),
                     P<float4>(c->d_wrot), st);
        ev_end(c, st, e);
    }
    {
        ProjectArgs a{};
        a.world_mo = conv ? P<float4>(c->d_wmo) : nullptr;
        a.world_rot = conv ? P<float4>(c->d_wrot) : nullptr;
        a.rec_mu = want_mu ? P<float4>(c->d_recmu) : nullptr;
        a.means_opacity = reinterpret_cast<const float4*>(sc->means_opacity);
        a.scales = reinterpret_cast<const float4*>(sc->scales);
        a.rotations = reinterpret_cast<const float4*>(sc->rotations);
        a.colors = reinterpret_cast<const float4*>(sc->colors);
        a.ids = sc->instance_ids;
        a.life = reinterpret_cast<float2*>(sc->life);
        a.num_instances = sc->num_instances;
        a.n = N;
        a.views = c->p_views;
        a.n_views = nv;
        a.tidx = P<int32_t>(c->d_tidx);
        a.idx_stride = Ns;
        a.max_tiles = k2_tiles;
        a.rec = P<float4>(c->d_rec);
        a.dkey = P<unsigned long long>(c->d_dkey);
        a.gbits = c->gbits;
        a.gidx = c->debug ? P<int32_t>(c->d_gidx) : nullptr;
        a.counters = c->p_ctr;
        a.err = P<uint32_t>(c->d_err);
        a.dbg_keys = c->debug ? P<float>(c->d_dbg_keys) : nullptr;
        a.dbg_flags = c->debug ? P<uint8_t>(c->d_dbg_flags) : nullptr;
        a.dbg_rect = c->debug ? P<int16_t>(c->d_dbg_rect) : nullptr;
        a.lean = (!conv && !want_mu && !c->debug && c->lod_jitter[0] == 0.0f &&
                  c->lod_jitter[1] == 0.0f && c->lod_jitter[2] == 0.0f) ? 1 : 0;
        StageEvent e;
        ev_begin(c, S3R_STAGE_PROJECT, st, e);
        launch_project(a, st);
        ev_end(c, st, e);
    }
    CU(cudaGetLastError());
    ViewCounters* h_ctr = (ViewCounters*)stage_alloc(c, (size_t)std::max(nv, 1) * sizeof(ViewCounters));
    // ================= sizes of the sort / emit / raster phase
    c->stats.assign(nv, s3r_stats{});
    std::vector<int> dt0(nv + 1, 0);
    long long total_pairs = 0, total_cnt = 0, max_r = 0;
    int max_chunks = 0;
    long long total_tlist = 0;
    bool bad = false;
    const int stile = onesweep64_tile();
    int dtiles = 0;
    bool any_small = false, all_small = true;   // views for k_small.cu / for the big path
    if ((rc = ensure(c, c->d_dsegs, (size_t)std::max(nv, 1) * sizeof(Seg)))) return rc;
    if ((rc = ensure(c, c->d_dtile0, (size_t)(nv + 1) * sizeof(int)))) return rc;
    if (capm) {
        // the device plans the rest (k_plan_bins); the host sizes every buffer and
        // grid from the reservation
        max_r = c->cap.rendered_view;
        max_chunks = (int)((max_r + bin_chunk() - 1) / bin_chunk());
        for (int v = 0; v < nv; ++v) total_cnt += (long long)c->hv[v].nbins * max_chunks;
        total_pairs = c->cap.bin_pairs;
        total_tlist = c->cap.tile_entries;
        // sort tiles: sum over views of ceil(n_rendered / stile), bounded by both
        // the records and the per-view rendered capacity
        dtiles = (int)std::min<long long>((cap + stile - 1) / stile + nv,
                                          (long long)nv * ((max_r + stile - 1) / stile));
        // which views the device will mark small is not known here: launch the
        // one-CTA path whenever a view may be small, the big path unless all are
        any_small = false;
        for (int v = 0; v < nv; ++v) any_small = any_small || small_view(0, c->hv[v].ntiles);
        all_small = small_view(max_r, max_tiles);
        if (all_small) dtiles = 0;
        if (self_plan) total_tlist = (long long)std::max(nv, 1) * SMALL_WORK;
        PlanCaps pc;
        pc.rendered_view = max_r;
        pc.bin_pairs = total_pairs;
        pc.tile_entries = total_tlist;
        pc.counts = total_cnt;
        pc.bin_chunk = bin_chunk();
        pc.sort_tile = stile;
        c->cap_h_ctr = h_ctr;
        if (!self_plan)
            launch_plan_bins(c->p_views, nv, c->p_ctr, P<Seg>(c->d_dsegs),
                             P<int>(c->d_dtile0), pc, (ViewCounters*)mapped(c, h_ctr),
                             P<uint32_t>(c->d_err), st);
        c->cap_pending = true;
    } else {
        if (nv) launch_readback(mapped(c, h_ctr), c->p_ctr, nv * sizeof(ViewCounters), st);
        CU(cudaStreamSynchronize(st));
        for (int v = 0; v < nv; ++v) {
            DevView& d = c->hv[v];
            const ViewCounters& k = h_ctr[v];
            d.n_rendered = (long long)k.n_rendered;
            d.n_pairs = (long long)k.n_pairs;
            if (d.n_pairs >= (1ll << 31))
                return fail(c, S3R_EINVAL, "view %d: %lld tile pairs exceed 2^31", v, d.n_pairs);
            d.small = small_view(d.n_rendered, d.ntiles) ? 1 : 0;
            any_small = any_small || d.small;
            all_small = all_small && d.small;
            d.nchunks = d.small ? 0 : (int)((d.n_rendered + bin_chunk() - 1) / bin_chunk());
            d.cnt_off = total_cnt;
            d.pair_off = total_pairs;
            d.tlist_off = total_tlist;
            const long long SS = 1ll << (2 * d.sshift);
            if (SS * (long long)k.n_spairs >= (1ll << 31))
                return fail(c, S3R_EINVAL, "view %d: tile-list area exceeds 2^31 entries", v);
            total_tlist += SS * (long long)k.n_spairs;
            total_cnt += (long long)d.nbins * d.nchunks;
            total_pairs += (long long)k.n_spairs;
            max_chunks = std::max(max_chunks, d.nchunks);
            max_r = std::max(max_r, d.n_rendered);
            dt0[v + 1] = dt0[v] + (d.small ? 0 : (int)((d.n_rendered + stile - 1) / stile));
            s3r_stats& s = c->stats[v];
            s.n_scene = N;
            s.n_temporal = d.n_temporal;
            s.n_visible = (long long)k.n_visible;
            s.n_lod_small = (long long)k.n_small;
            s.n_lod_dropped = (long long)k.n_dropped;
            s.n_rendered = d.n_rendered;
            s.n_pairs = d.n_pairs;
            s.n_bin_pairs = (long long)k.n_spairs;
            s.n_bad_instance = (long long)k.n_bad;
            if (k.n_bad) bad = true;
        }
        dtiles = dt0[nv];
        // device-side metadata for the rest of the batch
        Seg* h_dsegs = (Seg*)stage_alloc(c, (size_t)std::max(nv, 1) * sizeof(Seg));
        int* h_dt0 = (int*)stage_alloc(c, (size_t)(nv + 1) * sizeof(int));
        DevView* h_views2 = (DevView*)stage_alloc(c, (size_t)std::max(nv, 1) * sizeof(DevView));
        for (int v = 0; v < nv; ++v) {
            const DevView& d = c->hv[v];
            h_dsegs[v] = Seg{d.cap_off, d.small ? 0 : d.n_rendered, dt0[v], dt0[v + 1] - dt0[v]};
        }
        std::memcpy(h_dt0, dt0.data(), (nv + 1) * sizeof(int));
        std::memcpy(h_views2, c->hv.data(), (size_t)nv * sizeof(DevView));
        if (nv) {
            CU(cudaMemcpyAsync(c->d_dsegs.p, h_dsegs, nv * sizeof(Seg), cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(c->d_dtile0.p, h_dt0, (nv + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
            CU(cudaMemcpyAsync(c->p_views, h_views2, nv * sizeof(DevView), cudaMemcpyHostToDevice, st));
        }
        // what this batch needed (s3r_capacity_from_last)
        s3r_capacity need{};
        need.records = cap;
        need.bin_pairs = total_pairs;
        need.tile_entries = total_tlist;
        for (int v = 0; v < nv; ++v) {
            need.rendered_view = std::max<long long>(need.rendered_view, c->hv[v].n_rendered);
            need.temporal_view = std::max<long long>(need.temporal_view, c->hv[v].n_temporal);
        }
        c->last_need = need;
        c->last_need_valid = true;
    }
    for (int i = 0; i < 2; ++i) {
        if ((rc = ensure(c, c->d_sortk[i], (size_t)capS * 8))) return rc;
        if ((rc = ensure(c, c->d_sortv[i], (size_t)capS * 4))) return rc;
    }
    if ((rc = ensure(c, c->d_recs, (size_t)capS * 48))) return rc;
    if ((rc = ensure(c, c->d_rects, (size_t)capS * 8))) return rc;
    if ((rc = ensure(c, c->d_lists, (size_t)std::max<long long>(total_pairs, 1) * 4))) return rc;
    if ((rc = ensure(c, c->d_tlists, (size_t)std::max<long long>(total_tlist, 1) * 4))) return rc;
    if ((rc = ensure(c, c->d_tranges, (size_t)std::max(total_tiles, 1) * sizeof(int2)))) return rc;
    if ((rc = ensure(c, c->d_cnt, (size_t)std::max<long long>(total_cnt, 1) * 4))) return rc;
    const int dpasses = (32 + c->gbits + RADIX_BITS - 1) / RADIX_BITS;
    if ((rc = ensure(c, c->d_hist, (size_t)std::max(nv, 1) * dpasses * RADIX * 4))) return rc;
    if ((rc = ensure(c, c->d_ranges, (size_t)std::max(total_bins, 1) * sizeof(int2)))) return rc;
    if ((rc = ensure(c, c->d_lb, (size_t)std::max(dtiles, 1) * RADIX * sizeof(uint32_t)))) return rc;

    // ================= K6: NeurF colour query (NEXT-4) into the compacted records
    if (neurf && nv) {
        int* h_toff = (int*)stage_alloc(c, (size_t)(nv + 1) * sizeof(int));
        int tt = 0;
        for (int v = 0; v < nv; ++v) {
            h_toff[v] = tt;
            tt += (int)((c->hv[v].n_rendered + 127) / 128);
        }
        h_toff[nv] = tt;
        if ((rc = ensure(c, c->d_toff, (size_t)(nv + 1) * sizeof(int)))) return rc;
        CU(cudaMemcpyAsync(c->d_toff.p, h_toff, (nv + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
        StageEvent e;
        ev_begin(c, S3R_STAGE_COLOR, st, e);
        NeurfArgs na{};
        na.views = c->p_views;
        na.n_views = nv;
        na.tile_off = P<int>(c->d_toff);
        na.total_tiles = tt;
        na.rec_mu = P<float4>(c->d_recmu);
        na.rec = P<float4>(c->d_rec);
        na.wpack = c->d_nw.p;
        na.bias = P<float>(c->d_nb);
        na.time_emb = P<float>(c->d_temb);
        na.n_time = c->neurf_ntime;
        na.class_emb = P<float>(c->d_cemb);
        na.pos_scale = c->neurf_scale;
        launch_neurf(na, st);
        ev_end(c, st, e);
        CU(cudaGetLastError());
    }

    const int dpasses_run = all_small ? 0 : dpasses;
    c->final_order = (dpasses - 1) & 1;
    // ================= a4 of the small views: one CTA each (k_small.cu)
    if (any_small && nv) {
        StageEvent e;
        ev_begin(c, S3R_STAGE_DEPTH_SORT, st, e);
        SmallPlan sp{};
        if (self_plan) {
            sp.ctr = c->p_ctr;
            sp.h_ctr = (ViewCounters*)mapped(c, h_ctr);
            sp.err = P<uint32_t>(c->d_err);
            sp.cap_rendered = c->cap.rendered_view;
        }
        launch_small_sortbin(c->p_views, nv, P<unsigned long long>(c->d_dkey),
                             P<float4>(c->d_rec), P<unsigned long long>(c->d_sortk[c->final_order]),
                             P<uint32_t>(c->d_sortv[c->final_order]), P<float4>(c->d_recs),
                             P<uint2>(c->d_rects), P<uint32_t>(c->d_tlists),
                             P<int2>(c->d_tranges), sp, st);
        ev_end(c, st, e);
    }
    // ================= K5a: depth sort: 8-bit LSD passes over (depth << gbits | index),
    // values = compacted slot j; gives the unique (depth, index) order (R11)
    if (!all_small) {
        StageEvent e;
        ev_begin(c, S3R_STAGE_DEPTH_SORT, st, e);
        CU(cudaMemsetAsync(c->d_hist.p, 0, (size_t)std::max(nv, 1) * dpasses * RADIX * 4, st));
        launch_hist64(P<unsigned long long>(c->d_dkey), P<Seg>(c->d_dsegs), nv,
                      P<int>(c->d_dtile0), dtiles, 0, dpasses, P<uint32_t>(c->d_hist), st);
        launch_hist_scan(P<uint32_t>(c->d_hist), nv, dpasses, st);
        const unsigned long long* kin = P<unsigned long long>(c->d_dkey);
        const uint32_t* vin = nullptr;
        for (int pass = 0; pass < dpasses_run; ++pass) {
            const int o = pass & 1;
            if (dtiles) CU(cudaMemsetAsync(c->d_lb.p, 0, (size_t)dtiles * RADIX * 4, st));
            launch_onesweep64kv(kin, vin, P<unsigned long long>(c->d_sortk[o]),
                                P<uint32_t>(c->d_sortv[o]), P<Seg>(c->d_dsegs), nv,
                                P<int>(c->d_dtile0), dtiles, P<uint32_t>(c->d_hist), pass,
                                dpasses, P<uint32_t>(c->d_lb), next_ticket(c), 8 * pass, st);
            kin = P<unsigned long long>(c->d_sortk[o]);
            vin = P<uint32_t>(c->d_sortv[o]);
        }
        ev_end(c, st, e);
    }
    CU(cudaGetLastError());

    // ================= K3/K4: depth-ordered permute + supertile counting sort
    if (!all_small) {
        StageEvent e;
        ev_begin(c, S3R_STAGE_BIN, st, e);
        launch_permute(c->p_views, nv, max_r, P<uint32_t>(c->d_sortv[c->final_order]),
                       P<float4>(c->d_rec), P<float4>(c->d_recs), P<uint2>(c->d_rects), st);
        launch_bin(c->p_views, nv, max_chunks, max_bins, P<uint2>(c->d_rects),
                   P<uint32_t>(c->d_cnt), P<int2>(c->d_ranges), P<uint32_t>(c->d_lists),
                   P<uint32_t>(c->d_tlists), P<int2>(c->d_tranges), st);
        ev_end(c, st, e);
    }
    CU(cudaGetLastError());

    // ================= K7: rasterizer
    {
        StageEvent e;
        ev_begin(c, S3R_STAGE_RASTER, st, e);
        RasterArgs a{};
        a.views = c->p_views;
        a.n_views = nv;
        a.max_tiles = max_tiles;
        a.tranges = P<int2>(c->d_tranges);
        a.tlists = P<uint32_t>(c->d_tlists);
        a.rec_sorted = P<float4>(c->d_recs);
        a.evals = nullptr;
        if (c->counters && nv) {
            if ((rc = ensure(c, c->d_evals, (size_t)nv * 16))) return rc;
            CU(cudaMemsetAsync(c->d_evals.p, 0, (size_t)nv * 16, st));
            a.evals = P<unsigned long long>(c->d_evals);
        }
        a.train_T = c->training ? P<float>(c->d_train_T) : nullptr;
        a.train_n = c->training ? P<int>(c->d_train_n) : nullptr;
        a.fast_exp = c->fast_exp ? 1 : 0;
        launch_raster(a, st);
        ev_end(c, st, e);
        c->last_counters = a.evals != nullptr;
        c->evals_fetched = false;
    }
    CU(cudaGetLastError());
    c->last_training = c->training;
    c->last_nviews = nv;
    c->last_max_tiles = max_tiles;
    c->last_max_r = max_r;
    c->last_N = N;
    if (c->timing && !c->capture_now) c->timed_renders++;
    if ((rc = stage_end(c, st))) return rc;
    c->have_render = true;
    if (c->ticket_overflow) return fail(c, S3R_EINTERNAL, "work-counter slots exhausted");
    if (bad) return fail(c, S3R_EINSTANCE, "a Gaussian had an instance id outside [0, %d]",
                         sc->num_instances - 1);
    c->err.clear();
    return S3R_OK;
}

}  // namespace

// ============================================================== C ABI
extern "C" {

int s3r_version(void) { return S3R_VERSION; }

int s3r_create(int device, s3r_ctx** out)
{
    if (!out) return S3R_EINVAL;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return S3R_ECUDA;
    }
    s3r_ctx* c = new (std::nothrow) s3r_ctx();
    if (!c) return S3R_ENOMEM;
    c->device = device;
    if (const char* e = std::getenv("S3R_OVERLAP")) c->overlap = e[0] && e[0] != '0';
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return S3R_ECUDA;
    }
    if (ensure(c, c->d_err, sizeof(uint32_t)) || cudaMemset(c->d_err.p, 0, sizeof(uint32_t)) != cudaSuccess) {
        delete c;
        return S3R_ECUDA;
    }
    *out = c;
    return S3R_OK;
}

void s3r_destroy(s3r_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->twin) s3r_destroy(c->twin);
    if (c->twin_stream) cudaStreamDestroy(c->twin_stream);
    if (c->fork_ev) cudaEventDestroy(c->fork_ev);
    if (c->join_ev) cudaEventDestroy(c->join_ev);
    Buf* bufs[] = {&c->d_nw, &c->d_nb, &c->d_temb, &c->d_cemb, &c->d_recmu, &c->d_toff,
                   &c->d_wmo, &c->d_wrot, &c->d_zero, &c->d_up, &c->d_tidx, &c->d_lb,
                   &c->d_rec, &c->d_dkey, &c->d_gidx, &c->d_sortk[0], &c->d_sortk[1],
                   &c->d_sortv[0], &c->d_sortv[1], &c->d_recs, &c->d_rects, &c->d_lists,
                   &c->d_tlists, &c->d_tranges, &c->d_train_T, &c->d_train_n, &c->d_sgrads,
                   &c->d_cots,
                   &c->d_cnt, &c->d_hist, &c->d_dsegs, &c->d_dtile0, &c->d_ranges, &c->d_err,
                   &c->d_dbg_keys, &c->d_dbg_flags, &c->d_dbg_rect, &c->d_dbg_tcnt, &c->d_evals};
    for (Buf* b : bufs)
        if (b->p) cudaFree(b->p);
    for (auto& b : c->m_scene)
        if (b.p) cudaFree(b.p);
    for (auto* vec : {&c->m_tab, &c->m_rgb, &c->m_depth, &c->m_T, &c->m_vis})
        for (auto& b : *vec)
            if (b.p) cudaFree(b.p);
    for (auto& e : c->ev) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    for (auto& S : c->ring) {
        if (S.h) cudaFreeHost(S.h);
        if (S.ev) cudaEventDestroy(S.ev);
    }
    for (char* h : c->graph_blocks) cudaFreeHost(h);
    if (c->graph_spare) cudaFreeHost(c->graph_spare);
    for (cudaEvent_t e : c->chunk_done) cudaEventDestroy(e);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    delete c;
}

const char* s3r_last_error(const s3r_ctx* c) { return c ? c->err.c_str() : "null context"; }

int s3r_set_debug(s3r_ctx* c, int enable)
{
    if (!c) return S3R_EINVAL;
    c->debug = enable != 0;
    return S3R_OK;
}

int s3r_set_counters(s3r_ctx* c, int enable)
{
    if (!c) return S3R_EINVAL;
    c->counters = enable != 0;
    return S3R_OK;
}

int s3r_set_timing(s3r_ctx* c, int enable)
{
    if (!c) return S3R_EINVAL;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto& e : c->ev) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    c->ev.clear();
    for (double& m : c->stage_ms) m = 0;
    c->timed_renders = 0;
    c->timing = enable != 0;
    if (c->twin) s3r_set_timing(c->twin, enable);
    return S3R_OK;
}

int s3r_get_stage_times(s3r_ctx* c, double* out_ms, int64_t* out_count)
{
    if (!c) return S3R_EINVAL;
    CU(cudaSetDevice(c->device));
    cudaError_t err = cudaSuccess;
    for (auto& e : c->ev) {       // every event is consumed (and destroyed) once
        float ms = 0;
        if (err == cudaSuccess) err = cudaEventSynchronize(e.b);
        if (err == cudaSuccess) err = cudaEventElapsedTime(&ms, e.a, e.b);
        if (err == cudaSuccess) c->stage_ms[e.stage] += ms;
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    c->ev.clear();
    if (err != cudaSuccess)
        return fail(c, S3R_ECUDA, "get_stage_times: %s", cudaGetErrorString(err));
    if (c->twin) {            // the second halves of overlapped batches
        double tw[S3R_NUM_STAGES];
        int64_t tc = 0;
        if (int r = s3r_get_stage_times(c->twin, tw, &tc)) return fail(c, r, "%s", c->twin->err.c_str());
        for (int i = 0; i < S3R_NUM_STAGES; ++i) c->stage_ms[i] += tw[i];
        c->twin->stage_ms[0] = 0;
        for (double& m : c->twin->stage_ms) m = 0;
    }
    if (out_ms)
        for (int i = 0; i < S3R_NUM_STAGES; ++i) out_ms[i] = c->stage_ms[i];
    if (out_count) *out_count = c->timed_renders;
    return S3R_OK;
}

int s3r_compose_instance_cameras(s3r_ctx* c, const float* w2c, const float* i2g, int32_t n_views,
                                 int32_t K, float* out, void* stream)
{
    if (!c) return S3R_EINVAL;
    if (n_views < 0 || K < 0 || K > 4095 || (n_views > 0 && (!w2c || !out)) ||
        (n_views > 0 && K > 0 && !i2g))
        return fail(c, S3R_EINVAL, "compose: bad arguments");
    CU(cudaSetDevice(c->device));
    launch_compose(w2c, i2g, n_views, K, out, (cudaStream_t)stream);
    CU(cudaGetLastError());
    return S3R_OK;
}

int s3r_render_batch(s3r_ctx* c, const s3r_scene* scene, const s3r_view* views, int32_t n_views,
                     const s3r_outputs* outs, void* stream)
{
    if (!c) return S3R_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    // Overlapped halves: the second half renders in the twin context on its own
    // stream, forked from and joined back into `stream`, so its latency-bound
    // front stages (K1-K5, with their two host syncs) overlap the first half's
    // compute-bound rasterization.  Modes whose state must describe one batch
    // (debug dumps, counters, training, NeurF) render in one piece.
    const bool split = c->overlap && n_views >= 16 && !c->debug && !c->counters &&
                       !c->training && !c->neurf && !c->cap_on;   // (the capacity mode has no host syncs to hide)
    if (!split) return render_impl(c, scene, views, n_views, outs, st);
    CU(cudaSetDevice(c->device));
    if (!c->twin) {
        int rc = s3r_create(c->device, &c->twin);
        if (rc) return fail(c, rc, "overlap: creating the twin context failed");
        c->twin->overlap = false;
        CU(cudaStreamCreateWithFlags(&c->twin_stream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
    }
    s3r_ctx* t = c->twin;
    t->pipeline = c->pipeline;
    t->fast_exp = c->fast_exp;
    for (int a = 0; a < 3; ++a) t->lod_jitter[a] = c->lod_jitter[a];
    if (t->timing != c->timing) s3r_set_timing(t, c->timing);
    CU(cudaEventRecord(c->fork_ev, st));
    CU(cudaStreamWaitEvent(c->twin_stream, c->fork_ev, 0));
    const int n1 = n_views / 2;
    int rc1 = render_impl(c, scene, views, n1, outs, st);
    if (rc1 != S3R_OK && rc1 != S3R_EINSTANCE) return rc1;
    int rc2 = render_impl(t, scene, views + n1, n_views - n1, outs + n1, c->twin_stream);
    if (rc2 != S3R_OK && rc2 != S3R_EINSTANCE) {
        cudaStreamSynchronize(c->twin_stream);
        return fail(c, rc2, "%s", t->err.c_str());
    }
    CU(cudaEventRecord(c->join_ev, c->twin_stream));
    CU(cudaStreamWaitEvent(st, c->join_ev, 0));
    c->stats.insert(c->stats.end(), t->stats.begin(), t->stats.end());
    c->host_chunked = true;        // per-view intermediates live in two contexts
    return rc1 ? rc1 : rc2;
}

int s3r_render(s3r_ctx* c, const s3r_scene* scene, const s3r_view* view, const s3r_outputs* out,
               void* stream)
{
    if (!c) return S3R_EINVAL;
    return render_impl(c, scene, view, 1, out, (cudaStream_t)stream);
}

int s3r_render_batch_host(s3r_ctx* c, const s3r_scene* hs, const s3r_view* hviews,
                          int32_t nv, const s3r_outputs* houts, void* stream)
{
    if (!c) return S3R_EINVAL;
    if (!hs || nv < 0 || (nv > 0 && (!hviews || !houts)))
        return fail(c, S3R_EINVAL, "render_batch_host: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(c->device));
    const long long N = hs->n;
    if (N < 0 || N >= (1ll << 30)) return fail(c, S3R_EINVAL, "n out of range");
    // this entry point synchronises anyway and collects per-chunk stats on the
    // host: it keeps the synchronous sizing
    struct Suspend {
        s3r_ctx* c;
        ~Suspend() { c->cap_suspend = false; }
    } suspend_{c};
    c->cap_suspend = true;
    int rc;
    const size_t sz[7] = {16, 16, 16, 16, 4, 8, 8};
    const void* src[7] = {hs->means_opacity, hs->scales, hs->rotations, hs->colors,
                          hs->instance_ids, hs->visibility, hs->life};
    s3r_scene ds = *hs;
    void* dst[7];
    for (int i = 0; i < 7; ++i) {
        dst[i] = nullptr;
        if (!src[i] || N == 0) continue;
        if ((rc = ensure(c, c->m_scene[i], (size_t)N * sz[i]))) return rc;
        dst[i] = c->m_scene[i].p;
        CU(cudaMemcpyAsync(dst[i], src[i], (size_t)N * sz[i], cudaMemcpyHostToDevice, st));
    }
    ds.means_opacity = (const float*)dst[0];
    ds.scales = (const float*)dst[1];
    ds.rotations = (const float*)dst[2];
    ds.colors = (const float*)dst[3];
    ds.instance_ids = (const int32_t*)dst[4];
    ds.visibility = (float*)dst[5];
    ds.life = (float*)dst[6];
    c->m_tab.resize(std::max<size_t>(c->m_tab.size(), nv));
    c->m_rgb.resize(std::max<size_t>(c->m_rgb.size(), nv));
    c->m_depth.resize(std::max<size_t>(c->m_depth.size(), nv));
    c->m_T.resize(std::max<size_t>(c->m_T.size(), nv));
    c->m_vis.resize(std::max<size_t>(c->m_vis.size(), nv));
    std::vector<s3r_view> dv(hviews, hviews + nv);
    std::vector<s3r_outputs> dout(nv);
    for (int v = 0; v < nv; ++v) {
        const size_t tb = (size_t)hs->num_instances * 12 * sizeof(float);
        if (!hviews[v].instance_w2c || !houts[v].rgb)
            return fail(c, S3R_EINVAL, "render_batch_host: view %d has NULL table/rgb", v);
        if ((rc = ensure(c, c->m_tab[v], tb))) return rc;
        CU(cudaMemcpyAsync(c->m_tab[v].p, hviews[v].instance_w2c, tb, cudaMemcpyHostToDevice, st));
        dv[v].instance_w2c = P<float>(c->m_tab[v]);
        const size_t px = (size_t)std::max(hviews[v].width, 1) * std::max(hviews[v].height, 1);
        if ((rc = ensure(c, c->m_rgb[v], px * 12))) return rc;
        dout[v].rgb = P<float>(c->m_rgb[v]);
        if (houts[v].depth) {
            if ((rc = ensure(c, c->m_depth[v], px * 4))) return rc;
            dout[v].depth = P<float>(c->m_depth[v]);
        }
        if (houts[v].final_T) {
            if ((rc = ensure(c, c->m_T[v], px * 4))) return rc;
            dout[v].final_T = P<float>(c->m_T[v]);
        }
        if (houts[v].visible && N > 0) {
            if ((rc = ensure(c, c->m_vis[v], (size_t)N))) return rc;
            dout[v].visible = P<uint8_t>(c->m_vis[v]);
        }
    }
    auto d2h = [&](int v, cudaStream_t cs) -> int {
        const size_t px = (size_t)hviews[v].width * hviews[v].height;
        CU(cudaMemcpyAsync(houts[v].rgb, dout[v].rgb, px * 12, cudaMemcpyDeviceToHost, cs));
        if (houts[v].depth)
            CU(cudaMemcpyAsync(houts[v].depth, dout[v].depth, px * 4, cudaMemcpyDeviceToHost, cs));
        if (houts[v].final_T)
            CU(cudaMemcpyAsync(houts[v].final_T, dout[v].final_T, px * 4, cudaMemcpyDeviceToHost, cs));
        if (houts[v].visible && N > 0)
            CU(cudaMemcpyAsync(houts[v].visible, dout[v].visible, (size_t)N, cudaMemcpyDeviceToHost, cs));
        return S3R_OK;
    };
    // Chunked pipeline: the views are rendered HOST_CHUNK at a time on `st`
    // while the finished chunks' outputs stream back to the host on a second
    // stream, so the device->host copies (the bound of this entry point) overlap
    // the rendering.  Debug / counters / timing / training keep the one-batch
    // semantics of s3r_render_batch (their state describes one whole batch).
    constexpr int HOST_CHUNK = 8;
    const bool chunked = nv > HOST_CHUNK && !(c->debug || c->counters || c->timing || c->training);
    if (!chunked) {
        rc = render_impl(c, &ds, dv.data(), nv, dout.data(), st);
        if (rc != S3R_OK && rc != S3R_EINSTANCE) return rc;
        for (int v = 0; v < nv; ++v)
            if (int r2 = d2h(v, st)) return r2;
    } else {
        if (!c->copy_stream) CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        const int nchunks = (nv + HOST_CHUNK - 1) / HOST_CHUNK;
        while ((int)c->chunk_done.size() < nchunks) {
            cudaEvent_t e;
            CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->chunk_done.push_back(e);
        }
        std::vector<s3r_stats> all(nv);
        int worst = S3R_OK;
        for (int k = 0; k < nchunks; ++k) {
            const int v0 = k * HOST_CHUNK, n = std::min(HOST_CHUNK, nv - v0);
            rc = render_impl(c, &ds, dv.data() + v0, n, dout.data() + v0, st);
            if (rc != S3R_OK && rc != S3R_EINSTANCE) {
                cudaStreamSynchronize(c->copy_stream);
                return rc;
            }
            if (rc) worst = rc;
            std::copy(c->stats.begin(), c->stats.begin() + n, all.begin() + v0);
            CU(cudaEventRecord(c->chunk_done[k], st));
            CU(cudaStreamWaitEvent(c->copy_stream, c->chunk_done[k], 0));
            for (int v = v0; v < v0 + n; ++v)
                if (int r2 = d2h(v, c->copy_stream)) return r2;
        }
        rc = worst;
        c->stats = all;
        c->host_chunked = true;
        CU(cudaStreamSynchronize(c->copy_stream));
    }
    if (hs->life && N > 0)
        CU(cudaMemcpyAsync(hs->life, ds.life, (size_t)N * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    return rc;
}

int s3r_get_stats(const s3r_ctx* c, int32_t view_index, s3r_stats* out)
{
    if (!c || !out) return S3R_EINVAL;
    if (!c->have_render || view_index < 0 || view_index >= (int)c->stats.size())
        return S3R_ESTATE;
    s3r_ctx* m = const_cast<s3r_ctx*>(c);
    if (m->cap_pending) {
        // capacity mode: the planner wrote the counts into mapped staging memory
        cudaSetDevice(m->device);
        if (cudaDeviceSynchronize() != cudaSuccess)
            return fail(m, S3R_ECUDA, "get_stats: %s", cudaGetErrorString(cudaGetLastError()));
        for (size_t v = 0; v < m->stats.size(); ++v) {
            const ViewCounters& k = m->cap_h_ctr[v];
            s3r_stats& s = m->stats[v];
            s.n_scene = m->N_last;
            s.n_temporal = m->cap_h_ntemp[v];
            s.n_visible = (long long)k.n_visible;
            s.n_lod_small = (long long)k.n_small;
            s.n_lod_dropped = (long long)k.n_dropped;
            s.n_rendered = (long long)k.n_rendered;
            s.n_pairs = (long long)k.n_pairs;
            s.n_bin_pairs = (long long)k.n_spairs;
            s.n_bad_instance = (long long)k.n_bad;
        }
        m->cap_pending = false;
    }
    if (m->last_counters && !m->evals_fetched) {
        // E_alg / E_exec are produced by the rasterizer: fetch them once
        const size_t nv = m->stats.size();
        std::vector<unsigned long long> ev(2 * nv);
        cudaSetDevice(m->device);
        if (cudaMemcpy(ev.data(), m->d_evals.p, nv * 16, cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(m, S3R_ECUDA, "get_stats: fetching counters failed");
        for (size_t v = 0; v < nv; ++v) {
            m->stats[v].n_blend_evals = (int64_t)ev[2 * v];
            m->stats[v].n_blend_exec = (int64_t)ev[2 * v + 1];
        }
        m->evals_fetched = true;
    }
    *out = c->stats[view_index];
    return S3R_OK;
}

int s3r_dump_intermediates(s3r_ctx* c, int32_t vi, const s3r_debug* dbg, void* stream)
{
    if (!c || !dbg) return S3R_EINVAL;
    if (!c->have_render || vi < 0 || vi >= (int)c->hv.size())
        return fail(c, S3R_ESTATE, "dump: no render or view index out of range");
    if (c->host_chunked)
        return fail(c, S3R_ESTATE, "dump: the last render was a chunked s3r_render_batch_host "
                                   "batch (enable debug mode to dump it)");
    if (c->last_capm)
        return fail(c, S3R_ESTATE, "dump: the last render was planned on the device (capacity "
                                   "mode); enable debug mode to dump it");
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(c->device));
    const DevView& d = c->hv[vi];
    const long long Ns = std::max<long long>(c->N_last, 1);
    if (dbg->temporal_idx && d.n_temporal)
        CU(cudaMemcpyAsync(dbg->temporal_idx, P<int32_t>(c->d_tidx) + (long long)d.tslot * Ns,
                           d.n_temporal * 4, cudaMemcpyDeviceToDevice, st));
    const bool need_dbg = dbg->keys || dbg->flags || dbg->rect || dbg->depth_order || dbg->pair_gauss;
    if (need_dbg && !c->last_debug)
        return fail(c, S3R_ESTATE, "dump: keys/flags/rect/depth_order/pair_gauss need s3r_set_debug(1) before the render");
    if (dbg->keys && d.n_temporal)
        CU(cudaMemcpyAsync(dbg->keys, P<float>(c->d_dbg_keys) + 6 * d.dbg_off, d.n_temporal * 24,
                           cudaMemcpyDeviceToDevice, st));
    if (dbg->flags && d.n_temporal)
        CU(cudaMemcpyAsync(dbg->flags, P<uint8_t>(c->d_dbg_flags) + d.dbg_off, d.n_temporal,
                           cudaMemcpyDeviceToDevice, st));
    if (dbg->rect && d.n_temporal)
        CU(cudaMemcpyAsync(dbg->rect, P<int16_t>(c->d_dbg_rect) + 4 * d.dbg_off, d.n_temporal * 8,
                           cudaMemcpyDeviceToDevice, st));
    if (dbg->splat_rgb && d.n_rendered)   // .xyz of the third float4 of each sorted record
        CU(cudaMemcpy2DAsync(dbg->splat_rgb, 12, P<char>(c->d_recs) + 48 * d.cap_off + 32, 48, 12,
                             (size_t)d.n_rendered, cudaMemcpyDeviceToDevice, st));
    const uint32_t* order = P<uint32_t>(c->d_sortv[c->final_order]);
    if (dbg->depth_order)
        launch_dump_order(order, P<int32_t>(c->d_gidx), d.cap_off, d.n_rendered, dbg->depth_order, st);
    if (dbg->pair_tile || dbg->pair_gauss || dbg->ranges) {
        // pack the view's per-tile lists in tile order (exclusive scan of their
        // lengths on the host; debug path) as (tile, Gaussian) pairs + ranges
        int rc;
        const int nt = d.ntiles;
        if ((rc = ensure(c, c->d_dbg_tcnt, (size_t)(nt + 1) * 4))) return rc;
        uint32_t* toff = P<uint32_t>(c->d_dbg_tcnt);
        std::vector<int2> tr(nt);
        CU(cudaMemcpyAsync(tr.data(), P<int2>(c->d_tranges) + d.trange_off, (size_t)nt * sizeof(int2),
                           cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        std::vector<uint32_t> h(nt);
        uint32_t run = 0;
        for (int t = 0; t < nt; ++t) {
            h[t] = run;
            run += (uint32_t)(tr[t].y - tr[t].x);
        }
        if ((long long)run != d.n_pairs)
            return fail(c, S3R_ECUDA, "dump: tile lists hold %u pairs, expected %lld", run, d.n_pairs);
        CU(cudaMemcpyAsync(toff, h.data(), (size_t)nt * 4, cudaMemcpyHostToDevice, st));
        launch_dbg_tile_pairs(c->p_views, vi, nt, P<uint32_t>(c->d_tlists),
                              P<int2>(c->d_tranges), toff, order,
                              c->last_debug ? P<int32_t>(c->d_gidx) : nullptr, dbg->pair_tile,
                              dbg->pair_gauss, dbg->ranges, st);
        CU(cudaStreamSynchronize(st));
    }
    CU(cudaGetLastError());
    return S3R_OK;
}

int s3r_commit_visibility(s3r_ctx* c, const s3r_scene* s, float margin, void* stream)
{
    if (!c || !s) return S3R_EINVAL;
    if (s->n < 0 || (s->n > 0 && (!s->visibility || !s->life)) || !std::isfinite(margin))
        return fail(c, S3R_EINVAL, "commit: bad arguments (visibility and life required)");
    CU(cudaSetDevice(c->device));
    launch_commit(reinterpret_cast<float2*>(s->visibility), reinterpret_cast<float2*>(s->life),
                  s->n, margin, (cudaStream_t)stream);
    CU(cudaGetLastError());
    return S3R_OK;
}

int s3r_reset_visibility(s3r_ctx* c, const s3r_scene* s, void* stream)
{
    if (!c || !s) return S3R_EINVAL;
    if (s->n < 0 || (s->n > 0 && !s->visibility))
        return fail(c, S3R_EINVAL, "reset: bad arguments");
    CU(cudaSetDevice(c->device));
    launch_reset(reinterpret_cast<float2*>(s->visibility), s->n, (cudaStream_t)stream);
    CU(cudaGetLastError());
    return S3R_OK;
}

int s3r_set_training(s3r_ctx* c, int enable)
{
    if (!c) return S3R_EINVAL;
    c->training = enable != 0;
    return S3R_OK;
}

int s3r_set_lod_jitter(s3r_ctx* c, float dx, float dy, float dz)
{
    if (!c) return S3R_EINVAL;
    if (!(std::isfinite(dx) && std::isfinite(dy) && std::isfinite(dz)))
        return fail(c, S3R_EINVAL, "set_lod_jitter: non-finite offset scale");
    c->lod_jitter[0] = dx;
    c->lod_jitter[1] = dy;
    c->lod_jitter[2] = dz;
    return S3R_OK;
}

int s3r_set_neural_colors(s3r_ctx* c, const s3r_neurf* p, void* stream)
{
    if (!c) return S3R_EINVAL;
    if (!p) {
        c->neurf = false;
        return S3R_OK;
    }
    if (!p->w1 || !p->b1 || !p->w2 || !p->b2 || !p->w3 || !p->b3 || !p->time_emb ||
        !p->class_emb || p->n_time < 1 || p->num_instances < 1 || !(p->pos_scale > 0.0f) ||
        !std::isfinite(p->pos_scale))
        return fail(c, S3R_EINVAL, "set_neural_colors: bad parameters");
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(c->device));
    int rc;
    if ((rc = ensure(c, c->d_nw, neurf_pack_bytes()))) return rc;
    if ((rc = ensure(c, c->d_nb, (size_t)neurf_bias_count() * 4))) return rc;
    if ((rc = ensure(c, c->d_temb, (size_t)p->n_time * 8 * 4))) return rc;
    if ((rc = ensure(c, c->d_cemb, (size_t)p->num_instances * 4 * 4))) return rc;
    launch_neurf_pack(p->w1, p->b1, p->w2, p->b2, p->w3, p->b3, c->d_nw.p, P<float>(c->d_nb), st);
    CU(cudaMemcpyAsync(c->d_temb.p, p->time_emb, (size_t)p->n_time * 32, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(c->d_cemb.p, p->class_emb, (size_t)p->num_instances * 16,
                       cudaMemcpyDeviceToDevice, st));
    CU(cudaGetLastError());
    c->neurf = true;
    c->neurf_ntime = p->n_time;
    c->neurf_ninst = p->num_instances;
    c->neurf_scale = p->pos_scale;
    return S3R_OK;
}

int s3r_set_overlap(s3r_ctx* c, int enable)
{
    if (!c) return S3R_EINVAL;
    c->overlap = enable != 0;
    return S3R_OK;
}

int s3r_set_fast_exp(s3r_ctx* c, int enable)
{
    if (!c) return S3R_EINVAL;
    c->fast_exp = enable != 0;
    return S3R_OK;
}

int s3r_set_pipeline(s3r_ctx* c, int pipeline)
{
    if (!c) return S3R_EINVAL;
    if (pipeline != S3R_PIPELINE_STREAMLINED && pipeline != S3R_PIPELINE_CONVENTIONAL)
        return fail(c, S3R_EINVAL, "set_pipeline: unknown pipeline %d", pipeline);
    c->pipeline = pipeline;
    return S3R_OK;
}

int s3r_render_backward(s3r_ctx* c, const s3r_scene* sc, const s3r_view* views, int32_t nv,
                        const s3r_cotangents* cots, const s3r_grads* grads, void* stream)
{
    if (!c || !sc || !grads) return S3R_EINVAL;
    if (!c->have_render || !c->last_training)
        return fail(c, S3R_ESTATE, "backward: no training forward (s3r_set_training(1) + render)");
    if (c->last_pipeline != S3R_PIPELINE_STREAMLINED)
        return fail(c, S3R_ESTATE, "backward: the last render used the conventional pipeline");
    if (c->last_neurf)
        return fail(c, S3R_ESTATE, "backward: the last render used NeurF colours");
    if (nv != c->last_nviews || sc->n != c->last_N)
        return fail(c, S3R_ESTATE, "backward: scene/views differ from the last forward");
    if (nv > 0 && (!views || !cots)) return fail(c, S3R_EINVAL, "backward: views/cots NULL");
    if (sc->n > 0 && (!grads->means_opacity || !grads->scales || !grads->rotations ||
                      !grads->colors))
        return fail(c, S3R_EINVAL, "backward: gradient arrays required");
    for (int v = 0; v < nv; ++v) {
        if (!cots[v].rgb) return fail(c, S3R_EINVAL, "backward: cots[%d].rgb is NULL", v);
        if (views[v].width != c->hv[v].W || views[v].height != c->hv[v].H)
            return fail(c, S3R_ESTATE, "backward: view %d differs from the last forward", v);
    }
    cudaStream_t st = (cudaStream_t)stream;
    CU(cudaSetDevice(c->device));
    int rc;
    long long cap = 0;
    for (int v = 0; v < nv; ++v) cap = std::max(cap, c->hv[v].cap_off + c->hv[v].n_temporal);
    const size_t sg_bytes = (size_t)std::max(cap, 1ll) * 4 * splat_grad_stride();
    if ((rc = ensure(c, c->d_sgrads, sg_bytes))) return rc;
    CU(cudaMemsetAsync(c->d_sgrads.p, 0, sg_bytes, st));
    if ((rc = ensure(c, c->d_cots, (size_t)std::max(nv, 1) * sizeof(s3r_cot)))) return rc;
    if ((rc = stage_begin(c, (size_t)std::max(nv, 1) * sizeof(s3r_cot) + 512, st))) return rc;
    s3r_cot* h = (s3r_cot*)stage_alloc(c, (size_t)std::max(nv, 1) * sizeof(s3r_cot));
    for (int v = 0; v < nv; ++v) h[v] = s3r_cot{cots[v].rgb, cots[v].depth, cots[v].final_T};
    if (nv) CU(cudaMemcpyAsync(c->d_cots.p, h, nv * sizeof(s3r_cot), cudaMemcpyHostToDevice, st));
    BackwardArgs a{};
    a.views = c->p_views;
    a.n_views = nv;
    a.cots = P<s3r_cot>(c->d_cots);
    a.tranges = P<int2>(c->d_tranges);
    a.tlists = P<uint32_t>(c->d_tlists);
    a.rec_sorted = P<float4>(c->d_recs);
    a.train_T = P<float>(c->d_train_T);
    a.train_n = P<int>(c->d_train_n);
    a.splat_grads = P<float>(c->d_sgrads);
    a.dkey_sorted = P<unsigned long long>(c->d_sortk[c->final_order]);
    // noisy offset: the splats' moved means by compacted slot, and rank -> slot
    a.rec_mu = c->last_jitter && c->last_recmu ? P<float4>(c->d_recmu) : nullptr;
    a.order = P<uint32_t>(c->d_sortv[c->final_order]);
    a.gmask = (1ull << c->gbits) - 1ull;
    a.ids = sc->instance_ids;
    a.means_opacity = reinterpret_cast<const float4*>(sc->means_opacity);
    a.scales = reinterpret_cast<const float4*>(sc->scales);
    a.rotations = reinterpret_cast<const float4*>(sc->rotations);
    a.g_means = grads->means_opacity;
    a.g_scales = grads->scales;
    a.g_rot = grads->rotations;
    a.g_colors = grads->colors;
    a.g_table = grads->table;
    a.num_instances = sc->num_instances;
    a.smem_table = sc->num_instances <= 1024;
    for (int v = 0; v < nv; ++v) {
        if (cots[v].depth) a.has_depth_cot = 1;
        if (cots[v].final_T) a.has_T_cot = 1;
    }
    launch_backward(a, c->last_max_tiles, c->last_max_r, st);
    if ((rc = stage_end(c, st))) return rc;
    CU(cudaGetLastError());
    return S3R_OK;
}

int s3r_mse(s3r_ctx* c, const float* x, const float* y, int64_t n, float scale, float* grad,
            float* loss, void* stream)
{
    if (!c) return S3R_EINVAL;
    if (n < 0 || (n > 0 && (!x || !y || !grad || !loss)))
        return fail(c, S3R_EINVAL, "mse: bad arguments");
    CU(cudaSetDevice(c->device));
    launch_mse(x, y, n, scale, grad, loss, (cudaStream_t)stream);
    CU(cudaGetLastError());
    return S3R_OK;
}

int s3r_life_flip(s3r_ctx* c, float* life, int64_t n, void* stream)
{
    if (!c) return S3R_EINVAL;
    if (n < 0 || (n > 0 && (!life || !aligned(life, 8))))
        return fail(c, S3R_EINVAL, "life_flip: bad arguments");
    CU(cudaSetDevice(c->device));
    launch_life_flip(reinterpret_cast<float2*>(life), n, (cudaStream_t)stream);
    CU(cudaGetLastError());
    return S3R_OK;
}

int s3r_set_capacity(s3r_ctx* c, const s3r_capacity* cap)
{
    if (!c) return S3R_EINVAL;
    if (!cap) {
        c->cap_on = false;
        return S3R_OK;
    }
    if (cap->records < 1 || cap->rendered_view < 1 || cap->bin_pairs < 1 ||
        cap->tile_entries < 1 || cap->temporal_view < 1)
        return fail(c, S3R_EINVAL, "set_capacity: every capacity must be >= 1");
    if (cap->records >= (1ll << 32) || cap->rendered_view >= (1ll << 31) ||
        cap->bin_pairs >= (1ll << 32) || cap->tile_entries >= (1ll << 32))
        return fail(c, S3R_EINVAL, "set_capacity: capacities must fit 32-bit list positions");
    c->cap = *cap;
    c->cap_on = true;
    return S3R_OK;
}

int s3r_capacity_from_last(s3r_ctx* c, float margin, s3r_capacity* out)
{
    if (!c || !out || !(margin >= 1.0f) || !std::isfinite(margin)) return S3R_EINVAL;
    if (!c->have_render) return fail(c, S3R_ESTATE, "capacity_from_last: no render yet");
    if (c->last_capm) {
        // planned on the device: the needs are the counters of that batch
        s3r_stats tmp;
        if (int r = s3r_get_stats(c, 0, &tmp)) return r;
        s3r_capacity need{};
        for (size_t v = 0; v < c->stats.size(); ++v) {
            const s3r_stats& s = c->stats[v];
            const long long SS = 1ll << (2 * c->hv[v].sshift);
            need.records += s.n_temporal;
            need.bin_pairs += s.n_bin_pairs;
            need.tile_entries += SS * s.n_bin_pairs;
            need.rendered_view = std::max<long long>(need.rendered_view, s.n_rendered);
            need.temporal_view = std::max<long long>(need.temporal_view, s.n_temporal);
        }
        c->last_need = need;
        c->last_need_valid = true;
    }
    if (!c->last_need_valid) return fail(c, S3R_ESTATE, "capacity_from_last: no sized render");
    auto sc = [&](long long x) {
        return std::max<long long>(1, (long long)std::ceil((double)x * (double)margin));
    };
    out->records = sc(c->last_need.records);
    out->rendered_view = sc(c->last_need.rendered_view);
    out->bin_pairs = sc(c->last_need.bin_pairs);
    out->tile_entries = sc(c->last_need.tile_entries);
    out->temporal_view = sc(c->last_need.temporal_view);
    return S3R_OK;
}

int s3r_check(s3r_ctx* c, void* stream)
{
    if (!c) return S3R_EINVAL;
    CU(cudaSetDevice(c->device));
    CU(cudaStreamSynchronize((cudaStream_t)stream));
    uint32_t e = 0;
    CU(cudaMemcpy(&e, c->d_err.p, sizeof e, cudaMemcpyDeviceToHost));
    CU(cudaMemset(c->d_err.p, 0, sizeof e));
    if (c->twin && c->twin_stream) {
        uint32_t e2 = 0;
        CU(cudaStreamSynchronize(c->twin_stream));
        CU(cudaMemcpy(&e2, c->twin->d_err.p, sizeof e2, cudaMemcpyDeviceToHost));
        CU(cudaMemset(c->twin->d_err.p, 0, sizeof e2));
        e |= e2;
    }
    if (e & ERR_PRECULL)
        return fail(c, S3R_EINTERNAL, "K2 frustum pre-test culled a visible Gaussian");
    if (e & ERR_CAPACITY)
        return fail(c, S3R_ECAPACITY, "capacity mode: a view exceeded the reserved scratch and was "
                                      "rendered empty (s3r_capacity_from_last / s3r_set_capacity)");
    if (e & ERR_BADID) return fail(c, S3R_EINSTANCE, "a Gaussian had an out-of-range instance id");
    return S3R_OK;
}

}  // extern "C"
