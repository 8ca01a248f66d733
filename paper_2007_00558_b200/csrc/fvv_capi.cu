// C ABI of libfvvb200.so (include/fvv_b200.h): context, resident camera
// slots, keyed z canvases with generation tags, and the launch sequence
// preprocess -> forward warp -> resolve for each view.

#include <cmath>
#include <cstdarg>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "fvv_capture.cuh"
#include "fvv_codec.cuh"
#include "fvv_kernels.cuh"
#include "fvv_mvd.cuh"

using namespace fvv;

namespace {

struct Slot {
    bool has_cam = false, has_bg = false, has_frame = false;
    fvv_camera cam{};
    DevCam dev{};
    size_t cap = 0;  // pixels allocated
    double *rays = nullptr;  // rx[W] then ry[H]
    uint32_t *texel = nullptr;
    float *fgd = nullptr;
    float *bgd = nullptr;
    void release() {
        cudaFree(rays);
        cudaFree(texel);
        cudaFree(fgd);
        cudaFree(bgd);
        rays = nullptr; texel = nullptr; fgd = nullptr; bgd = nullptr;
        cap = 0;
        has_cam = has_bg = has_frame = false;
    }
};

}  // namespace

struct fvv_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    int64_t launches = 0;
    Slot slots[FVV_MAX_SLOTS];
    Slot tmp[FVV_MAX_REFS + 1];  // one-shot calls (synthesize_view / warp_layer)
    // keyed z canvases: n contributions of (H+2r)(W+2r) keys
    uint64_t *canvas = nullptr;
    size_t canvas_cap = 0;  // keys allocated
    int cW = -1, cH = -1, cr = -1, cn = 0;
    int gen = -1;  // generation of the last view; -1 = canvases need a fill
    // device-resident generation (fvv_ctx_device_generation): every view
    // runs k_gen_fill, which advances dgen[0] on the device, so a captured
    // CUDA graph of views stays correct when replayed
    bool dev_gen = false;
    int *dgen = nullptr;  // [generation, CTA counter]
    // per contribution: K2's exact z of every source pixel (zcap doubles each)
    double *zsrc = nullptr;
    size_t zcap = 0, zn = 0;
    // inpainting scratch (provenance + composite depth) when the caller
    // passes no provenance buffer
    uint8_t *iprov = nullptr;
    float *idepth = nullptr;
    int16_t *idist = nullptr;   // 4 x [px] K4 distance planes
    size_t icap = 0;
    // K3's TMA map of the canvases and what it was built for
    CUtensorMap kmap;
    const void *kmap_base = nullptr;
    long long kmap_pitch = 0, kmap_rows = 0, kmap_n = 0, kmap_per = 0;
    // K2 -> K3 FG tile occupancy (TileFlags), 0xFF-initialised
    uint8_t *tflag = nullptr;
    size_t tflag_cap = 0;
    // K1 candidate list (camera << 26 | pixel) + its length
    uint32_t *cand = nullptr;
    int *ncand = nullptr;
    size_t cand_cap = 0;
    // MED + Rice plane codec scratch
    RiceScratch rice;
    // MVD container validity run-length encoder scratch
    RleScratch rle;
    // K1 range-weight table for range_sigma (kRangeTableLen doubles)
    double *range_w = nullptr;
    double range_sigma = -1.0;
    // per-kernel event timing (fvv_profile_enable)
    bool prof = false;
    struct Rec { int kid; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    double prof_ms[5] = {0, 0, 0, 0, 0};
    int64_t prof_n[5] = {0, 0, 0, 0, 0};
    unsigned long long *prof_atomics = nullptr;  // [256] K2 z-buffer atomics while counting
    bool count_atomics = false;
    // dequantize12 of every 12-bit code for the depth range (dq_span, dq_zf)
    float *dq = nullptr;
    double dq_span = 0.0, dq_zf = 0.0;
};

namespace {

int fail(fvv_ctx *ctx, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    return code;
}

#define CK(expr)                                                                       \
    do {                                                                               \
        cudaError_t e__ = (expr);                                                      \
        if (e__ != cudaSuccess)                                                        \
            return fail(ctx, FVV_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e__)); \
    } while (0)

cudaEvent_t prof_event(fvv_ctx *ctx) {
    if (!ctx->pool.empty()) {
        cudaEvent_t e = ctx->pool.back();
        ctx->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

#define LAUNCH_K(kid, expr)                                              \
    do {                                                                 \
        cudaEvent_t a__ = nullptr, b__ = nullptr;                        \
        if (ctx->prof) {                                                 \
            a__ = prof_event(ctx);                                       \
            b__ = prof_event(ctx);                                       \
            CK(cudaEventRecord(a__, ctx->stream));                       \
        }                                                                \
        CK(expr);                                                        \
        if (ctx->prof) {                                                 \
            CK(cudaEventRecord(b__, ctx->stream));                       \
            ctx->recs.push_back({kid, a__, b__});                        \
        }                                                                \
        ctx->launches += 1 + take_extra_launches();                      \
    } while (0)
#define LAUNCH(expr) LAUNCH_K(FVV_K_OTHER, expr)

int enter(fvv_ctx *ctx) {
    if (!ctx) return FVV_EINVAL;
    ctx->err.clear();
    CK(cudaSetDevice(ctx->device));
    return FVV_OK;
}

int check_cam(fvv_ctx *ctx, const fvv_camera *c, const char *what) {
    if (!c) return fail(ctx, FVV_EINVAL, "%s camera is NULL", what);
    if (c->width <= 0 || c->height <= 0 || c->width % 2 || c->height % 2)
        return fail(ctx, FVV_EINVAL, "%s camera: width and height must be positive and even", what);
    if (!(c->fx > 0 && c->fy > 0))
        return fail(ctx, FVV_EINVAL, "%s camera: focal lengths must be positive", what);
    if ((long long)c->width * c->height > (1ll << 26))
        return fail(ctx, FVV_EINVAL, "%s camera: more than 2^26 pixels", what);
    return FVV_OK;
}

int check_cfg(fvv_ctx *ctx, const fvv_synth_cfg *cfg) {
    if (!cfg) return fail(ctx, FVV_EINVAL, "config is NULL");
    if (cfg->splat_radius < 0 || cfg->crack_fill_window < 1)
        return fail(ctx, FVV_EINVAL, "bad splat/crack parameters");
    if (cfg->splat_radius > 3 || cfg->crack_fill_window > 5)
        return fail(ctx, FVV_EINVAL, "splat_radius > 3 or crack_fill_window > 5 not supported");
    if (cfg->angular_weight && !(cfg->angular_epsilon > 0 && std::isfinite(cfg->angular_epsilon)))
        return fail(ctx, FVV_EINVAL, "angular_epsilon must be positive and finite");
    if (cfg->inpaint && (cfg->inpaint_radius < 1 || cfg->inpaint_radius > 4096))
        return fail(ctx, FVV_EINVAL, "inpaint_radius must be in [1, 4096]");
    return FVV_OK;
}

int slot_alloc(fvv_ctx *ctx, Slot &s, const fvv_camera &cam) {
    const size_t n = (size_t)cam.width * cam.height;
    if (n > s.cap) {
        s.release();
        CK(cudaMalloc(&s.texel, n * sizeof(uint32_t)));
        CK(cudaMalloc(&s.fgd, n * sizeof(float)));
        CK(cudaMalloc(&s.bgd, n * sizeof(float)));
        s.cap = n;
    }
    CK(cudaFree(s.rays));
    s.rays = nullptr;
    CK(cudaMalloc(&s.rays, (size_t)(cam.width + cam.height) * sizeof(double)));
    s.cam = cam;
    s.dev = to_dev(cam);
    LAUNCH(launch_rays(s.dev, s.rays, s.rays + cam.width, ctx->stream));
    s.has_cam = true;
    s.has_bg = s.has_frame = false;
    return FVV_OK;
}

int slot_camera(fvv_ctx *ctx, Slot &s, const fvv_camera &cam) {
    if (s.has_cam && memcmp(&s.cam, &cam, sizeof(cam)) == 0) return FVV_OK;
    if (s.has_cam && s.cam.width == cam.width && s.cam.height == cam.height) {
        // same size: only the calibration changed; keep buffers, refresh
        // rays. The slot's BG model and live frame belonged to the old
        // calibration: a render now needs new ones ("missing inputs").
        s.cam = cam;
        s.dev = to_dev(cam);
        LAUNCH(launch_rays(s.dev, s.rays, s.rays + cam.width, ctx->stream));
        s.has_bg = s.has_frame = false;
        return FVV_OK;
    }
    return slot_alloc(ctx, s, cam);
}

PreprocParams base_pre(const Slot &s) {
    PreprocParams p{};
    p.W = s.cam.width;
    p.H = s.cam.height;
    return p;
}

// Install the range-weight table exp(-d2 * inv_2sr), d2 = 0 .. 3*255^2, for
// sigma_r. `host` (kRangeTableLen doubles) comes from the caller; NULL builds
// it with libm exp. A table already resident for sigma_r is kept, so the
// Python host's np.exp table (installed first) is never replaced by libm's.
int range_table(fvv_ctx *ctx, double sigma_r, const double *host) {
    if (!host && ctx->range_w && ctx->range_sigma == sigma_r) return FVV_OK;
    if (!ctx->range_w) CK(cudaMalloc(&ctx->range_w, kRangeTableLen * sizeof(double)));
    std::vector<double> t;
    if (!host) {
        // depthproc.py:200,212: inv_2sr = 1/(2 sr^2); w = exp(-d2 * inv_2sr)
        const double inv_2sr = 1.0 / (2.0 * (sigma_r * sigma_r));
        t.resize(kRangeTableLen);
        for (int d = 0; d < kRangeTableLen; ++d) t[d] = std::exp(-(double)d * inv_2sr);
        host = t.data();
    }
    // synchronous: the table is rebuilt only when sigma_range changes
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(ctx->range_w, host, kRangeTableLen * sizeof(double), cudaMemcpyHostToDevice));
    ctx->range_sigma = sigma_r;
    return FVV_OK;
}

int bilateral_params(fvv_ctx *ctx, BilateralParams &p, int radius, double sigma_s, double sigma_r,
                     int min_valid) {
    // depthproc.py:199-200, 211-212: spatial factor via libm exp on the host
    // (Python's math.exp is the same libm call); range factor from the table
    p.radius = radius;
    p.min_valid = min_valid;
    const double inv_2ss = 1.0 / (2.0 * (sigma_s * sigma_s));
    for (int dy = -radius; dy <= radius; ++dy)
        for (int dx = -radius; dx <= radius; ++dx)
            p.sw[dy + radius][dx + radius] = std::exp((double)(-(dy * dy + dx * dx)) * inv_2ss);
    if (radius > 0) {
        int rc = range_table(ctx, sigma_r, nullptr);
        if (rc) return rc;
    }
    p.range_w = ctx->range_w;
    return FVV_OK;
}

// reference defaults, depthproc.py:174-177
int bilateral_defaults(fvv_ctx *ctx, BilateralParams &p) {
    return bilateral_params(ctx, p, 2, 2.0, 10.0, 6);
}

// K0/K1 read a 12-bit code's depth from the context's table for the code's
// depth range (built by k_dq_table with the exact formula, once per range)
int dq_table(fvv_ctx *ctx, PreprocCore &c) {
    if (!ctx->dq) CK(cudaMalloc(&ctx->dq, 4096 * sizeof(float)));
    if (ctx->dq_span != c.inv_span || ctx->dq_zf != c.inv_zf) {
        LAUNCH(launch_dq_table(ctx->dq, c.inv_span, c.inv_zf, ctx->stream));
        // once per range: later calls may come on another stream
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->dq_span = c.inv_span;
        ctx->dq_zf = c.inv_zf;
    }
    c.dq = ctx->dq;
    return FVV_OK;
}

// room for `px` K1 candidates (a batch's pixel count bounds it)
int fill_list(fvv_ctx *ctx, size_t px, uint32_t *&cand, int *&ncand) {
    if (!ctx->ncand) CK(cudaMalloc(&ctx->ncand, sizeof(int)));
    if (px > ctx->cand_cap) {
        CK(cudaFree(ctx->cand));
        ctx->cand = nullptr;
        CK(cudaMalloc(&ctx->cand, px * sizeof(uint32_t)));
        ctx->cand_cap = px;
    }
    cand = ctx->cand;
    ncand = ctx->ncand;
    return FVV_OK;
}

int with_fill(fvv_ctx *ctx, PreprocParams &p) {
    if (p.radius <= 0) return FVV_OK;
    return fill_list(ctx, (size_t)p.W * p.H, p.cand, p.ncand);
}

int canvas_pitch(int W, int r) { return (W + 2 * r + 2) & ~1; }  // even, >= W+2r+1

size_t canvas_per(int W, int H, int r) { return (size_t)canvas_pitch(W, r) * (H + 2 * r); }

int ensure_canvas(fvv_ctx *ctx, int n, int W, int H, int r) {
    const size_t per = canvas_per(W, H, r);
    const size_t need = per * (size_t)n + 2;  // +1 leading offset, +1 slack
    if (need > ctx->canvas_cap) {
        CK(cudaFree(ctx->canvas));
        ctx->canvas = nullptr;
        CK(cudaMalloc(&ctx->canvas, need * sizeof(uint64_t)));
        ctx->canvas_cap = need;
        ctx->gen = -1;
    }
    if (ctx->cW != W || ctx->cH != H || ctx->cr != r || ctx->cn < n) {
        ctx->cW = W; ctx->cH = H; ctx->cr = r; ctx->cn = n;
        ctx->gen = -1;
    }
    if (ctx->dev_gen) {
        if (ctx->gen < 0) {   // new canvases: the device generation restarts
            CK(cudaMemsetAsync(ctx->dgen, 0xFF, sizeof(int), ctx->stream));
            ctx->gen = 0;
        }
        LAUNCH_K(FVV_K_FILL, launch_gen_fill(ctx->canvas, per * (size_t)ctx->cn + 2, ctx->dgen,
                                             ctx->stream));
        return FVV_OK;
    }
    // generation tags: keys of this view carry gen; anything else is empty.
    // One fill per 127 views instead of a clear per view.
    if (ctx->gen <= 0) {
        LAUNCH_K(FVV_K_FILL, launch_fill_u64(ctx->canvas, per * (size_t)ctx->cn + 2, kEmpty,
                                             ctx->stream));
        ctx->gen = 126;
    } else {
        ctx->gen -= 1;
    }
    return FVV_OK;
}

// n per-contribution z planes of `px` source pixels each (never cleared: K3
// reads only the entries of this view's winners, which K2 just wrote)
int ensure_zsrc(fvv_ctx *ctx, int n, size_t px) {
    if (px > ctx->zcap || (size_t)n > ctx->zn) {
        const size_t cap = px > ctx->zcap ? px : ctx->zcap;
        const size_t nn = (size_t)n > ctx->zn ? (size_t)n : ctx->zn;
        CK(cudaFree(ctx->zsrc));
        ctx->zsrc = nullptr;
        CK(cudaMalloc(&ctx->zsrc, cap * nn * sizeof(double)));
        ctx->zcap = cap;
        ctx->zn = nn;
    }
    return FVV_OK;
}

// codec scratch for n pixels (ns in the skewed rebuild layout, ne strip-edge
// slots) and c chunks
int rice_scratch(fvv_ctx *ctx, size_t n, size_t c, size_t ns = 0, size_t ne = 0) {
    RiceScratch &r = ctx->rice;
    if (!r.costs) {
        CK(cudaMalloc(&r.costs, 2 * kRiceMaxPlanes * sizeof(unsigned long long)));
        CK(cudaMalloc(&r.total, kRiceMaxPlanes * sizeof(unsigned long long)));
        CK(cudaMalloc(&r.changed, sizeof(int)));
        CK(cudaMalloc(&r.wave, 2 * sizeof(int)));
    }
    if (ne > r.e_cap) {
        CK(cudaFree(r.edge));
        r.edge = nullptr;
        CK(cudaMalloc(&r.edge, ne * sizeof(unsigned long long)));
        // no slot carries a tag (the rebuild runs on the same stream)
        CK(cudaMemsetAsync(r.edge, 0, ne * sizeof(unsigned long long), ctx->stream));
        r.e_cap = ne;
    }
    const size_t blocks = (n + 1023) / 1024 + 1;
    const size_t bneed = blocks > c + 1 ? blocks : c + 1;
    const size_t nn = n > ns ? n : ns;
    if (nn > r.n_cap) {
        CK(cudaFree(r.zz));
        CK(cudaFree(r.res));
        CK(cudaFree(r.skew));
        r.zz = nullptr;
        r.res = nullptr;
        r.skew = nullptr;
        CK(cudaMalloc(&r.zz, nn * sizeof(uint16_t)));
        CK(cudaMalloc(&r.res, nn * sizeof(int32_t)));
        CK(cudaMalloc(&r.skew, nn));
        r.n_cap = nn;
    }
    const size_t cneed = bneed;
    if (cneed > r.c_cap) {
        for (void **q : {(void **)&r.block, (void **)&r.entry, (void **)&r.exit,
                         (void **)&r.exit_prev, (void **)&r.count}) {
            CK(cudaFree(*q));
            *q = nullptr;
        }
        CK(cudaMalloc(&r.block, cneed * sizeof(unsigned long long)));
        CK(cudaMalloc(&r.entry, cneed * sizeof(long long)));
        CK(cudaMalloc(&r.exit, cneed * sizeof(long long)));
        CK(cudaMalloc(&r.exit_prev, cneed * sizeof(long long)));
        CK(cudaMalloc(&r.count, cneed * sizeof(unsigned long long)));
        r.c_cap = cneed;
    }
    return FVV_OK;
}

// cuTensorMapEncodeTiled from the driver, through the runtime (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    // function-local static: initialised once, thread-safely
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        cudaGetLastError();
        return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    }();
    return fn;
}

// K3's 3-D TMA map {pitch, rows, n} over the canvas allocation (cached)
int canvas_tensor_map(fvv_ctx *ctx, int n, int W, int H, int r, ResolveParams &rp) {
    const long long pitch = canvas_pitch(W, r), rows = H + 2 * r;
    const long long per = (long long)canvas_per(W, H, r);
    if (!(ctx->kmap_base == ctx->canvas && ctx->kmap_pitch == pitch && ctx->kmap_rows == rows &&
          ctx->kmap_n == n && ctx->kmap_per == per)) {
        auto enc = tensor_map_encoder();
        if (!enc) return fail(ctx, FVV_ECUDA, "cuTensorMapEncodeTiled unavailable");
        const cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)rows, (cuuint64_t)n};
        const cuuint64_t strides[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)per * 8};
        // K3's key tile: the 32 x FTY tile plus a 2-cell ring
        const cuuint32_t box[3] = {32 + 4, (cuuint32_t)resolve_tile_rows() + 4, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        const CUresult e = enc(&ctx->kmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, ctx->canvas, dims,
                               strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (e != CUDA_SUCCESS) return fail(ctx, FVV_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)e);
        ctx->kmap_base = ctx->canvas;
        ctx->kmap_pitch = pitch;
        ctx->kmap_rows = rows;
        ctx->kmap_n = n;
        ctx->kmap_per = per;
    }
    rp.kmap = ctx->kmap;
    rp.has_kmap = 1;
    return FVV_OK;
}

double host_weight(const fvv_camera &a, const fvv_camera &b, double eps) {
    const double dx = a.C[0] - b.C[0], dy = a.C[1] - b.C[1], dz = a.C[2] - b.C[2];
    return 1.0 / (std::sqrt((dx * dx + dy * dy) + dz * dz) + eps);
}

// FG tile occupancy for n FG contributions of a W x H view on K3's fast
// path (r == 1, 3 x 3 crack window): stale entries only cost K3 work
// (flags are compared with the view's generation), so the buffer is filled
// with 0xFF once per growth and never cleared.
int tile_flags(fvv_ctx *ctx, int n, int W, int H, WarpParams &wp, ResolveParams &rp) {
    TileFlags tf{};
    tf.n_fg = n;
    tf.ntx = (W + kTileFlagW - 1) / kTileFlagW;
    tf.nty = (H + kTileFlagH - 1) / kTileFlagH;
    const size_t need = (size_t)n * tf.ntx * tf.nty * kTileFlagStride;
    if (need > ctx->tflag_cap) {
        CK(cudaFree(ctx->tflag));
        ctx->tflag = nullptr;
        CK(cudaMalloc(&ctx->tflag, need));
        CK(cudaMemsetAsync(ctx->tflag, 0xFF, need, ctx->stream));
        ctx->tflag_cap = need;
    }
    tf.flag = ctx->tflag;
    wp.tf = tf;
    rp.tf = tf;
    return FVV_OK;
}

// One view from n reference slots: K2 over 2n contributions, then K3.
int render_view(fvv_ctx *ctx, const fvv_camera &virt, Slot *const *refs, const double *weights,
                int n, const fvv_synth_cfg &cfg, uint8_t *rgb_out, uint8_t *prov_out,
                const fvv_debug *dbg) {
    const int r = cfg.splat_radius;
    int rc = ensure_canvas(ctx, 2 * n, virt.width, virt.height, r);
    if (rc) return rc;
    const size_t per = canvas_per(virt.width, virt.height, r);
    const DevCam dst = to_dev(virt);
    uint64_t *cbase = ctx->canvas + 1;

    WarpParams wp{};
    wp.dst = dst;
    wp.r = r;
    wp.pitch = canvas_pitch(virt.width, r);
    wp.n = 2 * n;
    wp.gen_hi = (uint64_t)ctx->gen << kGenShift;
    wp.gen_ptr = ctx->dev_gen ? ctx->dgen : nullptr;
    wp.n_atomics = ctx->count_atomics ? ctx->prof_atomics : nullptr;
    ResolveParams rp{};
    rp.dst = dst;
    rp.gen_ptr = wp.gen_ptr;
    rp.r = r;
    rp.window = cfg.crack_fill_window;
    rp.need = cfg.crack_fill_window * cfg.crack_fill_window / 2 + 1;
    rp.pitch = wp.pitch;
    rp.gen = (uint64_t)ctx->gen;
    rp.n_fg = n;
    rp.n_bg = n;
    rp.band_rel = cfg.depth_band_rel;
    for (int q = 0; q < 3; ++q) {
        rp.hole[q] = (double)cfg.hole_color[q];
        rp.hole_rgb |= (uint32_t)cfg.hole_color[q] << (8 * q);
    }
    rp.rgb_out = rgb_out;
    rp.prov_out = prov_out;
    if (dbg) rp.dbg = *dbg;
    long long maxpx = 0;
    for (int j = 0; j < n; ++j) {
        const long long np = (long long)refs[j]->cam.width * refs[j]->cam.height;
        maxpx = np > maxpx ? np : maxpx;
    }
    if ((rc = ensure_zsrc(ctx, 2 * n, (size_t)maxpx))) return rc;
    for (int j = 0; j < n; ++j) {
        const Slot &s = *refs[j];
        const double w = (weights && weights[j] > 0) ? weights[j]
                                                     : host_weight(s.cam, virt, cfg.mixing_epsilon);
        const int b = index_bits((long long)s.cam.width * s.cam.height);
        const double *rx = s.rays, *ry = s.rays + s.cam.width;
        for (int L = 0; L < 2; ++L) {
            const int k = L * n + j;
            const float *d = L == 0 ? s.fgd : s.bgd;
            double *zs = ctx->zsrc + ctx->zcap * k;
            wp.c[k] = WarpContrib{s.dev, relative_pose(s.dev, dst), d, rx, ry, cbase + per * k,
                                  zs, b};
            rp.c[k] = ResolveContrib{s.dev, relative_pose(dst, s.dev), s.texel, zs,
                                     cbase + per * k, w, b,
                                     L == 0 ? kFlagLiveValid : kFlagLiveBackground, L == 0};
        }
    }
    rp.ang = cfg.angular_weight ? 1 : 0;
    rp.ang_eps = cfg.angular_epsilon;
    InpaintParams ip{};
    if (cfg.inpaint && rgb_out) {
        const size_t px = (size_t)virt.width * virt.height;
        if (px > ctx->icap) {
            CK(cudaFree(ctx->iprov));
            CK(cudaFree(ctx->idepth));
            CK(cudaFree(ctx->idist));
            ctx->iprov = nullptr;
            ctx->idepth = nullptr;
            ctx->idist = nullptr;
            CK(cudaMalloc(&ctx->iprov, px));
            CK(cudaMalloc(&ctx->idepth, px * sizeof(float)));
            CK(cudaMalloc(&ctx->idist, 4 * px * sizeof(int16_t)));
            ctx->icap = px;
        }
        if (!rp.prov_out) rp.prov_out = ctx->iprov;
        rp.depth_out = ctx->idepth;
        ip.W = virt.width;
        ip.H = virt.height;
        ip.radius = cfg.inpaint_radius;
        ip.bg_band = 0.05;
        ip.rgb = rgb_out;
        ip.prov = rp.prov_out;
        ip.depth = ctx->idepth;
        ip.dist_l = ctx->idist;
        ip.dist_r = ctx->idist + px;
        ip.dist_u = ctx->idist + 2 * px;
        ip.dist_d = ctx->idist + 3 * px;
    }
    if (r == 1 && resolve_uses_tma() &&
        (rc = canvas_tensor_map(ctx, ctx->cn, virt.width, virt.height, r, rp)))
        return rc;
    if (FVV_K3_SKIP && r == 1 && cfg.crack_fill_window == 3 &&
        (rc = tile_flags(ctx, n, virt.width, virt.height, wp, rp)))
        return rc;
    LAUNCH_K(FVV_K_FORWARD_WARP, launch_forward_warp(wp, maxpx, ctx->stream));
    LAUNCH_K(FVV_K_RESOLVE, launch_resolve(rp, ctx->stream));
    if (ip.rgb) {
        LAUNCH(launch_inpaint(ip, ctx->stream));
        ctx->launches += 2;   // rows, columns and fill passes
    }
    return FVV_OK;
}

int check_slot_ready(fvv_ctx *ctx, int slot) {
    if (slot < 0 || slot >= FVV_MAX_SLOTS) return fail(ctx, FVV_EINVAL, "slot %d out of range", slot);
    const Slot &s = ctx->slots[slot];
    if (!s.has_cam) return fail(ctx, FVV_EINVAL, "slot %d has no camera", slot);
    if (!s.has_frame) return fail(ctx, FVV_EINVAL, "missing inputs for reference slot %d", slot);
    if (!s.has_bg) return fail(ctx, FVV_EINVAL, "slot %d has no background model", slot);
    return FVV_OK;
}

}  // namespace

extern "C" {

const char *fvv_version(void) { return "fvv_b200 0.1 sm_100a"; }

int fvv_ctx_create(int32_t device, fvv_ctx **out) {
    if (!out) return FVV_EINVAL;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return FVV_ECUDA;
    }
    if (device < 0 || device >= count) return FVV_EINVAL;
    fvv_ctx *ctx = new fvv_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return FVV_ECUDA;
    }
    *out = ctx;
    return FVV_OK;
}

int fvv_ctx_destroy(fvv_ctx *ctx) {
    if (!ctx) return FVV_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto &s : ctx->slots) s.release();
    for (auto &s : ctx->tmp) s.release();
    cudaFree(ctx->canvas);
    cudaFree(ctx->zsrc);
    cudaFree(ctx->dgen);
    cudaFree(ctx->prof_atomics);
    cudaFree(ctx->dq);
    cudaFree(ctx->rle.block);
    cudaFree(ctx->rle.n_runs);
    for (void *q : {(void *)ctx->rice.zz, (void *)ctx->rice.res, (void *)ctx->rice.skew,
                    (void *)ctx->rice.block,
                    (void *)ctx->rice.costs, (void *)ctx->rice.total, (void *)ctx->rice.entry,
                    (void *)ctx->rice.exit, (void *)ctx->rice.exit_prev, (void *)ctx->rice.count,
                    (void *)ctx->rice.changed, (void *)ctx->rice.edge, (void *)ctx->rice.wave})
        cudaFree(q);
    cudaFree(ctx->cand);
    cudaFree(ctx->tflag);
    cudaFree(ctx->ncand);
    cudaFree(ctx->iprov);
    cudaFree(ctx->idepth);
    cudaFree(ctx->idist);
    cudaFree(ctx->range_w);
    for (auto &r : ctx->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : ctx->pool) cudaEventDestroy(e);
    delete ctx;
    return FVV_OK;
}

int fvv_ctx_set_stream(fvv_ctx *ctx, void *stream) {
    if (!ctx) return FVV_EINVAL;
    ctx->stream = (cudaStream_t)stream;
    return FVV_OK;
}

int fvv_sync(fvv_ctx *ctx) {
    int rc = enter(ctx);
    if (rc) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    return FVV_OK;
}

const char *fvv_last_error(const fvv_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t fvv_launch_count(const fvv_ctx *ctx) { return ctx ? ctx->launches : 0; }

static int prof_drain(fvv_ctx *ctx) {
    for (auto &r : ctx->recs) {
        CK(cudaEventSynchronize(r.b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.a, r.b));
        ctx->prof_ms[r.kid] += ms;
        ctx->prof_n[r.kid] += 1;
        ctx->pool.push_back(r.a);
        ctx->pool.push_back(r.b);
    }
    ctx->recs.clear();
    return FVV_OK;
}

int fvv_selftest_division(fvv_ctx *ctx, int64_t n, uint64_t seed, int32_t mode,
                          uint64_t *mismatches_dev) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (n < 0 || mode < 0 || mode > 5 || !mismatches_dev)
        return fail(ctx, FVV_EINVAL, "selftest_division: bad arguments");
    LAUNCH(launch_selftest_div(n, seed, mode, (unsigned long long *)mismatches_dev, ctx->stream));
    return FVV_OK;
}

int fvv_profile_enable(fvv_ctx *ctx, int32_t enable) {
    int rc = enter(ctx);
    if (rc) return rc;
    if ((rc = prof_drain(ctx))) return rc;
    ctx->prof = enable != 0;
    for (int i = 0; i < 5; ++i) { ctx->prof_ms[i] = 0; ctx->prof_n[i] = 0; }
    return FVV_OK;
}

int fvv_count_atomics(fvv_ctx *ctx, int32_t enable) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (enable) {
        if (!ctx->prof_atomics) CK(cudaMalloc(&ctx->prof_atomics, 256 * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(ctx->prof_atomics, 0, 256 * sizeof(unsigned long long), ctx->stream));
    }
    ctx->count_atomics = enable != 0;
    return FVV_OK;
}

int fvv_profile_atomics(fvv_ctx *ctx, int64_t *atomics) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (!atomics) return fail(ctx, FVV_EINVAL, "profile_atomics: NULL");
    *atomics = 0;
    if (!ctx->prof_atomics) return FVV_OK;
    unsigned long long v[256];
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(v, ctx->prof_atomics, sizeof(v), cudaMemcpyDeviceToHost));
    for (int i = 0; i < 256; ++i) *atomics += (int64_t)v[i];
    return FVV_OK;
}

int fvv_profile_read(fvv_ctx *ctx, int32_t kernel_id, double *total_ms, int64_t *launches) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (kernel_id < 0 || kernel_id > 4 || !total_ms || !launches)
        return fail(ctx, FVV_EINVAL, "profile_read: bad arguments");
    if ((rc = prof_drain(ctx))) return rc;
    *total_ms = ctx->prof_ms[kernel_id];
    *launches = ctx->prof_n[kernel_id];
    return FVV_OK;
}

int fvv_decode_mm(fvv_ctx *ctx, const uint16_t *mm, const uint8_t *validity_in, int32_t width,
                  int32_t height, float *depth_out, uint8_t *validity_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (width < 0 || height < 0 || !mm || !depth_out || !validity_out)
        return fail(ctx, FVV_EINVAL, "decode_mm: bad arguments");
    if (width == 0 || height == 0) return FVV_OK;
    PreprocParams p{};
    p.W = width;
    p.H = height;
    p.src = kSrcMM;
    p.mm = mm;
    p.validity = validity_in;
    p.depth_out = depth_out;
    p.validity_out = validity_out;
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    return FVV_OK;
}

int fvv_decode_yuv420_12(fvv_ctx *ctx, const uint8_t *y, const uint8_t *u, const uint8_t *v,
                         int32_t width, int32_t height, double z_near, double z_far,
                         float *depth_out, uint8_t *validity_out, uint16_t *codes_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (width < 0 || height < 0 || width % 2 || height % 2)
        return fail(ctx, FVV_EINVAL, "YUV420 dimensions must be even");
    if (!(0 < z_near && z_near < z_far))
        return fail(ctx, FVV_EINVAL, "need 0 < z_near < z_far");
    if (!y || !u || !v || !depth_out || !validity_out)
        return fail(ctx, FVV_EINVAL, "decode_yuv420_12: NULL buffer");
    if (width == 0 || height == 0) return FVV_OK;
    PreprocParams p{};
    p.W = width;
    p.H = height;
    p.src = kSrcYUV;
    p.y = y; p.u = u; p.v = v;
    p.inv_span = 1.0 / z_near - 1.0 / z_far;  // depthcodec.py:121
    p.inv_zf = 1.0 / z_far;
    if ((rc = dq_table(ctx, p))) return rc;
    p.depth_out = depth_out;
    p.validity_out = validity_out;
    p.codes_out = codes_out;
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    return FVV_OK;
}

int fvv_dequantize12(fvv_ctx *ctx, const uint16_t *codes, int32_t width, int32_t height,
                     double z_near, double z_far, float *depth_out, uint8_t *validity_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (width < 0 || height < 0 || !codes || !depth_out || !validity_out)
        return fail(ctx, FVV_EINVAL, "dequantize12: bad arguments");
    if (!(0 < z_near && z_near < z_far)) return fail(ctx, FVV_EINVAL, "need 0 < z_near < z_far");
    if (width == 0 || height == 0) return FVV_OK;
    PreprocParams p{};
    p.W = width;
    p.H = height;
    p.src = kSrcCodes;
    p.codes = codes;
    p.inv_span = 1.0 / z_near - 1.0 / z_far;
    p.inv_zf = 1.0 / z_far;
    if ((rc = dq_table(ctx, p))) return rc;
    p.depth_out = depth_out;
    p.validity_out = validity_out;
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    return FVV_OK;
}

int fvv_set_range_weights(fvv_ctx *ctx, double sigma_range, const double *table, int32_t n) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (!table || n != kRangeTableLen)
        return fail(ctx, FVV_EINVAL, "range-weight table must hold %d doubles", kRangeTableLen);
    if (!(sigma_range != 0.0 && std::isfinite(sigma_range)))
        return fail(ctx, FVV_EINVAL, "sigma_range must be finite and non-zero");
    return range_table(ctx, sigma_range, table);
}

int fvv_bilateral_close_holes(fvv_ctx *ctx, const float *depth, const uint8_t *validity,
                              const uint8_t *rgb, int32_t width, int32_t height, int32_t radius,
                              double sigma_spatial, double sigma_range, int32_t min_valid,
                              float *depth_out, uint8_t *validity_out, int32_t *n_holes_dev) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (width < 0 || height < 0 || !depth || !validity || !rgb || !depth_out || !validity_out)
        return fail(ctx, FVV_EINVAL, "bilateral_close_holes: bad arguments");
    if (radius < 0 || radius > 4)
        return fail(ctx, FVV_EINVAL, "bilateral radius must be in [0, 4]");
    if (width == 0 || height == 0) return FVV_OK;
    PreprocParams p{};
    p.W = width;
    p.H = height;
    p.src = kSrcF32;
    p.depth = depth;
    p.validity = validity;
    p.rgb = rgb;
    if ((rc = bilateral_params(ctx, p, radius, sigma_spatial, sigma_range, min_valid))) return rc;
    if ((rc = with_fill(ctx, p))) return rc;
    p.depth_out = depth_out;
    p.validity_out = validity_out;
    p.n_holes = n_holes_dev;
    if (n_holes_dev) CK(cudaMemsetAsync(n_holes_dev, 0, sizeof(int32_t), ctx->stream));
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    return FVV_OK;
}

static QuantParams quant_params(double zn, double zf) {
    QuantParams q;
    q.zn = zn;
    q.zf = zf;
    q.lo = zn * (1.0 - 0.01);  // depthcodec.py:101-102 (GUARD_BAND = 0.01)
    q.hi = zf * (1.0 + 0.01);
    q.inv_zf = 1.0 / zf;
    q.inv_span = 1.0 / zn - 1.0 / zf;
    return q;
}

#define NEED(cond, msg) \
    do {                \
        if (!(cond)) return fail(ctx, FVV_EINVAL, "%s", msg); \
    } while (0)

int fvv_correct_depth(fvv_ctx *ctx, const float *depth, const uint8_t *validity, int32_t width,
                      int32_t height, double alpha, double beta, float *depth_out,
                      uint8_t *validity_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width >= 0 && height >= 0 && depth && validity && depth_out && validity_out,
         "correct_depth: bad arguments");
    NEED(std::isfinite(alpha) && std::isfinite(beta), "correction model parameters must be finite");
    if (!width || !height) return FVV_OK;
    LAUNCH_K(FVV_K_OTHER, launch_correct_depth(depth, validity, (size_t)width * height, alpha, beta,
                                               depth_out, validity_out, ctx->stream));
    return FVV_OK;
}

int fvv_bg_train(fvv_ctx *ctx, const uint8_t *rgb, int32_t width, int32_t height, double *mean,
                 double *var, int32_t first, double learning_rate, double var_floor) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width >= 0 && height >= 0 && rgb && mean && var, "bg_train: bad arguments");
    if (!width || !height) return FVV_OK;
    LAUNCH_K(FVV_K_OTHER, launch_bg_train(rgb, (size_t)width * height, mean, var, first != 0,
                                          learning_rate, var_floor, ctx->stream));
    return FVV_OK;
}

int fvv_classify_fg(fvv_ctx *ctx, const uint8_t *rgb, const double *mean, const double *var,
                    int32_t width, int32_t height, double threshold, uint8_t *fg_mask_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width >= 0 && height >= 0 && rgb && mean && var && fg_mask_out,
         "classify_fg: bad arguments");
    if (!width || !height) return FVV_OK;
    LAUNCH_K(FVV_K_OTHER, launch_classify_fg(rgb, mean, var, (size_t)width * height,
                                             threshold * threshold, fg_mask_out, ctx->stream));
    return FVV_OK;
}

int fvv_remove_bg_depth(fvv_ctx *ctx, const float *depth, const uint8_t *validity,
                        const uint8_t *fg_mask, int32_t width, int32_t height, float *depth_out,
                        uint8_t *validity_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width >= 0 && height >= 0 && depth && validity && fg_mask && depth_out && validity_out,
         "remove_bg_depth: bad arguments");
    if (!width || !height) return FVV_OK;
    LAUNCH_K(FVV_K_OTHER, launch_remove_bg(depth, validity, fg_mask, (size_t)width * height,
                                           depth_out, validity_out, ctx->stream));
    return FVV_OK;
}

int fvv_quantize12(fvv_ctx *ctx, const float *depth, const uint8_t *validity, int32_t width,
                   int32_t height, double z_near, double z_far, uint16_t *codes_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width >= 0 && height >= 0 && depth && validity && codes_out, "quantize12: bad arguments");
    NEED(0 < z_near && z_near < z_far, "need 0 < z_near < z_far");
    if (!width || !height) return FVV_OK;
    LAUNCH_K(FVV_K_OTHER, launch_quantize12(depth, validity, (size_t)width * height,
                                            quant_params(z_near, z_far), codes_out, ctx->stream));
    return FVV_OK;
}

int fvv_pack_yuv420(fvv_ctx *ctx, const uint16_t *codes, int32_t width, int32_t height,
                    uint8_t *y_out, uint8_t *u_out, uint8_t *v_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width >= 0 && height >= 0 && codes && y_out && u_out && v_out, "pack_yuv420: bad arguments");
    NEED(width % 2 == 0 && height % 2 == 0, "disparity map dimensions must be even");
    if (!width || !height) return FVV_OK;
    LAUNCH_K(FVV_K_OTHER, launch_pack_yuv420(codes, width, height, y_out, u_out, v_out, ctx->stream));
    return FVV_OK;
}

int fvv_capture_encode(fvv_ctx *ctx, const float *depth, const uint8_t *validity,
                       const uint8_t *rgb, int32_t width, int32_t height, int32_t do_correct,
                       double alpha, double beta, const double *bg_mean, const double *bg_var,
                       double threshold, double z_near, double z_far, uint8_t *y_out,
                       uint8_t *u_out, uint8_t *v_out, uint16_t *codes_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width >= 0 && height >= 0 && depth && validity && y_out && u_out && v_out,
         "capture_encode: bad arguments");
    NEED(width % 2 == 0 && height % 2 == 0, "YUV420 dimensions must be even");
    NEED(0 < z_near && z_near < z_far, "need 0 < z_near < z_far");
    NEED(!bg_mean || (bg_var && rgb), "BG removal needs the colour frame and model variance");
    if (!width || !height) return FVV_OK;
    CaptureParams p{};
    p.W = width;
    p.H = height;
    p.depth = depth;
    p.validity = validity;
    p.rgb = rgb;
    p.correct = do_correct != 0;
    p.alpha = alpha;
    p.beta = beta;
    p.bg_mean = bg_mean;
    p.bg_var = bg_var;
    p.tau2 = threshold * threshold;
    p.quant = quant_params(z_near, z_far);
    p.y = y_out;
    p.u = u_out;
    p.v = v_out;
    p.codes_out = codes_out;
    LAUNCH_K(FVV_K_OTHER, launch_capture_encode(p, ctx->stream));
    return FVV_OK;
}

int64_t fvv_rice_stream_bound(int32_t width, int32_t height) {
    if (width < 0 || height < 0) return -1;
    return rice_stream_bound(width, height);
}

// ---------------------------------------------------------------------------
// MVD disk container rasters (mvdio.py, core.py:246-255)

int fvv_encode_mm(fvv_ctx *ctx, const float *depth, const uint8_t *validity, int32_t width,
                  int32_t height, uint16_t *mm_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width >= 0 && height >= 0 && depth && validity && mm_out, "encode_mm: bad arguments");
    if (!width || !height) return FVV_OK;
    LAUNCH_K(FVV_K_OTHER, launch_encode_mm(depth, validity, (long long)width * height, mm_out,
                                           ctx->stream));
    return FVV_OK;
}

int fvv_rle_decode(fvv_ctx *ctx, const uint8_t *codes, const int64_t *ends, int64_t n_runs,
                   int64_t n, uint8_t *out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(n >= 0 && n_runs >= 0 && (n == 0 || (n_runs > 0 && codes && ends && out)),
         "rle_decode: bad arguments");
    if (!n) return FVV_OK;
    LAUNCH_K(FVV_K_OTHER, launch_rle_decode(codes, reinterpret_cast<const long long *>(ends),
                                            n_runs, n, out, ctx->stream));
    return FVV_OK;
}

int fvv_rle_encode(fvv_ctx *ctx, const uint8_t *flat, int64_t n, int64_t *starts_out,
                   uint8_t *codes_out, int64_t *n_runs_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(n >= 0 && n_runs_out && (n == 0 || (flat && starts_out && codes_out)),
         "rle_encode: bad arguments");
    const size_t nb = (size_t)((n + kRlePx - 1) / kRlePx);
    if (nb + 1 > ctx->rle.cap || !ctx->rle.n_runs) {
        CK(cudaFree(ctx->rle.block));
        ctx->rle.block = nullptr;
        CK(cudaMalloc(&ctx->rle.block, (nb + 1) * sizeof(unsigned long long)));
        if (!ctx->rle.n_runs) CK(cudaMalloc(&ctx->rle.n_runs, sizeof(long long)));
        ctx->rle.cap = nb + 1;
    }
    LAUNCH(launch_rle_encode(flat, n, reinterpret_cast<long long *>(starts_out), codes_out,
                             ctx->rle, ctx->stream));
    ctx->launches += n > 0 ? 2 : 0;   // k_rle_count, k_rle_scan, k_rle_write
    long long nr = 0;
    CK(cudaMemcpyAsync(&nr, ctx->rle.n_runs, sizeof(nr), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *n_runs_out = nr;
    return FVV_OK;
}

int fvv_rice_encode_plane(fvv_ctx *ctx, const uint8_t *plane, int32_t width, int32_t height,
                          uint8_t *stream_out, int32_t *k_out, int64_t *nbits_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width > 0 && height > 0 && plane && stream_out && k_out && nbits_out,
         "rice_encode_plane: bad arguments");
    const size_t n = (size_t)width * height;
    if ((rc = rice_scratch(ctx, n, 0))) return rc;
    int k = 0;
    long long nbits = 0;
    LAUNCH(rice_encode(plane, width, height, ctx->rice, stream_out, &k, &nbits, ctx->stream));
    ctx->launches += 3;  // k_med_zz, k_rice_lens, k_scan_blocks, k_rice_write
    *k_out = k;
    *nbits_out = nbits;
    return FVV_OK;
}

int fvv_rice_decode_planes(fvv_ctx *ctx, int32_t n, const uint8_t *const *streams,
                           const int64_t *nbytes, const int32_t *ks, const int32_t *widths,
                           const int32_t *heights, uint8_t *const *planes_out,
                           uint32_t *adlers_out, int32_t *status_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(n >= 0 && n <= kRiceMaxPlanes, "rice_decode_planes: 0..48 planes per call");
    if (!n) return FVV_OK;
    NEED(streams && nbytes && ks && widths && heights && planes_out && adlers_out && status_out,
         "rice_decode_planes: NULL argument array");
    RicePlane pl[kRiceMaxPlanes];
    size_t px = 0, skew = 0, edge = 0, chunks = 0;
    for (int i = 0; i < n; ++i) {
        NEED(widths[i] > 0 && heights[i] > 0 && planes_out[i] && nbytes[i] >= 0 &&
                 (streams[i] || !nbytes[i]),
             "rice_decode_planes: bad plane");
        NEED(ks[i] >= 0 && ks[i] <= 48, "rice parameter out of range");
        NEED(widths[i] <= kMedMaxWidth && heights[i] <= 4096, "plane too large for the MED rebuild");
        pl[i] = RicePlane{};
        pl[i].s = streams[i];
        pl[i].nbytes = nbytes[i];
        pl[i].k = ks[i];
        pl[i].W = widths[i];
        pl[i].H = heights[i];
        pl[i].out = planes_out[i];
        px += (size_t)widths[i] * heights[i];
        skew += rice_skew_size(widths[i], heights[i]);
        edge += rice_edge_size(widths[i], heights[i]);
        chunks += (size_t)((nbytes[i] * 8 + kRiceChunkBits - 1) / kRiceChunkBits);
    }
    if ((rc = rice_scratch(ctx, px, chunks + n, skew, edge))) return rc;
    {
        const cudaError_t e = rice_decode_batch(pl, n, ctx->rice, ctx->stream);
        if (e == cudaErrorLaunchTimeout)  // the rebuild's stall flag (k_med_rebuild_wave)
            return fail(ctx, FVV_ECUDA, "MED rebuild: a strip never received the row above it");
        LAUNCH(e);
    }
    ctx->launches += 12;  // spec, >= 2 sync rounds, 4 scan kernels, emit, rebuild, deskew, adler
    for (int i = 0; i < n; ++i) {
        status_out[i] = pl[i].status;
        adlers_out[i] = pl[i].status ? 0u : pl[i].adler;
    }
    return FVV_OK;
}

int fvv_rice_decode_plane(fvv_ctx *ctx, const uint8_t *stream, int64_t nbytes, int32_t k,
                          int64_t n_symbols, int32_t width, int32_t height, uint8_t *plane_out,
                          uint32_t *adler_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    NEED(width > 0 && height > 0 && plane_out && adler_out && nbytes >= 0 && (stream || !nbytes),
         "rice_decode_plane: bad arguments");
    NEED(n_symbols == (int64_t)width * height, "plane symbol count mismatch");
    int32_t status = 0;
    if ((rc = fvv_rice_decode_planes(ctx, 1, &stream, &nbytes, &k, &width, &height, &plane_out,
                                     adler_out, &status)))
        return rc;
    if (status) return fail(ctx, FVV_EINVAL, "rice stream truncated");
    return FVV_OK;
}

int fvv_slot_set_camera(fvv_ctx *ctx, int32_t slot, const fvv_camera *cam) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (slot < 0 || slot >= FVV_MAX_SLOTS) return fail(ctx, FVV_EINVAL, "slot %d out of range", slot);
    if ((rc = check_cam(ctx, cam, "slot"))) return rc;
    return slot_camera(ctx, ctx->slots[slot], *cam);
}

int fvv_ctx_device_generation(fvv_ctx *ctx, int32_t enable) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (enable && !ctx->dgen) CK(cudaMalloc(&ctx->dgen, 2 * sizeof(int)));
    if (enable && !ctx->dev_gen) {
        CK(cudaMemsetAsync(ctx->dgen, 0, 2 * sizeof(int), ctx->stream));
        CK(cudaMemsetAsync(ctx->dgen, 0xFF, sizeof(int), ctx->stream));   // fill first
    }
    if (!enable && ctx->dev_gen) ctx->gen = -1;   // host rule restarts with a fill
    ctx->dev_gen = enable != 0;
    return FVV_OK;
}

int fvv_slot_reset(fvv_ctx *ctx, int32_t slot) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (slot < 0 || slot >= FVV_MAX_SLOTS) return fail(ctx, FVV_EINVAL, "slot %d out of range", slot);
    ctx->slots[slot].has_bg = ctx->slots[slot].has_frame = false;
    return FVV_OK;
}

int fvv_slot_set_bg(fvv_ctx *ctx, int32_t slot, const float *bg_depth, const uint8_t *bg_validity) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (slot < 0 || slot >= FVV_MAX_SLOTS || !ctx->slots[slot].has_cam)
        return fail(ctx, FVV_EINVAL, "slot %d has no camera", slot);
    if (!bg_depth || !bg_validity) return fail(ctx, FVV_EINVAL, "bg model: NULL buffer");
    Slot &s = ctx->slots[slot];
    PreprocParams p = base_pre(s);
    p.src = kSrcF32;
    p.depth = bg_depth;
    p.validity = bg_validity;
    p.warp_depth = s.bgd;
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    s.has_bg = true;
    return FVV_OK;
}

int fvv_slot_ingest(fvv_ctx *ctx, int32_t slot, const uint8_t *rgb, const float *depth,
                    const uint8_t *validity, int32_t hole_closing) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (slot < 0 || slot >= FVV_MAX_SLOTS || !ctx->slots[slot].has_cam)
        return fail(ctx, FVV_EINVAL, "slot %d has no camera", slot);
    if (!rgb || !depth || !validity) return fail(ctx, FVV_EINVAL, "ingest: NULL buffer");
    Slot &s = ctx->slots[slot];
    PreprocParams p = base_pre(s);
    p.src = kSrcF32;
    p.depth = depth;
    p.validity = validity;
    p.rgb = rgb;
    if (hole_closing && (rc = bilateral_defaults(ctx, p))) return rc;
    if ((rc = with_fill(ctx, p))) return rc;
    p.texel = s.texel;
    p.warp_depth = s.fgd;
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    s.has_frame = true;
    return FVV_OK;
}

int fvv_slot_ingest_mm(fvv_ctx *ctx, int32_t slot, const uint8_t *rgb, const uint16_t *mm,
                       const uint8_t *validity, int32_t hole_closing, float *depth_out,
                       uint8_t *validity_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (slot < 0 || slot >= FVV_MAX_SLOTS || !ctx->slots[slot].has_cam)
        return fail(ctx, FVV_EINVAL, "slot %d has no camera", slot);
    if (!rgb || !mm) return fail(ctx, FVV_EINVAL, "ingest_mm: NULL buffer");
    Slot &s = ctx->slots[slot];
    PreprocParams p = base_pre(s);
    p.src = kSrcMM;
    p.mm = mm;
    p.validity = validity;
    p.rgb = rgb;
    if (hole_closing && (rc = bilateral_defaults(ctx, p))) return rc;
    if ((rc = with_fill(ctx, p))) return rc;
    p.texel = s.texel;
    p.warp_depth = s.fgd;
    p.depth_out = depth_out;
    p.validity_out = validity_out;
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    s.has_frame = true;
    return FVV_OK;
}

int fvv_slots_ingest_mm(fvv_ctx *ctx, int32_t n, const int32_t *slots,
                        const uint8_t *const *rgb, const uint16_t *const *mm,
                        const uint8_t *const *validity, int32_t hole_closing) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (n < 0 || n > FVV_MAX_REFS || (n && (!slots || !rgb || !mm)))
        return fail(ctx, FVV_EINVAL, "slots_ingest_mm: bad arguments");
    PreprocBatch b{};
    if (hole_closing && (rc = bilateral_defaults(ctx, b.bil))) return rc;
    b.n = n;
    for (int i = 0; i < n; ++i) {
        const int sl = slots[i];
        if (sl < 0 || sl >= FVV_MAX_SLOTS || !ctx->slots[sl].has_cam)
            return fail(ctx, FVV_EINVAL, "slot %d has no camera", sl);
        if (!rgb[i] || !mm[i]) return fail(ctx, FVV_EINVAL, "slots_ingest_mm: NULL buffer");
        Slot &s = ctx->slots[sl];
        PreprocCore &c = b.cam[i];
        c.W = s.cam.width;
        c.H = s.cam.height;
        c.src = kSrcMM;
        c.mm = mm[i];
        c.validity = validity ? validity[i] : nullptr;
        c.rgb = rgb[i];
        c.texel = s.texel;
        c.warp_depth = s.fgd;
    }
    if (hole_closing) {
        size_t px = 0;
        for (int i = 0; i < n; ++i) px += (size_t)b.cam[i].W * b.cam[i].H;
        if ((rc = fill_list(ctx, px, b.cand, b.ncand))) return rc;
    }
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess_batch(b, ctx->stream));
    for (int i = 0; i < n; ++i) ctx->slots[slots[i]].has_frame = true;
    return FVV_OK;
}

int fvv_slots_ingest_yuv(fvv_ctx *ctx, int32_t n, const int32_t *slots,
                         const uint8_t *const *rgb, const uint8_t *const *y,
                         const uint8_t *const *u, const uint8_t *const *v, double z_near,
                         double z_far, int32_t hole_closing) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (n < 0 || n > FVV_MAX_REFS || (n && (!slots || !rgb || !y || !u || !v)))
        return fail(ctx, FVV_EINVAL, "slots_ingest_yuv: bad arguments");
    if (!(0 < z_near && z_near < z_far)) return fail(ctx, FVV_EINVAL, "need 0 < z_near < z_far");
    PreprocBatch b{};
    if (hole_closing && (rc = bilateral_defaults(ctx, b.bil))) return rc;
    b.n = n;
    for (int i = 0; i < n; ++i) {
        const int sl = slots[i];
        if (sl < 0 || sl >= FVV_MAX_SLOTS || !ctx->slots[sl].has_cam)
            return fail(ctx, FVV_EINVAL, "slot %d has no camera", sl);
        if (!rgb[i] || !y[i] || !u[i] || !v[i])
            return fail(ctx, FVV_EINVAL, "slots_ingest_yuv: NULL buffer");
        Slot &s = ctx->slots[sl];
        PreprocCore &c = b.cam[i];
        c.W = s.cam.width;
        c.H = s.cam.height;
        c.src = kSrcYUV;
        c.y = y[i];
        c.u = u[i];
        c.v = v[i];
        // host-evaluated like numpy's 1/zn - 1/zf, 1/zf (depthcodec.py:113-125)
        c.inv_span = 1.0 / z_near - 1.0 / z_far;
        c.inv_zf = 1.0 / z_far;
        if ((rc = dq_table(ctx, c))) return rc;
        c.rgb = rgb[i];
        c.texel = s.texel;
        c.warp_depth = s.fgd;
    }
    if (hole_closing) {
        size_t px = 0;
        for (int i = 0; i < n; ++i) px += (size_t)b.cam[i].W * b.cam[i].H;
        if ((rc = fill_list(ctx, px, b.cand, b.ncand))) return rc;
    }
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess_batch(b, ctx->stream));
    for (int i = 0; i < n; ++i) ctx->slots[slots[i]].has_frame = true;
    return FVV_OK;
}

int fvv_slot_ingest_yuv(fvv_ctx *ctx, int32_t slot, const uint8_t *rgb, const uint8_t *y,
                        const uint8_t *u, const uint8_t *v, double z_near, double z_far,
                        int32_t hole_closing, float *depth_out, uint8_t *validity_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (slot < 0 || slot >= FVV_MAX_SLOTS || !ctx->slots[slot].has_cam)
        return fail(ctx, FVV_EINVAL, "slot %d has no camera", slot);
    if (!rgb || !y || !u || !v) return fail(ctx, FVV_EINVAL, "ingest_yuv: NULL buffer");
    if (!(0 < z_near && z_near < z_far)) return fail(ctx, FVV_EINVAL, "need 0 < z_near < z_far");
    Slot &s = ctx->slots[slot];
    PreprocParams p = base_pre(s);
    p.src = kSrcYUV;
    p.y = y; p.u = u; p.v = v;
    p.inv_span = 1.0 / z_near - 1.0 / z_far;
    p.inv_zf = 1.0 / z_far;
    if ((rc = dq_table(ctx, p))) return rc;
    p.rgb = rgb;
    if (hole_closing && (rc = bilateral_defaults(ctx, p))) return rc;
    if ((rc = with_fill(ctx, p))) return rc;
    p.texel = s.texel;
    p.warp_depth = s.fgd;
    p.depth_out = depth_out;
    p.validity_out = validity_out;
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    s.has_frame = true;
    return FVV_OK;
}

int fvv_render_views(fvv_ctx *ctx, const fvv_camera *virts, int32_t n_views,
                     const int32_t *ref_slots, const double *weights, int32_t n_refs,
                     const fvv_synth_cfg *cfg, uint8_t *rgb_out, uint8_t *provenance_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (n_views < 0 || !virts || !ref_slots) return fail(ctx, FVV_EINVAL, "render_views: bad arguments");
    if (n_refs < 1) return fail(ctx, FVV_EINVAL, "need at least one reference camera");
    if (n_refs > FVV_MAX_REFS) return fail(ctx, FVV_EINVAL, "more than %d references", FVV_MAX_REFS);
    if ((rc = check_cfg(ctx, cfg))) return rc;
    for (int i = 0; i < n_views; ++i) {
        if ((rc = check_cam(ctx, &virts[i], "virtual"))) return rc;
        if (virts[i].width != virts[0].width || virts[i].height != virts[0].height)
            return fail(ctx, FVV_EINVAL, "all virtual views of a batch must share one size");
        Slot *refs[FVV_MAX_REFS];
        for (int j = 0; j < n_refs; ++j) {
            const int sl = ref_slots[(size_t)i * n_refs + j];
            if ((rc = check_slot_ready(ctx, sl))) return rc;
            refs[j] = &ctx->slots[sl];
        }
        const size_t px = (size_t)virts[i].width * virts[i].height;
        rc = render_view(ctx, virts[i], refs, weights ? weights + (size_t)i * n_refs : nullptr,
                         n_refs, *cfg, rgb_out ? rgb_out + px * 3 * i : nullptr,
                         provenance_out ? provenance_out + px * i : nullptr, nullptr);
        if (rc) return rc;
    }
    return FVV_OK;
}

int fvv_synthesize_view(fvv_ctx *ctx, const fvv_camera *virt, const fvv_ref_frame *refs,
                        int32_t n_refs, const fvv_synth_cfg *cfg, uint8_t *rgb_out,
                        uint8_t *provenance_out, const fvv_debug *dbg) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (n_refs < 1 || !refs) return fail(ctx, FVV_EINVAL, "need at least one reference camera");
    if (n_refs > FVV_MAX_REFS) return fail(ctx, FVV_EINVAL, "more than %d references", FVV_MAX_REFS);
    if ((rc = check_cfg(ctx, cfg))) return rc;
    if ((rc = check_cam(ctx, virt, "virtual"))) return rc;
    Slot *sl[FVV_MAX_REFS];
    double w[FVV_MAX_REFS];
    for (int j = 0; j < n_refs; ++j) {
        const fvv_ref_frame &f = refs[j];
        if ((rc = check_cam(ctx, &f.cam, "reference"))) return rc;
        if (!f.rgb || !f.live_depth || !f.live_validity || !f.bg_depth || !f.bg_validity)
            return fail(ctx, FVV_EINVAL, "missing inputs for reference camera %d", f.cam.id);
        Slot &s = ctx->tmp[j];
        if ((rc = slot_camera(ctx, s, f.cam))) return rc;
        PreprocParams p = base_pre(s);
        p.src = kSrcF32;
        p.depth = f.live_depth;
        p.validity = f.live_validity;
        p.rgb = f.rgb;
        p.texel = s.texel;
        p.warp_depth = s.fgd;
        LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
        PreprocParams q = base_pre(s);
        q.src = kSrcF32;
        q.depth = f.bg_depth;
        q.validity = f.bg_validity;
        q.warp_depth = s.bgd;
        LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(q, ctx->stream));
        sl[j] = &s;
        w[j] = f.weight;
    }
    return render_view(ctx, *virt, sl, w, n_refs, *cfg, rgb_out, provenance_out, dbg);
}

int fvv_warp_layer(fvv_ctx *ctx, const fvv_camera *src, const fvv_camera *dst, const uint8_t *rgb,
                   const float *depth, const uint8_t *validity, const uint8_t *color_valid,
                   int32_t layer_fg, const fvv_synth_cfg *cfg, double *color_out,
                   double *depth_out, uint8_t *valid_out, int32_t *winner_out,
                   uint8_t *stage_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if ((rc = check_cfg(ctx, cfg))) return rc;
    if ((rc = check_cam(ctx, src, "source"))) return rc;
    if ((rc = check_cam(ctx, dst, "virtual"))) return rc;
    if (!rgb || !depth || !validity || !valid_out)
        return fail(ctx, FVV_EINVAL, "warp_layer: NULL buffer");
    Slot &s = ctx->tmp[FVV_MAX_REFS];
    if ((rc = slot_camera(ctx, s, *src))) return rc;
    PreprocParams p = base_pre(s);
    p.src = kSrcF32;
    p.depth = depth;
    p.validity = validity;
    p.rgb = rgb;
    p.color_valid = color_valid;
    p.texel = s.texel;
    p.warp_depth = s.fgd;
    if (!color_valid) {
        // colour validity defaults to the depth validity (synthesis.py:185-186):
        // flag bit 0 is exactly that
    }
    LAUNCH_K(FVV_K_PREPROCESS, launch_preprocess(p, ctx->stream));
    const int r = cfg->splat_radius;
    if ((rc = ensure_canvas(ctx, 1, dst->width, dst->height, r))) return rc;
    const DevCam dd = to_dev(*dst);
    const int b = index_bits((long long)src->width * src->height);
    const double *rx = s.rays, *ry = s.rays + src->width;
    WarpParams wp{};
    wp.dst = dd;
    wp.r = r;
    wp.pitch = canvas_pitch(dst->width, r);
    wp.n = 1;
    wp.gen_hi = (uint64_t)ctx->gen << kGenShift;
    wp.gen_ptr = ctx->dev_gen ? ctx->dgen : nullptr;
    if ((rc = ensure_zsrc(ctx, 1, (size_t)src->width * src->height))) return rc;
    wp.c[0] = WarpContrib{s.dev, relative_pose(s.dev, dd), s.fgd, rx, ry, ctx->canvas + 1,
                          ctx->zsrc, b};
    LAUNCH_K(FVV_K_FORWARD_WARP, launch_forward_warp(wp, (long long)src->width * src->height, ctx->stream));
    ResolveParams rp{};
    rp.dst = dd;
    rp.r = r;
    rp.window = cfg->crack_fill_window;
    rp.need = cfg->crack_fill_window * cfg->crack_fill_window / 2 + 1;
    rp.pitch = wp.pitch;
    rp.gen = (uint64_t)ctx->gen;
    rp.gen_ptr = wp.gen_ptr;
    rp.n_fg = layer_fg ? 1 : 0;
    rp.n_bg = layer_fg ? 0 : 1;
    rp.band_rel = cfg->depth_band_rel;
    rp.dbg.contrib_color = color_out;
    rp.dbg.contrib_depth = depth_out;
    rp.dbg.contrib_valid = valid_out;
    rp.dbg.contrib_winner = winner_out;
    rp.dbg.contrib_stage = stage_out;
    rp.c[0] = ResolveContrib{s.dev, relative_pose(dd, s.dev), s.texel, ctx->zsrc, ctx->canvas + 1,
                             host_weight(*src, *dst, cfg->mixing_epsilon), b, kFlagLiveValid,
                             layer_fg ? 1 : 0};
    if (r == 1 && resolve_uses_tma() &&
        (rc = canvas_tensor_map(ctx, ctx->cn, dst->width, dst->height, r, rp)))
        return rc;
    LAUNCH_K(FVV_K_RESOLVE, launch_resolve(rp, ctx->stream));
    return FVV_OK;
}

int fvv_mix_layer(fvv_ctx *ctx, int32_t n, const double *const *colors, const double *const *depths,
                  const uint8_t *const *valids, const double *weights, int32_t width,
                  int32_t height, double depth_band_rel, double *color_out, double *depth_out,
                  uint8_t *valid_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (n < 1) return fail(ctx, FVV_EINVAL, "need at least one contribution");
    if (n > 2 * FVV_MAX_REFS) return fail(ctx, FVV_EINVAL, "too many contributions");
    if (!colors || !depths || !valids || !weights || !color_out || !depth_out || !valid_out)
        return fail(ctx, FVV_EINVAL, "mix_layer: NULL buffer");
    MixParams p{};
    p.n = n;
    p.W = width;
    p.H = height;
    p.band_rel = depth_band_rel;
    for (int j = 0; j < n; ++j) {
        if (!(weights[j] > 0)) return fail(ctx, FVV_EINVAL, "contribution weight must be positive");
        p.color[j] = colors[j];
        p.depth[j] = depths[j];
        p.valid[j] = valids[j];
        p.weight[j] = weights[j];
    }
    p.color_out = color_out;
    p.depth_out = depth_out;
    p.valid_out = valid_out;
    LAUNCH(launch_mix(p, ctx->stream));
    return FVV_OK;
}

int fvv_composite(fvv_ctx *ctx, const double *fg_color, const uint8_t *fg_valid,
                  const double *bg_color, const uint8_t *bg_valid, int32_t width, int32_t height,
                  const uint8_t hole_color[3], uint8_t *rgb_out, uint8_t *provenance_out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (!fg_color || !fg_valid || !bg_color || !bg_valid || !hole_color || !rgb_out)
        return fail(ctx, FVV_EINVAL, "composite: NULL buffer");
    const double hole[3] = {(double)hole_color[0], (double)hole_color[1], (double)hole_color[2]};
    LAUNCH(launch_composite(fg_color, fg_valid, bg_color, bg_valid, width, height, hole, rgb_out,
                            provenance_out, ctx->stream));
    return FVV_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Render-tick queue: the e2e edge-server loop (pipeline.py:514-547 render
// tick, 762-763 on_display) fed from pinned host memory, with every per-tick
// stream and event operation in native code. Tick t uses buffer slot
// t % depth: its span is copied into stage[slot] on the H2D stream (after the
// compute of tick t - depth finished reading that slot), the context's
// stream waits for it and for the download of tick t - depth out of
// dout[slot], runs the tick's ingest (K0 + K1) and render (K2 + K3) into
// dout[slot] — eagerly, or as the CUDA graph captured on the key's second
// occurrence — and the D2H stream copies the views to the caller's pinned
// buffer. depth ticks are in flight, so the copies of ticks t+1 / t-1
// overlap the compute of tick t.

struct fvv_tickq {
    fvv_ctx *ctx = nullptr;
    int depth = 0;
    int64_t span_cap = 0, out_cap = 0;
    int max_graphs = 0;
    std::vector<uint8_t *> stage, dout;
    std::vector<cudaEvent_t> up, done, down;  // span landed / tick's compute done / views landed
    std::vector<bool> used;
    // ticks run on the queue's own compute stream (capturable, unlike the
    // legacy default stream a context may be bound to), ordered after the
    // context stream's work at submission and before its later work
    cudaStream_t h2d = nullptr, d2h = nullptr, comp = nullptr;
    cudaEvent_t entry = nullptr;
    cudaStream_t saved = nullptr;
    int64_t n = 0;
    int64_t h2d_bytes = 0, d2h_bytes = 0, replays = 0;
    struct Graph {
        cudaGraphExec_t exec;
        int64_t span_bytes, out_bytes, launches;
        uint64_t last_use;
    };
    std::map<std::pair<uint64_t, int>, Graph> graphs;  // (key, slot)
    std::map<std::pair<uint64_t, int>, uint64_t> seen;  // eager ticks per (key, slot)
};

namespace {

int tickq_begin(fvv_tickq *q, const void *host_span, int64_t span_bytes, int slot) {
    fvv_ctx *ctx = q->ctx;
    if (q->used[slot]) CK(cudaStreamWaitEvent(q->h2d, q->done[slot], 0));
    CK(cudaMemcpyAsync(q->stage[slot], host_span, (size_t)span_bytes, cudaMemcpyHostToDevice,
                       q->h2d));
    CK(cudaEventRecord(q->up[slot], q->h2d));
    CK(cudaEventRecord(q->entry, ctx->stream));
    CK(cudaStreamWaitEvent(q->comp, q->entry, 0));
    CK(cudaStreamWaitEvent(q->comp, q->up[slot], 0));
    if (q->used[slot]) CK(cudaStreamWaitEvent(q->comp, q->down[slot], 0));
    q->h2d_bytes += span_bytes;
    // the tick's library calls go to the compute stream
    q->saved = ctx->stream;
    ctx->stream = q->comp;
    return FVV_OK;
}

// the context's stream back (after a tick, or after a failed one)
void tickq_restore(fvv_tickq *q) {
    if (q->ctx->stream == q->comp) q->ctx->stream = q->saved;
}

int tickq_end(fvv_tickq *q, void *host_out, int64_t out_bytes, int slot, int64_t *ticket) {
    fvv_ctx *ctx = q->ctx;
    tickq_restore(q);
    CK(cudaEventRecord(q->done[slot], q->comp));
    CK(cudaStreamWaitEvent(ctx->stream, q->done[slot], 0));
    CK(cudaStreamWaitEvent(q->d2h, q->done[slot], 0));
    CK(cudaMemcpyAsync(host_out, q->dout[slot], (size_t)out_bytes, cudaMemcpyDeviceToHost,
                       q->d2h));
    CK(cudaEventRecord(q->down[slot], q->d2h));
    q->used[slot] = true;
    q->d2h_bytes += out_bytes;
    if (ticket) *ticket = q->n;
    ++q->n;
    return FVV_OK;
}

void tickq_evict(fvv_tickq *q) {
    while ((int)q->graphs.size() > q->max_graphs) {
        auto lru = q->graphs.begin();
        for (auto it = q->graphs.begin(); it != q->graphs.end(); ++it)
            if (it->second.last_use < lru->second.last_use) lru = it;
        cudaGraphExecDestroy(lru->second.exec);
        q->graphs.erase(lru);
    }
    while ((int)q->seen.size() > 4 * q->max_graphs) {
        auto old = q->seen.begin();
        for (auto it = q->seen.begin(); it != q->seen.end(); ++it)
            if (it->second < old->second) old = it;
        q->seen.erase(old);
    }
}

}  // namespace

extern "C" {

int fvv_tickq_create(fvv_ctx *ctx, int32_t depth, int64_t span_bytes, int64_t out_bytes,
                     int32_t max_graphs, fvv_tickq **out) {
    int rc = enter(ctx);
    if (rc) return rc;
    if (!out || depth < 1 || depth > 16 || span_bytes <= 0 || out_bytes <= 0 || max_graphs < 0)
        return fail(ctx, FVV_EINVAL, "tickq_create: bad arguments");
    *out = nullptr;
    fvv_tickq *q = new fvv_tickq();
    q->ctx = ctx;
    q->depth = depth;
    q->span_cap = span_bytes;
    q->out_cap = out_bytes;
    q->max_graphs = max_graphs;
    q->stage.assign(depth, nullptr);
    q->dout.assign(depth, nullptr);
    q->up.assign(depth, nullptr);
    q->done.assign(depth, nullptr);
    q->down.assign(depth, nullptr);
    q->used.assign(depth, false);
    cudaError_t e = cudaStreamCreateWithFlags(&q->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&q->d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&q->comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q->entry, cudaEventDisableTiming);
    for (int i = 0; i < depth && e == cudaSuccess; ++i) {
        e = cudaMalloc(&q->stage[i], (size_t)span_bytes);
        if (e == cudaSuccess) e = cudaMalloc(&q->dout[i], (size_t)out_bytes);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q->up[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q->done[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q->down[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        fvv_tickq_destroy(q);
        return fail(ctx, FVV_ECUDA, "tickq_create: %s", cudaGetErrorString(e));
    }
    // captured ticks need the device-resident canvas generation
    if (max_graphs > 0 && (rc = fvv_ctx_device_generation(ctx, 1))) {
        fvv_tickq_destroy(q);
        return rc;
    }
    *out = q;
    return FVV_OK;
}

int fvv_tickq_destroy(fvv_tickq *q) {
    if (!q) return FVV_EINVAL;
    cudaSetDevice(q->ctx->device);
    if (q->h2d) cudaStreamSynchronize(q->h2d);
    if (q->d2h) cudaStreamSynchronize(q->d2h);
    if (q->comp) cudaStreamSynchronize(q->comp);
    for (auto &g : q->graphs) cudaGraphExecDestroy(g.second.exec);
    for (int i = 0; i < q->depth; ++i) {
        cudaFree(q->stage[i]);
        cudaFree(q->dout[i]);
        if (q->up[i]) cudaEventDestroy(q->up[i]);
        if (q->done[i]) cudaEventDestroy(q->done[i]);
        if (q->down[i]) cudaEventDestroy(q->down[i]);
    }
    if (q->h2d) cudaStreamDestroy(q->h2d);
    if (q->d2h) cudaStreamDestroy(q->d2h);
    if (q->comp) cudaStreamDestroy(q->comp);
    if (q->entry) cudaEventDestroy(q->entry);
    delete q;
    return FVV_OK;
}

int fvv_tickq_submit(fvv_tickq *q, const void *host_span, int64_t span_bytes, int32_t kind,
                     int32_t n_cams, const int32_t *slots, const int64_t *offs, double z_near,
                     double z_far, int32_t hole_closing, const fvv_camera *virts,
                     int32_t n_views, const int32_t *ref_slots, const double *weights,
                     int32_t n_refs, const fvv_synth_cfg *cfg, void *host_out, uint64_t key,
                     int64_t *ticket) {
    if (!q) return FVV_EINVAL;
    fvv_ctx *ctx = q->ctx;
    int rc = enter(ctx);
    if (rc) return rc;
    if (!host_span || !host_out || !offs || !slots || !virts || n_views < 1 || n_cams < 1 ||
        n_cams > FVV_MAX_REFS || (kind != 0 && kind != 1))
        return fail(ctx, FVV_EINVAL, "tickq_submit: bad arguments");
    if (span_bytes <= 0 || span_bytes > q->span_cap)
        return fail(ctx, FVV_EINVAL, "tickq_submit: span of %lld bytes, the queue holds %lld",
                    (long long)span_bytes, (long long)q->span_cap);
    const int64_t out_bytes = (int64_t)n_views * virts[0].width * virts[0].height * 3;
    if (out_bytes > q->out_cap)
        return fail(ctx, FVV_EINVAL, "tickq_submit: %d views need %lld output bytes, the queue "
                    "holds %lld", n_views, (long long)out_bytes, (long long)q->out_cap);
    for (int i = 0; i < n_cams; ++i) {
        if (!(slots[i] >= 0 && slots[i] < FVV_MAX_SLOTS && ctx->slots[slots[i]].has_cam))
            return fail(ctx, FVV_EINVAL, "slot %d has no camera", slots[i]);
        const fvv_camera &c = ctx->slots[slots[i]].cam;
        const int64_t px = (int64_t)c.width * c.height;
        // bytes each raster of the camera occupies in the span
        const int64_t need[4] = {3 * px, kind == 0 ? 2 * px : px, kind == 0 ? px : px / 4,
                                 kind == 0 ? 0 : px / 4};
        for (int r = 0; r < 4; ++r) {
            const int64_t o = offs[4 * i + r];
            if (o < 0 && (r == 0 || r == 1 || (kind == 1 && r > 0)))
                return fail(ctx, FVV_EINVAL, "tickq_submit: camera %d lacks raster %d", i, r);
            // 16-byte aligned like a device allocation (K0's vector loads)
            if (o >= 0 && (o + need[r] > span_bytes || (o & 15)))
                return fail(ctx, FVV_EINVAL, "tickq_submit: raster %d of camera %d lies outside "
                            "the span or is not 16-byte aligned", r, i);
        }
    }
    const int slot = (int)(q->n % q->depth);
    const auto gk = std::make_pair(key, slot);
    if ((rc = tickq_begin(q, host_span, span_bytes, slot))) return rc;
    // the tick's ingest + render (the context's stream is the queue's now)
    auto tick = [&]() -> int {
        const uint8_t *base = q->stage[slot];
        const uint8_t *p[4][FVV_MAX_REFS];
        for (int i = 0; i < n_cams; ++i)
            for (int r = 0; r < 4; ++r)
                p[r][i] = offs[4 * i + r] >= 0 ? base + offs[4 * i + r] : nullptr;
        int e;
        if (kind == 0) {
            bool all_v = true;
            for (int i = 0; i < n_cams; ++i) all_v = all_v && p[2][i];
            e = fvv_slots_ingest_mm(ctx, n_cams, slots, p[0],
                                    reinterpret_cast<const uint16_t *const *>(p[1]),
                                    all_v ? p[2] : nullptr, hole_closing);
        } else {
            e = fvv_slots_ingest_yuv(ctx, n_cams, slots, p[0], p[1], p[2], p[3], z_near, z_far,
                                     hole_closing);
        }
        if (e) return e;
        return fvv_render_views(ctx, virts, n_views, ref_slots, weights, n_refs, cfg,
                                q->dout[slot], nullptr);
    };
    // eager, or captured on the key's second occurrence and launched
    auto run = [&]() -> int {
        auto it = key != 0 && q->max_graphs > 0 ? q->seen.find(gk) : q->seen.end();
        if (it != q->seen.end() && it->second != UINT64_MAX) {
            const int64_t l0 = ctx->launches;
            CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            const int e = tick();
            cudaGraph_t g = nullptr;
            const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &g);
            cudaGraphExec_t exec = nullptr;
            cudaError_t ei = ec;
            if (!e && ec == cudaSuccess) ei = cudaGraphInstantiate(&exec, g, 0);
            if (g) cudaGraphDestroy(g);
            if (e) return e;  // an argument error: the eager tick would fail alike
            if (ei == cudaSuccess) {
                q->seen.erase(it);
                q->graphs[gk] = {exec, span_bytes, out_bytes, ctx->launches - l0,
                                 (uint64_t)q->n};
                tickq_evict(q);
                CK(cudaGraphLaunch(exec, ctx->stream));
                return FVV_OK;
            }
            // not capturable (e.g. a first-use allocation): this key stays eager
            cudaGetLastError();
            ctx->launches = l0;
            it->second = UINT64_MAX;
        } else if (it == q->seen.end() && key != 0 && q->max_graphs > 0) {
            q->seen[gk] = (uint64_t)q->n;
            tickq_evict(q);
        }
        return tick();
    };
    if ((rc = run())) {
        tickq_restore(q);
        return rc;
    }
    return tickq_end(q, host_out, out_bytes, slot, ticket);
}

int fvv_tickq_replay(fvv_tickq *q, const void *host_span, int64_t span_bytes, void *host_out,
                     uint64_t key, int64_t *ticket) {
    if (!q || !ticket) return FVV_EINVAL;
    fvv_ctx *ctx = q->ctx;
    *ticket = -1;
    if (key == 0) return FVV_OK;
    const int slot = (int)(q->n % q->depth);
    auto it = q->graphs.find(std::make_pair(key, slot));
    if (it == q->graphs.end()) return FVV_OK;  // not captured (yet): submit the tick
    int rc = enter(ctx);
    if (rc) return rc;
    if (!host_span || !host_out || span_bytes != it->second.span_bytes)
        return fail(ctx, FVV_EINVAL, "tickq_replay: span of %lld bytes, the tick was captured "
                    "with %lld", (long long)span_bytes, (long long)it->second.span_bytes);
    if ((rc = tickq_begin(q, host_span, span_bytes, slot))) return rc;
    const cudaError_t el = cudaGraphLaunch(it->second.exec, ctx->stream);
    if (el != cudaSuccess) {
        tickq_restore(q);
        return fail(ctx, FVV_ECUDA, "tick graph launch: %s", cudaGetErrorString(el));
    }
    ctx->launches += it->second.launches;
    it->second.last_use = (uint64_t)q->n;
    ++q->replays;
    return tickq_end(q, host_out, it->second.out_bytes, slot, ticket);
}

int fvv_tickq_wait(fvv_tickq *q, int64_t ticket) {
    if (!q) return FVV_EINVAL;
    fvv_ctx *ctx = q->ctx;
    if (ticket < 0 || ticket >= q->n) return fail(ctx, FVV_EINVAL, "tickq_wait: no tick %lld", (long long)ticket);
    // the slot's latest download is this tick's or a later one (the D2H
    // stream runs in order)
    CK(cudaEventSynchronize(q->down[ticket % q->depth]));
    return FVV_OK;
}

int fvv_tickq_fence(fvv_tickq *q, void *cuda_stream) {
    if (!q) return FVV_EINVAL;
    fvv_ctx *ctx = q->ctx;
    int rc = enter(ctx);
    if (rc) return rc;
    for (int i = 0; i < q->depth; ++i)
        if (q->used[i]) CK(cudaStreamWaitEvent((cudaStream_t)cuda_stream, q->down[i], 0));
    return FVV_OK;
}

int fvv_tickq_stats(fvv_tickq *q, int64_t *ticks, int64_t *h2d_bytes, int64_t *d2h_bytes,
                    int64_t *replays, int64_t *graphs) {
    if (!q) return FVV_EINVAL;
    if (ticks) *ticks = q->n;
    if (h2d_bytes) *h2d_bytes = q->h2d_bytes;
    if (d2h_bytes) *d2h_bytes = q->d2h_bytes;
    if (replays) *replays = q->replays;
    if (graphs) *graphs = (int64_t)q->graphs.size();
    return FVV_OK;
}

}  // extern "C"
