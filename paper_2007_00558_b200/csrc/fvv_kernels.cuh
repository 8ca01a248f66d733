// Kernel parameter blocks and host launchers (implemented in fvv_kernels.cu).
#pragma once

#include <cuda.h>  // CUtensorMap

#include "fvv_common.cuh"

namespace fvv {

// Texel flags (byte 3 of the packed RGBA texel).
constexpr uint32_t kFlagLiveValid = 1u;       // live validity == VALID  -> FG colour source
constexpr uint32_t kFlagLiveBackground = 2u;  // live validity == BACKGROUND -> BG colour source

// Where a per-camera live depth comes from.
enum DepthSource : int { kSrcF32 = 0, kSrcMM = 1, kSrcYUV = 2, kSrcCodes = 3 };

// Per-camera buffers of one preprocessing pass (K0 decode + K1 fill + ingest).
struct PreprocCore {
    int W, H;
    int src;                 // DepthSource
    const float *depth;      // kSrcF32
    const uint8_t *validity; // kSrcF32 / kSrcMM (may be null for MM -> all Valid)
    const uint16_t *mm;      // kSrcMM
    const uint8_t *y, *u, *v;// kSrcYUV
    const uint16_t *codes;   // kSrcCodes
    double inv_span, inv_zf; // kSrcYUV/Codes: 1/zn - 1/zf, 1/zf (host-evaluated like numpy)
    const float *dq;         // kSrcYUV/Codes: dequantize12 of every code 0..4095 for
                             // (inv_span, inv_zf) (k_dq_table; same formula), or null
    const uint8_t *rgb;      // guide / colour (H*W*3)
    const uint8_t *color_valid; // optional explicit colour-valid mask -> flag bit 0
    // outputs (any may be null)
    uint32_t *texel;         // packed RGB + flags
    float *warp_depth;       // depth where Valid else 0
    float *depth_out;        // decoded / filled DepthFrame depth
    uint8_t *validity_out;   // decoded / filled DepthFrame validity
    uint16_t *codes_out;     // kSrcYUV 12-bit codes
    int *n_holes;            // count of Invalid pixels before filling
};

// joint bilateral parameters (depthproc.py:171-224); radius 0 disables
struct BilateralParams {
    int radius, min_valid;
    double sw[9][9];         // spatial weights math.exp(-(dy^2+dx^2)/(2 s^2)), host evaluated
    // range weights exp(-d2 / (2 sigma_range^2)) for every integer colour
    // distance d2 in [0, 3*255^2], evaluated on the host by the same exp the
    // reference calls (np.exp, installed by the Python host; libm otherwise)
    const double *range_w;
};

constexpr int kRangeTableLen = 3 * 255 * 255 + 1;

struct PreprocParams : PreprocCore, BilateralParams {
    uint32_t *cand;          // K1 candidate list (see PreprocBatch)
    int *ncand;
};

// several cameras in one launch (blockIdx.z = camera), same bilateral params
struct PreprocBatch {
    BilateralParams bil;
    int n;
    // K1 candidate list (camera << 26 | pixel) and its length, device memory
    // owned by the context; needed when bil.radius > 0
    uint32_t *cand;
    int *ncand;
    PreprocCore cam[FVV_MAX_REFS];
};

struct WarpContrib {
    DevCam src;
    Rel rel;                 // src camera -> virtual camera (relative_pose)
    const float *depth;      // > 0 marks a source pixel (Valid), else 0
    const double *rx, *ry;   // src ray slope tables (core.py:224-227)
    uint64_t *canvas;        // (Hd+2r) x (Wd+2r) keys
    double *zsrc;            // [Hs*Ws] exact f64 target-camera z of every source
                             // pixel that scattered a key (read back by K3 for
                             // the winners); may be null
    int b;                   // index bits
};

// Canvas layout: element (cy, cx) of a (Hd+2r) x (Wd+2r) canvas lives at
// ptr[cy * pitch + cx], where ptr = allocation + 1 + k * per and pitch is even
// and >= Wd+2r+1, so that tile rows starting at image column x0 (a multiple
// of 32) are 16-byte aligned for cp.async staging.
// FG tile occupancy: for contributions k < n_fg, K2 stores the view's
// generation into tflag[k * ntx * nty + tile] of every flag tile (kTileFlagW x
// kTileFlagH target pixels) a source lands in; K3 skips an FG contribution for
// a tile none of whose 3 x 3 neighbour tiles is flagged (its key tile,
// halo included, holds no key of this view). Null: no flags.
#ifndef FVV_RGB_CVT
#define FVV_RGB_CVT 1
#endif
#ifndef FVV_TF_STRIDE
#define FVV_TF_STRIDE 8
#endif
constexpr int kTileFlagStride = FVV_TF_STRIDE;  // bytes per flag
#ifndef FVV_TF_W
#define FVV_TF_W 32   // flag tile width (target pixels)
#endif
#ifndef FVV_TF_H
#define FVV_TF_H 8    // flag tile height
#endif
constexpr int kTileFlagW = FVV_TF_W, kTileFlagH = FVV_TF_H;
#ifndef FVV_K3_SKIP
#define FVV_K3_SKIP 1
#endif
struct TileFlags {
    uint8_t *flag;
    int n_fg, ntx, nty;      // flag tiles are kTileFlagW x kTileFlagH target pixels
};

struct WarpParams {
    DevCam dst;
    int r;
    int pitch;
    int n;
    uint64_t gen_hi;         // generation code << 57
    const int *gen_ptr;      // non-null: the generation is read from here (k_gen_fill)
    unsigned long long *n_atomics;  // non-null (profiling): += atomics issued
    TileFlags tf;
    WarpContrib c[2 * FVV_MAX_REFS];
};

struct ResolveContrib {
    DevCam src;
    Rel rel;                 // virtual camera -> src camera (relative_pose)
    const uint32_t *texel;
    const double *zsrc;      // K2's exact z per source pixel (WarpContrib::zsrc)
    const uint64_t *canvas;
    double weight;
    int b;
    uint32_t flag;           // texel flag bit that marks colour-valid source pixels
    int layer_fg;
};

struct ResolveParams {
    // TMA map of the keyed canvases: dims {pitch, Hd + 2r, n contributions}
    // over the canvas allocation, so canvas element (k, cy, cx) is tensor
    // element (cx + 1, cy, k) (the +1 allocation offset). Used by the fast
    // path (r = 1, window 3) when has_kmap.
    CUtensorMap kmap;
    int has_kmap;
    DevCam dst;
    int r, window, need;
    int pitch;
    uint64_t gen;            // generation code (0..127)
    const int *gen_ptr;      // non-null: the generation is read from here (k_gen_fill)
    TileFlags tf;            // FG tile occupancy written by K2 (fast path, non-debug)
    int n_fg, n_bg;
    double band_rel;
    double hole[3];
    uint32_t hole_rgb;       // hole[] as composite's u8 R | G << 8 | B << 16
    uint8_t *rgb_out;        // H*W*3 (may be null)
    uint8_t *prov_out;       // H*W (may be null)
    // extensions outside the reference (off in parity mode, fvv_synth_cfg):
    int ang;                 // 1: per-pixel angular factor on the blend weights
    double ang_eps;          // rad, factor = 1 / (theta + ang_eps)
    float *depth_out;        // H*W composite depth (inpainting input; may be null)
    fvv_debug dbg;
    ResolveContrib c[2 * FVV_MAX_REFS];
};

// K4 (extension): background-biased disocclusion inpainting of the holes of
// a composited view
struct InpaintParams {
    int W, H;
    int radius;              // max distance to a candidate, pixels (<= 4096)
    double bg_band;          // candidates within (1 - bg_band) * z_max count as background
    uint8_t *rgb;            // in/out: holes are filled in place
    uint8_t *prov;           // in/out: 0 hole -> 3 inpainted
    const float *depth;      // composite depth (0 at holes)
    int16_t *dist_l, *dist_r, *dist_u, *dist_d;  // scratch [H*W]: distances to the
                                        // nearest non-hole pixel (-1 none within radius)
};

struct MixParams {
    int n, W, H;
    double band_rel;
    const double *color[FVV_MAX_REFS * 2];
    const double *depth[FVV_MAX_REFS * 2];
    const uint8_t *valid[FVV_MAX_REFS * 2];
    double weight[FVV_MAX_REFS * 2];
    double *color_out, *depth_out;
    uint8_t *valid_out;
};

// host launchers; return cudaGetLastError()
cudaError_t launch_preprocess(const PreprocParams &p, cudaStream_t s);
cudaError_t launch_preprocess_batch(const PreprocBatch &b, cudaStream_t s);
cudaError_t launch_rays(const DevCam &c, double *rx, double *ry, cudaStream_t s);
cudaError_t launch_forward_warp(const WarpParams &p, long long max_src_pixels, cudaStream_t s);
cudaError_t launch_resolve(const ResolveParams &p, cudaStream_t s);
bool resolve_uses_tma();  // the fast path stages key tiles by TMA (needs ResolveParams::kmap)
cudaError_t launch_mix(const MixParams &p, cudaStream_t s);
cudaError_t launch_composite(const double *fg_c, const uint8_t *fg_v, const double *bg_c,
                             const uint8_t *bg_v, int W, int H, const double hole[3],
                             uint8_t *rgb, uint8_t *prov, cudaStream_t s);
cudaError_t launch_selftest_div(long long n, uint64_t seed, int mode, unsigned long long *mism,
                                cudaStream_t s);
cudaError_t launch_inpaint(const InpaintParams &p, cudaStream_t s);
int take_extra_launches();  // kernels beyond one issued by the last launcher call
cudaError_t launch_fill_u64(uint64_t *p, size_t n, uint64_t v, cudaStream_t s);
cudaError_t launch_dq_table(float *t, double inv_span, double inv_zf, cudaStream_t s);
cudaError_t launch_gen_fill(uint64_t *p, size_t n, int *g, cudaStream_t s);
size_t resolve_smem_bytes(int maxr);
int resolve_tile_rows();  // K3 fast-path tile height (the tile width is 32)

}  // namespace fvv
