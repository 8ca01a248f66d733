/*
 * fvv_b200.h — C ABI of the B200-native edge-server view-synthesis library
 * (libfvvb200.so, sm_100a).
 *
 * This is the drop-in boundary for the reference's synthesis path. The
 * reference (/root/reference/pkg/src/fvv) is pure Python/numpy and has no
 * FFI of its own; each entry point below replaces one reference function and
 * is bound from Python with ctypes (paper_2007_00558_b200/_native.py). The
 * reference function each one replaces is cited next to it.
 *
 * Conventions
 *  - Image buffers are caller-owned DEVICE pointers, tightly packed, row-major
 *    (pitch = width elements; RGB pitch = 3*width bytes).
 *  - Every call is asynchronous on the context's stream (fvv_ctx_set_stream);
 *    fvv_sync() waits for it.
 *  - Status codes: FVV_OK, FVV_EINVAL (-> Python ValueError, mirroring the
 *    reference's ValueError cases), FVV_ECUDA (-> RuntimeError). The message
 *    is available from fvv_last_error(ctx). The library never aborts.
 *  - Contexts are independent; a context is not thread-safe, distinct
 *    contexts may be used from distinct threads.
 */
#ifndef FVV_B200_H
#define FVV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FVV_OK 0
#define FVV_EINVAL 1
#define FVV_ECUDA 2

#define FVV_VALID 0      /* core.Validity, core.py:28-33 */
#define FVV_INVALID 1
#define FVV_BACKGROUND 2

#define FVV_MAX_REFS 16  /* transport.CameraSetCommand bitmask, transport.py:241-263 */
#define FVV_MAX_SLOTS 64

typedef struct fvv_ctx fvv_ctx;

/* core.CameraCalibration (core.py:36-86): intrinsics + world->camera pose. */
typedef struct fvv_camera {
    int32_t id, width, height, reserved;
    double fx, fy, cx, cy;
    double R[9]; /* row-major world->camera rotation (core.py:62) */
    double C[3]; /* camera centre in world metres (core.py:63) */
} fvv_camera;

/* synthesis.SynthesisConfig (synthesis.py:36-49). reference_count is a
 * host-side selection parameter and is not needed by the kernels. */
typedef struct fvv_synth_cfg {
    int32_t splat_radius;      /* synthesis.py:39, 0..3 */
    int32_t crack_fill_window; /* synthesis.py:40, 1..5 */
    double mixing_epsilon;     /* synthesis.py:41 */
    double depth_band_rel;     /* synthesis.py:42 */
    uint8_t hole_color[3];     /* synthesis.py:43 */
    /* Extensions outside the reference. All 0 in
     * parity mode, which is what the reference computes. */
    uint8_t angular_weight;    /* 1: blend weight 1/(dist+eps) is multiplied per pixel
                                  by 1/(theta + angular_epsilon), theta the angle at
                                  the surface point between the reference and the
                                  virtual camera rays */
    uint8_t inpaint;           /* 1: K4 fills each hole from the nearest non-hole
                                  pixels left/right/up/down, background side
                                  only; provenance 3 marks inpainted pixels */
    uint8_t reserved[3];
    double angular_epsilon;    /* rad, > 0 (default 0.0175 = 1 degree) */
    int32_t inpaint_radius;    /* max distance to a candidate, pixels, 1..4096 (default 64) */
    int32_t reserved2;
} fvv_synth_cfg;

/* synthesis.CameraStreamInputs (synthesis.py:321-328), device pointers. */
typedef struct fvv_ref_frame {
    fvv_camera cam;
    const uint8_t *rgb;           /* H*W*3 live colour */
    const float *live_depth;      /* H*W metres; FG Valid, BG Background, holes Invalid */
    const uint8_t *live_validity; /* H*W Validity codes */
    const float *bg_depth;        /* H*W static background model */
    const uint8_t *bg_validity;   /* H*W */
    double weight;                /* 1/(camera_distance + eps) (synthesis.py:249,257);
                                     <= 0 -> computed on device */
} fvv_ref_frame;

/* Optional intermediate rasters (synthesis.DebugBundle, synthesis.py:365-397)
 * plus the winner-index/stage maps the reference never materialises.
 * Contribution k in [0, 2*n_refs): FG contributions in reference order, then
 * BG contributions. Any pointer may be NULL. */
typedef struct fvv_debug {
    double *contrib_color;   /* [2R][H][W][3] */
    double *contrib_depth;   /* [2R][H][W] (0 where not valid) */
    uint8_t *contrib_valid;  /* [2R][H][W] */
    int32_t *contrib_winner; /* [2R][H][W] source pixel index, -1 none/crack-filled */
    uint8_t *contrib_stage;  /* [2R][H][W] 0 none, 1 centre, 2 splat, 3 crack median */
    double *merged_color;    /* [2][H][W][3] FG then BG (synthesis.MergedLayer) */
    double *merged_depth;    /* [2][H][W] */
    uint8_t *merged_valid;   /* [2][H][W] */
} fvv_debug;

/* ---- context ------------------------------------------------------------ */
int fvv_ctx_create(int32_t device, fvv_ctx **out);
int fvv_ctx_destroy(fvv_ctx *ctx);
int fvv_ctx_set_stream(fvv_ctx *ctx, void *cuda_stream); /* NULL = legacy default */
int fvv_sync(fvv_ctx *ctx);
const char *fvv_last_error(const fvv_ctx *ctx);
const char *fvv_version(void);
int64_t fvv_launch_count(const fvv_ctx *ctx); /* kernels launched by this context */
/* 1: the canvases' generation tag lives in device memory and every view
 * advances it with a kernel (k_gen_fill, which also does the periodic canvas
 * fill), so the launch sequence of a view is identical from call to call and
 * can be captured once in a CUDA graph and replayed (cudaStreamBeginCapture on
 * the context's stream around fvv_slots_ingest_mm + fvv_render_views; the
 * first call for a new view size must run outside capture, it allocates).
 * 0 (default): the host keeps the tag and passes it as a kernel argument. */
int fvv_ctx_device_generation(fvv_ctx *ctx, int32_t enable);

/* Per-kernel device timing: when enabled, every launch is bracketed by CUDA
 * events on the context's stream (the stream the kernel runs on).
 * kernel ids: 0 preprocess (K0 decode/ingest + K1 hole fill), 1 forward warp (K2),
 * 2 resolve (K3), 3 canvas fill, 4 other. fvv_profile_read synchronises. */
#define FVV_K_PREPROCESS 0
#define FVV_K_FORWARD_WARP 1
#define FVV_K_RESOLVE 2
#define FVV_K_FILL 3
#define FVV_K_OTHER 4
int fvv_profile_enable(fvv_ctx *ctx, int32_t enable); /* also resets */
int fvv_profile_read(fvv_ctx *ctx, int32_t kernel_id, double *total_ms, int64_t *launches);
/* Counting pass (not for timing: the counters add work): with 1, K2 counts
 * the 64-bit z-buffer atomicMin operations it issues (counters reset);
 * fvv_profile_atomics returns the count so far (synchronises). */
int fvv_count_atomics(fvv_ctx *ctx, int32_t enable);
int fvv_profile_atomics(fvv_ctx *ctx, int64_t *atomics);

/* Numerics self-test of the shared-reciprocal division and K2's filtered
 * rint(f*x/z + c) against the correctly rounded __ddiv_rn path, on n seeded
 * samples of operand class `mode` (0 bilinear, 1 projection, 2 mix, 3 wide
 * log-uniform, 4 near-half projections, 5 all u16 mm -> m quotients).
 * Adds mismatches to *mismatches_dev. */
int fvv_selftest_division(fvv_ctx *ctx, int64_t n, uint64_t seed, int32_t mode,
                          uint64_t *mismatches_dev);

/* ---- K0: depth decode ----------------------------------------------------- */
/* core.depth_from_millimeters (core.py:260-269): f32 = (f32)mm / 1000.0f,
 * Valid & mm==0 -> Invalid, non-Valid depth = 0. validity_in may be NULL
 * (= all Valid). */
int fvv_decode_mm(fvv_ctx *ctx, const uint16_t *mm, const uint8_t *validity_in,
                  int32_t width, int32_t height, float *depth_out, uint8_t *validity_out);

/* depthcodec.unpack_yuv420 (depthcodec.py:213-222) + dequantize12
 * (depthcodec.py:113-138). y: H*W, u/v: (H/2)*(W/2). codes_out may be NULL. */
int fvv_decode_yuv420_12(fvv_ctx *ctx, const uint8_t *y, const uint8_t *u, const uint8_t *v,
                         int32_t width, int32_t height, double z_near, double z_far,
                         float *depth_out, uint8_t *validity_out, uint16_t *codes_out);

/* depthcodec.dequantize12 (depthcodec.py:113-138) from 12-bit codes. */
int fvv_dequantize12(fvv_ctx *ctx, const uint16_t *codes, int32_t width, int32_t height,
                     double z_near, double z_far, float *depth_out, uint8_t *validity_out);

/* ---- K1: joint-bilateral hole closing -------------------------------------- */
/* depthproc.bilateral_close_holes (depthproc.py:171-224). n_holes_dev (device
 * int32, may be NULL) receives the number of Invalid input pixels, so the
 * host can mirror the reference's "same object when nothing to fill". */
int fvv_bilateral_close_holes(fvv_ctx *ctx, const float *depth, const uint8_t *validity,
                              const uint8_t *rgb, int32_t width, int32_t height,
                              int32_t radius, double sigma_spatial, double sigma_range,
                              int32_t min_valid_neighbors, float *depth_out,
                              uint8_t *validity_out, int32_t *n_holes_dev);

/* K1's range factor np.exp(-color_d2 / (2 sigma_range^2)) (depthproc.py:
 * 200, 211-212) has an exact integer argument color_d2 in [0, 3*255^2], so
 * K1 reads it from a resident table of 3*255^2+1 doubles. This call installs
 * the caller's table for sigma_range (the Python host passes the np.exp values
 * the reference computes, which differ from libm's in the last bit on ~5 % of
 * entries); without it the library builds the table with libm exp. */
int fvv_set_range_weights(fvv_ctx *ctx, double sigma_range, const double *table, int32_t n);

/* ---- K2+K3: one synthesized view (synthesis.synthesize_view, synthesis.py:331-362) */
int fvv_synthesize_view(fvv_ctx *ctx, const fvv_camera *virt, const fvv_ref_frame *refs,
                        int32_t n_refs, const fvv_synth_cfg *cfg, uint8_t *rgb_out,
                        uint8_t *provenance_out, const fvv_debug *dbg);

/* synthesis.warp_layer (synthesis.py:162-258): one contribution. color_valid
 * may be NULL (= depth validity == Valid). Outputs may be NULL except valid. */
int fvv_warp_layer(fvv_ctx *ctx, const fvv_camera *src, const fvv_camera *dst,
                   const uint8_t *rgb, const float *depth, const uint8_t *validity,
                   const uint8_t *color_valid, int32_t layer_fg, const fvv_synth_cfg *cfg,
                   double *color_out, double *depth_out, uint8_t *valid_out,
                   int32_t *winner_out, uint8_t *stage_out);

/* synthesis.mix_layer (synthesis.py:261-292) over n host arrays of device
 * pointers (colour H*W*3 f64, depth H*W f64, valid H*W u8). */
int fvv_mix_layer(fvv_ctx *ctx, int32_t n, const double *const *colors,
                  const double *const *depths, const uint8_t *const *valids,
                  const double *weights, int32_t width, int32_t height,
                  double depth_band_rel, double *color_out, double *depth_out,
                  uint8_t *valid_out);

/* synthesis.composite (synthesis.py:295-318). provenance_out may be NULL. */
int fvv_composite(fvv_ctx *ctx, const double *fg_color, const uint8_t *fg_valid,
                  const double *bg_color, const uint8_t *bg_valid, int32_t width,
                  int32_t height, const uint8_t hole_color[3], uint8_t *rgb_out,
                  uint8_t *provenance_out);

/* ---- capture-server chain ------------------------
 * The producer side of the MVD stream, CaptureServer.capture
 * (pipeline.py:381-397). All rasters device pointers; mean/var are the
 * GaussianBgModel's (H,W,3) float64 arrays (depthproc.py:91-118). */
/* depthproc.correct_depth (depthproc.py:67-84) */
int fvv_correct_depth(fvv_ctx *ctx, const float *depth, const uint8_t *validity, int32_t width,
                      int32_t height, double alpha, double beta, float *depth_out,
                      uint8_t *validity_out);
/* depthproc.bg_train (depthproc.py:121-136); first != 0 on the model's first frame */
int fvv_bg_train(fvv_ctx *ctx, const uint8_t *rgb, int32_t width, int32_t height, double *mean,
                 double *var, int32_t first, double learning_rate, double var_floor);
/* depthproc.classify_fg (depthproc.py:139-149): mask 1 = FG */
int fvv_classify_fg(fvv_ctx *ctx, const uint8_t *rgb, const double *mean, const double *var,
                    int32_t width, int32_t height, double threshold, uint8_t *fg_mask_out);
/* depthproc.remove_bg_depth (depthproc.py:152-164) */
int fvv_remove_bg_depth(fvv_ctx *ctx, const float *depth, const uint8_t *validity,
                        const uint8_t *fg_mask, int32_t width, int32_t height, float *depth_out,
                        uint8_t *validity_out);
/* depthcodec.quantize12 (depthcodec.py:83-110) */
int fvv_quantize12(fvv_ctx *ctx, const float *depth, const uint8_t *validity, int32_t width,
                   int32_t height, double z_near, double z_far, uint16_t *codes_out);
/* depthcodec.pack_yuv420 (depthcodec.py:180-193) */
int fvv_pack_yuv420(fvv_ctx *ctx, const uint16_t *codes, int32_t width, int32_t height,
                    uint8_t *y_out, uint8_t *u_out, uint8_t *v_out);
/* correct -> classify -> remove BG -> quantize12 -> pack_yuv420 in one pass.
 * do_correct = 0 skips the correction; bg_mean = NULL skips BG removal.
 * codes_out may be NULL. */
int fvv_capture_encode(fvv_ctx *ctx, const float *depth, const uint8_t *validity,
                       const uint8_t *rgb, int32_t width, int32_t height, int32_t do_correct,
                       double alpha, double beta, const double *bg_mean, const double *bg_var,
                       double threshold, double z_near, double z_far, uint8_t *y_out,
                       uint8_t *u_out, uint8_t *v_out, uint16_t *codes_out);

/* ---- MED + Golomb-Rice lossless plane codec ----------
 * The Rice stage of depthcodec's CODEC_PRED_RICE (depthcodec.py:281-409):
 * LOCO-I median prediction, zig-zag, one Rice parameter per plane, MSB-first
 * bits. The plane header (">BBIII") and the optional zlib stage around the
 * stream stay with the caller, as the reference's struct/zlib calls. Both
 * calls are synchronous. */
/* bytes a stream buffer must hold for a width x height plane */
int64_t fvv_rice_stream_bound(int32_t width, int32_t height);
/* _compress_plane's MED + Rice part (depthcodec.py:376-383): k_out = the
 * cheapest k of 0..14 (ties -> smaller k), nbits_out = stream length in bits;
 * stream_out (device) receives (nbits+7)/8 bytes. */
int fvv_rice_encode_plane(fvv_ctx *ctx, const uint8_t *plane, int32_t width, int32_t height,
                          uint8_t *stream_out, int32_t *k_out, int64_t *nbits_out);
/* _decompress_plane's Rice + MED part (depthcodec.py:386-409): decodes
 * n_symbols (must be width*height) symbols of parameter k from the device
 * stream, rebuilds the plane and returns its adler32 (the caller compares it
 * with the header's). FVV_EINVAL "rice stream truncated" when the stream runs
 * out early (the reference's DecodeError). */
int fvv_rice_decode_plane(fvv_ctx *ctx, const uint8_t *stream, int64_t nbytes, int32_t k,
                          int64_t n_symbols, int32_t width, int32_t height, uint8_t *plane_out,
                          uint32_t *adler_out);
/* The same for n planes at once (up to 48: e.g. Y, U, V of every reference
 * camera of a render tick): the Rice segmentation of all streams runs in the
 * same kernels and the planes' MED recurrences run concurrently, one CTA
 * each. Host arrays of n entries; status_out[i] = 1 when stream i runs out
 * early (adlers_out[i] then 0). */
int fvv_rice_decode_planes(fvv_ctx *ctx, int32_t n, const uint8_t *const *streams,
                           const int64_t *nbytes, const int32_t *ks, const int32_t *widths,
                           const int32_t *heights, uint8_t *const *planes_out,
                           uint32_t *adlers_out, int32_t *status_out);

/* ---- MVD disk container rasters (mvdio.py) -------------
 * The container's files (PNG colour, u16le mm depth, JSON sidecar with the
 * validity run-length code) are read and written by the host; these are the
 * per-pixel parts. Device pointers. */
/* core.depth_to_millimeters (core.py:246-255): Valid pixels ->
 * clip(rint(f32(depth * 1000)), 1, 65535), all others 0. */
int fvv_encode_mm(fvv_ctx *ctx, const float *depth, const uint8_t *validity, int32_t width,
                  int32_t height, uint16_t *mm_out);
/* mvdio.rle_decode (mvdio.py:43-52) after the host checked the runs cover
 * exactly n pixels (the reference's ValueError): run r = codes[r] over
 * [ends[r-1], ends[r]) (ends = cumulative run lengths). */
int fvv_rle_decode(fvv_ctx *ctx, const uint8_t *codes, const int64_t *ends, int64_t n_runs,
                   int64_t n, uint8_t *out);
/* mvdio.rle_encode (mvdio.py:34-40): the starts and codes of the runs of
 * flat[0..n) in order (starts_out / codes_out hold up to n entries);
 * *n_runs_out (host) after the call, which synchronises. */
int fvv_rle_encode(fvv_ctx *ctx, const uint8_t *flat, int64_t n, int64_t *starts_out,
                   uint8_t *codes_out, int64_t *n_runs_out);

/* ---- session path: resident camera slots, batched views ---------------------
 * The edge server keeps a slot per rig camera: its calibration, its static
 * BG model (uploaded once, pipeline.py:445) and its latest live frame. */
int fvv_slot_set_camera(fvv_ctx *ctx, int32_t slot, const fvv_camera *cam);
/* Forget a slot's BG model and live frame (a renderer taking over a slot
 * must supply both again before rendering from it: "missing inputs"). */
int fvv_slot_reset(fvv_ctx *ctx, int32_t slot);
int fvv_slot_set_bg(fvv_ctx *ctx, int32_t slot, const float *bg_depth,
                    const uint8_t *bg_validity);
/* Live frame from f32 depth + validity (MvdFrame / DepthFrame); hole_closing
 * runs K1 with the reference defaults first (pipeline.py:518-519). */
int fvv_slot_ingest(fvv_ctx *ctx, int32_t slot, const uint8_t *rgb, const float *depth,
                    const uint8_t *validity, int32_t hole_closing);
/* Live frame from the 16-bit mm raster: K0 decode + ingest (listing the hole
 * candidates) then K1 hole fill (pipeline.py:518-519). hole_closing=0 skips
 * K1. depth_out /
 * validity_out (may be NULL) receive the preprocessed DepthFrame. */
int fvv_slot_ingest_mm(fvv_ctx *ctx, int32_t slot, const uint8_t *rgb, const uint16_t *mm,
                       const uint8_t *validity, int32_t hole_closing, float *depth_out,
                       uint8_t *validity_out);
/* Several slots' live frames from mm rasters in ONE launch (one CTA grid
 * layer per camera): the form a render tick uses for its reference cameras.
 * rgb / mm / validity are host arrays of n device pointers. */
int fvv_slots_ingest_mm(fvv_ctx *ctx, int32_t n, const int32_t *slots,
                        const uint8_t *const *rgb, const uint16_t *const *mm,
                        const uint8_t *const *validity, int32_t hole_closing);
/* Live frame from the 12-bit YUV420 depth raster (pipeline.py:469-472). */
int fvv_slot_ingest_yuv(fvv_ctx *ctx, int32_t slot, const uint8_t *rgb, const uint8_t *y,
                        const uint8_t *u, const uint8_t *v, double z_near, double z_far,
                        int32_t hole_closing, float *depth_out, uint8_t *validity_out);
/* fvv_slot_ingest_yuv for n cameras of a render tick in one K0 launch (one
 * grid layer per camera), then one K1 over all of their fill candidates:
 * the edge server's wire-format decode (pipeline.py:466-472,518-519). */
int fvv_slots_ingest_yuv(fvv_ctx *ctx, int32_t n, const int32_t *slots,
                         const uint8_t *const *rgb, const uint8_t *const *y,
                         const uint8_t *const *u, const uint8_t *const *v, double z_near,
                         double z_far, int32_t hole_closing);
/* n_views views; view i blends slots ref_slots[i*n_refs .. +n_refs) in that
 * order with weights[i*n_refs ..] (NULL or <= 0 -> computed on device).
 * rgb_out: n_views*H*W*3; provenance_out: n_views*H*W or NULL. */
int fvv_render_views(fvv_ctx *ctx, const fvv_camera *virts, int32_t n_views,
                     const int32_t *ref_slots, const double *weights, int32_t n_refs,
                     const fvv_synth_cfg *cfg, uint8_t *rgb_out, uint8_t *provenance_out);

/* ---- render-tick queue (the e2e edge-server loop) ------------------------
 * pipeline.py:514-547 (EdgeServer.render_tick) fed from host memory, with its
 * per-tick stream/event work native: each tick's rasters arrive in ONE
 * pinned host span (a receive buffer); the queue copies it into an HBM
 * staging slot on its H2D stream, runs the tick's ingest (K0 + K1) and
 * render (K2 + K3) on the context's stream and copies the views into the
 * caller's pinned host buffer on its D2H stream (pipeline.py:762-763
 * on_display), `depth` ticks in flight: tick t reuses the slot of tick
 * t - depth once that tick's compute and download are done. A tick with a
 * non-zero key is captured as a CUDA graph on the second occurrence of
 * (key, slot) and replayed by fvv_tickq_replay (at most max_graphs kept,
 * least recently used dropped; 0 = never capture). Keys are the caller's
 * identity of a tick: same cameras, raster offsets, views and references. */
typedef struct fvv_tickq fvv_tickq;
int fvv_tickq_create(fvv_ctx *ctx, int32_t depth, int64_t span_bytes, int64_t out_bytes,
                     int32_t max_graphs, fvv_tickq **out);
int fvv_tickq_destroy(fvv_tickq *q);
/* kind 0: offs[4i..4i+3] = byte offsets of camera i's rgb, mm (uint16),
 * validity (-1: none), unused; kind 1: rgb, y, u, v (12-bit YUV420 codes,
 * z_near/z_far its depth range). Offsets 16-byte aligned. Views as
 * fvv_render_views; host_out receives n_views*H*W*3 bytes. *ticket = the
 * tick's number (fvv_tickq_wait). */
int fvv_tickq_submit(fvv_tickq *q, const void *host_span, int64_t span_bytes, int32_t kind,
                     int32_t n_cams, const int32_t *slots, const int64_t *offs, double z_near,
                     double z_far, int32_t hole_closing, const fvv_camera *virts,
                     int32_t n_views, const int32_t *ref_slots, const double *weights,
                     int32_t n_refs, const fvv_synth_cfg *cfg, void *host_out, uint64_t key,
                     int64_t *ticket);
/* Replays the graph captured for (key, next slot): *ticket >= 0, or -1 when
 * there is none (submit the tick instead). */
int fvv_tickq_replay(fvv_tickq *q, const void *host_span, int64_t span_bytes, void *host_out,
                     uint64_t key, int64_t *ticket);
/* Blocks until tick `ticket`'s views are in its host buffer. */
int fvv_tickq_wait(fvv_tickq *q, int64_t ticket);
/* cuda_stream waits (on the device) for every download queued so far. */
int fvv_tickq_fence(fvv_tickq *q, void *cuda_stream);
int fvv_tickq_stats(fvv_tickq *q, int64_t *ticks, int64_t *h2d_bytes, int64_t *d2h_bytes,
                    int64_t *replays, int64_t *graphs);

#ifdef __cplusplus
}
#endif
#endif /* FVV_B200_H */
