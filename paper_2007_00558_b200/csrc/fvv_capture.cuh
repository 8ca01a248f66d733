// Capture-server chain kernels (fvv_capture.cu): parameter blocks and launchers.
#pragma once

#include "fvv_common.cuh"

namespace fvv {

// quantize12 constants, evaluated on the host exactly as the reference's
// Python scalars (depthcodec.py:97-105)
struct QuantParams {
    double zn, zf;        // DepthRange
    double lo, hi;        // zn * (1 - 0.01), zf * (1 + 0.01): guard band
    double inv_zf;        // 1.0 / zf
    double inv_span;      // 1.0 / zn - 1.0 / zf
};

struct CaptureParams {
    int W, H;
    const float *depth;
    const uint8_t *validity;
    const uint8_t *rgb;
    int correct;          // apply correct_depth
    double alpha, beta;
    const double *bg_mean, *bg_var;  // null -> no BG removal
    double tau2;          // threshold ** 2
    QuantParams quant;
    uint8_t *y, *u, *v;
    uint16_t *codes_out;  // optional
};

cudaError_t launch_correct_depth(const float *d, const uint8_t *v, size_t n, double alpha,
                                 double beta, float *d_out, uint8_t *v_out, cudaStream_t s);
cudaError_t launch_bg_train(const uint8_t *rgb, size_t n, double *mean, double *var, int first,
                            double rho, double var_floor, cudaStream_t s);
cudaError_t launch_classify_fg(const uint8_t *rgb, const double *mean, const double *var, size_t n,
                               double tau2, uint8_t *mask, cudaStream_t s);
cudaError_t launch_remove_bg(const float *d, const uint8_t *v, const uint8_t *fg, size_t n,
                             float *d_out, uint8_t *v_out, cudaStream_t s);
cudaError_t launch_quantize12(const float *d, const uint8_t *v, size_t n, const QuantParams &q,
                              uint16_t *codes, cudaStream_t s);
cudaError_t launch_pack_yuv420(const uint16_t *codes, int W, int H, uint8_t *y, uint8_t *u,
                               uint8_t *v, cudaStream_t s);
cudaError_t launch_capture_encode(const CaptureParams &p, cudaStream_t s);

}  // namespace fvv
