// Capture-server side of the MVD stream: the
// per-frame producer chain of CaptureServer.capture (pipeline.py:381-397) as
// sm_100a kernels, bit-exact with the reference's float64 numpy code.
//
//   k_correct_depth    depthproc.correct_depth      depthproc.py:67-84
//   k_bg_train         depthproc.bg_train           depthproc.py:121-136
//   k_classify_fg      depthproc.classify_fg        depthproc.py:139-149
//   k_remove_bg        depthproc.remove_bg_depth    depthproc.py:152-164
//   k_quantize12       depthcodec.quantize12        depthcodec.py:83-110
//   k_pack_yuv420      depthcodec.pack_yuv420       depthcodec.py:141-193
//   k_capture_encode   all of the above fused, one thread per 2x2 block:
//                      depth + colour (+ BG model) in, YUV420 planes out

#include "fvv_capture.cuh"

namespace fvv {

__device__ __forceinline__ void correct_px(double alpha, double beta, float &d, uint8_t &v) {
    // z_post = (alpha * z + beta) * z on Valid pixels; <= 0 -> Invalid; non-Valid -> 0
    if (v == FVV_VALID) {
        const double z = (double)d;
        const double zp = dmul(dadd(dmul(alpha, z), beta), z);
        if (zp <= 0.0) v = FVV_INVALID;
        d = (v == FVV_VALID) ? __double2float_rn(zp) : 0.0f;
    } else {
        d = 0.0f;
    }
}

// sum over channels of (x - mu)^2 / var (sequential, like np.sum over a
// length-3 axis) > tau^2
__device__ __forceinline__ bool fg_px(const uint8_t *rgb, const double *mean, const double *var,
                                      double tau2) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double dlt = dsub((double)rgb[c], mean[c]);
        const double t = ddiv(dmul(dlt, dlt), var[c]);
        s = c == 0 ? t : dadd(s, t);
    }
    return s > tau2;
}

// quantize12: code 0 Background, 1 Invalid / out of the guard band, else
// floor(4093 * frac + 2 + 0.5) clipped to [2, 4095]
__device__ __forceinline__ uint32_t quant_px(const QuantParams &q, float d, uint8_t v) {
    if (v == FVV_BACKGROUND) return 0u;
    if (v != FVV_VALID) return 1u;
    const double z = (double)d;
    if (!(z >= q.lo && z <= q.hi)) return 1u;
    const double zc = fmin(fmax(z, q.zn), q.zf);
    const double frac = ddiv(dsub(ddiv(1.0, zc), q.inv_zf), q.inv_span);
    double code = floor(dadd(dadd(dmul(4093.0, frac), 2.0), 0.5));
    code = fmin(fmax(code, 2.0), 4095.0);
    return (uint32_t)code;
}

__device__ __forceinline__ uint32_t fold_lsb(uint32_t code) {
    const uint32_t msb = code >> 8, lsb = code & 0xFFu;
    return (msb & 1u) ? 255u - lsb : lsb;
}

// nibble interleave a3 b3 a2 b2 a1 b1 a0 b0 (a3 at bit 7), depthcodec.py:141-151
__device__ __forceinline__ uint32_t interleave(uint32_t a, uint32_t b) {
    uint32_t o = 0;
#pragma unroll
    for (int bit = 0; bit < 4; ++bit) {
        o |= ((a >> bit) & 1u) << (2 * bit + 1);
        o |= ((b >> bit) & 1u) << (2 * bit);
    }
    return o;
}

__global__ void k_correct_depth(const float *d, const uint8_t *v, size_t n, double alpha,
                                double beta, float *d_out, uint8_t *v_out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        float z = d[i];
        uint8_t val = v[i];
        correct_px(alpha, beta, z, val);
        d_out[i] = z;
        v_out[i] = val;
    }
}

__global__ void k_bg_train(const uint8_t *rgb, size_t n, double *mean, double *var, int first,
                           double rho, double var_floor) {
    const double omr = 1.0 - rho;  // Python float (1.0 - rho), depthproc.py:131
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * 3;
         i += (size_t)gridDim.x * blockDim.x) {
        const double x = (double)rgb[i];
        if (first) {
            mean[i] = x;
            var[i] = var_floor;
        } else {
            const double m = dadd(dmul(omr, mean[i]), dmul(rho, x));
            const double dl = dsub(x, m);
            mean[i] = m;
            var[i] = fmax(dadd(dmul(omr, var[i]), dmul(rho, dmul(dl, dl))), var_floor);
        }
    }
}

__global__ void k_classify_fg(const uint8_t *rgb, const double *mean, const double *var, size_t n,
                              double tau2, uint8_t *mask) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        mask[i] = fg_px(rgb + 3 * i, mean + 3 * i, var + 3 * i, tau2) ? 1 : 0;
}

__global__ void k_remove_bg(const float *d, const uint8_t *v, const uint8_t *fg, size_t n,
                            float *d_out, uint8_t *v_out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        const bool bg = fg[i] == 0;
        v_out[i] = bg ? (uint8_t)FVV_BACKGROUND : v[i];
        d_out[i] = bg ? 0.0f : d[i];
    }
}

__global__ void k_quantize12(const float *d, const uint8_t *v, size_t n, QuantParams q,
                             uint16_t *codes) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        codes[i] = (uint16_t)quant_px(q, d[i], v[i]);
}

// one thread per 2x2 block
__global__ void k_pack_yuv420(const uint16_t *codes, int W, int H, uint8_t *y, uint8_t *u,
                              uint8_t *vv) {
    const int bx = blockIdx.x * blockDim.x + threadIdx.x, by = blockIdx.y;
    if (bx >= W / 2 || by >= H / 2) return;
    const size_t r0 = (size_t)(2 * by) * W + 2 * bx, r1 = r0 + W;
    const uint32_t c00 = codes[r0], c01 = codes[r0 + 1], c10 = codes[r1], c11 = codes[r1 + 1];
    y[r0] = (uint8_t)fold_lsb(c00);
    y[r0 + 1] = (uint8_t)fold_lsb(c01);
    y[r1] = (uint8_t)fold_lsb(c10);
    y[r1 + 1] = (uint8_t)fold_lsb(c11);
    const size_t ci = (size_t)by * (W / 2) + bx;
    u[ci] = (uint8_t)interleave(c00 >> 8, c01 >> 8);
    vv[ci] = (uint8_t)interleave(c10 >> 8, c11 >> 8);
}

// CaptureServer.capture's per-frame chain (pipeline.py:384-397) fused:
// correct_depth -> classify_fg -> remove_bg_depth -> quantize12 -> pack_yuv420
__global__ void k_capture_encode(const __grid_constant__ CaptureParams p) {
    const int bx = blockIdx.x * blockDim.x + threadIdx.x, by = blockIdx.y;
    const int W = p.W;
    if (bx >= W / 2 || by >= p.H / 2) return;
    uint32_t code[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const size_t i = (size_t)(2 * by + (q >> 1)) * W + 2 * bx + (q & 1);
        float d = p.depth[i];
        uint8_t v = p.validity[i];
        if (p.correct) correct_px(p.alpha, p.beta, d, v);
        if (p.bg_mean && !fg_px(p.rgb + 3 * i, p.bg_mean + 3 * i, p.bg_var + 3 * i, p.tau2)) {
            v = FVV_BACKGROUND;
            d = 0.0f;
        }
        code[q] = quant_px(p.quant, d, v);
        p.y[i] = (uint8_t)fold_lsb(code[q]);
        if (p.codes_out) p.codes_out[i] = (uint16_t)code[q];
    }
    const size_t ci = (size_t)by * (W / 2) + bx;
    p.u[ci] = (uint8_t)interleave(code[0] >> 8, code[1] >> 8);
    p.v[ci] = (uint8_t)interleave(code[2] >> 8, code[3] >> 8);
}

static unsigned grid1(size_t n) {
    const size_t b = (n + 255) / 256;
    return (unsigned)(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

cudaError_t launch_correct_depth(const float *d, const uint8_t *v, size_t n, double alpha,
                                 double beta, float *d_out, uint8_t *v_out, cudaStream_t s) {
    k_correct_depth<<<grid1(n), 256, 0, s>>>(d, v, n, alpha, beta, d_out, v_out);
    return cudaGetLastError();
}

cudaError_t launch_bg_train(const uint8_t *rgb, size_t n, double *mean, double *var, int first,
                            double rho, double var_floor, cudaStream_t s) {
    k_bg_train<<<grid1(3 * n), 256, 0, s>>>(rgb, n, mean, var, first, rho, var_floor);
    return cudaGetLastError();
}

cudaError_t launch_classify_fg(const uint8_t *rgb, const double *mean, const double *var, size_t n,
                               double tau2, uint8_t *mask, cudaStream_t s) {
    k_classify_fg<<<grid1(n), 256, 0, s>>>(rgb, mean, var, n, tau2, mask);
    return cudaGetLastError();
}

cudaError_t launch_remove_bg(const float *d, const uint8_t *v, const uint8_t *fg, size_t n,
                             float *d_out, uint8_t *v_out, cudaStream_t s) {
    k_remove_bg<<<grid1(n), 256, 0, s>>>(d, v, fg, n, d_out, v_out);
    return cudaGetLastError();
}

cudaError_t launch_quantize12(const float *d, const uint8_t *v, size_t n, const QuantParams &q,
                              uint16_t *codes, cudaStream_t s) {
    k_quantize12<<<grid1(n), 256, 0, s>>>(d, v, n, q, codes);
    return cudaGetLastError();
}

cudaError_t launch_pack_yuv420(const uint16_t *codes, int W, int H, uint8_t *y, uint8_t *u,
                               uint8_t *v, cudaStream_t s) {
    dim3 grid((W / 2 + 127) / 128, H / 2);
    k_pack_yuv420<<<grid, 128, 0, s>>>(codes, W, H, y, u, v);
    return cudaGetLastError();
}

cudaError_t launch_capture_encode(const CaptureParams &p, cudaStream_t s) {
    dim3 grid((p.W / 2 + 127) / 128, p.H / 2);
    k_capture_encode<<<grid, 128, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace fvv
