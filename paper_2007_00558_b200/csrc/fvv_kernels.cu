// sm_100a kernels of the edge-server view-synthesis path.
//
//   K0  k_preprocess     decode (mm / YUV420-12 / f32), pack RGB+flags texels
//                        and warp depth, list the hole-fill candidates
//   K1  k_fill_g8/k_fill joint-bilateral fill of the listed candidates
//   K2  k_forward_warp   forward 3-D warp, one 64-bit atomicMin per source
//                        pixel into a padded keyed z canvas, exact z kept;
//                        FG contributions flag the target tiles they reach
//   K3  k_resolve_fast   per 32x8 target tile and per contribution (BG ones
//       (k_resolve_generic  and the flagged FG ones): splat
//        for other splat radii / crack windows)
//                        ring + FG cull + crack median in shared memory, f64
//                        backward projection, masked bilinear fetch; then the
//                        two layer mixes and the FG-over-BG composite -> RGB8
//                        + provenance
//   K4  k_inpaint_rows/cols (extension) background-biased hole fill
//
// Each kernel cites the reference lines it replaces; the numerics contract is
// in fvv_common.cuh and oracle/fvv_oracle.py.

#include <atomic>
#include <type_traits>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "fvv_kernels.cuh"

namespace fvv {

// ---------------------------------------------------------------------------
// helpers

__global__ void k_fill_u64(uint64_t *p, size_t n, uint64_t v) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) p[i] = v;
}

cudaError_t launch_fill_u64(uint64_t *p, size_t n, uint64_t v, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    k_fill_u64<<<blocks, 256, 0, s>>>(p, n, v);
    return cudaGetLastError();
}

// Device-resident canvas generation (graph-replayable views): g[0] is the
// generation K2/K3 of the coming view read, g[1] a CTA counter. The host
// rule of ensure_canvas, on the device: a previous generation <= 0 fills
// every canvas with empty keys and restarts at 126, else it counts down. All
// CTAs read g[0] before the last one to finish (counter) writes it.
__global__ void k_gen_fill(uint64_t *p, size_t n, int *g) {
    __shared__ int prev;
    if (threadIdx.x == 0) prev = *(volatile int *)g;
    __syncthreads();
    const int old = prev;
    if (old <= 0) {
        // 16-byte stores from the first 16-byte aligned key on
        const size_t head = (reinterpret_cast<uintptr_t>(p) & 15) ? 1 : 0;
        const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        const size_t stride = (size_t)gridDim.x * blockDim.x;
        if (t == 0 && head) p[0] = kEmpty;
        ulonglong2 *q = reinterpret_cast<ulonglong2 *>(p + head);
        const size_t n2 = (n - head) / 2;
        for (size_t i = t; i < n2; i += stride) q[i] = make_ulonglong2(kEmpty, kEmpty);
        if (t == 0 && ((n - head) & 1)) p[n - 1] = kEmpty;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned t = atomicAdd(reinterpret_cast<unsigned *>(g + 1), 1u);
        if (t == gridDim.x - 1) {
            *(volatile int *)g = old <= 0 ? 126 : old - 1;
            *(volatile int *)(g + 1) = 0;
            __threadfence();
        }
    }
}

cudaError_t launch_gen_fill(uint64_t *p, size_t n, int *g, cudaStream_t s) {
    // one CTA per SM: cheap when only the generation advances (126 of 127
    // views), enough 16-byte stores in flight for the periodic fill
    k_gen_fill<<<148, 512, 0, s>>>(p, n, g);
    return cudaGetLastError();
}

// ray slopes (u - cx)/fx and (v - cy)/fy, core.py:224-227
__global__ void k_rays(DevCam c, double *rx, double *ry) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < c.W) rx[i] = ddiv(dsub((double)i, c.cx), c.fx);
    if (i < c.H) ry[i] = ddiv(dsub((double)i, c.cy), c.fy);
}

cudaError_t launch_rays(const DevCam &c, double *rx, double *ry, cudaStream_t s) {
    const int n = c.W > c.H ? c.W : c.H;
    k_rays<<<(n + 255) / 256, 256, 0, s>>>(c, rx, ry);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K0 + K1 + ingest

#ifndef FVV_PRE_MINB
#define FVV_PRE_MINB 4
#endif
#ifndef FVV_PRE_ROWS
#define FVV_PRE_ROWS 2
#endif
// tile: PY rows x 128 px; a thread owns 4 px of PROWS rows
constexpr int PROWS = FVV_PRE_ROWS, PX = 128, PY = 8 * PROWS, PMAXR = 4;
constexpr int PSC = PX + 2 * PMAXR, PSR = PY + 2 * PMAXR;

// 12-bit code at (iy, ix) from the folded/interleaved YUV420 raster
// (depthcodec.py:154-177, 213-222): MSB nibble from U (even rows) or V (odd
// rows), A = odd bit positions for even columns, B = even positions for odd
// columns; LSB mirrored when the MSB is odd.
__device__ __forceinline__ uint32_t yuv_code(const PreprocCore &p, int iy, int ix) {
    const uint8_t *plane = (iy & 1) ? p.v : p.u;
    const uint32_t c = plane[(size_t)(iy >> 1) * (p.W >> 1) + (ix >> 1)];
    const uint32_t sh = (ix & 1) ? 0u : 1u;
    uint32_t msb = 0;
#pragma unroll
    for (int bit = 0; bit < 4; ++bit) msb |= ((c >> (2 * bit + sh)) & 1u) << bit;
    uint32_t lsb = p.y[(size_t)iy * p.W + ix];
    if (msb & 1u) lsb = 255u - lsb;
    return (msb << 8) | lsb;
}

// (float)mm / 1000.0f correctly rounded: product with the rounded reciprocal
// and one FMA residual correction. Equal to the IEEE quotient for every u16
// (verified exhaustively with exact rational arithmetic, and on the device by
// fvv_selftest_division mode 5).
__device__ __forceinline__ float mm_to_m(uint32_t mm) {
    const float a = (float)mm, r = 1.0f / 1000.0f;
    const float q = __fmul_rn(a, r);
    return __fmaf_rn(__fmaf_rn(-1000.0f, q, a), r, q);
}

// core.depth_from_millimeters (core.py:260-269): fp32 TRUE division by 1000
__device__ __forceinline__ void decode_mm(uint32_t mm, uint8_t &val, float &z) {
    if (val == FVV_VALID && mm == 0) val = FVV_INVALID;
    z = (val == FVV_VALID) ? mm_to_m(mm) : 0.0f;
}

// depthcodec.dequantize_codes (depthcodec.py:113-125) of one code >= 2:
// f64 frac = (c - 2) / 4093, z = 1 / (frac * inv_span + inv_zf), cast to f32
__device__ __forceinline__ float dequant_code(uint32_t c, double inv_span, double inv_zf) {
    const double frac = ddiv((double)c - 2.0, 4093.0);
    return __double2float_rn(ddiv(1.0, dadd(dmul(frac, inv_span), inv_zf)));
}

// the 4096-entry table of dequant_code for one depth range (entries 0, 1:
// the reserved codes, unused)
__global__ void k_dq_table(float *t, double inv_span, double inv_zf) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < 4096) t[c] = c < 2 ? 0.0f : dequant_code((uint32_t)c, inv_span, inv_zf);
}

cudaError_t launch_dq_table(float *t, double inv_span, double inv_zf, cudaStream_t s) {
    k_dq_table<<<16, 256, 0, s>>>(t, inv_span, inv_zf);
    return cudaGetLastError();
}

// depthcodec.dequantize12 / dequantize_codes (depthcodec.py:113-138)
__device__ __forceinline__ void decode_code(const PreprocCore &p, uint32_t c, uint8_t &val,
                                            float &z) {
    if (c < 2) {
        val = (c == 0) ? (uint8_t)FVV_BACKGROUND : (uint8_t)FVV_INVALID;
        z = 0.0f;
    } else {
        val = FVV_VALID;
        z = p.dq ? __ldg(p.dq + c) : dequant_code(c, p.inv_span, p.inv_zf);
    }
}

// codes of 4 consecutive pixels xb..xb+3 (xb % 4 == 0) of row iy from the
// Y word (4 LSB bytes) and the 2 chroma bytes of the U (even rows) or V (odd
// rows) plane that cover them (yuv_code, depthcodec.py:154-177, 213-222)
__device__ __forceinline__ void yuv_codes4(uint32_t yw, uint32_t cw, uint32_t code[4]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t c = (cw >> (8 * (q >> 1))) & 0xFFu;
        const uint32_t sh = (q & 1) ? 0u : 1u;   // even column: odd bit positions
        uint32_t msb = 0;
#pragma unroll
        for (int bit = 0; bit < 4; ++bit) msb |= ((c >> (2 * bit + sh)) & 1u) << bit;
        uint32_t lsb = (yw >> (8 * q)) & 0xFFu;
        if (msb & 1u) lsb = 255u - lsb;
        code[q] = (msb << 8) | lsb;
    }
}

// Decoded (depth, validity) of one pixel, per source format.
__device__ __forceinline__ void load_depth(const PreprocCore &p, int iy, int ix, float &z,
                                           uint8_t &val, uint32_t *code) {
    const size_t i = (size_t)iy * p.W + ix;
    if (p.src == kSrcMM) {
        val = p.validity ? p.validity[i] : (uint8_t)FVV_VALID;
        decode_mm(p.mm[i], val, z);
    } else if (p.src == kSrcYUV || p.src == kSrcCodes) {
        const uint32_t c = p.src == kSrcYUV ? yuv_code(p, iy, ix) : (uint32_t)p.codes[i];
        if (code) *code = c;
        decode_code(p, c, val, z);
    } else {
        z = p.depth[i];
        val = p.validity[i];
    }
}

__device__ __forceinline__ uchar4 load_rgb(const PreprocCore &p, size_t i) {
    if (!p.rgb) return make_uchar4(0, 0, 0, 0);
    const uint8_t *c = p.rgb + i * 3;
    return make_uchar4(c[0], c[1], c[2], 0);
}

// K0 + K1 + ingest. Each thread owns 4 consecutive pixels of PROWS rows
// (8 apart); a warp owns 128-px row segments (coalesced 8/4/12-byte loads,
// 16-byte stores), all rows' loads issued before any is used so twice the
// bytes are in flight per thread (the kernel streams from HBM and is bound by
// memory-level parallelism). The 5x5 joint-bilateral fill
// (depthproc.py:171-224) only runs when the tile holds an Invalid pixel: then
// the 2-px halo is staged in shared memory (zero-padded like
// scenegen._shift2d: outside pixels are never Valid).
__global__ void __launch_bounds__(256, FVV_PRE_MINB) k_preprocess(const __grid_constant__ PreprocBatch batch) {
    const PreprocCore &p = batch.cam[blockIdx.z];
    const BilateralParams &bl = batch.bil;
    __shared__ __align__(8) uint8_t sv[PSR * PSC + 8];
    __shared__ int s_holes, s_base;
    __shared__ int s_wcnt[8];

    const int tid = threadIdx.x, lane = tid & 31, ty = tid >> 5;
    const int x0 = blockIdx.x * PX, y0 = blockIdx.y * PY;
    if (x0 >= p.W || y0 >= p.H) return;  // batch grids cover the largest camera
    const int xb = x0 + lane * 4;
    const int R = bl.radius;
    const int SC = PX + 2 * R;
    if (tid == 0) s_holes = 0;

    // phase 1: every row's vector loads (raw words only, to keep registers
    // for more bytes in flight)
    bool vec[PROWS];
    uint2 rm[PROWS];
    uint32_t rv[PROWS], rc[PROWS][3];
    const bool vcols = xb + 3 < p.W && (p.W & 3) == 0 && p.rgb &&
                       ((p.src == kSrcMM && p.validity) || p.src == kSrcYUV);
#pragma unroll
    for (int r = 0; r < PROWS; ++r) {
        const int iy = y0 + ty + 8 * r;
        vec[r] = vcols && iy < p.H;
        if (vec[r]) {
            // 16-B aligned vector path (W % 4 == 0; torch/cudaMalloc bases are 256-B aligned)
            const size_t i0 = (size_t)iy * p.W + xb;
            if (p.src == kSrcMM) {
                rm[r] = __ldcs(reinterpret_cast<const uint2 *>(p.mm + i0));
                rv[r] = __ldcs(reinterpret_cast<const uint32_t *>(p.validity + i0));
            } else {
                // wire format: 4 Y bytes + the 2 chroma bytes under them
                const uint8_t *plane = (iy & 1) ? p.v : p.u;
                rm[r].x = __ldcs(reinterpret_cast<const uint32_t *>(p.y + i0));
                rm[r].y = __ldcs(reinterpret_cast<const uint16_t *>(
                    plane + (size_t)(iy >> 1) * (p.W >> 1) + (xb >> 1)));
                rv[r] = 0;
            }
            const uint32_t *c3 = reinterpret_cast<const uint32_t *>(p.rgb + i0 * 3);
            rc[r][0] = __ldcs(c3);
            rc[r][1] = __ldcs(c3 + 1);
            rc[r][2] = __ldcs(c3 + 2);
        }
    }
    // phase 2: decode, write the outputs (K1 later rewrites the pixels it
    // fills, so the stores need not wait for the candidate test below) and
    // keep each row's decoded validity (packed) for that test
    uint32_t vp[PROWS];
    int nh = 0;
#pragma unroll
    for (int r = 0; r < PROWS; ++r) {
        const int iy = y0 + ty + 8 * r;
        const size_t rowbase = (size_t)iy * p.W;
        if (vec[r] && !p.color_valid) {
            // the 4 pixels as packed bytes: validity word, flag word, texels
            // by byte permutes (same values as the per-pixel path below)
            float z[4];
            uint32_t v4;
            if (p.src == kSrcYUV) {
                uint32_t code[4];
                uint8_t val[4];
                yuv_codes4(rm[r].x, rm[r].y, code);
#pragma unroll
                for (int q = 0; q < 4; ++q) decode_code(p, code[q], val[q], z[q]);
                v4 = (uint32_t)val[0] | ((uint32_t)val[1] << 8) | ((uint32_t)val[2] << 16) |
                     ((uint32_t)val[3] << 24);
            } else {
                // decode_mm: Valid with mm == 0 becomes Invalid; z = mm / 1000 on Valid
                const uint32_t zero =
                    __byte_perm(__vcmpeq2(rm[r].x, 0u), __vcmpeq2(rm[r].y, 0u), 0x6420);
                const uint32_t fix = __vcmpeq4(rv[r], 0u) & zero;
                v4 = (rv[r] & ~fix) | (fix & (0x01010101u * FVV_INVALID));
                const uint32_t vm = __vcmpeq4(v4, 0u);
                const uint32_t mm4[4] = {rm[r].x & 0xFFFFu, rm[r].x >> 16, rm[r].y & 0xFFFFu,
                                         rm[r].y >> 16};
#pragma unroll
                for (int q = 0; q < 4; ++q) z[q] = ((vm >> (8 * q)) & 1u) ? mm_to_m(mm4[q]) : 0.0f;
            }
            static_assert(FVV_VALID == 0 && kFlagLiveValid == 1 && kFlagLiveBackground == 2,
                          "packed flag word");
            vp[r] = v4;
            nh += __popc(__vcmpeq4(v4, 0x01010101u * FVV_INVALID)) >> 3;
            const uint32_t fl = (__vcmpeq4(v4, 0u) & 0x01010101u) |
                                (__vcmpeq4(v4, 0x01010101u * FVV_BACKGROUND) & 0x02020202u);
            const uint32_t ca = rc[r][0], cb = rc[r][1], cc = rc[r][2];
            const size_t i0 = rowbase + xb;
            if (p.texel)
                *reinterpret_cast<uint4 *>(p.texel + i0) = make_uint4(
                    __byte_perm(ca, fl, 0x4210), __byte_perm(__byte_perm(ca, cb, 0x0543), fl, 0x5210),
                    __byte_perm(__byte_perm(cb, cc, 0x0432), fl, 0x6210), __byte_perm(cc, fl, 0x7321));
            // z is 0 wherever the pixel is not Valid, so the warp depth is z
            if (p.warp_depth) *reinterpret_cast<float4 *>(p.warp_depth + i0) = make_float4(z[0], z[1], z[2], z[3]);
            if (p.depth_out) *reinterpret_cast<float4 *>(p.depth_out + i0) = make_float4(z[0], z[1], z[2], z[3]);
            if (p.validity_out) *reinterpret_cast<uint32_t *>(p.validity_out + i0) = v4;
            continue;
        }
        float z[4];
        uint8_t val[4];
        uchar4 g[4];
        uint32_t code[4] = {0, 0, 0, 0};
        if (vec[r] && p.src == kSrcYUV) {
            yuv_codes4(rm[r].x, rm[r].y, code);
#pragma unroll
            for (int q = 0; q < 4; ++q) decode_code(p, code[q], val[q], z[q]);
        } else if (vec[r]) {
            const uint32_t mm4[4] = {rm[r].x & 0xFFFFu, rm[r].x >> 16, rm[r].y & 0xFFFFu,
                                     rm[r].y >> 16};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                val[q] = (uint8_t)(rv[r] >> (8 * q));
                decode_mm(mm4[q], val[q], z[q]);
            }
        }
        if (vec[r]) {
            const uint32_t ca = rc[r][0], cb = rc[r][1], cc = rc[r][2];
            g[0] = make_uchar4(ca & 255, (ca >> 8) & 255, (ca >> 16) & 255, 0);
            g[1] = make_uchar4(ca >> 24, cb & 255, (cb >> 8) & 255, 0);
            g[2] = make_uchar4((cb >> 16) & 255, cb >> 24, cc & 255, 0);
            g[3] = make_uchar4((cc >> 8) & 255, (cc >> 16) & 255, cc >> 24, 0);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                z[q] = 0.0f;
                val[q] = 0xFF;
                g[q] = make_uchar4(0, 0, 0, 0);
                if (iy < p.H && xb + q < p.W) {
                    load_depth(p, iy, xb + q, z[q], val[q], &code[q]);
                    g[q] = load_rgb(p, rowbase + xb + q);
                }
            }
        }
        vp[r] = (uint32_t)val[0] | ((uint32_t)val[1] << 8) | ((uint32_t)val[2] << 16) |
                ((uint32_t)val[3] << 24);
#pragma unroll
        for (int q = 0; q < 4; ++q) nh += (val[q] == FVV_INVALID);
        if (iy >= p.H) continue;
        uint32_t tex[4];
        float wd[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t flags;
            if (p.color_valid) {
                flags = (xb + q < p.W && p.color_valid[rowbase + xb + q]) ? kFlagLiveValid : 0u;
            } else {
                flags = (val[q] == FVV_VALID ? kFlagLiveValid : 0u) |
                        (val[q] == FVV_BACKGROUND ? kFlagLiveBackground : 0u);
            }
            tex[q] = (uint32_t)g[q].x | ((uint32_t)g[q].y << 8) | ((uint32_t)g[q].z << 16) |
                     (flags << 24);
            wd[q] = (val[q] == FVV_VALID) ? z[q] : 0.0f;
        }
        if (vec[r]) {
            const size_t i0 = rowbase + xb;
            if (p.texel) *reinterpret_cast<uint4 *>(p.texel + i0) = make_uint4(tex[0], tex[1], tex[2], tex[3]);
            if (p.warp_depth) *reinterpret_cast<float4 *>(p.warp_depth + i0) = make_float4(wd[0], wd[1], wd[2], wd[3]);
            if (p.depth_out) *reinterpret_cast<float4 *>(p.depth_out + i0) = make_float4(z[0], z[1], z[2], z[3]);
            if (p.validity_out) *reinterpret_cast<uint32_t *>(p.validity_out + i0) = vp[r];
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (xb + q >= p.W) break;
                const size_t i = rowbase + xb + q;
                if (p.texel) p.texel[i] = tex[q];
                if (p.warp_depth) p.warp_depth[i] = wd[q];
                if (p.depth_out) p.depth_out[i] = z[q];
                if (p.validity_out) p.validity_out[i] = val[q];
                if (p.codes_out) p.codes_out[i] = (uint16_t)code[q];
            }
        }
    }
    if (p.n_holes) {
        const int m = __reduce_add_sync(0xffffffffu, nh);
        if (lane == 0 && m) atomicAdd(&s_holes, m);
        __syncthreads();
        if (tid == 0 && s_holes) atomicAdd(p.n_holes, s_holes);
    }

    if (R > 0 && __syncthreads_or(nh)) {
        // K1 candidates: Invalid pixels with >= min_valid Valid pixels in
        // their window (depthproc.py:218). Only the validity of the tile and
        // its R-px ring is staged (zero-padded like scenegen._shift2d: outside
        // pixels are never Valid); the candidates go to a global list that
        // k_fill drains densely after this kernel (a tile holds a few dozen of
        // them, so filling them here would idle most of its lanes).
#pragma unroll
        for (int r = 0; r < PROWS; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) sv[(ty + 8 * r + R) * SC + lane * 4 + q + R] = (uint8_t)(vp[r] >> (8 * q));
        const int SR = PY + 2 * R;
        // block-uniform choice (a thread's own `vec` is false on rows / columns
        // past the image, which must not change how the halo is split up)
        const bool hvec = R == 2 && (p.W & 3) == 0 && p.src == kSrcMM && p.validity;
        const int ring = hvec ? 0 : SR * SC - PY * PX;
        if (hvec) {
            // halo validity with 16-byte-group loads: rows y0-2, y0-1, y0+PY,
            // y0+PY+1 as 34 aligned 4-px groups each (columns x0-4 .. x0+131),
            // then the 2-px side columns of the PY tile rows
            if (tid < 4 * 34) {
                const int hr = tid / 34, gq = tid - hr * 34;
                const int ry = hr < 2 ? hr : PY + hr;  // smem row
                const int qy = y0 - 2 + ry, gx = x0 - 4 + 4 * gq;
                uint32_t v4 = 0xFFFFFFFFu;
                if (qy >= 0 && qy < p.H && gx >= 0 && gx + 3 < p.W) {
                    const size_t gi = (size_t)qy * p.W + gx;
                    const uint2 m = __ldg(reinterpret_cast<const uint2 *>(p.mm + gi));
                    v4 = __ldg(reinterpret_cast<const uint32_t *>(p.validity + gi));
                    const uint32_t mm4[4] = {m.x & 0xFFFFu, m.x >> 16, m.y & 0xFFFFu, m.y >> 16};
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (((v4 >> (8 * q)) & 0xFFu) == FVV_VALID && mm4[q] == 0)
                            v4 = (v4 & ~(0xFFu << (8 * q))) | ((uint32_t)FVV_INVALID << (8 * q));
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int sx = 4 * gq - 2 + q;  // smem column of pixel gx + q
                    if (sx >= 0 && sx < SC) sv[ry * SC + sx] = (uint8_t)(v4 >> (8 * q));
                }
            } else if (tid < 4 * 34 + PY * 4) {
                const int j = tid - 4 * 34, ry = 2 + (j >> 2), c = j & 3;
                const int rx = c < 2 ? c : PX + c;  // smem columns 0,1 and PX+2, PX+3
                const int qy = y0 - 2 + ry, qx = x0 - 2 + rx;
                float zz;
                uint8_t vv = 0xFF;
                if (qy < p.H && qx >= 0 && qx < p.W) load_depth(p, qy, qx, zz, vv, nullptr);
                sv[ry * SC + rx] = vv;
            }
        }
        for (int i = tid; i < ring; i += 256) {
            int ry, rx;
            const int top = R * SC;
            if (i < top) { ry = i / SC; rx = i - ry * SC; }
            else if (i < 2 * top) { ry = PY + R + (i - top) / SC; rx = (i - top) % SC; }
            else { const int j = i - 2 * top; ry = R + j / (2 * R); rx = j % (2 * R);
                   if (rx >= R) rx += PX; }
            const int qy = y0 - R + ry, qx = x0 - R + rx;
            float zz = 0.0f;
            uint8_t vv = 0xFF;
            if (qy >= 0 && qy < p.H && qx >= 0 && qx < p.W) load_depth(p, qy, qx, zz, vv, nullptr);
            sv[ry * SC + rx] = vv;
        }
        __syncthreads();
        // no Valid pixel in the tile and its ring (sky, ray misses): no
        // candidate can reach min_valid > 0, skip the per-pixel counts
        // (R = 2: the staged rows as Valid bitmasks, bit j of sbits[y][w] =
        // smem pixel (y, 32 w + j), so a window row is one funnel shift and a
        // popcount)
        __shared__ uint32_t sbits[PSR][5];
        {
            int anyv = 0;
            if (R == 2) {
                for (int i = tid; i < SR * 5; i += 256) {
                    const int y = i / 5, w = i - 5 * y;
                    uint32_t bits = 0;
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        const int c = 32 * w + 4 * g;
                        if (c < SC) {   // Valid == 0; 4 byte flags -> 4 bits
                            const uint32_t m =
                                __vcmpeq4(*reinterpret_cast<const uint32_t *>(sv + y * SC + c), 0u) &
                                0x01010101u;
                            bits |= (((m * 0x01020408u) >> 24) & 0xFu) << (4 * g);
                        }
                    }
                    sbits[y][w] = bits;
                    anyv |= bits != 0u;
                }
            } else {
                const int nw = (SR * SC + 3) / 4;
                for (int i = tid; i < nw; i += 256) {
                    const uint32_t w = reinterpret_cast<const uint32_t *>(sv)[i];
                    anyv |= __vcmpeq4(w, 0u) != 0u;   // a Valid (0) byte
                }
            }
            if (!__syncthreads_or(anyv) && bl.min_valid > 0) return;
        }
        unsigned cm[PROWS][4];
        int wc = 0;
#pragma unroll
        for (int r = 0; r < PROWS; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                bool cand = false;
                const int x = lane * 4 + q;  // tile column; window columns x..x+2R in smem
                const int row = ty + 8 * r;  // tile row
                if (((vp[r] >> (8 * q)) & 0xFFu) == FVV_INVALID) {
                    int cnt = 0;
                    if (R == 2) {
                        // window columns x..x+4 of smem rows row..row+4
                        const int w = x >> 5, sh = x & 31;
#pragma unroll
                        for (int dy = 0; dy < 5; ++dy)
                            cnt += __popc(__funnelshift_r(sbits[row + dy][w], sbits[row + dy][w + 1], sh) &
                                          0x1Fu);
                    } else {
                        for (int dy = -R; dy <= R; ++dy)
                            for (int dx = -R; dx <= R; ++dx)
                                cnt += sv[(row + R + dy) * SC + x + R + dx] == FVV_VALID;
                    }
                    cand = cnt >= bl.min_valid;
                }
                cm[r][q] = __ballot_sync(0xffffffffu, cand);
                wc += __popc(cm[r][q]);
            }
        // one global atomic per tile (a single list counter is hit by every
        // tile with candidates): warp counts -> tile prefix -> list slots
        if (lane == 0) s_wcnt[ty] = wc;
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < 8; ++w) {
                const int c = s_wcnt[w];
                s_wcnt[w] = tot;
                tot += c;
            }
            s_base = tot ? atomicAdd(batch.ncand, tot) : 0;
        }
        __syncthreads();
        int base = s_base + s_wcnt[ty];
#pragma unroll
        for (int r = 0; r < PROWS; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if ((cm[r][q] >> lane) & 1u)
                    batch.cand[base + __popc(cm[r][q] & ((1u << lane) - 1u))] =
                        ((uint32_t)blockIdx.z << 26) |
                        (uint32_t)((size_t)(y0 + ty + 8 * r) * p.W + xb + q);
                base += __popc(cm[r][q]);
            }
    }
}



// K1 proper: the joint-bilateral fill (depthproc.py:196-222) of the
// candidates k_preprocess listed, one thread per candidate, reading the
// window straight from the (L2-resident) inputs. Taps in dy-major order with
// the centre skipped; w = exp_s(dy,dx) * exp(-|g - g_nb|^2 / (2 sr^2)) on
// Valid taps; the colour distance is an exact integer (u8 channels), so the
// range factor np.exp(-d2 * inv_2sr) is one table read. A filled pixel's
// outputs (depth, validity, texel flags, warp depth) are rewritten; k_preprocess
// already wrote it as Invalid.
__device__ __forceinline__ void fill_tap(const PreprocCore &p, int x, int y, int dy, int dx,
                                         float &z, bool &ok, uchar4 &g) {
    const int qy = y + dy, qx = x + dx;
    ok = false;
    z = 0.0f;
    g = make_uchar4(0, 0, 0, 0);
    if (qy >= 0 && qy < p.H && qx >= 0 && qx < p.W) {
        uint8_t v;
        // the colour load does not wait for the validity test (one dependent
        // load fewer per tap; a non-Valid tap's colour is never used)
        g = load_rgb(p, (size_t)qy * p.W + qx);
        load_depth(p, qy, qx, z, v, nullptr);
        ok = v == FVV_VALID;
    }
}

// Radius 2, the default: 32/LPC candidates per warp, LPC lanes per
// candidate, lane t evaluating taps t, t+LPC, ... (loads + table read +
// weight products); the products go through shared memory and the group's
// first lane adds the 24 taps in the reference's order. All groups
// accumulate in the same instructions. K1 is latency-bound (a chain of
// dependent loads per candidate): 4 lanes per candidate (8 candidates per
// warp pass, 6 independent taps per lane) halve the passes of 8 lanes.
#ifndef FVV_K1_CTAS
#define FVV_K1_CTAS 4   // CTAs per SM of the K1 grid, all resident (<= 64 registers;
                        // at 87 only 2 fit and the grid ran in two latency-bound waves)
#endif
#ifndef FVV_K1_LPC
#define FVV_K1_LPC 4
#endif
template <int LPC>
__global__ void __launch_bounds__(256, FVV_K1_CTAS) k_fill_g8(const __grid_constant__ PreprocBatch batch) {
    constexpr int G = 32 / LPC, TPL = 24 / LPC;   // candidates per warp, taps per lane
    __shared__ double2 s_w[8][G][24];   // [warp][group][tap] = (w, w * z)
    const BilateralParams &bl = batch.bil;
    const int n = *batch.ncand;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane / LPC, t = lane % LPC;
    const unsigned gmask = ((1u << LPC) - 1u) << (LPC * g);
    for (int base = (blockIdx.x * 8 + warp) * G; base < n; base += gridDim.x * 8 * G) {
        const int e = base + g;
        const bool live = e < n;
        const uint32_t ent = live ? batch.cand[e] : 0u;
        const PreprocCore &p = batch.cam[ent >> 26];
        const int i = (int)(ent & ((1u << 26) - 1));
        const int y = i / p.W, x = i - y * p.W;
        const uchar4 gc = live ? load_rgb(p, (size_t)i) : make_uchar4(0, 0, 0, 0);
        int cnt = 0;
        float zn[TPL];
        bool ok[TPL];
        uchar4 n4[TPL];
#pragma unroll
        for (int m = 0; m < TPL; ++m) {   // every tap's loads first
            const int k = t + LPC * m, kk = k < 12 ? k : k + 1;  // skip the centre
            zn[m] = 0.0f;
            ok[m] = false;
            n4[m] = make_uchar4(0, 0, 0, 0);
            if (live) fill_tap(p, x, y, kk / 5 - 2, kk % 5 - 2, zn[m], ok[m], n4[m]);
        }
#pragma unroll
        for (int m = 0; m < TPL; ++m) {
            const int k = t + LPC * m, kk = k < 12 ? k : k + 1;
            double w = 0.0;
            if (ok[m]) {
                const int e0 = gc.x - n4[m].x, e1 = gc.y - n4[m].y, e2 = gc.z - n4[m].z;
                w = dmul(bl.sw[kk / 5][kk % 5], __ldg(bl.range_w + (e0 * e0 + e1 * e1 + e2 * e2)));
            }
            s_w[warp][g][k] = make_double2(w, dmul(w, (double)zn[m]));
            cnt += __popc(__ballot_sync(0xffffffffu, ok[m]) & gmask);
        }
        __syncwarp();
        if (t == 0 && live) {
            double num = 0.0, den = 0.0;
#pragma unroll
            for (int k = 0; k < 24; ++k) {
                const double2 v = s_w[warp][g][k];
                num = dadd(num, v.y);
                den = dadd(den, v.x);
            }
            if (cnt >= bl.min_valid && den > 0.0) {
                const float z = __double2float_rn(ddiv(num, den));
                if (p.depth_out) p.depth_out[i] = z;
                if (p.validity_out) p.validity_out[i] = FVV_VALID;
                if (p.warp_depth) p.warp_depth[i] = z;
                if (p.texel && !p.color_valid)
                    reinterpret_cast<uint8_t *>(p.texel + i)[3] = (uint8_t)kFlagLiveValid;
            }
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(256) k_fill(const __grid_constant__ PreprocBatch batch) {
    // one warp per candidate: lane k evaluates tap k (its loads and table read
    // in parallel with the other taps'), then lane 0 accumulates the taps in
    // the reference's order. A non-Valid tap contributes w = 0 exactly as in
    // the reference (np.where(nb_valid, w, 0): adding +0.0 changes nothing).
    const BilateralParams &bl = batch.bil;
    const int n = *batch.ncand;
    const int R = bl.radius, D = 2 * R + 1, ntaps = D * D - 1;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int e = warp; e < n; e += nwarps) {
        const uint32_t ent = batch.cand[e];
        const PreprocCore &p = batch.cam[ent >> 26];
        const int i = (int)(ent & ((1u << 26) - 1));
        const int y = i / p.W, x = i - y * p.W;
        const uchar4 gc = load_rgb(p, (size_t)i);
        double num = 0.0, den = 0.0;
        int cnt = 0;
        for (int c0 = 0; c0 < ntaps; c0 += 32) {
            const int k = c0 + lane;
            double w = 0.0, wz = 0.0;
            bool ok = false;
            if (k < ntaps) {
                const int kk = k < ntaps / 2 ? k : k + 1;  // skip the centre
                const int dy = kk / D - R, dx = kk % D - R;
                float zn;
                uchar4 n4;
                fill_tap(p, x, y, dy, dx, zn, ok, n4);
                if (ok) {
                    const int e0 = gc.x - n4.x, e1 = gc.y - n4.y, e2 = gc.z - n4.z;
                    w = dmul(bl.sw[dy + R][dx + R],
                             __ldg(bl.range_w + (e0 * e0 + e1 * e1 + e2 * e2)));
                    wz = dmul(w, (double)zn);
                }
            }
            cnt += __popc(__ballot_sync(0xffffffffu, ok));
            const int m = ntaps - c0 < 32 ? ntaps - c0 : 32;
            for (int t = 0; t < m; ++t) {
                const double wt = __shfl_sync(0xffffffffu, w, t);
                const double wzt = __shfl_sync(0xffffffffu, wz, t);
                num = dadd(num, wzt);
                den = dadd(den, wt);
            }
        }
        if (lane != 0 || !(cnt >= bl.min_valid && den > 0.0)) continue;
        const float z = __double2float_rn(ddiv(num, den));
        if (p.depth_out) p.depth_out[i] = z;
        if (p.validity_out) p.validity_out[i] = FVV_VALID;
        if (p.warp_depth) p.warp_depth[i] = z;
        if (p.texel && !p.color_valid)
            reinterpret_cast<uint8_t *>(p.texel + i)[3] = (uint8_t)kFlagLiveValid;
    }
}

// kernels a launcher issued beyond the one LAUNCH_K counts (fvv_launch_count)
static thread_local int t_extra_launches = 0;

cudaError_t launch_preprocess_batch(const PreprocBatch &b, cudaStream_t s) {
    if (b.n <= 0) return cudaSuccess;
    int W = 0, H = 0;
    for (int i = 0; i < b.n; ++i) {
        W = b.cam[i].W > W ? b.cam[i].W : W;
        H = b.cam[i].H > H ? b.cam[i].H : H;
    }
    const bool fill = b.bil.radius > 0;
    if (fill) {
        cudaError_t e = cudaMemsetAsync(b.ncand, 0, sizeof(int), s);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((W + PX - 1) / PX, (H + PY - 1) / PY, b.n);
    k_preprocess<<<grid, 256, 0, s>>>(b);
    if (fill) {
        if (b.bil.radius == 2) k_fill_g8<FVV_K1_LPC><<<148 * FVV_K1_CTAS, 256, 0, s>>>(b);
        else k_fill<<<148 * 8, 256, 0, s>>>(b);
        ++t_extra_launches;
    }
    return cudaGetLastError();
}

int take_extra_launches() {
    const int n = t_extra_launches;
    t_extra_launches = 0;
    return n;
}

cudaError_t launch_preprocess(const PreprocParams &p, cudaStream_t s) {
    PreprocBatch b{};
    b.bil = static_cast<const BilateralParams &>(p);
    b.n = 1;
    b.cand = p.cand;
    b.ncand = p.ncand;
    b.cam[0] = static_cast<const PreprocCore &>(p);
    return launch_preprocess_batch(b, s);
}

// ---------------------------------------------------------------------------
// K2: forward warp (synthesis.py:188-205)
//
// One thread per source pixel: unproject with the f32 depth (as f64), move
// to the virtual camera, project, rint (np.round, half-even) and scatter ONE
// key into the canvas padded by r. The 9-way splat of the reference becomes
// the ring min in K3 (verified equivalent).

// rint((f*x)/z + c) — the target pixel of np.round(uv) (synthesis.py:193-194).
// The quotient is first formed with a Newton-refined reciprocal r of z
// (shared by u and v, relative error ~1e-16); only when the result lies within
// 1e-6 of a rounding boundary (k + 0.5) is the correctly rounded __ddiv_rn
// path taken, so the rounded target is always the one the exact float64
// expression gives (tests/test_gpu_numerics.py, mode 4).
__device__ __forceinline__ double proj_rint_r(double f, double x, double z, double r, double c) {
    const double num = dmul(f, x);
    const double ua = fma(num, r, c);
    // |ua - rint(ua)| is ua's exact distance to the nearest integer: more
    // than 1e-6 away from k + 0.5, the approximate quotient rounds as the
    // exact one does
    const double ri = rint(ua);
    if (fabs(ua - ri) < 0.5 - 1e-6 && fabs(ua) < 1e8) return ri;
    return rint(dadd(ddiv(num, z), c));
}

__device__ __forceinline__ double rcp_approx2(double z) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z));
    double e = fma(-z, r, 1.0);
    r = fma(r, e, r);
    e = fma(-z, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ double proj_rint(double f, double x, double z, double c) {
    if (!(z > 1e-200)) return rint(dadd(ddiv(dmul(f, x), z), c));
    return proj_rint_r(f, x, z, rcp_approx2(z), c);
}

constexpr int K2_THREADS = 128, K2_PX = 4;

// FG tile flags (TileFlags). Every CTA warping a view's FG region stores into
// the same few flags, and same-sector stores serialise in L2: flags are spread
// kTileFlagStride (8) bytes apart, one store per run of a tile per warp. At c4
// (4K, L2-thrashing canvases) packed bytes cost K2 +35%, 8-byte spacing +15%;
// a read-before-store (L1) or coarser 64/128-px flag tiles were slower still.
__device__ __forceinline__ uint8_t *tile_flag(const TileFlags &tf, int k, int t) {
    return tf.flag + ((size_t)k * tf.ntx * tf.nty + t) * kTileFlagStride;
}

__device__ __forceinline__ void mark_tile(uint8_t *f, uint8_t gen8) { *f = gen8; }

// 12 CTAs of 128 threads per SM (40 registers, a few bytes of spill): K2
// is issue-bound with its atomics' latency to hide; 46 registers (10 CTAs)
// measured 68.1 us at c1, 40 registers 66.1, 32 registers (16 CTAs) 68.2.
#ifndef FVV_K2_MINB
#define FVV_K2_MINB 12
#endif
__global__ void __launch_bounds__(K2_THREADS, FVV_K2_MINB) k_forward_warp(const __grid_constant__ WarpParams p) {
    const WarpContrib &c = p.c[blockIdx.z];
    const int Ws = c.src.W, Hs = c.src.H;
    const int sv = blockIdx.y;
    const int u0 = (blockIdx.x * K2_THREADS + threadIdx.x) * K2_PX;
    if (sv >= Hs) return;
    // lanes past the row end stay for the warp shuffle below (no pixels)
    const size_t row = (size_t)sv * Ws;
    float d[K2_PX];
    if (u0 >= Ws) {
#pragma unroll
        for (int q = 0; q < K2_PX; ++q) d[q] = 0.0f;
    } else if ((Ws & 3) == 0) {
        const float4 v = __ldcs(reinterpret_cast<const float4 *>(c.depth + row + u0));
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    } else {
#pragma unroll
        for (int q = 0; q < K2_PX; ++q) d[q] = (u0 + q < Ws) ? c.depth[row + u0 + q] : 0.0f;
    }
    const int r = p.r;
    const int Wd = p.dst.W, Hd = p.dst.H, P = p.pitch;
    const double lo = -(double)r, uhi = (double)(Wd + r), vhi = (double)(Hd + r);
    const double ry = __ldg(c.ry + sv);
    // the row part of the rotated ray, once per thread (its 4 pixels share a row)
    const double q0 = rel_q(c.rel, 0, ry), q1 = rel_q(c.rel, 1, ry), q2 = rel_q(c.rel, 2, ry);
    const bool fgk = p.tf.flag && (int)blockIdx.z < p.tf.n_fg;
    const uint64_t gen_hi = p.gen_ptr ? (uint64_t)__ldg(p.gen_ptr) << kGenShift : p.gen_hi;
    const uint8_t gen8 = (uint8_t)(gen_hi >> kGenShift);
    int first_t = -1, last_t = -1;
    double zq[K2_PX];
    unsigned stored = 0;
#pragma unroll
    for (int q = 0; q < K2_PX; ++q) {
        zq[q] = 0.0;
        if (!(d[q] > 0.0f)) continue;
        const int su = u0 + q;
        const double dd = (double)d[q];
        const double rx = __ldg(c.rx + su);
        const double x = rel_c(c.rel, 0, rx, q0, dd), y = rel_c(c.rel, 1, rx, q1, dd),
                     z = rel_c(c.rel, 2, rx, q2, dd);
        if (!(z > 0.0)) continue;
        double ur, vr;
        if (z > 1e-200) {
            const double rz = rcp_approx2(z);
            ur = proj_rint_r(p.dst.fx, x, z, rz, p.dst.cx);
            vr = proj_rint_r(p.dst.fy, y, z, rz, p.dst.cy);
        } else {
            ur = rint(dadd(ddiv(dmul(p.dst.fx, x), z), p.dst.cx));
            vr = rint(dadd(ddiv(dmul(p.dst.fy, y), z), p.dst.cy));
        }
        if (!(ur >= lo && ur < uhi && vr >= lo && vr < vhi)) continue;
        const size_t cell = (size_t)((int)vr + r) * P + (size_t)((int)ur + r);
        atomicMin((unsigned long long *)(c.canvas + cell),
                  (unsigned long long)(gen_hi | zkey(z, (uint32_t)(row + su), c.b)));
        if (fgk) {
            // the K3 tile of the target (padding columns/rows clamp to the edge
            // tiles, whose neighbourhood check covers them); a plain store
            // (no read-back on the critical path), once per tile change
            const int tx = min(max((int)ur, 0) / kTileFlagW, p.tf.ntx - 1);
            const int ty = min(max((int)vr, 0) / kTileFlagH, p.tf.nty - 1);
            const int t = ty * p.tf.ntx + tx;
            if (t != last_t) {
                // the thread's first tile is stored after the loop, unless the
                // previous lane's run already ended in it
                if (first_t < 0) first_t = t;
                else mark_tile(tile_flag(p.tf, blockIdx.z, t), gen8);
                last_t = t;
            }
        }
        zq[q] = z;
        stored |= 1u << q;
    }
    if (p.n_atomics) {
        // counting pass (untimed): the warp's z-buffer atomics, added to one
        // of 256 counters (the host sums them) so the adds do not serialise
        unsigned n = __popc(stored);
#pragma unroll
        for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
        const unsigned slot = (blockIdx.x * 131u + blockIdx.y * 31u + blockIdx.z * 7u +
                               (threadIdx.x >> 5)) & 255u;
        if ((threadIdx.x & 31) == 0 && n) atomicAdd(p.n_atomics + slot, (unsigned long long)n);
    }
    if (fgk) {
        // lanes hold consecutive source pixels: one store per run of a tile
        const int prev = __shfl_up_sync(0xffffffffu, last_t, 1);
        if (first_t >= 0 && ((threadIdx.x & 31) == 0 || first_t != prev))
            mark_tile(tile_flag(p.tf, blockIdx.z, first_t), gen8);
    }
    // the exact z of every scattering source, so K3 reads a winner's depth
    // instead of re-deriving it: one 32-byte run per thread where all four
    // pixels scattered (dense BG layers), single stores otherwise
    if (c.zsrc && stored) {
        double *o = c.zsrc + row + u0;
        if (stored == 0xFu && (Ws & 1) == 0) {
            reinterpret_cast<double2 *>(o)[0] = make_double2(zq[0], zq[1]);
            reinterpret_cast<double2 *>(o)[1] = make_double2(zq[2], zq[3]);
        } else {
#pragma unroll
            for (int q = 0; q < K2_PX; ++q)
                if (stored & (1u << q)) o[q] = zq[q];
        }
    }
}

cudaError_t launch_forward_warp(const WarpParams &p, long long max_src_pixels, cudaStream_t s) {
    if (p.n == 0) return cudaSuccess;
    int maxw = 0, maxh = 0;
    for (int k = 0; k < p.n; ++k) {
        maxw = p.c[k].src.W > maxw ? p.c[k].src.W : maxw;
        maxh = p.c[k].src.H > maxh ? p.c[k].src.H : maxh;
    }
    (void)max_src_pixels;
    const int per = K2_THREADS * K2_PX;
    dim3 grid((maxw + per - 1) / per, maxh, p.n);
    k_forward_warp<<<grid, K2_THREADS, 0, s>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K3: resolve + backward fetch + mix + composite

constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int MAXH = 5;   // max(r,1) + window/2 with r <= 3, window <= 5
constexpr int MAXRC = 2;  // window/2
constexpr int KMAX = (TY + 2 * MAXH) * (TX + 2 * MAXH);
constexpr int BMAX = (TY + 2 * MAXRC) * (TX + 2 * MAXRC);

size_t resolve_smem_bytes(int maxr) { return (size_t)maxr * 5 * NT * sizeof(double); }

// Median of the valid (finite) ring values around `center` (np.nanmedian,
// synthesis.py:123): odd count -> middle, even -> (lo + hi) / 2.
__device__ __forceinline__ double ring_median(const double *sz, int BC, int center, int rc,
                                              int cnt) {
    const int lo_rank = (cnt - 1) >> 1, hi_rank = cnt >> 1;
    double lo = 0.0, hi = 0.0;
    int a = 0;
    for (int ay = -rc; ay <= rc; ++ay) {
        for (int ax = -rc; ax <= rc; ++ax) {
            if (ay == 0 && ax == 0) continue;
            const double va = sz[center + ay * BC + ax];
            if (!(va < INFINITY)) { ++a; continue; }
            int rank = 0, b = 0;
            for (int by = -rc; by <= rc; ++by) {
                for (int bx = -rc; bx <= rc; ++bx) {
                    if (by == 0 && bx == 0) continue;
                    const double vb = sz[center + by * BC + bx];
                    if (vb < INFINITY && (vb < va || (vb == va && b < a))) ++rank;
                    ++b;
                }
            }
            if (rank == lo_rank) lo = va;
            if (rank == hi_rank) hi = va;
            ++a;
        }
    }
    return (cnt & 1) ? lo : ddiv(dadd(lo, hi), 2.0);
}

// Extension (not in the reference): angular factor of a blend weight,
// 1 / (theta + eps), theta = angle at the surface point X (the virtual pixel's
// ray at depth z) between the rays to the reference and to the virtual camera
// centres. Free-order f64 (the arccos in f32): this path has no reference
// to match.
__device__ __forceinline__ double angular_factor(const DevCam &dst, const DevCam &src, double rxd,
                                                 double ryd, double z, double eps) {
    const double px = rxd * z, py = ryd * z, pz = z;
    const double wx = px * dst.R[0] + py * dst.R[3] + pz * dst.R[6] + dst.C[0];
    const double wy = px * dst.R[1] + py * dst.R[4] + pz * dst.R[7] + dst.C[1];
    const double wz = px * dst.R[2] + py * dst.R[5] + pz * dst.R[8] + dst.C[2];
    const double ax = wx - src.C[0], ay = wy - src.C[1], az = wz - src.C[2];
    const double bx = wx - dst.C[0], by = wy - dst.C[1], bz = wz - dst.C[2];
    const double den = sqrt((ax * ax + ay * ay + az * az) * (bx * bx + by * by + bz * bz));
    double cs = den > 0.0 ? (ax * bx + ay * by + az * bz) / den : 1.0;
    cs = fmin(fmax(cs, -1.0), 1.0);
    // a blend weight, not a parity quantity: the angle in single precision
    return 1.0 / ((double)acosf((float)cs) + eps);
}

template <int MAXR>
__global__ void __launch_bounds__(NT) k_resolve_generic(const __grid_constant__ ResolveParams p) {
    __shared__ uint64_t sk[KMAX];
    __shared__ double sz[BMAX];
    __shared__ int swin[BMAX];
    __shared__ uint8_t sst[BMAX];
    extern __shared__ double sres[];  // [MAXR][5][NT]: colour rgb, depth, weight

    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const DevCam &dst = p.dst;
    const int Wd = dst.W, Hd = dst.H;
    const int ix = x0 + tx, iy = y0 + ty;
    const bool inimg = ix < Wd && iy < Hd;
    const uint64_t gen = p.gen_ptr ? (uint64_t)__ldg(p.gen_ptr) : p.gen;
    const size_t pix = (size_t)iy * Wd + ix;
    const int r = p.r, rc = p.window >> 1;
    const int Hh = (r > 1 ? r : 1) + rc;
    const int KC = TX + 2 * Hh, KR = TY + 2 * Hh;
    const int BC = TX + 2 * rc, BR = TY + 2 * rc;
    const int Wc = Wd + 2 * r, Hc = Hd + 2 * r;
    const size_t plane = (size_t)Wd * Hd;
    // virtual-camera ray of this pixel (pixel_rays, core.py:224-227)
    const double rxd = ddiv(dsub((double)ix, dst.cx), dst.fx);
    const double ryd = ddiv(dsub((double)iy, dst.cy), dst.fy);

    double lc[2][3] = {{0, 0, 0}, {0, 0, 0}};
    double ld[2] = {0.0, 0.0};
    bool lv[2] = {false, false};

    for (int L = 0; L < 2; ++L) {
        const int n = L == 0 ? p.n_fg : p.n_bg;
        const int k0 = L == 0 ? 0 : p.n_fg;
        uint32_t vmask = 0;
        for (int j = 0; j < n; ++j) {
            const int k = k0 + j;
            const ResolveContrib &c = p.c[k];
            __syncthreads();  // smem reuse across contributions
            // -- phase A: keys of tile + halo; stale generations read as empty
            int any = 0;
            for (int i = tid; i < KR * KC; i += NT) {
                const int ky = i / KC, kx = i - ky * KC;
                const int cy = y0 - Hh + ky + r, cx = x0 - Hh + kx + r;
                uint64_t key = kEmpty;
                if (cy >= 0 && cy < Hc && cx >= 0 && cx < Wc) {
                    const uint64_t v = c.canvas[(size_t)cy * p.pitch + cx];
                    if ((v >> kGenShift) == gen) { key = v; any = 1; }
                }
                sk[i] = key;
            }
            any = __syncthreads_or(any);
            double z = INFINITY;
            int win = -1;
            uint8_t st = kStageNone;
            if (any) {
                // -- phase B: splat policy + FG cull (synthesis.py:207-219)
                for (int i = tid; i < BR * BC; i += NT) {
                    const int by = i / BC, bx = i - by * BC;
                    const int qy = y0 - rc + by, qx = x0 - rc + bx;
                    double zq = INFINITY;
                    int wq = -1;
                    uint8_t sq = kStageNone;
                    if (qy >= 0 && qy < Hd && qx >= 0 && qx < Wd) {
                        const int kc = (by + Hh - rc) * KC + bx + Hh - rc;
                        uint64_t w = sk[kc];
                        if (w != kEmpty) {
                            sq = kStageCenter;
                        } else {
                            for (int dy = -r; dy <= r; ++dy)
                                for (int dx = -r; dx <= r; ++dx)
                                    if (dy || dx) {
                                        const uint64_t kk = sk[kc + dy * KC + dx];
                                        w = kk < w ? kk : w;
                                    }
                            if (w != kEmpty) {
                                sq = kStageSplat;
                                if (c.layer_fg) {
                                    // _neighbor_count of centre coverage, zero padded (:79-87)
                                    int cnt = 0;
                                    for (int dy = -1; dy <= 1; ++dy)
                                        for (int dx = -1; dx <= 1; ++dx) {
                                            if (!(dy || dx)) continue;
                                            const int ny = qy + dy, nx = qx + dx;
                                            if (ny >= 0 && ny < Hd && nx >= 0 && nx < Wd &&
                                                sk[kc + dy * KC + dx] != kEmpty)
                                                ++cnt;
                                        }
                                    if (cnt < 5) { w = kEmpty; sq = kStageNone; }
                                }
                            }
                        }
                        if (w != kEmpty) {
                            // exact f64 z of the winner, as K2 computed it
                            const uint32_t idx = (uint32_t)(w & ((1ull << c.b) - 1));
                            zq = __ldg(c.zsrc + idx);
                            wq = (int)idx;
                        }
                    }
                    sz[i] = zq;
                    swin[i] = wq;
                    sst[i] = sq;
                }
                __syncthreads();
                // -- phase C: crack median (synthesis.py:90-125)
                if (inimg) {
                    const int bi = (ty + rc) * BC + tx + rc;
                    z = sz[bi];
                    win = swin[bi];
                    st = sst[bi];
                    if (!(z < INFINITY) && rc > 0) {
                        int cnt = 0;
                        for (int dy = -rc; dy <= rc; ++dy)
                            for (int dx = -rc; dx <= rc; ++dx)
                                if ((dy || dx) && sz[bi + dy * BC + dx] < INFINITY) ++cnt;
                        if (cnt >= p.need) {
                            z = ring_median(sz, BC, bi, rc, cnt);
                            st = kStageCrack;
                            win = -1;
                        }
                    }
                }
            }
            // -- backward colour fetch (synthesis.py:224-247, _bilinear_fetch :128-159)
            bool ok = false;
            double c0 = 0.0, c1 = 0.0, c2 = 0.0;
            if (z < INFINITY) {
                double xs, ys, zs;
                transfer(c.rel, rxd, ryd, z, xs, ys, zs);
                if (zs > 0.0) {
                    const int Ws = c.src.W, Hs = c.src.H;
                    const double us = proj(c.src.fx, xs, zs, c.src.cx);
                    const double vs = proj(c.src.fy, ys, zs, c.src.cy);
                    if (us >= -0.5 && us <= (double)Ws - 0.5 && vs >= -0.5 &&
                        vs <= (double)Hs - 0.5) {
                        const double uc = fmin(fmax(us, 0.0), (double)(Ws - 1));
                        const double vc = fmin(fmax(vs, 0.0), (double)(Hs - 1));
                        const double u0 = floor(uc), v0 = floor(vc);
                        const int iu = (int)u0, iv = (int)v0;
                        const double fu = dsub(uc, u0), fv = dsub(vc, v0);
                        const double omu = dsub(1.0, fu), omv = dsub(1.0, fv);
                        const double wt[4] = {dmul(omu, omv), dmul(fu, omv), dmul(omu, fv),
                                              dmul(fu, fv)};
                        const bool inu = iu + 1 < Ws, inv = iv + 1 < Hs;
                        const uint32_t *row0 = c.texel + (size_t)iv * Ws + iu;
                        const uint32_t *row1 = row0 + Ws;
                        const uint32_t t[4] = {__ldg(row0), inu ? __ldg(row0 + 1) : 0u,
                                               inv ? __ldg(row1) : 0u,
                                               (inu && inv) ? __ldg(row1 + 1) : 0u};
                        const uint32_t fl = c.flag << 24;
                        double s = 0.0;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if (t[q] & fl) {
                                c0 = dadd(c0, dmul(wt[q], (double)(t[q] & 0xFFu)));
                                c1 = dadd(c1, dmul(wt[q], (double)((t[q] >> 8) & 0xFFu)));
                                c2 = dadd(c2, dmul(wt[q], (double)((t[q] >> 16) & 0xFFu)));
                                s = dadd(s, wt[q]);
                            }
                        }
                        if (s > 1e-12) {
                            ok = true;
                            c0 = ddiv(c0, s);
                            c1 = ddiv(c1, s);
                            c2 = ddiv(c2, s);
                        }
                    }
                }
            }
            if (!ok) { c0 = c1 = c2 = 0.0; }
            const double zd = ok ? z : 0.0;
            if (j < MAXR) {
                sres[(j * 5 + 0) * NT + tid] = c0;
                sres[(j * 5 + 1) * NT + tid] = c1;
                sres[(j * 5 + 2) * NT + tid] = c2;
                sres[(j * 5 + 3) * NT + tid] = zd;
                sres[(j * 5 + 4) * NT + tid] =
                    (p.ang && ok) ? c.weight * angular_factor(dst, c.src, rxd, ryd, z, p.ang_eps)
                                  : c.weight;
            }
            if (ok) vmask |= 1u << j;
            if (inimg) {
                const size_t o = (size_t)k * plane + pix;
                if (p.dbg.contrib_color) {
                    p.dbg.contrib_color[o * 3 + 0] = c0;
                    p.dbg.contrib_color[o * 3 + 1] = c1;
                    p.dbg.contrib_color[o * 3 + 2] = c2;
                }
                if (p.dbg.contrib_depth) p.dbg.contrib_depth[o] = zd;
                if (p.dbg.contrib_valid) p.dbg.contrib_valid[o] = ok ? 1 : 0;
                if (p.dbg.contrib_winner) p.dbg.contrib_winner[o] = win;
                if (p.dbg.contrib_stage) p.dbg.contrib_stage[o] = st;
            }
        }
        // -- mix_layer (synthesis.py:261-292)
        double zmin = INFINITY;
        for (int j = 0; j < n && j < MAXR; ++j) {
            const double zj = sres[(j * 5 + 3) * NT + tid];
            if (((vmask >> j) & 1u) && zj < zmin) zmin = zj;
        }
        const double thr = dadd(zmin, dmul(p.band_rel, zmin));
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, ad = 0.0, aw = 0.0;
        for (int j = 0; j < n && j < MAXR; ++j) {
            const double zj = sres[(j * 5 + 3) * NT + tid];
            if (((vmask >> j) & 1u) && zj <= thr) {
                const double w = sres[(j * 5 + 4) * NT + tid];
                a0 = dadd(a0, dmul(w, sres[(j * 5 + 0) * NT + tid]));
                a1 = dadd(a1, dmul(w, sres[(j * 5 + 1) * NT + tid]));
                a2 = dadd(a2, dmul(w, sres[(j * 5 + 2) * NT + tid]));
                ad = dadd(ad, dmul(w, zj));
                aw = dadd(aw, w);
            }
        }
        lv[L] = aw > 0.0;
        if (lv[L]) {
            lc[L][0] = ddiv(a0, aw);
            lc[L][1] = ddiv(a1, aw);
            lc[L][2] = ddiv(a2, aw);
        }
        if (inimg) {
            const size_t o = (size_t)L * plane + pix;
            if (p.dbg.merged_color) {
                p.dbg.merged_color[o * 3 + 0] = lc[L][0];
                p.dbg.merged_color[o * 3 + 1] = lc[L][1];
                p.dbg.merged_color[o * 3 + 2] = lc[L][2];
            }
            if (p.dbg.merged_depth) p.dbg.merged_depth[o] = lv[L] ? ddiv(ad, aw) : 0.0;
            if (p.dbg.merged_valid) p.dbg.merged_valid[o] = lv[L] ? 1 : 0;
        }
        ld[L] = lv[L] ? ddiv(ad, aw) : 0.0;
    }
    // -- composite (synthesis.py:295-318): hole, then BG, then FG; rint, clip
    if (inimg) {
        const int src = lv[0] ? 0 : (lv[1] ? 1 : -1);
        if (p.rgb_out) {
            uint8_t *o = p.rgb_out + pix * 3;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double v = src >= 0 ? lc[src][q] : p.hole[q];
                o[q] = (uint8_t)fmin(fmax(rint(v), 0.0), 255.0);
            }
        }
        if (p.prov_out) p.prov_out[pix] = lv[0] ? 2 : (lv[1] ? 1 : 0);
        if (p.depth_out) p.depth_out[pix] = (float)(src >= 0 ? ld[src] : 0.0);
    }
}

// ---------------------------------------------------------------------------
// K3 fast path: splat_radius 1, crack window 3 (the reference defaults,
// synthesis.py:39-40) with every tile dimension a compile-time constant.
//
// Per 32x8 target tile and per contribution:
//   keys   12x36 canvas cells (tile + 2-px halo) staged by TMA (or cp.async)
//          into a double buffer (next contribution's tile in flight while the
//          current one is resolved). Keys of stale generations compare
//          larger than any fresh key, so the ring min needs no sanitising.
//   cells  10x34 (tile + 1-px halo): centre key or 8-ring min (splat), FG cull
//          on < 5 centre-covered 8-neighbours.
//   pixel  winner z from K2's exact z plane, crack median (8-value sorting
//          network), backward projection and masked bilinear fetch; valid
//          per-contribution results kept in smem.
// then mix_layer x2 (valid contributions only) and the composite per pixel,
// the merged layers held as rounded packed colours in registers.

#ifndef FVV_K3_MINB
#define FVV_K3_MINB 6
#endif
#ifndef FVV_K3_TY
#define FVV_K3_TY 8
#endif
constexpr int FTY = FVV_K3_TY, FNT = TX * FTY;                   // fast-path tile: 32 x FTY
constexpr int FKR = FTY + 4, FKC = TX + 4, FKEYS = FKR * FKC;  // 12 x 36 (FTY = 8)
constexpr int FBR = FTY + 2, FBC = TX + 2, FCELLS = FBR * FBC;  // 10 x 34
// each key buffer is a TMA destination: 128-byte aligned (FTY = 4 or 8)
static_assert(FKEYS * sizeof(uint64_t) % 128 == 0, "K3 key buffers must stay 128-byte aligned");
// 32-bit winner cells from this many contributions per layer on (default:
// always). They save 2.7 KB of shared memory, which keeps 5 CTAs/SM with a
// 4-reference sres (c4: K3 1,078 -> 943 us) and trims K3 at c1 by 3 %.
#ifndef FVV_K3_W32_FROM
#define FVV_K3_W32_FROM 1
#endif
template <int MAXR>
using WinnerT = typename std::conditional<(MAXR >= FVV_K3_W32_FROM), uint32_t, uint64_t>::type;

constexpr int FCHUNKS = FKR * (FKC / 2);                       // 216 16-byte chunks

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
                 "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 12 x 36 keys (tile + 2-px halo) as 216 16-byte chunks, one per thread.
// Tile column x0-2 is canvas column x0-1 (r = 1), which the +1 allocation
// offset puts on an even element: every chunk is 16-byte aligned. Chunks
// outside the canvas rows / pitch are zero-filled; they only ever feed
// out-of-image cells, which are never resolved.
__device__ __forceinline__ void stage_keys(uint64_t *dst, const uint64_t *canvas, int x0, int y0,
                                           int P, int Hc, int tid) {
    if (tid < FCHUNKS) {
        const int ky = tid / (FKC / 2), kq = tid - ky * (FKC / 2);
        const int cy = y0 - 1 + ky, cx = x0 - 1 + 2 * kq;
        const bool ok = cy >= 0 && cy < Hc && cx >= -1 && cx + 1 <= P - 2;
        cp_async16(dst + ky * FKC + 2 * kq, ok ? canvas + (ptrdiff_t)cy * P + cx : canvas,
                   ok ? 16 : 0);
    }
}

// TMA (cp.async.bulk.tensor) staging of a key tile with mbarrier completion:
// one elected thread issues a 36 x 12 box of the 3-D canvas map; every
// thread waits on the buffer's mbarrier with the item's phase parity.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// composite's per-channel conversion: np.clip(np.round(v), 0, 255) -> uint8
// (half-even rint, synthesis.py:312)
// One F2I: cvt.rni rounds half to even like rint, .sat clamps to 0..255
// and NaN converts to 0 (what fmin(fmax(rint(NaN), 0), 255) gives).
__device__ __forceinline__ uint32_t rgb_u8(double v) {
#if FVV_RGB_CVT
    unsigned short r;
    asm("cvt.rni.sat.u8.f64 %0, %1;" : "=h"(r) : "d"(v));
    return r;
#else
    return (uint32_t)fmin(fmax(rint(v), 0.0), 255.0);
#endif
}

// exact f64 z of a winner index: the value K2 computed and stored for it
__device__ __forceinline__ double winner_z(const ResolveContrib &c, const DevCam &,
                                           uint32_t idx) {
    return __ldg(c.zsrc + idx);
}

// A cell's winner as K3 keeps it in shared memory: the whole 64-bit key, or
// (WT = uint32_t, for the wider contribution counts, whose mixes need the
// shared memory) just its source index — the key's depth bits only order the
// z-buffer, the exact z comes from zsrc. All ones = no winner either way
// (resolve_cells packs them).
template <typename WT>
__device__ __forceinline__ bool w_none(WT w) { return w == (WT)~(WT)0; }
template <typename WT>
__device__ __forceinline__ uint32_t w_idx(WT w, int b) {
    return sizeof(WT) == 8 ? (uint32_t)((uint64_t)w & ((1ull << b) - 1)) : (uint32_t)w;
}

template <typename WT>
__device__ __forceinline__ double key_z(const ResolveContrib &c, const DevCam &dst, WT w) {
    return w_none(w) ? INFINITY : winner_z(c, dst, w_idx(w, c.b));
}

// compare-exchange of two non-NaN depths (finite or +inf): one compare and
// selects (fmin + fmax would compare twice for their NaN rules)
#ifndef FVV_K3_CSWAP1
#define FVV_K3_CSWAP1 1
#endif
#ifndef FVV_K3_RAYRCP
#define FVV_K3_RAYRCP 0
#endif
__device__ __forceinline__ void cswap(double &a, double &b) {
#if FVV_K3_CSWAP1
    const bool sw = b < a;
    const double lo = sw ? b : a, hi = sw ? a : b;
#else
    const double lo = fmin(a, b), hi = fmax(a, b);
#endif
    a = lo;
    b = hi;
}


// min of 8 keys: the high words' min by three-input VIMNMX3, then the min of
// the low words among the keys holding it (exact; 23 instructions against
// 28 for seven 64-bit compare-and-selects: K3 135.6 -> 134.2 us at c1)
__device__ __forceinline__ uint64_t min8_u64(uint64_t n0, uint64_t n1, uint64_t n2, uint64_t n3,
                                             uint64_t n4, uint64_t n5, uint64_t n6, uint64_t n7) {
    const uint32_t h0 = (uint32_t)(n0 >> 32), h1 = (uint32_t)(n1 >> 32), h2 = (uint32_t)(n2 >> 32),
                   h3 = (uint32_t)(n3 >> 32), h4 = (uint32_t)(n4 >> 32), h5 = (uint32_t)(n5 >> 32),
                   h6 = (uint32_t)(n6 >> 32), h7 = (uint32_t)(n7 >> 32);
    const uint32_t hm = __vimin3_u32(__vimin3_u32(h0, h1, h2), __vimin3_u32(h3, h4, h5), min(h6, h7));
    const uint32_t l0 = h0 == hm ? (uint32_t)n0 : ~0u, l1 = h1 == hm ? (uint32_t)n1 : ~0u,
                   l2 = h2 == hm ? (uint32_t)n2 : ~0u, l3 = h3 == hm ? (uint32_t)n3 : ~0u,
                   l4 = h4 == hm ? (uint32_t)n4 : ~0u, l5 = h5 == hm ? (uint32_t)n5 : ~0u,
                   l6 = h6 == hm ? (uint32_t)n6 : ~0u, l7 = h7 == hm ? (uint32_t)n7 : ~0u;
    const uint32_t lm = __vimin3_u32(__vimin3_u32(l0, l1, l2), __vimin3_u32(l3, l4, l5), min(l6, l7));
    return ((uint64_t)hm << 32) | lm;
}

// Cells-phase descriptors: a thread's cells (tid, tid + FNT) are the same
// for every contribution of the tile, so their key-tile offset, in-image bit
// and in-image neighbour mask are formed once per CTA (c1: K3 141.0 -> 135.5
// us together with the popcount neighbour test and the 32-bit index mask;
// formed per contribution instead, 137.7)
struct CellDesc {
    uint32_t d[2];   // kc | in-image << 15 | neighbour mask << 16; 0 = no cell
};

__device__ __forceinline__ CellDesc cell_desc(int Wd, int Hd, int x0, int y0, int tid) {
    CellDesc cd;
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
        const int i = tid + rep * FNT;
        cd.d[rep] = 0;
        if (i >= FCELLS) continue;
        const int by = i / FBC, bx = i - by * FBC;
        const int qy = y0 - 1 + by, qx = x0 - 1 + bx;
        const uint32_t kc = (uint32_t)((by + 1) * FKC + bx + 1);
        // neighbour bits n0..n7 (up-left, up, up-right, left, right,
        // down-left, down, down-right), out-of-image ones cleared
        uint32_t im = 0xFFu;
        if (!(qy > 0)) im &= ~0x07u;
        if (!(qy + 1 < Hd)) im &= ~0xE0u;
        if (!(qx > 0)) im &= ~0x29u;
        if (!(qx + 1 < Wd)) im &= ~0x94u;
        const bool inb = (unsigned)qy < (unsigned)Hd && (unsigned)qx < (unsigned)Wd;
        cd.d[rep] = kc | ((uint32_t)inb << 15) | (im << 16);
    }
    return cd;
}

// Phase "cells" of one contribution: splat policy + FG cull (synthesis.py:
// 207-219) for the 10x34 cells around the tile -> winner (all ones = none).
template <bool DBG, typename WT>
__device__ __forceinline__ int resolve_cells(const ResolveContrib &c, const CellDesc &cd,
                                             const uint64_t *K, WT *swk, uint8_t *sst,
                                             uint64_t gen, int tid) {
    int any = 0;
    // a key is fresh (this view's generation) iff it is below `lim`: older
    // generations carry larger tags and empty is all ones, so the ring min of
    // a cell is fresh iff any of its neighbours is (the BG splat test), and a
    // fresh key is never kEmpty (packs without the empty test)
    const uint64_t lim = (gen + 1) << kGenShift;
    const bool fgl = c.layer_fg;
    // b <= 26: a key's source index lies in its low word
    const uint32_t imask = (1u << c.b) - 1u;
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
        const int i = tid + rep * FNT;
        if (i >= FCELLS) break;
        const uint32_t dsc = cd.d[rep];
        uint64_t w = kEmpty;
        uint8_t sq = kStageNone;
        if (dsc & 0x8000u) {
            const int kc = (int)(dsc & 0x7FFFu);
            w = K[kc];
            if (w < lim) {
                sq = kStageCenter;
            } else {
                const uint64_t n0 = K[kc - FKC - 1], n1 = K[kc - FKC], n2 = K[kc - FKC + 1];
                const uint64_t n3 = K[kc - 1], n4 = K[kc + 1];
                const uint64_t n5 = K[kc + FKC - 1], n6 = K[kc + FKC], n7 = K[kc + FKC + 1];
                bool keep;
                if (fgl) {
                    // _neighbor_count (synthesis.py:79-87): in-image centre
                    // hits, as a population count of the fresh-neighbour bits
                    const unsigned fm = (unsigned)(n0 < lim) | ((unsigned)(n1 < lim) << 1) |
                                        ((unsigned)(n2 < lim) << 2) | ((unsigned)(n3 < lim) << 3) |
                                        ((unsigned)(n4 < lim) << 4) | ((unsigned)(n5 < lim) << 5) |
                                        ((unsigned)(n6 < lim) << 6) | ((unsigned)(n7 < lim) << 7);
                    keep = __popc(fm & (dsc >> 16)) >= 5;
                    if (keep) w = min8_u64(n0, n1, n2, n3, n4, n5, n6, n7);
                } else {
                    // the 8-ring min; stale keys compare larger than any fresh one
                    w = min8_u64(n0, n1, n2, n3, n4, n5, n6, n7);
                    keep = w < lim;
                }
                if (keep) sq = kStageSplat;
            }
            any |= sq != kStageNone;
        }
        if (sizeof(WT) == 8) swk[i] = sq != kStageNone ? (WT)w : (WT)kEmpty;
        else swk[i] = sq != kStageNone ? (WT)((uint32_t)w & imask) : (WT)~(WT)0;
        if (DBG) sst[i] = sq;
    }
    return any;
}

// crack median of a hole pixel from its 8 neighbours' winner keys. About 8 %
// of (pixel, contribution) pairs at c1, ~2.5 lanes per warp that enters it;
// a CTA crack queue (one warp resolving all of an item's cracks after an
// extra barrier, layer mixes deferred) was 16 % slower.
#ifndef FVV_K3_CRACK_NOINLINE
#define FVV_K3_CRACK_NOINLINE 0
#endif
template <typename WT>
#if FVV_K3_CRACK_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
double crack_z(const ResolveContrib &c, const DevCam &dst,
                                       const WT *W, int bi, int *stage) {
    const WT k0 = W[bi - FBC - 1], k1 = W[bi - FBC], k2 = W[bi - FBC + 1], k3 = W[bi - 1],
             k4 = W[bi + 1], k5 = W[bi + FBC - 1], k6 = W[bi + FBC], k7 = W[bi + FBC + 1];
    const int cnt = !w_none(k0) + !w_none(k1) + !w_none(k2) + !w_none(k3) + !w_none(k4) +
                    !w_none(k5) + !w_none(k6) + !w_none(k7);
    if (cnt < 5) return INFINITY;
    double v0 = key_z(c, dst, k0), v1 = key_z(c, dst, k1), v2 = key_z(c, dst, k2),
           v3 = key_z(c, dst, k3), v4 = key_z(c, dst, k4), v5 = key_z(c, dst, k5),
           v6 = key_z(c, dst, k6), v7 = key_z(c, dst, k7);
    cswap(v0, v1); cswap(v2, v3); cswap(v4, v5); cswap(v6, v7);
    cswap(v0, v2); cswap(v1, v3); cswap(v4, v6); cswap(v5, v7);
    cswap(v1, v2); cswap(v5, v6);
    cswap(v0, v4); cswap(v1, v5); cswap(v2, v6); cswap(v3, v7);
    cswap(v2, v4); cswap(v3, v5);
    cswap(v1, v2); cswap(v3, v4); cswap(v5, v6);
    *stage = kStageCrack;
    const double lo = cnt <= 6 ? v2 : v3;
    // even count: mean of the middle pair; halving is exact, so * 0.5 == / 2
    return (cnt & 1) ? lo : dmul(dadd(lo, cnt == 6 ? v3 : v4), 0.5);
}

// np.clip(v, 0, hi) of a finite v: two compares and selects (fmin/fmax
// would add their NaN handling)
#ifndef FVV_K3_CLIP
#define FVV_K3_CLIP 1
#endif
__device__ __forceinline__ double clip_finite(double v, double hi) {
#if FVV_K3_CLIP
    v = v < 0.0 ? 0.0 : v;
    return v > hi ? hi : v;
#else
    return fmin(fmax(v, 0.0), hi);
#endif
}

// backward projection + masked bilinear fetch of one covered pixel
// (synthesis.py:224-247, _bilinear_fetch :128-159)
__device__ __forceinline__ bool fetch(const ResolveContrib &c, const DevCam &dst, double rxd,
                                      double ryd, double z, double &c0, double &c1, double &c2) {
    double xs, ys, zs;
    transfer(c.rel, rxd, ryd, z, xs, ys, zs);
    if (!(zs > 0.0)) return false;
    const int Ws = c.src.W, Hs = c.src.H;
    double us, vs;
    if (zs > 1e-100) {
        const double rz = rcp_nr(zs);
        us = dadd(div_rcp(dmul(c.src.fx, xs), zs, rz), c.src.cx);
        vs = dadd(div_rcp(dmul(c.src.fy, ys), zs, rz), c.src.cy);
    } else {
        us = proj(c.src.fx, xs, zs, c.src.cx);
        vs = proj(c.src.fy, ys, zs, c.src.cy);
    }
    if (!(us >= -0.5 && us <= (double)Ws - 0.5 && vs >= -0.5 && vs <= (double)Hs - 0.5))
        return false;
    const double uc = clip_finite(us, (double)(Ws - 1)), vc = clip_finite(vs, (double)(Hs - 1));
    const double u0 = floor(uc), v0 = floor(vc);
    const int iu = (int)u0, iv = (int)v0;
    const double fu = dsub(uc, u0), fv = dsub(vc, v0);
    const double omu = dsub(1.0, fu), omv = dsub(1.0, fv);
    const bool inu = iu + 1 < Ws, inv = iv + 1 < Hs;
    const uint32_t *row0 = c.texel + (size_t)iv * Ws + iu;
    const uint32_t fl = c.flag << 24;
    const uint32_t t0 = __ldg(row0);
    const uint32_t t1 = inu ? __ldg(row0 + 1) : 0u;
    const uint32_t t2 = inv ? __ldg(row0 + Ws) : 0u;
    const uint32_t t3 = (inu && inv) ? __ldg(row0 + Ws + 1) : 0u;
    // a masked tap weight of +0.0 adds exactly nothing (synthesis.py:154)
    const double w0 = (t0 & fl) ? dmul(omu, omv) : 0.0;
    const double w1 = (t1 & fl) ? dmul(fu, omv) : 0.0;
    const double w2 = (t2 & fl) ? dmul(omu, fv) : 0.0;
    const double w3 = (t3 & fl) ? dmul(fu, fv) : 0.0;
#define FVV_CH(T, SH) (double)(((T) >> (SH)) & 0xFFu)
    c0 = dadd(dadd(dadd(dmul(w0, FVV_CH(t0, 0)), dmul(w1, FVV_CH(t1, 0))), dmul(w2, FVV_CH(t2, 0))),
              dmul(w3, FVV_CH(t3, 0)));
    c1 = dadd(dadd(dadd(dmul(w0, FVV_CH(t0, 8)), dmul(w1, FVV_CH(t1, 8))), dmul(w2, FVV_CH(t2, 8))),
              dmul(w3, FVV_CH(t3, 8)));
    c2 = dadd(dadd(dadd(dmul(w0, FVV_CH(t0, 16)), dmul(w1, FVV_CH(t1, 16))),
                   dmul(w2, FVV_CH(t2, 16))), dmul(w3, FVV_CH(t3, 16)));
#undef FVV_CH
    const double s = dadd(dadd(dadd(w0, w1), w2), w3);
    if (!(s > 1e-12)) return false;
    if (s != 1.0) {  // x / 1.0 is x: most all-Valid windows need no division
        const double rs = rcp_nr(s);
        c0 = div_rcp(c0, s, rs);
        c1 = div_rcp(c1, s, rs);
        c2 = div_rcp(c2, s, rs);
    }
    return true;
}

#ifndef FVV_K3_MIXUNROLL
#define FVV_K3_MIXUNROLL 1
#endif
#ifndef FVV_K3_NBUF
#define FVV_K3_NBUF 2
#endif
// K3 key staging: 1 = cp.async.bulk.tensor (TMA) + mbarrier (default: at 5
// CTAs/SM it measured 209.4 vs 212.9 us for cp.async; at 4 CTAs/SM, before
// the merged layers left shared memory, cp.async had been 3 % faster),
// 0 = per-thread 16-byte cp.async
#ifndef FVV_K3_TMA
#define FVV_K3_TMA 1
#endif
constexpr int NBUF = FVV_K3_NBUF;  // key tiles in flight (NBUF-1 items ahead of the one shaded)

// One 32x8 tile per CTA; the 12x36 key tiles of the next three contributions
// are in flight (cp.async groups) while the current one is shaded, and the
// cells phase of contribution q+1 runs in the same barrier interval as the
// per-pixel work of contribution q.
// dynamic shared memory of a k_resolve_fast CTA: key tiles, winner cells,
// per-contribution results, rays, (ANG) weights, (DBG) stage bytes
template <int MAXR, bool ANG>
constexpr size_t fast_smem() {
    return NBUF * FKEYS * sizeof(uint64_t) + 2 * FCELLS * sizeof(WinnerT<MAXR>) +
           (size_t)MAXR * 4 * FNT * sizeof(double) + (TX + FTY) * sizeof(double) +
           (ANG && MAXR <= 3 ? (size_t)MAXR * FNT * sizeof(double) : 0) + 2 * FCELLS;
}

// Resident CTAs per SM the register budget is sized for: FVV_K3_MINB (6:
// 40 registers) where that many CTAs' shared memory fits the SM's 228 KB
// (1 KB reserved per CTA, ~0.2 KB static), else 5 (48 registers). At c1 (3
// references) 6 CTAs measured 140.7 us against 145.7 at 5 with this build;
// 7 or 8 (32 registers) spill heavily.
template <int MAXR, bool ANG>
constexpr int k3_min_blocks() {
    return (fast_smem<MAXR, ANG>() + 1024 + 256) * FVV_K3_MINB <= 228 * 1024 ? FVV_K3_MINB : 5;
}

template <int MAXR, bool DBG, bool ANG>
__global__ void __launch_bounds__(FNT, (k3_min_blocks<MAXR, ANG>())) k_resolve_fast(const __grid_constant__ ResolveParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[NBUF];                // TMA completion per buffer
    uint64_t *sk = reinterpret_cast<uint64_t *>(smem);          // [NBUF][FKEYS]
    using WT = WinnerT<MAXR>;
    WT *swk = reinterpret_cast<WT *>(sk + NBUF * FKEYS);          // [2][FCELLS] winners
    double *sres = reinterpret_cast<double *>(swk + 2 * FCELLS); // [MAXR][4][FNT]
    double *sray = sres + MAXR * 4 * FNT;                         // [TX] rx, [FTY] ry
    // ANG weights: kept per contribution in shared memory up to 3 references;
    // for more, evaluated in the mix (the raster would cost the 5th CTA/SM)
    constexpr bool WSTORE = ANG && MAXR <= 3;
    double *swt = sray + TX + FTY;                                // [MAXR][FNT] (WSTORE)
    uint8_t *sst = reinterpret_cast<uint8_t *>(swt + (WSTORE ? MAXR * FNT : 0));  // [2][FCELLS] (DBG)

    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const DevCam &dst = p.dst;
    const int Wd = dst.W, Hd = dst.H;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * FTY;
    const int ix = x0 + tx, iy = y0 + ty;
    const bool inimg = ix < Wd && iy < Hd;
    const size_t pix = (size_t)iy * Wd + ix;
    const int P = p.pitch, Hc = Hd + 2;
    const size_t plane = (size_t)Wd * Hd;
    const uint64_t gen = p.gen_ptr ? (uint64_t)__ldg(p.gen_ptr) : p.gen;
    const int ntot = p.n_fg + p.n_bg;
    // the contributions this tile resolves, in reference order: every BG
    // contribution, and the FG ones K2 flagged near this tile (all of them
    // when debug rasters are requested)
    __shared__ int8_t s_item[2 * FVV_MAX_REFS];
    __shared__ int s_nitems;
    __shared__ int s_needbg;   // some in-image pixel's merged FG layer is invalid
#if FVV_K3_TMA
    // key tiles by TMA: thread 0 arms buffer q % NBUF's mbarrier and issues
    // the box; canvas column x0-1 .. x0+34 is tensor x = x0 .. x0+35 (the
    // allocation's +1 offset), out-of-canvas boxes are zero-filled (they only
    // feed out-of-image cells, which are never resolved)
    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) mbar_init(&s_bar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    auto stage = [&](int q, int n) {
        if (tid == 0 && q < n) {
            uint64_t *bar = &s_bar[q % NBUF];
            mbar_expect_tx(bar, FKEYS * sizeof(uint64_t));
            tma_load_3d(sk + (q % NBUF) * FKEYS, &p.kmap, x0, y0 - 1, s_item[q], bar);
        }
    };
#endif
    if (tid < 32) {
        bool act = false;
        if (tid < ntot) {
            act = DBG || !p.tf.flag || tid >= p.n_fg;
            if (!act) {
                // the flag tiles covering the staged key tile (target pixels
                // x0-2 .. x0+TX+1, y0-2 .. y0+FTY+1; K2 clamps the canvas
                // padding into the edge tiles): at most NXF x NYF of them
                // (3 x 3 for 32 x 8 flag tiles); the loads are independent
                // (clamped duplicates are harmless), so they cost one round
                // trip. 16x8, 16x4 and 8x8 flag tiles measured the same.
                const int fx0 = max(x0 - 2, 0) / kTileFlagW;
                const int fx1 = min((x0 + TX + 1) / kTileFlagW, p.tf.ntx - 1);
                const int fy0 = max(y0 - 2, 0) / kTileFlagH;
                const int fy1 = min((y0 + FTY + 1) / kTileFlagH, p.tf.nty - 1);
                constexpr int NXF = (TX + 3) / kTileFlagW + 2, NYF = (FTY + 3) / kTileFlagH + 2;
                uint8_t f[NXF * NYF];
#pragma unroll
                for (int e = 0; e < NXF * NYF; ++e) {
                    const int tx2 = min(fx0 + e % NXF, fx1), ty2 = min(fy0 + e / NXF, fy1);
                    f[e] = *tile_flag(p.tf, tid, ty2 * p.tf.ntx + tx2);
                }
#pragma unroll
                for (int e = 0; e < NXF * NYF; ++e) act |= f[e] == (uint8_t)gen;
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, act);
        if (act) s_item[__popc(m & ((1u << tid) - 1u))] = (int8_t)tid;
        if (tid == 0) {
            s_nitems = __popc(m);
            s_needbg = 0;
        }
#if FVV_K3_TMA
        // the first key tiles go out before the CTA barrier
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NBUF; ++q) stage(q, __popc(m));
#endif
    } else if (tid < 32 + TX + FTY) {
        // virtual-camera rays of the tile's columns and rows (pixel_rays,
        // core.py:224-227), once per CTA, while warp 0 picks the contributions
        // (the correctly rounded quotient from a Newton reciprocal, div_rcp)
        const int t = tid - 32;
#if FVV_K3_RAYRCP
        if (t < TX) sray[t] = div_rcp(dsub((double)(x0 + t), dst.cx), dst.fx, rcp_nr(dst.fx));
        else sray[t] = div_rcp(dsub((double)(y0 + t - TX), dst.cy), dst.fy, rcp_nr(dst.fy));
#else
        if (t < TX) sray[t] = ddiv(dsub((double)(x0 + t), dst.cx), dst.fx);
        else sray[t] = ddiv(dsub((double)(y0 + t - TX), dst.cy), dst.fy);
#endif
    }
    __syncthreads();
    const int nitems = s_nitems;
    if (nitems == 0) {
        // no BG contribution and no FG key near the tile: all holes
        if (inimg) {
            if (p.rgb_out)
                for (int ch = 0; ch < 3; ++ch) p.rgb_out[pix * 3 + ch] = (uint8_t)(p.hole_rgb >> (8 * ch));
            if (p.prov_out) p.prov_out[pix] = 0;
            if (p.depth_out) p.depth_out[pix] = 0.0f;
        }
        return;
    }
#if FVV_K3_TMA
    auto wait_keys = [&](int q) {
        if (q < nitems) mbar_wait(&s_bar[q % NBUF], (unsigned)((q / NBUF) & 1));
    };
    wait_keys(0);
#else
    auto stage = [&](int q) {
        if (q < nitems)
            stage_keys(sk + (q % NBUF) * FKEYS, p.c[s_item[q]].canvas, x0, y0, P, Hc, tid);
        cp_async_commit();  // (possibly empty) group per item keeps the accounting uniform
    };

#pragma unroll
    for (int q = 0; q < NBUF; ++q) stage(q);
    cp_async_wait<NBUF - 1>();
    __syncthreads();
#endif
        const CellDesc cdesc = cell_desc(Wd, Hd, x0, y0, tid);
    int any_next = resolve_cells<DBG>(p.c[s_item[0]], cdesc, sk, swk, sst, gen, tid);

    bool fv = false, bv = false;
    uint32_t fgc = 0, bgc = 0;   // rounded merged layer colours (R | G << 8 | B << 16)
    float fgz = 0.0f, bgz = 0.0f;
    uint32_t vmask = 0;
    // -- end of a layer: mix_layer (synthesis.py:261-292) over the layer's
    // valid contributions (kb = its first contribution index)
    auto mix = [&](bool fgl, int kb) {
        // valid contributions only, in ascending (reference) order
        double zmin = INFINITY;
#if FVV_K3_MIXUNROLL
#pragma unroll
        for (int qq = 0; qq < MAXR; ++qq) {
            if (!((vmask >> qq) & 1u)) continue;
#else
        for (unsigned m = vmask; m; m &= m - 1) {
            const int qq = __ffs(m) - 1;
#endif
            const double zj = sres[(qq * 4 + 3) * FNT + tid];
            if (zj < zmin) zmin = zj;
        }
        const double thr = dadd(zmin, dmul(p.band_rel, zmin));
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, ad = 0.0, aw = 0.0;
#if FVV_K3_MIXUNROLL
#pragma unroll
        for (int qq = 0; qq < MAXR; ++qq) {
            if (!((vmask >> qq) & 1u)) continue;
#else
        for (unsigned m = vmask; m; m &= m - 1) {
            const int qq = __ffs(m) - 1;
#endif
            const double zj = sres[(qq * 4 + 3) * FNT + tid];
            if (zj <= thr) {
                // ANG without WSTORE: the angular factor of the participating
                // contributions from the stored exact z (same value)
                const double w = WSTORE ? swt[qq * FNT + tid]
                                 : ANG ? p.c[kb + qq].weight *
                                             angular_factor(dst, p.c[kb + qq].src, sray[tx],
                                                            sray[TX + ty], zj, p.ang_eps)
                                       : p.c[kb + qq].weight;
                a0 = dadd(a0, dmul(w, sres[(qq * 4 + 0) * FNT + tid]));
                a1 = dadd(a1, dmul(w, sres[(qq * 4 + 1) * FNT + tid]));
                a2 = dadd(a2, dmul(w, sres[(qq * 4 + 2) * FNT + tid]));
                if (DBG || p.depth_out) ad = dadd(ad, dmul(w, zj));
                aw = dadd(aw, w);
            }
        }
        const bool mv = aw > 0.0;
        double m0 = 0.0, m1 = 0.0, m2 = 0.0;
        if (mv) {
            const double ra = rcp_nr(aw);
            m0 = div_rcp(a0, aw, ra);
            m1 = div_rcp(a1, aw, ra);
            m2 = div_rcp(a2, aw, ra);
        }
        const float mz = (p.depth_out && mv) ? (float)ddiv(ad, aw) : 0.0f;
        if (fgl) {
            // composite needs only the FG layer's rounded colour (it wins
            // wherever valid, synthesis.py:309-312): one packed register
            fv = mv;
            fgc = rgb_u8(m0) | (rgb_u8(m1) << 8) | (rgb_u8(m2) << 16);
            fgz = mz;
        } else {
            bv = mv;
            bgc = rgb_u8(m0) | (rgb_u8(m1) << 8) | (rgb_u8(m2) << 16);
            bgz = mz;
        }
        vmask = 0;
        if (DBG && inimg) {
            const size_t o = (size_t)(fgl ? 0 : 1) * plane + pix;
            if (p.dbg.merged_color) {
                p.dbg.merged_color[o * 3 + 0] = m0;
                p.dbg.merged_color[o * 3 + 1] = m1;
                p.dbg.merged_color[o * 3 + 2] = m2;
            }
            if (p.dbg.merged_depth) p.dbg.merged_depth[o] = mv ? ddiv(ad, aw) : 0.0;
            if (p.dbg.merged_valid) p.dbg.merged_valid[o] = mv ? 1 : 0;
        }
    };
#pragma unroll 1
    for (int q = 0; q < nitems; ++q) {
        const int k = s_item[q];
        const bool fgl = k < p.n_fg;
        const int j = fgl ? k : k - p.n_fg;
        // keys of q+1 must have landed (groups q+1 done, q+2 may pend); cells of q
        // complete
#if FVV_K3_TMA
        wait_keys(q + 1);
        const int any = __syncthreads_or(any_next);
        // every in-image pixel has a valid merged FG layer: the BG layer cannot
        // change the composite (FG wins wherever valid, synthesis.py:309-311),
        // so the tile skips its BG contributions (no key tile is in flight:
        // q+1's landed above, q+2's is issued below)
        if (!DBG && !fgl && q > 0 && s_item[q - 1] < p.n_fg && !s_needbg) break;
        // keys of q+NBUF into the buffer item q's cells phase used (all reads of
        // it by the generic proxy are ordered before the barrier above)
        if (tid == 0) fence_proxy_async();
        stage(q + NBUF, nitems);
#else
        cp_async_wait<NBUF - 2>();
        const int any = __syncthreads_or(any_next);
        if (!DBG && !fgl && q > 0 && s_item[q - 1] < p.n_fg && !s_needbg) break;
        // keys of q+NBUF into the buffer item q's cells phase (iteration q-1) used
        stage(q + NBUF);
#endif
        // cells of q+1 (other warps' per-pixel work of q overlaps it)
        any_next = 0;
        if (q + 1 < nitems)
            any_next = resolve_cells<DBG>(p.c[s_item[q + 1]], cdesc,
                                          sk + ((q + 1) % NBUF) * FKEYS, swk + ((q + 1) & 1) * FCELLS,
                                          sst + ((q + 1) & 1) * FCELLS, gen, tid);
        const ResolveContrib &c = p.c[k];
        const WT *W = swk + (q & 1) * FCELLS;
        double z = INFINITY;
        int win = -1;
        uint8_t st = kStageNone;
        bool ok = false;
        double c0 = 0.0, c1 = 0.0, c2 = 0.0;
        // BG contributions cannot change a pixel whose merged FG layer is valid
        // (composite = FG over BG, synthesis.py:309-311): skip their fetch
        // there unless every intermediate raster is requested (DBG)
        if (any && inimg && (DBG || fgl || !fv)) {
            const int bi = (ty + 1) * FBC + tx + 1;
            const WT wk = W[bi];
            if (DBG) st = sst[(q & 1) * FCELLS + bi];
            if (!w_none(wk)) {
                const uint32_t idx = w_idx(wk, c.b);
                z = winner_z(c, dst, idx);
                win = (int)idx;
            } else {
                // crack median (synthesis.py:90-125)
                int stc = st;
                z = crack_z(c, dst, W, bi, &stc);
                st = (uint8_t)stc;
            }
            if (z < INFINITY) ok = fetch(c, dst, sray[tx], sray[TX + ty], z, c0, c1, c2);
        }
        if (!ok) { c0 = c1 = c2 = 0.0; }
        const double zd = ok ? z : 0.0;
        // the mixes read only contributions whose vmask bit is set
        if (ok) {
            sres[(j * 4 + 0) * FNT + tid] = c0;
            sres[(j * 4 + 1) * FNT + tid] = c1;
            sres[(j * 4 + 2) * FNT + tid] = c2;
            sres[(j * 4 + 3) * FNT + tid] = zd;
            if (WSTORE)
                swt[j * FNT + tid] =
                    c.weight * angular_factor(dst, c.src, sray[tx], sray[TX + ty], z, p.ang_eps);
            vmask |= 1u << j;
        }
        if (DBG && inimg) {
            const size_t o = (size_t)k * plane + pix;
            if (p.dbg.contrib_color) {
                p.dbg.contrib_color[o * 3 + 0] = c0;
                p.dbg.contrib_color[o * 3 + 1] = c1;
                p.dbg.contrib_color[o * 3 + 2] = c2;
            }
            if (p.dbg.contrib_depth) p.dbg.contrib_depth[o] = zd;
            if (p.dbg.contrib_valid) p.dbg.contrib_valid[o] = ok ? 1 : 0;
            if (p.dbg.contrib_winner) p.dbg.contrib_winner[o] = win;
            if (p.dbg.contrib_stage) p.dbg.contrib_stage[o] = st;
        }
        // the last resolved contribution of its layer ends it
        const bool last = q + 1 == nitems || (fgl && s_item[q + 1] >= p.n_fg);
        if (last) {
            mix(fgl, k - j);
            if (!DBG && fgl && inimg && !fv) s_needbg = 1;
        }
    }
    // -- end of a tile: composite (synthesis.py:295-318): hole, BG, FG; rint, clip
    if (inimg) {
        const uint32_t oc = fv ? fgc : (bv ? bgc : p.hole_rgb);
        if (p.rgb_out) {
            uint8_t *o = p.rgb_out + pix * 3;
            o[0] = (uint8_t)oc;
            o[1] = (uint8_t)(oc >> 8);
            o[2] = (uint8_t)(oc >> 16);
        }
        if (p.prov_out) p.prov_out[pix] = fv ? 2 : (bv ? 1 : 0);
        if (p.depth_out) p.depth_out[pix] = fv ? fgz : (bv ? bgz : 0.0f);
    }
#if !FVV_K3_TMA
    cp_async_wait<0>();
#endif
}

// The dynamic shared-memory limit is a per-device function attribute: raise
// it once per (kernel, device). `done` is the kernel's bitmask of devices.
template <typename K>
static void raise_smem(K kernel, size_t bytes, std::atomic<uint64_t> &done) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    done.fetch_or(bit, std::memory_order_acq_rel);
}


template <int MAXR, bool DBG, bool ANG>
static void launch_fast(const ResolveParams &p, dim3 grid, cudaStream_t s) {
    static std::atomic<uint64_t> done{0};
    raise_smem(k_resolve_fast<MAXR, DBG, ANG>, fast_smem<MAXR, ANG>(), done);
    k_resolve_fast<MAXR, DBG, ANG><<<grid, FNT, fast_smem<MAXR, ANG>(), s>>>(p);
}

template <int MAXR>
static void launch_fast_r(const ResolveParams &p, bool dbg, dim3 grid, cudaStream_t s) {
    if (p.ang) {
        if (dbg) launch_fast<MAXR, true, true>(p, grid, s);
        else launch_fast<MAXR, false, true>(p, grid, s);
    } else {
        if (dbg) launch_fast<MAXR, true, false>(p, grid, s);
        else launch_fast<MAXR, false, false>(p, grid, s);
    }
}


bool resolve_uses_tma() { return FVV_K3_TMA != 0; }
int resolve_tile_rows() { return FTY; }

cudaError_t launch_resolve(const ResolveParams &p, cudaStream_t s) {
    dim3 grid((p.dst.W + TX - 1) / TX, (p.dst.H + TY - 1) / TY);
    dim3 fgrid((p.dst.W + TX - 1) / TX, (p.dst.H + FTY - 1) / FTY);
    const int maxn = p.n_fg > p.n_bg ? p.n_fg : p.n_bg;
    const bool dbg = p.dbg.contrib_color || p.dbg.contrib_depth || p.dbg.contrib_valid ||
                     p.dbg.contrib_winner || p.dbg.contrib_stage || p.dbg.merged_color ||
                     p.dbg.merged_depth || p.dbg.merged_valid;
    if (p.r == 1 && p.window == 3 && p.n_fg + p.n_bg > 0 && (p.has_kmap || !FVV_K3_TMA)) {
        if (maxn <= 3) launch_fast_r<3>(p, dbg, fgrid, s);
        else if (maxn <= 4) launch_fast_r<4>(p, dbg, fgrid, s);
        else launch_fast_r<FVV_MAX_REFS>(p, dbg, fgrid, s);
        return cudaGetLastError();
    }
    if (maxn <= 4) {
        static std::atomic<uint64_t> done4{0};
        raise_smem(k_resolve_generic<4>, resolve_smem_bytes(4), done4);
        k_resolve_generic<4><<<grid, NT, resolve_smem_bytes(4), s>>>(p);
    } else {
        static std::atomic<uint64_t> done16{0};
        raise_smem(k_resolve_generic<FVV_MAX_REFS>, resolve_smem_bytes(FVV_MAX_REFS), done16);
        k_resolve_generic<FVV_MAX_REFS><<<grid, NT, resolve_smem_bytes(FVV_MAX_REFS), s>>>(p);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K4 (extension, not in the reference: SPEC.md:548 leaves holes at hole_color)
//
// Background-biased disocclusion fill. A hole of a forward-warped view is
// where the virtual camera sees past a foreground edge that no reference saw
// behind, so the right colour is the background beside it. Each hole pixel
// takes the first non-hole pixel to its left, right, top and bottom (within
// `radius` pixels), keeps the candidates whose depth lies within bg_band of
// the farthest one and averages their colours with 1/distance weights;
// provenance 3 marks it. Two passes, O(1) per pixel however large the holes:
//   rows     one warp per row, 512-px steps (16 px per lane, one 16-byte
//            load), nearest-source carries by warp max/min scans, left->right
//            and right->left; stores each hole's left / right distances
//            (int16, -1 = none);
//   columns  32 adjacent columns per CTA, each split into 32 row chunks
//            (one thread each, so every row step of a warp is one coalesced
//            load): chunk boundaries first, then every chunk rescans with the
//            carries from above and below: up / down distances;
//   fill     every hole pixel in parallel from its four distances.
// Prov is only written by the fill pass, so the passes see the composite's
// holes (0) and sources (1, 2) only.

__device__ __forceinline__ bool inpaint_src(uint8_t pv) { return pv == 1 || pv == 2; }

__global__ void k_inpaint_rows(const InpaintParams p) {
    // one warp per row; lane l owns 16 contiguous pixels of each 512-px step
    // (one 16-byte load), carries of the nearest source come from warp scans
    const int lane = threadIdx.x & 31;
    const int y = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (y >= p.H) return;
    const uint8_t *row = p.prov + (size_t)y * p.W;
    int16_t *L = p.dist_l + (size_t)y * p.W, *R = p.dist_r + (size_t)y * p.W;
    const bool vec = (p.W & 15) == 0 && ((uintptr_t)row & 15) == 0;
    const int nsteps = (p.W + 511) / 512;
    auto load16 = [&](int x0, uint8_t (&v)[16]) {
        if (vec && x0 + 15 < p.W) {
            const uint4 q = __ldg(reinterpret_cast<const uint4 *>(row + x0));
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = x0 + k < p.W ? row[x0 + k] : 0;
        }
    };
    int carry = -1;   // last source column left of this step
    for (int st = 0; st < nsteps; ++st) {
        const int x0 = st * 512 + lane * 16;
        uint8_t v[16];
        load16(x0, v);
        int mine = -1;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (x0 + k < p.W && inpaint_src(v[k])) mine = x0 + k;
        // exclusive max-scan over lanes: the last source before this lane
        int incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl = max(incl, t);
        }
        int left = __shfl_up_sync(0xffffffffu, incl, 1);
        left = lane ? max(left, carry) : carry;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int x = x0 + k;
            if (x >= p.W) break;
            if (inpaint_src(v[k])) left = x;
            else L[x] = (left >= 0 && x - left <= p.radius) ? (int16_t)(x - left) : -1;
        }
        carry = max(carry, __shfl_sync(0xffffffffu, incl, 31));
    }
    carry = -1;   // first source column right of this step
    for (int st = nsteps - 1; st >= 0; --st) {
        const int x0 = st * 512 + lane * 16;
        uint8_t v[16];
        load16(x0, v);
        int mine = -1;
#pragma unroll
        for (int k = 15; k >= 0; --k)
            if (x0 + k < p.W && inpaint_src(v[k])) mine = x0 + k;
        // exclusive min-scan from the right (-1 = none)
        int incl = mine;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_down_sync(0xffffffffu, incl, o);
            if (lane + o < 32 && t >= 0 && (incl < 0 || t < incl)) incl = t;
        }
        int right = __shfl_down_sync(0xffffffffu, incl, 1);
        if (lane == 31) right = -1;
        if (right < 0) right = carry;
#pragma unroll
        for (int k = 15; k >= 0; --k) {
            const int x = x0 + k;
            if (x >= p.W) continue;
            if (inpaint_src(v[k])) right = x;
            else R[x] = (right >= 0 && right - x <= p.radius) ? (int16_t)(right - x) : -1;
        }
        const int first = __shfl_sync(0xffffffffu, incl, 0);
        if (first >= 0) carry = first;
    }
}

// the fill of one hole pixel from its four candidates (left, right, up,
// down distances; <= 0 = none), f32, in that order
__device__ __forceinline__ void inpaint_pixel(const InpaintParams &p, size_t i, int dl, int dr,
                                              int du, int dd) {
    const size_t ci[4] = {i - (size_t)(dl > 0 ? dl : 0), i + (size_t)(dr > 0 ? dr : 0),
                          i - (size_t)(du > 0 ? du : 0) * p.W, i + (size_t)(dd > 0 ? dd : 0) * p.W};
    const int cd[4] = {dl, dr, du, dd};
    float zmax = 0.0f, cz[4];
    int n = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        cz[k] = cd[k] > 0 ? p.depth[ci[k]] : 0.0f;
        if (cd[k] > 0) { zmax = fmaxf(zmax, cz[k]); ++n; }
    }
    if (n == 0) return;
    const float zlo = zmax * (float)(1.0 - p.bg_band);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, aw = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        if (cd[k] <= 0 || cz[k] < zlo) continue;
        const float w = 1.0f / (float)cd[k];
        const uint8_t *c = p.rgb + ci[k] * 3;
        a0 += w * c[0];
        a1 += w * c[1];
        a2 += w * c[2];
        aw += w;
    }
    uint8_t *o = p.rgb + i * 3;
    o[0] = (uint8_t)fminf(fmaxf(rintf(a0 / aw), 0.f), 255.f);
    o[1] = (uint8_t)fminf(fmaxf(rintf(a1 / aw), 0.f), 255.f);
    o[2] = (uint8_t)fminf(fmaxf(rintf(a2 / aw), 0.f), 255.f);
    p.prov[i] = 3;
}

// Columns: a 32 x 32 CTA owns 32 adjacent columns; thread (tx, ty) scans row
// chunk ty of column tx. Chunks publish their first / last non-hole rows,
// then each thread rescans its chunk with the carries of the chunks above
// and below, writing the vertical distances and filling its holes.
__global__ void __launch_bounds__(1024) k_inpaint_cols(const InpaintParams p) {
    __shared__ int s_first[32][33], s_last[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int x = blockIdx.x * 32 + tx;
    const int rows = (p.H + 31) / 32;
    const int ya = ty * rows, yb = min(p.H, ya + rows);
    int first = -1, last = -1;
    if (x < p.W)
        for (int y0 = ya; y0 < yb; y0 += 8) {
            uint8_t v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)   // 8 independent loads in flight
                v[k] = y0 + k < yb ? p.prov[(size_t)(y0 + k) * p.W + x] : 0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (y0 + k < yb && inpaint_src(v[k])) {
                    if (first < 0) first = y0 + k;
                    last = y0 + k;
                }
        }
    s_first[ty][tx] = first;
    s_last[ty][tx] = last;
    __syncthreads();
    if (x >= p.W) return;
    int up = -1, down = -1;   // carries: last source above the chunk, first below
    for (int c = ty - 1; c >= 0 && up < 0; --c) up = s_last[c][tx];
    for (int c = ty + 1; c < 32 && down < 0; ++c) down = s_first[c][tx];
    for (int y0 = ya; y0 < yb; y0 += 8) {
        uint8_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = y0 + k < yb ? p.prov[(size_t)(y0 + k) * p.W + x] : 1;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int y = y0 + k;
            if (y >= yb) break;
            if (inpaint_src(v[k])) up = y;
            else p.dist_u[(size_t)y * p.W + x] = (up >= 0 && y - up <= p.radius) ? (int16_t)(y - up) : -1;
        }
    }
    for (int y1 = yb - 1; y1 >= ya; y1 -= 8) {
        uint8_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = y1 - k >= ya ? p.prov[(size_t)(y1 - k) * p.W + x] : 1;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int y = y1 - k;
            if (y < ya) break;
            if (inpaint_src(v[k])) down = y;
            else p.dist_d[(size_t)y * p.W + x] =
                (down >= 0 && down - y <= p.radius) ? (int16_t)(down - y) : -1;
        }
    }
}

// every hole pixel in parallel, from its four distances
__global__ void k_inpaint_fill(const InpaintParams p) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= p.W) return;
    const size_t i = (size_t)y * p.W + x;
    if (p.prov[i] != 0) return;
    inpaint_pixel(p, i, p.dist_l[i], p.dist_r[i], p.dist_u[i], p.dist_d[i]);
}

cudaError_t launch_inpaint(const InpaintParams &p, cudaStream_t s) {
    if (p.W <= 0 || p.H <= 0) return cudaSuccess;
    k_inpaint_rows<<<(p.H + 7) / 8, 256, 0, s>>>(p);
    k_inpaint_cols<<<(p.W + 31) / 32, dim3(32, 32), 0, s>>>(p);
    k_inpaint_fill<<<dim3((p.W + 127) / 128, p.H), 128, 0, s>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// numerics self-test: div_rcp / proj_rint against the correctly rounded path

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ double unit(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

__global__ void k_selftest_div(long long n, uint64_t seed, int mode,
                               unsigned long long *mism) {
    unsigned long long bad = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const uint64_t r1 = splitmix(seed ^ (uint64_t)i * 2 + 1), r2 = splitmix(r1), r3 = splitmix(r2);
        double a, b;
        if (mode == 0) {        // bilinear normalisation: sum(w*c) / sum(w)
            b = 1e-12 + unit(r2) * (1.0 - 1e-12);
            a = unit(r1) * 255.0 * b;
        } else if (mode == 1) { // projection: (f*x) / z
            a = (unit(r1) * 2.0 - 1.0) * 1e7;
            b = exp(log(1e-3) + unit(r2) * log(1e6));
        } else if (mode == 2) { // mix: sum(w*c) / sum(w)
            b = 0.01 + unit(r2) * 1600.0;
            a = unit(r1) * 255.0 * b;
        } else {                // wide log-uniform magnitudes, both signs
            a = exp((unit(r1) * 2.0 - 1.0) * 69.0) * ((r3 & 1) ? -1.0 : 1.0);
            b = exp((unit(r2) * 2.0 - 1.0) * 69.0) * ((r3 & 2) ? -1.0 : 1.0);
        }
        if (mode == 5) {
            if (i < 65536) {
                const float t = __fdiv_rn((float)(uint32_t)i, 1000.0f);
                bad += __float_as_uint(mm_to_m((uint32_t)i)) != __float_as_uint(t);
            }
            continue;
        }
        if (mode <= 3) {
            const double q = div_rcp(a, b, rcp_nr(b));
            const double t = __ddiv_rn(a, b);
            bad += (__double_as_longlong(q) != __double_as_longlong(t)) && !(q == 0.0 && t == 0.0);
        } else {                // K2's filtered rint(f*x/z + c), incl. near-half quotients
            const double f = 500.0 + unit(r1) * 3000.0, z = 0.3 + unit(r2) * 20.0;
            const double c = 100.0 + unit(r3) * 2000.0;
            double u = floor(unit(splitmix(r3)) * 4000.0) - 100.0 + 0.5;  // a half-integer target
            const double jitter = (unit(splitmix(r2 ^ 7)) - 0.5) * ((r3 & 4) ? 1e-9 : 1e-3);
            const double x = ((u + jitter - c) * z) / f;
            const double a1 = proj_rint(f, x, z, c);
            const double a2 = rint(dadd(ddiv(dmul(f, x), z), c));
            // compared as values: rint(-0.3) is -0.0 where the fast path gives
            // +0.0; both convert to the same integer target
            bad += !(a1 == a2);
        }
    }
    if (bad) atomicAdd(mism, bad);
}

cudaError_t launch_selftest_div(long long n, uint64_t seed, int mode, unsigned long long *mism,
                                cudaStream_t s) {
    k_selftest_div<<<148 * 8, 256, 0, s>>>(n, seed, mode, mism);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// standalone mix_layer / composite over caller-provided rasters

__global__ void k_mix(const __grid_constant__ MixParams p) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)p.W * p.H) return;
    double zmin = INFINITY;
    for (int j = 0; j < p.n; ++j)
        if (p.valid[j][i] && p.depth[j][i] < zmin) zmin = p.depth[j][i];
    const double thr = dadd(zmin, dmul(p.band_rel, zmin));
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, ad = 0.0, aw = 0.0;
    for (int j = 0; j < p.n; ++j) {
        // every contribution is added (w = 0 when not participating), exactly
        // like the reference, so NaN/inf colours propagate the same way
        const double w = (p.valid[j][i] && p.depth[j][i] <= thr) ? p.weight[j] : 0.0;
        a0 = dadd(a0, dmul(w, p.color[j][i * 3 + 0]));
        a1 = dadd(a1, dmul(w, p.color[j][i * 3 + 1]));
        a2 = dadd(a2, dmul(w, p.color[j][i * 3 + 2]));
        ad = dadd(ad, dmul(w, p.depth[j][i]));
        aw = dadd(aw, w);
    }
    const bool v = aw > 0.0;
    p.color_out[i * 3 + 0] = v ? ddiv(a0, aw) : 0.0;
    p.color_out[i * 3 + 1] = v ? ddiv(a1, aw) : 0.0;
    p.color_out[i * 3 + 2] = v ? ddiv(a2, aw) : 0.0;
    p.depth_out[i] = v ? ddiv(ad, aw) : 0.0;
    p.valid_out[i] = v ? 1 : 0;
}

cudaError_t launch_mix(const MixParams &p, cudaStream_t s) {
    const size_t n = (size_t)p.W * p.H;
    if (n == 0) return cudaSuccess;
    k_mix<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p);
    return cudaGetLastError();
}

__global__ void k_composite(const double *fg_c, const uint8_t *fg_v, const double *bg_c,
                            const uint8_t *bg_v, size_t n, double h0, double h1, double h2,
                            uint8_t *rgb, uint8_t *prov) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool f = fg_v[i] != 0, b = bg_v[i] != 0;
    const double hole[3] = {h0, h1, h2};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const double v = f ? fg_c[i * 3 + q] : (b ? bg_c[i * 3 + q] : hole[q]);
        rgb[i * 3 + q] = (uint8_t)fmin(fmax(rint(v), 0.0), 255.0);
    }
    if (prov) prov[i] = f ? 2 : (b ? 1 : 0);
}

cudaError_t launch_composite(const double *fg_c, const uint8_t *fg_v, const double *bg_c,
                             const uint8_t *bg_v, int W, int H, const double hole[3],
                             uint8_t *rgb, uint8_t *prov, cudaStream_t s) {
    const size_t n = (size_t)W * H;
    if (n == 0) return cudaSuccess;
    k_composite<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(fg_c, fg_v, bg_c, bg_v, n, hole[0],
                                                           hole[1], hole[2], rgb, prov);
    return cudaGetLastError();
}

}  // namespace fvv
