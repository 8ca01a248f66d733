// sm_100a kernels of the edge-server view-synthesis path.
//
//   K0+K1+ingest  k_preprocess   decode (mm / YUV420-12 / f32), joint-bilateral
//                                hole fill, pack RGB+flags texels, warp depth
//   K2            k_forward_warp forward 3-D warp, one 64-bit atomicMin per
//                                source pixel into a padded keyed z canvas
//   K3            k_resolve      per 32x8 target tile and per contribution:
//                                splat ring + FG cull + crack median in shared
//                                memory, f64 backward projection, masked
//                                bilinear fetch; then the two layer mixes and
//                                the FG-over-BG composite -> RGB8 + provenance
//
// Each kernel cites the reference lines it replaces; the numerics contract is
// in fvv_common.cuh and oracle/fvv_oracle.py.

#include <cfloat>
#include <cmath>

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

constexpr int PX = 32, PY = 8, PMAXR = 4;

// 12-bit code at (iy, ix) from the folded/interleaved YUV420 raster
// (depthcodec.py:154-177, 213-222): MSB nibble from U (even rows) or V (odd
// rows), A = odd bit positions for even columns, B = even positions for odd
// columns; LSB mirrored when the MSB is odd.
__device__ __forceinline__ uint32_t yuv_code(const PreprocParams &p, int iy, int ix) {
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

// Decoded (depth, validity) of pixel (iy, ix), per source format.
__device__ __forceinline__ void load_depth(const PreprocParams &p, int iy, int ix, float &z,
                                           uint8_t &val, uint32_t *code) {
    const size_t i = (size_t)iy * p.W + ix;
    if (p.src == kSrcMM) {
        // core.depth_from_millimeters (core.py:260-269): fp32 TRUE division
        const uint16_t mm = p.mm[i];
        val = p.validity ? p.validity[i] : (uint8_t)FVV_VALID;
        if (val == FVV_VALID && mm == 0) val = FVV_INVALID;
        z = (val == FVV_VALID) ? __fdiv_rn((float)mm, 1000.0f) : 0.0f;
    } else if (p.src == kSrcYUV || p.src == kSrcCodes) {
        // depthcodec.dequantize12 / dequantize_codes (depthcodec.py:113-138)
        const uint32_t c = p.src == kSrcYUV ? yuv_code(p, iy, ix) : (uint32_t)p.codes[i];
        if (code) *code = c;
        if (c < 2) {
            val = (c == 0) ? (uint8_t)FVV_BACKGROUND : (uint8_t)FVV_INVALID;
            z = 0.0f;
        } else {
            val = FVV_VALID;
            const double frac = ddiv((double)c - 2.0, 4093.0);
            z = __double2float_rn(ddiv(1.0, dadd(dmul(frac, p.inv_span), p.inv_zf)));
        }
    } else {
        z = p.depth[i];
        val = p.validity[i];
    }
}

__global__ void __launch_bounds__(256) k_preprocess(const __grid_constant__ PreprocParams p) {
    __shared__ float sz[(PY + 2 * PMAXR) * (PX + 2 * PMAXR)];
    __shared__ uint8_t sv[(PY + 2 * PMAXR) * (PX + 2 * PMAXR)];
    __shared__ uchar4 sg[(PY + 2 * PMAXR) * (PX + 2 * PMAXR)];
    __shared__ int s_holes;

    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int x0 = blockIdx.x * PX, y0 = blockIdx.y * PY;
    const int R = p.radius;
    const int SC = PX + 2 * R, SR = PY + 2 * R;
    if (tid == 0) s_holes = 0;

    if (R > 0) {
        for (int i = tid; i < SR * SC; i += 256) {
            const int qy = y0 - R + i / SC, qx = x0 - R + i % SC;
            float z = 0.0f;
            uint8_t val = 0xFF;  // outside the image: never a valid neighbour
            uchar4 g = make_uchar4(0, 0, 0, 0);
            if (qy >= 0 && qy < p.H && qx >= 0 && qx < p.W) {
                load_depth(p, qy, qx, z, val, nullptr);
                const uint8_t *c = p.rgb + ((size_t)qy * p.W + qx) * 3;
                g = make_uchar4(c[0], c[1], c[2], 0);
            }
            sz[i] = z;
            sv[i] = val;
            sg[i] = g;
        }
        __syncthreads();
    }

    const int ix = x0 + tx, iy = y0 + ty;
    int hole = 0;
    if (ix < p.W && iy < p.H) {
        const size_t i = (size_t)iy * p.W + ix;
        float z;
        uint8_t val;
        uint32_t code = 0;
        uchar4 g;
        if (R > 0) {
            const int si = (ty + R) * SC + tx + R;
            z = sz[si];
            val = sv[si];
            g = sg[si];
            if (p.src == kSrcYUV && p.codes_out) code = yuv_code(p, iy, ix);
        } else {
            load_depth(p, iy, ix, z, val, &code);
            const uint8_t *c = p.rgb ? p.rgb + i * 3 : nullptr;
            g = c ? make_uchar4(c[0], c[1], c[2], 0) : make_uchar4(0, 0, 0, 0);
        }
        if (val == FVV_INVALID) {
            hole = 1;
            if (R > 0) {
                // depthproc.bilateral_close_holes (depthproc.py:196-222): 24 taps
                // in dy-major order; w = exp_s(dy,dx) * exp(-|g - g_nb|^2 / (2 sr^2))
                const double g0 = g.x, g1 = g.y, g2 = g.z;
                double num = 0.0, den = 0.0;
                int cnt = 0;
                for (int dy = -R; dy <= R; ++dy) {
                    for (int dx = -R; dx <= R; ++dx) {
                        if (dy == 0 && dx == 0) continue;
                        const int ni = (ty + R + dy) * SC + tx + R + dx;
                        if (sv[ni] != FVV_VALID) continue;
                        const uchar4 n = sg[ni];
                        const double e0 = dsub(g0, (double)n.x), e1 = dsub(g1, (double)n.y),
                                     e2 = dsub(g2, (double)n.z);
                        const double d2 = dadd(dadd(dmul(e0, e0), dmul(e1, e1)), dmul(e2, e2));
                        const double w = dmul(p.sw[dy + R][dx + R], exp(dmul(-d2, p.inv_2sr)));
                        num = dadd(num, dmul(w, (double)sz[ni]));
                        den = dadd(den, w);
                        ++cnt;
                    }
                }
                if (cnt >= p.min_valid && den > 0.0) {
                    z = __double2float_rn(ddiv(num, den));
                    val = FVV_VALID;
                }
            }
        }
        if (p.texel) {
            uint32_t flags;
            if (p.color_valid) flags = p.color_valid[i] ? kFlagLiveValid : 0u;
            else flags = (val == FVV_VALID ? kFlagLiveValid : 0u) |
                         (val == FVV_BACKGROUND ? kFlagLiveBackground : 0u);
            p.texel[i] = (uint32_t)g.x | ((uint32_t)g.y << 8) | ((uint32_t)g.z << 16) | (flags << 24);
        }
        if (p.warp_depth) p.warp_depth[i] = (val == FVV_VALID) ? z : 0.0f;
        if (p.depth_out) p.depth_out[i] = z;
        if (p.validity_out) p.validity_out[i] = val;
        if (p.codes_out) p.codes_out[i] = (uint16_t)code;
    }
    if (p.n_holes) {
        const unsigned m = __ballot_sync(0xffffffffu, hole);
        __syncthreads();
        if ((tid & 31) == 0 && m) atomicAdd(&s_holes, __popc(m));
        __syncthreads();
        if (tid == 0 && s_holes) atomicAdd(p.n_holes, s_holes);
    }
}

cudaError_t launch_preprocess(const PreprocParams &p, cudaStream_t s) {
    dim3 grid((p.W + PX - 1) / PX, (p.H + PY - 1) / PY);
    k_preprocess<<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K2: forward warp (synthesis.py:188-205)
//
// One thread per source pixel: unproject with the f32 depth (as f64), move
// to the virtual camera, project, rint (np.round, half-even) and scatter ONE
// key into the canvas padded by r. The 9-way splat of the reference becomes
// the ring min in K3 (verified equivalent).

__global__ void __launch_bounds__(256) k_forward_warp(const __grid_constant__ WarpParams p) {
    const WarpContrib &c = p.c[blockIdx.y];
    const int Ws = c.src.W;
    const long long N = (long long)Ws * c.src.H;
    const int r = p.r;
    const int Wd = p.dst.W, Hd = p.dst.H, Wc = Wd + 2 * r;
    const double ulo = -(double)r, uhi = (double)(Wd + r), vhi = (double)(Hd + r);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x) {
        const float d = __ldcs(c.depth + i);
        if (!(d > 0.0f)) continue;
        const int sv = (int)(i / Ws), su = (int)(i - (long long)sv * Ws);
        const double dd = (double)d;
        double x, y, z;
        transfer(c.src, p.dst, dmul(__ldg(c.rx + su), dd), dmul(__ldg(c.ry + sv), dd), dd, x, y, z);
        if (!(z > 0.0)) continue;
        const double ur = rint(proj(p.dst.fx, x, z, p.dst.cx));
        const double vr = rint(proj(p.dst.fy, y, z, p.dst.cy));
        if (!(ur >= ulo && ur < uhi && vr >= ulo && vr < vhi)) continue;
        const size_t cell = (size_t)((int)vr + r) * Wc + (size_t)((int)ur + r);
        atomicMin((unsigned long long *)(c.canvas + cell),
                  (unsigned long long)(p.gen_hi | zkey(z, (uint32_t)i, c.b)));
    }
}

cudaError_t launch_forward_warp(const WarpParams &p, long long max_src_pixels, cudaStream_t s) {
    if (p.n == 0) return cudaSuccess;
    long long blocks = (max_src_pixels + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    dim3 grid((unsigned)blocks, (unsigned)p.n);
    k_forward_warp<<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K3: resolve + backward fetch + mix + composite

constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int MAXH = 5;   // max(r,1) + window/2 with r <= 3, window <= 5
constexpr int MAXRC = 2;  // window/2
constexpr int KMAX = (TY + 2 * MAXH) * (TX + 2 * MAXH);
constexpr int BMAX = (TY + 2 * MAXRC) * (TX + 2 * MAXRC);

size_t resolve_smem_bytes(int maxr) { return (size_t)maxr * 4 * NT * sizeof(double); }

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

template <int MAXR>
__global__ void __launch_bounds__(NT) k_resolve(const __grid_constant__ ResolveParams p) {
    __shared__ uint64_t sk[KMAX];
    __shared__ double sz[BMAX];
    __shared__ int swin[BMAX];
    __shared__ uint8_t sst[BMAX];
    extern __shared__ double sres[];  // [MAXR][4][NT]: colour rgb, depth

    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const DevCam &dst = p.dst;
    const int Wd = dst.W, Hd = dst.H;
    const int ix = x0 + tx, iy = y0 + ty;
    const bool inimg = ix < Wd && iy < Hd;
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
                    const uint64_t v = c.canvas[(size_t)cy * Wc + cx];
                    if ((v >> kGenShift) == p.gen) { key = v; any = 1; }
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
                            // exact f64 z of the winner, recomputed from its index
                            const uint32_t idx = (uint32_t)(w & ((1ull << c.b) - 1));
                            const int sv = (int)(idx / (uint32_t)c.src.W);
                            const int su = (int)(idx - (uint32_t)sv * c.src.W);
                            const double d = (double)__ldg(c.depth + idx);
                            zq = transfer_z(c.src, dst, dmul(__ldg(c.rx + su), d),
                                            dmul(__ldg(c.ry + sv), d), d);
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
                transfer(dst, c.src, dmul(rxd, z), dmul(ryd, z), z, xs, ys, zs);
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
                sres[(j * 4 + 0) * NT + tid] = c0;
                sres[(j * 4 + 1) * NT + tid] = c1;
                sres[(j * 4 + 2) * NT + tid] = c2;
                sres[(j * 4 + 3) * NT + tid] = zd;
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
            const double zj = sres[(j * 4 + 3) * NT + tid];
            if (((vmask >> j) & 1u) && zj < zmin) zmin = zj;
        }
        const double thr = dadd(zmin, dmul(p.band_rel, zmin));
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, ad = 0.0, aw = 0.0;
        for (int j = 0; j < n && j < MAXR; ++j) {
            const double zj = sres[(j * 4 + 3) * NT + tid];
            if (((vmask >> j) & 1u) && zj <= thr) {
                const double w = p.c[k0 + j].weight;
                a0 = dadd(a0, dmul(w, sres[(j * 4 + 0) * NT + tid]));
                a1 = dadd(a1, dmul(w, sres[(j * 4 + 1) * NT + tid]));
                a2 = dadd(a2, dmul(w, sres[(j * 4 + 2) * NT + tid]));
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
    }
}

cudaError_t launch_resolve(const ResolveParams &p, cudaStream_t s) {
    dim3 grid((p.dst.W + TX - 1) / TX, (p.dst.H + TY - 1) / TY);
    const int maxn = p.n_fg > p.n_bg ? p.n_fg : p.n_bg;
    if (maxn <= 4) {
        k_resolve<4><<<grid, NT, resolve_smem_bytes(4), s>>>(p);
    } else {
        static bool attr_set = false;
        if (!attr_set) {
            cudaFuncSetAttribute(k_resolve<FVV_MAX_REFS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)resolve_smem_bytes(FVV_MAX_REFS));
            attr_set = true;
        }
        k_resolve<FVV_MAX_REFS><<<grid, NT, resolve_smem_bytes(FVV_MAX_REFS), s>>>(p);
    }
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
