/*
 * CPU ORACLE (C) — TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of oracle/fvv_oracle.py (itself a restatement of the
 * reference's edge-server path, /root/reference/pkg/src/fvv). Same explicit
 * float64 operation order (compiled with -ffp-contract=off so no FMA is
 * formed), same keyed z-buffer, same rint/true-division/median semantics; the
 * tests check it bit-for-bit against the numpy oracle. Used by bench.py as
 * the timed CPU baseline ("port") and never by the product package.
 *
 *   fo_decode_mm        core.depth_from_millimeters        core.py:260-269
 *   fo_bilateral        depthproc.bilateral_close_holes    depthproc.py:171-224
 *   fo_synthesize_view  synthesis.synthesize_view          synthesis.py:331-362
 *     forward warp      warp_layer stage 1                 synthesis.py:184-205
 *     resolve           splat policy, FG cull, crack median synthesis.py:79-125,207-222
 *     backward fetch    warp_layer stage 3, _bilinear_fetch synthesis.py:128-159,224-247
 *     mix / composite   mix_layer, composite               synthesis.py:261-318
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define VALID 0
#define INVALID 1
#define BACKGROUND 2
#define KEY_EMPTY 0xFFFFFFFFFFFFFFFFull
#define KEY_EXP_MIN (1023 - 16)

typedef struct {
    int32_t width, height;
    double fx, fy, cx, cy;
    double R[9], C[3];
} fo_cam;

typedef struct {
    fo_cam cam;
    const uint8_t *rgb;
    const float *live_depth;
    const uint8_t *live_validity;
    const float *bg_depth;
    const uint8_t *bg_validity;
    double weight;
} fo_ref;

typedef struct {
    int32_t splat_radius, crack_fill_window;
    double depth_band_rel;
    uint8_t hole_color[3];
} fo_cfg;

/* ------------------------------------------------------------------------ */

void fo_decode_mm(const uint16_t *mm, const uint8_t *val_in, int W, int H, float *depth,
                  uint8_t *val) {
    const long n = (long)W * H;
    for (long i = 0; i < n; ++i) {
        uint8_t v = val_in ? val_in[i] : VALID;
        if (v == VALID && mm[i] == 0) v = INVALID;
        val[i] = v;
        depth[i] = (v == VALID) ? (float)mm[i] / 1000.0f : 0.0f;
    }
}

/* returns the number of Invalid input pixels. range_w (may be NULL = libm
 * exp) holds exp(-d2 * inv_2sr) for every integer d2 in [0, 3*255^2]: the
 * Python wrapper passes the np.exp values the reference computes
 * (depthproc.py:212), since numpy's SIMD exp and libm's differ in the last bit
 * on some arguments. */
long fo_bilateral(const float *d, const uint8_t *v, const uint8_t *rgb, int W, int H, int R,
                  double sigma_s, double sigma_r, int min_valid, float *out_d, uint8_t *out_v,
                  const double *range_w) {
    const long n = (long)W * H;
    memcpy(out_d, d, n * sizeof(float));
    memcpy(out_v, v, n);
    long holes = 0;
    const double inv_2ss = 1.0 / (2.0 * (sigma_s * sigma_s));
    const double inv_2sr = 1.0 / (2.0 * (sigma_r * sigma_r));
    double sw[9][9];
    for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx)
            sw[dy + R][dx + R] = exp((double)(-(dy * dy + dx * dx)) * inv_2ss);
    for (int y = 0; y < H; ++y) {
        for (int x = 0; x < W; ++x) {
            const long i = (long)y * W + x;
            if (v[i] != INVALID) continue;
            ++holes;
            const double g0 = rgb[i * 3], g1 = rgb[i * 3 + 1], g2 = rgb[i * 3 + 2];
            double num = 0.0, den = 0.0;
            int cnt = 0;
            for (int dy = -R; dy <= R; ++dy) {
                for (int dx = -R; dx <= R; ++dx) {
                    if (dy == 0 && dx == 0) continue;
                    const int ny = y + dy, nx = x + dx;
                    if (ny < 0 || ny >= H || nx < 0 || nx >= W) continue;
                    const long j = (long)ny * W + nx;
                    if (v[j] != VALID) continue;
                    const double e0 = g0 - rgb[j * 3], e1 = g1 - rgb[j * 3 + 1],
                                 e2 = g2 - rgb[j * 3 + 2];
                    const double d2 = (e0 * e0 + e1 * e1) + e2 * e2;
                    const double w = sw[dy + R][dx + R] *
                                     (range_w ? range_w[(long)d2] : exp(-d2 * inv_2sr));
                    num += w * (double)d[j];
                    den += w;
                    ++cnt;
                }
            }
            if (cnt >= min_valid && den > 0.0) {
                out_d[i] = (float)(num / den);
                out_v[i] = VALID;
            }
        }
    }
    return holes;
}

/* ------------------------------------------------------------------------ */

static int index_bits(long n) {
    int b = 0;
    long v = n - 1;
    while (v > 0) { ++b; v >>= 1; }
    return b < 1 ? 1 : b;
}

static uint64_t zkey(double z, uint64_t idx, int b) {
    uint64_t bits;
    memcpy(&bits, &z, 8);
    const int e = (int)((bits >> 52) & 0x7FF);
    const int m = 52 - b;
    uint64_t zc;
    if (e < KEY_EXP_MIN) zc = 0;
    else if (e > KEY_EXP_MIN + 31) zc = (1ull << (5 + m)) - 1;
    else zc = ((uint64_t)(e - KEY_EXP_MIN) << m) | ((bits & ((1ull << 52) - 1)) >> (52 - m));
    return (zc << b) | idx;
}

/* src camera -> dst camera motion, composed once per pair in a fixed order
 * (oracle relative_pose): M = R_t R_s^T, tt = R_t (C_s - C_t). */
typedef struct {
    double M[9], t[3];
} fo_rel;

static fo_rel relative_pose(const fo_cam *s, const fo_cam *t) {
    fo_rel r;
    const double *Rs = s->R, *Rt = t->R;
    const double dc[3] = {s->C[0] - t->C[0], s->C[1] - t->C[1], s->C[2] - t->C[2]};
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j)
            r.M[3 * i + j] = (Rt[3 * i] * Rs[3 * j] + Rt[3 * i + 1] * Rs[3 * j + 1]) +
                             Rt[3 * i + 2] * Rs[3 * j + 2];
        r.t[i] = (Rt[3 * i] * dc[0] + Rt[3 * i + 1] * dc[1]) + Rt[3 * i + 2] * dc[2];
    }
    return r;
}

/* (x, y, z) in the target camera of the source ray (rx, ry, 1) at depth d:
 * per coordinate ((M_i0 rx) + ((M_i1 ry) + M_i2)) d + t_i (oracle transfer) */
static void transfer(const fo_rel *m, double rx, double ry, double d, double *x, double *y,
                     double *z) {
    const double *M = m->M;
    *x = (M[0] * rx + (M[1] * ry + M[2])) * d + m->t[0];
    *y = (M[3] * rx + (M[4] * ry + M[5])) * d + m->t[1];
    *z = (M[6] * rx + (M[7] * ry + M[8])) * d + m->t[2];
}

typedef struct {
    uint64_t *canvas; /* (H+2r) x (W+2r) */
    double *zsrc;     /* per source pixel */
    int b;
} warp_t;

static void forward_warp(const float *depth, const uint8_t *valid_src, const fo_cam *src,
                         const fo_cam *dst, int r, warp_t *w) {
    const int Ws = src->width, Hs = src->height, Wd = dst->width, Hd = dst->height;
    const int Wc = Wd + 2 * r;
    const long nc = (long)Wc * (Hd + 2 * r);
    for (long i = 0; i < nc; ++i) w->canvas[i] = KEY_EMPTY;
    w->b = index_bits((long)Ws * Hs);
    const fo_rel m = relative_pose(src, dst);
    for (int v = 0; v < Hs; ++v) {
        const double ry = ((double)v - src->cy) / src->fy;
        for (int u = 0; u < Ws; ++u) {
            const long i = (long)v * Ws + u;
            w->zsrc[i] = 0.0;
            if (valid_src[i] != VALID) continue;
            const double d = (double)depth[i];
            const double rx = ((double)u - src->cx) / src->fx;
            double x, y, z;
            transfer(&m, rx, ry, d, &x, &y, &z);
            w->zsrc[i] = z;
            if (!(z > 0.0)) continue;
            const double ui = rint((dst->fx * x) / z + dst->cx);
            const double vi = rint((dst->fy * y) / z + dst->cy);
            if (!(ui >= -r && ui < Wd + r && vi >= -r && vi < Hd + r)) continue;
            const long cell = ((long)vi + r) * Wc + ((long)ui + r);
            const uint64_t key = zkey(z, (uint64_t)i, w->b);
            if (key < w->canvas[cell]) w->canvas[cell] = key;
        }
    }
}

static double key_z(const warp_t *w, uint64_t key) {
    return w->zsrc[key & ((1ull << w->b) - 1)];
}

static int cmp_double(const void *a, const void *b) {
    const double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* zbuf: f64 with INFINITY = uncovered */
static void resolve_zbuf(const warp_t *w, int Wd, int Hd, int r, int layer_fg, int window,
                         double *zpre, double *zbuf) {
    const int Wc = Wd + 2 * r;
    for (int y = 0; y < Hd; ++y) {
        for (int x = 0; x < Wd; ++x) {
            const uint64_t cen = w->canvas[(long)(y + r) * Wc + (x + r)];
            uint64_t win = cen;
            if (cen == KEY_EMPTY) {
                uint64_t m = KEY_EMPTY;
                for (int dy = -r; dy <= r; ++dy)
                    for (int dx = -r; dx <= r; ++dx)
                        if (dy || dx) {
                            const uint64_t k = w->canvas[(long)(y + r + dy) * Wc + (x + r + dx)];
                            if (k < m) m = k;
                        }
                win = m;
                if (m != KEY_EMPTY && layer_fg) {
                    int cnt = 0;
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (!(dy || dx)) continue;
                            const int ny = y + dy, nx = x + dx;
                            if (ny < 0 || ny >= Hd || nx < 0 || nx >= Wd) continue;
                            cnt += w->canvas[(long)(ny + r) * Wc + (nx + r)] != KEY_EMPTY;
                        }
                    if (cnt < 5) win = KEY_EMPTY;
                }
            }
            zpre[(long)y * Wd + x] = win == KEY_EMPTY ? INFINITY : key_z(w, win);
        }
    }
    const int rc = window / 2, need = window * window / 2 + 1;
    double vals[64];
    for (int y = 0; y < Hd; ++y) {
        for (int x = 0; x < Wd; ++x) {
            const long i = (long)y * Wd + x;
            double z = zpre[i];
            if (!(z < INFINITY) && rc > 0) {
                int n = 0;
                for (int dy = -rc; dy <= rc; ++dy)
                    for (int dx = -rc; dx <= rc; ++dx) {
                        if (!(dy || dx)) continue;
                        const int ny = y + dy, nx = x + dx;
                        if (ny < 0 || ny >= Hd || nx < 0 || nx >= Wd) continue;
                        const double zz = zpre[(long)ny * Wd + nx];
                        if (zz < INFINITY) vals[n++] = zz;
                    }
                if (n >= need) {
                    qsort(vals, n, sizeof(double), cmp_double);
                    z = (n & 1) ? vals[(n - 1) / 2] : (vals[(n - 1) / 2] + vals[n / 2]) / 2;
                }
            }
            zbuf[i] = z;
        }
    }
}

/* colour + depth of one contribution at every covered pixel */
static void backward_fetch(const double *zbuf, const fo_cam *src, const fo_cam *dst,
                           const uint8_t *rgb, const uint8_t *cvalid_val, uint8_t cvalid_code,
                           double *col, double *dep, uint8_t *ok_out) {
    const int Wd = dst->width, Hd = dst->height, Ws = src->width, Hs = src->height;
    const fo_rel m = relative_pose(dst, src);
    for (int y = 0; y < Hd; ++y) {
        const double ry = ((double)y - dst->cy) / dst->fy;
        for (int x = 0; x < Wd; ++x) {
            const long i = (long)y * Wd + x;
            const double z = zbuf[i];
            col[i * 3] = col[i * 3 + 1] = col[i * 3 + 2] = 0.0;
            dep[i] = 0.0;
            ok_out[i] = 0;
            if (!(z < INFINITY)) continue;
            const double rx = ((double)x - dst->cx) / dst->fx;
            double xs, ys, zs;
            transfer(&m, rx, ry, z, &xs, &ys, &zs);
            if (!(zs > 0.0)) continue;
            const double us = (src->fx * xs) / zs + src->cx;
            const double vs = (src->fy * ys) / zs + src->cy;
            if (!(us >= -0.5 && us <= Ws - 0.5 && vs >= -0.5 && vs <= Hs - 0.5)) continue;
            const double uc = fmin(fmax(us, 0.0), (double)(Ws - 1));
            const double vc = fmin(fmax(vs, 0.0), (double)(Hs - 1));
            const double u0 = floor(uc), v0 = floor(vc);
            const int iu = (int)u0, iv = (int)v0;
            const double fu = uc - u0, fv = vc - v0;
            const double wt[4] = {(1 - fu) * (1 - fv), fu * (1 - fv), (1 - fu) * fv, fu * fv};
            const int du[4] = {0, 1, 0, 1}, dv[4] = {0, 0, 1, 1};
            double c0 = 0.0, c1 = 0.0, c2 = 0.0, s = 0.0;
            for (int q = 0; q < 4; ++q) {
                const int uu = iu + du[q], vv = iv + dv[q];
                if (uu >= Ws || vv >= Hs) continue;
                const long j = (long)vv * Ws + uu;
                if (cvalid_val[j] != cvalid_code) continue;
                c0 += wt[q] * (double)rgb[j * 3];
                c1 += wt[q] * (double)rgb[j * 3 + 1];
                c2 += wt[q] * (double)rgb[j * 3 + 2];
                s += wt[q];
            }
            if (!(s > 1e-12)) continue;
            col[i * 3] = c0 / s;
            col[i * 3 + 1] = c1 / s;
            col[i * 3 + 2] = c2 / s;
            dep[i] = z;
            ok_out[i] = 1;
        }
    }
}

static void mix_layer(int n, double *const *col, double *const *dep, uint8_t *const *ok,
                      const double *weight, long npx, double band_rel, double *mcol,
                      uint8_t *mvalid) {
    for (long i = 0; i < npx; ++i) {
        double zmin = INFINITY;
        for (int k = 0; k < n; ++k)
            if (ok[k][i] && dep[k][i] < zmin) zmin = dep[k][i];
        const double thr = zmin + band_rel * zmin;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, aw = 0.0;
        for (int k = 0; k < n; ++k) {
            if (!(ok[k][i] && dep[k][i] <= thr)) continue;
            const double w = weight[k];
            a0 += w * col[k][i * 3];
            a1 += w * col[k][i * 3 + 1];
            a2 += w * col[k][i * 3 + 2];
            aw += w;
        }
        mvalid[i] = aw > 0.0;
        mcol[i * 3] = mvalid[i] ? a0 / aw : 0.0;
        mcol[i * 3 + 1] = mvalid[i] ? a1 / aw : 0.0;
        mcol[i * 3 + 2] = mvalid[i] ? a2 / aw : 0.0;
    }
}

static uint8_t to_u8(double v) { return (uint8_t)fmin(fmax(rint(v), 0.0), 255.0); }

int fo_synthesize_view(const fo_cam *virt, const fo_ref *refs, int n, const fo_cfg *cfg,
                       uint8_t *rgb_out, uint8_t *prov_out) {
    if (n < 1) return 1;
    const int Wd = virt->width, Hd = virt->height, r = cfg->splat_radius;
    const long npx = (long)Wd * Hd;
    long maxs = 0;
    for (int k = 0; k < n; ++k) {
        const long s = (long)refs[k].cam.width * refs[k].cam.height;
        if (s > maxs) maxs = s;
    }
    warp_t w;
    w.canvas = malloc(sizeof(uint64_t) * (size_t)(Wd + 2 * r) * (Hd + 2 * r));
    w.zsrc = malloc(sizeof(double) * maxs);
    double *zpre = malloc(sizeof(double) * npx), *zbuf = malloc(sizeof(double) * npx);
    double *col[32], *dep[32];
    uint8_t *ok[32];
    double wts[32];
    for (int k = 0; k < 2 * n; ++k) {
        col[k] = malloc(sizeof(double) * 3 * npx);
        dep[k] = malloc(sizeof(double) * npx);
        ok[k] = malloc(npx);
    }
    for (int L = 0; L < 2; ++L) {
        for (int j = 0; j < n; ++j) {
            const fo_ref *f = &refs[j];
            const int k = L * n + j;
            const float *d = L == 0 ? f->live_depth : f->bg_depth;
            const uint8_t *vv = L == 0 ? f->live_validity : f->bg_validity;
            forward_warp(d, vv, &f->cam, virt, r, &w);
            resolve_zbuf(&w, Wd, Hd, r, L == 0, cfg->crack_fill_window, zpre, zbuf);
            backward_fetch(zbuf, &f->cam, virt, f->rgb, f->live_validity,
                           L == 0 ? VALID : BACKGROUND, col[k], dep[k], ok[k]);
            wts[k] = f->weight;
        }
    }
    double *fc = malloc(sizeof(double) * 3 * npx), *bc = malloc(sizeof(double) * 3 * npx);
    uint8_t *fvld = malloc(npx), *bvld = malloc(npx);
    mix_layer(n, col, dep, ok, wts, npx, cfg->depth_band_rel, fc, fvld);
    mix_layer(n, col + n, dep + n, ok + n, wts + n, npx, cfg->depth_band_rel, bc, bvld);
    for (long i = 0; i < npx; ++i) {
        for (int q = 0; q < 3; ++q) {
            const double v = fvld[i] ? fc[i * 3 + q] : (bvld[i] ? bc[i * 3 + q]
                                                                 : (double)cfg->hole_color[q]);
            rgb_out[i * 3 + q] = to_u8(v);
        }
        if (prov_out) prov_out[i] = fvld[i] ? 2 : (bvld[i] ? 1 : 0);
    }
    for (int k = 0; k < 2 * n; ++k) {
        free(col[k]);
        free(dep[k]);
        free(ok[k]);
    }
    free(fc); free(bc); free(fvld); free(bvld);
    free(zpre); free(zbuf); free(w.canvas); free(w.zsrc);
    return 0;
}
