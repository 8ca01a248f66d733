// MED + Golomb-Rice lossless plane codec on sm_100a.
//
// The reference compresses each 8-bit plane of the 12-bit depth YUV420 raster
// (depthcodec.py:281-409): LOCO-I median (MED) prediction, zig-zag residuals,
// one Rice parameter k per plane (the cheapest of 0..14), an MSB-first bit
// stream, then zlib when that is smaller (the zlib step stays on the host, as
// the reference's zlib call). Both directions are sequential in the reference
// (numba loops); here:
//
//   encode  k_med_zz      residual + zig-zag per pixel, per-k bit costs
//           k_rice_lens   symbol lengths q + 1 + k, per-block sums
//           k_scan_blocks exclusive scan of the block sums (one CTA)
//           k_rice_write  per-block scan, each symbol ORs its k+1 bits into
//                         the zeroed stream (its q leading zeros are implicit)
//   decode  k_rice_sync   chunked speculative decoding: every 256-bit chunk
//                         decodes from an entry guess to its exit; rounds
//                         re-decode chunks whose entry (= previous chunk's
//                         exit) changed until none does. Rice codes
//                         resynchronise within a few symbols, so 2-3 rounds
//                         settle an exact symbol segmentation
//           k_scan_blocks symbol base of every chunk
//           k_rice_emit   each chunk writes its residuals
//           k_med_rebuild the MED recurrence as a wavefront: one CTA per
//                         plane, a warp per 32-row strip with lane = row and
//                         columns skewed by lane; strips hand their last row
//                         to the next strip's warp through shared memory
//           k_adler       adler32 of the rebuilt plane (zlib.adler32 check)

#include <cstdint>
#include <cstdio>

#include "fvv_codec.cuh"

#ifdef FVV_CODEC_TRACE
#define TRACE_EV(name)                                                       \
    do {                                                                     \
        cudaEvent_t e_; cudaEventCreate(&e_); cudaEventRecord(e_, s);        \
        cudaEventSynchronize(e_);                                            \
        float ms_ = 0; cudaEventElapsedTime(&ms_, t0_, e_);                  \
        fprintf(stderr, "[codec] %-10s %8.1f us\n", name, ms_ * 1e3f);       \
    } while (0)
#else
#define TRACE_EV(name) do { } while (0)
#endif

namespace fvv {

// ---------------------------------------------------------------------------
// encode

// LOCO-I median predictor (depthcodec.py:281-298): a left, b up, c up-left,
// 0 outside the plane
__device__ __forceinline__ int med(int a, int b, int c) {
    const int mx = a > b ? a : b, mn = a < b ? a : b;
    return c >= mx ? mn : (c <= mn ? mx : a + b - c);
}

__global__ void k_med_zz(const uint8_t *x, int W, int H, uint16_t *zz,
                         unsigned long long *costs) {
    __shared__ unsigned long long s_cost[kRiceKMax + 1];
    if (threadIdx.x <= kRiceKMax) s_cost[threadIdx.x] = 0;
    __syncthreads();
    const long long n = (long long)W * H;
    unsigned long long c[kRiceKMax + 1];
#pragma unroll
    for (int k = 0; k <= kRiceKMax; ++k) c[k] = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / W), col = (int)(i - (long long)row * W);
        const int a = col > 0 ? x[i - 1] : 0;
        const int b = row > 0 ? x[i - W] : 0;
        const int cc = (row > 0 && col > 0) ? x[i - W - 1] : 0;
        const int r = (int)x[i] - med(a, b, cc);
        const int z = r >= 0 ? 2 * r : -2 * r - 1;  // depthcodec.py:379
        zz[i] = (uint16_t)z;
#pragma unroll
        for (int k = 0; k <= kRiceKMax; ++k) c[k] += (unsigned)((z >> k) + 1 + k);
    }
#pragma unroll
    for (int k = 0; k <= kRiceKMax; ++k) {
        unsigned long long v = c[k];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_cost[k], v);
    }
    __syncthreads();
    if (threadIdx.x <= kRiceKMax && s_cost[threadIdx.x])
        atomicAdd(&costs[threadIdx.x], s_cost[threadIdx.x]);
}

constexpr int kScanB = 1024;  // symbols per scan block (256 threads x 4)

__global__ void k_rice_lens(const uint16_t *zz, long long n, int k,
                            unsigned long long *block_sum) {
    const long long b0 = (long long)blockIdx.x * kScanB;
    unsigned long long s = 0;
    for (int t = threadIdx.x; t < kScanB; t += blockDim.x) {
        const long long i = b0 + t;
        if (i < n) s += (unsigned)((zz[i] >> k) + 1 + k);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ unsigned long long ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
        block_sum[blockIdx.x] = t;
    }
}

// exclusive scan of v[0..n) in place (one CTA of 1024 threads); total in *total
__global__ void __launch_bounds__(1024) k_scan_blocks(unsigned long long *v, long long n,
                                                      unsigned long long *total) {
    __shared__ unsigned long long ws[32];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (long long base = 0; base < n; base += 1024) {
        const long long i = base + threadIdx.x;
        const unsigned long long x = i < n ? v[i] : 0;
        unsigned long long inc = x;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) ws[w] = inc;
        __syncthreads();
        if (w == 0) {
            unsigned long long s = ws[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            ws[lane] = s;  // inclusive over warps
        }
        __syncthreads();
        const unsigned long long before = carry + (w ? ws[w - 1] : 0) + inc - x;
        if (i < n) v[i] = before;
        __syncthreads();
        if (threadIdx.x == 1023) carry = before + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Symbol i = q zeros, a one, then the k low bits of zz MSB-first
// (depthcodec.py:319-334). The stream is zeroed beforehand, so a symbol only
// ORs its k+1 trailing bits into at most two big-endian 32-bit words.
__global__ void k_rice_write(const uint16_t *zz, long long n, int k,
                             const unsigned long long *block_off, uint32_t *words) {
    __shared__ unsigned long long ws[8];
    const long long b0 = (long long)blockIdx.x * kScanB;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // 4 consecutive symbols per thread
    unsigned len[4];
    unsigned tsum = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const long long i = b0 + threadIdx.x * 4 + t;
        len[t] = i < n ? (unsigned)((zz[i] >> k) + 1 + k) : 0u;
        tsum += len[t];
    }
    unsigned long long inc = tsum;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    unsigned long long pre = 0;
    for (int q = 0; q < w; ++q) pre += ws[q];
    unsigned long long off = block_off[blockIdx.x] + pre + inc - tsum;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const long long i = b0 + threadIdx.x * 4 + t;
        if (i < n) {
            const unsigned z = zz[i];
            const unsigned q = z >> k;
            const unsigned long long p = off + q;  // the terminating one
            const unsigned long long v = (1ull << k) | (z & ((1u << k) - 1u));  // k+1 bits
            const unsigned sh = (unsigned)(p & 31);
            const unsigned long long be = v << (64 - (k + 1) - sh);
            const long long wi = (long long)(p >> 5);
            atomicOr(words + wi, bswap32((uint32_t)(be >> 32)));
            const uint32_t lo = (uint32_t)be;
            if (lo) atomicOr(words + wi + 1, bswap32(lo));
        }
        off += len[t];
    }
}

// ---------------------------------------------------------------------------
// decode

// 64 stream bits starting at bit p (MSB-first), zero past the end
__device__ __forceinline__ unsigned long long bswap64(unsigned long long x) {
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((unsigned long long)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
}

__device__ __forceinline__ unsigned long long peek64(const uint8_t *s, long long nbytes,
                                                     long long p) {
    const long long b = p >> 3;
    const long long w = b >> 3;
    if ((((uintptr_t)s) & 7) == 0 && (w + 2) * 8 <= nbytes) {
        // two aligned big-endian words hold bits p .. p+63
        const unsigned long long *q = reinterpret_cast<const unsigned long long *>(s);
        const unsigned long long hi = bswap64(__ldg(q + w)), lo = bswap64(__ldg(q + w + 1));
        const int sh = (int)(p - w * 64);
        return sh ? (hi << sh) | (lo >> (64 - sh)) : hi;
    }
    unsigned long long v = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        const long long bi = b + i;
        const unsigned long long byte = bi < nbytes ? (unsigned long long)__ldg(s + bi) : 0ull;
        if (i < 8) v |= byte << (56 - 8 * i);
        else v = (v << (p & 7)) | (byte >> (8 - (p & 7)));  // p & 7 == 0: byte >> 8 == 0
    }
    return v;
}

// Decode one symbol starting at bit p; returns its length (0 = truncated:
// the unary run or the remainder runs past nbits, depthcodec.py:337-355).
__device__ __forceinline__ long long rice_one(const uint8_t *s, long long nbytes, long long nbits,
                                              int k, long long p, unsigned long long &zz) {
    long long q = 0;
    long long t = p;
    while (true) {
        if (t >= nbits) return 0;
        const unsigned long long w = peek64(s, nbytes, t);
        if (w) {
            const int lz = __clzll(w);
            t += lz;
            q += lz;
            break;
        }
        t += 64;
        q += 64;
    }
    if (t >= nbits) return 0;            // the one lies in the zero padding
    if (t + 1 + k > nbits) return 0;
    const unsigned long long rem =
        k ? (peek64(s, nbytes, t + 1) >> (64 - k)) : 0ull;
    zz = ((unsigned long long)q << k) | rem;
    return t + 1 + k - p;
}

struct RiceChunks {
    const uint8_t *s;
    long long nbytes, nbits;
    int k;
    long long nchunks;
    long long *entry;              // symbol start the chunk decodes from
    long long *exit;               // first symbol start at or past the chunk end
    unsigned long long *count;     // symbols starting inside the chunk
    int *trunc;                    // 1: the chunk's last symbol is truncated
};

__device__ void chunk_decode(const RiceChunks &c, long long j, long long e) {
    const long long end = (j + 1) * kRiceChunkBits < c.nbits ? (j + 1) * kRiceChunkBits : c.nbits;
    long long p = e;
    unsigned long long n = 0;
    int tr = 0;
    while (p < end) {
        unsigned long long zz;
        const long long len = rice_one(c.s, c.nbytes, c.nbits, c.k, p, zz);
        if (!len) { tr = 1; p = c.nbits; break; }
        p += len;
        ++n;
    }
    c.entry[j] = e;
    c.exit[j] = p;
    c.count[j] = n;
    c.trunc[j] = tr;
}

// round 0: every chunk guesses that a symbol starts at its first bit
__global__ void k_rice_spec(RiceChunks c) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < c.nchunks) chunk_decode(c, j, j == 0 ? 0 : j * kRiceChunkBits);
}

// later rounds: entry(j) = exit(j-1) of the previous round (Jacobi); chunks
// whose entry changed decode again. `exit_prev` is the previous round's
// exits; `changed` counts the chunks that moved.
__global__ void k_rice_sync(RiceChunks c, const long long *exit_prev, int *changed) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= c.nchunks || j == 0) return;
    const long long e = exit_prev[j - 1];
    if (e == c.entry[j]) return;
    chunk_decode(c, j, e);
    atomicAdd(changed, 1);
}

// Position of residual (row, col) in the rebuild's skewed layout: strip
// (32 rows) by strip, step t = col + lane by step, 32 lanes contiguous, so the
// wavefront's warp reads (and writes) 32 consecutive words per step.
#ifndef FVV_MED_DIAG
#define FVV_MED_DIAG 1
#endif

__device__ __forceinline__ long long skew_index(long long idx, int W, int H) {
    const int row = (int)(idx / W), col = (int)(idx - (long long)row * W);
#if FVV_MED_DIAG
    // anti-diagonal major: diagonal t = row + col holds rows 0..H-1 at t*H + row
    (void)W;
    return (long long)(row + col) * H + row;
#else
    (void)H;
    const int lane = row & 31;
    return ((long long)(row >> 5) * (W + 31) + col + lane) * 32 + lane;
#endif
}

// residuals of the first n symbols (zig-zag inverse, depthcodec.py:389)
__global__ void k_rice_emit(RiceChunks c, const unsigned long long *base, long long n, int W,
                            int H, int32_t *res) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= c.nchunks) return;
    long long p = c.entry[j];
    unsigned long long idx = base[j];
    const unsigned long long cnt = c.count[j];
    for (unsigned long long s = 0; s < cnt && (long long)idx < n; ++s, ++idx) {
        unsigned long long zz = 0;
        p += rice_one(c.s, c.nbytes, c.nbits, c.k, p, zz);
        const long long z = (long long)zz;
        res[skew_index((long long)idx, W, H)] = (int32_t)((z & 1) == 0 ? z / 2 : -(z + 1) / 2);
    }
}

// The MED recurrence x = r + med(left, up, up-left) (depthcodec.py:301-316)
// on one plane per CTA. Warp w rebuilds 32-row strips w, w+32, ...; lane l
// holds row 32*strip + l and reaches column j at step j + l, so its up and
// up-left neighbours are lane l-1's values of the two previous steps
// (shuffles). Lane 0 takes them from the previous strip's last row, which
// that strip's lane 31 publishes column by column into one of two shared-
// memory row slots as 64-bit (strip tag << 32 | x) words: one aligned 8-byte
// store is atomic, so the consumer spins on the word itself and needs no
// fence. Two slots are enough: strip S+1 overwrites column j of slot (S+1)%2
// only after its lane 0 consumed column j of strip S, i.e. after strip S's
// lane 0 read column j of strip S-1 from that slot.
#ifndef FVV_MED_SLEEP
#define FVV_MED_SLEEP 32
#endif
#ifndef FVV_MED_PF
#define FVV_MED_PF 4
#endif
constexpr int kPf = FVV_MED_PF;  // residual prefetch depth of the MED rebuild

__global__ void __launch_bounds__(1024, 1) k_med_rebuild(const int32_t *res, int W, int H,
                                                         uint8_t *out_skew) {
    extern __shared__ long long s_rows[];       // [2][W] (strip << 32 | x)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nstrips = (H + 31) / 32;
    for (int i = threadIdx.x; i < 2 * W; i += blockDim.x) s_rows[i] = -1ll << 32;
    __syncthreads();
    volatile long long *vrows = s_rows;
    for (int strip = warp; strip < nstrips; strip += 32) {
        const int row = strip * 32 + lane;
        const bool live = row < H;
        const int slot = strip & 1, pslot = slot ^ 1;
        int cur = 0, prev = 0;   // this lane's x at columns j-1 and j-2
        int bprev = 0;           // lane 0: the previous strip's x at column j-1
        const int steps = W + 31;
        // residuals and outputs in the skewed layout (skew_index): step t of
        // this strip is 32 consecutive words / bytes. The residuals stream
        // through a kPf-deep register window loaded kPf steps ahead.
        const long long sbase = (long long)strip * (W + 31) * 32 + lane;
        int32_t win[kPf];
#pragma unroll
        for (int q = 0; q < kPf; ++q) {
            const int jq = q - lane;
            win[q] = (live && jq >= 0 && jq < W) ? __ldg(res + sbase + (long long)q * 32) : 0;
        }
        // unrolled by kPf so window slot u is consumed at step t0 + u and
        // refilled for step t0 + u + kPf: each load has kPf steps to land
        for (int t0 = 0; t0 < steps; t0 += kPf) {
#pragma unroll
            for (int u = 0; u < kPf; ++u) {
                const int t = t0 + u;
                if (t >= steps) break;
                const int j = t - lane;
                // up / up-left: lane l-1's values from the last two steps
                const int up_l = __shfl_up_sync(0xffffffffu, cur, 1);
                const int upl_l = __shfl_up_sync(0xffffffffu, prev, 1);
                int x = 0;
                if (j >= 0 && j < W && live) {
                    int b, c;
                    if (lane == 0) {
                        if (strip == 0) {
                            b = 0;
                        } else {
                            long long w;
                            // a waiting lane backs off, leaving issue slots
                            // to the producing warps on the same SM
                            while ((int)((w = vrows[pslot * W + j]) >> 32) != strip - 1)
                                __nanosleep(FVV_MED_SLEEP);
                            b = (int)(uint32_t)w;
                        }
                        c = j > 0 ? bprev : 0;
                        bprev = b;
                    } else {
                        b = up_l;
                        c = j > 0 ? upl_l : 0;
                    }
                    const int a = j > 0 ? cur : 0;
                    x = win[u] + med(a, b, c);
                    out_skew[sbase + (long long)t * 32] = (uint8_t)x;   // astype(uint8): mod 256
                    if (lane == 31 && strip + 1 < nstrips)
                        vrows[slot * W + j] = ((long long)strip << 32) | (uint32_t)x;
                }
                if (j >= 0 && j < W) {
                    prev = cur;
                    cur = x;
                }
                const int jn = j + kPf;
                win[u] = (live && jn >= 0 && jn < W)
                             ? __ldg(res + sbase + (long long)(t + kPf) * 32) : 0;
            }
        }
    }
}

// The MED recurrence as an anti-diagonal wavefront in one CTA: step t
// computes every (row, t - row) at once, since x(i, j) needs only diagonal
// t-1 (left (i, j-1), up (i-1, j)) and t-2 (up-left). The last two diagonals
// live in shared memory indexed by row; residuals and outputs use the
// anti-diagonal-major layout, so each step reads and writes contiguous
// words. One barrier per step; each thread owns rows tid, tid + blockDim, ...
constexpr int kDiagPf = 8;  // residual prefetch depth (steps)

template <int ROWS>
__global__ void __launch_bounds__(1024, 1) k_med_rebuild_diag(const int32_t *res, int W, int H,
                                                              uint8_t *out_diag) {
    extern __shared__ int32_t s_diag[];   // [3][H]: diagonals t, t-1, t-2 (rotating)
    const int nt = blockDim.x;
    const int steps = W + H - 1;
    // residuals of this thread's rows, kDiagPf steps ahead: ring slot u
    // holds step t0 + u and is refilled with step t0 + u + kDiagPf
    int32_t ring[kDiagPf][ROWS];
    auto fetch = [&](int t, int q) -> int32_t {
        const int i = threadIdx.x + q * nt;
        return (i < H && i <= t && t - i < W) ? __ldg(res + (long long)t * H + i) : 0;
    };
#pragma unroll
    for (int u = 0; u < kDiagPf; ++u)
#pragma unroll
        for (int q = 0; q < ROWS; ++q) ring[u][q] = fetch(u, q);
    for (int t0 = 0; t0 < steps; t0 += kDiagPf) {
#pragma unroll
        for (int u = 0; u < kDiagPf; ++u) {
            const int t = t0 + u;
            if (t >= steps) break;
            int32_t *d0 = s_diag + (t % 3) * H;
            const int32_t *d1 = s_diag + ((t + 2) % 3) * H;   // t - 1
            const int32_t *d2 = s_diag + ((t + 1) % 3) * H;   // t - 2
#pragma unroll
            for (int q = 0; q < ROWS; ++q) {
                const int i = threadIdx.x + q * nt;
                const int j = t - i;
                if (i < H && j >= 0 && j < W) {
                    const int a = j > 0 ? d1[i] : 0;
                    const int b = i > 0 ? d1[i - 1] : 0;
                    const int c = (i > 0 && j > 0) ? d2[i - 1] : 0;
                    const int x = ring[u][q] + med(a, b, c);
                    d0[i] = x;
                    out_diag[(long long)t * H + i] = (uint8_t)x;   // astype(uint8): modulo 256
                }
                ring[u][q] = fetch(t + kDiagPf, q);
            }
            __syncthreads();
        }
    }
}

// skewed rebuild output -> raster plane
__global__ void k_deskew(const uint8_t *skew, int W, int H, uint8_t *out) {
    const long long n = (long long)W * H;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = skew[skew_index(i, W, H)];
}

// adler32 (zlib) of n bytes: A = 1 + sum d_i, B = n + sum (n - i) d_i, mod 65521
__global__ void k_adler(const uint8_t *d, long long n, unsigned long long *sums) {
    unsigned long long a = 0, b = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long v = d[i];
        a += v;
        b += (unsigned long long)(n - i) * v;
    }
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sums[0], a % 65521ull);
        atomicAdd(&sums[1], b % 65521ull);
    }
}

// ---------------------------------------------------------------------------
// host launchers

cudaError_t rice_encode(const uint8_t *plane, int W, int H, RiceScratch &sc, uint8_t *stream,
                        int *k_out, long long *nbits_out, cudaStream_t s) {
    const long long n = (long long)W * H;
    cudaError_t e;
    if ((e = cudaMemsetAsync(sc.costs, 0, sizeof(unsigned long long) * (kRiceKMax + 1), s)))
        return e;
    k_med_zz<<<148 * 8, 256, 0, s>>>(plane, W, H, sc.zz, sc.costs);
    unsigned long long costs[kRiceKMax + 1];
    if ((e = cudaMemcpyAsync(costs, sc.costs, sizeof(costs), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    // depthcodec.py:380-381: min over (cost, k) -> smallest cost, then smallest k
    int k = 0;
    for (int q = 1; q <= kRiceKMax; ++q)
        if (costs[q] < costs[k]) k = q;
    const long long nb = (n + kScanB - 1) / kScanB;
    k_rice_lens<<<(unsigned)nb, 256, 0, s>>>(sc.zz, n, k, sc.block);
    k_scan_blocks<<<1, 1024, 0, s>>>(sc.block, nb, sc.total);
    const long long nbits = (long long)costs[k];
    const long long nwords = (nbits + 31) / 32 + 1;
    if ((e = cudaMemsetAsync(stream, 0, (size_t)nwords * 4, s))) return e;
    k_rice_write<<<(unsigned)nb, 256, 0, s>>>(sc.zz, n, k, sc.block,
                                              reinterpret_cast<uint32_t *>(stream));
    *k_out = k;
    *nbits_out = nbits;
    return cudaGetLastError();
}

cudaError_t rice_decode(const uint8_t *stream, long long nbytes, int k, long long n, int W, int H,
                        RiceScratch &sc, uint8_t *plane, uint32_t *adler_out, int *status,
                        cudaStream_t s) {
    *status = 0;
    cudaError_t e;
    const long long nbits = nbytes * 8;
    RiceChunks c{};
    c.s = stream;
    c.nbytes = nbytes;
    c.nbits = nbits;
    c.k = k;
    c.nchunks = nbits ? (nbits + kRiceChunkBits - 1) / kRiceChunkBits : 0;
    c.entry = sc.entry;
    c.exit = sc.exit;
    c.count = sc.count;
    c.trunc = sc.trunc;
    const unsigned g = (unsigned)((c.nchunks + 127) / 128);
#ifdef FVV_CODEC_TRACE
    cudaEvent_t t0_;
    cudaEventCreate(&t0_);
    cudaEventRecord(t0_, s);
    int rounds_ = 0;
#endif
    if (c.nchunks) {
        k_rice_spec<<<g, 128, 0, s>>>(c);
        TRACE_EV("spec");
        for (int round = 0;; round += 2) {
            // two Jacobi rounds per host check: segmentations settle after
            // the first round in practice, so one read-back confirms them
            for (int r2 = 0; r2 < 2; ++r2) {
                if ((e = cudaMemcpyAsync(sc.exit_prev, sc.exit, sizeof(long long) * c.nchunks,
                                         cudaMemcpyDeviceToDevice, s)))
                    return e;
                if ((e = cudaMemsetAsync(sc.changed, 0, sizeof(int), s))) return e;
                k_rice_sync<<<g, 128, 0, s>>>(c, sc.exit_prev, sc.changed);
            }
            int changed = 0;
            if ((e = cudaMemcpyAsync(&changed, sc.changed, sizeof(int), cudaMemcpyDeviceToHost, s)))
                return e;
            if ((e = cudaStreamSynchronize(s))) return e;
#ifdef FVV_CODEC_TRACE
            ++rounds_;
            fprintf(stderr, "[codec] round %d changed %d\n", rounds_, changed);
#endif
            if (!changed) break;
            if (round > c.nchunks) return cudaErrorUnknown;  // cannot happen: one chunk per round
        }
        if ((e = cudaMemcpyAsync(sc.block, sc.count, sizeof(unsigned long long) * c.nchunks,
                                 cudaMemcpyDeviceToDevice, s)))
            return e;
        k_scan_blocks<<<1, 1024, 0, s>>>(sc.block, c.nchunks, sc.total);
    } else if ((e = cudaMemsetAsync(sc.total, 0, sizeof(unsigned long long), s))) {
        return e;
    }
    // the symbol a truncated chunk stopped at must lie past the n we need
    unsigned long long total = 0;
    if ((e = cudaMemcpyAsync(&total, sc.total, sizeof(total), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    if ((long long)total < n) { *status = 1; return cudaSuccess; }   // stream runs out early
    TRACE_EV("sync+scan");
    if (c.nchunks) k_rice_emit<<<g, 128, 0, s>>>(c, sc.block, n, W, H, sc.res);
    TRACE_EV("emit");
#if FVV_MED_DIAG
    {
        // one row per thread up to 1024 rows (fewer warps per barrier), else
        // 1024 threads with up to kDiagRows rows each
        const size_t sm = (size_t)3 * H * sizeof(int32_t);
        if (H <= 1024)
            k_med_rebuild_diag<1><<<1, (H + 31) / 32 * 32, sm, s>>>(sc.res, W, H, sc.skew);
        else if (H <= 2048)
            k_med_rebuild_diag<2><<<1, 1024, sm, s>>>(sc.res, W, H, sc.skew);
        else
            k_med_rebuild_diag<4><<<1, 1024, sm, s>>>(sc.res, W, H, sc.skew);
    }
#else
    const size_t smem = (size_t)2 * W * sizeof(long long);
    if (smem > 48 * 1024)   // per-device attribute: set on every launch of this variant
        cudaFuncSetAttribute(k_med_rebuild, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    k_med_rebuild<<<1, 1024, smem, s>>>(sc.res, W, H, sc.skew);
#endif
    k_deskew<<<148 * 4, 256, 0, s>>>(sc.skew, W, H, plane);
    TRACE_EV("rebuild");
    if ((e = cudaMemsetAsync(sc.costs, 0, 2 * sizeof(unsigned long long), s))) return e;
    k_adler<<<148 * 4, 256, 0, s>>>(plane, n, sc.costs);
    unsigned long long ab[2];
    if ((e = cudaMemcpyAsync(ab, sc.costs, sizeof(ab), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    const uint32_t A = (uint32_t)((1 + ab[0]) % 65521ull);
    const uint32_t B = (uint32_t)(((unsigned long long)n % 65521ull + ab[1]) % 65521ull);
    *adler_out = (B << 16) | A;
    return cudaGetLastError();
}

}  // namespace fvv
