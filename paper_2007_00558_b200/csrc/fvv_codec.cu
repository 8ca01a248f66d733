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
//   decode  k_rice_spec / k_rice_sync  chunked speculative decoding: every
//                         128-bit chunk decodes from an entry guess to its
//                         exit; rounds re-decode chunks whose entry (= the
//                         previous chunk's exit) changed until none does.
//                         Rice codes resynchronise within a few symbols, so
//                         2-3 rounds settle an exact symbol segmentation
//           k_count_sums / k_scan_blocks / k_count_scan / k_plane_totals
//                         symbol base of every chunk (one scan over the batch)
//           k_rice_emit   each chunk writes its residuals
//           k_med_rebuild_wave  the MED recurrence, one warp per 128-row
//                         strip (lane = 4 rows, one column of skew per row,
//                         neighbours by shuffle), strip edges handed down
//                         through epoch-tagged global slots; every strip of
//                         every plane of a batch runs concurrently
//           k_deskew      strip layout -> raster plane
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
// 0 outside the plane. The reference's three cases (c >= max(a, b): min;
// c <= min(a, b): max; else a + b - c) are all max(a, b, c) + min(a, b, c) - c:
// two 3-input min/max and one add, no compare-and-select chain, and exact in
// wrapping int32 arithmetic (the true value lies between min and max).
__device__ __forceinline__ int med(int a, int b, int c) {
    const int mx = max(max(a, b), c), mn = min(min(a, b), c);
    return (int)((unsigned)mx + (unsigned)mn - (unsigned)c);
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

// exclusive scan of v[0..n) in place by one CTA of 1024 threads; total in
// *total. Warp w owns a contiguous range, read 32 consecutive elements at a
// time (coalesced): pass 1 sums it, one CTA barrier scans the 32 warp sums,
// pass 2 scans the range slice by slice with shuffles and a running carry.
__device__ void scan_segment(unsigned long long *v, long long n, unsigned long long *total) {
    __shared__ unsigned long long ws[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long per = ((n + 31) / 32 + 31) / 32 * 32;  // whole slices per warp
    const long long i0 = (long long)w * per;
    const long long i1 = i0 + per < n ? i0 + per : n;
#ifndef FVV_SCAN_B
#define FVV_SCAN_B 8
#endif
    constexpr int B = FVV_SCAN_B;  // slices whose loads are in flight together
    unsigned long long x = 0;
    for (long long b0 = i0; b0 < i1; b0 += 32 * B) {
        unsigned long long y[B];
#pragma unroll
        for (int q = 0; q < B; ++q) {
            const long long i = b0 + 32 * q + lane;
            y[q] = i < i1 ? v[i] : 0;
        }
#pragma unroll
        for (int q = 0; q < B; ++q) x += y[q];
    }
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned long long t = ws[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        ws[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    unsigned long long carry = w ? ws[w - 1] : 0;
    for (long long b0 = i0; b0 < i1; b0 += 32 * B) {
        unsigned long long y[B];
#pragma unroll
        for (int q = 0; q < B; ++q) {
            const long long i = b0 + 32 * q + lane;
            y[q] = i < i1 ? v[i] : 0;
        }
#pragma unroll
        for (int q = 0; q < B; ++q) {
            const long long i = b0 + 32 * q + lane;
            unsigned long long inc = y[q];
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (i < i1) v[i] = carry + inc - y[q];
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
    if (threadIdx.x == 0) *total = ws[31];
}

__global__ void __launch_bounds__(1024) k_scan_blocks(unsigned long long *v, long long n,
                                                      unsigned long long *total) {
    scan_segment(v, n, total);
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

// MSB-first bit reader for the chunk decoders: a 64-bit buffer refilled from
// big-endian 32-bit words with the next word loaded one refill ahead, so a
// symbol costs shifts and a clz instead of the two dependent 64-bit peeks of
// rice_one (same results; bytes past the stream read as zero). Streams of
// any alignment: bits are counted from the 4-byte boundary below s.
struct BitReader {
    const uint32_t *w;       // aligned base (<= s)
    long long nbytes;        // stream bytes (from s)
    int skew;                // s - w, bytes
    unsigned long long buf;  // bits [pos, pos + nb), MSB-aligned, zero below
    int nb;
    long long pos;           // stream bit of buf's MSB
    long long wi;            // aligned index of the prefetched word
    uint32_t next;

    __device__ __forceinline__ uint32_t word(long long i) const {
        const long long b0 = 4 * i - skew;  // stream byte of the word's first byte
        if (b0 >= 0 && b0 + 3 < nbytes) return bswap32(__ldg(w + i));
        uint32_t v = 0;
        const uint8_t *s = reinterpret_cast<const uint8_t *>(w) + skew;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const long long b = b0 + q;
            v = (v << 8) | (b >= 0 && b < nbytes ? (uint32_t)__ldg(s + b) : 0u);
        }
        return v;
    }
    __device__ __forceinline__ void refill() {
        while (nb <= 32) {
            buf |= (unsigned long long)next << (32 - nb);
            nb += 32;
            next = word(++wi);
        }
    }
    __device__ __forceinline__ void start(const uint8_t *s, long long nbytes_, long long p) {
        skew = (int)((uintptr_t)s & 3);
        w = reinterpret_cast<const uint32_t *>(s - skew);
        nbytes = nbytes_;
        const long long a = p + 8 * skew;  // aligned bit position
        wi = a >> 5;
        const int off = (int)(a & 31);
        buf = (unsigned long long)word(wi) << (32 + off);
        nb = 32 - off;
        next = word(++wi);
        pos = p;
        refill();
    }
    __device__ __forceinline__ void skip(int n) {  // n <= nb
        buf = n < 64 ? buf << n : 0ull;
        nb -= n;
        pos += n;
        refill();
    }
    // one symbol (depthcodec.py:337-355); false (truncated) if its unary run
    // or remainder runs past nbits; requires k <= 32
    __device__ __forceinline__ bool symbol(long long nbits, int k, unsigned long long &zz) {
        unsigned long long q = 0;
        while (true) {
            if (pos >= nbits) return false;
            const int lz = __clzll(buf);  // 64 when buf == 0
            if (lz < nb) {
                q += lz;
                if (pos + lz >= nbits) return false;  // the one lies in the padding
                if (pos + lz + 1 + k > nbits) return false;
                skip(lz + 1);
                break;
            }
            q += nb;
            skip(nb);
        }
        const unsigned long long rem = k ? buf >> (64 - k) : 0ull;
        if (k) skip(k);
        zz = (q << k) | rem;
        return true;
    }
};

// Position of residual (row, col) in the rebuild's strip layout
// (rice_skew_size): row = kWaveStrip s + kWaveRows l + h runs in lane l of
// strip s's warp as its row h, computing column col at step
// u = col + kWaveRows l + h; each strip stores [u / 4][h][l][u % 4], so a
// warp reads a row's 4 steps as one 16-byte word per lane and writes its 4
// output bytes as one word.
__device__ __forceinline__ long long skew_rc(int row, int col, int W) {
    const int st = row / kWaveStrip, rr = row - st * kWaveStrip;
    const int l = rr / kWaveRows, h = rr - l * kWaveRows, u = col + rr;
    return (long long)st * kWaveStrip * rice_wave_steps(W) +
           ((long long)(u >> 2) * kWaveRows + h) * 128 + l * 4 + (u & 3);
}

// A batch of planes decoded together (all depth planes of a render tick):
// their chunks are numbered consecutively, plane p owning chunks
// [pl[p].c0, pl[p].c0 + pl[p].nchunks).
struct RiceBatch {
    int np;
    RicePlane pl[kRiceMaxPlanes];
    long long nchunks;             // over all planes
    int ngroups;                   // rebuild CTAs over all planes
    long long *entry;              // symbol start the chunk decodes from (plane bits)
    long long *exit;               // first symbol start at or past the chunk end
    unsigned long long *count;     // symbols starting inside the chunk
};

__device__ __forceinline__ int plane_of(const RiceBatch &b, long long j) {
    int p = 0;
    while (p + 1 < b.np && j >= b.pl[p + 1].c0) ++p;
    return p;
}

__device__ void chunk_decode(const RiceBatch &b, const RicePlane &pl, long long j, long long lj,
                             long long e) {
    const long long end =
        (lj + 1) * kRiceChunkBits < pl.nbits ? (lj + 1) * kRiceChunkBits : pl.nbits;
    long long p = e;
    unsigned long long n = 0;
    if (pl.k <= 32) {
        BitReader br;
        if (p < end) br.start(pl.s, pl.nbytes, p);
        while (p < end) {
            unsigned long long zz;
            if (!br.symbol(pl.nbits, pl.k, zz)) { p = pl.nbits; break; }  // truncated
            p = br.pos;
            ++n;
        }
    } else {
        while (p < end) {
            unsigned long long zz;
            const long long len = rice_one(pl.s, pl.nbytes, pl.nbits, pl.k, p, zz);
            if (!len) { p = pl.nbits; break; }   // truncated: no further symbols
            p += len;
            ++n;
        }
    }
    b.entry[j] = e;
    b.exit[j] = p;
    b.count[j] = n;
}

// round 0: every chunk guesses that a symbol starts at its first bit
__global__ void k_rice_spec(const __grid_constant__ RiceBatch b) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= b.nchunks) return;
    const RicePlane &pl = b.pl[plane_of(b, j)];
    const long long lj = j - pl.c0;
    chunk_decode(b, pl, j, lj, lj * kRiceChunkBits);
}

// later rounds: entry(j) = exit(j-1) of the previous round (Jacobi, within a
// plane); chunks whose entry changed decode again, `changed` counts them
__global__ void k_rice_sync(const __grid_constant__ RiceBatch b, const long long *exit_prev,
                            int *changed) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= b.nchunks) return;
    const RicePlane &pl = b.pl[plane_of(b, j)];
    const long long lj = j - pl.c0;
    if (lj == 0) return;
    const long long e = exit_prev[j - 1];
    if (e == b.entry[j]) return;
    chunk_decode(b, pl, j, lj, e);
    atomicAdd(changed, 1);
}

// Symbol bases: one exclusive scan of the chunk counts over the whole batch,
// spread over the GPU (block sums, one CTA over the block sums, block-local
// scans); a plane's symbol index is then base[j] - base[c0 of its plane].
__global__ void __launch_bounds__(1024) k_count_sums(const unsigned long long *cnt, long long n,
                                                     unsigned long long *bsum) {
    __shared__ unsigned long long ws[32];
    const long long i = (long long)blockIdx.x * 1024 + threadIdx.x;
    unsigned long long x = i < n ? cnt[i] : 0;
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
        x = ws[threadIdx.x];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (threadIdx.x == 0) bsum[blockIdx.x] = x;
    }
}

__global__ void __launch_bounds__(1024) k_count_scan(const unsigned long long *cnt, long long n,
                                                     const unsigned long long *boff,
                                                     unsigned long long *base) {
    __shared__ unsigned long long ws[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long i = (long long)blockIdx.x * 1024 + threadIdx.x;
    const unsigned long long x = i < n ? cnt[i] : 0;
    unsigned long long inc = x;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) ws[w] = inc;
    __syncthreads();
    if (w == 0) {
        unsigned long long t = ws[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        ws[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    if (i < n) base[i] = boff[blockIdx.x] + (w ? ws[w - 1] : 0) + inc - x;
}

// symbols per plane (the batch's grand total closes the last plane)
__global__ void k_plane_totals(const __grid_constant__ RiceBatch b, const unsigned long long *base,
                               const unsigned long long *grand, unsigned long long *totals) {
    const int p = threadIdx.x;
    if (p >= b.np) return;
    const RicePlane &pl = b.pl[p];
    if (!pl.nchunks) {
        totals[p] = 0;
        return;
    }
    const long long e = pl.c0 + pl.nchunks;
    totals[p] = (e < b.nchunks ? base[e] : *grand) - base[pl.c0];
}

// residuals of each plane's first n symbols (zig-zag inverse,
// depthcodec.py:389), into the rebuild's strip layout (skew_rc)
__global__ void k_rice_emit(const __grid_constant__ RiceBatch b, const unsigned long long *base,
                            int32_t *res) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= b.nchunks) return;
    const RicePlane &pl = b.pl[plane_of(b, j)];
    long long p = b.entry[j];
    unsigned long long idx = base[j] - base[pl.c0];  // the plane's symbol index
    const unsigned long long cnt = b.count[j];
    int32_t *r = res + pl.rbase;
    // raster position of the first symbol; later ones step along the row
    int row = (int)(idx / (unsigned long long)pl.W), col = (int)(idx - (unsigned long long)row * pl.W);
    BitReader br;
    const bool fast = pl.k <= 32;
    if (fast && cnt) br.start(pl.s, pl.nbytes, p);
    for (unsigned long long s = 0; s < cnt && (long long)idx < pl.n; ++s, ++idx) {
        unsigned long long zz = 0;
        if (fast)
            br.symbol(pl.nbits, pl.k, zz);  // counted symbols decode (chunk_decode)
        else
            p += rice_one(pl.s, pl.nbytes, pl.nbits, pl.k, p, zz);
        const long long z = (long long)zz;
        r[skew_rc(row, col, pl.W)] = (int32_t)((z & 1) == 0 ? z / 2 : -(z + 1) / 2);
        if (++col == pl.W) {
            col = 0;
            ++row;
        }
    }
}

// The MED recurrence (depthcodec.py:301-317) as a wavefront of strips of
// kWaveStrip rows, one warp each, lane l holding rows R l .. R l + R - 1
// (R = kWaveRows). Row h of a lane runs h steps behind row h - 1 and lane l
// runs R steps behind lane l - 1, so at step u every row needs only values
// of steps u - 1 and u - 2: its own (left), the row above (up, up-left), from
// a register for h > 0 and by shuffle from lane l - 1 for h = 0. The R rows
// of a step are independent (instruction-level parallelism) and a value
// crosses lanes once per R steps.
//
// Lane 0 of strip s reads strip s - 1's last row from global memory: 64-bit
// slots tagged with the batch's epoch, stored by the producer (lane 31) per
// column. Residuals and those slots are staged kWavePf blocks (of 4 steps)
// ahead into shared memory by cp.async, so no load latency and no register
// ring sits on the step chain; a slot whose tag is still stale when its
// block comes is re-read (warp-uniformly) until it is current, and at its
// start a consumer waits until the producer is kWaveLead columns ahead, past
// the staging window. The producer belongs to the same CTA or to a CTA with
// a smaller ticket (taken at CTA start), which has started and waits only on
// smaller tickets: every wait ends (a lost producer would set wave[1] after
// kWaveSpinLimit re-reads instead of hanging).
constexpr int kWavePf = 5;                        // blocks staged ahead
constexpr int kWaveLead = 4 * kWavePf + 4;  // producer lead at a consumer's start (past the staging window)
constexpr long long kWaveSpinLimit = 1ll << 26;

__device__ __forceinline__ unsigned long long ld_edge(const unsigned long long *ptr) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ptr));
    return v;
}
__device__ __forceinline__ void st_edge(unsigned long long *ptr, int p, unsigned long long v) {
    // no "memory" clobber: nothing else in the kernel reads these slots
    // through ordinary accesses, and keeping the compiler free to move the
    // next block's shared-memory loads across this store matters
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
        " @q st.relaxed.gpu.global.u64 [%0], %1;\n}" ::"l"(ptr),
        "l"(v), "r"(p));
}
__device__ __forceinline__ void wave_cp16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
// A slot's value once its tag is the batch's: the whole warp re-reads the
// same slot while any lane sees a stale tag (v: the value each lane last
// read). Warp-uniform on purpose: a wait taken by lane 0 alone would leave
// the warp diverged, and every later shuffle would go through the divergent
// (collective) path.
__device__ __forceinline__ unsigned long long edge_wait(const unsigned long long *slot,
                                                        unsigned long long v, unsigned epoch,
                                                        int *stall) {
    long long n = 0;
#pragma unroll 1
    while (__any_sync(0xffffffffu, (uint32_t)(v >> 32) != epoch)) {
        if (++n == kWaveSpinLimit) {  // a lost producer: report, never hang
            if ((threadIdx.x & 31) == 0) atomicExch(stall, 1);
            break;
        }
        v = ld_edge(slot);
    }
    return v;
}

template <bool C>
struct WaveCheck {
    static constexpr bool value = C;
};

__global__ void __launch_bounds__(32 * kWaveWarps) k_med_rebuild_wave(
    const __grid_constant__ RiceBatch b, const int32_t *res_all, uint8_t *skew_all,
    unsigned long long *edge_all, int *wave, unsigned epoch) {
    constexpr int R = kWaveRows, PF = kWavePf;
    // per warp: PF staged blocks of residuals [R][32 lanes] and edge slots [4]
    __shared__ __align__(16) int4 s_res[kWaveWarps][PF][R][32];
    __shared__ __align__(16) unsigned long long s_top[kWaveWarps][PF][4];
    __shared__ int s_ticket;
    if (threadIdx.x == 0) s_ticket = atomicAdd(wave, 1);
    __syncthreads();
    const int g = s_ticket;
    int p = 0;
    while (p + 1 < b.np && g >= b.pl[p + 1].g0) ++p;
    const RicePlane &pl = b.pl[p];
    const int W = pl.W, H = pl.H, ns = (H + kWaveStrip - 1) / kWaveStrip;
    const int wid = threadIdx.x >> 5;
    const int st = (g - pl.g0) * kWaveWarps + wid;
    if (st >= ns) return;
    const int lane = threadIdx.x & 31;
    const int U = rice_wave_steps(W), nblk = U >> 2, Wp = (W + 3) & ~3;
    const long long sbase = pl.rbase + (long long)st * kWaveStrip * U;
    // block k, row h of this lane: res[32 (R k + h)]
    const int4 *res = reinterpret_cast<const int4 *>(res_all + sbase) + lane;
    uint32_t *out = reinterpret_cast<uint32_t *>(skew_all + sbase) + lane;
    const bool up = st > 0 && lane == 0, down = st + 1 < ns && lane == 31;
    const unsigned long long *top = edge_all + pl.ebase + (long long)(st > 0 ? st - 1 : 0) * Wp;
    unsigned long long *mine = edge_all + pl.ebase + (long long)st * Wp;
    const unsigned long long tag = (unsigned long long)epoch << 32;
    const int l0 = R * lane;  // this lane's first row within the strip
    int4(*sres)[R][32] = s_res[wid];
    unsigned long long(*stop)[4] = s_top[wid];
    if (st > 0) {  // start once the producer is kWaveLead columns ahead
        const int c = min(kWaveLead, W - 1);
        edge_wait(top + c, ld_edge(top + c), epoch, wave + 1);
    }
    // stage block k (clamped to the strip; past-the-end stages are unused):
    // this lane's R residual words, and for lane 0 the 4 edge slots above
    auto stage = [&](int k) {
        const int kc = min(k, nblk - 1), slot = k % PF;
#pragma unroll
        for (int h = 0; h < R; ++h) wave_cp16(&sres[slot][h][lane], res + 32 * (R * kc + h));
        if (up) {
            const unsigned long long *src = top + min(4 * kc, Wp - 4);
            wave_cp16(&stop[slot][0], src);
            wave_cp16(&stop[slot][2], src + 2);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#pragma unroll
    for (int k = 0; k < PF - 1; ++k) stage(k);
    int x1[R], x2[R];
#pragma unroll
    for (int h = 0; h < R; ++h) x1[h] = x2[h] = 0;
    int tprev = 0;
    // One block of 4 steps. CHECK: some row of some step may lie outside
    // columns 0..W-1 (the strip's first 32R - 1 and last steps); elsewhere
    // every row's column is inside and the range tests go.
    // the staged inputs of block k: this lane's residuals and the 4 edge slots
    // (every lane reads the slots, a broadcast; only lane 0 of a strip > 0
    // uses them)
    struct Staged {
        int4 r[R];
        ulonglong2 v01, v23;
    };
    auto load = [&](int k) {
        Staged d;
        const int slot = k % PF;
#pragma unroll
        for (int h = 0; h < R; ++h) d.r[h] = sres[slot][h][lane];
        d.v01 = *reinterpret_cast<const ulonglong2 *>(&stop[slot][0]);
        d.v23 = *reinterpret_cast<const ulonglong2 *>(&stop[slot][2]);
        return d;
    };
    // One block of 4 steps. CHECK: some row of some step may lie outside
    // columns 0..W-1 (the strip's first 32R - 1 and last steps); elsewhere
    // every row's column is inside and the range tests go.
    auto block = [&](auto check, int k, const Staged &d) {
        constexpr bool CHECK = decltype(check)::value;
        const int4 *r = d.r;
        // lane 0: columns 4k..4k+3 of the row above (stale tags are rare)
        int t[4];
        bool stale = false;
        {
            const unsigned long long v[4] = {d.v01.x, d.v01.y, d.v23.x, d.v23.y};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                t[e] = up ? (int)(uint32_t)v[e] : 0;
                stale |= up && 4 * k + e < W && (uint32_t)(v[e] >> 32) != epoch;
            }
        }
        if (__any_sync(0xffffffffu, stale)) {  // warp-uniform slow path
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (4 * k + e < W)
                    t[e] = (int)(uint32_t)edge_wait(top + 4 * k + e, ld_edge(top + 4 * k + e),
                                                    epoch, wave + 1);
            if (!up) t[0] = t[1] = t[2] = t[3] = 0;
        }
        int xs[4][R];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            int bu = __shfl_up_sync(0xffffffffu, x1[R - 1], 1);
            int cu = __shfl_up_sync(0xffffffffu, x2[R - 1], 1);
            if (lane == 0) {  // strip 0: t and tprev stay 0 (row -1 is 0)
                bu = t[e];
                cu = e ? t[e - 1] : tprev;
            }
#pragma unroll
            for (int h = 0; h < R; ++h) {
                const int bb = h ? x1[h - 1] : bu, cc = h ? x2[h - 1] : cu;
                const int rv = e == 0 ? r[h].x : e == 1 ? r[h].y : e == 2 ? r[h].z : r[h].w;
                const int x = (int)((unsigned)rv + (unsigned)med(x1[h], bb, cc));
                // x1 is 0 left of column 0, so a = 0 there (as in the reference)
                xs[e][h] = !CHECK || (unsigned)(4 * k + e - l0 - h) < (unsigned)W ? x : 0;
            }
#pragma unroll
            for (int h = 0; h < R; ++h) {
                x2[h] = x1[h];
                x1[h] = xs[e][h];
            }
        }
        tprev = t[3];
#pragma unroll
        for (int h = 0; h < R; ++h)  // astype(uint8): the low bytes of 4 steps
            out[32 * (R * k + h)] = __byte_perm(__byte_perm(xs[0][h], xs[1][h], 0x0040),
                                                __byte_perm(xs[2][h], xs[3][h], 0x0040), 0x5410);
        // lane 31: this block's columns of the strip's last row
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = 4 * k + e - (kWaveStrip - 1);
            st_edge(mine + j, down && (!CHECK || (unsigned)j < (unsigned)W),
                    tag | (uint32_t)xs[e][R - 1]);
        }
    };
    // blocks whose steps u all have u >= 32R - 1 and u <= W - 1
    const int km0 = (kWaveStrip - 1 + 3) / 4, km1 = W / 4;
#pragma unroll 1
    for (int k = 0; k < nblk; ++k) {
        stage(k + PF - 1);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(PF - 1) : "memory");
        if (k >= km0 && k < km1)
            block(WaveCheck<false>{}, k, load(k));
        else
            block(WaveCheck<true>{}, k, load(k));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");  // no copy outlives the CTA
}

// strip-layout rebuild output -> raster plane (blockIdx.y = plane)
// (4 consecutive pixels of a row per thread: 4-byte stores when W % 4 == 0)
__global__ void k_deskew(const __grid_constant__ RiceBatch b, const uint8_t *skew_all) {
    const RicePlane &pl = b.pl[blockIdx.y];
    const uint8_t *skew = skew_all + pl.rbase;
    const int W = pl.W, W4 = (W + 3) >> 2;
    const long long n4 = (long long)W4 * pl.H;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / W4), c0 = (int)(i - (long long)row * W4) * 4;
        uint8_t v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = c0 + q < W ? skew[skew_rc(row, c0 + q, W)] : 0;
        uint8_t *o = pl.out + (long long)row * W + c0;
        if ((W & 3) == 0 && ((uintptr_t)pl.out & 3) == 0) {
            *reinterpret_cast<uint32_t *>(o) = (uint32_t)v[0] | ((uint32_t)v[1] << 8) |
                                               ((uint32_t)v[2] << 16) | ((uint32_t)v[3] << 24);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (c0 + q < W) o[q] = v[q];
        }
    }
}

// adler32 (zlib) of each rebuilt plane: A = 1 + sum d_i, B = n + sum (n - i) d_i,
// mod 65521 (blockIdx.y = plane; sums[2p], sums[2p+1])
__global__ void k_adler(const __grid_constant__ RiceBatch b, unsigned long long *sums) {
    const RicePlane &pl = b.pl[blockIdx.y];
    const long long n = pl.n;
    unsigned long long a = 0, c = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long v = pl.out[i];
        a += v;
        c += (unsigned long long)(n - i) * v;
    }
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sums[2 * blockIdx.y], a % 65521ull);
        atomicAdd(&sums[2 * blockIdx.y + 1], c % 65521ull);
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

cudaError_t rice_decode_batch(RicePlane *planes, int np, RiceScratch &sc, cudaStream_t s) {
    cudaError_t e;
    RiceBatch b{};
    b.np = np;
    long long c0 = 0, rbase = 0, ebase = 0;
    int g0 = 0;
    for (int p = 0; p < np; ++p) {
        RicePlane &pl = planes[p];
        pl.nbits = pl.nbytes * 8;
        pl.n = (long long)pl.W * pl.H;
        pl.c0 = c0;
        pl.nchunks = pl.nbits ? (pl.nbits + kRiceChunkBits - 1) / kRiceChunkBits : 0;
        pl.rbase = rbase;
        pl.status = 0;
        c0 += pl.nchunks;
        pl.ebase = ebase;
        pl.g0 = g0;
        rbase += (long long)rice_skew_size(pl.W, pl.H);
        ebase += (long long)rice_edge_size(pl.W, pl.H);
        g0 += (rice_wave_strips(pl.H) + kWaveWarps - 1) / kWaveWarps;
        b.pl[p] = pl;
    }
    b.nchunks = c0;
    b.ngroups = g0;
    b.entry = sc.entry;
    b.exit = sc.exit;
    b.count = sc.count;
    const unsigned g = (unsigned)((b.nchunks + 127) / 128);
    unsigned long long tot[kRiceMaxPlanes] = {0};
#ifdef FVV_CODEC_TRACE
    cudaEvent_t t0_;
    cudaEventCreate(&t0_);
    cudaEventRecord(t0_, s);
#endif
    if (b.nchunks) {
        k_rice_spec<<<g, 128, 0, s>>>(b);
        for (long long round = 0;; round += 2) {
            // two Jacobi rounds per host check: segmentations settle after
            // the first round in practice, so one read-back confirms them
            for (int r2 = 0; r2 < 2; ++r2) {
                if ((e = cudaMemcpyAsync(sc.exit_prev, sc.exit, sizeof(long long) * b.nchunks,
                                         cudaMemcpyDeviceToDevice, s)))
                    return e;
                if ((e = cudaMemsetAsync(sc.changed, 0, sizeof(int), s))) return e;
                k_rice_sync<<<g, 128, 0, s>>>(b, sc.exit_prev, sc.changed);
            }
            int changed = 0;
            if ((e = cudaMemcpyAsync(&changed, sc.changed, sizeof(int), cudaMemcpyDeviceToHost, s)))
                return e;
            if ((e = cudaStreamSynchronize(s))) return e;
            if (!changed) break;
            if (round > b.nchunks) return cudaErrorUnknown;  // cannot happen: >= 1 chunk settles per round
        }
        TRACE_EV("segment");
        // block sums in exit_prev (free after the rounds), grand total in
        // costs[0] (free until the adler32 pass)
        const long long nblk = (b.nchunks + 1023) / 1024;
        unsigned long long *bsum = reinterpret_cast<unsigned long long *>(sc.exit_prev);
        k_count_sums<<<(unsigned)nblk, 1024, 0, s>>>(b.count, b.nchunks, bsum);
        k_scan_blocks<<<1, 1024, 0, s>>>(bsum, nblk, sc.costs);
        k_count_scan<<<(unsigned)nblk, 1024, 0, s>>>(b.count, b.nchunks, bsum, sc.block);
        k_plane_totals<<<1, kRiceMaxPlanes, 0, s>>>(b, sc.block, sc.costs, sc.total);
        TRACE_EV("scan");
    }
    // no host round trip here: a plane whose stream runs out before its n
    // symbols (a truncated symbol ends its chain) is found from the totals
    // read back with the checksums at the end, and reported (its rebuilt
    // bytes are then meaningless)
    if (b.nchunks) k_rice_emit<<<g, 128, 0, s>>>(b, sc.block, sc.res);
    TRACE_EV("emit");
    // edge tags: a fresh epoch per batch (the slots start zeroed, epoch 0 is
    // never used, so no stale slot matches)
    if (++sc.epoch == 0) {
        if ((e = cudaMemsetAsync(sc.edge, 0, sc.e_cap * sizeof(unsigned long long), s))) return e;
        sc.epoch = 1;
    }
    if ((e = cudaMemsetAsync(sc.wave, 0, 2 * sizeof(int), s))) return e;
    k_med_rebuild_wave<<<b.ngroups, 32 * kWaveWarps, 0, s>>>(b, sc.res, sc.skew, sc.edge, sc.wave,
                                                            sc.epoch);
    TRACE_EV("rebuild");
    k_deskew<<<dim3(148 * 2, np), 256, 0, s>>>(b, sc.skew);
    TRACE_EV("deskew");
    if ((e = cudaMemsetAsync(sc.costs, 0, 2 * np * sizeof(unsigned long long), s))) return e;
    k_adler<<<dim3(148, np), 256, 0, s>>>(b, sc.costs);
    unsigned long long ab[2 * kRiceMaxPlanes];
    int stall = 0;
    if ((e = cudaMemcpyAsync(ab, sc.costs, 2 * np * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s)))
        return e;
    if ((e = cudaMemcpyAsync(&stall, sc.wave + 1, sizeof(int), cudaMemcpyDeviceToHost, s)))
        return e;
    if (b.nchunks && (e = cudaMemcpyAsync(tot, sc.total, sizeof(unsigned long long) * np,
                                          cudaMemcpyDeviceToHost, s)))
        return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    TRACE_EV("adler");
    if (stall) return cudaErrorLaunchTimeout;  // a strip never received the row above
    for (int p = 0; p < np; ++p) {
        planes[p].status = (long long)tot[p] < planes[p].n ? 1 : 0;
        const unsigned long long n = (unsigned long long)planes[p].n;
        const uint32_t A = (uint32_t)((1 + ab[2 * p]) % 65521ull);
        const uint32_t B = (uint32_t)((n % 65521ull + ab[2 * p + 1]) % 65521ull);
        planes[p].adler = (B << 16) | A;
    }
    return cudaGetLastError();
}

}  // namespace fvv
