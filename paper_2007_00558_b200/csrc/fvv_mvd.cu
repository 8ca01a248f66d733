// MVD disk-container rasters (second half).
//
//   k_encode_mm     core.depth_to_millimeters (core.py:246-255): Valid pixels
//                   np.round(f32 depth * 1000.0) clipped to [1, 65535] (the
//                   product is float32 under numpy 2's scalar promotion, the
//                   rounding half-to-even), every other pixel 0. 4 px/thread.
//   k_rle_*         mvdio.rle_encode (mvdio.py:34-40): a run starts at 0 and
//                   wherever flat[i] != flat[i-1]. Boundary counts per
//                   1024-px block, one exclusive scan over the blocks, then
//                   every block writes its run starts (and their codes) in
//                   order with a ballot prefix — the runs come out ascending.
//   k_rle_decode    mvdio.rle_decode (mvdio.py:43-52): each pixel finds its run
//                   by binary search over the runs' cumulative ends (the host
//                   checks they cover exactly the raster, as the reference
//                   does).

#include "fvv_mvd.cuh"

namespace fvv {

__global__ void k_encode_mm(const float *__restrict__ depth, const uint8_t *__restrict__ val,
                            long long n, uint16_t *__restrict__ mm) {
    const long long i0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long i = i0 + q;
        if (i >= n) return;
        uint16_t o = 0;
        if (val[i] == 0) {  // Validity.VALID
            const float r = rintf(__fmul_rn(depth[i], 1000.0f));
            o = (uint16_t)fminf(fmaxf(r, 1.0f), 65535.0f);
        }
        mm[i] = o;
    }
}

cudaError_t launch_encode_mm(const float *depth, const uint8_t *validity, long long n,
                             uint16_t *mm, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const long long threads = (n + 3) / 4;
    k_encode_mm<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(depth, validity, n, mm);
    return cudaGetLastError();
}

__global__ void k_rle_decode(const uint8_t *__restrict__ codes, const long long *__restrict__ ends,
                             long long n_runs, long long n, uint8_t *__restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // first run whose end exceeds i (zero-length runs are skipped over)
    long long lo = 0, hi = n_runs - 1;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (ends[mid] > i) hi = mid;
        else lo = mid + 1;
    }
    out[i] = codes[lo];
}

cudaError_t launch_rle_decode(const uint8_t *codes, const long long *ends, long long n_runs,
                              long long n, uint8_t *out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_rle_decode<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(codes, ends, n_runs, n, out);
    return cudaGetLastError();
}

// boundary flags of the 4 pixels a thread owns in block b
__device__ __forceinline__ unsigned rle_bounds(const uint8_t *flat, long long n, long long i0) {
    unsigned m = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const long long i = i0 + q;
        if (i < n && (i == 0 || flat[i] != flat[i - 1])) m |= 1u << q;
    }
    return m;
}

__global__ void k_rle_count(const uint8_t *__restrict__ flat, long long n,
                            unsigned long long *__restrict__ block) {
    __shared__ int s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const long long i0 = (long long)blockIdx.x * kRlePx + threadIdx.x * 4;
    const int c = __popc(rle_bounds(flat, n, i0));
    const int w = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(&s_cnt, w);
    __syncthreads();
    if (threadIdx.x == 0) block[blockIdx.x] = (unsigned long long)s_cnt;
}

// exclusive scan of nb block counts in one CTA; block[nb] = total
__global__ void k_rle_scan(unsigned long long *block, long long nb, long long *n_runs) {
    __shared__ unsigned long long s_w[32];
    __shared__ unsigned long long s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (long long base = 0; base < nb; base += blockDim.x) {
        const long long i = base + threadIdx.x;
        const unsigned long long v = i < nb ? block[i] : 0ull;
        unsigned long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned long long t = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0ull;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            s_w[lane] = t;   // inclusive warp totals
        }
        __syncthreads();
        const unsigned long long before = s_carry + (warp ? s_w[warp - 1] : 0ull) + x - v;
        if (i < nb) block[i] = before;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = before + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        block[nb] = s_carry;
        *n_runs = (long long)s_carry;
    }
}

__global__ void k_rle_write(const uint8_t *__restrict__ flat, long long n,
                            const unsigned long long *__restrict__ block,
                            long long *__restrict__ starts, uint8_t *__restrict__ codes) {
    __shared__ int s_wc[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long i0 = (long long)blockIdx.x * kRlePx + threadIdx.x * 4;
    const unsigned m = rle_bounds(flat, n, i0);
    const int c = __popc(m);
    // rank of this thread's first run inside the block: lanes, then warps
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_wc[warp] = x;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_wc[w];
    long long r = (long long)block[blockIdx.x] + wbase + x - c;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (m & (1u << q)) {
            starts[r] = i0 + q;
            codes[r] = flat[i0 + q];
            ++r;
        }
    }
}

cudaError_t launch_rle_encode(const uint8_t *flat, long long n, long long *starts,
                              uint8_t *codes, const RleScratch &sc, cudaStream_t s) {
    const long long nb = (n + kRlePx - 1) / kRlePx;
    if (n > 0) k_rle_count<<<(unsigned)nb, 256, 0, s>>>(flat, n, sc.block);
    k_rle_scan<<<1, 1024, 0, s>>>(sc.block, nb, sc.n_runs);
    if (n > 0) k_rle_write<<<(unsigned)nb, 256, 0, s>>>(flat, n, sc.block, starts, codes);
    return cudaGetLastError();
}

}  // namespace fvv
