// MED + Golomb-Rice plane codec (fvv_codec.cu): scratch and host launchers.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fvv {

constexpr int kRiceKMax = 14;          // depthcodec.py:380: k in range(15)
#ifndef FVV_RICE_CHUNK
#define FVV_RICE_CHUNK 128
#endif
constexpr int kRiceChunkBits = FVV_RICE_CHUNK;  // decode chunk (speculative segmentation unit)
constexpr int kMedMaxWidth = 12288;    // MED rebuild: widest plane (strip rows of W + 31 steps)

constexpr int kRiceMaxPlanes = 48;     // planes per decode batch (16 cameras x Y, U, V)

// one plane of a decode batch; the caller fills s, nbytes, k, W, H, out
struct RicePlane {
    const uint8_t *s;       // device stream
    long long nbytes;
    int k;
    int W, H;
    uint8_t *out;           // device plane (W x H)
    // filled by rice_decode_batch
    long long nbits, n, c0, nchunks, rbase;
    long long ebase;        // first strip-edge slot of the plane (rice_edge_size)
    int g0;                 // first rebuild CTA of the plane (kWaveWarps strips each)
    int status;             // 1: the stream runs out before W*H symbols
    uint32_t adler;         // adler32 of the rebuilt plane
};

// per-context device scratch, sized for n pixels / c chunks
struct RiceScratch {
    uint16_t *zz = nullptr;                 // [n] encoder symbols
    int32_t *res = nullptr;                 // [skewed n] decoder residuals (rice_skew_size)
    uint8_t *skew = nullptr;                // [skewed n] rebuilt plane, skewed layout
    unsigned long long *block = nullptr;    // [max(n/1024, c) + 1] scan buffer
    unsigned long long *costs = nullptr;    // [2 * kRiceMaxPlanes] per-k costs / adler sums
    unsigned long long *total = nullptr;    // [kRiceMaxPlanes] per-plane symbol totals
    long long *entry = nullptr, *exit = nullptr, *exit_prev = nullptr;  // [c] over all planes
    unsigned long long *count = nullptr;    // [c]
    int *changed = nullptr;                 // [1]
    unsigned long long *edge = nullptr;     // [sum rice_edge_size] strip edges, epoch-tagged
    int *wave = nullptr;                    // [2] rebuild CTA ticket, stall flag
    unsigned epoch = 0;                     // tag of the current batch's strip edges
    size_t e_cap = 0;
    size_t n_cap = 0, c_cap = 0;
};

// Encode one u8 plane: MED residuals, zig-zag, cheapest k, Rice bits into
// `stream` (zeroed here; needs rice_stream_bound bytes). Synchronises once
// (the choice of k).
cudaError_t rice_encode(const uint8_t *plane, int W, int H, RiceScratch &sc, uint8_t *stream,
                        int *k_out, long long *nbits_out, cudaStream_t s);

// Decode np planes together: W*H symbols of parameter k from each stream,
// rebuild every plane (one warp per 32-row strip, all planes concurrently)
// and its adler32. Scratch must hold sum(rice_skew_size) residuals,
// sum(rice_edge_size) edge slots and sum(chunks) + np chunk entries.
// Synchronous.
cudaError_t rice_decode_batch(RicePlane *planes, int np, RiceScratch &sc, cudaStream_t s);

// The MED rebuild (fvv_codec.cu, k_med_rebuild_wave) runs one warp per strip
// of 32 x kWaveRows rows, lane l on rows kWaveRows l .. kWaveRows l + R - 1,
// skewed so that step u computes column u - (row within the strip): a strip
// takes W + 32 kWaveRows - 1 steps, padded to a multiple of 4.
#ifndef FVV_WAVE_R
#define FVV_WAVE_R 4
#endif
constexpr int kWaveRows = FVV_WAVE_R;     // rows per lane
constexpr int kWaveStrip = 32 * kWaveRows;  // rows per strip (warp)
#ifndef FVV_WAVE_WARPS
#define FVV_WAVE_WARPS 4
#endif
constexpr int kWaveWarps = FVV_WAVE_WARPS;  // strips per rebuild CTA
__host__ __device__ inline int rice_wave_steps(int W) { return (W + kWaveStrip - 1 + 3) & ~3; }
inline int rice_wave_strips(int H) { return (H + kWaveStrip - 1) / kWaveStrip; }

// elements of the rebuild's skewed layout for a W x H plane (residuals in,
// bytes out): per strip, [steps / 4][kWaveRows][32 lanes][4 steps]
inline size_t rice_skew_size(int W, int H) {
    return (size_t)rice_wave_strips(H) * kWaveStrip * (size_t)rice_wave_steps(W);
}

// 64-bit strip-edge slots for a W x H plane: the last row of every strip, as
// the next strip reads it (row stride W rounded up to 4)
inline size_t rice_edge_size(int W, int H) {
    return (size_t)rice_wave_strips(H) * (size_t)((W + 3) & ~3);
}

// bytes `stream` must hold for a W x H plane: the cheapest k costs at most
// what k = 8 does (<= 10 bits per symbol for zz <= 510), plus a spill word
inline long long rice_stream_bound(int W, int H) {
    return ((long long)W * H * 10 + 31) / 32 * 4 + 8;
}

}  // namespace fvv
