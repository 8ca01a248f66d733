// MED + Golomb-Rice plane codec (fvv_codec.cu): scratch and host launchers.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fvv {

constexpr int kRiceKMax = 14;          // depthcodec.py:380: k in range(15)
constexpr int kRiceChunkBits = 256;    // decode chunk (speculative segmentation unit)
constexpr int kMedMaxWidth = 12288;    // MED rebuild: 2 x W x 8 B of row slots in shared memory

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
    size_t n_cap = 0, c_cap = 0;
};

// Encode one u8 plane: MED residuals, zig-zag, cheapest k, Rice bits into
// `stream` (zeroed here; needs rice_stream_bound bytes). Synchronises once
// (the choice of k).
cudaError_t rice_encode(const uint8_t *plane, int W, int H, RiceScratch &sc, uint8_t *stream,
                        int *k_out, long long *nbits_out, cudaStream_t s);

// Decode np planes together: W*H symbols of parameter k from each stream,
// rebuild each plane (one CTA per plane, concurrently) and its adler32.
// Scratch must hold sum(rice_skew_size) residuals and sum(chunks) + np chunk
// entries. Synchronous.
cudaError_t rice_decode_batch(RicePlane *planes, int np, RiceScratch &sc, cudaStream_t s);

// elements of the rebuild's skewed layout for a W x H plane
inline size_t rice_skew_size(int W, int H) {
    const size_t strips = (size_t)((H + 31) / 32) * (size_t)(W + 31) * 32;
    const size_t diags = (size_t)(W + H - 1) * (size_t)H;
    return strips > diags ? strips : diags;
}

// bytes `stream` must hold for a W x H plane: the cheapest k costs at most
// what k = 8 does (<= 10 bits per symbol for zz <= 510), plus a spill word
inline long long rice_stream_bound(int W, int H) {
    return ((long long)W * H * 10 + 31) / 32 * 4 + 8;
}

}  // namespace fvv
