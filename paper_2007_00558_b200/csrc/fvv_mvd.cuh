// MVD disk-container rasters on the device (fvv_mvd.cu): the 16-bit mm
// quantisation of a depth frame (core.depth_to_millimeters, core.py:246-255)
// and the run-length code of the validity sidecar (mvdio.rle_encode /
// rle_decode, mvdio.py:34-52).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fvv {

constexpr int kRlePx = 1024;   // pixels per run-boundary block (256 threads x 4)

// per-context scratch of the run-length encoder
struct RleScratch {
    unsigned long long *block = nullptr;  // [blocks + 1] boundary counts -> offsets
    long long *n_runs = nullptr;          // [1]
    size_t cap = 0;                       // blocks allocated
};

// mm[i] = Valid ? clip(rint(f32(depth * 1000)), 1, 65535) : 0
cudaError_t launch_encode_mm(const float *depth, const uint8_t *validity, long long n,
                             uint16_t *mm, cudaStream_t s);

// out[i] = code of the run whose half-open [end[r-1], end[r]) holds i
cudaError_t launch_rle_decode(const uint8_t *codes, const long long *ends, long long n_runs,
                              long long n, uint8_t *out, cudaStream_t s);

// run starts (ascending) and codes of flat[0..n); *n_runs on the device.
// starts / codes need room for n entries (the worst case); sc sized for n.
cudaError_t launch_rle_encode(const uint8_t *flat, long long n, long long *starts,
                              uint8_t *codes, const RleScratch &sc, cudaStream_t s);

}  // namespace fvv
