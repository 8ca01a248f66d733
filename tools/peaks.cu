// Measured B200 peaks for the limits SURVEY.md §8(d) names besides HBM:
//   * L2 64-bit atomicMin throughput (RED.E.MIN.64, no return value) — the
//     z-buffer scatter of K2 (replaces synthesis.py:196-205's np.minimum.at);
//   * FP64 rates (DFMA, DMUL, DADD, correctly rounded DDIV) — the parity
//     geometry of K2/K3 (core.py:160-227 in float64);
//   * FP32 FFMA issue rate — the SM's instruction-issue ceiling that K3 hits.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu
//   /tmp/peaks > profiles/r02_peaks.json
//
// Each figure is the best of 5 CUDA-event-timed launches after 2 warm-ups,
// grids of 148 x (resident CTAs per SM); one JSON object on stdout.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// mode 0: every lane an independent uniformly random canvas cell
// mode 1: a warp's 32 lanes hit 32 consecutive cells at a random base
//         (K2's pattern: consecutive source pixels land on consecutive targets)
// mode 2: as 1, but lanes pair up on 16 cells (z-collisions)
// mode 3: a warp's 32 lanes hit 8 cells 4 lanes each
__global__ void k_red_min64(unsigned long long* canvas, uint32_t cells, int iters, int mode,
                            uint32_t seed) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31, warp = tid >> 5;
  for (int i = 0; i < iters; ++i) {
    uint32_t cell;
    if (mode == 0) {
      cell = hash32(tid * 0x9E3779B9U + i * 0x85EBCA6BU + seed) % cells;
    } else {
      uint32_t base = hash32(warp * 0x9E3779B9U + i * 0x85EBCA6BU + seed) % (cells - 32);
      cell = base + (mode == 1 ? lane : mode == 2 ? (lane >> 1) : (lane >> 2));
    }
    unsigned long long key = ((unsigned long long)hash32(tid + i) << 32) | tid;
    atomicMin(canvas + cell, key);   // result unused -> RED.E.MIN.64
  }
}

template <int OP>
__global__ void k_fp64(double* out, int iters, double seed) {
  // 8 independent chains per thread so the pipe, not latency, is the limit
  double a[8];
  const double m = 1.0000001 + threadIdx.x * 1e-12, c = 1e-9;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + j + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] = fma(a[j], m, c);
      else if (OP == 1) a[j] = __dmul_rn(a[j], m);
      else a[j] = __dadd_rn(a[j], c);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_ddiv(double* out, int iters, double seed) {
  double a[4], b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { a[j] = seed + j + threadIdx.x; b[j] = 1.5 + 0.25 * j + 1e-6 * threadIdx.x; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = __ddiv_rn(a[j], b[j]) + 1.0;
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += a[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_ffma(float* out, int iters, float seed) {
  float a[8];
  const float m = 1.0000001f, c = 1e-7f;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + j + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], m, c);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.678f) out[0] = s;
}

template <class F>
static float best_ms(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_attr_mhz\": %.0f,\n", p.name, sms,
         clk_khz / 1e3);

  // ---- L2 64-bit atomicMin ----------------------------------------------
  const uint32_t sizes[2] = {1922u * 1082u, 3842u * 2162u};   // c1 / c4 padded canvases
  const char* size_name[2] = {"c1_canvas_16.6MB", "c4_canvas_66.5MB"};
  const char* mode_name[4] = {"random", "warp_consecutive", "pairs_colliding", "quads_colliding"};
  unsigned long long* canvas;
  CK(cudaMalloc(&canvas, sizes[1] * sizeof(unsigned long long)));
  const int threads = 256, blocks = sms * 8, iters = 256;
  const double ops = double(threads) * blocks * iters;
  printf("\"red_min_u64\": {\"unit\": \"G atomics/s\", \"atomics_per_launch\": %.0f", ops);
  for (int s = 0; s < 2; ++s) {
    for (int m = 0; m < 4; ++m) {
      CK(cudaMemset(canvas, 0xff, sizes[s] * sizeof(unsigned long long)));
      float ms = best_ms([&] {
        k_red_min64<<<blocks, threads>>>(canvas, sizes[s], iters, m, 12345u);
      });
      CK(cudaGetLastError());
      printf(", \"%s/%s\": %.2f", size_name[s], mode_name[m], ops / (ms * 1e-3) / 1e9);
    }
  }
  printf("},\n");

  // ---- FP64 / FP32 pipes ---------------------------------------------------
  double* dout;
  CK(cudaMalloc(&dout, 64));
  const int fb = sms * 8, ft = 256, fit = 4096;
  const double lanes_ops = double(fb) * ft * fit * 8;
  float ms_fma = best_ms([&] { k_fp64<0><<<fb, ft>>>(dout, fit, 1.0); });
  float ms_mul = best_ms([&] { k_fp64<1><<<fb, ft>>>(dout, fit, 1.0); });
  float ms_add = best_ms([&] { k_fp64<2><<<fb, ft>>>(dout, fit, 1.0); });
  const int dit = 512;
  float ms_div = best_ms([&] { k_ddiv<<<fb, ft>>>(dout, dit, 1.0); });
  float ms_ffma = best_ms([&] { k_ffma<<<fb, ft>>>((float*)dout, fit, 1.0f); });
  CK(cudaGetLastError());
  const double divs = double(fb) * ft * dit * 4;
  printf("\"fp64\": {\"dfma_per_s\": %.4g, \"tflops_fma\": %.3f, \"dmul_per_s\": %.4g, "
         "\"dadd_per_s\": %.4g, \"ddiv_rn_per_s\": %.4g},\n",
         lanes_ops / (ms_fma * 1e-3), 2 * lanes_ops / (ms_fma * 1e-3) / 1e12,
         lanes_ops / (ms_mul * 1e-3), lanes_ops / (ms_add * 1e-3), divs / (ms_div * 1e-3));
  const double warp_inst = lanes_ops / 32.0;
  printf("\"issue\": {\"ffma_lanes_per_s\": %.4g, \"ffma_warp_inst_per_s\": %.4g, "
         "\"warp_inst_per_clk_per_sm_at_attr_clock\": %.3f}\n}\n",
         lanes_ops / (ms_ffma * 1e-3), warp_inst / (ms_ffma * 1e-3),
         warp_inst / (ms_ffma * 1e-3) / (sms * clk_khz * 1e3));
  cudaFree(canvas);
  cudaFree(dout);
  return 0;
}
