// Blockwise absmax int8 hidden-state codec — bit-exact with SP/quantize.py:36-58.
//
// One warp per 64-element block (2 elements per lane).  Arithmetic mirrors
// numpy exactly:  scale = f32(absmax / 127)  (IEEE division, __fdiv_rn),
// code = rint(x / scale) (f32 division, round-half-even = __float2int_rn),
// scale 0 -> all codes 0; dequant = f32(code) * scale (single rounding).
// HBM-bound: 4 B read + 1.0625 B written per element.
#include "common.cuh"
#include "kernels.cuh"

namespace sp {

__global__ void __launch_bounds__(256) quantize_kernel(const float* __restrict__ x,
                                                       int8_t* __restrict__ codes,
                                                       float* __restrict__ scales, int64_t n) {
  int64_t blk = (int64_t)blockIdx.x * (blockDim.x / kWarp) + threadIdx.x / kWarp;
  int lane = threadIdx.x & 31;
  int64_t nblk = (n + kCodecBlock - 1) / kCodecBlock;
  if (blk >= nblk) return;
  int64_t i0 = blk * kCodecBlock + lane * 2;
  float a = (i0 < n) ? x[i0] : 0.f;
  float b = (i0 + 1 < n) ? x[i0 + 1] : 0.f;
  float m = warp_max(fmaxf(fabsf(a), fabsf(b)));
  float s = __fdiv_rn(m, 127.0f);
  int ca = 0, cb = 0;
  if (s > 0.f) {
    ca = __float2int_rn(__fdiv_rn(a, s));
    cb = __float2int_rn(__fdiv_rn(b, s));
  }
  if (i0 < n) codes[i0] = (int8_t)ca;
  if (i0 + 1 < n) codes[i0 + 1] = (int8_t)cb;
  if (lane == 0) scales[blk] = s;
}

__global__ void __launch_bounds__(256) dequantize_kernel(const int8_t* __restrict__ codes,
                                                         const float* __restrict__ scales,
                                                         float* __restrict__ x, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  x[i] = __fmul_rn((float)codes[i], scales[i / kCodecBlock]);
}

void launch_quantize(const float* x, int8_t* codes, float* scales, int64_t n, cudaStream_t st) {
  int64_t nblk = (n + kCodecBlock - 1) / kCodecBlock;
  if (nblk == 0) return;
  int64_t grid = (nblk + 7) / 8;
  quantize_kernel<<<(unsigned)grid, 256, 0, st>>>(x, codes, scales, n); count_launch();
}

void launch_dequantize(const int8_t* codes, const float* scales, float* x, int64_t n,
                       cudaStream_t st) {
  if (n == 0) return;
  dequantize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(codes, scales, x, n); count_launch();
}

}  // namespace sp
