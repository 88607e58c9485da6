// Prefill / replay linear layers (n_new > 1) — SIMT fp32 tile GEMM.
//
// y[m, n] = sum_k x[m, k] * W[n, k]: 64x64 output tiles, k-steps of 16 staged
// in shared memory; every output is accumulated by one thread in ascending k
// (FFMA chain), so a row's result does not depend on M or on its tile
// position (the micro-batch invariance of T/test_server.py:247-255).
// This is the exact-f32 path (the reference computes in f32, SP/model.py:9);
// the tensor-core prefill GEMM (gemm_tc.cu) takes over for bf16/int8 weights.
#include "common.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__device__ __forceinline__ float load_w(const LinearArgs& a, int64_t n, int64_t k) {
  if (a.wdtype == kF32) return reinterpret_cast<const float*>(a.w)[n * a.K + k];
  if (a.wdtype == kBF16)
    return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
        reinterpret_cast<const uint8_t*>(a.w) + cm_offset(n, 2 * k, 2 * a.K)));
  if (a.wdtype == kNF4) {   // exact integer CB7 * q; channel scale in the epilogue
    int nib;
    const uint8_t* b = reinterpret_cast<const uint8_t*>(a.w);
    const int code = (b[nf4_offset(n, k, a.K, &nib)] >> (4 * nib)) & 15;
    return (float)(nf4_cb7(code) * (int)b[nf4_qs_offset(n, k, a.N, a.K)]);
  }
  int q = (int)reinterpret_cast<const int8_t*>(a.w)[cm_offset(n, k, a.K)];
  return (float)q;  // per-row scale applied in the epilogue
}

__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

__global__ void __launch_bounds__(256) gemm_simt_kernel(LinearArgs a) {
  __shared__ float Xs[BK][BM + 4];
  __shared__ float Ws[BK][BN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = 0; k0 < a.K; k0 += BK) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      int idx = threadIdx.x + l * 256;  // 0..1023
      int mm = idx >> 4, kk = idx & 15;
      int64_t m = m0 + mm;
      Xs[kk][mm] = (m < a.R) ? a.x[m * a.ldx + k0 + kk] : 0.f;
      int64_t n = n0 + mm;
      Ws[kk][mm] = (n < a.N) ? load_w(a, n, k0 + kk) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float xv[4], wv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = Xs[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xv[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t m = m0 + ty * 4 + i;
    if (m >= a.R) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t n = n0 + tx * 4 + j;
      if (n >= a.N) continue;
      float v = acc[i][j];
      if (a.wdtype == kI8 || a.wdtype == kNF4) v *= a.wscale[n];
      float* dst = a.y + m * a.ldy + n;
      if (a.epi == EPI_RESID) v = a.res[m * a.ldy + n] + v;
      else if (a.epi == EPI_GELU) v = gelu_f(v);
      *dst = v;
    }
  }
}

__global__ void swiglu_rows_kernel(const float* in, float* out, int64_t R, int64_t F) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R * F) return;
  int64_t r = i / F, j = i % F;
  int64_t ng = (j / 64) * 128 + (j % 64);
  float g = in[r * 2 * F + ng], u = in[r * 2 * F + ng + 64];
  out[i] = silu_f(g) * u;
}

}  // namespace

void launch_gemm(const LinearArgs& a, cudaStream_t st) {
  dim3 grid((unsigned)((a.N + BN - 1) / BN), (unsigned)((a.R + BM - 1) / BM));
  gemm_simt_kernel<<<grid, 256, 0, st>>>(a); count_launch();
}

void launch_swiglu_rows(const float* in, float* out, int64_t R, int64_t F, cudaStream_t st) {
  int64_t n = R * F;
  if (n == 0) return;
  swiglu_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, out, R, F); count_launch();
}

}  // namespace sp
