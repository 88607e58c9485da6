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

__global__ void gelu_rows_kernel(const float* in, float* out, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = gelu_f(in[i]);
}

// one warp = one nf4 unit (128 channels x 64 k): the 4 KB of codes are read in
// their fragment order (lane L, tile t: 16 bytes at (t*32 + L)*16, coalesced),
// each lane writes 4-byte runs of both int8 planes; 8 lanes (g8) cover 128
// contiguous bytes of a core-matrix column, so the stores are coalesced too
__global__ void nf4_split_kernel(const uint8_t* __restrict__ w, const float* __restrict__ sc,
                                 int64_t N, int64_t K, int8_t* hi, int8_t* lo, float* sc128) {
  const int64_t unit = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t KT = K >> 6;
  if (unit >= (N >> 7) * KT) return;
  const int64_t grp = unit / KT, kt = unit % KT;
  const int g8 = lane >> 2, t4 = lane & 3;
  const uint4 qv = *reinterpret_cast<const uint4*>(w + N * K / 2 + unit * 128 + g8 * 16);
  const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w};
  const uint8_t* base = w + unit * 4096;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const uint4 wv = *reinterpret_cast<const uint4*>(base + (t * 32 + lane) * 16);
    const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int reg = 0; reg < 4; ++reg) {
        const int h = reg & 1, kc = reg >> 1;
        const uint32_t lv = nf4_expand(ww[2 * s + (reg >> 1)] >> (16 * (reg & 1)));  // CB7 + 63
        const int q = (qw[t >> 1] >> (16 * (t & 1) + 8 * h)) & 0xFF;
        const int q63 = 63 * q;
        uint32_t ph = 0, pl = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int v = (int)((lv >> (8 * e)) & 0xFF) * q - q63;     // CB7 * q, |v| <= 16065
          const int vh = (v + 64) >> 7;                                 // floor((v + 64) / 128)
          ph |= (uint32_t)(uint8_t)(int8_t)vh << (8 * e);
          pl |= (uint32_t)(uint8_t)(int8_t)(v - vh * 128) << (8 * e);   // [-64, 63]
        }
        const int64_t r = grp * 128 + t * 16 + h * 8 + g8;
        const int64_t k = kt * 64 + s * 32 + kc * 16 + t4 * 4;
        const int64_t off = cm_offset(r, k, K);
        *reinterpret_cast<uint32_t*>(hi + off) = ph;
        *reinterpret_cast<uint32_t*>(lo + off) = pl;
      }
  }
  if (kt == 0)
    for (int rr = lane; rr < 128; rr += 32) sc128[grp * 128 + rr] = 128.0f * sc[grp * 128 + rr];
}

}  // namespace

void launch_gelu_rows(const float* in, float* out, int64_t R, int64_t F, cudaStream_t st) {
  const int64_t n = R * F;
  if (n == 0) return;
  gelu_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, out, n); count_launch();
}

void launch_nf4_split(const uint8_t* w, const float* sc, int64_t N, int64_t K, int8_t* hi,
                      int8_t* lo, float* sc128, cudaStream_t st) {
  const int64_t warps = (N >> 7) * (K >> 6);
  nf4_split_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(w, sc, N, K, hi, lo, sc128);
  count_launch();
}

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
