// Deterministic weight generation on the GPU, bit-identical to the reference
// recipe (SP/model.py:40-60 splitmix64 streams, f64 affine map, f64->f32 RN),
// plus the bf16 / int8 roundings defined in oracle/model.py:
//   bf16: round-to-nearest-even of the f32 value
//   int8: per output channel scale = f32(absmax/127), code = rint(w/scale)
//         (the SP/quantize.py:43-47 arithmetic, one channel = one block)
//   nf4:  oracle/model.py quantize_columns_nf4 (codes + uint8 block scales +
//         f32 channel scale, layout common.cuh nf4_offset)
//
// Reference orientation is x @ W with W [d_in = K, d_out = N] row-major, i.e.
// element (k, n) is stream index k*N + n.  Storage here is output-major
// [N][K] (row per output channel), f32 plain or bf16/int8 fragment-tiled.
#include "common.cuh"
#include "kernels.cuh"

namespace sp {

__global__ void gen_stream_kernel(uint64_t stream, int64_t n, double scale, float* dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = uniform_value(stream, (uint64_t)i, scale);
}

// buffer row of output channel n for a matrix placed at `row0` with 16-row
// tiles interleaved every `tstride` tiles at tile offset `toff`
__device__ __forceinline__ int64_t buf_row(int64_t n, const MatPlace& p) {
  return p.row0 + ((n / kPlaceGranule) * p.tstride + p.toff) * kPlaceGranule + (n % kPlaceGranule);
}

// f32 storage, row-major [rows][K]
__global__ void gen_f32_rows_kernel(uint64_t stream, int64_t K, int64_t N, double scale,
                                    MatPlace place, float* dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K * N) return;
  int64_t n = i / K, k = i % K;
  dst[buf_row(n, place) * K + k] = uniform_value(stream, (uint64_t)(k * N + n), scale);
}

// int8 pass 1: per-output-channel absmax -> scale (warp per channel)
__global__ void gen_i8_scales_kernel(uint64_t stream, int64_t K, int64_t N, double scale,
                                     MatPlace place, float* scales) {
  int64_t n = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  int lane = threadIdx.x & 31;
  if (n >= N) return;
  float m = 0.f;
  for (int64_t k = lane; k < K; k += 32)
    m = fmaxf(m, fabsf(uniform_value(stream, (uint64_t)(k * N + n), scale)));
  m = warp_max(m);
  if (lane == 0) scales[buf_row(n, place)] = __fdiv_rn(m, 127.0f);
}

// int8 pass 2: one thread writes one 16-byte core-matrix row (16 k of one
// output channel), layout common.cuh cm_offset
__global__ void gen_i8_pack_kernel(uint64_t stream, int64_t K, int64_t N, double scale,
                                   MatPlace place, const float* __restrict__ scales,
                                   int8_t* dst) {
  const int64_t chunk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // (n, k16)
  const int64_t KC = K >> 4;
  if (chunk >= N * KC) return;
  const int64_t n = chunk / KC, k0 = (chunk % KC) * 16;
  const int64_t r = buf_row(n, place);
  const float s = scales[r];
  __align__(16) int8_t out[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int64_t k = k0 + q;
    const float w = uniform_value(stream, (uint64_t)(k * N + n), scale);
    out[q] = (int8_t)((s > 0.f) ? __float2int_rn(__fdiv_rn(w, s)) : 0);
  }
  *reinterpret_cast<uint4*>(dst + cm_offset(r, k0, K)) = *reinterpret_cast<uint4*>(out);
}

// bf16: one thread writes one 16-byte core-matrix row (8 k of one channel)
__global__ void gen_bf16_pack_kernel(uint64_t stream, int64_t K, int64_t N, double scale,
                                     MatPlace place, __nv_bfloat16* dst) {
  const int64_t chunk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // (n, k8)
  const int64_t KC = K >> 3;
  if (chunk >= N * KC) return;
  const int64_t n = chunk / KC, k0 = (chunk % KC) * 8;
  const int64_t r = buf_row(n, place);
  __align__(16) __nv_bfloat16 out[8];
#pragma unroll
  for (int q = 0; q < 8; ++q)
    out[q] = __float2bfloat16_rn(uniform_value(stream, (uint64_t)((k0 + q) * N + n), scale));
  *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(dst) + cm_offset(r, 2 * k0, 2 * K)) =
      *reinterpret_cast<uint4*>(out);
}

// nf4: one warp per output channel — channel absmax -> f32 channel scale, then
// each lane quantises whole 64-wide blocks (uint8 block scale + 64 codes,
// oracle/model.py quantize_columns_nf4 arithmetic, same IEEE roundings)
__global__ void gen_nf4_kernel(uint64_t stream, int64_t K, int64_t N, double scale,
                               MatPlace place, int64_t nbuf, uint8_t* dst, float* scales) {
  const int64_t n = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  const int64_t r = buf_row(n, place);
  float m = 0.f;
  for (int64_t k = lane; k < K; k += 32)
    m = fmaxf(m, fabsf(uniform_value(stream, (uint64_t)(k * N + n), scale)));
  m = warp_max(m);
  const float sr = m > 0.f ? __fdiv_rn(m, 16065.0f) : 0.f;
  if (lane == 0) scales[r] = sr;
  for (int64_t blk = lane; blk < K / 64; blk += 32) {
    float w[64];
    float a = 0.f;
#pragma unroll
    for (int e = 0; e < 64; ++e) {
      w[e] = uniform_value(stream, (uint64_t)((blk * 64 + e) * N + n), scale);
      a = fmaxf(a, fabsf(w[e]));
    }
    const int q = m > 0.f ? __float2int_rn(__fdiv_rn(__fmul_rn(255.0f, a), m)) : 0;
#pragma unroll
    for (int g = 0; g < 16; ++g) {
      uint32_t packed = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        int best = 7;
        if (q > 0) {
          const float t = __fdiv_rn(w[g * 4 + e], sr);
          float bd = fabsf(__fsub_rn(t, (float)(nf4_cb7(0) * q)));
          best = 0;
#pragma unroll
          for (int c = 1; c < 16; ++c) {
            const float dd = fabsf(__fsub_rn(t, (float)(nf4_cb7(c) * q)));
            if (dd < bd) { bd = dd; best = c; }
          }
        }
        packed |= (uint32_t)best << (4 * e);
      }
      int nib;
      *reinterpret_cast<uint16_t*>(dst + nf4_offset(r, blk * 64 + g * 4, K, &nib)) = (uint16_t)packed;
    }
    dst[nf4_qs_offset(r, blk * 64, nbuf, K)] = (uint8_t)q;
  }
}

void launch_gen_stream(uint64_t stream, int64_t n, double scale, float* dst, cudaStream_t st) {
  if (n <= 0) return;
  gen_stream_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(stream, n, scale, dst); count_launch();
}

void launch_gen_matrix(int wdtype, uint64_t stream, int64_t K, int64_t N, double scale,
                       MatPlace place, void* dst, float* scales, cudaStream_t st, int64_t nbuf) {
  if (wdtype == kNF4) {
    gen_nf4_kernel<<<(unsigned)((N + 7) / 8), 256, 0, st>>>(stream, K, N, scale, place, nbuf,
                                                             (uint8_t*)dst, scales); count_launch();
  } else if (wdtype == kF32) {
    int64_t n = K * N;
    gen_f32_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(stream, K, N, scale, place,
                                                                      (float*)dst); count_launch();
  } else if (wdtype == kBF16) {
    int64_t chunks = N * (K / 8);
    gen_bf16_pack_kernel<<<(unsigned)((chunks + 255) / 256), 256, 0, st>>>(
        stream, K, N, scale, place, (__nv_bfloat16*)dst); count_launch();
  } else {
    gen_i8_scales_kernel<<<(unsigned)((N + 7) / 8), 256, 0, st>>>(stream, K, N, scale, place,
                                                                   scales); count_launch();
    int64_t chunks = N * (K / 16);
    gen_i8_pack_kernel<<<(unsigned)((chunks + 255) / 256), 256, 0, st>>>(
        stream, K, N, scale, place, scales, (int8_t*)dst); count_launch();
  }
}

// read back: dst [K][N] f32 (reference orientation), effective values
__global__ void read_matrix_kernel(int wdtype, const void* src, const float* scales, int64_t K,
                                   int64_t N, int64_t bufK, MatPlace place, int64_t nbuf,
                                   float* dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K * N) return;
  int64_t k = i / N, n = i % N;
  int64_t r = buf_row(n, place);
  float v;
  if (wdtype == kF32) {
    v = ((const float*)src)[r * bufK + k];
  } else if (wdtype == kBF16) {
    v = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
        (const uint8_t*)src + cm_offset(r, 2 * k, 2 * bufK)));
  } else if (wdtype == kNF4) {
    int nib;
    const uint8_t* b = (const uint8_t*)src;
    const int code = (b[nf4_offset(r, k, bufK, &nib)] >> (4 * nib)) & 15;
    const int q = b[nf4_qs_offset(r, k, nbuf, bufK)];
    v = __fmul_rn((float)(nf4_cb7(code) * q), scales[r]);
  } else {
    int q = (int)((const int8_t*)src)[cm_offset(r, k, bufK)];
    v = __fmul_rn((float)q, scales[r]);
  }
  dst[i] = v;
}

void launch_read_matrix(int wdtype, const void* src, const float* scales, int64_t K, int64_t N,
                        MatPlace place, float* dst, cudaStream_t st, int64_t nbuf) {
  int64_t n = K * N;
  read_matrix_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(wdtype, src, scales, K, N, K,
                                                                   place, nbuf, dst); count_launch();
}

}  // namespace sp
