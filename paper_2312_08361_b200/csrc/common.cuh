// Shared device helpers for the span-forward kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/spanpipe.h"

namespace sp {

constexpr int kWarp = 32;
constexpr int kPageTokens = 64;      // KV page = 64 positions of one block
constexpr int kCodecBlock = 64;      // SP/quantize.py:15

enum Family { kToy = 0, kLlama = 1, kBloom = 2 };
enum WDtype { kF32 = 0, kBF16 = 1, kI8 = 2 };
enum KVDtype { kKVF32 = 0, kKVBF16 = 1 };

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// splitmix64, SP/model.py:40-46 in counter form: output number (i+1) of the
// stream started at `seed` is mix((i+1)*GOLDEN + seed).
__host__ __device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t i) {
  uint64_t z = (i + 1ull) * 0x9E3779B97F4A7C15ull + seed;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// SP/model.py:55-60: u = (bits >> 11) * 2^-53 (exact), ((2u - 1) * scale) in
// f64, then one f64 -> f32 round-to-nearest.  Written with explicit _rn
// intrinsics so no FMA contraction changes the rounding.
__device__ __forceinline__ float uniform_value(uint64_t stream, uint64_t idx, double scale) {
  uint64_t bits = splitmix64_at(stream, idx);
  double u = __dmul_rn((double)(bits >> 11), 1.0 / 9007199254740992.0);
  double c = __dadd_rn(__dmul_rn(2.0, u), -1.0);  // exact
  return __double2float_rn(__dmul_rn(c, scale));
}

__device__ __forceinline__ float bf16_to_f32(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }

// Fragment-tiled weight layout of the tensor-core decode GEMV (DESIGN.md
// "weights in HBM").  A tile is 512 bytes = 32 lanes x 16 B and lane L's 16
// bytes are exactly its mma A fragment, so a coalesced LDG.128 per lane feeds
// the MMA with no shuffles or shared-memory staging.  Tiles are row-tile major:
// tile(rt, kt) at ((rt * KT) + kt) * 512 B.
//   bf16: tile = 16 rows x 16 k, mma.m16n8k16 A layout (lane = g*4+t holds
//         rows g, g+8 x k {2t, 2t+1, 2t+8, 2t+9})
//   int8: tile = 16 rows x 32 k, mma.m16n8k32 s8 A layout (lane = g*4+t holds
//         4-byte groups: (g, 4t..), (g+8, 4t..), (g, 16+4t..), (g+8, 16+4t..))
__host__ __device__ __forceinline__ int64_t frag_offset_bf16(int64_t n, int64_t k, int64_t K) {
  const int i = (int)(n & 15), j = (int)(k & 15);
  const int g = i & 7, hi = i >> 3, c4 = (j & 7) >> 1, jj = j & 1, k8 = j >> 3;
  const int lane = g * 4 + c4, pos = (k8 * 2 + hi) * 2 + jj;
  return (((n >> 4) * (K >> 4) + (k >> 4)) << 8) + lane * 8 + pos;
}
__host__ __device__ __forceinline__ int64_t frag_offset_i8(int64_t n, int64_t k, int64_t K) {
  const int i = (int)(n & 15), j = (int)(k & 31);
  const int g = i & 7, hi = i >> 3, t = (j & 15) >> 2, q = j & 3, k16 = j >> 4;
  const int lane = g * 4 + t, reg = k16 * 2 + hi;
  return (((n >> 4) * (K >> 5) + (k >> 5)) << 9) + lane * 16 + reg * 4 + q;
}

// host-side count of kernels launched by this library (bench `gpu_launches`)
void count_launch();

}  // namespace sp

#define SP_CUDA_TRY(expr)                                       \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) {                                    \
      sp_set_error(__FILE__, __LINE__, cudaGetErrorString(_e)); \
      return SP_ERR_CUDA;                                       \
    }                                                           \
  } while (0)

void sp_set_error(const char* file, int line, const char* msg);
