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
enum WDtype { kF32 = 0, kBF16 = 1, kI8 = 2, kNF4 = 3 };
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

// Weight layout in HBM for bf16 / int8 ("core-matrix tiles", DESIGN.md
// "weights in HBM").  Rows (output channels) come in groups of 128; within a
// group the K dimension is cut into units of 32 bytes, each unit stored as
// 2 x 16 core matrices of 8 rows x 16 bytes (128 contiguous bytes):
//   offset(n, kb) = ((g*KT + kt)*2 + kc)*2048 + r8*128 + rr*16 + b
//   g = n/128, r8 = (n%128)/8, rr = n%8, kt = kb/32, kc = (kb%32)/16, b = kb%16
// (kb = byte offset along K: k for int8, 2k for bf16; KT = K bytes / 32).
// One decode unit (128 rows x 32 B = 4 KB) is contiguous -> one TMA bulk copy;
// ldmatrix.x4 on it yields mma.m16n8k32 (int8) / m16n8k16 (bf16) A fragments;
// and the same bytes are the UMMA canonical K-major SWIZZLE_NONE layout
// (LBO = 2048 B between K-adjacent core matrices, SBO = 128 B between
// row-adjacent ones) for the tcgen05 prefill GEMM.
constexpr int kGroupRows = 128;
__host__ __device__ __forceinline__ int64_t cm_offset(int64_t n, int64_t kb, int64_t Kbytes) {
  const int64_t g = n >> 7, r8 = (n & 127) >> 3, rr = n & 7;
  const int64_t kt = kb >> 5, kc = (kb & 31) >> 4, b = kb & 15;
  return ((g * (Kbytes >> 5) + kt) * 2 + kc) * 2048 + r8 * 128 + rr * 16 + b;
}

// the same layout with rt-row tiles instead of 128 (rt a multiple of 8): the
// wide-decode digit planes use rt = 16 / 32 so a tile's rows are contiguous
__host__ __device__ __forceinline__ int64_t cm_offset_rt(int64_t n, int64_t kb, int64_t Kbytes,
                                                         int rt) {
  const int64_t g = n / rt, r8 = (n % rt) >> 3, rr = n & 7;
  const int64_t kt = kb >> 5, kc = (kb & 31) >> 4, b = kb & 15;
  return ((g * (Kbytes >> 5) + kt) * 2 + kc) * (int64_t)(rt * 16) + r8 * 128 + rr * 16 + b;
}

// NF4 weights (oracle/model.py quantize_columns_nf4): 4-bit codes in units of
// 128 output channels x 64 k (4 KB, the same unit size as int8), stored in the
// decode GEMV's mma.m16n8k32 A-fragment order so a lane's 16-byte load holds
// its two k-steps of one 16-row tile: byte ((t*32 + lane)*16 + s*8 + reg*2 +
// e/2), low nibble for even e, with t = 16-row tile, lane = g8*4 + t4,
// reg = h + 2*kc (A register), s = 32-k step.  Block scales (uint8, one per
// channel per 64 k) follow all codes, 128 per unit ordered [g8][t][h].
// CB7 = rint(63 * NF4 level); A operand = CB7 + 63 (7-bit, unsigned).
__host__ __device__ __forceinline__ int64_t nf4_offset(int64_t n, int64_t k, int64_t K, int* nib) {
  const int64_t unit = (n >> 7) * (K >> 6) + (k >> 6);
  const int rr = (int)(n & 127), t = rr >> 4, h = (rr >> 3) & 1, g8 = rr & 7;
  const int kk = (int)(k & 63), st = kk >> 5, kc = (kk >> 4) & 1, t4 = (kk >> 2) & 3, e = kk & 3;
  *nib = e & 1;
  return unit * 4096 + (t * 32 + g8 * 4 + t4) * 16 + st * 8 + (h + 2 * kc) * 2 + (e >> 1);
}
__host__ __device__ __forceinline__ int64_t nf4_qs_offset(int64_t n, int64_t k, int64_t N, int64_t K) {
  const int64_t unit = (n >> 7) * (K >> 6) + (k >> 6);
  const int rr = (int)(n & 127);
  return N * K / 2 + unit * 128 + (rr & 7) * 16 + (rr >> 4) * 2 + ((rr >> 3) & 1);
}
__host__ __device__ __forceinline__ int nf4_cb7(int c) {
  // CB7 + 63 as bytes of two 64-bit words (register shifts, no local-memory table)
  constexpr unsigned long long lo = 0x3F39332D261E1300ull, hi = 0x7E6D625B544F4944ull;
  c &= 15;
  return (int)(((c < 8 ? lo : hi) >> (8 * (c & 7))) & 0xFF) - 63;
}
// NF4 level bytes (CB7 + 63, common.cuh) for prmt lookups: entries 0-7, 8-15
constexpr uint32_t kLA0 = 0u | 19u << 8 | 30u << 16 | 38u << 24;
constexpr uint32_t kLA1 = 45u | 51u << 8 | 57u << 16 | 63u << 24;
constexpr uint32_t kLB0 = 68u | 73u << 8 | 79u << 16 | 84u << 24;
constexpr uint32_t kLB1 = 91u | 98u << 8 | 109u << 16 | 126u << 24;
__device__ __forceinline__ uint32_t prmt_b32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// four 4-bit codes (the selector nibbles of `sel`) -> four level bytes: a nibble
// >= 8 selects, with its msb set, the replicated sign (0) of a table byte in
// the first lookup, and entry c - 8 of the second (and vice versa)
__device__ __forceinline__ uint32_t nf4_expand(uint32_t sel) {
  return prmt_b32(kLA0, kLA1, sel) | prmt_b32(kLB0, kLB1, sel ^ 0x8888u);
}

// bytes of an N x K NF4 matrix (codes + block scales)
__host__ __device__ __forceinline__ int64_t nf4_bytes(int64_t N, int64_t K) {
  return N * K / 2 + N * K / 64;
}

// 2^x on the SFU (MUFU.EX2, ~2^-22 relative error): the bf16-class softmax of
// the attention kernels; exp2f() carries a multi-instruction accurate path
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// device-side phase tracing (tools): compiled in only with -DSP_DEV_TRACE=1
#ifndef SP_DEV_TRACE
#define SP_DEV_TRACE 0
#endif

// host-side count of kernels launched by this library (bench `gpu_launches`)
void count_launch();

// kernel attributes (max dynamic smem) are per device: launchers remember
// them per device index
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < kMaxDevices ? d : kMaxDevices - 1;
}

// ---- programmatic dependent launch (decode chain) ----------------------------
// A kernel launched with launch_pdl() may start while the previous kernel in
// the stream is still running: everything before pdl_wait() must touch only
// data no earlier kernel of the chain writes (weights, old KV rows, page
// tables); pdl_wait() returns once the previous grid has completed and its
// memory is visible.  pdl_trigger() lets the next grid be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
extern bool g_pdl;   // sp_span_set_option(.., 1, ..): decode kernels use PDL (default on)

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// launch_pdl() with a thread-block cluster of `cy` CTAs along grid.y
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t st, int cy, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = cy;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

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

// Every ABI entry point that touches a device makes the span's (or head's)
// device current for the duration of the call and restores the caller's
// device on return (several GPUs in one process; destructors run at GC time).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

