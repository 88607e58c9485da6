// Decode linear layers for f32 weights (the reference toy model, which is
// computed in f32 end to end, SP/model.py:9 and SURVEY.md §0.8): warp per
// output channel, fixed shuffle-tree reduction (deterministic, batch-invariant).
// bf16 / int8 weights use the tensor-pipe GEMV in gemv3.cu.
#include "common.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

__device__ __forceinline__ void epi_store(const LinearArgs& a, int r, int64_t n, float v) {
  float* dst = a.y + (int64_t)r * a.ldy + n;
  if (a.epi == EPI_RESID) v = a.res[(int64_t)r * a.ldy + n] + v;
  else if (a.epi == EPI_GELU) v = gelu_f(v);
  *dst = v;
}

__global__ void __launch_bounds__(256) gemv_f32_kernel(LinearArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t o = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const float* W = reinterpret_cast<const float*>(a.w);
  if (a.epi == EPI_SWIGLU) {
    const int64_t F = a.N / 2;
    if (o >= F) return;
    const int64_t ng = (o / 64) * 128 + (o % 64), nu = ng + 64;
    for (int r = 0; r < a.R; ++r) {
      const float* x = a.x + (int64_t)r * a.ldx;
      float sg = 0.f, su = 0.f;
      for (int64_t k = lane; k < a.K; k += 32) {
        float xv = x[k];
        sg = fmaf(W[ng * a.K + k], xv, sg);
        su = fmaf(W[nu * a.K + k], xv, su);
      }
      sg = warp_sum(sg);
      su = warp_sum(su);
      if (lane == 0) a.y[(int64_t)r * a.ldy + o] = silu_f(sg) * su;
    }
    return;
  }
  if (o >= a.N) return;
  for (int r = 0; r < a.R; ++r) {
    const float* x = a.x + (int64_t)r * a.ldx;
    float sacc = 0.f;
    for (int64_t k = lane; k < a.K; k += 32) sacc = fmaf(W[o * a.K + k], x[k], sacc);
    sacc = warp_sum(sacc);
    if (lane == 0) epi_store(a, r, o, sacc);
  }
}

}  // namespace

void launch_gemv(const LinearArgs& a, cudaStream_t st) {
  int64_t outs = (a.epi == EPI_SWIGLU) ? a.N / 2 : a.N;
  gemv_f32_kernel<<<(unsigned)((outs + 7) / 8), 256, 0, st>>>(a);
  count_launch();
}

}  // namespace sp
