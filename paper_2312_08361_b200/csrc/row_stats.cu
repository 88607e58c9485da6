// Span-input row statistics for the first decode GEMV's folded pre-norm:
// P = d/128 fixed-slot partials {sum, sumsq, max|x*g|} per row, the layout the
// GEMV epilogues write for the next consumer (decode.cuh RowStat).
#include "common.cuh"
#include "decode.cuh"

namespace sp {

namespace {

__global__ void row_stats_kernel(const float* x, int64_t d, const float* g, RowStat* st, int Rs) {
  const int p = blockIdx.x, r = blockIdx.y;
  const int t = threadIdx.x;   // 128 threads: one element each
  __shared__ float vs[128], vg[128];
  const int64_t k = (int64_t)p * 128 + t;
  float v = x[(int64_t)r * d + k];
  vs[t] = v;
  vg[t] = fabsf(v * (g ? g[k] : 1.f));
  __syncthreads();
  if (t == 0) {            // fixed order: deterministic partials
    float S = 0.f, Q = 0.f, M = 0.f;
    for (int i = 0; i < 128; ++i) {
      S += vs[i];
      Q = fmaf(vs[i], vs[i], Q);
      M = fmaxf(M, vg[i]);
    }
    st[(int64_t)p * Rs + r] = RowStat{S, Q, M, 0.f};
  }
}

}  // namespace

void launch_row_stats(const float* x, int R, int64_t d, const float* g_next, RowStat* st_out,
                      cudaStream_t st) {
  dim3 grid((unsigned)(d / 128), (unsigned)R);
  row_stats_kernel<<<grid, 128, 0, st>>>(x, d, g_next, st_out, R);
  count_launch();
}

}  // namespace sp
