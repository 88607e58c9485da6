// Client head on the GPU: the tied embedding
// (SP/model.py:196-198, splitmix64 role 11 keyed by block n_blocks,
// bit-identical), embedding gather (SP/model.py:388-391), tied logits
// row @ E^T (SP/model.py:393-395, no final norm) and greedy argmax with ties
// to the lowest id (SP/model.py:398-400).  Logits: warp per vocab row, fixed
// shuffle-tree reduction; argmax: fixed-order tree — deterministic.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

void sp_set_error(const char* file, int line, const char* msg);

namespace sp {
namespace {

__global__ void gen_embedding_kernel(uint64_t stream, int64_t n, double scale, float* dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = uniform_value(stream, (uint64_t)i, scale);
}

__global__ void gather_kernel(const float* E, const int* tok, int n, int d, float* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n * d) return;
  out[i] = E[(int64_t)tok[i / d] * d + i % d];
}

__global__ void logits_kernel(const float* E, const float* x, int vocab, int d, float* logits) {
  const int v = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (v >= vocab) return;
  const float* e = E + (int64_t)v * d;
  float s = 0.f;
  for (int k = lane; k < d; k += 32) s = fmaf(e[k], x[k], s);
  s = warp_sum(s);
  if (lane == 0) logits[v] = s;
}

// logits of R rows (beam search: SP/client.py:624, 634): warp per vocab row,
// the embedding row streamed once for all R rows
template <int R>
__global__ void logits_rows_kernel(const float* E, const float* x, int vocab, int d,
                                   float* logits) {
  const int v = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (v >= vocab) return;
  const float* e = E + (int64_t)v * d;
  float s[R];
#pragma unroll
  for (int r = 0; r < R; ++r) s[r] = 0.f;
  for (int k = lane; k < d; k += 32) {
    const float ev = e[k];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = fmaf(ev, x[(int64_t)r * d + k], s[r]);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const float t = warp_sum(s[r]);
    if (lane == 0) logits[(int64_t)r * vocab + v] = t;
  }
}

// single CTA: (max value, lowest index) over the vocabulary
__global__ void argmax_kernel(const float* logits, int vocab, int* out) {
  __shared__ float bv[1024];
  __shared__ int bi[1024];
  float best = -INFINITY;
  int idx = 0x7fffffff;
  for (int v = threadIdx.x; v < vocab; v += blockDim.x) {
    const float l = logits[v];
    if (l > best) { best = l; idx = v; }    // ascending v per thread: first max kept
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = idx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const float o = bv[threadIdx.x + s];
      const int oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = bi[0];
}

}  // namespace
}  // namespace sp

struct sp_head {
  int device, vocab, d;
  float* E = nullptr;
  float* logits = nullptr;
  int* tok = nullptr;
  float* row = nullptr;
};

extern "C" {

uint64_t sp_stream_seed(uint64_t seed, int32_t block, int32_t role_id);

int sp_head_create(const sp_config* cfg, int32_t device, sp_head** out) {
  if (!cfg || !out) return SP_ERR_ARG;
  DeviceGuard dg(device);
  sp_head* h = new sp_head();
  h->device = device;
  h->vocab = cfg->vocab_size;
  h->d = cfg->hidden_dim;
  const int64_t n = (int64_t)h->vocab * h->d;
  SP_CUDA_TRY(cudaMalloc(&h->E, n * sizeof(float)));
  SP_CUDA_TRY(cudaMalloc(&h->logits, h->vocab * sizeof(float)));
  SP_CUDA_TRY(cudaMalloc(&h->tok, 4096 * sizeof(int)));
  SP_CUDA_TRY(cudaMalloc(&h->row, (size_t)h->d * sizeof(float)));
  const double scale = 1.0 / std::sqrt((double)h->d);
  sp::gen_embedding_kernel<<<(unsigned)((n + 255) / 256), 256>>>(
      sp_stream_seed(cfg->seed, cfg->n_blocks, 11), n, scale, h->E);
  sp::count_launch();
  SP_CUDA_TRY(cudaDeviceSynchronize());
  *out = h;
  return SP_OK;
}

int sp_head_destroy(sp_head* h) {
  if (!h) return SP_OK;
  DeviceGuard dg(h->device);
  cudaFree(h->E); cudaFree(h->logits); cudaFree(h->tok); cudaFree(h->row);
  delete h;
  return SP_OK;
}

int sp_head_embed(sp_head* h, const int32_t* tokens_host, int32_t n, float* out_dev,
                  void* stream) {
  if (!h || n < 0 || n > 4096) return SP_ERR_ARG;
  for (int i = 0; i < n; ++i)
    if (tokens_host[i] < 0 || tokens_host[i] >= h->vocab) return SP_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  DeviceGuard dg(h->device);
  SP_CUDA_TRY(cudaMemcpyAsync(h->tok, tokens_host, n * sizeof(int), cudaMemcpyHostToDevice, st));
  const int64_t tot = (int64_t)n * h->d;
  if (tot) {
    sp::gather_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(h->E, h->tok, n, h->d,
                                                                      out_dev);
    sp::count_launch();
  }
  SP_CUDA_TRY(cudaStreamSynchronize(st));
  return SP_OK;
}

int sp_head_greedy(sp_head* h, const float* row_dev, int32_t* token_host, void* stream) {
  if (!h || !row_dev || !token_host) return SP_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  DeviceGuard dg(h->device);
  sp::logits_kernel<<<(h->vocab + 7) / 8, 256, 0, st>>>(h->E, row_dev, h->vocab, h->d, h->logits);
  sp::argmax_kernel<<<1, 1024, 0, st>>>(h->logits, h->vocab, h->tok);
  sp::count_launch();
  sp::count_launch();
  SP_CUDA_TRY(cudaMemcpyAsync(token_host, h->tok, sizeof(int), cudaMemcpyDeviceToHost, st));
  SP_CUDA_TRY(cudaStreamSynchronize(st));
  return SP_OK;
}

// logits [n_rows, vocab] of device rows [n_rows, d] (row @ E^T, SP/model.py:393-395);
// the same per-row reduction order as sp_head_greedy's logits
int sp_head_logits(sp_head* h, const float* rows_dev, int32_t n_rows, float* logits_dev,
                   void* stream) {
  if (!h || !rows_dev || !logits_dev || n_rows < 0) return SP_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  DeviceGuard dg(h->device);
  const unsigned grid = (h->vocab + 7) / 8;
  for (int r0 = 0; r0 < n_rows; r0 += 4) {
    const int n = n_rows - r0 < 4 ? n_rows - r0 : 4;
    const float* x = rows_dev + (int64_t)r0 * h->d;
    float* out = logits_dev + (int64_t)r0 * h->vocab;
    switch (n) {
      case 1: sp::logits_rows_kernel<1><<<grid, 256, 0, st>>>(h->E, x, h->vocab, h->d, out); break;
      case 2: sp::logits_rows_kernel<2><<<grid, 256, 0, st>>>(h->E, x, h->vocab, h->d, out); break;
      case 3: sp::logits_rows_kernel<3><<<grid, 256, 0, st>>>(h->E, x, h->vocab, h->d, out); break;
      default: sp::logits_rows_kernel<4><<<grid, 256, 0, st>>>(h->E, x, h->vocab, h->d, out); break;
    }
    sp::count_launch();
  }
  SP_CUDA_TRY(cudaGetLastError());
  return SP_OK;
}

int sp_head_read_embedding(sp_head* h, float* dst_host) {
  if (!h) return SP_ERR_ARG;
  DeviceGuard dg(h->device);
  SP_CUDA_TRY(cudaMemcpy(dst_host, h->E, (size_t)h->vocab * h->d * sizeof(float),
                         cudaMemcpyDeviceToHost));
  return SP_OK;
}

}  // extern "C"
