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

// ---- beam selection (SP/model.py:470-491) -----------------------------------
// row log-sum-exp in float64 like the reference: z = logit - max, lse = log(sum exp z)
__global__ void beam_lse_kernel(const float* logits, int vocab, double* mx, double* lse) {
  __shared__ double red[1024];
  const float* l = logits + (int64_t)blockIdx.x * vocab;
  double m = -INFINITY;
  for (int v = threadIdx.x; v < vocab; v += blockDim.x) m = fmax(m, (double)l[v]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  m = red[0];
  __syncthreads();
  double acc = 0.0;
  for (int v = threadIdx.x; v < vocab; v += blockDim.x) acc += exp((double)l[v] - m);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {           // fixed-order tree
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) { mx[blockIdx.x] = m; lse[blockIdx.x] = log(red[0]); }
}

constexpr int KMAX = 16;
struct Cand { double s; int i; };
// ranking of SP/model.py:485-488: score descending, then (parent, token)
// ascending = flat index ascending
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  return a.s > b.s || (a.s == b.s && a.i < b.i);
}

// one CTA: every thread keeps its own top-k, warps then the block merge them by
// k rounds of a shuffle arg-best
__global__ void __launch_bounds__(1024) beam_topk_kernel(const float* logits, const double* scores,
                                                         const double* mx, const double* lse,
                                                         int w, int vocab, int k, int* parents,
                                                         int* tokens, double* out_scores) {
  __shared__ Cand wl[32][KMAX];
  Cand top[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) top[j] = Cand{-INFINITY, 0x7fffffff};
  const int n = w * vocab;
  for (int f = threadIdx.x; f < n; f += blockDim.x) {
    const int r = f / vocab;
    const double z = (double)logits[f] - mx[r];
    const Cand c{scores[r] + (z - lse[r]), f};
    if (!better(c, top[k - 1])) continue;
    int j = k - 1;                                    // insertion into the sorted list
    while (j > 0 && better(c, top[j - 1])) { top[j] = top[j - 1]; --j; }
    top[j] = c;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto warp_merge = [&](Cand* list, Cand* out) {     // list: this lane's sorted k; out: warp's k
    int head = 0;
    for (int j = 0; j < k; ++j) {
      Cand c = head < k ? list[head] : Cand{-INFINITY, 0x7fffffff};
      Cand b = c;
      int who = lane;
      for (int off = 16; off > 0; off >>= 1) {
        const double os = __shfl_xor_sync(0xffffffffu, b.s, off);
        const int oi = __shfl_xor_sync(0xffffffffu, b.i, off);
        const int ow = __shfl_xor_sync(0xffffffffu, who, off);
        if (better(Cand{os, oi}, b)) { b = Cand{os, oi}; who = ow; }
      }
      if (lane == who) ++head;
      if (lane == 0) out[j] = b;
    }
  };
  warp_merge(top, wl[warp]);
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    Cand mine[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      mine[j] = (lane < nw && j < k) ? wl[lane][j] : Cand{-INFINITY, 0x7fffffff};
    __shared__ Cand fin[KMAX];
    warp_merge(mine, fin);
    __syncwarp();
    if (lane < k) {
      parents[lane] = fin[lane].i / vocab;
      tokens[lane] = fin[lane].i % vocab;
      out_scores[lane] = fin[lane].s;
    }
  }
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

// SP/model.py:470-491 on the GPU: log-softmax of each row (float64), candidates
// scores[r] + logp, the k best by (score desc, parent asc, token asc)
int sp_beam_select(const float* logits_dev, const double* scores_host, int32_t w, int32_t vocab,
                   int32_t k, int32_t* parents_host, int32_t* tokens_host, double* new_scores_host,
                   void* stream) {
  if (!logits_dev || !scores_host || w < 1 || vocab < 1 || k < 1 || k > sp::KMAX ||
      (int64_t)w * vocab < k || (int64_t)w * vocab > (1ll << 31) - 1)
    return SP_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  double* buf = nullptr;           // scores, mx, lse, out_scores
  int* ibuf = nullptr;             // parents, tokens
  SP_CUDA_TRY(cudaMallocAsync(&buf, (3 * (size_t)w + sp::KMAX) * sizeof(double), st));
  SP_CUDA_TRY(cudaMallocAsync(&ibuf, 2 * sp::KMAX * sizeof(int), st));
  SP_CUDA_TRY(cudaMemcpyAsync(buf, scores_host, w * sizeof(double), cudaMemcpyHostToDevice, st));
  sp::beam_lse_kernel<<<w, 1024, 0, st>>>(logits_dev, vocab, buf + w, buf + 2 * w);
  sp::beam_topk_kernel<<<1, 1024, 0, st>>>(logits_dev, buf, buf + w, buf + 2 * w, w, vocab, k,
                                           ibuf, ibuf + sp::KMAX, buf + 3 * w);
  sp::count_launch();
  sp::count_launch();
  SP_CUDA_TRY(cudaGetLastError());
  SP_CUDA_TRY(cudaMemcpyAsync(parents_host, ibuf, k * sizeof(int), cudaMemcpyDeviceToHost, st));
  SP_CUDA_TRY(cudaMemcpyAsync(tokens_host, ibuf + sp::KMAX, k * sizeof(int),
                              cudaMemcpyDeviceToHost, st));
  SP_CUDA_TRY(cudaMemcpyAsync(new_scores_host, buf + 3 * w, k * sizeof(double),
                              cudaMemcpyDeviceToHost, st));
  SP_CUDA_TRY(cudaFreeAsync(buf, st));
  SP_CUDA_TRY(cudaFreeAsync(ibuf, st));
  SP_CUDA_TRY(cudaStreamSynchronize(st));
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
