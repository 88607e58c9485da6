// Norms, RoPE + paged KV append, and attention over the paged KV cache.
//
// KV pool layout (per block of the span): [page][K|V][kv_head][64 pos][hd],
// kv dtype f32 or bf16.  A session's page table is int32 [width][max_pages];
// page p of slot s holds positions [64p, 64p+64).  Beam reorder permutes page
// tables (copy-on-write of a shared tail page), SP/model.py:169-175.
//
// Attention follows SP/model.py:263-275: scores = q.k / f32(sqrt(hd)),
// (+ ALiBi slope_h * (j - i) for BLOOM), causal -1e30 mask only when
// n_new > 1, max-subtracted softmax.  Decode splits the key range by page and
// merges the partial (max, sum, out) in a fixed order — deterministic.
#include "common.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr float kLnEps = 1e-5f;  // SP/model.py:23

// deterministic block reduction (fixed tree) — blockDim.x == 256
__device__ float block_sum_256(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = (l < 8) ? sh[l] : 0.f;
    t = warp_sum(t);
    if (l == 0) sh[8] = t;
  }
  __syncthreads();
  t = sh[8];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(256) norm_kernel(int family, const float* __restrict__ x,
                                                   const float* __restrict__ g,
                                                   const float* __restrict__ b,
                                                   float* __restrict__ out, int64_t d) {
  __shared__ float sh[9];
  const float* xr = x + (int64_t)blockIdx.x * d;
  float* orow = out + (int64_t)blockIdx.x * d;
  const float inv_d = 1.0f / (float)d;
  if (family == kLlama) {
    float s = 0.f;
    for (int64_t i = threadIdx.x; i < d; i += 256) s = fmaf(xr[i], xr[i], s);
    float ms = block_sum_256(s, sh) * inv_d;
    float den = sqrtf(ms + kLnEps);
    for (int64_t i = threadIdx.x; i < d; i += 256) orow[i] = xr[i] / den * g[i];
  } else {
    float s = 0.f;
    for (int64_t i = threadIdx.x; i < d; i += 256) s += xr[i];
    float mu = block_sum_256(s, sh) * inv_d;
    float q = 0.f;
    for (int64_t i = threadIdx.x; i < d; i += 256) {
      float c = xr[i] - mu;
      q = fmaf(c, c, q);
    }
    float var = block_sum_256(q, sh) * inv_d;
    float den = sqrtf(var + kLnEps);
    for (int64_t i = threadIdx.x; i < d; i += 256) orow[i] = (xr[i] - mu) / den * g[i] + b[i];
  }
}

template <typename KT>
__device__ __forceinline__ KT* kv_ptr(void* pool, int page, int kvsel, int kvh, int h, int off,
                                      int hd) {
  return reinterpret_cast<KT*>(pool) +
         ((((int64_t)page * 2 + kvsel) * kvh + h) * kPageTokens + off) * hd;
}

// one CTA per new row: RoPE q,k in place (llama) and write k,v into the pages
template <typename KT>
__global__ void rope_append_kernel(AttnArgs a) {
  const int row = blockIdx.x;
  const int slot = row / a.n_new, i = row % a.n_new;
  const int pos = a.t0 + i;
  const int hd = a.hd, half = hd / 2;
  float* q = a.qkv + (int64_t)row * a.ldqkv;
  float* k = q + a.H * hd;
  float* v = k + a.kvh * hd;
  const int page = a.page_table[slot * a.max_pages + pos / kPageTokens];
  const int off = pos % kPageTokens;
  if (a.family == kLlama) {
    const float* cs = a.rope_cos + (int64_t)pos * half;
    const float* sn = a.rope_sin + (int64_t)pos * half;
    for (int p = threadIdx.x; p < a.H * half; p += blockDim.x) {
      int h = p / half, j = p % half;
      float x1 = q[h * hd + j], x2 = q[h * hd + j + half];
      float c = cs[j], s = sn[j];
      q[h * hd + j] = __fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, s));
      q[h * hd + j + half] = __fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, s));
    }
    for (int p = threadIdx.x; p < a.kvh * half; p += blockDim.x) {
      int h = p / half, j = p % half;
      float x1 = k[h * hd + j], x2 = k[h * hd + j + half];
      float c = cs[j], s = sn[j];
      float r1 = __fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, s));
      float r2 = __fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, s));
      KT* dst = kv_ptr<KT>(a.kv_pool, page, 0, a.kvh, h, off, hd);
      dst[j] = from_f32<KT>(r1);
      dst[j + half] = from_f32<KT>(r2);
    }
  } else {
    for (int p = threadIdx.x; p < a.kvh * hd; p += blockDim.x) {
      int h = p / hd, j = p % hd;
      kv_ptr<KT>(a.kv_pool, page, 0, a.kvh, h, off, hd)[j] = from_f32<KT>(k[p]);
    }
  }
  for (int p = threadIdx.x; p < a.kvh * hd; p += blockDim.x) {
    int h = p / hd, j = p % hd;
    kv_ptr<KT>(a.kv_pool, page, 1, a.kvh, h, off, hd)[j] = from_f32<KT>(v[p]);
  }
}

// ---------------------------------------------------------------------------
// decode: grid (width*kvh, n_pages_used); one CTA = one (slot, kv head, page)
// ---------------------------------------------------------------------------
template <int HD, typename KT>
__global__ void __launch_bounds__(128) attn_decode_kernel(AttnArgs a, int nsplit) {
  extern __shared__ float smem[];
  const int G = a.H / a.kvh;
  float* qs = smem;                         // [G][HD]
  float* Ks = qs + G * HD;                  // [64][HD+1]
  float* Vs = Ks + kPageTokens * (HD + 1);  // [64][HD]
  float* ps = Vs + kPageTokens * HD;        // [G][64]
  float* stat = ps + G * kPageTokens;       // [G][2]

  const int slot = blockIdx.x / a.kvh, kh = blockIdx.x % a.kvh;
  const int sp = blockIdx.y;
  const int T = a.t0 + 1;
  const int j0 = sp * kPageTokens;
  const int nv = min(kPageTokens, T - j0);
  const int row = slot;  // n_new == 1
  const float* q = a.qkv + (int64_t)row * a.ldqkv + kh * G * HD;
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) qs[i] = q[i];
  const int page = a.page_table[slot * a.max_pages + sp];
  const KT* kp = kv_ptr<KT>(a.kv_pool, page, 0, a.kvh, kh, 0, HD);
  const KT* vp = kv_ptr<KT>(a.kv_pool, page, 1, a.kvh, kh, 0, HD);
  for (int i = threadIdx.x; i < nv * HD; i += blockDim.x) {
    int j = i / HD, dd = i % HD;
    Ks[j * (HD + 1) + dd] = to_f32(kp[i]);
    Vs[i] = to_f32(vp[i]);
  }
  __syncthreads();
  const float inv_sqrt = 1.0f / sqrtf((float)HD);
  const float rs = sqrtf((float)HD);
  (void)inv_sqrt;
  for (int pidx = threadIdx.x; pidx < G * nv; pidx += blockDim.x) {
    int g = pidx / nv, j = pidx % nv;
    float s = 0.f;
#pragma unroll 8
    for (int dd = 0; dd < HD; ++dd) s = fmaf(qs[g * HD + dd], Ks[j * (HD + 1) + dd], s);
    s = s / rs;
    if (a.family == kBloom) s += a.alibi[kh * G + g] * (float)(j0 + j - (T - 1));
    ps[g * kPageTokens + j] = s;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int g = warp; g < G; g += 4) {
    float m = -INFINITY;
    for (int j = lane; j < nv; j += 32) m = fmaxf(m, ps[g * kPageTokens + j]);
    m = warp_max(m);
    float l = 0.f;
    for (int j = lane; j < nv; j += 32) {
      float e = expf(ps[g * kPageTokens + j] - m);
      ps[g * kPageTokens + j] = e;
      l += e;
    }
    l = warp_sum(l);
    if (lane == 0) {
      stat[g * 2] = m;
      stat[g * 2 + 1] = l;
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < G * HD; o += blockDim.x) {
    int g = o / HD, dd = o % HD;
    float acc = 0.f;
    for (int j = 0; j < nv; ++j) acc = fmaf(ps[g * kPageTokens + j], Vs[j * HD + dd], acc);
    if (nsplit == 1) {
      a.ctx[(int64_t)row * a.H * HD + (kh * G + g) * HD + dd] = acc / stat[g * 2 + 1];
    } else {
      float* w = a.workspace + (((int64_t)(slot * a.kvh + kh) * nsplit + sp) * G + g) * (HD + 2);
      w[dd] = acc;
      if (dd == 0) {
        w[HD] = stat[g * 2];
        w[HD + 1] = stat[g * 2 + 1];
      }
    }
  }
}

// merge page partials in ascending page order: grid width*H, block HD
template <int HD>
__global__ void attn_combine_kernel(AttnArgs a, int nsplit) {
  const int G = a.H / a.kvh;
  const int slot = blockIdx.x / a.H, h = blockIdx.x % a.H;
  const int kh = h / G, g = h % G;
  const float* base = a.workspace + ((int64_t)(slot * a.kvh + kh) * nsplit) * G * (HD + 2);
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, base[((int64_t)s * G + g) * (HD + 2) + HD]);
  float L = 0.f, O = 0.f;
  const int dd = threadIdx.x;
  for (int s = 0; s < nsplit; ++s) {
    const float* w = base + ((int64_t)s * G + g) * (HD + 2);
    float f = expf(w[HD] - M);
    L = fmaf(w[HD + 1], f, L);
    O = fmaf(w[dd], f, O);
  }
  a.ctx[(int64_t)slot * a.H * HD + h * HD + dd] = O / L;
}

// ---------------------------------------------------------------------------
// prefill: grid (width*H, ceil(n_new/16)); 128 threads = 16 rows x 8 lanes
// ---------------------------------------------------------------------------
template <int HD, typename KT>
__global__ void __launch_bounds__(128) attn_prefill_kernel(AttnArgs a) {
  extern __shared__ float smem[];
  constexpr int QT = 16;
  constexpr int DPT = (HD + 7) / 8;  // dims per thread
  float* qs = smem;                          // [16][HD]
  float* Ks = qs + QT * HD;                  // [64][HD+1]
  float* Vs = Ks + kPageTokens * (HD + 1);   // [64][HD]
  float* Ps = Vs + kPageTokens * HD;         // [16][64]

  const int G = a.H / a.kvh;
  const int slot = blockIdx.x / a.H, h = blockIdx.x % a.H, kh = h / G;
  const int i0 = blockIdx.y * QT;
  const int r = threadIdx.x >> 3, c = threadIdx.x & 7;
  const int i = i0 + r;
  const bool valid = i < a.n_new;
  const int pos = a.t0 + (valid ? i : (a.n_new - 1));
  for (int idx = threadIdx.x; idx < QT * HD; idx += 128) {
    int rr = idx / HD, dd = idx % HD;
    int ii = min(i0 + rr, a.n_new - 1);
    qs[idx] = a.qkv[(int64_t)(slot * a.n_new + ii) * a.ldqkv + h * HD + dd];
  }
  const int last_pos = a.t0 + min(i0 + QT, a.n_new) - 1;
  const int npages = last_pos / kPageTokens + 1;
  const float rs = sqrtf((float)HD);
  const float slope = (a.family == kBloom) ? a.alibi[h] : 0.f;
  float m = -INFINITY, l = 0.f;
  float o[DPT];
#pragma unroll
  for (int q = 0; q < DPT; ++q) o[q] = 0.f;

  for (int pg = 0; pg < npages; ++pg) {
    __syncthreads();
    const int page = a.page_table[slot * a.max_pages + pg];
    const KT* kp = kv_ptr<KT>(a.kv_pool, page, 0, a.kvh, kh, 0, HD);
    const KT* vp = kv_ptr<KT>(a.kv_pool, page, 1, a.kvh, kh, 0, HD);
    const int nv = min(kPageTokens, last_pos + 1 - pg * kPageTokens);
    for (int idx = threadIdx.x; idx < kPageTokens * HD; idx += 128) {
      int j = idx / HD, dd = idx % HD;
      float kv = 0.f, vv = 0.f;
      if (j < nv) {
        kv = to_f32(kp[idx]);
        vv = to_f32(vp[idx]);
      }
      Ks[j * (HD + 1) + dd] = kv;
      Vs[idx] = vv;
    }
    __syncthreads();
    float sc[8];
    float pm = -INFINITY;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      int j = c + 8 * jj;
      int jabs = pg * kPageTokens + j;
      float s = 0.f;
#pragma unroll 8
      for (int dd = 0; dd < HD; ++dd) s = fmaf(qs[r * HD + dd], Ks[j * (HD + 1) + dd], s);
      s = s / rs;
      if (a.family == kBloom) s += slope * (float)(jabs - pos);
      if (jabs > pos || j >= nv) s = -1e30f;
      sc[jj] = s;
      pm = fmaxf(pm, s);
    }
    pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 1));
    pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 2));
    pm = fmaxf(pm, __shfl_xor_sync(0xffffffffu, pm, 4));
    const float mn = fmaxf(m, pm);
    const float alpha = expf(m - mn);
    float ls = 0.f;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      float e = expf(sc[jj] - mn);
      Ps[r * kPageTokens + c + 8 * jj] = e;
      ls += e;
    }
    ls += __shfl_xor_sync(0xffffffffu, ls, 1);
    ls += __shfl_xor_sync(0xffffffffu, ls, 2);
    ls += __shfl_xor_sync(0xffffffffu, ls, 4);
    l = l * alpha + ls;
    m = mn;
    __syncwarp();
    __syncthreads();
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
      int dd = c + 8 * q;
      if (dd < HD) {
        float acc = o[q] * alpha;
        for (int j = 0; j < kPageTokens; ++j) acc = fmaf(Ps[r * kPageTokens + j], Vs[j * HD + dd], acc);
        o[q] = acc;
      }
    }
  }
  if (valid) {
#pragma unroll
    for (int q = 0; q < DPT; ++q) {
      int dd = c + 8 * q;
      if (dd < HD) a.ctx[(int64_t)(slot * a.n_new + i) * a.H * HD + h * HD + dd] = o[q] / l;
    }
  }
}

__global__ void page_copy_kernel(char* pool, int64_t block_stride, int64_t page_bytes, int src,
                                 int dst) {
  const int b = blockIdx.y;
  char* base = pool + b * block_stride;
  const int4* s = reinterpret_cast<const int4*>(base + src * page_bytes);
  int4* d = reinterpret_cast<int4*>(base + dst * page_bytes);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < page_bytes / 16;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

template <typename KT>
__global__ void kv_gather_kernel(const void* pool, const int* table, int t, int kvh, int hd,
                                 float* k_out, float* v_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t n = (int64_t)t * kvh * hd;
  if (i >= n) return;
  int pos = (int)(i / (kvh * hd));
  int h = (int)((i / hd) % kvh), dd = (int)(i % hd);
  int page = table[pos / kPageTokens];
  const KT* base = reinterpret_cast<const KT*>(pool);
  k_out[i] = to_f32(base[((((int64_t)page * 2 + 0) * kvh + h) * kPageTokens + pos % kPageTokens) * hd + dd]);
  v_out[i] = to_f32(base[((((int64_t)page * 2 + 1) * kvh + h) * kPageTokens + pos % kPageTokens) * hd + dd]);
}

template <int HD, typename KT>
void decode_t(const AttnArgs& a, cudaStream_t st) {
  const int T = a.t0 + 1;
  const int nsplit = (T + kPageTokens - 1) / kPageTokens;
  const int G = a.H / a.kvh;
  size_t sm = (size_t)(G * HD + kPageTokens * (HD + 1) + kPageTokens * HD + G * kPageTokens +
                       2 * G) * sizeof(float);
  auto kern = attn_decode_kernel<HD, KT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 grid(a.width * a.kvh, nsplit);
  kern<<<grid, 128, sm, st>>>(a, nsplit); count_launch();
  if (nsplit > 1) {
    attn_combine_kernel<HD><<<a.width * a.H, HD, 0, st>>>(a, nsplit);
    count_launch();
  }
}

template <int HD, typename KT>
void prefill_t(const AttnArgs& a, cudaStream_t st) {
  size_t sm = (size_t)(16 * HD + kPageTokens * (HD + 1) + kPageTokens * HD + 16 * kPageTokens) *
              sizeof(float);
  auto kern = attn_prefill_kernel<HD, KT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 grid(a.width * a.H, (a.n_new + 15) / 16);
  kern<<<grid, 128, sm, st>>>(a); count_launch();
}

template <typename KT>
void dispatch_hd(const AttnArgs& a, bool decode, cudaStream_t st) {
  switch (a.hd) {
#define SP_HD_CASE(V)                 \
  case V:                             \
    if (decode) decode_t<V, KT>(a, st); \
    else prefill_t<V, KT>(a, st);     \
    break;
    SP_HD_CASE(4)
    SP_HD_CASE(16)
    SP_HD_CASE(32)
    SP_HD_CASE(64)
    SP_HD_CASE(128)
#undef SP_HD_CASE
    default:
      break;
  }
}

}  // namespace

void launch_norm(int family, const float* x, const float* g, const float* b, float* out,
                 int64_t R, int64_t d, cudaStream_t st) {
  if (R == 0) return;
  norm_kernel<<<(unsigned)R, 256, 0, st>>>(family, x, g, b, out, d); count_launch();
}

void launch_rope_append(const AttnArgs& a, cudaStream_t st) {
  int R = a.width * a.n_new;
  if (R == 0) return;
  if (a.kv_dtype == kKVBF16) rope_append_kernel<__nv_bfloat16><<<R, 256, 0, st>>>(a);
  else rope_append_kernel<float><<<R, 256, 0, st>>>(a);
  count_launch();
}

int64_t attn_workspace_floats(int width, int H, int hd, int max_seq) {
  int64_t nsplit = (max_seq + kPageTokens - 1) / kPageTokens;
  return (int64_t)width * H * nsplit * (hd + 2);
}

void launch_attention_decode(const AttnArgs& a, cudaStream_t st) {
  if (a.kv_dtype == kKVBF16) dispatch_hd<__nv_bfloat16>(a, true, st);
  else dispatch_hd<float>(a, true, st);
}

void launch_attention_prefill(const AttnArgs& a, cudaStream_t st) {
  if (a.kv_dtype == kKVBF16) dispatch_hd<__nv_bfloat16>(a, false, st);
  else dispatch_hd<float>(a, false, st);
}

void launch_page_copy(void* pool, int64_t block_stride_bytes, int n_blocks, int64_t page_bytes,
                      int src_page, int dst_page, cudaStream_t st) {
  dim3 grid(64, n_blocks);
  page_copy_kernel<<<grid, 256, 0, st>>>((char*)pool, block_stride_bytes, page_bytes, src_page,
                                         dst_page); count_launch();
}

void launch_kv_gather_slot(const void* pool, int kv_dtype, const int* table, int t, int kvh,
                           int hd, float* k_out, float* v_out, cudaStream_t st) {
  int64_t n = (int64_t)t * kvh * hd;
  if (n == 0) return;
  if (kv_dtype == kKVBF16)
    kv_gather_kernel<__nv_bfloat16><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pool, table, t, kvh, hd, k_out, v_out);
  else
    kv_gather_kernel<float><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pool, table, t, kvh, hd, k_out, v_out);
  count_launch();
}

}  // namespace sp
