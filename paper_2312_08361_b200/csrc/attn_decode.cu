// Fused decode attention (n_new == 1) over the paged KV cache.
//
// Grid: (slot x kv head, chunk of 128 positions).  4 warps per CTA, one warp
// per 32 positions; all K/V loads are issued up front.  In one launch:
//   * RoPE (llama) of the G query heads of the kv group (kept transposed in
//     smem, [dim][head], so one LDS.128 feeds 4 heads),
//   * the CTA whose chunk holds the new position t0 RoPEs k_new, rounds k/v to
//     the cache dtype and appends them to the page (KVCache.append,
//     SP/model.py:163-167) before anyone reads the page,
//   * scores = q.k / f32(sqrt(hd)) (+ ALiBi), lane = position, G independent
//     accumulators; softmax partials per warp; P.V with lane = dims,
//     (SP/model.py:263-275 — no mask at n = 1),
//   * the 4 warp partials merge in a fixed order into one chunk partial; the
//     last-arriving CTA of the (slot, kv head) merges the chunk partials in
//     ascending order (deterministic) and writes ctx plus the per-head
//     partial statistics the O-projection GEMV folds in.
// Bytes per launch: K+V of the visible positions (2*T*kvh*hd*elt) + q/ctx.
#include <type_traits>

#include "common.cuh"
#include "decode.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int NTH = 128;
constexpr int CHUNK = 128;          // positions per CTA (two pages)
constexpr int GMAX = 16;            // max query heads per kv head

template <typename KT>
__device__ __forceinline__ KT* page_ptr(void* pool, int page, int kvsel, int kvh, int h, int hd) {
  return reinterpret_cast<KT*>(pool) + (((int64_t)page * 2 + kvsel) * kvh + h) * kPageTokens * hd;
}

__device__ __forceinline__ float rope_val(const float* x, int dd, int half, const float* cs,
                                          const float* sn) {
  const int j = dd % half;
  const float c = cs[j], s = sn[j];
  return dd < half ? __fsub_rn(__fmul_rn(x[j], c), __fmul_rn(x[j + half], s))
                   : __fadd_rn(__fmul_rn(x[j + half], c), __fmul_rn(x[j], s));
}

template <int HD, typename KT>
__global__ void __launch_bounds__(NTH) attn_dec2_kernel(AttnDecArgs a) {
  constexpr int DPL = HD >= 32 ? HD / 32 : 1;     // dims per lane in P.V
  constexpr int ACT = HD >= 32 ? 32 : HD;         // lanes active in P.V
  __shared__ __align__(16) float qT[HD][GMAX];    // [dim][head]
  __shared__ __align__(16) float ps[4][32][GMAX]; // [warp][position][head]
  __shared__ float wm[4][GMAX], wl[4][GMAX];
  __shared__ int last_flag;
  extern __shared__ __align__(16) float dsm[];
  const int G = a.H / a.kvh;
  float* wo = dsm;                                // [4][G][HD]
  float* pm = dsm + 4 * G * HD;                   // [max_pages][GMAX] chunk maxima
  float* pl = pm + a.max_pages * GMAX;            // [max_pages][GMAX] chunk sums

  const int slot = blockIdx.x / a.kvh, kh = blockIdx.x % a.kvh;
  const int chunk = blockIdx.y;
  const int T = a.t0 + 1;
  const int nchunk = (T + CHUNK - 1) / CHUNK;
  if (chunk >= nchunk) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = HD / 2;
  const float* qrow = a.qkv + (int64_t)slot * a.ldqkv;
  const float* cs = a.rope_cos ? a.rope_cos + (int64_t)a.t0 * half : nullptr;
  const float* sn = a.rope_sin ? a.rope_sin + (int64_t)a.t0 * half : nullptr;

  // ---- q (RoPE at t0), transposed ----
  for (int i = threadIdx.x; i < G * HD; i += NTH) {
    const int g = i / HD, dd = i % HD;
    const float* q = qrow + (kh * G + g) * HD;
    qT[dd][g] = (a.family == kLlama) ? rope_val(q, dd, half, cs, sn) : q[dd];
  }
  for (int i = G + threadIdx.x; i < GMAX; i += NTH)   // zero unused head columns
    for (int dd = 0; dd < HD; ++dd) qT[dd][i] = 0.f;
  // ---- append the new position (the CTA whose chunk holds t0) ----
  if (a.t0 / CHUNK == chunk) {
    const int page = a.page_table[slot * a.max_pages + a.t0 / kPageTokens];
    KT* kp = page_ptr<KT>(a.kv_pool, page, 0, a.kvh, kh, HD) + (a.t0 % kPageTokens) * HD;
    KT* vp = page_ptr<KT>(a.kv_pool, page, 1, a.kvh, kh, HD) + (a.t0 % kPageTokens) * HD;
    const float* kn = qrow + a.H * HD + kh * HD;
    const float* vn = qrow + a.H * HD + a.kvh * HD + kh * HD;
    for (int dd = threadIdx.x; dd < HD; dd += NTH) {
      kp[dd] = from_f32<KT>((a.family == kLlama) ? rope_val(kn, dd, half, cs, sn) : kn[dd]);
      vp[dd] = from_f32<KT>(vn[dd]);
    }
  }
  __syncthreads();

  // ---- this warp's 32 positions ----
  const int p0 = chunk * CHUNK + warp * 32;
  const int nv = max(0, min(32, T - p0));
  const int page = a.page_table[slot * a.max_pages + min(p0, T - 1) / kPageTokens];
  const int off0 = p0 % kPageTokens;
  const KT* kbase = page_ptr<KT>(a.kv_pool, page, 0, a.kvh, kh, HD) + off0 * HD;
  const KT* vbase = page_ptr<KT>(a.kv_pool, page, 1, a.kvh, kh, HD) + off0 * HD;
  // V rows for P.V, loaded now (lane = dims), consumed after the softmax
  float vreg[32][DPL];
  if constexpr (DPL * sizeof(KT) == 8 || DPL * sizeof(KT) == 16) {
    using VV = typename std::conditional<DPL * sizeof(KT) == 8, uint2, uint4>::type;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      VV raw{};
      if (j < nv && lane < ACT) raw = __ldcg(reinterpret_cast<const VV*>(vbase + j * HD + lane * DPL));
      const KT* e8 = reinterpret_cast<const KT*>(&raw);
#pragma unroll
      for (int e = 0; e < DPL; ++e) vreg[j][e] = to_f32(e8[e]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
#pragma unroll
      for (int e = 0; e < DPL; ++e)
        vreg[j][e] = (j < nv && lane < ACT) ? to_f32(__ldcg(vbase + j * HD + lane * DPL + e)) : 0.f;
  }
  // ---- scores: lane = position (its K row read straight from the page, 16 B
  // at a time: whole sectors), G accumulators ----
  float s[GMAX];
#pragma unroll
  for (int g = 0; g < GMAX; ++g) s[g] = 0.f;
  if (lane < nv) {
    constexpr int VE = 16 / sizeof(KT) < HD ? 16 / sizeof(KT) : HD;   // elements per load
    constexpr int NCH = HD / VE;
    constexpr int BLK = NCH < 8 ? NCH : 8;                             // loads in flight
    const KT* krow = kbase + lane * HD;
#pragma unroll
    for (int c0 = 0; c0 < NCH; c0 += BLK) {
      KT kv[BLK][VE];
#pragma unroll
      for (int c = 0; c < BLK; ++c) {
        if constexpr (VE * sizeof(KT) == 16)
          *reinterpret_cast<uint4*>(kv[c]) = __ldcg(reinterpret_cast<const uint4*>(krow + (c0 + c) * VE));
        else
#pragma unroll
          for (int e = 0; e < VE; ++e) kv[c][e] = krow[(c0 + c) * VE + e];
      }
#pragma unroll
      for (int c = 0; c < BLK; ++c)
#pragma unroll
        for (int e = 0; e < VE; ++e) {
          const int dd = (c0 + c) * VE + e;
          const float k = to_f32(kv[c][e]);
          const float4* q4 = reinterpret_cast<const float4*>(qT[dd]);
#pragma unroll
          for (int g4 = 0; g4 < GMAX / 4; ++g4) {
            if (g4 * 4 >= G) break;
            const float4 qv = q4[g4];
            s[g4 * 4 + 0] = fmaf(qv.x, k, s[g4 * 4 + 0]);
            s[g4 * 4 + 1] = fmaf(qv.y, k, s[g4 * 4 + 1]);
            s[g4 * 4 + 2] = fmaf(qv.z, k, s[g4 * 4 + 2]);
            s[g4 * 4 + 3] = fmaf(qv.w, k, s[g4 * 4 + 3]);
          }
        }
    }
  }
  const float rs = sqrtf((float)HD);
  const int pos = p0 + lane;
#pragma unroll
  for (int g = 0; g < GMAX; ++g) {
    if (g >= G) break;
    float sc = -INFINITY;
    if (lane < nv) {
      sc = s[g] / rs;
      if (a.family == kBloom) sc += a.alibi[kh * G + g] * (float)(pos - (T - 1));
    }
    const float m = warp_max(sc);
    const float e = (lane < nv) ? expf(sc - m) : 0.f;
    const float l = warp_sum(e);
    ps[warp][lane][g] = e;
    if (lane == 0) { wm[warp][g] = m; wl[warp][g] = l; }
  }
  for (int g = G; g < GMAX; ++g) ps[warp][lane][g] = 0.f;
  __syncwarp();

  // ---- P.V: lane = dims, G x DPL accumulators ----
  if (lane < ACT && nv > 0) {
    float o[GMAX][DPL];
#pragma unroll
    for (int g = 0; g < GMAX; ++g)
#pragma unroll
      for (int e = 0; e < DPL; ++e) o[g][e] = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float4* p4 = reinterpret_cast<const float4*>(ps[warp][j]);
#pragma unroll
      for (int g4 = 0; g4 < GMAX / 4; ++g4) {
        if (g4 * 4 >= G) break;
        const float4 pv = p4[g4];
#pragma unroll
        for (int e = 0; e < DPL; ++e) {
          o[g4 * 4 + 0][e] = fmaf(pv.x, vreg[j][e], o[g4 * 4 + 0][e]);
          o[g4 * 4 + 1][e] = fmaf(pv.y, vreg[j][e], o[g4 * 4 + 1][e]);
          o[g4 * 4 + 2][e] = fmaf(pv.z, vreg[j][e], o[g4 * 4 + 2][e]);
          o[g4 * 4 + 3][e] = fmaf(pv.w, vreg[j][e], o[g4 * 4 + 3][e]);
        }
      }
    }
#pragma unroll
    for (int g = 0; g < GMAX; ++g) {
      if (g >= G) break;
#pragma unroll
      for (int e = 0; e < DPL; ++e) wo[(warp * G + g) * HD + lane * DPL + e] = o[g][e];
    }
  }
  __syncthreads();

  // ---- merge the 4 warps (fixed order) -> chunk partial ----
  const int64_t pstride = (int64_t)G * (HD + 2);
  float* part = a.part + ((int64_t)(slot * a.kvh + kh) * a.max_pages + chunk) * pstride;
  for (int i = threadIdx.x; i < G * HD; i += NTH) {
    const int g = i / HD, dd = i % HD;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w][g]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < 4; ++w) {
      if (chunk * CHUNK + w * 32 >= T) continue;      // warp had no positions
      const float f = expf(wm[w][g] - M);
      L = fmaf(wl[w][g], f, L);
      O = fmaf(wo[(w * G + g) * HD + dd], f, O);
    }
    part[g * (HD + 2) + dd] = O;
    if (dd == 0) {
      part[g * (HD + 2) + HD] = M;
      part[g * (HD + 2) + HD + 1] = L;
    }
  }

  // ---- last CTA of this (slot, kv head): merge chunks in ascending order ----
  if (nchunk > 1) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
      last_flag = (atomicAdd(a.counters + slot * a.kvh + kh, 1) == nchunk - 1);
    __syncthreads();
    if (!last_flag) return;
    __threadfence();
  } else {
    __syncthreads();
  }
  const float* pall = a.part + (int64_t)(slot * a.kvh + kh) * a.max_pages * pstride;
  for (int e = threadIdx.x; e < nchunk * G; e += NTH) {
    const int c = e / G, g = e % G;
    pm[c * GMAX + g] = __ldcg(pall + c * pstride + g * (HD + 2) + HD);
    pl[c * GMAX + g] = __ldcg(pall + c * pstride + g * (HD + 2) + HD + 1);
  }
  __syncthreads();
  float* outh = wo;
  for (int i = threadIdx.x; i < G * HD; i += NTH) {
    const int g = i / HD, dd = i % HD;
    float M = -INFINITY;
    for (int c = 0; c < nchunk; ++c) M = fmaxf(M, pm[c * GMAX + g]);
    float L = 0.f, O = 0.f;
    for (int c0 = 0; c0 < nchunk; c0 += 8) {
      float wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        wv[u] = (c0 + u < nchunk) ? __ldcg(pall + (c0 + u) * pstride + g * (HD + 2) + dd) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (c0 + u < nchunk) {
          const float f = expf(pm[(c0 + u) * GMAX + g] - M);
          L = fmaf(pl[(c0 + u) * GMAX + g], f, L);
          O = fmaf(wv[u], f, O);
        }
      }
    }
    const float c = O / L;
    outh[i] = c;
    a.ctx[(int64_t)slot * a.H * HD + (kh * G + g) * HD + dd] = c;
  }
  if (threadIdx.x == 0 && nchunk > 1) a.counters[slot * a.kvh + kh] = 0;
  __syncthreads();
  if (a.st_out && threadIdx.x < G) {
    const int g = threadIdx.x;
    float S = 0.f, Q = 0.f, Mx = 0.f;
    for (int dd = 0; dd < HD; ++dd) {
      const float c = outh[g * HD + dd];
      S += c;
      Q = fmaf(c, c, Q);
      Mx = fmaxf(Mx, fabsf(c));
    }
    a.st_out[(int64_t)(kh * G + g) * a.width + slot] = RowStat{S, Q, Mx, 0.f};
  }
}

template <int HD, typename KT>
void launch_t(const AttnDecArgs& a, cudaStream_t st) {
  const int T = a.t0 + 1;
  dim3 grid(a.width * a.kvh, (T + CHUNK - 1) / CHUNK);
  const int G = a.H / a.kvh;
  const size_t smem = (size_t)(4 * G * HD + 2 * a.max_pages * GMAX) * sizeof(float);
  static size_t set = 0;
  if (smem > set) {
    cudaFuncSetAttribute(attn_dec2_kernel<HD, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    set = smem;
  }
  attn_dec2_kernel<HD, KT><<<grid, NTH, smem, st>>>(a);
  count_launch();
}

template <typename KT>
void dispatch(const AttnDecArgs& a, cudaStream_t st) {
  switch (a.hd) {
    case 16: launch_t<16, KT>(a, st); break;
    case 32: launch_t<32, KT>(a, st); break;
    case 64: launch_t<64, KT>(a, st); break;
    case 128: launch_t<128, KT>(a, st); break;
    default: launch_t<4, KT>(a, st); break;
  }
}

}  // namespace

int64_t attn_dec_part_floats(int width, int H, int hd, int max_pages) {
  return (int64_t)width * H * max_pages * (hd + 2);
}

void launch_attn_decode_fused(const AttnDecArgs& a, cudaStream_t st) {
  if (a.kv_dtype == kKVBF16) dispatch<__nv_bfloat16>(a, st);
  else dispatch<float>(a, st);
}

}  // namespace sp
