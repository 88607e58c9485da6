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
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "decode.cuh"
#include "kernels.cuh"

namespace sp {

extern int g_attn_cluster;  // option 6: decode-attention cluster size (0 auto, -1 off, 8, 16)
extern int g_attn_nsub;   // sp_span_set_option(.., 5, n): forced sub-chunks per CTA (0 = auto)

namespace {

constexpr int NTH = 128;
constexpr int CHUNK = 128;          // positions per CTA (two pages)
constexpr int GMAX = 16;            // max query heads per kv head
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void trace_mark(const AttnDecArgs& a, int ph) {
  if (SP_DEV_TRACE && a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    a.trace[(blockIdx.y * gridDim.x + blockIdx.x) * 12 + ph] = t;
  }
}

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

// merge the 4 warp partials (fixed order) into this chunk's partial; the
// last-arriving CTA of (slot, kv head) merges all chunks in ascending order,
// writes ctx and the per-head partial stats of ctx
// LOG2: the partial maxima are in the log2 domain (scores pre-scaled by log2 e)
template <int HD, bool LOG2, int GT = 0>
__device__ void merge_tail(const AttnDecArgs& a, int G_rt, int slot, int kh, int chunk, int nchunk,
                           int T, const float (*wm)[GMAX], const float (*wl)[GMAX], float* wo,
                           float* pm, float* pl, int* last_flag, int CH = CHUNK,
                           float* stg = nullptr, int stg_cap = 0) {
  const int G = GT ? GT : G_rt;            // compile-time group size where known
  __shared__ float wf[4][GMAX];        // per (warp, head) rescale factors
  __shared__ float hM[GMAX], hL[GMAX];
  // ---- merge the 4 warps (fixed order) -> chunk partial ----
  if (threadIdx.x < G) {
    const int g = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w)
      if (chunk * CH + w * 32 < T) M = fmaxf(M, wm[w][g]);
    float L = 0.f;
    for (int w = 0; w < 4; ++w) {
      const float f = (chunk * CH + w * 32 < T) ? (LOG2 ? ex2_approx(wm[w][g] - M) : expf(wm[w][g] - M))
                                                   : 0.f;  // empty warp: 0
      wf[w][g] = f;
      L = fmaf(wl[w][g] * (f > 0.f ? 1.f : 0.f), f, L);
    }
    hM[g] = M;
    hL[g] = L;
  }
  __syncthreads();
  // partials: O [(slot, kv head, chunk)][G][HD] (16-byte aligned rows), then
  // the (max, sum) pairs [(slot, kv head, chunk)][G][2] after all O rows
  const int64_t sk = (int64_t)slot * a.kvh + kh;
  const int GH = G * HD;
  float* partO = a.part + (sk * a.max_pages + chunk) * GH;
  float* stats = a.part + (int64_t)a.width * a.H * a.max_pages * HD;
  for (int i = threadIdx.x * 4; i < GH; i += NTH * 4) {
    const int g = i / HD;
    float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float4 v = *reinterpret_cast<const float4*>(wo + w * GH + i);
      const float f = wf[w][g];
      O.x = fmaf(v.x, f, O.x); O.y = fmaf(v.y, f, O.y);
      O.z = fmaf(v.z, f, O.z); O.w = fmaf(v.w, f, O.w);
    }
    __stcg(reinterpret_cast<float4*>(partO + i), O);
  }
  if (threadIdx.x < G) {
    float* st = stats + ((sk * a.max_pages + chunk) * G + threadIdx.x) * 2;
    __stcg(st, hM[threadIdx.x]);
    __stcg(st + 1, hL[threadIdx.x]);
  }

  // ---- last CTA of this (slot, kv head): merge chunks in ascending order ----
  if (nchunk > 1) {
    __syncthreads();
    if (threadIdx.x == 0) {
      int old;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                   : "=r"(old) : "l"(a.counters + slot * a.kvh + kh) : "memory");
      *last_flag = (old == nchunk - 1);
    }
    __syncthreads();
    trace_mark(a, 4);
    if (!*last_flag) return;
  } else {
    __syncthreads();
  }
  const float* sall = stats + sk * a.max_pages * G * 2;
  const float* oall = a.part + sk * a.max_pages * GH;
  // when the chunk partials fit the (now idle) K/V staging buffer, one burst of
  // cp.async pulls all of them from L2 in one round trip, under the stats merge
  const bool staged = stg != nullptr && nchunk * GH <= stg_cap;
  if (staged) {
    for (int i = threadIdx.x * 4; i < nchunk * GH; i += NTH * 4)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(stg + i)), "l"(oall + i));
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // every load below is issued before its first use: the merge costs one L2
  // round trip for the (max, sum) pairs and one per 8 chunks of O
  {
    float2 mv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * NTH;
      mv[u] = e < nchunk * G ? __ldcg(reinterpret_cast<const float2*>(sall) + e)
                             : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * NTH;
      if (e < nchunk * G) { pm[(e / G) * GMAX + e % G] = mv[u].x; pl[(e / G) * GMAX + e % G] = mv[u].y; }
    }
    for (int e = threadIdx.x + 4 * NTH; e < nchunk * G; e += NTH) {
      pm[(e / G) * GMAX + e % G] = __ldcg(sall + 2 * e);
      pl[(e / G) * GMAX + e % G] = __ldcg(sall + 2 * e + 1);
    }
  }
  __syncthreads();
  // per head (one warp each): global max M, chunk factors f_c = exp(m_c - M)
  // (stored over pm) and L = sum_c l_c f_c, by a fixed shuffle tree
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int g = warp; g < G; g += NTH / 32) {
      float m = -INFINITY;
      for (int c = lane; c < nchunk; c += 32) m = fmaxf(m, pm[c * GMAX + g]);
      const float M = warp_max(m);
      float L = 0.f;
      for (int c = lane; c < nchunk; c += 32) {
        const float f = LOG2 ? ex2_approx(pm[c * GMAX + g] - M) : expf(pm[c * GMAX + g] - M);
        pm[c * GMAX + g] = f;
        L = fmaf(pl[c * GMAX + g], f, L);
      }
      L = warp_sum(L);
      if (lane == 0) hL[g] = L;
    }
  }
  if (staged) asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  trace_mark(a, 5);
  float* outh = wo;
  if (staged) {
    float* ctx = a.ctx + (int64_t)slot * a.H * HD + kh * GH;
    for (int i = threadIdx.x * 4; i < GH; i += NTH * 4) {
      float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int c = 0; c < nchunk; ++c) {               // ascending chunks, like the path below
        const float4 w = *reinterpret_cast<const float4*>(stg + c * GH + i);
        const float f = pm[c * GMAX + i / HD];
        O.x = fmaf(w.x, f, O.x); O.y = fmaf(w.y, f, O.y);
        O.z = fmaf(w.z, f, O.z); O.w = fmaf(w.w, f, O.w);
      }
      const float L = hL[i / HD];
      const float4 cv = make_float4(O.x / L, O.y / L, O.z / L, O.w / L);
      *reinterpret_cast<float4*>(outh + i) = cv;
      *reinterpret_cast<float4*>(ctx + i) = cv;
    }
  }
  for (int ib = staged ? GH : threadIdx.x * 4; ib < GH; ib += 2 * NTH * 4) {
    const int i1 = ib + NTH * 4;
    const bool has1 = i1 < GH;
    float4 O0 = make_float4(0.f, 0.f, 0.f, 0.f), O1 = O0;
    for (int c0 = 0; c0 < nchunk; c0 += 8) {
      float4 w0[8], w1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = c0 + u < nchunk;
        const float4* src = reinterpret_cast<const float4*>(oall + (int64_t)(c0 + u) * GH);
        w0[u] = ok ? __ldcg(src + ib / 4) : make_float4(0.f, 0.f, 0.f, 0.f);
        w1[u] = (ok && has1) ? __ldcg(src + i1 / 4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = c0 + u < nchunk;
        const float f0 = ok ? pm[(c0 + u) * GMAX + ib / HD] : 0.f;
        const float f1 = (ok && has1) ? pm[(c0 + u) * GMAX + i1 / HD] : 0.f;
        O0.x = fmaf(w0[u].x, f0, O0.x); O0.y = fmaf(w0[u].y, f0, O0.y);
        O0.z = fmaf(w0[u].z, f0, O0.z); O0.w = fmaf(w0[u].w, f0, O0.w);
        O1.x = fmaf(w1[u].x, f1, O1.x); O1.y = fmaf(w1[u].y, f1, O1.y);
        O1.z = fmaf(w1[u].z, f1, O1.z); O1.w = fmaf(w1[u].w, f1, O1.w);
      }
    }
    float* ctx = a.ctx + (int64_t)slot * a.H * HD + kh * GH;
    {
      const float L = hL[ib / HD];
      const float4 c = make_float4(O0.x / L, O0.y / L, O0.z / L, O0.w / L);
      *reinterpret_cast<float4*>(outh + ib) = c;
      *reinterpret_cast<float4*>(ctx + ib) = c;
    }
    if (has1) {
      const float L = hL[i1 / HD];
      const float4 c = make_float4(O1.x / L, O1.y / L, O1.z / L, O1.w / L);
      *reinterpret_cast<float4*>(outh + i1) = c;
      *reinterpret_cast<float4*>(ctx + i1) = c;
    }
  }
  trace_mark(a, 6);
  if (threadIdx.x == 0 && nchunk > 1) a.counters[slot * a.kvh + kh] = 0;
  __syncthreads();
  if (a.st_out) {
    // one warp per head, fixed shuffle tree (deterministic)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int g = warp; g < G; g += NTH / 32) {
      float S = 0.f, Q = 0.f, Mx = 0.f;
      for (int dd = lane; dd < HD; dd += 32) {
        const float c = outh[g * HD + dd];
        S += c;
        Q = fmaf(c, c, Q);
        Mx = fmaxf(Mx, fabsf(c));
      }
      S = warp_sum(S); Q = warp_sum(Q); Mx = warp_max(Mx);
      if (lane == 0) a.st_out[(int64_t)(kh * G + g) * a.width + slot] = RowStat{S, Q, Mx, 0.f};
    }
  }
}

template <int HD, typename KT, int GT>
__global__ void __launch_bounds__(NTH) attn_dec2_kernel(AttnDecArgs a) {
  constexpr int GC = GT ? GT : GMAX;              // compile-time bound on heads per kv head
  constexpr int DPL = HD >= 32 ? HD / 32 : 1;     // dims per lane in P.V
  constexpr int ACT = HD >= 32 ? 32 : HD;         // lanes active in P.V
  __shared__ __align__(16) float qT[HD][GMAX];    // [dim][head]
  __shared__ __align__(16) float ps[4][32][GMAX]; // [warp][position][head]
  __shared__ float wm[4][GMAX], wl[4][GMAX];
  __shared__ int last_flag;
  extern __shared__ __align__(16) float dsm[];
  const int G = GT ? GT : a.H / a.kvh;
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
  float s[((GC + 3) / 4) * 4];
#pragma unroll
  for (int g = 0; g < ((GC + 3) / 4) * 4; ++g) s[g] = 0.f;
  if (lane < nv) {
    constexpr int VE = 16 / sizeof(KT) < HD ? 16 / sizeof(KT) : HD;   // elements per load
    constexpr int NCH = HD / VE;
    constexpr int BLK = NCH < 2 ? NCH : 2;                             // loads in flight
    const KT* krow = kbase + lane * HD;
#pragma unroll 1
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
          for (int g4 = 0; g4 < (GC + 3) / 4; ++g4) {
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
  for (int g = 0; g < GC; ++g) {
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
    float o[((GC + 3) / 4) * 4][DPL];
#pragma unroll
    for (int g = 0; g < ((GC + 3) / 4) * 4; ++g)
#pragma unroll
      for (int e = 0; e < DPL; ++e) o[g][e] = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float4* p4 = reinterpret_cast<const float4*>(ps[warp][j]);
#pragma unroll
      for (int g4 = 0; g4 < (GC + 3) / 4; ++g4) {
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
    for (int g = 0; g < GC; ++g) {
      if (g >= G) break;
#pragma unroll
      for (int e = 0; e < DPL; ++e) wo[(warp * G + g) * HD + lane * DPL + e] = o[g][e];
    }
  }
  __syncthreads();

  merge_tail<HD, false>(a, G, slot, kh, chunk, nchunk, T, wm, wl, wo, pm, pl, &last_flag);
}


// ---------------------------------------------------------------------------
// tensor-core variant (bf16 KV, hd % 16 == 0, G <= 8): per warp 32 positions,
// S = K.q^T and O^T = V^T.P on mma.m16n8k16 (q and P split hi+lo in bf16, so
// the products keep ~16 mantissa bits; K/V are exact cache values), K/V tiles
// staged by cp.async and fed by ldmatrix (.trans for V^T).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_bf16_16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0));
}

// Cluster merge (70B shape: G = 8 query heads per kv head, a cluster of CY = 8
// or 16 CTAs per (slot, kv head) along the positions): each CTA folds its 4 warps'
// partials into one (O[G][HD], max, sum) in shared memory; after one cluster
// barrier CTA r merges head r from the 8 CTAs' partials over DSMEM, in fixed
// rank order, and writes ctx and the head's row statistics.  No global partial
// round trip, no arrival counter, no serial last-CTA merge.
template <int HD, int CY>
__device__ void cluster_merge(const AttnDecArgs& a, int G, int slot, int kh, bool has_rows,
                              const float (*wm)[GMAX], const float (*wl)[GMAX], const float* wo,
                              int T, int base) {
  namespace cg = cooperative_groups;
  __shared__ __align__(16) float cO[8][HD];
  __shared__ float cM[8], cL[8], wf[4][8];
  __shared__ float red[3][4];
  cg::cluster_group cluster = cg::this_cluster();
  // ---- this CTA's partial: the 4 warps merged (warps without rows: weight 0) ----
  if (threadIdx.x < G) {
    const int g = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w)
      if (has_rows && base + w * 32 < T) M = fmaxf(M, wm[w][g]);
    float L = 0.f;
    for (int w = 0; w < 4; ++w) {
      const float f = (has_rows && base + w * 32 < T && M != -INFINITY) ? ex2_approx(wm[w][g] - M) : 0.f;
      wf[w][g] = f;
      L = fmaf(f > 0.f ? wl[w][g] : 0.f, f, L);
    }
    cM[g] = M;
    cL[g] = L;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * HD; i += NTH) {
    const int g = i / HD, dd = i % HD;
    float O = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w)                  // (a warp without rows holds no finite O)
      if (wf[w][g] != 0.f) O = fmaf(wo[(w * G + g) * HD + dd], wf[w][g], O);
    cO[g][dd] = O;
  }
  cluster.sync();
  // ---- CTA r merges head r over the 8 CTAs (DSMEM, ascending rank) ----
  const int g = (int)cluster.block_rank();
  if (g < G) {
    float Mc[CY], Lc[CY];
    float M = -INFINITY;
#pragma unroll
    for (int c = 0; c < CY; ++c) {
      Mc[c] = *cluster.map_shared_rank(&cM[g], c);
      Lc[c] = *cluster.map_shared_rank(&cL[g], c);
      M = fmaxf(M, Mc[c]);
    }
    float L = 0.f, f[CY];
#pragma unroll
    for (int c = 0; c < CY; ++c) {
      f[c] = Mc[c] == -INFINITY ? 0.f : ex2_approx(Mc[c] - M);
      L = fmaf(Lc[c], f[c], L);
    }
    const float inv = __frcp_rn(L);
    float S = 0.f, Q = 0.f, Mx = 0.f;
    for (int dd = threadIdx.x; dd < HD; dd += NTH) {
      float O = 0.f;
#pragma unroll
      for (int c = 0; c < CY; ++c)
        if (f[c] != 0.f) O = fmaf(*cluster.map_shared_rank(&cO[g][dd], c), f[c], O);
      const float v = O * inv;
      a.ctx[(int64_t)slot * a.H * HD + (kh * G + g) * HD + dd] = v;
      S += v;
      Q = fmaf(v, v, Q);
      Mx = fmaxf(Mx, fabsf(v));
    }
    if (a.st_out) {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      S = warp_sum(S); Q = warp_sum(Q); Mx = warp_max(Mx);
      if (lane == 0) { red[0][warp] = S; red[1][warp] = Q; red[2][warp] = Mx; }
      __syncthreads();
      if (threadIdx.x == 0) {
        float s2 = 0.f, q2 = 0.f, m2 = 0.f;
        for (int w = 0; w < NTH / 32; ++w) { s2 += red[0][w]; q2 += red[1][w]; m2 = fmaxf(m2, red[2][w]); }
        a.st_out[(int64_t)(kh * G + g) * a.width + slot] = RowStat{s2, q2, m2, 0.f};
      }
    }
  }
  cluster.sync();          // peers' shared memory stays valid until everyone has read it
}

template <int HD, int GT, int CL = 0>
__global__ void __launch_bounds__(NTH) attn_dec_mma_kernel(AttnDecArgs a) {
  constexpr int RS = HD + 8;                      // padded smem row (bf16), breaks ldmatrix conflicts
  __shared__ __align__(16) __nv_bfloat16 qh[8][RS], ql[8][RS];      // [head][dim]
  __shared__ __align__(16) __nv_bfloat16 ph[4][8][40], pl_[4][8][40]; // [warp][head][pos]
  __shared__ float wm[4][GMAX], wl[4][GMAX];
  __shared__ int last_flag;
  extern __shared__ __align__(16) float dsm[];
  const int G = GT ? GT : a.H / a.kvh;   // query heads per kv head (compile-time when known)
  typedef __nv_bfloat16 Row[RS];
  // K/V of a 128-position sub-chunk, double-buffered: [2][4*32][RS] each.  A
  // CTA streams a.nsub sub-chunks (MHA shapes: many kv heads, few positions per
  // CTA otherwise) with a running online softmax per warp
  // (one buffer when a CTA has a single sub-chunk: 70 KB instead of 139 KB, so
  // the next GEMV's CTA fits beside it and prefetches its weights)
  const int nbuf = a.nsub > 1 ? 2 : 1;
  Row* Kbuf = reinterpret_cast<Row*>(dsm);
  Row* Vbuf = Kbuf + nbuf * 4 * 32;
  float* wo = reinterpret_cast<float*>(Vbuf + nbuf * 4 * 32);   // [4][G][HD]
  float* pmv = wo + 4 * G * HD;
  float* plv = pmv + a.max_pages * GMAX;

  const int slot = blockIdx.x / a.kvh, kh = blockIdx.x % a.kvh;
  const int chunk = blockIdx.y;
  const int T = a.t0 + 1;
  const int nsub = a.nsub > 0 ? a.nsub : 1;
  const int CH = CHUNK * nsub;                    // positions per CTA
  const int nchunk = (T + CH - 1) / CH;
  if (CL == 0 && chunk >= nchunk) return;            // (cluster mode: every CTA joins the barriers)
  const int base = chunk * CH;
  const int nsub_here = base < T ? min(nsub, (T - base + CHUNK - 1) / CHUNK) : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int half = HD / 2;
  const float* qrow = a.qkv + (int64_t)slot * a.ldqkv;
  const float* cs = a.rope_cos ? a.rope_cos + (int64_t)a.t0 * half : nullptr;
  const float* sn = a.rope_sin ? a.rope_sin + (int64_t)a.t0 * half : nullptr;

  // ---- 1. stage this warp's 32 K/V rows of sub-chunk j (cp.async, zero-fill
  // past T) into buffer j & 1; sub-chunk 0 is issued first of all: the loads do
  // not depend on q, so their latency overlaps everything below.  Row t0 is
  // read stale and patched in smem after the append ----
  constexpr int CPR = HD / 8;                     // 16-byte chunks per row
  auto stage = [&](int j) {
    const int q0 = base + j * CHUNK + warp * 32;
    const int nvj = max(0, min(32, T - q0));
    const int page = a.page_table[slot * a.max_pages + min(q0, T - 1) / kPageTokens];
    const __nv_bfloat16* kbase = page_ptr<__nv_bfloat16>(a.kv_pool, page, 0, a.kvh, kh, HD) + (q0 % kPageTokens) * HD;
    const __nv_bfloat16* vbase = page_ptr<__nv_bfloat16>(a.kv_pool, page, 1, a.kvh, kh, HD) + (q0 % kPageTokens) * HD;
    Row* Kt = Kbuf + (j % nbuf) * 128;
    Row* Vt = Vbuf + (j % nbuf) * 128;
    for (int c = lane; c < 32 * CPR; c += 32) {
      const int r = c / CPR, e = (c % CPR) * 8;
      const bool ok = r < nvj;
      cp_async16(&Kt[warp * 32 + r][e], kbase + (ok ? r : 0) * HD + e, ok);
      cp_async16(&Vt[warp * 32 + r][e], vbase + (ok ? r : 0) * HD + e, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (nsub_here > 0) stage(0);
  trace_mark(a, 0);
  pdl_trigger();
  pdl_wait();        // q / k_new / v_new come from the QKV GEMV just before
  trace_mark(a, 1);

  // ---- 2. q (RoPE) -> bf16 hi/lo, [head][dim]; unused heads zero.  All loads
  // of the thread are issued before any arithmetic (one latency, not eight) ----
  {
    constexpr int PER = 8 * HD / NTH;
    float x1[PER], x2[PER], c[PER], sg[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = threadIdx.x + u * NTH, g = i / HD, dd = i % HD, j = dd % half;
      const float* q = qrow + (kh * G + min(g, G - 1)) * HD;
      x1[u] = q[j];
      x2[u] = q[j + half];
      c[u] = cs ? cs[j] : 1.f;
      sg[u] = sn ? sn[j] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = threadIdx.x + u * NTH, g = i / HD, dd = i % HD;
      float v = 0.f;
      if (g < G) {
        if (a.family == kLlama)
          v = dd < half ? __fsub_rn(__fmul_rn(x1[u], c[u]), __fmul_rn(x2[u], sg[u]))
                        : __fadd_rn(__fmul_rn(x2[u], c[u]), __fmul_rn(x1[u], sg[u]));
        else
          v = dd < half ? x1[u] : x2[u];
      }
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      qh[g][dd] = h;
      ql[g][dd] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
  }
  // ---- 3. append the new position (KVCache.append, SP/model.py:163-167) ----
  const bool appender = (a.t0 / CH == chunk);
  const int app_sub = (a.t0 - base) / CHUNK;       // the appender's sub-chunk holding t0
  __nv_bfloat16 knew[HD / NTH > 0 ? HD / NTH : 1], vnew[HD / NTH > 0 ? HD / NTH : 1];
  if (appender) {
    const int page = a.page_table[slot * a.max_pages + a.t0 / kPageTokens];
    __nv_bfloat16* kp = page_ptr<__nv_bfloat16>(a.kv_pool, page, 0, a.kvh, kh, HD) + (a.t0 % kPageTokens) * HD;
    __nv_bfloat16* vp = page_ptr<__nv_bfloat16>(a.kv_pool, page, 1, a.kvh, kh, HD) + (a.t0 % kPageTokens) * HD;
    const float* kn = qrow + a.H * HD + kh * HD;
    const float* vn = qrow + a.H * HD + a.kvh * HD + kh * HD;
#pragma unroll
    for (int u = 0; u * NTH < HD; ++u) {
      const int dd = threadIdx.x + u * NTH;
      if (dd < HD) {
        knew[u] = __float2bfloat16_rn((a.family == kLlama) ? rope_val(kn, dd, half, cs, sn) : kn[dd]);
        vnew[u] = __float2bfloat16_rn(vn[dd]);
        kp[dd] = knew[u];
        vp[dd] = vnew[u];
      }
    }
  }
  const float qscale = kLog2e / sqrtf((float)HD);
  const int jrow = (lane & 7) + ((lane >> 4) << 3);      // ldmatrix.trans source row (pos)
  const int dcol = ((lane >> 3) & 1) * 8;                // +8 dims for matrices 1 and 3
  float m2[2] = {-INFINITY, -INFINITY}, l2[2] = {0.f, 0.f};
  float oacc[HD / 16][4];
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;

  for (int js = 0; js < nsub_here; ++js) {
    if (js + 1 < nsub_here) {
      stage(js + 1);                              // next sub-chunk streams under this one
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (js == 0) trace_mark(a, 2);
    Row* Kt = Kbuf + (js % nbuf) * 128;
    Row* Vt = Vbuf + (js % nbuf) * 128;
    if (appender && js == app_sub) {
      const int r = a.t0 - base - js * CHUNK;
#pragma unroll
      for (int u = 0; u * NTH < HD; ++u) {
        const int dd = threadIdx.x + u * NTH;
        if (dd < HD) { Kt[r][dd] = knew[u]; Vt[r][dd] = vnew[u]; }
      }
      __syncthreads();
    }
    const int p0 = base + js * CHUNK + warp * 32;
    const int nv = max(0, min(32, T - p0));

    // ---- S[32 x 8] = K . q^T ----
    float sacc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
      const uint32_t bh0 = *reinterpret_cast<const uint32_t*>(&qh[g8][ks * 16 + 2 * t4]);
      const uint32_t bh1 = *reinterpret_cast<const uint32_t*>(&qh[g8][ks * 16 + 2 * t4 + 8]);
      const uint32_t bl0 = *reinterpret_cast<const uint32_t*>(&ql[g8][ks * 16 + 2 * t4]);
      const uint32_t bl1 = *reinterpret_cast<const uint32_t*>(&ql[g8][ks * 16 + 2 * t4 + 8]);
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        uint32_t af[4];
        ldsm_x4(af, &Kt[warp * 32 + mt * 16 + (lane & 15)][ks * 16 + (lane >> 4) * 8]);
        mma_bf16_16816(sacc[mt], af[0], af[1], af[2], af[3], bh0, bh1);
        mma_bf16_16816(sacc[mt], af[0], af[1], af[2], af[3], bl0, bl1);
      }
    }
    if (js == 0) trace_mark(a, 8);
    // ---- online softmax per head over the warp's 32 positions ----
    // lane holds S[pos mt*16 + g8 (+8)][head 2*t4 + {0,1}]
    float alpha[2];
#pragma unroll
    for (int hc = 0; hc < 2; ++hc) {
      const int head = 2 * t4 + hc;
      float mx = -INFINITY;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int pos = mt * 16 + g8 + hh * 8;
          // log2 domain: one multiply folds 1/sqrt(hd) and log2(e); exp2 below
          float v = sacc[mt][hh * 2 + hc] * qscale;
          if (a.family == kBloom && head < G)
            v = fmaf(a.alibi[kh * G + head] * kLog2e, (float)(p0 + pos - (T - 1)), v);
          if (pos >= nv) v = -INFINITY;
          sacc[mt][hh * 2 + hc] = v;
          mx = fmaxf(mx, v);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const float mnew = fmaxf(m2[hc], mx);
      alpha[hc] = (m2[hc] == -INFINITY) ? 0.f : ex2_approx(m2[hc] - mnew);
      float sum = 0.f;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int pos = mt * 16 + g8 + hh * 8;
          const float e = (pos < nv) ? ex2_approx(sacc[mt][hh * 2 + hc] - mnew) : 0.f;
          sum += e;
          const __nv_bfloat16 h = __float2bfloat16_rn(e);
          ph[warp][head][pos] = h;
          pl_[warp][head][pos] = __float2bfloat16_rn(e - __bfloat162float(h));
        }
      sum += __shfl_xor_sync(0xffffffffu, sum, 4);
      sum += __shfl_xor_sync(0xffffffffu, sum, 8);
      sum += __shfl_xor_sync(0xffffffffu, sum, 16);
      m2[hc] = mnew;
      l2[hc] = l2[hc] * alpha[hc] + sum;
    }
    __syncwarp();
    if (js == 0) trace_mark(a, 9);
    // ---- O^T[HD x 8] = alpha * O^T + V^T . P ----
#pragma unroll
    for (int mt = 0; mt < HD / 16; ++mt) {
      // oacc columns: head 2*t4 + (j & 1)
      oacc[mt][0] *= alpha[0]; oacc[mt][1] *= alpha[1];
      oacc[mt][2] *= alpha[0]; oacc[mt][3] *= alpha[1];
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        uint32_t af[4];
        ldsm_x4_t(af, &Vt[warp * 32 + ks * 16 + jrow][mt * 16 + dcol]);
        const uint32_t bh0 = *reinterpret_cast<const uint32_t*>(&ph[warp][g8][ks * 16 + 2 * t4]);
        const uint32_t bh1 = *reinterpret_cast<const uint32_t*>(&ph[warp][g8][ks * 16 + 2 * t4 + 8]);
        const uint32_t bl0 = *reinterpret_cast<const uint32_t*>(&pl_[warp][g8][ks * 16 + 2 * t4]);
        const uint32_t bl1 = *reinterpret_cast<const uint32_t*>(&pl_[warp][g8][ks * 16 + 2 * t4 + 8]);
        mma_bf16_16816(oacc[mt], af[0], af[1], af[2], af[3], bh0, bh1);
        mma_bf16_16816(oacc[mt], af[0], af[1], af[2], af[3], bl0, bl1);
      }
    }
    __syncthreads();                              // buffer js & 1 is refilled next
  }
  if (g8 == 0) {
#pragma unroll
    for (int hc = 0; hc < 2; ++hc) {
      const int head = 2 * t4 + hc;
      if (head < G) { wm[warp][head] = m2[hc]; wl[warp][head] = l2[hc]; }
    }
  }
  // oacc: O^T[dim mt*16 + g8 (+8)][head 2*t4 + {0,1}]
#pragma unroll
  for (int mt = 0; mt < HD / 16; ++mt)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int head = 2 * t4 + (j & 1);
      const int dim = mt * 16 + g8 + ((j >> 1) << 3);
      if (head < G) wo[(warp * G + head) * HD + dim] = oacc[mt][j];
    }
  trace_mark(a, 10);
  __syncthreads();
  trace_mark(a, 3);
  if constexpr (CL > 0)
    cluster_merge<HD, CL>(a, G, slot, kh, nsub_here > 0, wm, wl, wo, T, base);
  else
    merge_tail<HD, true, GT>(a, G, slot, kh, chunk, nchunk, T, wm, wl, wo, pmv, plv, &last_flag, CH,
                             reinterpret_cast<float*>(dsm), nbuf * 2 * 4 * 32 * RS / 2);
  trace_mark(a, 7);
}

template <int HD, int GT, int CL>
void launch_mma_cl(const AttnDecArgs& a_in, cudaStream_t st) {
  AttnDecArgs a = a_in;
  const int T = a.t0 + 1;
  // sub-chunks per CTA: one (136 CTAs for 70B GQA at 2 K positions) unless the
  // grid would exceed ~2 CTAs per SM (MHA: 112 kv heads x 17 chunks for BLOOM)
  const int64_t n128 = (int64_t)a.width * a.kvh * ((T + CHUNK - 1) / CHUNK);
  static int num_sms = 0;
  if (!num_sms) cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, current_device());
  int nsub = g_attn_nsub > 0 ? g_attn_nsub : (int)((n128 + 2 * num_sms - 1) / (2 * num_sms));
  if (CL > 0) nsub = (T + CHUNK * CL - 1) / (CHUNK * CL);   // CL CTAs cover the positions
  nsub = nsub < 1 ? 1 : (nsub > 32 ? 32 : nsub);
  a.nsub = nsub;
  dim3 grid(a.width * a.kvh, CL > 0 ? CL : (T + CHUNK * nsub - 1) / (CHUNK * nsub));
  const int G = a.H / a.kvh;
  const size_t smem = (size_t)(nsub > 1 ? 2 : 1) * 2 * 4 * 32 * (HD + 8) * 2 +
                      (size_t)(4 * G * HD + 2 * a.max_pages * GMAX) * sizeof(float);
  static size_t set[kMaxDevices] = {};
  const int dv = current_device();
  if (smem > set[dv]) {
    cudaFuncSetAttribute(attn_dec_mma_kernel<HD, GT, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    if (CL > 8)
      cudaFuncSetAttribute(attn_dec_mma_kernel<HD, GT, CL>,
                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    set[dv] = smem;
  }
  static int trace_call = getenv("SP_ATTN_TRACE") ? atoi(getenv("SP_ATTN_TRACE")) : -1;
  static int ncall = 0;
  static unsigned long long* tbuf = nullptr;
  AttnDecArgs b = a;
  const bool tr = trace_call >= 0 && ncall++ == trace_call;
  const size_t tn = (size_t)grid.x * grid.y * 12;
  if (tr) {
    cudaMalloc(&tbuf, tn * 8);
    cudaMemsetAsync(tbuf, 0, tn * 8, st);
    b.trace = tbuf;
  }
  if (CL > 0)
    launch_pdl_cluster(attn_dec_mma_kernel<HD, GT, CL>, grid, dim3(NTH), smem, st, CL, b);
  else
    launch_pdl(attn_dec_mma_kernel<HD, GT, CL>, grid, dim3(NTH), smem, st, b);
  count_launch();
  if (tr) {
    std::vector<unsigned long long> h(tn);
    cudaMemcpyAsync(h.data(), tbuf, tn * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long t0 = ~0ull;
    for (size_t i = 0; i < tn; i += 12) if (h[i] && h[i] < t0) t0 = h[i];
    for (size_t i = 0; i < tn; i += 12) {
      fprintf(stderr, "cta %3zu:", i / 12);
      for (int p = 0; p < 11; ++p)
        fprintf(stderr, " %7.2f", h[i + p] ? (double)(h[i + p] - t0) / 1e3 : -1.0);
      fprintf(stderr, "\n");
    }
    cudaFree(tbuf);
  }
}

// Cluster merge for G = 8 (70B GQA): 8 CTAs per (slot, kv head) up to 1 K
// positions, 16 beyond (one 128-position sub-chunk each at 2 K).  Measured on
// the 70B shape at 2 K positions: 8-CTA clusters tie the global last-CTA merge
// (0.118 ms per 8-block tick either way), 16-CTA clusters lose (0.167 ms), so
// the default (g_attn_cluster = -1, option 6 / SP_ATTN_CLUSTER) stays global;
// 0 = the size rule above, 8 or 16 = forced.

template <int HD, int GT>
void launch_mma(const AttnDecArgs& a, cudaStream_t st) {
  const int T = a.t0 + 1;
  int cy = 0;
  if (GT == 8 && g_attn_cluster >= 0) {
    cy = g_attn_cluster > 0 ? g_attn_cluster : (T > 8 * CHUNK ? 16 : 8);
    if (T > 32 * CHUNK * cy) cy = 0;
  }
  if (cy == 16) launch_mma_cl<HD, GT, GT == 8 ? 16 : 0>(a, st);
  else if (cy == 8) launch_mma_cl<HD, GT, GT == 8 ? 8 : 0>(a, st);
  else launch_mma_cl<HD, GT, 0>(a, st);
}

template <int HD, typename KT, int GT>
void launch_g(const AttnDecArgs& a, cudaStream_t st) {
  const int T = a.t0 + 1;
  dim3 grid(a.width * a.kvh, (T + CHUNK - 1) / CHUNK);
  const int G = a.H / a.kvh;
  const size_t smem = (size_t)(4 * G * HD + 2 * a.max_pages * GMAX) * sizeof(float);
  static size_t set[kMaxDevices] = {};
  const int dv = current_device();
  if (smem > set[dv]) {
    cudaFuncSetAttribute(attn_dec2_kernel<HD, KT, GT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    set[dv] = smem;
  }
  attn_dec2_kernel<HD, KT, GT><<<grid, NTH, smem, st>>>(a);
  count_launch();
}

template <int HD, typename KT>
void launch_t(const AttnDecArgs& a, cudaStream_t st) {
  switch (a.H / a.kvh) {
    case 1: launch_g<HD, KT, 1>(a, st); break;
    case 8: launch_g<HD, KT, 8>(a, st); break;
    default: launch_g<HD, KT, 0>(a, st); break;
  }
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

int g_attn_nsub = 0;
int g_attn_cluster = getenv("SP_ATTN_CLUSTER") ? atoi(getenv("SP_ATTN_CLUSTER")) : -1;

int64_t attn_dec_part_floats(int width, int H, int hd, int max_pages) {
  return (int64_t)width * H * max_pages * (hd + 2);
}

namespace {
// timing experiment only (SP_DEBUG_ATTN_EMPTY=1, wrong results): a trivial
// dependent kernel with the attention grid, to measure the cost of the kernel
// boundary itself in the PDL chain
__global__ void empty_pdl_kernel(int) {
  pdl_trigger();
  pdl_wait();
}
}  // namespace

bool g_attn_cl = getenv("SP_ATTN_CL") ? atoi(getenv("SP_ATTN_CL")) != 0 : true;

int launch_attn_decode_fused(const AttnDecArgs& a, cudaStream_t st) {
  static const bool empty = getenv("SP_DEBUG_ATTN_EMPTY") != nullptr;
  if (empty) {
    launch_pdl(empty_pdl_kernel, dim3(136), dim3(128), 0, st, 0);
    count_launch();
    return a.H;
  }
  if (attn_dec_mha_ok(a)) return launch_attn_decode_mha(a, st);
  if (g_attn_cl && attn_dec_cl_ok(a)) return launch_attn_decode_cl(a, st);
  const int G = a.H / a.kvh;
  if (a.kv_dtype == kKVBF16 && G <= 8 && (a.hd == 64 || a.hd == 128)) {
    // group size as a template constant for the shapes we serve (70B: 8,
    // MHA/BLOOM: 1); others keep it at run time
    auto go = [&](auto hdc) {
      constexpr int HDv = decltype(hdc)::value;
      switch (G) {
        case 8: launch_mma<HDv, 8>(a, st); break;
        case 1: launch_mma<HDv, 1>(a, st); break;
        default: launch_mma<HDv, 0>(a, st); break;
      }
    };
    if (a.hd == 128) go(std::integral_constant<int, 128>{});
    else go(std::integral_constant<int, 64>{});
    return a.H;
  }
  if (a.kv_dtype == kKVBF16) dispatch<__nv_bfloat16>(a, st);
  else dispatch<float>(a, st);
  return a.H;
}

}  // namespace sp
