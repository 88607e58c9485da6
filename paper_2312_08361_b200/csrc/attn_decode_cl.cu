// Decode attention (n_new == 1) with a thread-block-cluster merge — the
// default decode attention for a bf16 KV cache (head dim 64 / 128, up to 8
// query heads per kv head).
//
// SP/model.py:263-275 at n = 1: scores = q . k / sqrt(hd) (+ ALiBi), no mask,
// max-subtracted softmax, ctx = p . v; the new position's k (RoPE'd) and v are
// appended to the paged cache first (KVCache.append, SP/model.py:163-167).
//
// Work split.  One cluster of CL = 8 CTAs per (slot, kv head); CTA rank c holds
// NW warps, warp w the 32 positions [(s*CL + c)*NW*32 + w*32, +32) of pass s
// (one pass up to CL*NW*32 positions: 3072 with NW = 12).  Every warp's K/V
// rows are staged with cp.async BEFORE the programmatic-launch wait (positions
// < t0 are never rewritten), so after the QKV projection lands only the math
// remains:
//   * S[32 x 8] = K . q^T on mma.m16n8k16 (A = the warp's K rows by ldmatrix,
//     B columns = the kv group's query heads, q split hi + lo bf16 — two MMAs —
//     against the bf16 cache), online softmax per head in the exp2 domain,
//   * O^T[hd x 8] += V^T . P^T (A = V rows transposed by ldmatrix.trans; B = P
//     split hi + lo, turned from the S accumulator layout into B fragments by
//     movmatrix.trans) — no padded rows, 64 MMAs per 32 positions,
//   * the NW warp partials merge in a fixed order in shared memory, then the
//     CL CTA partials merge over distributed shared memory: rank r finalises
//     outputs [r*G*hd/CL, (r+1)*G*hd/CL) reading its 7 peers in rank order.
// No global partials, counters or last-CTA merge (the round-1 kernel's serial
// merge was most of its in-stream cost).  Deterministic: fixed merge orders.
// Each rank also writes the (sum, sumsq, max|x|) partial of its ctx slice:
// P_out = kvh * CL partials per row for the O-projection GEMV's prologue.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "decode.cuh"
#include "kernels.cuh"

namespace sp {

namespace cg = cooperative_groups;

namespace {

constexpr int CL = 8;            // CTAs per (slot, kv head)
constexpr int GM = 8;            // query heads per kv head (rows of the M = 16 tile)
constexpr int NWMAX = 12;        // warps per CTA
constexpr int kMinWarps = 4;     // q preparation and merges run on >= 4 warps
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// transpose of the warp's 8 x 8 b16 matrix fragment (lane (g8, t4) holds row g8,
// columns 2t4, 2t4 + 1 -> afterwards row g8 of the transpose)
__device__ __forceinline__ uint32_t movm_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ void ldsm4(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm4t(uint32_t* r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void cp16z(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(ok ? 16 : 0));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat16 h0 = __float2bfloat16_rn(x0), h1 = __float2bfloat16_rn(x1);
  hi = pack_bf16(__bfloat162float(h0), __bfloat162float(h1));
  lo = pack_bf16(x0 - __bfloat162float(h0), x1 - __bfloat162float(h1));
}

// debug (SP_BUILD_TRACE=1 build + SP_ATTN_TRACE=<call>): per-CTA phase times
__device__ __forceinline__ void cl_mark(const AttnDecArgs& a, int ph) {
  if (SP_DEV_TRACE && a.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    a.trace[(blockIdx.y * gridDim.x + blockIdx.x) * 12 + ph] = t;
  }
}

template <int HD>
struct Layout {
  static constexpr int RS = HD + 8;                      // padded bf16 row (ldmatrix banks)
  static constexpr int KV_WARP = 32 * RS * 2;            // bytes of one warp's K (or V) rows
  static constexpr int Q_BYTES = 2 * GM * RS * 2;        // q hi, lo
  static constexpr int OC_BYTES = GM * HD * 4;           // CTA partial O
  static size_t bytes(int nw) {
    return (size_t)2 * nw * KV_WARP + Q_BYTES + OC_BYTES + 2 * NWMAX * GM * 4 + 4 * GM * 4 + 256;
  }
};

template <int HD>
__global__ void __launch_bounds__(NWMAX * 32, 1) attn_dec_cl_kernel(AttnDecArgs a) {
  using L = Layout<HD>;
  constexpr int RS = L::RS;
  extern __shared__ __align__(128) uint8_t dsm[];
  const int NW = blockDim.x >> 5;
  typedef __nv_bfloat16 Row[RS];
  Row* Ks = reinterpret_cast<Row*>(dsm);                            // [NW*32]
  Row* Vs = reinterpret_cast<Row*>(dsm + (size_t)NW * L::KV_WARP);  // [NW*32]
  Row* Qh = reinterpret_cast<Row*>(dsm + (size_t)2 * NW * L::KV_WARP);   // [GM]
  Row* Ql = Qh + GM;
  float* Oc = reinterpret_cast<float*>(dsm + (size_t)2 * NW * L::KV_WARP + L::Q_BYTES);  // [GM][HD]
  float* mw = Oc + GM * HD;                       // [NWMAX][GM] warp maxima
  float* lw = mw + NWMAX * GM;                    // [NWMAX][GM] warp sums
  float* Mc = lw + NWMAX * GM;                    // [GM] CTA max
  float* Lc = Mc + GM;                            // [GM] CTA sum

  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int slot = blockIdx.x / a.kvh, kh = blockIdx.x % a.kvh;
  const int G = a.H / a.kvh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
  const int T = a.t0 + 1;
  const int PC = NW * 32;                          // positions per CTA per pass
  const int npass = (T + CL * PC - 1) / (CL * PC);
  const int half = HD / 2;
  const float* qrow = a.qkv + (int64_t)slot * a.ldqkv;
  Row* Kw = Ks + warp * 32;
  Row* Vw = Vs + warp * 32;

  // this warp's 32 K/V rows of pass s (zero-filled past T; the row of t0 is
  // stale until the append below patches it)
  auto stage = [&](int s) {
    const int p0 = (s * CL + rank) * PC + warp * 32;
    const int nv = max(0, min(32, T - p0));
    if (nv == 0) return;
    const int page = a.page_table[slot * a.max_pages + p0 / kPageTokens];
    const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(a.kv_pool) +
                              (((int64_t)page * 2 + 0) * a.kvh + kh) * kPageTokens * HD +
                              (p0 % kPageTokens) * HD;
    const __nv_bfloat16* vb = kb + (int64_t)a.kvh * kPageTokens * HD;
    constexpr int CPR = HD / 8;                   // 16-byte chunks per row
#pragma unroll 4
    for (int c = lane; c < 32 * CPR; c += 32) {
      const int r = c / CPR, e = (c % CPR) * 8;
      const bool ok = r < nv;
      cp16z(&Kw[r][e], kb + (ok ? r : 0) * HD + e, ok);
      cp16z(&Vw[r][e], vb + (ok ? r : 0) * HD + e, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  cl_mark(a, 0);
  stage(0);
  cl_mark(a, 1);
  pdl_trigger();
  pdl_wait();
  cl_mark(a, 2);

  // ---- q of the kv group (RoPE at t0), hi/lo bf16, rows >= G zero ----
  // (g, j < half) pairs; every load of a thread is issued before the first
  // store (one L2 round trip, not one per pair)
  const float* cs = a.rope_cos ? a.rope_cos + (int64_t)a.t0 * half : nullptr;
  const float* sn = a.rope_sin ? a.rope_sin + (int64_t)a.t0 * half : nullptr;
  const bool llama = a.family == kLlama;
  {
    constexpr int QI = GM * HD / 2 / (kMinWarps * 32);
    float x0[QI], x1[QI], c0[QI], s0[QI];
#pragma unroll
    for (int u = 0; u < QI; ++u) {
      const int i = threadIdx.x + u * blockDim.x, g = i / half, j = i % half;
      x0[u] = x1[u] = 0.f;
      c0[u] = 1.f;
      s0[u] = 0.f;
      if (i < GM * half && g < G) {
        const float* q = qrow + (kh * G + g) * HD;
        x0[u] = q[j];
        x1[u] = q[j + half];
        if (llama) { c0[u] = cs[j]; s0[u] = sn[j]; }
      }
    }
#pragma unroll
    for (int u = 0; u < QI; ++u) {
      const int i = threadIdx.x + u * blockDim.x, g = i / half, j = i % half;
      if (i < GM * half) {
        float v0 = x0[u], v1 = x1[u];
        if (llama) {
          v0 = __fsub_rn(__fmul_rn(x0[u], c0[u]), __fmul_rn(x1[u], s0[u]));
          v1 = __fadd_rn(__fmul_rn(x1[u], c0[u]), __fmul_rn(x0[u], s0[u]));
        }
        const __nv_bfloat16 h0 = __float2bfloat16_rn(v0), h1 = __float2bfloat16_rn(v1);
        Qh[g][j] = h0;
        Qh[g][j + half] = h1;
        Ql[g][j] = __float2bfloat16_rn(v0 - __bfloat162float(h0));
        Ql[g][j + half] = __float2bfloat16_rn(v1 - __bfloat162float(h1));
      }
    }
  }
  // the new position: k (RoPE'd) and v appended to the page by the warp that
  // owns t0 (patched into its staged rows after the wait below)
  const int app_pass = a.t0 / (CL * PC);
  const int app_off = a.t0 - app_pass * CL * PC - rank * PC - warp * 32;
  const bool appender = app_off >= 0 && app_off < 32;
  __nv_bfloat16 knew[HD / 32], vnew[HD / 32];
  if (appender) {
    const int page = a.page_table[slot * a.max_pages + a.t0 / kPageTokens];
    __nv_bfloat16* kp = reinterpret_cast<__nv_bfloat16*>(a.kv_pool) +
                        (((int64_t)page * 2 + 0) * a.kvh + kh) * kPageTokens * HD +
                        (a.t0 % kPageTokens) * HD;
    __nv_bfloat16* vp = kp + (int64_t)a.kvh * kPageTokens * HD;
    const float* kn = qrow + a.H * HD + kh * HD;
    const float* vn = qrow + a.H * HD + a.kvh * HD + kh * HD;
    float kv_[HD / 32], kr_[HD / 32], vv_[HD / 32], ck[HD / 32], sk[HD / 32];
#pragma unroll
    for (int u = 0; u < HD / 32; ++u) {
      const int dd = lane + 32 * u, j = dd % half;
      kv_[u] = kn[dd];
      kr_[u] = kn[dd < half ? dd + half : dd - half];
      vv_[u] = vn[dd];
      if (llama) { ck[u] = cs[j]; sk[u] = sn[j]; }
    }
#pragma unroll
    for (int u = 0; u < HD / 32; ++u) {
      const int dd = lane + 32 * u;
      float kx = kv_[u];
      if (llama)   // rope_at: x[j] c - x[j+half] s  /  x[j+half] c + x[j] s
        kx = dd < half ? __fsub_rn(__fmul_rn(kv_[u], ck[u]), __fmul_rn(kr_[u], sk[u]))
                       : __fadd_rn(__fmul_rn(kv_[u], ck[u]), __fmul_rn(kr_[u], sk[u]));
      knew[u] = __float2bfloat16_rn(kx);
      vnew[u] = __float2bfloat16_rn(vv_[u]);
      kp[dd] = knew[u];
      vp[dd] = vnew[u];
    }
  }
  __syncthreads();                                 // q visible
  cl_mark(a, 3);

  const float qscale = kLog2e / sqrtf((float)HD);
  // this lane's two heads (B / C columns 2*t4, 2*t4 + 1)
  const int hA = 2 * t4, hB = 2 * t4 + 1;
  const float slA = (a.family == kBloom && hA < G) ? a.alibi[kh * G + hA] * kLog2e : 0.f;
  const float slB = (a.family == kBloom && hB < G) ? a.alibi[kh * G + hB] * kLog2e : 0.f;

  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};   // heads hA, hB
  // O^T[dims x heads]: dim tile dt, c0/c1 = (dim dt*16 + g8, hA / hB), c2/c3 = (+8)
  float o[HD / 16][4];
#pragma unroll
  for (int i = 0; i < HD / 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;

  for (int s = 0; s < npass; ++s) {
    const int p0 = (s * CL + rank) * PC + warp * 32;
    const int nv = max(0, min(32, T - p0));
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if (s == 0) cl_mark(a, 4);
    if (nv > 0) {
      if (appender && s == app_pass) {
#pragma unroll
        for (int u = 0; u < HD / 32; ++u) {
          Kw[app_off][lane + 32 * u] = knew[u];
          Vw[app_off][lane + 32 * u] = vnew[u];
        }
        __syncwarp();
      }
      // ---- S[32 positions x 8 heads] = K . q^T (A = K rows, B = q hi / lo) ----
      float sc[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) sc[mt][0] = sc[mt][1] = sc[mt][2] = sc[mt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < HD / 16; ++ks) {
        const uint32_t h0 = *reinterpret_cast<const uint32_t*>(&Qh[g8][ks * 16 + 2 * t4]);
        const uint32_t h1 = *reinterpret_cast<const uint32_t*>(&Qh[g8][ks * 16 + 8 + 2 * t4]);
        const uint32_t l0 = *reinterpret_cast<const uint32_t*>(&Ql[g8][ks * 16 + 2 * t4]);
        const uint32_t l1 = *reinterpret_cast<const uint32_t*>(&Ql[g8][ks * 16 + 8 + 2 * t4]);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          uint32_t ka[4];
          const int m = lane >> 3;
          ldsm4(ka, &Kw[mt * 16 + (m & 1) * 8 + (lane & 7)][ks * 16 + (m >> 1) * 8]);
          mma16816(sc[mt], ka, h0, h1);
          mma16816(sc[mt], ka, l0, l1);
        }
      }
      // ---- online softmax per head: sc[mt][j] = (position mt*16 + g8 + 8*(j>>1), head 2*t4 + (j&1))
      float tmA = -INFINITY, tmB = -INFINITY;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int pos = p0 + mt * 16 + g8 + 8 * (j >> 1);
          float v = sc[mt][j] * qscale;
          if (a.family == kBloom) v = fmaf((j & 1) ? slB : slA, (float)(pos - a.t0), v);
          if (pos >= T) v = -INFINITY;
          sc[mt][j] = v;
          if (j & 1) tmB = fmaxf(tmB, v); else tmA = fmaxf(tmA, v);
        }
#pragma unroll
      for (int sh = 4; sh <= 16; sh <<= 1) {
        tmA = fmaxf(tmA, __shfl_xor_sync(0xffffffffu, tmA, sh));
        tmB = fmaxf(tmB, __shfl_xor_sync(0xffffffffu, tmB, sh));
      }
      const float mnA = fmaxf(m_run[0], tmA), mnB = fmaxf(m_run[1], tmB);
      const float alA = (m_run[0] == -INFINITY) ? 0.f : ex2_approx(m_run[0] - mnA);
      const float alB = (m_run[1] == -INFINITY) ? 0.f : ex2_approx(m_run[1] - mnB);
      float psA = 0.f, psB = 0.f;
      // P^T B fragments (k = positions, n = heads): the S accumulator holds (position g8,
      // heads 2t4..) pairs; movmatrix.trans turns each 8 x 8 block into (head g8,
      // positions 2t4..) pairs = the B fragment of the next MMA
      uint32_t bh[2][2], bl[2][2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {       // positions g8 (hh = 0) or g8 + 8
          const float pa = ex2_approx(sc[mt][2 * hh] - mnA);       // -inf -> +0
          const float pb = ex2_approx(sc[mt][2 * hh + 1] - mnB);
          psA += pa;
          psB += pb;
          uint32_t hi, lo;
          split2(pa, pb, hi, lo);
          bh[mt][hh] = movm_trans(hi);
          bl[mt][hh] = movm_trans(lo);
        }
#pragma unroll
      for (int sh = 4; sh <= 16; sh <<= 1) {
        psA += __shfl_xor_sync(0xffffffffu, psA, sh);
        psB += __shfl_xor_sync(0xffffffffu, psB, sh);
      }
      l_run[0] = l_run[0] * alA + psA;
      l_run[1] = l_run[1] * alB + psB;
      m_run[0] = mnA;
      m_run[1] = mnB;
#pragma unroll
      for (int i = 0; i < HD / 16; ++i) {
        o[i][0] *= alA; o[i][1] *= alB; o[i][2] *= alA; o[i][3] *= alB;
      }
      // ---- O^T[dims x heads] += V^T . P^T (A = V rows transposed by ldmatrix) ----
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
        for (int dt = 0; dt < HD / 16; ++dt) {
          uint32_t va[4];
          const int m = lane >> 3;
          ldsm4t(va, &Vw[kk * 16 + (m >> 1) * 8 + (lane & 7)][dt * 16 + (m & 1) * 8]);
          mma16816(o[dt], va, bh[kk][0], bh[kk][1]);
          mma16816(o[dt], va, bl[kk][0], bl[kk][1]);
        }
      }
    }
    if (s + 1 < npass) {
      __syncwarp();
      stage(s + 1);                                // this warp's slots are free again
    }
  }

  cl_mark(a, 5);
  // ---- warp partials -> shared (O over this warp's own K rows) ----
  float* Ow = reinterpret_cast<float*>(Kw);        // [GM][HD] f32 fits 32 K rows
  __syncwarp();
#pragma unroll
  for (int dt = 0; dt < HD / 16; ++dt) {
    if (hA < G) {
      Ow[hA * HD + dt * 16 + g8] = o[dt][0];
      Ow[hA * HD + dt * 16 + g8 + 8] = o[dt][2];
    }
    if (hB < G) {
      Ow[hB * HD + dt * 16 + g8] = o[dt][1];
      Ow[hB * HD + dt * 16 + g8 + 8] = o[dt][3];
    }
  }
  if (g8 == 0) {
    if (hA < G) { mw[warp * GM + hA] = m_run[0]; lw[warp * GM + hA] = l_run[0]; }
    if (hB < G) { mw[warp * GM + hB] = m_run[1]; lw[warp * GM + hB] = l_run[1]; }
  }
  __syncthreads();
  // ---- CTA merge over warps (fixed order): factors f_w = exp2(m_w - M),
  // recomputed by every thread for its own head (no serial factor phase);
  // four consecutive outputs (one head) per thread ----
  for (int i4 = threadIdx.x; i4 < G * HD / 4; i4 += blockDim.x) {
    const int g = i4 * 4 / HD;
    float M = -INFINITY;
    for (int w = 0; w < NW; ++w) M = fmaxf(M, mw[w * GM + g]);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float Ls = 0.f;
#pragma unroll 3
    for (int w = 0; w < NW; ++w) {
      const float m = mw[w * GM + g];
      const float f = (m == -INFINITY) ? 0.f : ex2_approx(m - M);
      Ls = fmaf(lw[w * GM + g], f, Ls);
      if (f != 0.f) {
        const float4 o = reinterpret_cast<const float4*>(Ks + w * 32)[i4];
        acc.x = fmaf(o.x, f, acc.x);
        acc.y = fmaf(o.y, f, acc.y);
        acc.z = fmaf(o.z, f, acc.z);
        acc.w = fmaf(o.w, f, acc.w);
      }
    }
    reinterpret_cast<float4*>(Oc)[i4] = acc;
    if (i4 * 4 % HD == 0) { Mc[g] = M; Lc[g] = Ls; }
  }
  cl_mark(a, 6);
  cluster.sync();                                   // every CTA partial visible cluster-wide
  cl_mark(a, 7);

  // ---- rank merge over the cluster (fixed rank order) ----
  // every distributed-shared-memory load of a thread is issued before its
  // first use (the 8 peers' (max, sum) and O values in flight together: one
  // DSMEM round trip, not a chain of 16)
  const int GH = G * HD;
  const int i0 = rank * GH / CL, i1 = (rank + 1) * GH / CL;
  float S = 0.f, Q = 0.f, Mx = 0.f;
  float* ctx = a.ctx + (int64_t)slot * a.H * HD + (int64_t)kh * G * HD;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const int g = i / HD;
    float pm[CL], pl[CL], po[CL];
#pragma unroll
    for (int c = 0; c < CL; ++c) {
      pm[c] = *cluster.map_shared_rank(&Mc[g], c);
      pl[c] = *cluster.map_shared_rank(&Lc[g], c);
      po[c] = *cluster.map_shared_rank(&Oc[i], c);
    }
    float M = -INFINITY;
#pragma unroll
    for (int c = 0; c < CL; ++c) M = fmaxf(M, pm[c]);
    float Ls = 0.f, acc = 0.f;
#pragma unroll
    for (int c = 0; c < CL; ++c) {
      const float f = (pm[c] == -INFINITY) ? 0.f : ex2_approx(pm[c] - M);
      Ls = fmaf(pl[c], f, Ls);
      acc = fmaf(po[c], f, acc);
    }
    const float v = acc / Ls;
    ctx[i] = v;
    S += v;
    Q = fmaf(v, v, Q);
    Mx = fmaxf(Mx, fabsf(v));
  }
  // (relaxed: the DSMEM loads have returned — their values are used above)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  cl_mark(a, 8);
  if (a.st_out) {
    // fixed-order block reduction of this rank's slice statistics
    S = warp_sum(S); Q = warp_sum(Q); Mx = warp_max(Mx);
    __shared__ float red[NWMAX][3];
    if (lane == 0) { red[warp][0] = S; red[warp][1] = Q; red[warp][2] = Mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      float s2 = 0.f, q2 = 0.f, m2 = 0.f;
      for (int w = 0; w < NW; ++w) { s2 += red[w][0]; q2 += red[w][1]; m2 = fmaxf(m2, red[w][2]); }
      a.st_out[(int64_t)(kh * CL + rank) * a.width + slot] = RowStat{s2, q2, m2, 0.f};
    }
  }
  cl_mark(a, 9);
  // peers' shared memory read by everyone before any CTA exits (arrived right
  // after this CTA's last DSMEM read, above)
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  cl_mark(a, 10);
}

template <int HD>
int launch_hd(const AttnDecArgs& a, cudaStream_t st) {
  const int T = a.t0 + 1;
  const int nw = max(kMinWarps, min(NWMAX, (T + CL * 32 - 1) / (CL * 32)));
  const size_t smem = Layout<HD>::bytes(nw);
  static bool set[kMaxDevices] = {};
  const int dv = current_device();
  if (!set[dv]) {
    cudaFuncSetAttribute(attn_dec_cl_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Layout<HD>::bytes(NWMAX));
    set[dv] = true;
  }
  static int trace_call = getenv("SP_ATTN_TRACE") ? atoi(getenv("SP_ATTN_TRACE")) : -1;
  static int ncall = 0;
  AttnDecArgs b = a;
  const dim3 grid(a.width * a.kvh, CL);
  const bool tr = SP_DEV_TRACE && trace_call >= 0 && ncall++ == trace_call;
  const size_t tn = (size_t)grid.x * grid.y * 12;
  unsigned long long* tbuf = nullptr;
  if (tr) {
    cudaMalloc(&tbuf, tn * 8);
    cudaMemsetAsync(tbuf, 0, tn * 8, st);
    b.trace = tbuf;
  }
  launch_pdl_cluster(attn_dec_cl_kernel<HD>, grid, dim3(nw * 32), smem, st, CL, b);
  count_launch();
  if (tr) {
    std::vector<unsigned long long> h(tn);
    cudaMemcpyAsync(h.data(), tbuf, tn * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long t0 = ~0ull;
    for (size_t i = 0; i < tn; i += 12) if (h[i] && h[i] < t0) t0 = h[i];
    fprintf(stderr, "attn_dec_cl T=%d nw=%d phases: start staged waited q cp_done computed "
            "cta_merged cl_sync merged stats end\n", T, nw);
    for (size_t i = 0; i < tn; i += 12) {
      fprintf(stderr, "cta %3zu:", i / 12);
      for (int p = 0; p < 11; ++p)
        fprintf(stderr, " %7.2f", h[i + p] ? (double)(h[i + p] - t0) / 1e3 : -1.0);
      fprintf(stderr, "\n");
    }
    cudaFree(tbuf);
  }
  return a.kvh * CL;
}

}  // namespace

// the cluster kernel serves bf16 KV caches with head dim 64 / 128 and up to 8
// query heads per kv head while one wave of clusters covers the grid
bool attn_dec_cl_ok(const AttnDecArgs& a) {
  const int G = a.H / a.kvh;
  return a.kv_dtype == kKVBF16 && (a.hd == 64 || a.hd == 128) && G <= GM &&
         (int64_t)a.width * a.kvh * CL <= 4 * 148;
}

int launch_attn_decode_cl(const AttnDecArgs& a, cudaStream_t st) {
  return a.hd == 128 ? launch_hd<128>(a, st) : launch_hd<64>(a, st);
}

}  // namespace sp
