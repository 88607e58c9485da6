// Prefill / replay attention (n_new > 1) on tensor cores, flash-style.
//
// CTA = (slot, query head, 128 query rows); 8 warps x 16 rows share each K/V tile.  Key/value pages
// (64 positions, bf16, head dim 64/128) stream through a double-buffered
// cp.async ring; S = Q K^T and O += P V run on mma.m16n8k16 with the online
// softmax of FlashAttention-2.  Q and P are rounded to bf16 like the cached
// K/V (the precision class the bf16 KV cache already sets); with
// sp_span_set_option(.., 3, 1) they are split hi + lo (two MMAs each) and the
// result tracks the f32 reference more closely.  Accumulation is f32 (SP/model.py:263-275: scores / f32(sqrt(hd)),
// (+ ALiBi), causal -1e30 mask for n > 1, max-subtracted softmax).
// Each query row's result depends only on its own row: batch/tile invariant.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int KTL = 64;           // keys per tile (one page)

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
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
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo_elem, float hi_elem) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);
  return *reinterpret_cast<uint32_t*>(&v);
}
// x -> (hi, lo) bf16 pairs for two consecutive elements
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat16 h0 = __float2bfloat16_rn(x0), h1 = __float2bfloat16_rn(x1);
  hi = pack_bf16(__bfloat162float(h0), __bfloat162float(h1));
  lo = pack_bf16(x0 - __bfloat162float(h0), x1 - __bfloat162float(h1));
}

template <int HD, bool HILO, int NWARP>
__global__ void __launch_bounds__(NWARP * 32) attn_prefill_mma_kernel(AttnArgs a) {
  constexpr int QT = 16 * NWARP;                    // query rows per CTA (share each K/V tile)
  constexpr int RS = HD + 8;                        // padded smem row (bf16)
  constexpr int NKS = HD / 16;                      // k-steps over dims
  extern __shared__ __align__(16) uint8_t dsm_[];
  typedef __nv_bfloat16 Tile[KTL][RS];
  Tile* Ks = reinterpret_cast<Tile*>(dsm_);        // [2]
  Tile* Vs = Ks + 2;                                // [2]

  const int G = a.H / a.kvh;
  const int slot = blockIdx.x / a.H, h = blockIdx.x % a.H, kh = h / G;
  // the heaviest (latest) query tiles launch first: causal work grows with q0
  const int q0 = (gridDim.y - 1 - blockIdx.y) * QT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g8 = lane >> 2, t4 = lane & 3;
  const int qrow0 = q0 + warp * 16;                 // this warp's first query row
  const float slope = (a.family == kBloom) ? a.alibi[h] : 0.f;
  const float qscale = 1.4426950408889634f / sqrtf((float)HD);   // log2(e) / sqrt(hd)
  const float slope_l2 = slope * 1.4426950408889634f;

  // ---- Q fragments (hi/lo bf16) for rows qrow0+g8 and qrow0+g8+8 ----
  uint32_t qh[NKS][4], ql[NKS][4];
  {
    const int r_a = min(qrow0 + g8, a.n_new - 1), r_b = min(qrow0 + g8 + 8, a.n_new - 1);
    const float* qa = a.qkv + (int64_t)(slot * a.n_new + r_a) * a.ldqkv + h * HD;
    const float* qb = a.qkv + (int64_t)(slot * a.n_new + r_b) * a.ldqkv + h * HD;
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
      const int c = ks * 16 + 2 * t4;
      const float2 a0 = *reinterpret_cast<const float2*>(qa + c);
      const float2 a1 = *reinterpret_cast<const float2*>(qb + c);
      const float2 a2 = *reinterpret_cast<const float2*>(qa + c + 8);
      const float2 a3 = *reinterpret_cast<const float2*>(qb + c + 8);
      split2(a0.x, a0.y, qh[ks][0], ql[ks][0]);
      split2(a1.x, a1.y, qh[ks][1], ql[ks][1]);
      split2(a2.x, a2.y, qh[ks][2], ql[ks][2]);
      split2(a3.x, a3.y, qh[ks][3], ql[ks][3]);
    }
  }

  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};

  const int last_q = min(q0 + QT, a.n_new) - 1;
  const int kend = a.t0 + last_q + 1;               // keys visible to this CTA
  const int ntiles = (kend + KTL - 1) / KTL;
  const int pos_a = a.t0 + qrow0 + g8, pos_b = pos_a + 8;

  auto load_tile = [&](int kt, int buf) {
    const int page = a.page_table[slot * a.max_pages + kt];
    const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(a.kv_pool) +
                              (((int64_t)page * 2 + 0) * a.kvh + kh) * kPageTokens * HD;
    const __nv_bfloat16* vp = reinterpret_cast<const __nv_bfloat16*>(a.kv_pool) +
                              (((int64_t)page * 2 + 1) * a.kvh + kh) * kPageTokens * HD;
    constexpr int CPR = HD / 8;                     // 16-byte chunks per row
    for (int c = threadIdx.x; c < KTL * CPR; c += NWARP * 32) {
      const int j = c / CPR, e = (c % CPR) * 8;
      cp16(&Ks[buf][j][e], kp + j * HD + e);
      cp16(&Vs[buf][j][e], vp + j * HD + e);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  load_tile(0, 0);
  for (int kt = 0; kt < ntiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ntiles) {
      load_tile(kt + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int kbase = kt * KTL;
    // ---- S = Q K^T : 8 n-tiles of 8 keys ----
    float s[KTL / 8][4];
#pragma unroll
    for (int nt = 0; nt < KTL / 8; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
    if (kbase <= a.t0 + qrow0 + 15) {               // warp-uniform: some key visible
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
#pragma unroll
        for (int np = 0; np < KTL / 16; ++np) {     // pairs of n-tiles
          uint32_t kb[4];
          const int m = lane >> 3;
          ldsm4(kb, &Ks[buf][np * 16 + (m >> 1) * 8 + (lane & 7)][ks * 16 + (m & 1) * 8]);
          mma16816(s[2 * np], qh[ks], kb[0], kb[1]);
          if (HILO) mma16816(s[2 * np], ql[ks], kb[0], kb[1]);
          mma16816(s[2 * np + 1], qh[ks], kb[2], kb[3]);
          if (HILO) mma16816(s[2 * np + 1], ql[ks], kb[2], kb[3]);
        }
      }
    }
    // ---- scale, ALiBi, causal mask, online softmax ----
    float tmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < KTL / 8; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int key = kbase + nt * 8 + 2 * t4 + (j & 1);
        const int pos = (j < 2) ? pos_a : pos_b;
        // log2-domain scores: exp(x - m) == exp2(x*log2e - m*log2e); the
        // 1/sqrt(hd) scale and log2(e) fold into one multiply (bf16-class)
        float v = s[nt][j] * qscale;
        if (a.family == kBloom) v = fmaf(slope_l2, (float)(key - pos), v);
        if (key > pos) v = -INFINITY;
        s[nt][j] = v;
        tmax[j >> 1] = fmaxf(tmax[j >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      tmax[r] = fmaxf(tmax[r], __shfl_xor_sync(0xffffffffu, tmax[r], 1));
      tmax[r] = fmaxf(tmax[r], __shfl_xor_sync(0xffffffffu, tmax[r], 2));
    }
    float mnew[2], alpha[2], psum[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(mrow[r], tmax[r]);
      alpha[r] = (mnew[r] == -INFINITY) ? 1.f : ex2_approx(mrow[r] - mnew[r]);
    }
    uint32_t ph[KTL / 16][4], pl[KTL / 16][4];
#pragma unroll
    for (int nt = 0; nt < KTL / 8; ++nt) {
      float p[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float mr = mnew[j >> 1];
        p[j] = (s[nt][j] == -INFINITY) ? 0.f : ex2_approx(s[nt][j] - mr);
        psum[j >> 1] += p[j];
      }
      // C layout of two n-tiles == A layout of one k16 step of P
      const int kk = nt >> 1, hi_half = nt & 1;
      split2(p[0], p[1], ph[kk][hi_half * 2 + 0], pl[kk][hi_half * 2 + 0]);
      split2(p[2], p[3], ph[kk][hi_half * 2 + 1], pl[kk][hi_half * 2 + 1]);
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      psum[r] += __shfl_xor_sync(0xffffffffu, psum[r], 1);
      psum[r] += __shfl_xor_sync(0xffffffffu, psum[r], 2);
      lrow[r] = lrow[r] * alpha[r] + psum[r];
      mrow[r] = mnew[r];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= alpha[0]; o[i][1] *= alpha[0];
      o[i][2] *= alpha[1]; o[i][3] *= alpha[1];
    }
    // ---- O += P V : 16 keys per k-step, 8 dims per n-tile ----
    if (kbase <= a.t0 + qrow0 + 15) {
#pragma unroll
      for (int kk = 0; kk < KTL / 16; ++kk) {
#pragma unroll
        for (int dp = 0; dp < HD / 16; ++dp) {      // pairs of dim n-tiles
          uint32_t vb[4];
          const int m = lane >> 3;
          ldsm4t(vb, &Vs[buf][kk * 16 + (m & 1) * 8 + (lane & 7)][dp * 16 + (m >> 1) * 8]);
          mma16816(o[2 * dp], ph[kk], vb[0], vb[1]);
          if (HILO) mma16816(o[2 * dp], pl[kk], vb[0], vb[1]);
          mma16816(o[2 * dp + 1], ph[kk], vb[2], vb[3]);
          if (HILO) mma16816(o[2 * dp + 1], pl[kk], vb[2], vb[3]);
        }
      }
    }
    __syncthreads();
  }
  // ---- write ctx rows (one reciprocal per row, then multiplies) ----
  const float inv0 = __frcp_rn(lrow[0]), inv1 = __frcp_rn(lrow[1]);
  const int ra = qrow0 + g8, rb = ra + 8;
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int dim = i * 8 + 2 * t4;
    if (ra < a.n_new) {
      float* dst = a.ctx + (int64_t)(slot * a.n_new + ra) * a.H * HD + h * HD + dim;
      *reinterpret_cast<float2*>(dst) = make_float2(o[i][0] * inv0, o[i][1] * inv0);
    }
    if (rb < a.n_new) {
      float* dst = a.ctx + (int64_t)(slot * a.n_new + rb) * a.H * HD + h * HD + dim;
      *reinterpret_cast<float2*>(dst) = make_float2(o[i][2] * inv1, o[i][3] * inv1);
    }
  }
}

}  // namespace

template <int HD, bool HILO, int NW>
void launch_hd(const AttnArgs& a, size_t smem, cudaStream_t st) {
  static bool set[kMaxDevices] = {};
  const int dv = current_device();
  if (!set[dv]) {
    cudaFuncSetAttribute(attn_prefill_mma_kernel<HD, HILO, NW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set[dv] = true;
  }
  dim3 grid(a.width * a.H, (a.n_new + 16 * NW - 1) / (16 * NW));
  attn_prefill_mma_kernel<HD, HILO, NW><<<grid, NW * 32, smem, st>>>(a);
}

bool g_attn_hilo = false;

template <int HD, bool HILO>
void launch_nw(const AttnArgs& a, size_t smem, cudaStream_t st) {
  static int nw = getenv("SP_ATTN_PF_WARPS") ? atoi(getenv("SP_ATTN_PF_WARPS")) : 4;
  if (nw == 8) launch_hd<HD, HILO, 8>(a, smem, st);
  else launch_hd<HD, HILO, 4>(a, smem, st);
}

bool launch_attention_prefill_mma(const AttnArgs& a, cudaStream_t st) {
  if (a.kv_dtype != kKVBF16 || !(a.hd == 64 || a.hd == 128)) return false;
  const size_t smem = (size_t)4 * KTL * (a.hd + 8) * 2;
  if (a.hd == 128) {
    if (g_attn_hilo) launch_nw<128, true>(a, smem, st);
    else launch_nw<128, false>(a, smem, st);
  } else {
    if (g_attn_hilo) launch_nw<64, true>(a, smem, st);
    else launch_nw<64, false>(a, smem, st);
  }
  count_launch();
  return true;
}

}  // namespace sp
