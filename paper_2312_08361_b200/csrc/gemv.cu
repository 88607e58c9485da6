// Decode linear layers (n_new == 1): y[r, n] = sum_k x[r, k] * W[n, k] (+ epilogue).
//
// Weight-streaming GEMV for bf16 / int8 weights on the tensor pipe:
//   * weights are stored fragment-tiled (common.cuh): every lane issues one
//     coalesced 16-byte LDG per tile and the bytes ARE its mma.m16n8k16 A
//     fragment — no shuffles, no shared-memory staging of weights;
//   * int8 codes are offset-binary u8; one PRMT builds two f16 (1024 + u) and
//     one HSUB2 removes the bias — exact, 1 op / element;
//   * the activation column is split hi/lo (x = hi + lo, both f16 or bf16),
//     packed as two MMA columns, so the product keeps ~22 mantissa bits
//     (f32-class) while the tensor pipe does the multiply-adds;
//   * for f16 the k-chunk of each row is pre-scaled by a power of two (exact)
//     so hi/lo never overflow or go subnormal;
//   * split-K over CTAs with a fixed-order, last-arriving-CTA reduction:
//     deterministic and independent of the batch size R.
// The bound is HBM: bytes = N*K*elt (+4N scales) per launch.
//
// f32 weights (the reference toy model) use a SIMT warp-per-
// row GEMV with a fixed shuffle-tree reduction.
#include "common.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int kNW = 8;        // warps per CTA (split K inside the CTA)
constexpr int kRT = 2;        // 16-row tiles per CTA
constexpr int kU = 4;         // k-tiles in flight per lane per row tile
constexpr int kMaxR = 4;      // batch rows per MMA column group (hi+lo -> 8 columns)

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// two offset-binary bytes -> f16x2 of (u - 128), exact
__device__ __forceinline__ uint32_t u8x2_to_f16x2(uint32_t w, uint32_t sel) {
  uint32_t h = prmt(w, 0x64646464u, sel);   // (1024 + u) as f16
  uint32_t r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(h), "r"(0x64806480u));
  return r;
}

__device__ __forceinline__ void mma_f16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int WT>
__device__ __forceinline__ uint32_t pack_split(float x0, float x1, int part) {
  if (WT == kI8) {
    __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
    if (part) {
      h0 = __float2half_rn(x0 - __half2float(h0));
      h1 = __float2half_rn(x1 - __half2float(h1));
    }
    __half2 v = __halves2half2(h0, h1);
    return *reinterpret_cast<uint32_t*>(&v);
  } else {
    __nv_bfloat16 h0 = __float2bfloat16_rn(x0), h1 = __float2bfloat16_rn(x1);
    if (part) {
      h0 = __float2bfloat16_rn(x0 - __bfloat162float(h0));
      h1 = __float2bfloat16_rn(x1 - __bfloat162float(h1));
    }
    __nv_bfloat162 v = __halves2bfloat162(h0, h1);
    return *reinterpret_cast<uint32_t*>(&v);
  }
}

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

// ---------------------------------------------------------------------------
// tensor-pipe GEMV (bf16 / int8 weights)
// ---------------------------------------------------------------------------
template <int WT>
__global__ void __launch_bounds__(kNW * 32, 2) gemv_mma_kernel(LinearArgs a, int KS, int Rn) {
  constexpr int KTILE = (WT == kI8) ? 32 : 16;  // k per 512-byte tile
  __shared__ float red[kNW][kRT][32][4];
  __shared__ float fin[kRT][32][2];
  __shared__ float rscale[kMaxR];
  __shared__ float ramax[kNW][kMaxR];
  __shared__ int last_flag;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = blockIdx.x;
  const int64_t grp = item / KS;
  const int s = (int)(item % KS);
  const int64_t KT = a.K / KTILE;
  const int64_t kt_item = KT / KS;
  const int64_t kt_warp = kt_item / kNW;
  const int64_t k_lo = (int64_t)s * kt_item * KTILE, k_hi = k_lo + kt_item * KTILE;

  // ---- per-row power-of-two prescale over this item's k-chunk (f16 only) ----
  if (WT == kI8) {
    float m[kMaxR];
#pragma unroll
    for (int r = 0; r < kMaxR; ++r) m[r] = 0.f;
    for (int64_t k = k_lo + threadIdx.x; k < k_hi; k += blockDim.x) {
#pragma unroll
      for (int r = 0; r < kMaxR; ++r)
        if (r < Rn) m[r] = fmaxf(m[r], fabsf(__ldg(a.x + (int64_t)r * a.ldx + k)));
    }
#pragma unroll
    for (int r = 0; r < kMaxR; ++r) {
      float v = warp_max(m[r]);
      if (lane == 0) ramax[warp][r] = v;
    }
    __syncthreads();
    if (threadIdx.x < kMaxR) {
      float v = 0.f;
      for (int w = 0; w < kNW; ++w) v = fmaxf(v, ramax[w][threadIdx.x]);
      int e = 0;
      if (v > 0.f) frexpf(v, &e);          // v < 2^e
      rscale[threadIdx.x] = (v > 0.f) ? ldexpf(1.0f, 14 - e) : 1.0f;
    }
    __syncthreads();
  }

  // ---- B fragment source for this lane: column = lane/4 -> (row r, hi|lo) ----
  const int col = lane >> 2, r_b = col >> 1, part = col & 1;
  const bool bvalid = r_b < Rn;
  const float* xrow = a.x + (int64_t)(bvalid ? r_b : 0) * a.ldx;
  const float xs = (WT == kI8 && bvalid) ? rscale[r_b] : 1.0f;
  const int cb = (lane & 3) * 2;

  float acc[kRT][4];
#pragma unroll
  for (int t = 0; t < kRT; ++t)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[t][j] = 0.f;

  const int64_t kt0 = (int64_t)s * kt_item + (int64_t)warp * kt_warp;
  const uint8_t* wbase = reinterpret_cast<const uint8_t*>(a.w);
  const int64_t rt0 = grp * kRT;

  uint4 wb[kU][kRT];
#pragma unroll
  for (int u = 0; u < kU; ++u)
#pragma unroll
    for (int t = 0; t < kRT; ++t)
      wb[u][t] = (u < kt_warp)
                     ? ldg_stream(wbase + (((rt0 + t) * KT + kt0 + u) << 9) + lane * 16)
                     : make_uint4(0, 0, 0, 0);

  for (int64_t it = 0; it < kt_warp; it += kU) {
    uint4 cur[kU][kRT];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int t = 0; t < kRT; ++t) cur[u][t] = wb[u][t];
    if (it + kU < kt_warp) {
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int t = 0; t < kRT; ++t)
          wb[u][t] = (it + kU + u < kt_warp)
                         ? ldg_stream(wbase + (((rt0 + t) * KT + kt0 + it + kU + u) << 9) +
                                      lane * 16)
                         : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (it + u >= kt_warp) break;
      const int64_t kbase = (kt0 + it + u) * KTILE;
      if (WT == kI8) {
        uint32_t b[2][2];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          float2 lo = make_float2(0.f, 0.f), hi = make_float2(0.f, 0.f);
          if (bvalid) {
            lo = __ldg(reinterpret_cast<const float2*>(xrow + kbase + ks * 16 + cb));
            hi = __ldg(reinterpret_cast<const float2*>(xrow + kbase + ks * 16 + cb + 8));
          }
          b[ks][0] = pack_split<WT>(lo.x * xs, lo.y * xs, part);
          b[ks][1] = pack_split<WT>(hi.x * xs, hi.y * xs, part);
        }
#pragma unroll
        for (int t = 0; t < kRT; ++t) {
          const uint4 w = cur[u][t];
          uint32_t a0[4] = {u8x2_to_f16x2(w.x, 0x5140u), u8x2_to_f16x2(w.x, 0x7362u),
                            u8x2_to_f16x2(w.y, 0x5140u), u8x2_to_f16x2(w.y, 0x7362u)};
          uint32_t a1[4] = {u8x2_to_f16x2(w.z, 0x5140u), u8x2_to_f16x2(w.z, 0x7362u),
                            u8x2_to_f16x2(w.w, 0x5140u), u8x2_to_f16x2(w.w, 0x7362u)};
          mma_f16(acc[t], a0, b[0][0], b[0][1]);
          mma_f16(acc[t], a1, b[1][0], b[1][1]);
        }
      } else {
        float2 lo = make_float2(0.f, 0.f), hi = make_float2(0.f, 0.f);
        if (bvalid) {
          lo = __ldg(reinterpret_cast<const float2*>(xrow + kbase + cb));
          hi = __ldg(reinterpret_cast<const float2*>(xrow + kbase + cb + 8));
        }
        uint32_t b0 = pack_split<WT>(lo.x, lo.y, part);
        uint32_t b1 = pack_split<WT>(hi.x, hi.y, part);
#pragma unroll
        for (int t = 0; t < kRT; ++t) {
          const uint4 w = cur[u][t];
          uint32_t a0[4] = {w.x, w.y, w.z, w.w};
          mma_bf16(acc[t], a0, b0, b1);
        }
      }
    }
  }

  // ---- fixed-order reduction over the CTA's warps ----
#pragma unroll
  for (int t = 0; t < kRT; ++t)
    *reinterpret_cast<float4*>(red[warp][t][lane]) =
        make_float4(acc[t][0], acc[t][1], acc[t][2], acc[t][3]);
  __syncthreads();
  float v0 = 0.f, v1 = 0.f;
  const int t_rt = threadIdx.x >> 5, t_l = threadIdx.x & 31;
  const int r_out = t_l & 3;
  if (threadIdx.x < kRT * 32) {
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    for (int w = 0; w < kNW; ++w) {
      float4 p = *reinterpret_cast<float4*>(red[w][t_rt][t_l]);
      c0 += p.x; c1 += p.y; c2 += p.z; c3 += p.w;
    }
    float inv = (WT == kI8 && r_out < Rn) ? 1.0f / rscale[r_out] : 1.0f;  // power of 2: exact
    v0 = (c0 + c1) * inv;
    v1 = (c2 + c3) * inv;
  }

  // ---- split-K across CTAs: fixed-order reduction by the last arrival ----
  if (KS > 1) {
    if (threadIdx.x < kRT * 32) {
      float2* ws = reinterpret_cast<float2*>(a.workspace) + (grp * KS + s) * (kRT * 32);
      ws[threadIdx.x] = make_float2(v0, v1);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      int prev = atomicAdd(a.counters + grp, 1);
      last_flag = (prev == KS - 1);
    }
    __syncthreads();
    if (!last_flag) return;
    __threadfence();
    if (threadIdx.x < kRT * 32) {
      const volatile float2* ws =
          reinterpret_cast<const volatile float2*>(a.workspace) + grp * KS * (kRT * 32);
      float s0 = 0.f, s1 = 0.f;
      for (int j = 0; j < KS; ++j) {
        s0 += ws[j * (kRT * 32) + threadIdx.x].x;
        s1 += ws[j * (kRT * 32) + threadIdx.x].y;
      }
      v0 = s0;
      v1 = s1;
    }
    if (threadIdx.x == 0) a.counters[grp] = 0;
  }

  // ---- epilogue ----
  if (threadIdx.x < kRT * 32) {
    const int64_t na = (rt0 + t_rt) * 16 + (t_l >> 2), nb = na + 8;
    if (WT == kI8) {
      v0 *= a.wscale[na];
      v1 *= a.wscale[nb];
    }
    fin[t_rt][t_l][0] = v0;
    fin[t_rt][t_l][1] = v1;
    if (a.epi != EPI_SWIGLU && r_out < Rn) {
      epi_store(a, r_out, na, v0);
      epi_store(a, r_out, nb, v1);
    }
  }
  if (a.epi == EPI_SWIGLU) {
    __syncthreads();
    if (threadIdx.x < 32 && r_out < Rn) {
      // row tile 0 of the CTA = gate tile, row tile 1 = up tile (same 16 outputs)
      const int64_t j = grp * 16 + (t_l >> 2);
      float g0 = fin[0][t_l][0], g1 = fin[0][t_l][1];
      float u0 = fin[1][t_l][0], u1 = fin[1][t_l][1];
      a.y[(int64_t)r_out * a.ldy + j] = silu_f(g0) * u0;
      a.y[(int64_t)r_out * a.ldy + j + 8] = silu_f(g1) * u1;
    }
  }
}

// ---------------------------------------------------------------------------
// f32 weights: warp per output channel, fixed shuffle-tree reduction
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gemv_f32_kernel(LinearArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t o = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const float* W = reinterpret_cast<const float*>(a.w);
  if (a.epi == EPI_SWIGLU) {
    const int64_t F = a.N / 2;
    if (o >= F) return;
    const int64_t ng = (o >> 4) * 32 + (o & 15), nu = ng + 16;
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

int choose_ks(int64_t N, int64_t K, int wdtype) {
  const int KTILE = (wdtype == kI8) ? 32 : 16;
  const int64_t KT = K / KTILE;
  const int64_t G = N / (16 * kRT);
  int best = 1;
  for (int ks = 1; ks <= 64; ++ks) {
    if (KT % (ks * kNW)) continue;
    if (KT / (ks * kNW) < 8) break;      // keep >= 8 tiles per warp
    best = ks;
    if (G * ks >= 1000) break;
  }
  return best;
}

}  // namespace

int64_t gemv_workspace_floats(int64_t N, int64_t K, int wdtype) {
  if (wdtype == kF32) return 0;
  int ks = choose_ks(N, K, wdtype);
  return (N / (16 * kRT)) * ks * kRT * 32 * 2;
}
int64_t gemv_counter_ints(int64_t N) { return N / (16 * kRT) + 1; }

void launch_gemv(const LinearArgs& a, cudaStream_t st) {
  if (a.wdtype == kF32) {
    int64_t outs = (a.epi == EPI_SWIGLU) ? a.N / 2 : a.N;
    gemv_f32_kernel<<<(unsigned)((outs + 7) / 8), 256, 0, st>>>(a); count_launch();
    return;
  }
  const int ks = choose_ks(a.N, a.K, a.wdtype);
  const int64_t grid = (a.N / (16 * kRT)) * ks;
  for (int r0 = 0; r0 < a.R; r0 += kMaxR) {
    LinearArgs b = a;
    b.x = a.x + (int64_t)r0 * a.ldx;
    b.y = a.y + (int64_t)r0 * a.ldy;
    if (a.res) b.res = a.res + (int64_t)r0 * a.ldy;
    int rn = a.R - r0 < kMaxR ? a.R - r0 : kMaxR;
    if (a.wdtype == kI8)
      gemv_mma_kernel<kI8><<<(unsigned)grid, kNW * 32, 0, st>>>(b, ks, rn);
    else
      gemv_mma_kernel<kBF16><<<(unsigned)grid, kNW * 32, 0, st>>>(b, ks, rn);
    count_launch();
  }
}

}  // namespace sp
