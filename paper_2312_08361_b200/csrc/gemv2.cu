// Decode linear layers on the tensor pipe, with the block's pre-norm folded in.
//
//   y[r, n] = epi( rstd_r * sum_k W[n, k] * ((x[r, k] - mu_r) * g[k]) )
//
// int8 weights (70B / BLOOM shapes): EXACT integer arithmetic.
//   * the input row is scaled by a power of two 2^(22-e_r) (e_r from the
//     row's max, produced by the previous kernel) and rounded to a 23-bit
//     integer q, written as three balanced base-256 digits (q + 0x808080 ->
//     bytes, minus 128): q = d0*2^16 + d1*2^8 + d2, each digit int8;
//   * the three digits of each batch row are three columns of one
//     mma.m16n8k32.s8.s8.s32 — the 16-byte weight load of each lane IS its A
//     fragment (fragment-tiled storage), no conversion of weights at all;
//   * per-digit int32 sums are exact; digits combine in int64, split-K
//     partials are int64 atomics (exact -> order-independent, deterministic);
//   * one rounding at the end: y = f32(D * 2^(e-22) * rstd * wscale[n]).
//   So the only error vs. exact arithmetic is the 23-bit rounding of the input.
// bf16 weights (7B shape): A = bf16 tiles straight from HBM, the input is split
//   hi + lo (both bf16, two MMA columns per row), f32 accumulation, fixed-order
//   split-K reduction.
// The norm (RMSNorm / LayerNorm) needs only per-row (sum, sumsq, max) which the
// producer of x wrote as fixed-slot partials; they are reduced here in a fixed
// order — no separate norm kernel, still deterministic and batch-invariant.
// Each output CTA writes the same partial stats for the next consumer.
#include <type_traits>

#include "common.cuh"
#include "decode.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int NW = 8;       // warps per CTA (split K inside the CTA)
constexpr int RT = 4;       // 16-row tiles per CTA (64 output channels)
constexpr int U = 2;        // k-tiles per prefetch batch
constexpr int RMAX = 8;     // batch rows per launch (more rows -> more launches)
constexpr int STAGES = 3;   // TMA ring depth per warp
constexpr int STAGE_BYTES = RT * U * 512;
constexpr size_t RING_BYTES = (size_t)NW * STAGES * STAGE_BYTES;

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D TMA (bulk async copy) global -> shared, completion counted on `bar`,
// L2 evict-first: weights are streamed exactly once per step
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void mma_s8(int* c, const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_bf16(float* c, const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + expf(-x)); }

struct RowParams {
  float mu[RMAX];
  float dscale[RMAX];   // int8: 2^(22-e)   (digit scale)
  double yscale[RMAX];  // int8: 2^(e-22)*rstd ; bf16: rstd
};

// reduce the P_in partial stats of every row in a fixed order -> per-row params
template <bool INT8>
__device__ void row_params(const GemvArgs& a, int r0, int Rn, int Rs, RowParams& rp,
                           float* scratch /* [NW][RMAX][3] */) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float s[RMAX], q[RMAX], m[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) { s[r] = 0.f; q[r] = 0.f; m[r] = 0.f; }
  for (int p = threadIdx.x; p < a.P_in; p += blockDim.x) {
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r < Rn) {
        RowStat t = a.st_in[(int64_t)p * Rs + r0 + r];
        s[r] += t.sum; q[r] += t.sumsq; m[r] = fmaxf(m[r], t.amax);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    float vs = warp_sum(s[r]), vq = warp_sum(q[r]), vm = warp_max(m[r]);
    if (lane == 0) {
      scratch[(warp * RMAX + r) * 3 + 0] = vs;
      scratch[(warp * RMAX + r) * 3 + 1] = vq;
      scratch[(warp * RMAX + r) * 3 + 2] = vm;
    }
  }
  __syncthreads();
  if (threadIdx.x < Rn) {
    const int r = threadIdx.x;
    float S = 0.f, Q = 0.f, M = 0.f;
    for (int w = 0; w < NW; ++w) {
      S += scratch[(w * RMAX + r) * 3 + 0];
      Q += scratch[(w * RMAX + r) * 3 + 1];
      M = fmaxf(M, scratch[(w * RMAX + r) * 3 + 2]);
    }
    const float invK = 1.0f / (float)a.K;
    float mu = 0.f, rstd = 1.f, bound = M;
    if (a.norm == NORM_RMS) {
      rstd = 1.0f / sqrtf(Q * invK + a.eps);
    } else if (a.norm == NORM_LN) {
      mu = S * invK;
      float var = fmaxf(Q * invK - mu * mu, 0.f);
      rstd = 1.0f / sqrtf(var + a.eps);
      bound = M + fabsf(mu) * a.gmax;
    }
    rp.mu[r] = mu;
    if (INT8) {
      int e = 0;
      if (bound > 0.f) frexpf(bound, &e);          // bound < 2^e
      rp.dscale[r] = bound > 0.f ? ldexpf(1.0f, 22 - e) : 0.f;
      rp.yscale[r] = ldexp(1.0, e - 22) * (double)rstd;
    } else {
      rp.dscale[r] = 1.0f;
      rp.yscale[r] = (double)rstd;
    }
  }
  __syncthreads();
}

// balanced base-256 digit `dg` (0 = most significant) of 4 integers, packed
__device__ __forceinline__ uint32_t digits4(int q0, int q1, int q2, int q3, int sh) {
  uint32_t u0 = (uint32_t)(q0 + 0x808080) >> sh, u1 = (uint32_t)(q1 + 0x808080) >> sh;
  uint32_t u2 = (uint32_t)(q2 + 0x808080) >> sh, u3 = (uint32_t)(q3 + 0x808080) >> sh;
  uint32_t lo = __byte_perm(u0, u1, 0x0040), hi = __byte_perm(u2, u3, 0x0040);
  return __byte_perm(lo, hi, 0x5410) ^ 0x80808080u;
}

__device__ __forceinline__ float4 xform4(const float4 x, const float4 g, float mu, float sc) {
  return make_float4((x.x - mu) * g.x * sc, (x.y - mu) * g.y * sc, (x.z - mu) * g.z * sc,
                     (x.w - mu) * g.w * sc);
}

template <int WT, int NT>
__global__ void __launch_bounds__(NW * 32, NT == 1 ? 2 : 1)
gemv2_kernel(GemvArgs a, int KS, int r0, int Rn, int Rs) {
  constexpr int KTILE = (WT == kI8) ? 32 : 16;
  constexpr int COLS_PER_ROW = (WT == kI8) ? 3 : 2;
  __shared__ RowParams rp;
  __shared__ float scratch[NW * RMAX * 3];
  extern __shared__ int4 dyn_smem[];
  int (*red)[RT][NT][32][4] = reinterpret_cast<int (*)[RT][NT][32][4]>(dyn_smem);
  __shared__ float outv[RT * 16][RMAX];
  __shared__ int last_flag;
  __shared__ __align__(8) uint64_t bars[NW][STAGES];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    for (int st = 0; st < STAGES; ++st) mbar_init(&bars[warp][st], 1);
    mbar_fence_init();
  }
  __syncwarp();
  const int64_t grp = blockIdx.x / KS;
  const int s = blockIdx.x % KS;
  const int64_t KT = a.K / KTILE;
  const int64_t kt_item = KT / KS;
  const int64_t kt_warp = kt_item / NW;
  const int64_t kt0 = s * kt_item + warp * kt_warp;
  const int64_t rt0 = grp * RT;

  row_params<WT == kI8>(a, r0, Rn, Rs, rp, scratch);

  // ---- this lane's B column: nt*8 + lane/4 -> (row, digit | hi/lo) ----
  int brow[NT], bsub[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    int c = nt * 8 + (lane >> 2);
    brow[nt] = c / COLS_PER_ROW;
    bsub[nt] = c % COLS_PER_ROW;
  }
  const int t4 = lane & 3;
  const bool has_g = a.norm != NORM_NONE;

  // ---- accumulators ----
  int iacc[RT][NT][4];
  float facc[RT][NT][4];
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) { iacc[t][nt][j] = 0; facc[t][nt][j] = 0.f; }

  // ---- weight stream: per-warp ring of STAGES x (RT tiles x U k-tiles), TMA ----
  const uint8_t* wbase = reinterpret_cast<const uint8_t*>(a.w);
  uint8_t* ring = reinterpret_cast<uint8_t*>(dyn_smem) + warp * STAGES * STAGE_BYTES;
  uint64_t* bar = bars[warp];
  const int64_t n_it = (kt_warp + U - 1) / U;
  const uint64_t policy = evict_first_policy();
  auto issue = [&](int64_t it) {
    const int st = (int)(it % STAGES);
    const int64_t kt = kt0 + it * U;
    const int nk = (int)min((int64_t)U, kt_warp - it * U);
    mbar_expect_tx(&bar[st], (uint32_t)(RT * nk * 512));
#pragma unroll
    for (int t = 0; t < RT; ++t)
      tma_load_1d(ring + st * STAGE_BYTES + t * U * 512, wbase + (((rt0 + t) * KT + kt) << 9),
                  (uint32_t)(nk * 512), &bar[st], policy);
  };
  if (lane == 0)
    for (int64_t it = 0; it < STAGES && it < n_it; ++it) issue(it);

  // the activation side of the B fragments is software-pipelined one
  // iteration ahead (its L1/L2 latency was the dominant stall)
  constexpr int XV = (WT == kI8) ? 4 : 2;          // floats per half-fragment
  using XVec = typename std::conditional<WT == kI8, float4, float2>::type;
  XVec xc[U][NT][2], gc[U][NT][2], xn[U][NT][2], gn[U][NT][2];
  auto load_x = [&](int64_t it, XVec (&xr_)[U][NT][2], XVec (&gr_)[U][NT][2]) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int r = brow[nt];
        const int64_t kt = kt0 + it * U + u;
        const bool ok = (r < Rn) && (it * U + u < kt_warp);
        const int64_t k0 = kt * KTILE + t4 * XV;
        const int64_t koff = (WT == kI8) ? 16 : 8;
        if (ok) {
          const float* xr = a.x + (int64_t)(r0 + r) * a.ldx;
          xr_[u][nt][0] = __ldg(reinterpret_cast<const XVec*>(xr + k0));
          xr_[u][nt][1] = __ldg(reinterpret_cast<const XVec*>(xr + k0 + koff));
          if (has_g) {
            gr_[u][nt][0] = __ldg(reinterpret_cast<const XVec*>(a.g + k0));
            gr_[u][nt][1] = __ldg(reinterpret_cast<const XVec*>(a.g + k0 + koff));
          }
        }
      }
  };
  if (n_it > 0) load_x(0, xc, gc);

  for (int64_t it = 0; it < n_it; ++it) {
    const int st = (int)(it % STAGES);
    if (it + 1 < n_it) load_x(it + 1, xn, gn);
    mbar_wait(&bar[st], (uint32_t)((it / STAGES) & 1));
    const int nk = (int)min((int64_t)U, kt_warp - it * U);
    const uint8_t* stage = ring + st * STAGE_BYTES;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u >= nk) break;
      uint4 wt[RT];
#pragma unroll
      for (int t = 0; t < RT; ++t)
        wt[t] = *reinterpret_cast<const uint4*>(stage + (t * U + u) * 512 + lane * 16);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        uint32_t b0 = 0, b1 = 0;
        const int r = brow[nt];
        if (r < Rn) {
          const float mu = rp.mu[r], sc = rp.dscale[r];
          if constexpr (WT == kI8) {
            const float4 one = make_float4(1.f, 1.f, 1.f, 1.f);
            float4 va = xform4(xc[u][nt][0], has_g ? gc[u][nt][0] : one, mu, sc);
            float4 vb = xform4(xc[u][nt][1], has_g ? gc[u][nt][1] : one, mu, sc);
            const int sh = 8 * (2 - bsub[nt]);
            b0 = digits4(__float2int_rn(va.x), __float2int_rn(va.y), __float2int_rn(va.z),
                         __float2int_rn(va.w), sh);
            b1 = digits4(__float2int_rn(vb.x), __float2int_rn(vb.y), __float2int_rn(vb.z),
                         __float2int_rn(vb.w), sh);
          } else {
            const float2 one = make_float2(1.f, 1.f);
            const float2 xa = xc[u][nt][0], xb = xc[u][nt][1];
            const float2 ga = has_g ? gc[u][nt][0] : one, gb = has_g ? gc[u][nt][1] : one;
            float v[4] = {(xa.x - mu) * ga.x, (xa.y - mu) * ga.y, (xb.x - mu) * gb.x,
                          (xb.y - mu) * gb.y};
            __nv_bfloat16 h[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              h[j] = __float2bfloat16_rn(v[j]);
              if (bsub[nt]) h[j] = __float2bfloat16_rn(v[j] - __bfloat162float(h[j]));
            }
            __nv_bfloat162 p0 = __halves2bfloat162(h[0], h[1]), p1 = __halves2bfloat162(h[2], h[3]);
            b0 = *reinterpret_cast<uint32_t*>(&p0);
            b1 = *reinterpret_cast<uint32_t*>(&p1);
          }
        }
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          if constexpr (WT == kI8) mma_s8(iacc[t][nt], wt[t], b0, b1);
          else mma_bf16(facc[t][nt], wt[t], b0, b1);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          xc[u][nt][h] = xn[u][nt][h];
          gc[u][nt][h] = gn[u][nt][h];
        }
    __syncwarp();
    if (lane == 0 && it + STAGES < n_it) issue(it + STAGES);
  }
  __syncthreads();   // every warp's ring is drained: the ring memory becomes `red`

  // ---- cross-warp reduction (fixed order) -> per (row, batch) value ----
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      if (WT == kI8)
        *reinterpret_cast<int4*>(red[warp][t][nt][lane]) =
            make_int4(iacc[t][nt][0], iacc[t][nt][1], iacc[t][nt][2], iacc[t][nt][3]);
      else
        *reinterpret_cast<float4*>(red[warp][t][nt][lane]) =
            make_float4(facc[t][nt][0], facc[t][nt][1], facc[t][nt][2], facc[t][nt][3]);
    }
  __syncthreads();
  // collapse warps: element e = ((t*NT + nt)*32 + l)*4 + j
  __shared__ __align__(16) int ctile[RT * 16][NT * 8];
  for (int e = threadIdx.x; e < RT * NT * 32 * 4; e += blockDim.x) {
    const int j = e & 3, l = (e >> 2) & 31, tn = e >> 7;
    const int t = tn / NT, nt = tn % NT;
    int isum = 0;
    float fsum = 0.f;
    for (int w = 0; w < NW; ++w) {
      int v = red[w][t][nt][l][j];
      if (WT == kI8) isum += v;
      else fsum += __int_as_float(v);
    }
    const int row = t * 16 + (l >> 2) + ((j >> 1) << 3);
    const int col = nt * 8 + (l & 3) * 2 + (j & 1);
    ctile[row][col] = (WT == kI8) ? isum : __float_as_int(fsum);
  }
  __syncthreads();

  // each thread owns NPAIR (output channel i, batch row r) pairs
  constexpr int NPAIR = (RT * 16 * RMAX) / (NW * 32);
  int pi[NPAIR], pr[NPAIR];
  bool mine[NPAIR];
  long long D[NPAIR];
  float F[NPAIR], v[NPAIR];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    const int e = threadIdx.x + q * NW * 32;
    pi[q] = e / RMAX;
    pr[q] = e % RMAX;
    mine[q] = pr[q] < Rn;
    D[q] = 0;
    F[q] = 0.f;
    if (mine[q]) {
      const int i = pi[q], r = pr[q];
      if (WT == kI8)
        D[q] = (long long)ctile[i][3 * r] * 65536 + (long long)ctile[i][3 * r + 1] * 256 +
               (long long)ctile[i][3 * r + 2];
      else
        F[q] = __int_as_float(ctile[i][2 * r]) + __int_as_float(ctile[i][2 * r + 1]);
    }
  }

  if (KS > 1) {
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) {
      if (!mine[q]) continue;
      const int64_t n = rt0 * 16 + pi[q];
      if (WT == kI8)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.ws) + (int64_t)(r0 + pr[q]) * a.N + n,
                  (unsigned long long)D[q]);
      else
        reinterpret_cast<float*>(a.ws)[((int64_t)s * Rs + r0 + pr[q]) * a.N + n] = F[q];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last_flag = (atomicAdd(a.counters + grp, 1) == KS - 1);
    __syncthreads();
    if (!last_flag) return;
    __threadfence();
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) {
      if (!mine[q]) continue;
      const int64_t n = rt0 * 16 + pi[q];
      if (WT == kI8) {
        D[q] = (long long)atomicExch(
            reinterpret_cast<unsigned long long*>(a.ws) + (int64_t)(r0 + pr[q]) * a.N + n, 0ull);
      } else {
        float acc = 0.f;
        const volatile float* ws = reinterpret_cast<const volatile float*>(a.ws);
        for (int j = 0; j < KS; ++j) acc += ws[((int64_t)j * Rs + r0 + pr[q]) * a.N + n];
        F[q] = acc;
      }
    }
    if (threadIdx.x == 0) a.counters[grp] = 0;
  }

#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    v[q] = 0.f;
    if (mine[q]) {
      const int64_t n = rt0 * 16 + pi[q];
      if (WT == kI8) v[q] = (float)((double)D[q] * rp.yscale[pr[q]] * (double)a.wscale[n]);
      else v[q] = (float)((double)F[q] * rp.yscale[pr[q]]);
    }
  }

  // ---- epilogue: outputs + this group's partial stats for the next consumer ----
  __shared__ float gsc[RT * 16][RMAX];
  if (a.epi == EPI_SWIGLU) {
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) outv[pi[q]][pr[q]] = v[q];
    __syncthreads();
  }
  float oval[NPAIR];
  int64_t ocol[NPAIR];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    const int i = pi[q], r = pr[q];
    const int64_t n = rt0 * 16 + i;
    ocol[q] = -1;
    oval[q] = 0.f;
    if (!mine[q]) continue;
    if (a.epi == EPI_SWIGLU) {
      // tiles (0,1) = (gate, up) of outputs [0,16); tiles (2,3) of outputs [16,32)
      if (i < 32) {
        const int pair = i >> 4, jj = i & 15;
        oval[q] = silu_f(outv[pair * 32 + jj][r]) * outv[pair * 32 + 16 + jj][r];
        ocol[q] = grp * 32 + i;
      }
    } else {
      ocol[q] = n;
      oval[q] = v[q];
      if (a.epi == EPI_RESID) oval[q] = a.res[(int64_t)(r0 + r) * a.ldy + n] + v[q];
      else if (a.epi == EPI_GELU) oval[q] = gelu_f(v[q]);
    }
    if (ocol[q] >= 0) a.y[(int64_t)(r0 + r) * a.ldy + ocol[q]] = oval[q];
  }
  if (a.st_out) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) {
      const bool ok = ocol[q] >= 0;
      outv[pi[q]][pr[q]] = ok ? oval[q] : 0.f;
      gsc[pi[q]][pr[q]] = ok ? fabsf(oval[q] * (a.g_next ? a.g_next[ocol[q]] : 1.f)) : 0.f;
    }
    __syncthreads();
    if (threadIdx.x < Rn) {
      const int rr = threadIdx.x;
      float S = 0.f, Q = 0.f, M = 0.f;
      for (int ii = 0; ii < RT * 16; ++ii) {
        const float o = outv[ii][rr];
        S += o;
        Q = fmaf(o, o, Q);
        M = fmaxf(M, gsc[ii][rr]);
      }
      a.st_out[grp * Rs + r0 + rr] = RowStat{S, Q, M, 0.f};
    }
  }
}

int choose_ks2(int64_t N, int64_t K, int wdtype) {
  const int KTILE = (wdtype == kI8) ? 32 : 16;
  const int64_t KT = K / KTILE;
  const int64_t G = N / (16 * RT);
  int best = 1;
  for (int ks = 1; ks <= 64; ++ks) {
    if (KT % (ks * NW)) continue;
    if (KT / (ks * NW) < 2 * U) break;
    best = ks;
    if (G * ks >= 296) break;
  }
  return best;
}

template <int WT>
void launch_wt(const GemvArgs& a, int ks, int r0, int rn, int Rs, cudaStream_t st) {
  const unsigned grid = (unsigned)((a.N / (16 * RT)) * ks);
  const int cols = rn * ((WT == kI8) ? 3 : 2);
  const int nt = cols <= 8 ? 1 : (cols <= 16 ? 2 : 3);
  const size_t red_bytes = (size_t)NW * RT * nt * 32 * 16;
  const size_t smem = red_bytes > RING_BYTES ? red_bytes : RING_BYTES;
  static bool attr_set_all[kMaxDevices][3] = {};
  bool* attr_set = attr_set_all[current_device()];
  if (nt == 1) {
    if (!attr_set[0]) {
      cudaFuncSetAttribute(gemv2_kernel<WT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set[0] = true;
    }
    gemv2_kernel<WT, 1><<<grid, NW * 32, smem, st>>>(a, ks, r0, rn, Rs);
  } else if (nt == 2) {
    if (!attr_set[1]) {
      cudaFuncSetAttribute(gemv2_kernel<WT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set[1] = true;
    }
    gemv2_kernel<WT, 2><<<grid, NW * 32, smem, st>>>(a, ks, r0, rn, Rs);
  } else {
    if (!attr_set[2]) {
      cudaFuncSetAttribute(gemv2_kernel<WT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_set[2] = true;
    }
    gemv2_kernel<WT, 3><<<grid, NW * 32, smem, st>>>(a, ks, r0, rn, Rs);
  }
  count_launch();
}

// ---- span-input statistics: P = d/128 partials (the layout GEMV outputs use) ----
__global__ void row_stats_kernel(const float* x, int64_t d, const float* g, RowStat* st, int Rs) {
  const int p = blockIdx.x, r = blockIdx.y;
  const int t = threadIdx.x;   // 128 threads: one element each
  __shared__ float vs[128], vg[128];
  const int64_t k = (int64_t)p * 128 + t;
  float v = x[(int64_t)r * d + k];
  vs[t] = v;
  vg[t] = fabsf(v * (g ? g[k] : 1.f));
  __syncthreads();
  if (t == 0) {
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

int gemv2_groups(int64_t N) { return (int)(N / (16 * RT)); }
int64_t gemv2_counters(int64_t N) { return N / (16 * RT) + 1; }

int64_t gemv2_ws_bytes(int wdtype, int64_t N, int64_t K, int Rmax) {
  if (wdtype == kI8) return (int64_t)Rmax * N * 8;
  return (int64_t)choose_ks2(N, K, wdtype) * Rmax * N * 4;
}

void launch_gemv2(int wdtype, const GemvArgs& a, cudaStream_t st) {
  const int ks = choose_ks2(a.N, a.K, wdtype);
  for (int r0 = 0; r0 < a.R; r0 += RMAX) {
    const int rn = a.R - r0 < RMAX ? a.R - r0 : RMAX;
    if (wdtype == kI8) launch_wt<kI8>(a, ks, r0, rn, a.R, st);
    else launch_wt<kBF16>(a, ks, r0, rn, a.R, st);
  }
}

void launch_row_stats(const float* x, int R, int64_t d, const float* g_next, RowStat* st_out,
                      cudaStream_t st) {
  dim3 grid((unsigned)(d / 128), (unsigned)R);
  row_stats_kernel<<<grid, 128, 0, st>>>(x, d, g_next, st_out, R);
  count_launch();
}

}  // namespace sp
