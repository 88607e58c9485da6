// Decode linear layers (n_new == 1) — persistent stream-K tensor-pipe GEMV.
//
//   y[r, n] = epi( rstd_r * sum_k W[n, k] * ((x[r, k] - mu_r) * g[k]) )
//
// Work split.  The weight matrix is a sequence of "units" = (group of 64 output
// channels, one k-tile); every warp of a persistent grid (2 CTAs x 8 warps per
// SM) owns an equal contiguous slice of units — identical byte counts per
// warp, no waves, no tail.  Each warp streams its slice through a private
// STAGES-deep ring of 1-D TMA bulk copies (cp.async.bulk + mbarrier, L2
// evict-first) and never synchronises with other warps.
//
// Arithmetic (int8 weights, 70B/BLOOM): exact for the coded input.  The input
// row is scaled by a power of two 2^(kQBits-e_r) and rounded to an integer
// q written as ND balanced base-256 digits (15-bit / 2 digits for every row
// count: width-independent numerics); the digits of each
// batch row are columns of mma.m16n8k32.s8.s8.s32 whose A fragment is the lane's
// 16-byte weight load (fragment-tiled storage, no conversion).  Digit sums are
// exact int32, combined in int64; partial sums of a group's k-range are int64
// atomics (exact => order-independent => deterministic and batch-invariant).
// One rounding at the end: y = f32(D * 2^(e-kQBits) * rstd * wscale[n]).
// bf16 weights (7B): A = bf16 tiles, input split hi+lo (two bf16 MMA columns),
// f32 accumulation; partials fixed-point (2^-32) int64 atomics => deterministic.
//
// The pre-norm (RMSNorm / LayerNorm) is folded in: the producer of x wrote
// per-row (sum, sumsq, max|x g|) partials, reduced here in a fixed order; mu
// and g are applied while building the B fragments, rstd in the epilogue.
// The last warp to finish a group writes the group's outputs (+ residual /
// SwiGLU / GELU epilogue) and the same partial stats for the next consumer.
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "decode.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int NW = 8;             // warps per CTA
constexpr int CTAS_PER_SM = 2;
constexpr int RT = 8;             // 16-row tiles per group (128 output channels)
constexpr int UNIT_BYTES = 4096;  // one unit = 128 rows x 32 bytes of K (common.cuh cm_offset)
constexpr int XSLOT = 128;        // per batch row: the unit's activation chunk (<= 32 f32)
// stage = weights + the activation chunks of the rows one launch handles
// (NT MMA column tiles hold 8*NT/3 int8 digit rows / 8*NT/2 bf16 hi-lo rows)
__host__ __device__ constexpr int stage_bytes(int nt) {
  return UNIT_BYTES + (nt == 1 ? 4 : (nt == 2 ? 8 : 8)) * XSLOT;
}
// nf4: 4 KB of codes (128 channels x 64 k), the unit's 128 uint8 block scales,
// and each batch row's 64-float activation chunk (1 row, or up to 4 rows: the
// 8 columns of one MMA tile at 2 digits per row)
constexpr int NF4_QS = 128, NF4_X = 256;
__host__ __device__ constexpr int stage_bytes_wt(int wt, int nt, int rm = 1) {
  return wt == kNF4 ? UNIT_BYTES + NF4_QS + (rm == 1 ? 1 : 4) * NF4_X : stage_bytes(nt);
}
constexpr int STAGES = 3;         // TMA ring depth per warp (units)
// multi-row nf4 stages are 5.1 KB: two of them per warp keep two CTAs per SM
__host__ __device__ constexpr int stages_of(int wt, int rm) {
  return (wt == kNF4 && rm != 1) ? 2 : STAGES;
}
constexpr int RMAX = 8;           // batch rows per launch
// int8 path: activation code width.  The row is scaled by 2^(kQBits - e)
// (|x| < 2^e) and rounded to an integer |q| <= 2^kQBits written as NDIG
// balanced int8 digits (MMA columns); 2 digits = 15-bit codes, the precision
// class of the prefill digit planes, and 4 batch rows per 8-column MMA tile.
constexpr int kNDig = 2;   // digits of the int8 path (see launch_gemv3)
constexpr double kFix = 4294967296.0;   // bf16 partial fixed point 2^32

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

__device__ __forceinline__ void ldsm_x4(uint4& r, const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
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

// digit of 4 integers: byte `sel` of (q + bias), packed; balanced digits:
// 2 digits: d1 = byte0(q), d0 = byte1(q + 0x80)  (|q| <= 2^14); 3 digits add byte2(q + 0x8080)
__device__ __forceinline__ uint32_t digits4(int q0, int q1, int q2, int q3, int bias,
                                            uint32_t sel_lo, uint32_t sel_hi) {
  const uint32_t u0 = q0 + bias, u1 = q1 + bias, u2 = q2 + bias, u3 = q3 + bias;
  const uint32_t lo = __byte_perm(u0, u1, sel_lo);    // bytes: u0.b, u1.b
  const uint32_t hi = __byte_perm(u2, u3, sel_lo);
  return __byte_perm(lo, hi, sel_hi);
}

// debug trace: per warp [start, after pdl_wait, after prologue, first stage, mainloop end, exit]
__device__ __forceinline__ void gtrace(const GemvArgs& a, int ph) {
  if (SP_DEV_TRACE && a.trace && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    a.trace[((int64_t)blockIdx.x * NW + (threadIdx.x >> 5)) * 8 + ph] = t;
    if (ph == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      a.trace[((int64_t)blockIdx.x * NW + (threadIdx.x >> 5)) * 8 + 6] = smid;
    }
  }
}

struct WarpSmem {
  float mu[RMAX], dscale[RMAX];
  double yscale[RMAX];
  uint64_t bar[STAGES];
};

template <int WT, int NT, int NORMT, bool HASG, int ND, int RM, int EP>
__global__ void __launch_bounds__(NW * 32, CTAS_PER_SM)
gemv3_kernel(GemvArgs a, int r0, int Rn, int Rs, int64_t units, int64_t warps_total) {
  constexpr int NDIG = ND;
  constexpr int kQBits = 8 * ND - 2;
  constexpr bool INT = (WT == kI8 || WT == kNF4);   // exact integer digit path
  constexpr int KTILE = (WT == kI8) ? 32 : (WT == kNF4 ? 64 : 16);
  constexpr int COLS = INT ? NDIG : 2;
  constexpr int XV = INT ? 4 : 2;
  using XVec = typename std::conditional<INT, float4, float2>::type;
  static_assert(WT != kNF4 || NT == 1, "nf4: one MMA column tile (up to 4 rows)");
  constexpr int XOFF = UNIT_BYTES + (WT == kNF4 ? NF4_QS : 0);   // activation chunks in a stage
  constexpr int XS = WT == kNF4 ? NF4_X : XSLOT;                 // bytes per row's chunk
  constexpr int ST = stages_of(WT, RM);                          // ring depth
  extern __shared__ __align__(128) uint8_t dyn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int STAGE_BYTES = stage_bytes_wt(WT, NT, RM);
  uint8_t* ring = dyn + (size_t)warp * ST * STAGE_BYTES;
  WarpSmem* ws_ = reinterpret_cast<WarpSmem*>(dyn + (size_t)NW * ST * STAGE_BYTES) + warp;

  const int64_t gw = (int64_t)blockIdx.x * NW + warp;
  // unit indices fit 32 bits (units = N/128 * K/KTILE < 2^31); the slice
  // bounds floor(gw * units / W) use one double division with an exact
  // integer fix-up instead of two 64-bit divisions (code size: see DESIGN)
  const int W32 = (int)warps_total, U32 = (int)units;
  auto slice_bound = [&](int w) {
    const long long num = (long long)w * U32;
    int q = (int)((double)num / (double)W32);
    if ((long long)q * W32 > num) --q;
    else if ((long long)(q + 1) * W32 <= num) ++q;
    return q;
  };
  const int u0 = slice_bound((int)gw), u1 = slice_bound((int)gw + 1);
  const int KT = (int)(a.K / KTILE);

  gtrace(a, 0);
  if (lane == 0) {
    for (int st = 0; st < ST; ++st) mbar_init(&ws_->bar[st], 1);
    mbar_fence_init();
  }
  __syncwarp();
  constexpr int XB = KTILE * 4;
  const uint8_t* wbase = reinterpret_cast<const uint8_t*>(a.w);
  const uint8_t* qsbase = wbase + (WT == kNF4 ? a.N * a.K / 2 : 0);   // nf4 block scales
  const uint64_t policy = evict_first_policy();
  uint64_t policy_x;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(policy_x));
  const int nunits = u1 > u0 ? (int)(u1 - u0) : 0;
  const int npre = nunits < ST ? nunits : ST;   // the whole ring before the wait
  // ---- before the dependency: the weights of the first STAGES units (no
  // kernel writes weights), so their DRAM latency overlaps the previous
  // kernel's tail; each stage's barrier also expects its activation bytes ----
  if (lane == 0)
    for (int i = 0; i < npre; ++i) {
      const int64_t u = (int64_t)u0 + i;
      mbar_expect_tx(&ws_->bar[i], XOFF + Rn * XB);
      tma_load_1d(ring + i * STAGE_BYTES, wbase + u * UNIT_BYTES,
                  UNIT_BYTES, &ws_->bar[i], policy);
      if constexpr (WT == kNF4)
        tma_load_1d(ring + i * STAGE_BYTES + UNIT_BYTES, qsbase + u * NF4_QS, NF4_QS,
                    &ws_->bar[i], policy);
    }
  pdl_trigger();
  pdl_wait();
  gtrace(a, 1);
  // ---- per-row parameters from the producer's partial stats ----
  // CTA-wide: 256 threads load the P_in x Rn partials with several loads in
  // flight each, then a fixed-order tree (warp shuffles, then warps in order)
  __shared__ float red_s[NW][RM][3];
  __shared__ uint32_t nf4_lut[2];
  if (WT == kNF4 && threadIdx.x == 0) { nf4_lut[0] = kLA0; nf4_lut[1] = kLB0; }
  __shared__ float prm_mu[RM], prm_ds[RM];
  __shared__ double prm_ys[RM];
  {
    float S[RM], Q[RM], M[RM];
#pragma unroll
    for (int r = 0; r < RM; ++r) { S[r] = 0.f; Q[r] = 0.f; M[r] = 0.f; }
    constexpr int PU = RM == 1 ? 2 : 4;   // P_in <= 2 * 256 for one row
    for (int p0 = threadIdx.x; p0 < a.P_in; p0 += PU * NW * 32) {
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        if (r >= Rn) break;
        RowStat t[PU];
#pragma unroll
        for (int j = 0; j < PU; ++j) {
          const int p = p0 + j * NW * 32;
          t[j] = p < a.P_in ? a.st_in[(int64_t)p * Rs + r0 + r] : RowStat{0.f, 0.f, 0.f, 0.f};
        }
#pragma unroll
        for (int j = 0; j < PU; ++j) {
          S[r] += t[j].sum; Q[r] += t[j].sumsq; M[r] = fmaxf(M[r], t[j].amax);
        }
      }
    }
  if (lane == 0)
    for (int i = 0, kt0 = u0 % KT; i < npre; ++i) {   // x chunks of the prefetched units
      // (issued right behind the stats loads, ahead of their reduction)
      const int64_t kt = kt0 + i < KT ? kt0 + i : kt0 + i - KT;
      for (int r = 0; r < (RM == 1 ? 1 : Rn); ++r)
        tma_load_1d(ring + i * STAGE_BYTES + XOFF + r * XS,
                    a.x + (int64_t)(r0 + r) * a.ldx + kt * KTILE, XB, &ws_->bar[i], policy_x);
    }
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const float vs = warp_sum(S[r]), vq = warp_sum(Q[r]), vm = warp_max(M[r]);
      if (lane == 0) { red_s[warp][r][0] = vs; red_s[warp][r][1] = vq; red_s[warp][r][2] = vm; }
    }
    __syncthreads();
    if (threadIdx.x < Rn) {
      const int r = threadIdx.x;
      float s = 0.f, q = 0.f, m = 0.f;
      for (int w = 0; w < NW; ++w) {
        s += red_s[w][r][0]; q += red_s[w][r][1]; m = fmaxf(m, red_s[w][r][2]);
      }
      const float invK = 1.0f / (float)a.K;
      float mu = 0.f, rstd = 1.f, bound = m;
      if (NORMT == NORM_RMS) {
        rstd = 1.0f / sqrtf(q * invK + a.eps);
      } else if (NORMT == NORM_LN) {
        mu = s * invK;
        rstd = 1.0f / sqrtf(fmaxf(q * invK - mu * mu, 0.f) + a.eps);
        bound = m + fabsf(mu) * a.gmax;
      }
      prm_mu[r] = mu;
      if (INT) {
        int e = 0;
        if (bound > 0.f) frexpf(bound, &e);          // bound < 2^e
        prm_ds[r] = bound > 0.f ? ldexpf(1.0f, kQBits - e) : 0.f;
        prm_ys[r] = ldexp(1.0, e - kQBits) * (double)rstd;
      } else {
        prm_ds[r] = 1.0f;
        prm_ys[r] = (double)rstd / kFix;
      }
    }
    __syncthreads();
  }
  gtrace(a, 2);
  if (u0 >= u1) return;
  if (lane < RM) {
    ws_->mu[lane] = prm_mu[lane];
    ws_->dscale[lane] = prm_ds[lane];
    ws_->yscale[lane] = prm_ys[lane];
  }
  __syncwarp();

  // ---- this lane's B column: nt*8 + lane/4 -> (batch row, digit | hi/lo) ----
  int brow[NT], bsub[NT];
  float bmu[NT], bsc[NT];
  int bbias[NT];
  uint32_t bsel_lo[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = nt * 8 + (lane >> 2);
    brow[nt] = c / COLS;
    bsub[nt] = c % COLS;
    if (brow[nt] >= Rn) brow[nt] = 0;   // unused column: computed, never read
    bmu[nt] = ws_->mu[brow[nt]];
    bsc[nt] = ws_->dscale[brow[nt]];
    // digit dg: byte (NDIG-1-dg) of q + bias_dg, bias_dg = 0x80 in every byte below it
    bbias[nt] = 0;
    for (int j = 0; j < NDIG - 1 - bsub[nt]; ++j) bbias[nt] |= 0x80 << (8 * j);
    const uint32_t b = NDIG - 1 - bsub[nt];
    bsel_lo[nt] = b | ((b + 4) << 4);
  }
  const int t4 = lane & 3;

  // ---- TMA producer (lane 0) ----
  // producer state (lane 0): next unit to issue as (group, k-tile, ring stage)
  int p_grp = (u0 + npre) / KT, p_kt = (u0 + npre) % KT;
  int p_st = npre % ST, p_left = nunits - npre;
  auto issue_next = [&]() {
    // the unit's weights and, alongside, each batch row's activation chunk:
    // both arrive on the same mbarrier (no separate activation-load latency)
    mbar_expect_tx(&ws_->bar[p_st], XOFF + Rn * XB);
    uint8_t* dstg = ring + p_st * STAGE_BYTES;
    tma_load_1d(dstg, wbase + ((int64_t)p_grp * KT + p_kt) * UNIT_BYTES, UNIT_BYTES,
                &ws_->bar[p_st], policy);
    if constexpr (WT == kNF4)
      tma_load_1d(dstg + UNIT_BYTES, qsbase + ((int64_t)p_grp * KT + p_kt) * NF4_QS, NF4_QS,
                  &ws_->bar[p_st], policy);
    for (int r = 0; r < (RM == 1 ? 1 : Rn); ++r)
      tma_load_1d(dstg + XOFF + r * XS, a.x + (int64_t)(r0 + r) * a.ldx + p_kt * KTILE,
                  XB, &ws_->bar[p_st], policy_x);
    if (++p_kt == KT) { p_kt = 0; ++p_grp; }
    if (++p_st == ST) p_st = 0;
    --p_left;
  };
  __syncwarp();

  // ---- activation side: read from the stage (arrived with the weights) ----
  XVec xc[NT][2], gc[NT][2];
  constexpr int KOFF = INT ? 16 : 8;
  int c_grp = u0 / KT, c_kt = u0 % KT, c_st = 0;
  uint32_t c_ph = 0;

  using AccT = typename std::conditional<INT, int, float>::type;
  // nf4: acc[t][0] sums (unit partial) x (block scale) in int32; a warp flushes
  // every kNf4Flush units, the bound that keeps the sum exact:
  // |partial| <= 64 * 63 * 128, x 255, x 16 < 2^31
  constexpr int kNf4Flush = 16;
  AccT acc[RT][NT][4];
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[t][nt][j] = 0;
  int seg_kt0 = c_kt;
  // nf4 table words in per-thread registers: loaded from shared memory, so
  // ptxas cannot treat them as uniform constants and re-copy them from uniform
  // registers before every lookup
  const uint32_t la0 = WT == kNF4 ? *reinterpret_cast<volatile uint32_t*>(&nf4_lut[0]) : 0u;
  const uint32_t lb0 = WT == kNF4 ? *reinterpret_cast<volatile uint32_t*>(&nf4_lut[1]) : 0u;

  for (int i = 0; i < nunits; ++i) {
    mbar_wait(&ws_->bar[c_st], c_ph);
    if (i == 0) gtrace(a, 3);
    const uint8_t* stage = ring + c_st * STAGE_BYTES;
    if constexpr (WT == kNF4) {
      // ---- nf4 unit: 2 k-steps of 32; B = the row's activation digits ----

      // this lane's B column = (batch row brow[0], digit bsub[0])
      const float* xs = reinterpret_cast<const float*>(stage + XOFF + brow[0] * XS);
      uint32_t bb[2][2];
      const float mu = bmu[0], sc = bsc[0];
#pragma unroll
      for (int st = 0; st < 2; ++st) {
        const float4 v0 = *reinterpret_cast<const float4*>(xs + st * 32 + t4 * 4);
        const float4 v1 = *reinterpret_cast<const float4*>(xs + st * 32 + 16 + t4 * 4);
        float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        if (HASG) {
          const int64_t k0 = (int64_t)c_kt * KTILE + st * 32 + t4 * 4;
          const float4 g0 = __ldg(reinterpret_cast<const float4*>(a.g + k0));
          const float4 g1 = __ldg(reinterpret_cast<const float4*>(a.g + k0 + 16));
          const float g8v[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] *= g8v[j];
        }
        int q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float tt = (NORMT == NORM_LN) ? (v[j] - mu) : v[j];
          // rint(tt * sc) by the 1.5 * 2^23 shift (sc is a power of two, so the
          // product is exact and this equals __float2int_rn(tt * sc), |q| < 2^22):
          // FFMA + integer add instead of FMUL + F2I on the slower conversion pipe
          q[j] = __float_as_int(fmaf(tt, sc, 12582912.0f)) - 0x4B400000;
        }
        bb[st][0] = digits4(q[0], q[1], q[2], q[3], bbias[0], bsel_lo[0], 0x5410);
        bb[st][1] = digits4(q[4], q[5], q[6], q[7], bbias[0], bsel_lo[0], 0x5410);
      }
      // the level bytes carry +63 (7-bit, unsigned): subtract 63 * sum(B) per column
      int off[4] = {0, 0, 0, 0};
      const uint4 a63 = make_uint4(0x3F3F3F3Fu, 0x3F3F3F3Fu, 0x3F3F3F3Fu, 0x3F3F3F3Fu);
      mma_s8(off, a63, bb[0][0], bb[0][1]);
      mma_s8(off, a63, bb[1][0], bb[1][1]);
      const uint4 qv = *reinterpret_cast<const uint4*>(stage + UNIT_BYTES + (lane >> 2) * 16);
      const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w};
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const uint4 wv = *reinterpret_cast<const uint4*>(stage + (t * 32 + lane) * 16);
        // the -63 * sum(B) level offset seeds the accumulator (no per-tile subtraction)
        int c[4] = {-off[0], -off[1], -off[2], -off[3]};
        // entries 0-7 and 8-15 go to the tensor pipe as two A fragments (each
        // zero where the other table holds the code) instead of being OR-ed
        const uint32_t hx = wv.x >> 16, hy = wv.y >> 16, hz = wv.z >> 16, hw = wv.w >> 16;
        mma_s8(c, make_uint4(prmt_b32(la0, kLA1, wv.x), prmt_b32(la0, kLA1, hx),
                             prmt_b32(la0, kLA1, wv.y), prmt_b32(la0, kLA1, hy)),
               bb[0][0], bb[0][1]);
        mma_s8(c, make_uint4(prmt_b32(lb0, kLB1, wv.x ^ 0x8888u), prmt_b32(lb0, kLB1, hx ^ 0x8888u),
                             prmt_b32(lb0, kLB1, wv.y ^ 0x8888u), prmt_b32(lb0, kLB1, hy ^ 0x8888u)),
               bb[0][0], bb[0][1]);
        mma_s8(c, make_uint4(prmt_b32(la0, kLA1, wv.z), prmt_b32(la0, kLA1, hz),
                             prmt_b32(la0, kLA1, wv.w), prmt_b32(la0, kLA1, hw)),
               bb[1][0], bb[1][1]);
        mma_s8(c, make_uint4(prmt_b32(lb0, kLB1, wv.z ^ 0x8888u), prmt_b32(lb0, kLB1, hz ^ 0x8888u),
                             prmt_b32(lb0, kLB1, wv.w ^ 0x8888u), prmt_b32(lb0, kLB1, hw ^ 0x8888u)),
               bb[1][0], bb[1][1]);
        // block scales of rows g8 (h = 0) and g8 + 8 (h = 1): bytes 2t, 2t + 1
        const int q0 = (qw[t >> 1] >> (16 * (t & 1))) & 0xFF;
        const int q1 = (qw[t >> 1] >> (16 * (t & 1) + 8)) & 0xFF;
        acc[t][0][0] += c[0] * q0;
        acc[t][0][1] += c[1] * q0;
        acc[t][0][2] += c[2] * q1;
        acc[t][0][3] += c[3] * q1;
      }
    } else {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const float* xs = reinterpret_cast<const float*>(stage + UNIT_BYTES + brow[nt] * XSLOT) + t4 * XV;
      xc[nt][0] = *reinterpret_cast<const XVec*>(xs);
      xc[nt][1] = *reinterpret_cast<const XVec*>(xs + KOFF);
      if (HASG) {
        const int64_t k0 = (int64_t)c_kt * KTILE + t4 * XV;
        gc[nt][0] = __ldg(reinterpret_cast<const XVec*>(a.g + k0));
        gc[nt][1] = __ldg(reinterpret_cast<const XVec*>(a.g + k0 + KOFF));
      }
    }
    // ldmatrix.x4: lane i addresses row (i%8) of core matrix (kc = i/16, r8 = 2t + (i/8)%2)
    const uint8_t* lrow = stage + (lane >> 4) * 2048 + ((lane >> 3) & 1) * 128 + (lane & 7) * 16;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      uint32_t b0 = 0, b1 = 0;
      {
        const float mu = bmu[nt], sc = bsc[nt];
        if constexpr (WT == kI8) {
          float v[8] = {xc[nt][0].x, xc[nt][0].y, xc[nt][0].z, xc[nt][0].w,
                        xc[nt][1].x, xc[nt][1].y, xc[nt][1].z, xc[nt][1].w};
          if (HASG) {
            const float g8[8] = {gc[nt][0].x, gc[nt][0].y, gc[nt][0].z, gc[nt][0].w,
                                 gc[nt][1].x, gc[nt][1].y, gc[nt][1].z, gc[nt][1].w};
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] *= g8[j];
          }
          int q[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float t = (NORMT == NORM_LN) ? (v[j] - mu) : v[j];
            q[j] = __float2int_rn(t * sc);
          }
          b0 = digits4(q[0], q[1], q[2], q[3], bbias[nt], bsel_lo[nt], 0x5410);
          b1 = digits4(q[4], q[5], q[6], q[7], bbias[nt], bsel_lo[nt], 0x5410);
        } else {
          float v[4] = {xc[nt][0].x, xc[nt][0].y, xc[nt][1].x, xc[nt][1].y};
          if (HASG) {
            const float g4[4] = {gc[nt][0].x, gc[nt][0].y, gc[nt][1].x, gc[nt][1].y};
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] *= g4[j];
          }
          __nv_bfloat16 h[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float t = (NORMT == NORM_LN) ? (v[j] - mu) : v[j];
            h[j] = __float2bfloat16_rn(t);
            if (bsub[nt]) h[j] = __float2bfloat16_rn(t - __bfloat162float(h[j]));
          }
          __nv_bfloat162 p0 = __halves2bfloat162(h[0], h[1]), p1 = __halves2bfloat162(h[2], h[3]);
          b0 = *reinterpret_cast<uint32_t*>(&p0);
          b1 = *reinterpret_cast<uint32_t*>(&p1);
        }
      }
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        uint4 wt;
        ldsm_x4(wt, lrow + t * 256);
        if constexpr (INT) mma_s8(reinterpret_cast<int*>(acc[t][nt]), wt, b0, b1);
        else mma_bf16(reinterpret_cast<float*>(acc[t][nt]), wt, b0, b1);
      }
    }
    }   // int8 / bf16 unit
    __syncwarp();
    if (lane == 0 && p_left > 0) issue_next();
    if (++c_st == ST) { c_st = 0; c_ph ^= 1; }

    // ---- end of this warp's contribution to a group: flush ----
    const int64_t grp = c_grp;
    const int nkt = c_kt + 1 - seg_kt0;
    const bool grp_end = (c_kt + 1 == KT) || (i + 1 == nunits);
    const bool chunk_end = (WT == kNF4) && nkt == kNf4Flush;   // exactness bound (above)
    if (++c_kt == KT) { c_kt = 0; ++c_grp; seg_kt0 = 0; }
    if (i + 1 == nunits) gtrace(a, 4);
    if (!grp_end && !chunk_end) continue;
    if (!grp_end) seg_kt0 = c_kt;                 // nf4 mid-group flush: next segment
    // combine this segment's digit/hi-lo columns per (row, batch row) in registers
    unsigned long long* acc64 = reinterpret_cast<unsigned long long*>(a.ws);
    const int g8 = lane >> 2;
#pragma unroll
    for (int t = 0; t < RT; ++t) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t n = grp * 128 + t * 16 + g8 + h * 8;
        for (int r = 0; r < (RM == 1 ? 1 : Rn); ++r) {
          long long D = 0;
          if constexpr (INT) {
#pragma unroll
            for (int dg = 0; dg < NDIG; ++dg) {
              const int c = NDIG * r + dg, nt = c >> 3, cw = c & 7;
              int val = 0;
#pragma unroll
              for (int q = 0; q < NT; ++q)
                if (q == nt) val = (cw & 1) ? (int)acc[t][q][1 + 2 * h] : (int)acc[t][q][2 * h];
              val = __shfl_sync(0xffffffffu, val, g8 * 4 + (cw >> 1));
              D += (long long)val << (8 * (NDIG - 1 - dg));
            }
          } else {
            const int c = 2 * r, nt = c >> 3, cw = c & 7;
            float hi = 0.f, lo = 0.f;
#pragma unroll
            for (int q = 0; q < NT; ++q)
              if (q == nt) { hi = (float)acc[t][q][2 * h]; lo = (float)acc[t][q][2 * h + 1]; }
            hi = __shfl_sync(0xffffffffu, hi, g8 * 4 + (cw >> 1));
            lo = __shfl_sync(0xffffffffu, lo, g8 * 4 + (cw >> 1));
            D = __double2ll_rn(((double)hi + (double)lo) * kFix);
          }
          if (t4 == 0) atomicAdd(acc64 + (int64_t)(r0 + r) * a.N + n, (unsigned long long)D);
        }
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[t][nt][j] = 0;
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      int old;
      asm volatile("atom.release.gpu.global.add.s32 %0, [%1], %2;"
                   : "=r"(old) : "l"(a.counters + grp), "r"(nkt) : "memory");
      last = (old + nkt == KT);
      if (last) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        a.counters[grp] = 0;
      }
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) continue;

    // ---- epilogue for the group (128 channels x Rn rows), last warp only ----
    // every load of the lane (4 accumulators, their scales, residuals, next
    // gains) is issued before the first is used: one round trip, not four
    // EP >= 0: the epilogue type is a template constant (single-row kernels:
    // the unused variants' code is not emitted)
    const int epi = EP >= 0 ? EP : a.epi;
    const bool swiglu = (epi == EPI_SWIGLU);
    const int nj = swiglu ? 2 : 4;         // outputs per lane (64 or 128 per group)
    for (int r = 0; r < (RM == 1 ? 1 : Rn); ++r) {
      unsigned long long* accr = acc64 + (int64_t)(r0 + r) * a.N + grp * 128;
      const double ys = ws_->yscale[r];
      const int64_t yrow = (int64_t)(r0 + r) * a.ldy;
      long long D[4];
      float wsc[4], rv[4], gn[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int row = lane + 32 * j;
        D[j] = (long long)atomicExch(accr + row, 0ull);
        wsc[j] = INT ? __ldg(a.wscale + grp * 128 + row) : 1.f;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t col = swiglu ? grp * 64 + lane + 32 * j : grp * 128 + lane + 32 * j;
        rv[j] = (j < nj && epi == EPI_RESID) ? a.res[yrow + col] : 0.f;
        gn[j] = (j < nj && a.g_next) ? __ldg(a.g_next + col) : 1.f;
      }
      auto val_of = [&](int k) {
        if (INT) return (float)((double)D[k] * ys * (double)wsc[k]);
        return (float)((double)D[k] * ys);
      };
      float S = 0.f, Q = 0.f, M = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= nj) break;
        float val;
        int64_t col;
        if (swiglu) {
          // group = [gate 64 rows | up 64 rows] of outputs grp*64 + o
          val = silu_f(val_of(j)) * val_of(j + 2);
          col = grp * 64 + lane + 32 * j;
        } else {
          col = grp * 128 + lane + 32 * j;
          val = val_of(j);
          if (epi == EPI_RESID) val += rv[j];
          else if (epi == EPI_GELU) val = gelu_f(val);
        }
        a.y[yrow + col] = val;
        S += val;
        Q = fmaf(val, val, Q);
        M = fmaxf(M, fabsf(val * gn[j]));
      }
      if (a.st_out) {
        S = warp_sum(S); Q = warp_sum(Q); M = warp_max(M);
        if (lane == 0) a.st_out[grp * Rs + r0 + r] = RowStat{S, Q, M, 0.f};
      }
    }
    __syncwarp();
  }
  gtrace(a, 5);
}

int g_num_sms = 0;

template <int WT, int NT, int NORMT, bool HASG, int ND, int RM, int EP>
void launch_cfg(const GemvArgs& a, int r0, int rn, cudaStream_t st) {
  const int KTILE = (WT == kI8) ? 32 : (WT == kNF4 ? 64 : 16);
  const int64_t units = (a.N / 128) * (a.K / KTILE);
  const int grid = g_num_sms * CTAS_PER_SM;
  const size_t smem =
      (size_t)NW * stages_of(WT, RM) * stage_bytes_wt(WT, NT, RM) + (size_t)NW * sizeof(WarpSmem) +
      128;
  static bool set[kMaxDevices] = {};
  const int dv = current_device();
  if (!set[dv]) {
    cudaFuncSetAttribute(gemv3_kernel<WT, NT, NORMT, HASG, ND, RM, EP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    set[dv] = true;
  }
  static int trace_call = getenv("SP_GEMV_TRACE") ? atoi(getenv("SP_GEMV_TRACE")) : -1;
  static int ncall = 0;   // per instantiation
  GemvArgs b = a;
  const bool tr = trace_call >= 0 && ncall++ == trace_call;
  const size_t tn = (size_t)grid * NW * 8;
  unsigned long long* tbuf = nullptr;
  if (tr) {
    cudaMalloc(&tbuf, tn * 8);
    cudaMemsetAsync(tbuf, 0, tn * 8, st);
    b.trace = tbuf;
  }
  launch_pdl(gemv3_kernel<WT, NT, NORMT, HASG, ND, RM, EP>, dim3(grid), dim3(NW * 32), smem, st, b, r0, rn,
             a.R, units, (int64_t)grid * NW);
  count_launch();
  if (tr) {
    std::vector<unsigned long long> h(tn);
    cudaMemcpyAsync(h.data(), tbuf, tn * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long t0 = ~0ull;
    for (size_t i = 0; i < tn; i += 8) if (h[i] && h[i] < t0) t0 = h[i];
    fprintf(stderr, "gemv N=%lld K=%lld\n", (long long)a.N, (long long)a.K);
    for (size_t i = 0; i < tn; i += 8) {
      fprintf(stderr, "w %4zu:", i / 8);
      for (int p = 0; p < 6; ++p)
        fprintf(stderr, " %7.2f", h[i + p] ? (double)(h[i + p] - t0) / 1e3 : -1.0);
      fprintf(stderr, " %llu", h[i + 6]);
      fprintf(stderr, "\n");
    }
    cudaFree(tbuf);
  }
}

template <int WT, int NT, int ND, int RM, int EP>
void launch_norm(const GemvArgs& a, int r0, int rn, cudaStream_t st) {
  const bool hg = a.g != nullptr;
  switch (a.norm) {
    case NORM_RMS: hg ? launch_cfg<WT, NT, NORM_RMS, true, ND, RM, EP>(a, r0, rn, st)
                      : launch_cfg<WT, NT, NORM_RMS, false, ND, RM, EP>(a, r0, rn, st); break;
    case NORM_LN: hg ? launch_cfg<WT, NT, NORM_LN, true, ND, RM, EP>(a, r0, rn, st)
                     : launch_cfg<WT, NT, NORM_LN, false, ND, RM, EP>(a, r0, rn, st); break;
    default: launch_cfg<WT, NT, NORM_NONE, false, ND, RM, EP>(a, r0, rn, st); break;
  }
}

template <int WT, int NT, int ND, int RM>
void launch_nt2(const GemvArgs& a, int r0, int rn, cudaStream_t st) {
  if constexpr (RM != 1) {
    launch_norm<WT, NT, ND, RM, -1>(a, r0, rn, st);
  } else {
    // single-row kernels: one instantiation per (pre-norm, epilogue) pair the
    // span uses — normed input -> STORE / SWIGLU / GELU, raw input -> RESID
    const bool hg = a.g != nullptr;
    if ((a.norm == NORM_NONE) != (a.epi == EPI_RESID)) {   // other pairs: generic kernel
      if constexpr (WT != kNF4) launch_norm<WT, NT, ND, RMAX, -1>(a, r0, rn, st);
      else fprintf(stderr, "nf4 gemv: unsupported (norm, epilogue) pair\n");
      return;
    }
    if (a.norm == NORM_NONE) {
      launch_cfg<WT, NT, NORM_NONE, false, ND, RM, EPI_RESID>(a, r0, rn, st);
      return;
    }
    auto pick = [&](auto ep) {
      constexpr int E = decltype(ep)::value;
      if (a.norm == NORM_RMS)
        hg ? launch_cfg<WT, NT, NORM_RMS, true, ND, RM, E>(a, r0, rn, st)
           : launch_cfg<WT, NT, NORM_RMS, false, ND, RM, E>(a, r0, rn, st);
      else
        hg ? launch_cfg<WT, NT, NORM_LN, true, ND, RM, E>(a, r0, rn, st)
           : launch_cfg<WT, NT, NORM_LN, false, ND, RM, E>(a, r0, rn, st);
    };
    switch (a.epi) {
      case EPI_STORE: pick(std::integral_constant<int, EPI_STORE>{}); break;
      case EPI_SWIGLU: pick(std::integral_constant<int, EPI_SWIGLU>{}); break;
      default: pick(std::integral_constant<int, EPI_GELU>{}); break;
    }
  }
}

// one-row launches get their own instantiation (RM = 1): the per-row loops of
// the prologue, flush and epilogue collapse, and the kernel is a third smaller
template <int WT, int NT, int ND>
void launch_nt(const GemvArgs& a, int r0, int rn, cudaStream_t st) {
  if (NT == 1 && rn == 1) launch_nt2<WT, NT, ND, 1>(a, r0, rn, st);
  else launch_nt2<WT, NT, ND, RMAX>(a, r0, rn, st);
}

template <int WT, int ND>
void launch_wt(const GemvArgs& a, int r0, int rn, cudaStream_t st) {
  const int cols = rn * ((WT == kI8) ? ND : 2);
  if (cols <= 8) launch_nt<WT, 1, ND>(a, r0, rn, st);
  else if (cols <= 16) launch_nt<WT, 2, ND>(a, r0, rn, st);
  else launch_nt<WT, 3, ND>(a, r0, rn, st);
}

}  // namespace

int64_t gemv3_ws_bytes(int64_t N, int Rmax) { return (int64_t)Rmax * N * 8; }
int64_t gemv3_counters(int64_t N) { return N / 128 + 1; }

void launch_gemv3(int wdtype, const GemvArgs& a, cudaStream_t st) {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  for (int r0 = 0; r0 < a.R; r0 += RMAX) {
    const int rn = a.R - r0 < RMAX ? a.R - r0 : RMAX;
    // activation code width: 15 bits (2 balanced int8 digits, the precision
    // class of the prefill digit planes) for every row count, so a row's
    // result never depends on how many rows share the launch (decode numerics
    // independent of beam width / batch).  The 3-digit (23-bit) variant is
    // kept for A/B only (SP_GEMV_NDIG=3): it measured no faster at batch 1.
    static int nd_env = getenv("SP_GEMV_NDIG") ? atoi(getenv("SP_GEMV_NDIG")) : 0;
    const int nd = nd_env ? nd_env : kNDig;
    if (wdtype == kNF4) {
      // one launch per 4 rows (8 MMA columns at 2 digits): the weights stream
      // once for the batch; the 15-bit code keeps a row's result independent
      // of the launch's row count
      for (int q0 = r0; q0 < r0 + rn; q0 += 4) {
        const int qn = r0 + rn - q0 < 4 ? r0 + rn - q0 : 4;
        if (qn == 1) launch_nt2<kNF4, 1, 2, 1>(a, q0, 1, st);
        else launch_nt2<kNF4, 1, 2, 4>(a, q0, qn, st);
      }
    } else if (wdtype == kI8) {
      if (nd == 3) launch_wt<kI8, 3>(a, r0, rn, st);
      else launch_wt<kI8, 2>(a, r0, rn, st);
    } else {
      launch_wt<kBF16, 2>(a, r0, rn, st);
    }
  }
}

}  // namespace sp
