// Prefill / replay linear layers on the 5th-gen tensor cores (tcgen05 + TMEM).
//
//   Y[m, n] = epi( 2^(e_m - 14) * wscale[n] * sum_k (d0[m,k]*256 + d1[m,k]) * W[n,k] )
//
// * Activations are two int8 "digit planes" of a per-row 15-bit fixed-point
//   code (q = rint(x * 2^(14-e)), q = 256*d0 + d1): written by the digitize
//   kernel below in the same UMMA-canonical core-matrix layout as the weights
//   (common.cuh cm_offset), so both operands reach shared memory as plain 1-D
//   TMA bulk copies (cp.async.bulk + mbarrier complete_tx).
// * int8 weights are consumed as stored (no dequantisation pass): the MMA is
//   tcgen05.mma.cta_group::1.kind::i8, M = 128 tokens x N = 128 channels x
//   K = 32, both operands K-major SWIZZLE_NONE (LBO = 2048 B along K, SBO = 128 B
//   per 8 rows).  The CTA-pair kernel below (cta_group::2, M = 256, N = 256) is
//   the default; this one is the reference it is checked against bit for bit.  One CTA owns a 128 x 256 output tile = 2 planes x 2 weight
//   groups = 4 int32 accumulators = all 512 TMEM columns.
// * Accumulation is exact (int32 per plane, int64 when the planes combine), so
//   every output row is independent of M and of its tile position — the
//   micro-batch invariance the reference pins (T/test_server.py:247-255) holds.
// * Warp roles: warp 0 = TMA producer (one lane), warp 1 = MMA issuer (one
//   lane), warp 2 = TMEM allocator, warps 4..7 = epilogue (tcgen05.ld, scale,
//   residual / GELU / SwiGLU, store).  3-stage smem ring of 64 KB stages.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "prefill.cuh"

namespace sp {

namespace {

constexpr int BM = 128;                 // tokens per tile
constexpr int NGRP = 2;                 // 128-channel weight groups per tile (N = 256)
constexpr int KU = 4;                   // 32-byte K units per stage (128 B of K)
constexpr int STAGES = 3;
constexpr int UNIT = 4096;              // one 128-row x 32-byte unit (common.cuh)
constexpr int A_BYTES = 2 * KU * UNIT;  // two digit planes
constexpr int B_BYTES = NGRP * KU * UNIT;
constexpr int STAGE = A_BYTES + B_BYTES;   // 64 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (cute::UMMA::SmemDescriptor)
__device__ __forceinline__ uint64_t umma_desc(const void* smem, uint32_t lbo, uint32_t sbo) {
  const uint32_t addr = smem_u32(smem);
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;             // version = 1 (sm100)
  // base_offset = 0, lbo_mode = 0, layout_type = 0 (SWIZZLE_NONE)
  return d;
}

// instruction descriptor: kind::i8, D = s32, A = B = s8, K-major, M = 128, N = 128
constexpr uint32_t kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) |
                              ((128u >> 4) << 24);

// bf16 operands, f32 accumulation (kind::f16; c_format F32, a/b_format BF16)
constexpr uint32_t kIdescBF16 = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) |
                                ((128u >> 4) << 24);
__device__ __forceinline__ void mma_bf16_tc(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdescBF16), "r"(acc));
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdescI8), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                   "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, int* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, int* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + tanhf(0.7978845608028654f * (x + 0.044715f * x * x * x)));
}

// Epilogue of one 128-channel weight group for this thread's token row m.
// TMEM columns: plane p, group j, channel c -> p * 256 + j * 128 + c (both
// kernels).  D = D0 * 256 + D1 is exact (int64); y = f32(D) * 2^(e-14) * wscale.
// All TMEM loads of a chunk are issued before one wait.
// BF: bf16 operands (hi + lo f32 accumulators); EP >= 0: epilogue type fixed
// at compile time (only that variant's code is emitted), -1: a.epi at run time
template <bool BF, int EP>
__device__ __forceinline__ void epilogue_group(const TcGemmArgs& a, uint32_t tb, int j, int ng0,
                                               int64_t m, bool valid, float ys) {
  const int64_t n0 = (int64_t)(ng0 + j) * 128;
  const float* wsc = a.wscale ? a.wscale + n0 : nullptr;
  // int8: D = D0 * 256 + D1 exact in int64; bf16: hi + lo f32 accumulators
  auto comb = [](int x0, int x1) {
    if constexpr (BF) return __fadd_rn(__int_as_float(x0), __int_as_float(x1));
    else return (float)((long long)x0 * 256 + x1);
  };
  const int epi = EP >= 0 ? EP : a.epi;
  if (epi == EPI_SWIGLU) {
    // group = [gate 64 | up 64] of outputs (ng0 + j) * 64 + c
    for (int c0 = 0; c0 < 64; c0 += 32) {
      int g0[32], g1[32], u0[32], u1[32];
      tmem_ld32_nw(tb + (uint32_t)(0 * 256 + j * 128 + c0), g0);
      tmem_ld32_nw(tb + (uint32_t)(1 * 256 + j * 128 + c0), g1);
      tmem_ld32_nw(tb + (uint32_t)(0 * 256 + j * 128 + 64 + c0), u0);
      tmem_ld32_nw(tb + (uint32_t)(1 * 256 + j * 128 + 64 + c0), u1);
      tmem_wait_ld();
      if (!valid) continue;
      float* out = a.y + m * a.ldy + (ng0 + j) * 64 + c0;
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        float o4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int cc = c + e;
          // explicit roundings (no FMA contraction): every instantiation and both
          // GEMM kernels give bit-identical outputs
          const float gd = __fmul_rn(__fmul_rn(comb(g0[cc], g1[cc]), ys), wsc ? __ldg(wsc + c0 + cc) : 1.f);
          const float ud = __fmul_rn(__fmul_rn(comb(u0[cc], u1[cc]), ys), wsc ? __ldg(wsc + 64 + c0 + cc) : 1.f);
          o4[e] = __fmul_rn(__fdividef(gd, __fadd_rn(1.0f, __expf(-gd))), ud);
        }
        *reinterpret_cast<float4*>(out + c) = make_float4(o4[0], o4[1], o4[2], o4[3]);
      }
    }
  } else {
    for (int c0 = 0; c0 < 128; c0 += 32) {
      int v0[32], v1[32];
      tmem_ld32_nw(tb + (uint32_t)(0 * 256 + j * 128 + c0), v0);
      tmem_ld32_nw(tb + (uint32_t)(1 * 256 + j * 128 + c0), v1);
      tmem_wait_ld();
      if (!valid) continue;
      float* out = a.y + m * a.ldy + n0 + c0;
      const float* res = a.res ? a.res + m * a.ldy + n0 + c0 : nullptr;
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        float r4[4] = {0.f, 0.f, 0.f, 0.f};
        if (epi == EPI_RESID) {
          const float4 rr = *reinterpret_cast<const float4*>(res + c);
          r4[0] = rr.x; r4[1] = rr.y; r4[2] = rr.z; r4[3] = rr.w;
        }
        float o4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int cc = c + e;
          float v = __fmul_rn(__fmul_rn(comb(v0[cc], v1[cc]), ys), wsc ? __ldg(wsc + c0 + cc) : 1.f);
          if (epi == EPI_RESID) v = __fadd_rn(v, r4[e]);
          else if (epi == EPI_GELU) v = gelu_f(v);
          o4[e] = v;
        }
        *reinterpret_cast<float4*>(out + c) = make_float4(o4[0], o4[1], o4[2], o4[3]);
      }
    }
  }
}

// split-K, phase 1: this CTA's exact partial D = D0 * 256 + D1 of one weight
// group for row m, added into the int64 workspace (order-independent => the
// result is deterministic)
__device__ __forceinline__ void partial_group(const TcGemmArgs& a, uint32_t tb, int j, int ng0,
                                              int64_t m, bool valid) {
  unsigned long long* ws = reinterpret_cast<unsigned long long*>(a.ws) + m * a.N +
                           (int64_t)(ng0 + j) * 128;
  for (int c0 = 0; c0 < 128; c0 += 32) {
    int v0[32], v1[32];
    tmem_ld32_nw(tb + (uint32_t)(0 * 256 + j * 128 + c0), v0);
    tmem_ld32_nw(tb + (uint32_t)(1 * 256 + j * 128 + c0), v1);
    tmem_wait_ld();
    if (!valid) continue;
#pragma unroll
    for (int c = 0; c < 32; ++c)
      atomicAdd(ws + c0 + c, (unsigned long long)((long long)v0[c] * 256 + v1[c]));
  }
}

// split-K, phase 2 (last CTA of the tile, all 256 threads, consecutive threads
// on consecutive outputs): the epilogue of epilogue_group on the summed
// workspace, which is zeroed for the next use.  Plain L2 loads: every partial
// was fenced before its CTA's arrival on the tile counter.
__device__ __forceinline__ void finish_tile(const TcGemmArgs& a, int mt, int ng0) {
  const int rows = (int)min((int64_t)BM, a.M - (int64_t)mt * BM);
  const bool swiglu = a.epi == EPI_SWIGLU;
  const int outs = swiglu ? 64 : 128;                // outputs per weight group
  const int total = rows * NGRP * outs;
  long long* ws = a.ws;
  // 8 outputs per thread per pass with every load issued before the first use
  // (one L2 round trip per pass instead of one per output: this tail runs on
  // the critical path of every split-K GEMM)
  constexpr int U = 8;
  for (int i0 = threadIdx.x; i0 < total; i0 += U * blockDim.x) {
    long long g0[U], g1[U];
    float wg[U], wu[U], rv[U], ys[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      g0[u] = g1[u] = 0;
      wg[u] = wu[u] = rv[u] = 0.f;
      ys[u] = 1.f;
      if (i >= total) continue;
      const int r = i / (NGRP * outs), rem = i % (NGRP * outs), j = rem / outs, c = rem % outs;
      const int64_t m = (int64_t)mt * BM + r;
      const int64_t n0 = (int64_t)(ng0 + j) * 128;
      const long long* wr = ws + m * a.N + n0;
      ys[u] = ldexpf(1.0f, a.exps[m] - 14);
      g0[u] = __ldcg(wr + c);
      wg[u] = __ldg(a.wscale + n0 + c);
      if (swiglu) {
        g1[u] = __ldcg(wr + 64 + c);
        wu[u] = __ldg(a.wscale + n0 + 64 + c);
      } else if (a.epi == EPI_RESID) {
        rv[u] = a.res[m * a.ldy + n0 + c];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i >= total) continue;
      const int r = i / (NGRP * outs), rem = i % (NGRP * outs), j = rem / outs, c = rem % outs;
      const int64_t m = (int64_t)mt * BM + r;
      const int64_t n0 = (int64_t)(ng0 + j) * 128;
      long long* wr = ws + m * a.N + n0;
      if (swiglu) {
        const float gd = __fmul_rn(__fmul_rn((float)g0[u], ys[u]), wg[u]);
        const float ud = __fmul_rn(__fmul_rn((float)g1[u], ys[u]), wu[u]);
        wr[c] = 0;
        wr[64 + c] = 0;
        a.y[m * a.ldy + (ng0 + j) * 64 + c] = __fmul_rn(__fdividef(gd, __fadd_rn(1.0f, __expf(-gd))), ud);
      } else {
        float v = __fmul_rn(__fmul_rn((float)g0[u], ys[u]), wg[u]);
        wr[c] = 0;
        if (a.epi == EPI_RESID) v = __fadd_rn(v, rv[u]);
        else if (a.epi == EPI_GELU) v = gelu_f(v);
        a.y[m * a.ldy + n0 + c] = v;
      }
    }
  }
}

template <bool BF, int EP>
__global__ void __launch_bounds__(256, 1) gemm_i8_tc_kernel(TcGemmArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], tmem_full;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // token tiles vary fastest: the CTAs resident together share one weight
  // tile, so each weight byte leaves DRAM once and the re-reads hit L2
  const int ng0 = blockIdx.y * NGRP;         // first weight group of this tile
  const int mt = blockIdx.x;                 // token tile (128 rows)
  const int64_t KT = a.K >> 5;               // 32-byte units along K
  const int KBT = (int)(KT / KU);            // stages along K
  const int S = a.ksplit > 1 ? a.ksplit : 1; // K split (blockIdx.z = part)
  const int kb0 = (int)((int64_t)blockIdx.z * KBT / S), kb1 = (int)((int64_t)(blockIdx.z + 1) * KBT / S);
  const int KB = kb1 - kb0;                  // stages of this CTA
  __shared__ int last_cta;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    const uint8_t* pa0 = a.planes;
    const uint8_t* pa1 = a.planes + a.plane_stride;
    const uint8_t* wb = reinterpret_cast<const uint8_t*>(a.w);
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      uint8_t* st = smem + (size_t)s * STAGE;
      mbar_expect_tx(&full[s], STAGE);
      const int64_t ua = ((int64_t)mt * KT + (int64_t)(kb0 + kb) * KU) * UNIT;
      tma_load_1d(st, pa0 + ua, KU * UNIT, &full[s]);
      tma_load_1d(st + KU * UNIT, pa1 + ua, KU * UNIT, &full[s]);
      for (int j = 0; j < NGRP; ++j) {
        const int64_t ub = ((int64_t)(ng0 + j) * KT + (int64_t)(kb0 + kb) * KU) * UNIT;
        tma_load_1d(st + A_BYTES + j * KU * UNIT, wb + ub, KU * UNIT, &full[s]);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* st = smem + (size_t)s * STAGE;
#pragma unroll
      for (int u = 0; u < KU; ++u) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint64_t ad = umma_desc(st + p * KU * UNIT + u * UNIT, 2048, 128);
#pragma unroll
          for (int j = 0; j < NGRP; ++j) {
            const uint64_t bd = umma_desc(st + A_BYTES + j * KU * UNIT + u * UNIT, 2048, 128);
            if (BF) mma_bf16_tc(tbase + (uint32_t)((p * NGRP + j) * 128), ad, bd, (kb | u) ? 1u : 0u);
            else mma_i8(tbase + (uint32_t)((p * NGRP + j) * 128), ad, bd, (kb | u) ? 1u : 0u);
          }
        }
      }
      mma_commit(&empty[s]);          // frees the stage when these MMAs complete
    }
    mma_commit(&tmem_full);
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int q = warp - 4;                          // TMEM lane quarter
    const int row = q * 32 + lane;
    const int64_t m = (int64_t)mt * BM + row;
    mbar_wait(&tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const bool valid = m < a.M;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    if (S == 1) {
      const float ys = (valid && !BF) ? ldexpf(1.0f, a.exps[m] - 14) : 1.f;
      for (int j = 0; j < NGRP; ++j) epilogue_group<BF, EP>(a, tbase + lane_addr, j, ng0, m, valid, ys);
    } else {
      for (int j = 0; j < NGRP; ++j) partial_group(a, tbase + lane_addr, j, ng0, m, valid);
      __threadfence();
    }
  }
  if (S > 1) {
    // split-K: the last CTA of this output tile applies the epilogue
    __syncthreads();
    if (threadIdx.x == 0) {
      int* cnt = a.counters + (int64_t)mt * gridDim.y + blockIdx.y;
      const int old = atomicAdd(cnt, 1);
      last_cta = (old == S - 1);
      if (last_cta) { __threadfence(); *cnt = 0; }
    }
    __syncthreads();
    if (last_cta) finish_tile(a, mt, ng0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase)
                 : "memory");
}

// ---- CTA-pair variant (cta_group::2) ------------------------------------------
// A cluster of two CTAs on one TPC computes a 256-token x 256-channel tile:
// CTA r stages its own 128 tokens (both digit planes) and weight group ng0 + r;
// the leader issues tcgen05.mma.cta_group::2 (M = 256, N = 256), which reads
// A and B halves from both CTAs' shared memory and writes each CTA's TMEM
// rows.  Per SM and K unit this moves 12 KB from L2 instead of 16 KB for the
// same MMA work — the single-CTA kernel is bound by L2->SM throughput, not by
// the tensor pipe.  The peer's stage arrivals are relayed to the leader with
// a cluster-scope mbarrier arrive; MMA completion is multicast to both CTAs.
// (KUP K units per stage, ST stages; both configurations keep 192 KB in flight)
constexpr uint32_t kIdescI8x2 = (2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) |
                                ((256u >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
constexpr uint32_t kIdescBF16x2 = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) |
                                  ((256u >> 4) << 24);
__device__ __forceinline__ void mma_bf16_x2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdescBF16x2), "r"(acc));
}
__device__ __forceinline__ void mma_i8_x2(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdescI8x2), "r"(acc));
}
__device__ __forceinline__ void mma_commit_x2(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void tc_trace(const TcGemmArgs& a, int ph) {
  if (SP_DEV_TRACE && a.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    a.trace[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * 4 + ph] = t;
  }
}

template <int KUP, int STAGES2, bool BF, int EP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_i8_tc2_kernel(TcGemmArgs a) {
  constexpr int A2_BYTES = 2 * KUP * UNIT;   // two digit planes, 128 tokens
  constexpr int STAGE2 = A2_BYTES + KUP * UNIT;   // + one 128-channel weight group
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[STAGES2], peer_full[STAGES2], empty[STAGES2], tmem_full;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) tc_trace(a, 0);
  const uint32_t rank = cluster_rank();
  const int mt = blockIdx.x >> 1;            // 256-token tile of the pair (token tiles fastest)
  const int ng0 = blockIdx.y * 2;            // the pair's two 128-channel weight groups
  const int64_t KT = a.K >> 5;
  const int KB = (int)(KT / KUP);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1); mbar_init(&peer_full[s], 1); mbar_init(&empty[s], 1);
    }
    mbar_init(&tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();      // both CTAs' barriers and TMEM exist before any cross-CTA use
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: this CTA's half of every stage ----------------
    const uint8_t* pa0 = a.planes;
    const uint8_t* pa1 = a.planes + a.plane_stride;
    const uint8_t* wb = reinterpret_cast<const uint8_t*>(a.w);
    const int64_t arow = (int64_t)mt * 2 + rank;         // this CTA's 128-token block
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES2;
      if (kb >= STAGES2) mbar_wait(&empty[s], ((kb / STAGES2) - 1) & 1);
      uint8_t* st = smem + (size_t)s * STAGE2;
      if (a.debug == 2) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        continue;
      }
      mbar_expect_tx(&full[s], STAGE2);
      const int64_t ua = (arow * KT + (int64_t)kb * KUP) * UNIT;
      tma_load_1d(st, pa0 + ua, KUP * UNIT, &full[s]);
      tma_load_1d(st + KUP * UNIT, pa1 + ua, KUP * UNIT, &full[s]);
      const int64_t ub = ((int64_t)(ng0 + rank) * KT + (int64_t)kb * KUP) * UNIT;
      tma_load_1d(st + A2_BYTES, wb + ub, KUP * UNIT, &full[s]);
    }
  } else if (warp == 3 && lane == 0 && rank == 1) {
    // ---------------- relay (peer): stage landed here -> leader ----------------
    const uint32_t pf = mapa_shared(smem_u32(&peer_full[0]), 0);
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES2;
      mbar_wait(&full[s], (kb / STAGES2) & 1);
      mbar_arrive_remote(pf + (uint32_t)s * 8u);
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (leader) ----------------
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES2;
      const uint32_t ph = (kb / STAGES2) & 1;
      mbar_wait(&full[s], ph);
      mbar_wait_cluster(&peer_full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* st = smem + (size_t)s * STAGE2;
#pragma unroll
      for (int u = 0; u < KUP; ++u) {
        if (a.debug == 1) break;
        const uint64_t bd = umma_desc(st + A2_BYTES + u * UNIT, 2048, 128);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint64_t ad = umma_desc(st + p * KUP * UNIT + u * UNIT, 2048, 128);
          if (BF) mma_bf16_x2(tbase + (uint32_t)(p * 256), ad, bd, (kb | u) ? 1u : 0u);
          else mma_i8_x2(tbase + (uint32_t)(p * 256), ad, bd, (kb | u) ? 1u : 0u);
        }
      }
      mma_commit_x2(&empty[s]);        // frees stage s in both CTAs when these MMAs finish
    }
    mma_commit_x2(&tmem_full);
  }
  {
    // ---------------- epilogue: this CTA's 128 tokens x 256 channels ----------------
    // all 8 warps, once their pipeline roles are done: warp w reads TMEM lane
    // quarter w % 4 (the lanes a warp may access) and weight group w / 4
    __syncwarp();                      // role lanes rejoin: tcgen05.ld is warp-aligned
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int64_t m = ((int64_t)mt * 2 + rank) * 128 + row;
    mbar_wait(&tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 128) tc_trace(a, 1);
    const bool valid = m < a.M;
    const float ys = (valid && !BF) ? ldexpf(1.0f, a.exps[m] - 14) : 1.f;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    epilogue_group<BF, EP>(a, tbase + lane_addr, warp >> 2, ng0, m, valid, ys);
  }
  if (threadIdx.x == 128) tc_trace(a, 2);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();      // the leader's MMAs wrote the peer's TMEM: free it only now
  if (threadIdx.x == 0) tc_trace(a, 3);
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase)
                 : "memory");
}

// ---- activation digit planes: one CTA per (padded) row -----------------------
// norm: 0 none, 1 RMSNorm, 2 LayerNorm (gains g, bias b; eps 1e-5)
__global__ void __launch_bounds__(256) digitize_kernel(const float* __restrict__ x, int64_t ldx,
                                                       int64_t M, int64_t K, int norm,
                                                       const float* g, const float* b,
                                                       uint8_t* planes, int64_t plane_stride,
                                                       int* exps, int rt) {
  __shared__ float sh[3][9];
  const int64_t m = blockIdx.x;
  const float* xr = x + m * ldx;
  const bool valid = m < M;
  float mu = 0.f, rstd = 1.f;
  auto bsum = [&](float v, int slot) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) sh[slot][threadIdx.x >> 5] = v;
    __syncthreads();
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += sh[slot][w];
    __syncthreads();
    return t;
  };
  if (valid && norm != 0) {
    float s = 0.f, s2 = 0.f;
    for (int64_t k = threadIdx.x; k < K; k += 256) { s += xr[k]; s2 = fmaf(xr[k], xr[k], s2); }
    if (norm == 2) {
      mu = bsum(s, 0) / (float)K;
      float q = 0.f;
      for (int64_t k = threadIdx.x; k < K; k += 256) { float c = xr[k] - mu; q = fmaf(c, c, q); }
      rstd = 1.0f / sqrtf(bsum(q, 1) / (float)K + 1e-5f);
    } else {
      rstd = 1.0f / sqrtf(bsum(s2, 1) / (float)K + 1e-5f);
    }
  }
  auto val = [&](int64_t k) -> float {
    if (!valid) return 0.f;
    float v = xr[k];
    if (norm == 1) v = v * rstd * g[k];
    else if (norm == 2) v = (v - mu) * rstd * g[k] + b[k];
    return v;
  };
  float amax = 0.f;
  for (int64_t k = threadIdx.x; k < K; k += 256) amax = fmaxf(amax, fabsf(val(k)));
  amax = warp_max(amax);
  if ((threadIdx.x & 31) == 0) sh[2][threadIdx.x >> 5] = amax;
  __syncthreads();
  amax = 0.f;
  for (int w = 0; w < 8; ++w) amax = fmaxf(amax, sh[2][w]);
  int e = 0;
  if (amax > 0.f) frexpf(amax, &e);                 // |v| < 2^e
  const float sc = amax > 0.f ? ldexpf(1.0f, 14 - e) : 0.f;
  if (threadIdx.x == 0 && valid) exps[m] = e;
  // 16 consecutive k per thread -> one 16-byte core-matrix row per plane
  for (int64_t k0 = (int64_t)threadIdx.x * 16; k0 < K; k0 += 256 * 16) {
    __align__(16) int8_t d0[16], d1[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int q = __float2int_rn(val(k0 + i) * sc);      // |q| <= 2^14
      const int lo = (int)(int8_t)(q & 0xFF);
      d1[i] = (int8_t)lo;
      d0[i] = (int8_t)((q - lo) >> 8);
    }
    const int64_t off = cm_offset_rt(m, k0, K, rt);
    *reinterpret_cast<uint4*>(planes + off) = *reinterpret_cast<uint4*>(d0);
    *reinterpret_cast<uint4*>(planes + plane_stride + off) = *reinterpret_cast<uint4*>(d1);
  }
}

// register-resident digitize: the row is read from HBM once (16 consecutive
// floats per thread and chunk, four float4 loads), normalised and reduced in
// registers, and written as one 16-byte core-matrix row per plane and chunk.
template <int NT, int NCH>
__global__ void __launch_bounds__(NT) digitize_reg_kernel(const float* __restrict__ x, int64_t ldx,
                                                          int64_t M, int64_t K, int norm,
                                                          const float* __restrict__ g,
                                                          const float* __restrict__ b,
                                                          uint8_t* planes, int64_t plane_stride,
                                                          int* exps, int rt) {
  constexpr int NW = NT / 32;
  __shared__ float red[3][NW];
  const int64_t m = blockIdx.x;
  const float* xr = x + m * ldx;
  const bool valid = m < M;
  const int nchunk = (int)(K >> 4);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float v[NCH][16];
  auto bsum = [&](float a, int slot) {
    a = warp_sum(a);
    if (lane == 0) red[slot][warp] = a;
    __syncthreads();
    float r = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) r += red[slot][w];
    return r;
  };
  float s = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = t + j * NT;
    if (valid && c < nchunk) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 f = __ldcs(reinterpret_cast<const float4*>(xr + (int64_t)c * 16) + q);
        v[j][4 * q] = f.x; v[j][4 * q + 1] = f.y; v[j][4 * q + 2] = f.z; v[j][4 * q + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[j][e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) { s += v[j][e]; s2 = fmaf(v[j][e], v[j][e], s2); }
  }
  if (norm != 0) {
    float mu = 0.f, rstd;
    if (norm == 2) {
      mu = bsum(s, 0) / (float)K;
      float q2 = 0.f;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int c = t + j * NT;
        if (c < nchunk)
#pragma unroll
          for (int e = 0; e < 16; ++e) { const float d = v[j][e] - mu; q2 = fmaf(d, d, q2); }
      }
      rstd = 1.0f / sqrtf(bsum(q2, 1) / (float)K + 1e-5f);
    } else {
      rstd = 1.0f / sqrtf(bsum(s2, 1) / (float)K + 1e-5f);
    }
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = t + j * NT;
      if (!(valid && c < nchunk)) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 gg = __ldg(reinterpret_cast<const float4*>(g + (int64_t)c * 16) + q);
        const float gq[4] = {gg.x, gg.y, gg.z, gg.w};
        float bq[4] = {0.f, 0.f, 0.f, 0.f};
        if (norm == 2) {
          const float4 bb = __ldg(reinterpret_cast<const float4*>(b + (int64_t)c * 16) + q);
          bq[0] = bb.x; bq[1] = bb.y; bq[2] = bb.z; bq[3] = bb.w;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float& vv = v[j][4 * q + e];
          vv = (norm == 1) ? vv * rstd * gq[e] : (vv - mu) * rstd * gq[e] + bq[e];
        }
      }
    }
  }
  float amax = 0.f;
#pragma unroll
  for (int j = 0; j < NCH; ++j)
#pragma unroll
    for (int e = 0; e < 16; ++e) amax = fmaxf(amax, fabsf(v[j][e]));
  amax = warp_max(amax);
  if (lane == 0) red[2][warp] = amax;
  __syncthreads();
  amax = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) amax = fmaxf(amax, red[2][w]);
  int e2 = 0;
  if (amax > 0.f) frexpf(amax, &e2);                 // |v| < 2^e
  const float sc = amax > 0.f ? ldexpf(1.0f, 14 - e2) : 0.f;
  if (t == 0 && valid) exps[m] = e2;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = t + j * NT;
    if (c >= nchunk) continue;
    __align__(16) int8_t d0[16], d1[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int qv = __float2int_rn(v[j][i] * sc);    // |q| <= 2^14
      const int lo = (int)(int8_t)(qv & 0xFF);
      d1[i] = (int8_t)lo;
      d0[i] = (int8_t)((qv - lo) >> 8);
    }
    const int64_t off = cm_offset_rt(m, (int64_t)c * 16, K, rt);
    *reinterpret_cast<uint4*>(planes + off) = *reinterpret_cast<uint4*>(d0);
    *reinterpret_cast<uint4*>(planes + plane_stride + off) = *reinterpret_cast<uint4*>(d1);
  }
}


// few-row digitize (wide decode, M <= 32 rows): one row per thread-block
// cluster of CL CTAs (grid (CL, M)), each CTA holding 1/CL of the row in
// registers; the row's sums and maximum are combined over distributed shared
// memory in rank order (every CTA gets the same totals), so a 57 K-element
// row is read by 8 SMs at once instead of one CTA streaming it alone.
template <int NCH>
__global__ void __launch_bounds__(256) digitize_cl_kernel(const float* __restrict__ x, int64_t ldx,
                                                         int64_t M, int64_t K, int norm,
                                                         const float* __restrict__ g,
                                                         const float* __restrict__ b,
                                                         uint8_t* planes, int64_t plane_stride,
                                                         int* exps, int rt) {
  namespace cgx = cooperative_groups;
  constexpr int NT = 256, NW = NT / 32;
  cgx::cluster_group cluster = cgx::this_cluster();
  const int CL = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  __shared__ float red[NW];
  __shared__ float part[3];                        // this CTA's (sum, centred sumsq, amax)
  const int64_t m = blockIdx.y;
  const float* xr = x + m * ldx;
  const int nchunk = (int)(K >> 4);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float v[NCH][16];
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = (rank + CL * j) * NT + t;
    if (c < nchunk) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 f = __ldcs(reinterpret_cast<const float4*>(xr + (int64_t)c * 16) + q);
        v[j][4 * q] = f.x; v[j][4 * q + 1] = f.y; v[j][4 * q + 2] = f.z; v[j][4 * q + 3] = f.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[j][e] = 0.f;
    }
  }
  // cluster-wide reduction of one value (sum or max), rank order
  auto csum = [&](float a, int slot, bool is_max) {
    a = is_max ? warp_max(a) : warp_sum(a);
    if (lane == 0) red[warp] = a;
    __syncthreads();
    if (t == 0) {
      float r = is_max ? 0.f : 0.f;
      for (int w = 0; w < NW; ++w) r = is_max ? fmaxf(r, red[w]) : r + red[w];
      part[slot] = r;
    }
    cluster.sync();
    float r = 0.f;
    for (int c = 0; c < CL; ++c) {
      const float pv = *cluster.map_shared_rank(&part[slot], c);
      r = is_max ? fmaxf(r, pv) : r + pv;
    }
    return r;
  };
  float s = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < NCH; ++j)
#pragma unroll
    for (int e = 0; e < 16; ++e) { s += v[j][e]; s2 = fmaf(v[j][e], v[j][e], s2); }
  if (norm != 0) {
    float mu = 0.f, rstd;
    if (norm == 2) {
      mu = csum(s, 0, false) / (float)K;
      float q2 = 0.f;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int c = (rank + CL * j) * NT + t;
        if (c < nchunk)
#pragma unroll
          for (int e = 0; e < 16; ++e) { const float d = v[j][e] - mu; q2 = fmaf(d, d, q2); }
      }
      rstd = 1.0f / sqrtf(csum(q2, 1, false) / (float)K + 1e-5f);
    } else {
      rstd = 1.0f / sqrtf(csum(s2, 1, false) / (float)K + 1e-5f);
    }
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = (rank + CL * j) * NT + t;
      if (c >= nchunk) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 gg = __ldg(reinterpret_cast<const float4*>(g + (int64_t)c * 16) + q);
        const float gq[4] = {gg.x, gg.y, gg.z, gg.w};
        float bq[4] = {0.f, 0.f, 0.f, 0.f};
        if (norm == 2) {
          const float4 bb = __ldg(reinterpret_cast<const float4*>(b + (int64_t)c * 16) + q);
          bq[0] = bb.x; bq[1] = bb.y; bq[2] = bb.z; bq[3] = bb.w;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float& vv = v[j][4 * q + e];
          vv = (norm == 1) ? vv * rstd * gq[e] : (vv - mu) * rstd * gq[e] + bq[e];
        }
      }
    }
  }
  float amax = 0.f;
#pragma unroll
  for (int j = 0; j < NCH; ++j)
#pragma unroll
    for (int e = 0; e < 16; ++e) amax = fmaxf(amax, fabsf(v[j][e]));
  amax = csum(amax, 2, true);
  int e2 = 0;
  if (amax > 0.f) frexpf(amax, &e2);                 // |v| < 2^e
  const float sc = amax > 0.f ? ldexpf(1.0f, 14 - e2) : 0.f;
  if (t == 0 && rank == 0) exps[m] = e2;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = (rank + CL * j) * NT + t;
    if (c >= nchunk) continue;
    __align__(16) int8_t d0[16], d1[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int qv = __float2int_rn(v[j][i] * sc);    // |q| <= 2^14
      const int lo = (int)(int8_t)(qv & 0xFF);
      d1[i] = (int8_t)lo;
      d0[i] = (int8_t)((qv - lo) >> 8);
    }
    const int64_t off = cm_offset_rt(m, (int64_t)c * 16, K, rt);
    *reinterpret_cast<uint4*>(planes + off) = *reinterpret_cast<uint4*>(d0);
    *reinterpret_cast<uint4*>(planes + plane_stride + off) = *reinterpret_cast<uint4*>(d1);
  }
  cluster.sync();                                  // peers' partials read before exit
}

// bf16 operands for the tcgen05 GEMM (bf16 weights, Llama-2-7B): the
// (normalised) row as hi = bf16(x) and lo = bf16(x - hi) planes in the same
// core-matrix layout (16-byte rows = 8 elements); no exponent
template <int NT, int NCH>
__global__ void __launch_bounds__(NT) digitize_bf16_kernel(const float* __restrict__ x, int64_t ldx,
                                                           int64_t M, int64_t K, int norm,
                                                           const float* __restrict__ g,
                                                           const float* __restrict__ b,
                                                           uint8_t* planes, int64_t plane_stride) {
  constexpr int NW = NT / 32;
  __shared__ float red[2][NW];
  const int64_t m = blockIdx.x;
  const float* xr = x + m * ldx;
  const int nchunk = (int)(K >> 3);               // 8 elements per 16-byte core-matrix row
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  float v[NCH][8];
  auto bsum = [&](float a, int slot) {
    a = warp_sum(a);
    if (lane == 0) red[slot][warp] = a;
    __syncthreads();
    float r = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) r += red[slot][w];
    return r;
  };
  float s = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = t + j * NT;
    if (c < nchunk) {
      const float4 f0 = __ldcs(reinterpret_cast<const float4*>(xr + (int64_t)c * 8));
      const float4 f1 = __ldcs(reinterpret_cast<const float4*>(xr + (int64_t)c * 8) + 1);
      v[j][0] = f0.x; v[j][1] = f0.y; v[j][2] = f0.z; v[j][3] = f0.w;
      v[j][4] = f1.x; v[j][5] = f1.y; v[j][6] = f1.z; v[j][7] = f1.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[j][e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) { s += v[j][e]; s2 = fmaf(v[j][e], v[j][e], s2); }
  }
  if (norm != 0) {
    float mu = 0.f, rstd;
    if (norm == 2) {
      mu = bsum(s, 0) / (float)K;
      float q2 = 0.f;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
        if (t + j * NT < nchunk)
#pragma unroll
          for (int e = 0; e < 8; ++e) { const float dd = v[j][e] - mu; q2 = fmaf(dd, dd, q2); }
      rstd = 1.0f / sqrtf(bsum(q2, 1) / (float)K + 1e-5f);
    } else {
      rstd = 1.0f / sqrtf(bsum(s2, 1) / (float)K + 1e-5f);
    }
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = t + j * NT;
      if (c >= nchunk) continue;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int64_t k = (int64_t)c * 8 + e;
        v[j][e] = (norm == 1) ? v[j][e] * rstd * g[k] : (v[j][e] - mu) * rstd * g[k] + b[k];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NCH; ++j) {
    const int c = t + j * NT;
    if (c >= nchunk) continue;
    __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      hi[e] = __float2bfloat16_rn(v[j][e]);
      lo[e] = __float2bfloat16_rn(v[j][e] - __bfloat162float(hi[e]));
    }
    const int64_t off = cm_offset(m, (int64_t)c * 16, 2 * K);
    *reinterpret_cast<uint4*>(planes + off) = *reinterpret_cast<uint4*>(hi);
    *reinterpret_cast<uint4*>(planes + plane_stride + off) = *reinterpret_cast<uint4*>(lo);
  }
}

}  // namespace

bool g_tc_pair = true;

void launch_digitize(const float* x, int64_t ldx, int64_t M, int64_t K, int norm, const float* g,
                     const float* b, uint8_t* planes, int64_t plane_stride, int* exps,
                     cudaStream_t st, int rt) {
  // padding rows of the planes are never written: a tile's rows are
  // independent in the MMA and the GEMM epilogue drops rows >= M
  const unsigned grid = (unsigned)M;
  const bool al = (K % 16 == 0) && (ldx % 4 == 0);
  static const bool cl_ok = getenv("SP_DIGITIZE_CL") ? atoi(getenv("SP_DIGITIZE_CL")) != 0 : true;
  if (cl_ok && al && M <= 32 && K > 256 * 16 * 2 && K <= 8 * 256 * 16 * 4) {
    // few rows (wide decode): a cluster of CL CTAs per row, 256 threads x 2-4 chunks each
    const int64_t nchunk = K / 16;
    int CLN = (int)((nchunk + 256 * 2 - 1) / (256 * 2));
    const bool four = CLN > 8;
    if (four) CLN = (int)((nchunk + 256 * 4 - 1) / (256 * 4));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)CLN, (unsigned)M);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CLN;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (four)
      cudaLaunchKernelEx(&cfg, digitize_cl_kernel<4>, x, ldx, M, K, norm, g, b, planes,
                         plane_stride, exps, rt);
    else
      cudaLaunchKernelEx(&cfg, digitize_cl_kernel<2>, x, ldx, M, K, norm, g, b, planes,
                         plane_stride, exps, rt);
    count_launch();
    return;
  }
  if (al && K <= 256 * 16 * 2)
    digitize_reg_kernel<256, 2><<<grid, 256, 0, st>>>(x, ldx, M, K, norm, g, b, planes, plane_stride, exps, rt);
  else if (al && K <= 256 * 16 * 4)
    digitize_reg_kernel<256, 4><<<grid, 256, 0, st>>>(x, ldx, M, K, norm, g, b, planes, plane_stride, exps, rt);
  else if (al && K <= 512 * 16 * 4)
    digitize_reg_kernel<512, 4><<<grid, 512, 0, st>>>(x, ldx, M, K, norm, g, b, planes, plane_stride, exps, rt);
  else if (al && K <= 1024 * 16 * 4)
    digitize_reg_kernel<1024, 4><<<grid, 1024, 0, st>>>(x, ldx, M, K, norm, g, b, planes, plane_stride, exps, rt);
  else
    digitize_kernel<<<grid, 256, 0, st>>>(x, ldx, M, K, norm, g, b, planes, plane_stride, exps, rt);
  count_launch();
}

template <int KUP, int ST, bool BF, int EP>
void launch_pair(const TcGemmArgs& a, cudaStream_t st) {
  static bool set2[kMaxDevices] = {};
  const int dv = current_device();
  const size_t smem2 = (size_t)ST * 3 * KUP * UNIT;
  if (!set2[dv]) {
    cudaFuncSetAttribute(gemm_i8_tc2_kernel<KUP, ST, BF, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem2);
    set2[dv] = true;
  }
  dim3 grid2((unsigned)(2 * ((a.M + 255) / 256)), (unsigned)(a.N / 256));
  static int dbg = getenv("SP_TC_DEBUG") ? atoi(getenv("SP_TC_DEBUG")) : 0;
  static int trc = getenv("SP_TC_TRACE") ? atoi(getenv("SP_TC_TRACE")) : -1;
  static int ncall = 0;
  TcGemmArgs b = a;
  b.debug = dbg;
  const bool tr = trc >= 0 && ncall++ == trc;
  const size_t tn = (size_t)grid2.x * grid2.y * 4;
  if (tr) {
    cudaMalloc(&b.trace, tn * 8);
    cudaMemsetAsync(b.trace, 0, tn * 8, st);
  }
  gemm_i8_tc2_kernel<KUP, ST, BF, EP><<<grid2, 256, smem2, st>>>(b);
  count_launch();
  if (tr) {
    std::vector<unsigned long long> h(tn);
    cudaMemcpyAsync(h.data(), b.trace, tn * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long t0 = ~0ull;
    for (size_t i = 0; i < tn; i += 4) if (h[i] && h[i] < t0) t0 = h[i];
    fprintf(stderr, "tcgemm M=%lld N=%lld K=%lld\n", (long long)a.M, (long long)a.N, (long long)a.K);
    for (size_t i = 0; i < tn; i += 4)
      fprintf(stderr, "c %zu %.2f %.2f %.2f %.2f\n", i / 4, (h[i] - t0) / 1e3, (h[i + 1] - t0) / 1e3,
              (h[i + 2] - t0) / 1e3, (h[i + 3] - t0) / 1e3);
    cudaFree(b.trace);
  }
}



// ---- the decode GEMV's activation code for the wide-decode GEMM ----------------
// (gemv3.cu prologue and unit loop, restated so that a row of a wide step gets
// exactly the GEMV's integers and scale): statistics from the producer's
// partials in the GEMV's reduction order (256 threads, partials p and p + 256
// per thread, warp butterflies, warps in order), bound -> exponent e,
// q = rint(t * 2^(14-e)) with t = x*g (- mu for LayerNorm), ys = 2^(e-14) * rstd.
__device__ __forceinline__ float silu_gemv(float x) { return x / (1.0f + expf(-x)); }

__global__ void __launch_bounds__(256) digitize_gemv_kernel(
    const float* __restrict__ x, int64_t ldx, int64_t M, int64_t K, int norm,
    const float* __restrict__ g, const float4* __restrict__ st_in, int P_in, float gmax, float eps,
    uint8_t* planes, int64_t plane_stride, double* ys_rows, int rt) {
  __shared__ float red[8][3];
  __shared__ float prm[2];                          // mu, dscale
  const int64_t m = blockIdx.y;                     // row; blockIdx.x = 4096-element slice
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nchunk = (int)(K >> 4);
  const int c = blockIdx.x * 256 + t;              // this thread's 16 elements
  float4 xv[4];                                    // loaded ahead of the statistics
  if (c < nchunk) {
#pragma unroll
    for (int qd = 0; qd < 4; ++qd)
      xv[qd] = __ldg(reinterpret_cast<const float4*>(x + m * ldx + (int64_t)c * 16) + qd);
  }
  float S = 0.f, Q = 0.f, Mx = 0.f;
  for (int p0 = t; p0 < P_in; p0 += 4 * 256) {
    float4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int p = p0 + j * 256;
      v[j] = p < P_in ? st_in[(int64_t)p * M + m] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) { S += v[j].x; Q += v[j].y; Mx = fmaxf(Mx, v[j].z); }
  }
  {
    const float vs = warp_sum(S), vq = warp_sum(Q), vm = warp_max(Mx);
    if (lane == 0) { red[warp][0] = vs; red[warp][1] = vq; red[warp][2] = vm; }
  }
  __syncthreads();
  if (t == 0) {
    float s = 0.f, q = 0.f, mm = 0.f;
    for (int w = 0; w < 8; ++w) { s += red[w][0]; q += red[w][1]; mm = fmaxf(mm, red[w][2]); }
    const float invK = 1.0f / (float)K;
    float mu = 0.f, rstd = 1.f, bound = mm;
    if (norm == 1) {
      rstd = 1.0f / sqrtf(q * invK + eps);
    } else if (norm == 2) {
      mu = s * invK;
      rstd = 1.0f / sqrtf(fmaxf(q * invK - mu * mu, 0.f) + eps);
      bound = mm + fabsf(mu) * gmax;
    }
    int e = 0;
    if (bound > 0.f) frexpf(bound, &e);             // bound < 2^e
    prm[0] = mu;
    prm[1] = bound > 0.f ? ldexpf(1.0f, 14 - e) : 0.f;
    if (blockIdx.x == 0) ys_rows[m] = ldexp(1.0, e - 14) * (double)rstd;
  }
  __syncthreads();
  const float mu = prm[0], sc = prm[1];
  // every CTA of the row recomputes the same statistics and codes one
  // 256-chunk slice of the row (no reduction over x: the coding is per element)
  {
    if (c >= nchunk) return;
    __align__(16) int8_t d0[16], d1[16];
#pragma unroll
    for (int qd = 0; qd < 4; ++qd) {
      const float4 f = xv[qd];
      float v[4] = {f.x, f.y, f.z, f.w};
      if (g) {
        const float4 gg = __ldg(reinterpret_cast<const float4*>(g + (int64_t)c * 16) + qd);
        v[0] *= gg.x; v[1] *= gg.y; v[2] *= gg.z; v[3] *= gg.w;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float tt = (norm == 2) ? (v[e] - mu) : v[e];
        const int qv = __float2int_rn(tt * sc);
        const int lo = (int)(int8_t)(qv & 0xFF);
        d1[4 * qd + e] = (int8_t)lo;
        d0[4 * qd + e] = (int8_t)((qv - lo) >> 8);
      }
    }
    const int64_t off = cm_offset_rt(m, (int64_t)c * 16, K, rt);
    *reinterpret_cast<uint4*>(planes + off) = *reinterpret_cast<uint4*>(d0);
    *reinterpret_cast<uint4*>(planes + plane_stride + off) = *reinterpret_cast<uint4*>(d1);
  }
}

// the GEMV's epilogue for rows x one 128-channel weight group: val =
// f32((double)D * ys * wscale) (+ residual / GELU, or SwiGLU of the group's two
// halves), then the group's (sum, sumsq, max|val * g_next|) partial, lanes and
// the warp butterfly in the GEMV's order.  vals(c) returns the pre-epilogue
// value of channel c (0..127) of the group for this row.
template <typename VAL>
__device__ __forceinline__ void gemv_epilogue_group(const TcGemmArgs& a, int grp, int64_t m,
                                                    int lane, VAL vals) {
  const bool swiglu = a.epi == EPI_SWIGLU;
  const int nj = swiglu ? 2 : 4;
  // every input of the lane first (the group's values, residuals): one round
  // trip instead of a load -> store chain per output (res may alias y)
  float v[4], rv[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = vals(lane + 32 * i);
  if (!swiglu && a.epi == EPI_RESID) {
#pragma unroll
    for (int i = 0; i < 4; ++i) rv[i] = a.res[m * a.ldy + (int64_t)grp * 128 + lane + 32 * i];
  }
  float S = 0.f, Q = 0.f, M = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j >= nj) break;
    float val;
    int64_t col;
    if (swiglu) {
      col = (int64_t)grp * 64 + lane + 32 * j;
      val = silu_gemv(v[j]) * v[j + 2];
    } else {
      col = (int64_t)grp * 128 + lane + 32 * j;
      val = v[j];
      if (a.epi == EPI_RESID) val += rv[j];
      else if (a.epi == EPI_GELU) val = gelu_f(val);
    }
    a.y[m * a.ldy + col] = val;
    const float gn = a.g_next ? __ldg(a.g_next + col) : 1.f;
    S += val;
    Q = fmaf(val, val, Q);
    M = fmaxf(M, fabsf(val * gn));
  }
  if (a.st_out) {
    S = warp_sum(S); Q = warp_sum(Q); M = warp_max(M);
    if (lane == 0) a.st_out[(int64_t)grp * a.stat_rs + m] = make_float4(S, Q, M, 0.f);
  }
}

// ---- wide decode (3..32 token rows, split-K): weights as the A operand -------
// The single-CTA kernel above puts the tokens on the MMA's M = 128 rows, so at
// decode widths of 3-32 rows 75-98 % of every MMA multiplies padding and the
// tensor pipe (fed at 8 KB of shared memory per MMA) becomes the limit: BLOOM
// batch 16 measured 77.6 % tensor-pipe active at 55 % of the HBM rate.  Here
// the operands swap: A = one 128-channel weight unit (the same core-matrix
// bytes, K-major), B = the NR token rows of the digit planes (N = NR = 16 or
// 32; the planes are digitised in NR-row core-matrix tiles, so a stage's rows
// are one contiguous copy per plane), D in
// TMEM with lane = output channel and column = token row.  Same exact integer
// products, same scaling and rounding sequence in the epilogue as
// epilogue_group / finish_tile, so the outputs are bit-identical to the
// single-CTA kernel's.  3 stages of 32 KB weights + NR KB of planes, two CTAs
// per SM; split-K over the int64 workspace as above.
template <int NR>
struct WideCfg {
  static constexpr int XU = NR * 32;                       // one plane unit: NR rows x 32 B
  static constexpr int W_BYTES = NGRP * KU * UNIT;         // 32 KB
  static constexpr int X_BYTES = 2 * KU * XU;
  static constexpr int STAGE = W_BYTES + X_BYTES;
  static constexpr int NST = 3;
  static constexpr int SMEM = NST * STAGE;
  static constexpr int TCOLS = 2 * NGRP * NR;              // D columns: (plane, group, row)
  static constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) |
                                    ((uint32_t)(NR >> 3) << 17) | ((128u >> 4) << 24);
};
static_assert(NGRP * 32 * 128 * 4 <= WideCfg<32>::SMEM && NGRP * 16 * 128 * 4 <= WideCfg<16>::SMEM,
              "the epilogue tile fits the drained stage ring");

__device__ __forceinline__ void mma_i8_id(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int NR, int EP>
__global__ void __launch_bounds__(256, 2) gemm_i8_wide_kernel(TcGemmArgs a) {
  using C = WideCfg<NR>;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[C::NST], empty[C::NST], tmem_full;
  __shared__ uint32_t tmem_base;
  __shared__ int last_cta;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ng0 = blockIdx.y * NGRP;
  const int64_t KT = a.K >> 5;
  const int KBT = (int)(KT / KU);
  const int S = a.ksplit > 1 ? a.ksplit : 1;
  const int kb0 = (int)((int64_t)blockIdx.z * KBT / S), kb1 = (int)((int64_t)(blockIdx.z + 1) * KBT / S);
  const int KB = kb1 - kb0;
  const int M = (int)a.M;                                  // <= NR

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)), "n"(C::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    const uint8_t* wb = reinterpret_cast<const uint8_t*>(a.w);
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % C::NST;
      if (kb >= C::NST) mbar_wait(&empty[s], ((kb / C::NST) - 1) & 1);
      uint8_t* st = smem + (size_t)s * C::STAGE;
      mbar_expect_tx(&full[s], C::STAGE);
      for (int j = 0; j < NGRP; ++j) {
        const int64_t ub = ((int64_t)(ng0 + j) * KT + (int64_t)(kb0 + kb) * KU) * UNIT;
        tma_load_1d(st + j * KU * UNIT, wb + ub, KU * UNIT, &full[s]);
      }
      // the planes are digitised with NR-row tiles (launch_digitize rt = NR):
      // a stage's KU units of one plane are KU * NR * 32 contiguous bytes
      for (int p = 0; p < 2; ++p)
        tma_load_1d(st + C::W_BYTES + p * KU * C::XU,
                    a.planes + p * a.plane_stride + (int64_t)(kb0 + kb) * KU * C::XU, KU * C::XU,
                    &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer: D[channel][row] += W . X^T ----------------
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % C::NST;
      mbar_wait(&full[s], (kb / C::NST) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint8_t* st = smem + (size_t)s * C::STAGE;
#pragma unroll
      for (int u = 0; u < KU; ++u)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const uint64_t bd = umma_desc(st + C::W_BYTES + (p * KU + u) * C::XU, NR * 16, 128);
#pragma unroll
          for (int j = 0; j < NGRP; ++j) {
            const uint64_t ad = umma_desc(st + j * KU * UNIT + u * UNIT, 2048, 128);
            mma_i8_id(tbase + (uint32_t)((p * NGRP + j) * NR), ad, bd, C::IDESC, (kb | u) ? 1u : 0u);
          }
        }
      mma_commit(&empty[s]);
    }
    mma_commit(&tmem_full);
  } else if (warp >= 4) {
    // ---------------- epilogue: thread = output channel ----------------
    const int q = warp - 4, ch = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    mbar_wait(&tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* tile = reinterpret_cast<float*>(smem);           // [NGRP][NR][128] (stages are drained)
    for (int j = 0; j < NGRP; ++j) {
      int d0[NR], d1[NR];
#pragma unroll
      for (int c = 0; c < NR; c += 16) {
        tmem_ld16_nw(tbase + lane_addr + (uint32_t)((0 * NGRP + j) * NR + c), d0 + c);
        tmem_ld16_nw(tbase + lane_addr + (uint32_t)((1 * NGRP + j) * NR + c), d1 + c);
      }
      tmem_wait_ld();
      const int64_t n = (int64_t)(ng0 + j) * 128 + ch;
      if (S == 1 && a.ys_rows) {                    // the decode GEMV's numerics
        const double wsc = (double)__ldg(a.wscale + n);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          if (r >= M) break;
          tile[(j * NR + r) * 128 + ch] =
              (float)((double)((long long)d0[r] * 256 + d1[r]) * a.ys_rows[r] * wsc);
        }
      } else if (S == 1) {
        const float wsc = __ldg(a.wscale + n);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          if (r >= M) break;
          const float ys = ldexpf(1.0f, a.exps[r] - 14);
          tile[(j * NR + r) * 128 + ch] =
              __fmul_rn(__fmul_rn((float)((long long)d0[r] * 256 + d1[r]), ys), wsc);
        }
      } else {
        unsigned long long* ws = reinterpret_cast<unsigned long long*>(a.ws);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          if (r >= M) break;
          atomicAdd(ws + (int64_t)r * a.N + n, (unsigned long long)((long long)d0[r] * 256 + d1[r]));
        }
      }
    }
    if (S == 1 && a.ys_rows) {
      asm volatile("bar.sync 1, 128;" ::: "memory");       // the 4 epilogue warps
      for (int pr = q; pr < NGRP * M; pr += 4) {
        const int j = pr / M, r = pr % M;
        gemv_epilogue_group(a, ng0 + j, r, lane,
                            [&](int c) { return tile[(j * NR + r) * 128 + c]; });
      }
    } else if (S == 1) {
      asm volatile("bar.sync 1, 128;" ::: "memory");       // the 4 epilogue warps
      const int t = threadIdx.x - 128;
      const int epi = EP >= 0 ? EP : a.epi;
      if (epi == EPI_SWIGLU) {
        for (int i = t; i < NGRP * M * 64; i += 128) {
          const int j = i / (M * 64), r = (i / 64) % M, c = i % 64;
          const float gd = tile[(j * NR + r) * 128 + c], ud = tile[(j * NR + r) * 128 + 64 + c];
          a.y[(int64_t)r * a.ldy + (ng0 + j) * 64 + c] =
              __fmul_rn(__fdividef(gd, __fadd_rn(1.0f, __expf(-gd))), ud);
        }
      } else {
        for (int i = t; i < NGRP * M * 128; i += 128) {
          const int j = i / (M * 128), r = (i / 128) % M, c = i % 128;
          const int64_t col = (int64_t)(ng0 + j) * 128 + c;
          float v = tile[(j * NR + r) * 128 + c];
          if (epi == EPI_RESID) v = __fadd_rn(v, a.res[(int64_t)r * a.ldy + col]);
          else if (epi == EPI_GELU) v = gelu_f(v);
          a.y[(int64_t)r * a.ldy + col] = v;
        }
      }
    } else {
      __threadfence();
    }
  }
  if (S > 1) {
    __syncthreads();
    if (threadIdx.x == 0) {
      int* cnt = a.counters + blockIdx.y;
      const int old = atomicAdd(cnt, 1);
      last_cta = (old == S - 1);
      if (last_cta) { __threadfence(); *cnt = 0; }
    }
    __syncthreads();
    if (last_cta) {
      if (a.ys_rows) {
        // the decode GEMV's epilogue on the summed int64 workspace (zeroed after)
        for (int pr = warp; pr < NGRP * M; pr += 8) {
          const int j = pr / M, r = pr % M;
          const int64_t n0 = (int64_t)(ng0 + j) * 128;
          long long* wr = a.ws + (int64_t)r * a.N + n0;
          const double ys = a.ys_rows[r];
          gemv_epilogue_group(a, ng0 + j, r, lane, [&](int c) {
            return (float)((double)__ldcg(wr + c) * ys * (double)__ldg(a.wscale + n0 + c));
          });
          __syncwarp();
          for (int c = lane; c < 128; c += 32) wr[c] = 0;
        }
      } else {
        finish_tile(a, 0, ng0);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TCOLS)
                 : "memory");
}

template <int NR, int EP>
void launch_wide_t(const TcGemmArgs& b, dim3 grid, cudaStream_t st) {
  static bool set[kMaxDevices] = {};
  const int dv = current_device();
  if (!set[dv]) {
    cudaFuncSetAttribute(gemm_i8_wide_kernel<NR, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         WideCfg<NR>::SMEM);
    set[dv] = true;
  }
  gemm_i8_wide_kernel<NR, EP><<<grid, 256, WideCfg<NR>::SMEM, st>>>(b);
}

template <int NR>
void launch_wide_nr(const TcGemmArgs& b, dim3 grid, cudaStream_t st) {
  switch (b.epi) {
    case EPI_STORE: launch_wide_t<NR, EPI_STORE>(b, grid, st); break;
    case EPI_RESID: launch_wide_t<NR, EPI_RESID>(b, grid, st); break;
    case EPI_SWIGLU: launch_wide_t<NR, EPI_SWIGLU>(b, grid, st); break;
    default: launch_wide_t<NR, EPI_GELU>(b, grid, st); break;
  }
}

bool g_tc_wide = getenv("SP_TC_WIDE") ? atoi(getenv("SP_TC_WIDE")) != 0 : true;

void launch_digitize_gemv(const float* x, int64_t ldx, int64_t M, int64_t K, int norm,
                          const float* g, const float4* st_in, int P_in, float gmax, float eps,
                          uint8_t* planes, int64_t plane_stride, double* ys_rows, int rt,
                          cudaStream_t st) {
  const dim3 grid((unsigned)((K / 16 + 255) / 256), (unsigned)M);
  digitize_gemv_kernel<<<grid, 256, 0, st>>>(x, ldx, M, K, norm, g, st_in, P_in, gmax, eps,
                                             planes, plane_stride, ys_rows, rt);
  count_launch();
}

int wide_rows(int64_t M) {
  if (!g_tc_wide) return 0;
  return M <= 16 ? 16 : (M <= 32 ? 32 : 0);
}

template <bool BF, int EP>
void launch_single_t(const TcGemmArgs& b, dim3 grid, cudaStream_t st) {
  static bool set[kMaxDevices] = {};
  const int dv = current_device();
  const size_t smem = (size_t)STAGES * STAGE;
  if (!set[dv]) {
    cudaFuncSetAttribute(gemm_i8_tc_kernel<BF, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    set[dv] = true;
  }
  gemm_i8_tc_kernel<BF, EP><<<grid, 256, smem, st>>>(b);
}

// one instantiation per (operand type, epilogue), like the pair kernel
void launch_single(const TcGemmArgs& b, dim3 grid, cudaStream_t st) {
  auto go = [&](auto bfc) {
    constexpr bool B = decltype(bfc)::value;
    switch (b.epi) {
      case EPI_STORE: launch_single_t<B, EPI_STORE>(b, grid, st); break;
      case EPI_RESID: launch_single_t<B, EPI_RESID>(b, grid, st); break;
      case EPI_SWIGLU: launch_single_t<B, EPI_SWIGLU>(b, grid, st); break;
      default: launch_single_t<B, EPI_GELU>(b, grid, st); break;
    }
  };
  if (b.bf16) go(std::true_type{});
  else go(std::false_type{});
}

void launch_gemm_i8_tc(const TcGemmArgs& a, cudaStream_t st) {
  // up to 128 tokens (wide decode, short prompts): one 128-token tile per CTA
  // does half the padded MMA work of a 256-token pair tile
  if (g_tc_pair && a.M > 128) {
    // (stage shapes measured: 4 units x 4 stages beats 2 x 8 by 35 % and 8 x 2 by 5 %)
    // one instantiation per (operand type, epilogue): each kernel carries only
    // its own epilogue's code (the GELU variant alone is ~12 KB of SASS)
    auto go = [&](auto bfc) {
      constexpr bool B = decltype(bfc)::value;
      switch (a.epi) {
        case EPI_STORE: launch_pair<4, 4, B, EPI_STORE>(a, st); break;
        case EPI_RESID: launch_pair<4, 4, B, EPI_RESID>(a, st); break;
        case EPI_SWIGLU: launch_pair<4, 4, B, EPI_SWIGLU>(a, st); break;
        default: launch_pair<4, 4, B, EPI_GELU>(a, st); break;
      }
    };
    if (a.bf16) go(std::true_type{});
    else go(std::false_type{});
    return;
  }
  if (!a.bf16 && a.ws && a.counters && wide_rows(a.M)) {
    // wide decode: weights on the MMA's M side (gemm_i8_wide_kernel); split K
    // as far as every CTA stays resident (two per SM): no second wave
    TcGemmArgs b = a;
    const int tiles = (int)(a.N / (128 * NGRP));
    const int kbt = (int)(a.K / 32 / KU);
    int S = (2 * 148) / tiles;                // every CTA resident at once (2 per SM)
    if (S > kbt / 4) S = kbt / 4;
    if (S < 1) S = 1;
    b.ksplit = S;
    const dim3 grid(1u, (unsigned)tiles, (unsigned)S);
    if (wide_rows(a.M) == 16) launch_wide_nr<16>(b, grid, st);
    else launch_wide_nr<32>(b, grid, st);
    count_launch();
    return;
  }
  TcGemmArgs b = a;
  const int tiles = (int)(((a.M + BM - 1) / BM) * (a.N / (128 * NGRP)));
  const int kbt = (int)(a.K / 32 / KU);
  int S = 1;
  if (a.ws && a.counters && tiles < 148 && !a.bf16) {   // few-token GEMM: fill the SMs along K
    S = (148 + tiles / 2) / tiles;
    if (S > kbt / 4) S = kbt / 4;
    if (S < 1) S = 1;
  }
  b.ksplit = S;
  dim3 grid((unsigned)((a.M + BM - 1) / BM), (unsigned)(a.N / (128 * NGRP)), (unsigned)S);
  launch_single(b, grid, st);
  count_launch();
}

int64_t tc_plane_bytes(int64_t M, int64_t K) { return tc_rows(M) * K; }

void launch_digitize_bf16(const float* x, int64_t ldx, int64_t M, int64_t K, int norm,
                          const float* g, const float* b, uint8_t* planes, int64_t plane_stride,
                          cudaStream_t st) {
  const unsigned grid = (unsigned)M;
  if (K <= 256 * 8 * 4)
    digitize_bf16_kernel<256, 4><<<grid, 256, 0, st>>>(x, ldx, M, K, norm, g, b, planes, plane_stride);
  else
    digitize_bf16_kernel<512, 4><<<grid, 512, 0, st>>>(x, ldx, M, K, norm, g, b, planes, plane_stride);
  count_launch();
}

}  // namespace sp
