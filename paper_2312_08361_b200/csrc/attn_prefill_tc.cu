// Prefill / replay causal attention (n_new > 1) on the 5th-gen tensor cores:
// tcgen05.mma with both A operands (Q, P) and both accumulators (S, O) in TMEM,
// K / V pages brought in by tensor-map TMA (bf16 KV cache, head dim 128).
//
// SP/model.py:263-275: scores = q . k / sqrt(hd) (+ ALiBi), causal mask for
// n > 1 (the reference fills -1e30; here -inf, identical after the
// max-subtracted exp), softmax over cache + new positions, ctx = p . v.
//
// CTA = (slot, query head, 128 query rows); keys stream 128 positions (two
// pages) per tile.  Warp roles (10 warps):
//   * warps 0-7  softmax / epilogue: TMEM lane = query row; the two warps of a
//                lane quarter split every tile's columns (64 scores, 64 output
//                dims each) and combine the row maxima through shared memory.
//                Q arrives pre-scaled by log2(e)/sqrt(hd), so the scores leave
//                the MMA in the exp2 domain.  Per tile: tcgen05.ld the scores,
//                ALiBi / causal mask (diagonal tiles only), max tree, exp2,
//                P (bf16) -> TMEM with tcgen05.st.  The output accumulates in
//                TMEM across tiles and is rescaled (tcgen05.ld / st) only when
//                a row's maximum grows by more than 2^8 over the one its P
//                values are normalised to (p <= 256).  At the end ctx = O / l.
//   * warp 8     producer: one lane issues each tile's K and V pages as 2-D
//                tensor-map TMA loads (cp.async.bulk.tensor, 128-byte swizzle,
//                [64 keys][64 dims] boxes) from the paged pool: K lands in the
//                K-major SW128 layout (B operand of S = Q K^T), V in the MN-major
//                SW128 layout (B operand of O = P V).  3 stages of 64 KB.
//   * warp 9     TMEM allocator + one elected lane issuing the MMAs:
//                S_j = (Qhi + Qlo) K_j^T  (M = 128, N = 128, K = 128; A in TMEM)
//                O  += P_j V_j            (M = 128, N = 128, K = 128; A in TMEM)
//                S_{j+1} is issued as soon as the softmax has read S_j out, so
//                the tensor pipe computes the next scores while the softmax
//                warps turn S_j into P_j.
// TMEM (512 columns): Q hi/lo 128, S 128, P 2 x 64 (double buffered), O 128.
// Q is split hi + lo bf16 (two MMAs) against the bf16 K cache, so the scores
// carry the cache's rounding, not a bf16 rounding of q; P (in [0, 256]) is
// bf16 with f32 accumulation.
// Each query row depends only on its own row: batch / tile invariant.
// Measured (profiles/r02_attn_pf.md): 173 us for 2048 tokens of one 70B block.
#include <cuda.h>   // CUtensorMap (the encoder is fetched from the driver at run time)

#include <array>
#include <cstdio>
#include <cstdlib>
#include <list>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "kernels.cuh"

namespace sp {

bool g_attn_tc = getenv("SP_ATTN_TC") ? atoi(getenv("SP_ATTN_TC")) != 0 : true;  // option 8

namespace {

constexpr int HD = 128;
constexpr int BQ = 128;                 // query rows per CTA
constexpr int BK = 128;                 // keys per tile (two pages)
constexpr int NSM = 8;                  // softmax warps: 2 per TMEM lane quarter
constexpr int NTHREADS = (NSM + 2) * 32;
constexpr int WP = NSM, WM = NSM + 1;   // producer warp, MMA warp
constexpr int K_BYTES = BK * HD * 2;    // 16 KB
constexpr int V_BYTES = BK * HD * 2;    // 16 KB
constexpr int STAGE_BYTES = K_BYTES + V_BYTES;
constexpr int NST = 3;                  // K/V stages
constexpr int BOX = kPageTokens * 64 * 2;   // one [64 keys][64 dims] TMA box (8 KB)
constexpr int HALF = BK * 128;          // one 64-dim half of a tile: [128 keys][128 B]
constexpr int SMEM_BYTES = NST * STAGE_BYTES + 1024;
// TMEM columns (32-bit): the A operands live in TMEM (one column = 2 bf16 of
// a row): Q hi 0..63, Q lo 64..127; S 128 (one tile, read out before the next
// is issued); P 2 x 64; O 128
constexpr int Q_COL = 0;
constexpr int S_COL = 128;
constexpr int P_COL = 256;
constexpr int O_COL = 384;
constexpr float kRescale = 8.0f;        // log2 growth of a row max that forces an O rescale
constexpr float kLog2e = 1.4426950408889634f;

// instruction descriptors (kind::f16: bf16 A/B, f32 D)
constexpr int SN = BK;                  // N of one score MMA (128 keys)
constexpr uint32_t kIdescS = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(SN >> 3) << 17) |
                             ((uint32_t)(BQ >> 4) << 24);                       // K-major B
constexpr uint32_t kIdescO = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                             ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(BQ >> 4) << 24);  // MN-major B

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor, version 1):
// layout 0 = SWIZZLE_NONE, 2 = SWIZZLE_128B (atoms 1024-byte aligned)
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo,
                                          uint32_t layout = 0) {
  uint64_t d = (uint64_t)((su32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
// A operand from TMEM (row = lane, K packed two bf16 per 32-bit column)
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                        uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(b))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t bf2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// debug (SP_BUILD_TRACE=1 build + SP_ATTN_PF_TRACE=1): per-phase clock sums of
// softmax warp 0 and the MMA lane of CTA (0, 0), printed by the launcher
__device__ unsigned long long g_pf_trace[16];
#define PF_T(slot, t0) \
  do { if (SP_DEV_TRACE && blockIdx.x == 0 && blockIdx.y == 0) { \
    const unsigned long long t_ = clock64(); pf_acc[slot] += t_ - (t0); (t0) = t_; } } while (0)

__global__ void __launch_bounds__(NTHREADS, 1)
attn_prefill_tc_kernel(AttnArgs a, const __grid_constant__ CUtensorMap kvmap, int64_t row0) {
  unsigned long long pf_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned long long pf_t = SP_DEV_TRACE ? clock64() : 0;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128-byte-swizzled TMA boxes / UMMA atoms
  uint8_t* smem = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  uint8_t* stages = smem;                                      // [NST][K box0 box1 | V box0 box1]
  __shared__ __align__(8) uint64_t kv_full[NST], kv_empty[NST], s_full, s_free, p_full[2],
      p_free[2], o_full, q_full;
  __shared__ uint32_t tmem_base;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.H / a.kvh;
  const int slot = blockIdx.x / a.H, h = blockIdx.x % a.H, kh = h / G;
  const int q0 = (gridDim.y - 1 - blockIdx.y) * BQ;          // heaviest tiles first
  const int last_q = min(q0 + BQ, a.n_new) - 1;
  const int ntiles = (a.t0 + last_q + 1 + BK - 1) / BK;

  // softmax warps: this row's 64 q values are loaded first of all, so their
  // latency overlaps the barrier / TMEM set-up and the first K/V loads
  float4 qv[16];
  if (warp < NSM) {
    const int row_ = (warp & 3) * 32 + lane;
    const int qi_ = min(q0 + row_, a.n_new - 1);
    const float* qsrc = a.qkv + (int64_t)(slot * a.n_new + qi_) * a.ldqkv + h * HD + (warp >> 2) * 64;
#pragma unroll
    for (int c = 0; c < 16; ++c) qv[c] = __ldcs(reinterpret_cast<const float4*>(qsrc + c * 4));
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(&s_full, 1);
    mbar_init(&s_free, NSM);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[i], NSM);
      mbar_init(&p_free[i], 1);
    }
    mbar_init(&o_full, 1);
    mbar_init(&q_full, NSM);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == WM) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;

  if (warp == WP) {
    // ---------------- producer: K / V pages by tensor-map TMA ----------------
    if (lane == 0) {
      for (int j = 0; j < ntiles; ++j) {
        const int st = j % NST;
        if (j >= NST) mbar_wait(&kv_empty[st], ((j / NST) - 1) & 1);
        uint8_t* Ks = stages + st * STAGE_BYTES;
        uint8_t* Vs = Ks + K_BYTES;
        mbar_expect_tx(&kv_full[st], STAGE_BYTES);
        // two pages; a tile's key rows 64p.. of dim half d at d * HALF + p * BOX
        // (beyond the table: page 0, whose finite rows the causal mask discards)
        for (int p = 0; p < BK / kPageTokens; ++p) {
          const int pi = (BK / kPageTokens) * j + p;
          const int page = pi < a.max_pages ? a.page_table[slot * a.max_pages + pi] : 0;
          // rows of the pool viewed as [(page, K|V, kv head, key)][hd]
          const int64_t rk = row0 + (((int64_t)page * 2 + 0) * a.kvh + kh) * kPageTokens;
          const int64_t rv = rk + (int64_t)a.kvh * kPageTokens;
          tma_2d(Ks + p * BOX, &kvmap, 0, (int)rk, &kv_full[st]);
          tma_2d(Ks + HALF + p * BOX, &kvmap, 64, (int)rk, &kv_full[st]);
          tma_2d(Vs + p * BOX, &kvmap, 0, (int)rv, &kv_full[st]);
          tma_2d(Vs + HALF + p * BOX, &kvmap, 64, (int)rv, &kv_full[st]);
        }
      }
    }
    __syncwarp();
  } else if (warp == WM) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      mbar_wait(&q_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      auto issue_s = [&](int j) {
        const int kst = j % NST;
        mbar_wait(&kv_full[kst], (j / NST) & 1);
        PF_T(3, pf_t);
        if (j >= 1) mbar_wait(&s_free, (j - 1) & 1);   // S_{j-1} read out
        PF_T(4, pf_t);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* Ks = stages + kst * STAGE_BYTES;
        const uint32_t d = tb + S_COL;
#pragma unroll
        for (int u = 0; u < HD / 16; ++u) {
          // K-major SW128: 16 dims = 32 bytes along the 128-byte swizzle atom row;
          // dims 64..127 are the second half; 8-key groups 1024 bytes apart.
          // A = Q hi / lo from TMEM: 16 dims = 8 columns
#pragma unroll
          for (int n = 0; n < BK / SN; ++n) {
            const uint64_t bd =
                sdesc(Ks + (u >> 2) * HALF + n * (SN * 128) + (u & 3) * 32, 16, 1024, 2);
            umma_ts(d + n * SN, tb + Q_COL + u * 8, bd, kIdescS, u > 0);
            umma_ts(d + n * SN, tb + Q_COL + 64 + u * 8, bd, kIdescS, 1);
          }
        }
        umma_commit(&s_full);
      };
      auto issue_o = [&](int j) {
        const int kst = j % NST, st = j & 1;
        mbar_wait(&p_full[st], (j >> 1) & 1);    // P_j written (and any O rescale done)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* Vs = stages + kst * STAGE_BYTES + K_BYTES;
#pragma unroll
        for (int u = 0; u < BK / 16; ++u)
          // MN-major SW128: 64 dims per 128-byte atom row, the second 64 dims one
          // box (LBO) further; 16 keys = 2 groups of 8 rows, 1024 bytes apart (SBO).
          // A = P_j from TMEM: 16 keys = 8 columns
          umma_ts(tb + O_COL, tb + P_COL + st * (BK / 2) + u * 8,
                  sdesc(Vs + u * 2048, HALF, 1024, 2), kIdescO, (j | u) ? 1u : 0u);
        umma_commit(&o_full);                    // O now holds tiles 0..j
        umma_commit(&p_free[st]);                // P buffer st read
        umma_commit(&kv_empty[kst]);             // K_j and V_j consumed
      };
      PF_T(0, pf_t);
      issue_s(0);
      PF_T(1, pf_t);
      for (int j = 0; j < ntiles; ++j) {
        if (j + 1 < ntiles) issue_s(j + 1);
        PF_T(1, pf_t);
        issue_o(j);
        PF_T(2, pf_t);
      }
      if (SP_DEV_TRACE && blockIdx.x == 0 && blockIdx.y == 0)
        for (int i = 0; i < 5; ++i) g_pf_trace[8 + i] = pf_acc[i];
    }
    __syncwarp();
  } else {
    // ---------------- softmax / epilogue ----------------
    // warp w: query rows (TMEM lanes) 32*(w%4) + lane, column half hf = w/4 of
    // every tile (scores 32*hf.., output dims 64*hf..); the two warps of a row
    // combine their tile maxima through shared memory (named barrier per pair)
    __shared__ float red_max[2][BQ][2];
    __shared__ float red_l[BQ];
    const int quarter = warp & 3, hf = warp >> 2;
    const int row = quarter * 32 + lane;
    const int qpos = a.t0 + q0 + row;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    auto pair_sync = [&]() {
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    };
    // Q row (this warp's 64 dims), pre-scaled by log2(e) / sqrt(hd) (scores come
    // out of the MMA in the exp2 domain), -> hi / lo bf16 pairs in TMEM (the A
    // operand of S = Q K^T: row = lane, column c = dims 2c, 2c + 1)
    const float qscale = kLog2e / sqrtf((float)HD);
    {
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float x[4] = {qv[c].x * qscale, qv[c].y * qscale, qv[c].z * qscale,
                            qv[c].w * qscale};
        float hh[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) hh[i] = __bfloat162float(__float2bfloat16_rn(x[i]));
        hi[2 * c] = bf2(hh[0], hh[1]);
        hi[2 * c + 1] = bf2(hh[2], hh[3]);
        lo[2 * c] = bf2(x[0] - hh[0], x[1] - hh[1]);
        lo[2 * c + 1] = bf2(x[2] - hh[2], x[3] - hh[3]);
      }
      tmem_st16(tb + lane_addr + Q_COL + hf * 32, hi);
      tmem_st16(tb + lane_addr + Q_COL + hf * 32 + 16, hi + 16);
      tmem_st16(tb + lane_addr + Q_COL + 64 + hf * 32, lo);
      tmem_st16(tb + lane_addr + Q_COL + 64 + hf * 32 + 16, lo + 16);
      tmem_wait_st();
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_full);
    }
    const float slope_l2 = (a.family == kBloom) ? a.alibi[h] * kLog2e : 0.f;
    constexpr int SC = BK / 2;                   // score columns per warp
    constexpr int OC = HD / 2;                   // output columns per warp
    float m_used = -INFINITY, l_run = 0.f;       // P_j = exp2(s - m_used); l in the same units
    PF_T(7, pf_t);
    for (int j = 0; j < ntiles; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full, j & 1);
      PF_T(0, pf_t);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float s[SC];
      tmem_ld32(tb + lane_addr + S_COL + hf * SC, s);
      if constexpr (SC > 32) tmem_ld32(tb + lane_addr + S_COL + hf * SC + 32, s + 32);
      tmem_wait_ld();
      PF_T(1, pf_t);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free);
      // ALiBi, causal mask (diagonal tiles only), tile max as a 3-input tree
      const int kbase = j * BK + hf * SC;
      const bool unmasked = j * BK + BK - 1 <= a.t0 + q0;   // every row sees every key
      if (a.family == kBloom) {
#pragma unroll
        for (int i = 0; i < SC; ++i) s[i] = fmaf(slope_l2, (float)(kbase + i - qpos), s[i]);
      }
      if (!unmasked) {
#pragma unroll
        for (int i = 0; i < SC; ++i) s[i] = (kbase + i > qpos) ? -INFINITY : s[i];
      }
      float mx[SC / 4];
#pragma unroll
      for (int i = 0; i < SC / 4; ++i)
        mx[i] = fmaxf(fmaxf(s[4 * i], s[4 * i + 1]), fmaxf(s[4 * i + 2], s[4 * i + 3]));
#pragma unroll
      for (int w = SC / 8; w >= 1; w >>= 1)
#pragma unroll
        for (int i = 0; i < w; ++i) mx[i] = fmaxf(mx[i], mx[i + w]);
      float tmax = mx[0];
      PF_T(2, pf_t);
      red_max[st][row][hf] = tmax;
      pair_sync();
      tmax = fmaxf(red_max[st][row][0], red_max[st][row][1]);
      PF_T(3, pf_t);
      // O rescale only when the row's max outgrows its reference by 2^8
      // (warp-uniform: tcgen05.ld/st are warp-collective; factor 1 elsewhere)
      float mnew = m_used;
      if (j == 0) mnew = tmax;
      else if (tmax > m_used + kRescale) mnew = tmax;
      const bool grow = j > 0 && mnew != m_used;
      // P buffer st free = O_{j-2} complete: also bounds o_full's phase below
      if (j >= 2) mbar_wait(&p_free[st], ((j >> 1) - 1) & 1);
      if (__any_sync(0xffffffffu, grow)) {
        const float f = grow ? ex2_approx(m_used - mnew) : 1.f;
        mbar_wait(&o_full, (j - 1) & 1);         // O holds tiles 0..j-1
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int c = 0; c < OC / 32; ++c) {
          float v[32];
          tmem_ld32(tb + lane_addr + O_COL + hf * OC + c * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= f;
          tmem_st32(tb + lane_addr + O_COL + hf * OC + c * 32, v);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        l_run *= f;
      }
      m_used = mnew;
      // P_j = exp2(s - m_used) (<= 2^8), bf16, -> TMEM buffer st, once the MMA
      // of tile j - 2 has read it
      PF_T(4, pf_t);
      PF_T(5, pf_t);
      // p = exp2(s - m) (ex2.approx.ftz(-inf) = +0: masked keys need no test);
      // four partial sums for instruction-level parallelism
      // (paired f32 arithmetic, FADD2: the softmax warps are issue-bound)
      uint64_t acc2[4] = {0, 0, 0, 0};
      uint32_t pk[SC / 2];
      uint64_t mm;
      asm("mov.b64 %0, {%1, %1};" : "=l"(mm) : "f"(m_used));
#pragma unroll
      for (int i = 0; i < SC; i += 2) {
        uint64_t x2, d2;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x2) : "f"(s[i]), "f"(s[i + 1]));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d2) : "l"(x2), "l"(mm));
        float d0, d1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d2));
        const float p0 = ex2_approx(d0);
        const float p1 = ex2_approx(d1);
        uint64_t p2;
        asm("mov.b64 %0, {%1, %2};" : "=l"(p2) : "f"(p0), "f"(p1));
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc2[(i >> 1) & 3]) : "l"(p2));
        pk[i / 2] = bf2(p0, p1);
      }
      float psum;
      {
        uint64_t t01, t23, t;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t01) : "l"(acc2[0]), "l"(acc2[1]));
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t23) : "l"(acc2[2]), "l"(acc2[3]));
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(t01), "l"(t23));
        float a0, a1;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(t));
        psum = a0 + a1;
      }
      // P_j -> TMEM (A operand of O += P V): this warp's 64 keys = 32 columns
      tmem_st16(tb + lane_addr + P_COL + st * (BK / 2) + hf * (SC / 2), pk);
      if constexpr (SC / 2 > 16)
        tmem_st16(tb + lane_addr + P_COL + st * (BK / 2) + hf * (SC / 2) + 16, pk + 16);
      tmem_wait_st();
      l_run += psum;
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[st]);
      PF_T(6, pf_t);
    }
    if (SP_DEV_TRACE && blockIdx.x == 0 && blockIdx.y == 0 && warp == 0 && lane == 0) {
      for (int i = 0; i < 8; ++i) g_pf_trace[i] = pf_acc[i];
      g_pf_trace[15] = ntiles;
    }
    // ---- ctx row = O / l  (l = the two halves' sums, same units) ----
    if (hf == 1) red_l[row] = l_run;
    pair_sync();
    if (hf == 0) red_l[row] += l_run;
    pair_sync();
    const float inv = __frcp_rn(red_l[row]);
    // every O MMA done = the last tile's P buffer released (one phase past the
    // one waited at that tile: an unambiguous parity wait)
    mbar_wait(&p_free[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* dst = a.ctx + (int64_t)(slot * a.n_new + q0 + row) * a.H * HD + h * HD + hf * OC;
#pragma unroll
    for (int c = 0; c < OC / 32; ++c) {
      float v[32];
      tmem_ld32(tb + lane_addr + O_COL + hf * OC + c * 32, v);
      tmem_wait_ld();
      if (q0 + row < a.n_new) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + c * 32 + i) =
              make_float4(v[i] * inv, v[i + 1] * inv, v[i + 2] * inv, v[i + 3] * inv);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == WM)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

}  // namespace

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
}  // namespace

// one 2-D tensor map per (KV pool, head dim, box rows): rows = (block, page,
// K|V, kv head, key), cols = hd; boxes of [box_rows keys][64 dims], 128-byte
// swizzle (prefill attention: a page per box; decode attention: 32 keys)
const CUtensorMap* kv_pool_map(const void* base, int64_t bytes, int hd, int box_rows) {
  static std::mutex mu;
  // std::list: the returned pointers stay valid as further maps are added
  static std::unordered_map<const void*, std::list<std::pair<std::array<int64_t, 3>,
                                                              CUtensorMap>>> maps;
  static EncodeTiledFn encode = nullptr;
  std::lock_guard<std::mutex> g(mu);
  auto& v = maps[base];
  for (auto& e : v)
    if (e.first[0] == bytes && e.first[1] == hd && e.first[2] == box_rows) return &e.second;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || !fn)
      return nullptr;
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  CUtensorMap m;
  const cuuint64_t dims[2] = {(cuuint64_t)hd, (cuuint64_t)(bytes / (hd * 2))};
  const cuuint64_t strides[1] = {(cuuint64_t)hd * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  if (encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return nullptr;
  v.push_back({{bytes, hd, box_rows}, m});
  return &v.back().second;
}

bool launch_attention_prefill_tc(const AttnArgs& a, cudaStream_t st) {
  if (!g_attn_tc || a.kv_dtype != kKVBF16 || a.hd != HD || !a.pool_base) return false;
  const CUtensorMap* map = kv_pool_map(a.pool_base, a.pool_bytes, HD, kPageTokens);
  if (!map) return false;
  static bool set[kMaxDevices] = {};
  const int dv = current_device();
  if (!set[dv]) {
    cudaFuncSetAttribute(attn_prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SMEM_BYTES);
    set[dv] = true;
  }
  const int64_t row0 = ((const char*)a.kv_pool - (const char*)a.pool_base) / (HD * 2);
  dim3 grid(a.width * a.H, (a.n_new + BQ - 1) / BQ);
  attn_prefill_tc_kernel<<<grid, NTHREADS, SMEM_BYTES, st>>>(a, *map, row0);
  count_launch();
  static const bool tr = SP_DEV_TRACE && getenv("SP_ATTN_PF_TRACE");
  if (tr) {
    unsigned long long h[16];
    cudaMemcpyFromSymbolAsync(h, g_pf_trace, sizeof(h), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "attn_pf_tc CTA(0,0) ntiles=%llu softmax clocks: s_wait %llu ld %llu "
            "scale %llu pair %llu rescale %llu p_free %llu exp_st %llu qload %llu | mma: "
            "prologue %llu issue_s %llu issue_o(wait P) %llu kv_full %llu s_free %llu\n", h[15],
            h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9], h[10], h[11], h[12]);
  }
  return true;
}

}  // namespace sp
