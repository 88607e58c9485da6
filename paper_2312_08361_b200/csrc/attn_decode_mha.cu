// Decode attention for multi-head attention (one query head per kv head:
// BLOOM-176B, Llama-2-7B shapes), every width — built for the batched decode
// of SURVEY.md C3 (batch 16: thousands of (row, head) pairs).  HBM-bound.
//
// SP/model.py:263-275 at n = 1: scores = q . k / sqrt(hd) (+ ALiBi), no mask,
// max-subtracted softmax, ctx = p . v; the new position's k (RoPE'd) and v are
// appended to the paged cache first (KVCache.append, SP/model.py:163-167).
//
// With one query row per kv head the products are matrix-vector: 2 flops per
// cached element, so the K/V bytes (2 * T * hd * 2 per pair) bound the kernel
// and no tensor-core tile is needed (the MMA kernel pads the single head to an
// 8-column tile and stages 64 KB sub-chunks through shared memory, which kept
// it at 57 % of HBM bandwidth with one CTA per SM).  Here:
//   * one CTA of 4 warps per (row, head, chunk); warp w takes the chunk's
//     32-position blocks w, w + 4, ...; all of a block's K rows (8 lanes per
//     row, 4 rows per load instruction: whole 128-byte lines) and V rows (lane
//     = 4 dims, one row per instruction) are loaded with streaming hints before
//     any arithmetic — 16 KB in flight per warp, 3 CTAs per SM — and the next
//     block is prefetched into L2 under this one's arithmetic;
//   * f32 q (RoPE at t0) in registers, f32 FMA dot products reduced over 8
//     lanes by shuffles, online softmax in the exp2 domain per warp, P
//     broadcast by shuffles into the P.V accumulation;
//   * the 4 warp partials merge in a fixed order; ctx and the head's (sum,
//     sumsq, max|x|) partial for the O-projection GEMV are written once.
// Bytes per launch: K+V of the visible positions (2 * T * H * hd * 2) + q/ctx.
// A (row, head) pair's positions are cut into chunks of a size that depends on
// the sequence length only (mha_chunk: >= T/16, 128..1024), one CTA each; with
// several chunks the last-arriving CTA merges the chunk partials in ascending
// order.  So a row's arithmetic is the same at every width (batch invariant)
// and batch 1 still spreads over up to 16 CTAs per head.
#include <cstdint>

#include "common.cuh"
#include "decode.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr int HD = 128;
constexpr int NW = 4;                  // warps per CTA
constexpr float kLog2e = 1.4426950408889634f;

// streaming loads (read once: evict-first in L2, no L1 allocation)
__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  return __ldcs(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ uint2 ld_stream8(const void* p) {
  return __ldcs(reinterpret_cast<const uint2*>(p));
}
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ float lo_bf(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_bf(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ float rope_at(const float* x, int dd, int half, const float* cs,
                                         const float* sn) {
  const int j = dd % half;
  const float c = cs[j], s = sn[j];
  return dd < half ? __fsub_rn(__fmul_rn(x[j], c), __fmul_rn(x[j + half], s))
                   : __fadd_rn(__fmul_rn(x[j + half], c), __fmul_rn(x[j], s));
}

// positions per CTA: a power of two >= T/div in [128, 1024] — a function of the
// sequence length only, so a row's arithmetic never depends on the step's width
__host__ __device__ __forceinline__ int mha_chunk(int T, int div) {
  int ch = 128;
  while (ch < 1024 && div * ch < T) ch *= 2;
  return ch;
}

__global__ void __launch_bounds__(NW * 32, 3) attn_dec_mha_kernel(AttnDecArgs a, int div) {
  __shared__ __align__(16) float qs[HD];
  __shared__ __align__(16) float wo[NW][HD];
  __shared__ float wm[NW], wl[NW], cf[32];
  __shared__ float red[3][NW];
  __shared__ int last;
  const int slot = blockIdx.x / a.kvh, kh = blockIdx.x % a.kvh;   // one query head: h = kh
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = a.t0 + 1;
  const int CH = mha_chunk(T, div);
  const int nchunk = (T + CH - 1) / CH;
  const int chunk = blockIdx.y;
  if (chunk >= nchunk) return;
  const int half = HD / 2;
  const int* ptab = a.page_table + slot * a.max_pages;
  const __nv_bfloat16* pool = reinterpret_cast<const __nv_bfloat16*>(a.kv_pool);
  const int b0 = chunk * (CH / 32), b1 = min((chunk + 1) * (CH / 32), (T + 31) / 32);
  auto block_k = [&](int b) {          // K rows of 32-position block b (V follows kvh pages on)
    const int page = ptab[(b * 32) / kPageTokens];
    return pool + (((int64_t)page * 2 + 0) * a.kvh + kh) * kPageTokens * HD +
           ((b * 32) % kPageTokens) * HD;
  };
  // before the dependency wait (page tables and cached rows are not written by
  // the kernels of this chain; L2 is coherent with the append below): the
  // warp's first two K/V blocks stream into L2 under the QKV projection's tail
  if (lane == 0)
    for (int b = b0 + warp, n = 0; b < b1 && n < 2; b += NW, ++n) {
      const __nv_bfloat16* kb = block_k(b);
      l2_prefetch(kb, 32 * HD * 2);
      l2_prefetch(kb + (int64_t)a.kvh * kPageTokens * HD, 32 * HD * 2);
    }
  pdl_trigger();
  pdl_wait();                          // q / k_new / v_new come from the QKV projection

  // ---- q (RoPE at t0) -> shared; the chunk holding t0 appends k / v to the page ----
  {
    const float* qrow = a.qkv + (int64_t)slot * a.ldqkv;
    const float* cs = a.rope_cos ? a.rope_cos + (int64_t)a.t0 * half : nullptr;
    const float* sn = a.rope_sin ? a.rope_sin + (int64_t)a.t0 * half : nullptr;
    const int dd = threadIdx.x;        // 128 threads = HD dims
    const bool rope = a.family == kLlama;
    const float* q = qrow + kh * HD;
    qs[dd] = rope ? rope_at(q, dd, half, cs, sn) : q[dd];
    if (a.t0 / CH == chunk) {
      const float* kn = qrow + a.H * HD + kh * HD;
      const float* vn = qrow + a.H * HD + a.kvh * HD + kh * HD;
      const int page = a.page_table[slot * a.max_pages + a.t0 / kPageTokens];
      __nv_bfloat16* kp = reinterpret_cast<__nv_bfloat16*>(a.kv_pool) +
                          (((int64_t)page * 2 + 0) * a.kvh + kh) * kPageTokens * HD +
                          (a.t0 % kPageTokens) * HD;
      __nv_bfloat16* vp = kp + (int64_t)a.kvh * kPageTokens * HD;
      kp[dd] = __float2bfloat16_rn(rope ? rope_at(kn, dd, half, cs, sn) : kn[dd]);
      vp[dd] = __float2bfloat16_rn(vn[dd]);
    }
  }
  __syncthreads();                     // q and the appended row visible to the block

  float qreg[16];                      // q dims [c*64 + (lane%8)*8, +8), c = 0, 1
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e) qreg[c * 8 + e] = qs[c * 64 + (lane & 7) * 8 + e];
  const float qscale = kLog2e / sqrtf((float)HD);
  const float slope = (a.family == kBloom) ? a.alibi[kh] * kLog2e : 0.f;
  float m = -INFINITY, l = 0.f;        // warp-uniform max, per-lane partial sum
  float o[4] = {0.f, 0.f, 0.f, 0.f};   // dims 4*lane .. 4*lane + 3
  for (int b = b0 + warp; b < b1; b += NW) {
    // a 32-position block lies inside one 64-position page (allocated: it holds b*32 < T)
    const __nv_bfloat16* kblk = block_k(b);
    const __nv_bfloat16* vblk = kblk + (int64_t)a.kvh * kPageTokens * HD;
    // the warp's block after next (K and V: 8 KB contiguous each) streams into
    // L2 under this block's arithmetic, so HBM stays busy between the register
    // loads of consecutive blocks (the first two were requested before the wait)
    if (lane == 0 && b + 2 * NW < b1) {
      const __nv_bfloat16* kn = block_k(b + 2 * NW);
      l2_prefetch(kn, 32 * HD * 2);
      l2_prefetch(kn + (int64_t)a.kvh * kPageTokens * HD, 32 * HD * 2);
    }
    // K: lane (rg = lane / 8, li = lane % 8) loads dims [c*64 + li*8, +8) of
    // rows i*4 + rg — each load instruction covers 4 whole 128-byte lines
    // (lane = position would touch 32 lines per instruction and saturate L1)
    uint4 kr[8][2];
    uint2 vr[32];
    const int rg = lane >> 3, li = lane & 7;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c < 2; ++c)
        kr[i][c] = ld_stream16(kblk + (i * 4 + rg) * HD + c * 64 + li * 8);
#pragma unroll
    for (int j = 0; j < 32; ++j) vr[j] = ld_stream8(vblk + j * HD + lane * 4);
    // ---- scores of rows i*4 + rg: 16 dims per lane, summed over the 8 lanes ----
    float sc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const float* qv = qreg + c * 8;
        acc[0] = fmaf(qv[0], lo_bf(kr[i][c].x), acc[0]);
        acc[1] = fmaf(qv[1], hi_bf(kr[i][c].x), acc[1]);
        acc[2] = fmaf(qv[2], lo_bf(kr[i][c].y), acc[2]);
        acc[3] = fmaf(qv[3], hi_bf(kr[i][c].y), acc[3]);
        acc[0] = fmaf(qv[4], lo_bf(kr[i][c].z), acc[0]);
        acc[1] = fmaf(qv[5], hi_bf(kr[i][c].z), acc[1]);
        acc[2] = fmaf(qv[6], lo_bf(kr[i][c].w), acc[2]);
        acc[3] = fmaf(qv[7], hi_bf(kr[i][c].w), acc[3]);
      }
      float d = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      d += __shfl_xor_sync(0xffffffffu, d, 1);
      d += __shfl_xor_sync(0xffffffffu, d, 2);
      d += __shfl_xor_sync(0xffffffffu, d, 4);
      const int p = b * 32 + i * 4 + rg;
      float v = d * qscale;
      if (a.family == kBloom) v = fmaf(slope, (float)(p - (T - 1)), v);
      sc[i] = p < T ? v : -INFINITY;
    }
    // ---- online softmax (exp2 domain); every lane of a row group holds its rows ----
    float bm = sc[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) bm = fmaxf(bm, sc[i]);
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 8));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
    const float mnew = fmaxf(m, bm);
    const float alpha = (m == -INFINITY) ? 0.f : ex2_approx(m - mnew);
    float pe[8], psum = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      pe[i] = ex2_approx(sc[i] - mnew);                 // -inf -> +0
      psum += pe[i];
    }
    l = fmaf(l, alpha, li == 0 ? psum : 0.f);           // one lane per row group counts
    m = mnew;
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] *= alpha;
    // ---- P . V: lane = 4 dims; rows past T carry p = 0 (finite pool rows) ----
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float pj = __shfl_sync(0xffffffffu, pe[j >> 2], (j & 3) * 8);   // row j = i*4 + rg
      o[0] = fmaf(pj, lo_bf(vr[j].x), o[0]);
      o[1] = fmaf(pj, hi_bf(vr[j].x), o[1]);
      o[2] = fmaf(pj, lo_bf(vr[j].y), o[2]);
      o[3] = fmaf(pj, hi_bf(vr[j].y), o[3]);
    }
  }
  l = warp_sum(l);
  *reinterpret_cast<float4*>(&wo[warp][lane * 4]) = make_float4(o[0], o[1], o[2], o[3]);
  if (lane == 0) { wm[warp] = m; wl[warp] = l; }
  __syncthreads();

  // ---- merge the 4 warps (fixed order) into this chunk's (max, sum, O); thread = dim ----
  const int dd = threadIdx.x;
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < NW; ++w) M = fmaxf(M, wm[w]);
  float L = 0.f, O = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const float f = (wm[w] == -INFINITY) ? 0.f : ex2_approx(wm[w] - M);
    L = fmaf(wl[w], f, L);
    O = fmaf(wo[w][dd], f, O);
  }
  const int64_t sk = (int64_t)slot * a.kvh + kh;
  if (nchunk > 1) {
    // chunk partial -> global; the last-arriving chunk merges all of them in
    // ascending order (deterministic, independent of arrival order)
    float* partO = a.part + (sk * a.max_pages + chunk) * HD;
    float* stats = a.part + (int64_t)a.width * a.H * a.max_pages * HD;
    __stcg(partO + dd, O);
    if (dd == 0) {
      __stcg(stats + (sk * a.max_pages + chunk) * 2, M);
      __stcg(stats + (sk * a.max_pages + chunk) * 2 + 1, L);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int old;
      asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                   : "=r"(old) : "l"(a.counters + sk) : "memory");
      last = (old == nchunk - 1);
    }
    __syncthreads();
    if (!last) return;
    const float* st = stats + sk * a.max_pages * 2;
    if (threadIdx.x < 32) {            // nchunk <= 32: lane = chunk
      const float mc = lane < nchunk ? __ldcg(st + 2 * lane) : -INFINITY;
      const float lc = lane < nchunk ? __ldcg(st + 2 * lane + 1) : 0.f;
      const float Mg = warp_max(mc);
      const float f = (mc == -INFINITY) ? 0.f : ex2_approx(mc - Mg);
      cf[lane] = f;
      const float Lg = warp_sum(lc * f);
      if (lane == 0) wl[0] = Lg;
    }
    __syncthreads();
    O = 0.f;
    const float* oall = a.part + sk * a.max_pages * HD;
    for (int c = 0; c < nchunk; ++c) O = fmaf(__ldcg(oall + (int64_t)c * HD + dd), cf[c], O);
    L = wl[0];
    if (threadIdx.x == 0) a.counters[sk] = 0;
  }
  const float v = O / L;
  a.ctx[(int64_t)slot * a.H * HD + (int64_t)kh * HD + dd] = v;
  if (a.st_out) {
    float S = warp_sum(v), Q = warp_sum(v * v), Mx = warp_max(fabsf(v));
    if (lane == 0) { red[0][warp] = S; red[1][warp] = Q; red[2][warp] = Mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      float s2 = 0.f, q2 = 0.f, m2 = 0.f;
      for (int w = 0; w < NW; ++w) { s2 += red[0][w]; q2 += red[1][w]; m2 = fmaxf(m2, red[2][w]); }
      a.st_out[(int64_t)kh * a.width + slot] = RowStat{s2, q2, m2, 0.f};
    }
  }
}

}  // namespace

bool g_attn_mha = getenv("SP_ATTN_MHA") ? atoi(getenv("SP_ATTN_MHA")) != 0 : true;
// chunk length >= T / div (128..1024 positions); measured (div 4 / 8 / 16):
// Llama-2-7B batch 1 at 1 K positions 312 / 336 / 346 steps/s (the cluster
// kernel: 341), BLOOM batch 16 at 2 K 163.0 / 160.4 / 159.2 per 8 blocks
static int g_mha_div = getenv("SP_MHA_DIV") ? atoi(getenv("SP_MHA_DIV")) : 16;

bool attn_dec_mha_ok(const AttnDecArgs& a) {
  // one query head per kv head, bf16 cache, hd 128; every width (the per-row
  // decomposition depends on the sequence length only); T / 128 chunks of the
  // smallest size must fit the partial buffers (max_pages) and one warp's merge
  const int T = a.t0 + 1;
  return g_attn_mha && a.kv_dtype == kKVBF16 && a.hd == HD && a.H == a.kvh &&
         (T + mha_chunk(T, g_mha_div) - 1) / mha_chunk(T, g_mha_div) <= 32;
}

int launch_attn_decode_mha(const AttnDecArgs& a, cudaStream_t st) {
  const int T = a.t0 + 1;
  const dim3 grid(a.width * a.kvh, (T + mha_chunk(T, g_mha_div) - 1) / mha_chunk(T, g_mha_div));
  launch_pdl(attn_dec_mha_kernel, grid, dim3(NW * 32), 0, st, a, g_mha_div);
  count_launch();
  return a.H;                          // P_out: one partial per head
}

}  // namespace sp
