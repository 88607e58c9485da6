// Fused decode-step interfaces (n_new == 1): tensor-pipe GEMVs with the
// pre-norm folded in, and the fused attention kernel.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {

// Per-row statistics of a GEMV input, written as P partials by the producing
// kernel (one partial per producer CTA/group, fixed slots -> deterministic):
//   x = sum(v), y = sum(v^2), z = max |v * g_next|   (w unused)
// The consumer reduces the P partials in a fixed order.
struct RowStat {
  float sum, sumsq, amax, pad;
};

enum Norm { NORM_NONE = 0, NORM_RMS = 1, NORM_LN = 2 };

struct GemvArgs {
  const void* w;          // fragment-tiled weights (int8 m16n8k32 / bf16 m16n8k16 layout)
  const float* wscale;    // int8 per-output-channel scales
  int64_t N, K;
  const float* x;         // [R][K] f32 (un-normalised)
  int64_t ldx;
  int R;
  int norm;               // Norm: the input transform folded into the GEMV
  const float* g;         // norm gains [K]
  float gmax;             // max |g| (LN exponent bound)
  float eps;
  const RowStat* st_in;   // [P_in][R]
  int P_in;
  float* y;               // [R][ldy]
  int64_t ldy;
  const float* res;       // residual [R][ldy] (may alias y)
  int epi;                // Epi (kernels.cuh)
  RowStat* st_out;        // [G][R] partial stats of the written outputs (or null)
  const float* g_next;    // gains for st_out.amax (null -> 1)
  long long* ws;          // split-K int64 accumulators [R][N] (int8) / f32 partials (bf16)
  int* counters;          // split-K arrival counters per row group (zero at rest)
  unsigned long long* trace;   // debug (SP_GEMV_TRACE): per-warp phase timestamps, or null
};

int64_t gemv3_ws_bytes(int64_t N, int Rmax);
int64_t gemv3_counters(int64_t N);
void launch_gemv3(int wdtype, const GemvArgs& a, cudaStream_t st);

// statistics of the span input rows (producer for the first block's norm)
void launch_row_stats(const float* x, int R, int64_t d, const float* g_next, RowStat* st_out,
                      cudaStream_t st);

struct AttnDecArgs {
  int family, kv_dtype;
  int width, t0;                 // the new token sits at position t0 (cache length before)
  int H, kvh, hd;
  const float* qkv;              // [width][H*hd + 2*kvh*hd] raw projections (no RoPE yet)
  int64_t ldqkv;
  void* kv_pool;
  const int* page_table;
  int max_pages;
  const float* rope_cos, *rope_sin, *alibi;
  float* ctx;                    // [width][H*hd]
  float* part;                   // O [width*kvh][max_pages][G][hd], then (max,sum) pairs
  int* counters;                 // [width*kvh] (zero at rest)
  RowStat* st_out;               // [H][width] partial stats of ctx (P = H)
  unsigned long long* trace;     // debug (SP_ATTN_TRACE): per-CTA phase timestamps, or null
  int nsub;                      // 128-position sub-chunks streamed per CTA (MMA kernel; 0 = 1)
};

// returns P_out: the number of ctx partial statistics per row written to
// st_out (the O-projection GEMV's P_in)
int launch_attn_decode_fused(const AttnDecArgs& a, cudaStream_t st);
bool attn_dec_cl_ok(const AttnDecArgs& a);              // attn_decode_cl.cu
int launch_attn_decode_cl(const AttnDecArgs& a, cudaStream_t st);
extern bool g_attn_cl;                                  // option 7 (default on)
bool attn_dec_mha_ok(const AttnDecArgs& a);             // attn_decode_mha.cu
int launch_attn_decode_mha(const AttnDecArgs& a, cudaStream_t st);
extern bool g_attn_mha;                                 // option 9 (default on)
int64_t attn_dec_part_floats(int width, int H, int hd, int max_pages);

}  // namespace sp
