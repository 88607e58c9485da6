// Prefill / replay (n_new > 1) tensor-core interfaces.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {

struct TcGemmArgs {
  const void* w;            // int8 weights, core-matrix layout (common.cuh)
  const float* wscale;      // per output channel
  int64_t N, K;
  const uint8_t* planes;    // activation digit planes d0 | d1 (core-matrix layout, M padded to 256)
  int64_t plane_stride;     // bytes between d0 and d1
  const int* exps;          // per-row exponents e_m (|x| < 2^e)
  int64_t M;
  float* y;
  int64_t ldy;
  const float* res;         // EPI_RESID (may alias y)
  int epi;
  int debug;                // (tools) 1: skip the MMAs, 2: skip the TMA loads — timing only
  unsigned long long* trace;  // (tools, SP_TC_TRACE) per-CTA globaltimer phases, or null
  // split-K (few-token GEMMs, single-CTA kernel): int64 partials [M][N] and one
  // arrival counter per output tile, both zero at rest; null = no split
  long long* ws;
  int* counters;
  int ksplit;               // set by the launcher
  int bf16;                 // bf16 weights and hi/lo bf16 planes (K counted in bytes)
  // decode-GEMV numerics (weight-side wide kernel only, ys_rows != null): the
  // planes carry the GEMV's activation code (digitize_gemv), the output is
  // f32((double)D * ys_rows[m] * wscale[n]) with the GEMV's epilogue order, and
  // the (sum, sumsq, max|x*g_next|) partial of every 128-channel group is
  // written to st_out[group * stat_rs + m] — a row's result equals the GEMV's
  const double* ys_rows;
  float4* st_out;
  const float* g_next;
  int64_t stat_rs;
};

extern bool g_tc_wide;    // option 10: wide-decode GEMM with the weights on the MMA's M side

// token rows of the digit planes: padded to the 256-token CTA-pair tile
inline int64_t tc_rows(int64_t M) { return (M + 255) / 256 * 256; }
int64_t tc_plane_bytes(int64_t M, int64_t K);
extern bool g_tc_pair;    // sp_span_set_option(.., 2, ..): CTA-pair tcgen05 GEMM (default on)
void launch_digitize(const float* x, int64_t ldx, int64_t M, int64_t K, int norm, const float* g,
                     const float* b, uint8_t* planes, int64_t plane_stride, int* exps,
                     cudaStream_t st, int rt = 128);   // rt: rows per core-matrix tile
int wide_rows(int64_t M);   // row tile of the wide-decode GEMM for M rows (0 = not used)
// the decode GEMV's activation code as digit planes (rt-row tiles): per row the
// statistics come from the producer's partials st_in[p * R + m] (p < P_in),
// reduced in the GEMV's order; ys_rows[m] = 2^(e-14) * rstd (double)
void launch_digitize_gemv(const float* x, int64_t ldx, int64_t M, int64_t K, int norm,
                          const float* g, const float4* st_in, int P_in, float gmax, float eps,
                          uint8_t* planes, int64_t plane_stride, double* ys_rows, int rt,
                          cudaStream_t st);
void launch_gemm_i8_tc(const TcGemmArgs& a, cudaStream_t st);
// bf16 operand planes (hi, lo) for bf16 weights; K <= 16384
void launch_digitize_bf16(const float* x, int64_t ldx, int64_t M, int64_t K, int norm,
                          const float* g, const float* b, uint8_t* planes, int64_t plane_stride,
                          cudaStream_t st);

}  // namespace sp
