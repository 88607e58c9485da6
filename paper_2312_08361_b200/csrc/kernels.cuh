// Kernel launch interfaces shared between the kernel files and the span runtime.
#pragma once
#include <cuda.h>   // CUtensorMap (tensor-map TMA of the KV pool)
#include <cuda_runtime.h>
#include <stdint.h>

namespace sp {

// Where a [K x N] matrix lives inside a fused weight buffer: output channel n
// goes to buffer row  row0 + ((n/64)*tstride + toff)*64 + n%64
// (tstride 2 interleaves gate/up in 64-row halves of each 128-row group).
struct MatPlace {
  int64_t row0;
  int64_t tstride;
  int64_t toff;
};
constexpr int kPlaceGranule = 64;

// GEMV / GEMM epilogues
enum Epi {
  EPI_STORE = 0,   // y = acc
  EPI_RESID = 1,   // y = res + acc   (res may alias y)
  EPI_GELU = 2,    // y = gelu(acc)                       SP/model.py:228-229
  EPI_SWIGLU = 3,  // y[:, j] = silu(gate_j) * up_j  (gate/up interleaved by 16-row tiles)
};

struct LinearArgs {
  const void* w;         // storage (f32 row-major / bf16,int8 fragment tiles)
  const float* wscale;   // int8 per-row scales (nullptr otherwise)
  int wdtype;
  int64_t N;             // buffer rows (output channels incl. interleave)
  int64_t K;
  const float* x;        // [R][K]
  int64_t ldx;
  float* y;              // [R][ldy]
  int64_t ldy;
  const float* res;      // residual [R][ldy] for EPI_RESID
  int epi;
  int R;
  float* workspace;      // split-K partials
  int* counters;         // split-K arrival counters (self-resetting, zero at rest)
};

void launch_quantize(const float* x, int8_t* codes, float* scales, int64_t n, cudaStream_t st);
void launch_dequantize(const int8_t* codes, const float* scales, float* x, int64_t n,
                       cudaStream_t st);

void launch_gen_stream(uint64_t stream, int64_t n, double scale, float* dst, cudaStream_t st);
// nbuf: rows of the destination buffer (nf4: the block scales follow its codes)
void launch_gen_matrix(int wdtype, uint64_t stream, int64_t K, int64_t N, double scale,
                       MatPlace place, void* dst, float* scales, cudaStream_t st, int64_t nbuf = 0);
void launch_read_matrix(int wdtype, const void* src, const float* scales, int64_t K, int64_t N,
                        MatPlace place, float* dst, cudaStream_t st, int64_t nbuf = 0);

// decode GEMV for f32 weights (any R; rows independent, batch-invariant)
void launch_gemv(const LinearArgs& a, cudaStream_t st);
// prefill GEMM (SIMT fp32, M-invariant)
void launch_gemm(const LinearArgs& a, cudaStream_t st);
// gate/up interleaved [R][2F] -> silu(gate)*up [R][F]
void launch_swiglu_rows(const float* in, float* out, int64_t R, int64_t F, cudaStream_t st);
void launch_gelu_rows(const float* in, float* out, int64_t R, int64_t F, cudaStream_t st);
// nf4 levels of an N x K matrix -> int8 planes hi, lo (hi * 128 + lo = CB7 * q,
// core-matrix layout) and sc128 = 128 * channel scale
void launch_nf4_split(const uint8_t* w, const float* sc, int64_t N, int64_t K, int8_t* hi,
                      int8_t* lo, float* sc128, cudaStream_t st);

// norms: out = LN(x)*g+b  (family toy/bloom) or RMS(x)*g (llama); one row per CTA
void launch_norm(int family, const float* x, const float* g, const float* b, float* out,
                 int64_t R, int64_t d, cudaStream_t st);

struct AttnArgs {
  int family;
  int kv_dtype;
  int width, n_new, t0;          // positions t0 .. t0+n_new-1 are being added
  int H, kvh, hd;
  float* qkv;                    // [width*n_new][H*hd + 2*kvh*hd] (q roped in place)
  int64_t ldqkv;
  void* kv_pool;                 // this block's pool: [pages][2][kvh][64][hd]
  const int* page_table;         // [width][max_pages]
  int max_pages;
  const float* rope_cos;         // [max_seq][hd/2]
  const float* rope_sin;
  const float* alibi;            // [H]
  float* ctx;                    // [width*n_new][H*hd]
  float* workspace;              // split partials
  const void* pool_base;         // the span's whole pool (all blocks): tensor-map base
  int64_t pool_bytes;
};

void launch_rope_append(const AttnArgs& a, cudaStream_t st);
int64_t attn_workspace_floats(int width, int H, int hd, int max_seq);
void launch_attention_decode(const AttnArgs& a, cudaStream_t st);
void launch_attention_prefill(const AttnArgs& a, cudaStream_t st);
// tensor-core flash prefill (bf16 KV, hd 64/128); false if the shape is unsupported
bool launch_attention_prefill_mma(const AttnArgs& a, cudaStream_t st);
// tcgen05 / TMEM flash prefill (bf16 KV, hd 128); false if the shape is unsupported
bool launch_attention_prefill_tc(const AttnArgs& a, cudaStream_t st);
extern bool g_attn_tc;    // option 8 (default on)
// 2-D tensor map over a span's KV pool (cols = hd, bf16, 128-byte swizzle,
// [box_rows][64] boxes); cached per pool; null if the driver entry point is missing
const CUtensorMap* kv_pool_map(const void* base, int64_t bytes, int hd, int box_rows);

// KV page copy (copy-on-write of a shared tail page): all blocks of the span
void launch_page_copy(void* pool, int64_t block_stride_bytes, int n_blocks,
                      int64_t page_bytes, int src_page, int dst_page, cudaStream_t st);
// gather one slot's K/V of one block into f32 [t][kvh][hd] x2
void launch_kv_gather_slot(const void* pool, int kv_dtype, const int* page_table_row, int t,
                           int kvh, int hd, float* k_out, float* v_out, cudaStream_t st);

// prompt-tuning backward of one toy-family block (backward.cu): float64
// recompute + backprop, f32 in/out; 0 or -1 (scratch allocation failed)
int block_backward_f64(const float* wqkv_t, const float* wo_t, const float* w1_t,
                       const float* w2_t, const float* ln1_g, const float* ln1_b,
                       const float* ln2_g, const float* ln2_b, int d, int H, int F,
                       const float* x, const float* dy, float* dx, int batch, int tokens,
                       cudaStream_t st);

}  // namespace sp
