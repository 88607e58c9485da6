/*
 * spanpipe — C ABI of the B200-native span-forward hot path of
 * Petals / swarmpipe (arXiv 2312.08361).
 *
 * Plain pointers and sizes only; device pointers are CUDA device addresses
 * on the span's device, `stream` is a cudaStream_t (NULL = legacy stream).
 * Every call returns SP_OK (0) or a negative SP_ERR_* code; sp_last_error()
 * returns the message of the most recent failure on the calling thread.
 *
 * Reference interfaces replaced (SP/ = /root/reference/pkg/src/swarmpipe/):
 *   sp_quantize_blockwise    <- quantize_hidden        SP/quantize.py:36-49
 *   sp_dequantize_blockwise  <- dequantize_hidden      SP/quantize.py:52-58
 *   sp_weights_generate      <- _uniform_weights       SP/model.py:55-60
 *   sp_span_create           <- RealServerEngine.__init__ / init_model
 *                                                      SP/server.py:80-82, SP/model.py:178-199
 *   sp_kv_create             <- RealServerEngine.make_caches  SP/server.py:84-85
 *   sp_kv_length             <- RealServerEngine.cache_length SP/server.py:87-91
 *   sp_span_forward          <- RealServerEngine.run_cached   SP/server.py:93-100
 *                               (block_forward_batched + KVCache.append,
 *                                SP/model.py:244-280, :163-167)
 *   sp_span_forward_stateless<- RealServerEngine.forward      SP/server.py:106-125
 *   sp_span_block_backward   <- block_backward (per block of RealServerEngine.backward)
 *                                                      SP/model.py:320-381, SP/server.py:127-139
 *   sp_kv_reorder            <- RealServerEngine.reorder / KVCache.gather
 *                                                      SP/server.py:102-104, SP/model.py:169-175
 *   sp_kv_read               <- KVCache.keys / .values views (test access,
 *                                T/test_server.py:173-178)
 *   sp_fnv1a64               <- fnv1a64 / RealServerEngine.blob_checksum
 *                                SP/wire.py:39-44, SP/server.py:141-142
 *   sp_content_hash(_verify) <- the relay checksum stamp / check of BlockServer._step
 *                                (SP/server.py:388-393, 413-426) for the device-resident
 *                                span-to-span wire
 */
#ifndef SPANPIPE_H_
#define SPANPIPE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_OK 0
#define SP_ERR_ARG (-1)
#define SP_ERR_CUDA (-2)
#define SP_ERR_CAPACITY (-3)
#define SP_ERR_STATE (-4)
#define SP_ERR_OOM (-5)

/* model families / dtypes (paper_2312_08361_b200/config.py) */
#define SP_FAMILY_TOY 0
#define SP_FAMILY_LLAMA 1
#define SP_FAMILY_BLOOM 2
#define SP_W_F32 0
#define SP_W_BF16 1
#define SP_W_I8 2
#define SP_W_NF4 3   /* 4-bit NF4 levels + uint8 block scales (oracle/model.py) */
#define SP_KV_F32 0
#define SP_KV_BF16 1

typedef struct sp_config {
  int32_t n_blocks;
  int32_t hidden_dim;
  int32_t n_heads;
  int32_t n_kv_heads;
  int32_t ffn_dim;
  int32_t vocab_size;
  int32_t max_seq_len;
  int32_t family;
  int32_t weight_dtype;
  int32_t kv_dtype;
  uint64_t seed;
  double rope_theta;
} sp_config;

typedef struct sp_span sp_span; /* weights + KV pool of blocks [start, end) on one device */
typedef struct sp_kv sp_kv;     /* one session's paged attention caches over the span */
typedef struct sp_head sp_head; /* client head: tied embedding + greedy pick */

const char* sp_last_error(void);
int sp_version(void);

/* ---- hidden-state codec (bit-exact with SP/quantize.py) ---------------- */
/* n elements of x (f32) -> codes int8 [n], scales f32 [ceil(n/64)] */
int sp_quantize_blockwise(const float* x, int8_t* codes, float* scales, int64_t n, void* stream);
int sp_dequantize_blockwise(const int8_t* codes, const float* scales, float* x, int64_t n,
                            void* stream);

/* ---- deterministic weights (bit-exact with SP/model.py:55-60) ----------- */
/* dst[i] = element i of the row-major [d_in, d_out] tensor of (seed, block, role_id) */
int sp_weights_generate(uint64_t seed, int32_t block, int32_t role_id, int64_t n_elements,
                        double scale, float* dst, void* stream);
/* splitmix64 stream seed of (seed, block, role_id) — SP/model.py:49-52 */
uint64_t sp_stream_seed(uint64_t seed, int32_t block, int32_t role_id);

/* ---- span lifecycle ----------------------------------------------------- */
/* kv_pool_tokens: KV capacity of the span's page pool, in positions
 * (summed over all sessions and beam slots). */
int sp_span_create(const sp_config* cfg, int32_t start, int32_t end, int32_t device,
                   int64_t kv_pool_tokens, sp_span** out);
int sp_span_destroy(sp_span* span);
int64_t sp_span_weight_bytes(const sp_span* span);
int64_t sp_span_free_pages(const sp_span* span);
/* copy block `block`'s matrix `role_id` back as f32 [d_in, d_out] (effective
 * values: bf16/int8 dequantised) — test access only */
int sp_span_read_weight(sp_span* span, int32_t block, int32_t role_id, float* dst_host);

/* ---- sessions ------------------------------------------------------------ */
int sp_kv_create(sp_span* span, int32_t width, sp_kv** out);
int sp_kv_destroy(sp_kv* kv);
int32_t sp_kv_length(const sp_kv* kv);
int32_t sp_kv_width(const sp_kv* kv);
/* new slot i <- old slot parents0[i]; new width = new_width (pages are shared
 * copy-on-write; only a shared partial tail page is copied) */
int sp_kv_reorder(sp_kv* kv, const int32_t* parents0, int32_t new_width, void* stream);
/* keys/values of one block (absolute block id) and slot, as f32
 * [length, n_kv_heads, head_dim] into host memory */
int sp_kv_read(sp_kv* kv, int32_t block, int32_t slot, float* keys_host, float* values_host);

/* ---- the hot path ----------------------------------------------------------
 * x: device f32 [width * n_new, hidden] (rows ordered slot-major), or NULL when
 * x_codes/x_scales carry the int8 codec form (dequantised in-kernel);
 * y: device f32 [width * n_new, hidden]; if y_codes != NULL the output is also
 * quantised (SP/server.py:100 with quantized=True) into y_codes/y_scales.
 * Appends n_new positions per slot to kv. */
int sp_span_forward(sp_span* span, sp_kv* kv, int32_t block_begin, int32_t block_end,
                    const float* x, const int8_t* x_codes, const float* x_scales, float* y,
                    int8_t* y_codes, float* y_scales, int32_t width, int32_t n_new,
                    void* stream);
/* stateless causal forward of `batch` independent sequences of `tokens`
 * (no cache kept), SP/server.py:106-125.  If record != NULL it receives the
 * input of every block: f32 [block_end - block_begin][batch * tokens][hidden]
 * (the `record` list of SP/server.py:113-121). */
int sp_span_forward_stateless(sp_span* span, int32_t block_begin, int32_t block_end,
                              const float* x, float* y, float* record, int32_t batch,
                              int32_t tokens, void* stream);
/* prompt-tuning backward of one block: dx = (d block / d x)^T dy for `batch`
 * sequences of `tokens` rows, recomputing the forward from the recorded block
 * input x in float64 (SP/model.py:320-381); x, dy, dx f32 [batch*tokens][hidden]
 * on the device.  Defined, like the reference, for the reference model family
 * (f32 weights, LayerNorm, MHA, GELU); SP_ERR_ARG otherwise. */
int sp_span_block_backward(sp_span* span, int32_t block, const float* x, const float* dy,
                           float* dx, int32_t batch, int32_t tokens, void* stream);

/* ---- client head (SP/model.py:388-400) -------------
 * embedding generated on the device bit-identically (role 11, block n_blocks);
 * embed = row gather; greedy = argmax(row @ E^T), ties to the lowest id */
int sp_head_create(const sp_config* cfg, int32_t device, sp_head** out);
int sp_head_destroy(sp_head* head);
int sp_head_embed(sp_head* head, const int32_t* tokens_host, int32_t n, float* out_dev,
                  void* stream);
int sp_head_greedy(sp_head* head, const float* row_dev, int32_t* token_host, void* stream);
int sp_head_read_embedding(sp_head* head, float* dst_host);
/* logits of n_rows device rows: logits_dev [n_rows, vocab] = rows @ E^T
 * (RealClientEngine.logits, SP/client.py:104-105, used by beam search) */
int sp_head_logits(sp_head* head, const float* rows_dev, int32_t n_rows, float* logits_dev,
                   void* stream);
/* one beam-search selection step (beam_select, SP/model.py:470-491) on device
 * logits [w, vocab]: float64 log-softmax per row, candidates scores[r] + logp,
 * the k (<= 16) best ranked by score desc, parent asc, token asc; results to host */
int sp_beam_select(const float* logits_dev, const double* scores_host, int32_t w, int32_t vocab,
                   int32_t k, int32_t* parents_host, int32_t* tokens_host, double* new_scores_host,
                   void* stream);

/* ---- measurement ----------------------------------------------------------
 * With profiling on, every launch of the span schedule is bracketed by CUDA
 * events on its stream; profile_read synchronises and returns, per class
 * (0 decode GEMV, 1 prefill GEMM, 2 decode attention, 3 prefill attention,
 * 4 norms/RoPE/KV-append/codec), the summed device ms, algorithmic bytes and
 * flops and the number of launches, then clears the records. */
int sp_span_set_profiling(sp_span* span, int32_t enable);
/* options: 0 = use the tcgen05 prefill GEMM when the shape allows (default 1;
 * 0 selects the exact-f32 SIMT GEMM, used by parity tests as a cross-check);
 * 1 = programmatic dependent launch of the decode chain (default 1);
 * 2 = CTA-pair (cta_group::2) prefill GEMM (default 1); 3 = bf16 hi/lo prefill
 * attention (default 0); 5 = decode-attention sub-chunks per CTA (0 = auto);
 * 6 = decode-attention cluster merge for 8 query heads per kv head
 * (-1 = global last-CTA merge, the default; 0 = auto; 8 or 16 = cluster size);
 * 7 = decode attention on the 8-CTA cluster kernel (default 1); 8 = prefill
 * attention on tcgen05 (default 1); 9 = multi-head decode attention
 * (one query head per kv head; default 1); 10 = wide decode (9..32 rows) GEMM
 * with the weights as the MMA's A operand (default 1; 0 = the token-tile GEMM,
 * bit-identical); 11 = the row count from which decode runs its linears on the
 * weight-side tcgen05 GEMM instead of the GEMV (default 3; up to 32 rows the
 * GEMM reproduces the GEMV's numerics, so rows are bit-identical either way).
 * Option 0 is per span; options 1-11 are kernel-selection switches shared by
 * every span in the process (set them before concurrent use). */
int sp_span_set_option(sp_span* span, int32_t option, int32_t value);
int sp_span_profile_read(sp_span* span, int32_t n_classes, double* ms, double* bytes,
                         double* flops, int64_t* launches);
/* measurement helper: only the 4 decode GEMVs of every block in [b0, b1)
 * (tensor-core path), reading the activations/statistics left by the last
 * decode step; *weight_bytes = algorithmic weight bytes of the sequence.
 * Used by bench.py to time the dominant kernel back to back with CUDA events. */
int sp_span_decode_gemv_only(sp_span* span, sp_kv* kv, int32_t block_begin, int32_t block_end,
                             float* y, int32_t width, void* stream, double* weight_bytes);
/* kernels launched by this library since load (all spans, all devices) */
int64_t sp_kernel_launches(void);

/* FNV-1a 64 over host bytes — SP/wire.py:39-44 (relay checksums,
 * SP/server.py:141-142); host-side helper */
uint64_t sp_fnv1a64(const uint8_t* data, int64_t n);

/* Content hash of n bytes of DEVICE memory, computed in `stream` with no host
 * synchronisation: H = (n + sum_i (w_i + 1) r^(i+1)) mod 2^61-1 over the
 * little-endian u32 words w_i (zero-padded tail), r = 0x0A3B1C5D7E9F2468 mod p
 * (definition: csrc/hash.cu; restatement: oracle/content_hash.py).
 * sp_content_hash writes H to *hash_out (device).  sp_content_hash_verify
 * compares H with *expect (device) and sets *mismatch (device int32) to 1 when
 * they differ (sticky: never cleared) — the relay-checksum check of
 * SP/server.py:388-393 done in the stream of the receiving span. */
int sp_content_hash(const void* data, int64_t n, uint64_t* hash_out, void* stream);
int sp_content_hash_verify(const void* data, int64_t n, const uint64_t* expect, int32_t* mismatch,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPANPIPE_H_ */
