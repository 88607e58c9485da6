// Span runtime: weights, paged KV pool, sessions and the per-block kernel
// schedule of RealServerEngine.run_cached (SP/server.py:93-100).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "decode.cuh"
#include "kernels.cuh"
#include "prefill.cuh"

namespace {
thread_local std::string g_err;
}

void sp_set_error(const char* file, int line, const char* msg) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s:%d: %s", file, line, msg);
  g_err = buf;
}

#define SP_FAIL(code, msg)                     \
  do {                                         \
    sp_set_error(__FILE__, __LINE__, (msg));   \
    return (code);                             \
  } while (0)

#define SP_CHECK_LAUNCH() SP_CUDA_TRY(cudaGetLastError())

namespace sp {
static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
bool g_pdl = true;
extern bool g_attn_hilo;   // attn_prefill.cu
extern int g_attn_nsub;    // attn_decode.cu, option 5
extern int g_attn_cluster; // attn_decode.cu, option 6
}  // namespace sp

using namespace sp;



namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kRoleMix = 0xC2B2AE3D27D4EB4Full;

enum Role { R_WQ = 1, R_WK = 2, R_WV = 3, R_WO = 4, R_W1 = 5, R_W2 = 6, R_W3 = 13 };

struct BlockW {
  void* qkv; float* s_qkv;
  void* o; float* s_o;
  void* up; float* s_up;      // llama: gate/up interleaved [2F]; else w1 [F]
  void* down; float* s_down;
  float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct sp_span {
  sp_config cfg;
  int start, end, device;
  int d, H, kvh, hd, F, kv;
  int64_t n_qkv, n_up;
  int64_t weight_bytes = 0;
  char* wmem = nullptr;
  std::vector<BlockW> blocks;
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  float* alibi = nullptr;
  // KV pool
  char* pool = nullptr;
  int64_t n_pages = 0;
  int64_t page_bytes = 0;        // one page, one block: 2*kvh*64*hd*elt
  int64_t block_stride = 0;      // bytes per block pool
  std::vector<int> refcount;
  std::vector<int> free_pages;
  int max_pages = 0;
  // scratch
  int64_t cap_rows = 0;
  float *h = nullptr, *qkvb = nullptr, *ctx = nullptr, *mlp = nullptr, *mlp_raw = nullptr;
  float* gemv_ws = nullptr;
  int* gemv_cnt = nullptr;
  // fused tensor-core decode path (decode.cuh)
  int64_t dec_cap_rows = 0;
  RowStat *st_norm1 = nullptr, *st_ctx = nullptr, *st_norm2 = nullptr, *st_mlp = nullptr;
  long long* ws2 = nullptr;
  int* cnt2 = nullptr;
  float* attn_part = nullptr;
  int* attn_cnt = nullptr;
  bool gains_one = true;   // LN/RMS gains are 1 at init (SP/model.py:192-195), never mutated
  // tcgen05 prefill path
  int64_t tc_cap_rows = 0;
  uint8_t* planes = nullptr;
  int* exps = nullptr;
  double* ys_rows = nullptr;   // wide decode: per-row scale of the GEMV-numerics code
  bool use_tc_prefill = true;
  // nf4 prefill: a linear's integer levels split into two int8 planes
  // (hi * 128 + lo) in core-matrix layout, and 128 x channel scale
  int64_t nf4_cap = 0;
  int8_t *nf4_hi = nullptr, *nf4_lo = nullptr;
  float* nf4_sc = nullptr;
  int64_t attn_ws_floats = 0;
  float* attn_ws = nullptr;
  std::mutex mu;
  // every call that uses the span's scratch (h/qkvb/ctx/mlp, digit planes, split-K
  // workspace and counters, attention partials) is ordered after the previous one,
  // whatever stream the caller passes: the new stream waits on `done` (recorded at
  // the end of the previous call's work) before its first launch
  cudaEvent_t done = nullptr;
  cudaStream_t done_stream = nullptr;
  bool done_valid = false;
  // sessions keep the span's host bookkeeping alive: destroying a span with
  // live sessions frees its device memory at once and the struct when the last
  // session goes (finalizer order in Python reference cycles is arbitrary)
  int live_kv = 0;
  bool dying = false;
  int last_p_ctx = 0;             // ctx partial stats the last decode attention wrote
  // live per-launch timing (bench roofline): CUDA events around each launch
  struct ProfRec { int cls; cudaEvent_t a, b; double bytes, flops; };
  bool prof = false;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
};

struct sp_kv {
  sp_span* span;
  int width;
  int length;
  std::vector<std::vector<int>> pages;
  int* d_table = nullptr;
  int table_cap_width = 0;
  int* h_table = nullptr;          // pinned staging copy of the table (async upload)
  cudaEvent_t table_ev = nullptr;  // completes when the last upload has read h_table
};

namespace {

uint64_t stream_seed(uint64_t seed, int block, int role) {
  uint64_t key = seed ^ ((uint64_t)(block + 1) * kGolden) ^ ((uint64_t)role * kRoleMix);
  return splitmix64_at(key, 0);
}

int wdtype_ktile(int wd) { return wd == kI8 ? 32 : 16; }

int elt_bytes(int wd) { return wd == kF32 ? 4 : (wd == kBF16 ? 2 : 1); }

// algorithmic bytes of one N x K weight matrix (codes + scales)
double weight_bytes_of(int wd, int64_t N, int64_t K) {
  if (wd == kNF4) return (double)nf4_bytes(N, K) + 4.0 * N;
  return (double)N * K * elt_bytes(wd) + (wd == kI8 ? 4.0 * N : 0.0);
}

int validate(const sp_config* c) {
  if (c->n_blocks < 1 || c->hidden_dim < 1 || c->n_heads < 1) return SP_ERR_ARG;
  if (c->hidden_dim % c->n_heads) return SP_ERR_ARG;
  int kvh = c->n_kv_heads ? c->n_kv_heads : c->n_heads;
  if (c->n_heads % kvh) return SP_ERR_ARG;
  int hd = c->hidden_dim / c->n_heads;
  if (!(hd == 4 || hd == 16 || hd == 32 || hd == 64 || hd == 128)) return SP_ERR_ARG;
  int F = c->ffn_dim ? c->ffn_dim : 4 * c->hidden_dim;
  int d = c->hidden_dim, kv = kvh * hd;
  if (c->weight_dtype < kF32 || c->weight_dtype > kNF4) return SP_ERR_ARG;
  if (c->weight_dtype != kF32) {
    // core-matrix layout: 128-row groups, K in 32-byte units (common.cuh)
    if (d % 32 || F % 32) return SP_ERR_ARG;
    if ((d + 2 * kv) % 128 || d % 128 || F % 64) return SP_ERR_ARG;
    if (c->family != kLlama && F % 128) return SP_ERR_ARG;
    if (c->weight_dtype == kNF4 && (d % 64 || F % 64)) return SP_ERR_ARG;   // 64-wide blocks
  } else {
    if (d % 16 || F % 16 || kv % 16) return SP_ERR_ARG;
  }
  return SP_OK;
}

int ensure_scratch(sp_span* s, int64_t rows) {
  if (rows <= s->cap_rows) return SP_OK;
  int64_t cap = rows < 64 ? 64 : rows;
  cudaFree(s->h); cudaFree(s->qkvb); cudaFree(s->ctx); cudaFree(s->mlp); cudaFree(s->mlp_raw);
  s->h = s->qkvb = s->ctx = s->mlp = s->mlp_raw = nullptr;
  int64_t wmax = s->d > s->F ? s->d : s->F;
  SP_CUDA_TRY(cudaMalloc(&s->h, cap * wmax * sizeof(float)));
  SP_CUDA_TRY(cudaMalloc(&s->qkvb, cap * s->n_qkv * sizeof(float)));
  SP_CUDA_TRY(cudaMalloc(&s->ctx, cap * s->d * sizeof(float)));
  SP_CUDA_TRY(cudaMalloc(&s->mlp, cap * s->F * sizeof(float)));
  SP_CUDA_TRY(cudaMalloc(&s->mlp_raw, cap * s->n_up * sizeof(float)));
  s->cap_rows = cap;
  return SP_OK;
}

int ensure_decode(sp_span* s, int64_t rows) {
  if (rows <= s->dec_cap_rows) return SP_OK;
  int64_t cap = rows < 8 ? 8 : rows;
  cudaFree(s->st_norm1); cudaFree(s->st_ctx); cudaFree(s->st_norm2); cudaFree(s->st_mlp);
  cudaFree(s->ws2); cudaFree(s->cnt2); cudaFree(s->attn_part); cudaFree(s->attn_cnt);
  // partial-statistics slots per row: the largest producer fan-out (GEMV groups,
  // decode-attention heads, or kv heads x cluster ranks)
  const int64_t P = std::max<int64_t>(std::max<int64_t>(s->d / 64, s->H),
                                      std::max<int64_t>(s->n_up / 64, 8 * (int64_t)s->kvh));
  for (RowStat** b : {&s->st_norm1, &s->st_ctx, &s->st_norm2, &s->st_mlp})
    SP_CUDA_TRY(cudaMalloc(b, P * cap * sizeof(RowStat)));
  int64_t ws = 0, cnt = 0;
  const int64_t shapes[4][2] = {{s->n_qkv, s->d}, {s->d, s->d}, {s->n_up, s->d}, {s->d, s->F}};
  for (auto& sh : shapes) {
    ws = std::max(ws, gemv3_ws_bytes(sh[0], (int)cap));
    cnt = std::max(cnt, gemv3_counters(sh[0]));
  }
  SP_CUDA_TRY(cudaMalloc(&s->ws2, ws + 16));
  SP_CUDA_TRY(cudaMemset(s->ws2, 0, ws + 16));
  SP_CUDA_TRY(cudaMalloc(&s->cnt2, cnt * sizeof(int)));
  SP_CUDA_TRY(cudaMemset(s->cnt2, 0, cnt * sizeof(int)));
  SP_CUDA_TRY(cudaMalloc(&s->attn_part,
                         attn_dec_part_floats((int)cap, s->H, s->hd, s->max_pages) * sizeof(float)));
  SP_CUDA_TRY(cudaMalloc(&s->attn_cnt, cap * s->kvh * sizeof(int)));
  SP_CUDA_TRY(cudaMemset(s->attn_cnt, 0, cap * s->kvh * sizeof(int)));
  s->dec_cap_rows = cap;
  return SP_OK;
}

int ensure_tc(sp_span* s, int64_t rows) {
  if (rows <= s->tc_cap_rows) return SP_OK;
  cudaFree(s->planes); cudaFree(s->exps); cudaFree(s->ys_rows);
  const int64_t Mp = tc_rows(rows);       // the CTA-pair GEMM tiles 256 tokens
  const int64_t K = std::max<int64_t>(s->d, s->F) * (s->cfg.weight_dtype == kBF16 ? 2 : 1);
  SP_CUDA_TRY(cudaMalloc(&s->planes, 2 * Mp * K));
  SP_CUDA_TRY(cudaMalloc(&s->exps, Mp * sizeof(int)));
  SP_CUDA_TRY(cudaMalloc(&s->ys_rows, Mp * sizeof(double)));
  s->tc_cap_rows = Mp;
  return SP_OK;
}

int ensure_nf4(sp_span* s) {
  if (s->nf4_cap) return SP_OK;
  cudaFree(s->nf4_hi); cudaFree(s->nf4_lo); cudaFree(s->nf4_sc);   // after a failed attempt
  s->nf4_hi = s->nf4_lo = nullptr;
  s->nf4_sc = nullptr;
  const int64_t d = s->d;
  const int64_t cap = std::max(std::max(s->n_qkv * d, d * d), std::max(s->n_up * d, d * s->F));
  SP_CUDA_TRY(cudaMalloc(&s->nf4_hi, cap));
  SP_CUDA_TRY(cudaMalloc(&s->nf4_lo, cap));
  SP_CUDA_TRY(cudaMalloc(&s->nf4_sc, std::max(s->n_qkv, s->n_up) * sizeof(float)));
  s->nf4_cap = cap;
  return SP_OK;
}

bool tc_ok(const sp_span* s) {
  const int wd = s->cfg.weight_dtype;
  // int8 / nf4 (as two int8 planes): K multiple of 128 elements (4 x 32-byte
  // units per stage); bf16: 64
  const int64_t kq = (wd == kI8 || wd == kNF4) ? 128 : 64;
  return (wd == kI8 || wd == kBF16 || wd == kNF4) && s->n_qkv % 256 == 0 && s->d % 256 == 0 &&
         s->n_up % 256 == 0 && s->d % kq == 0 && s->F % kq == 0 &&
         (wd != kBF16 || std::max(s->d, s->F) <= 16384);
}

int ensure_attn_ws(sp_span* s, int width) {
  int64_t need = attn_workspace_floats(width, s->H, s->hd, s->cfg.max_seq_len);
  if (need <= s->attn_ws_floats) return SP_OK;
  cudaFree(s->attn_ws);
  SP_CUDA_TRY(cudaMalloc(&s->attn_ws, need * sizeof(float)));
  s->attn_ws_floats = need;
  return SP_OK;
}

int alloc_page(sp_span* s) {
  if (s->free_pages.empty()) return -1;
  int p = s->free_pages.back();
  s->free_pages.pop_back();
  s->refcount[p] = 1;
  return p;
}

void release_page(sp_span* s, int p) {
  if (--s->refcount[p] == 0) s->free_pages.push_back(p);
}

int upload_table(sp_kv* kv, cudaStream_t st) {
  sp_span* s = kv->span;
  const size_t n = (size_t)kv->width * s->max_pages;
  if (kv->table_cap_width < kv->width) {
    if (kv->table_ev) SP_CUDA_TRY(cudaEventSynchronize(kv->table_ev));
    cudaFree(kv->d_table);
    cudaFreeHost(kv->h_table);
    kv->d_table = nullptr;
    kv->h_table = nullptr;
    kv->table_cap_width = 0;
    SP_CUDA_TRY(cudaMalloc(&kv->d_table, n * sizeof(int)));
    SP_CUDA_TRY(cudaMallocHost(&kv->h_table, n * sizeof(int)));
    kv->table_cap_width = kv->width;
  }
  if (!kv->table_ev) SP_CUDA_TRY(cudaEventCreateWithFlags(&kv->table_ev, cudaEventDisableTiming));
  // the previous upload must have read the staging copy before it is rewritten
  // (in practice long complete: uploads happen every 64 positions or on reorder)
  SP_CUDA_TRY(cudaEventSynchronize(kv->table_ev));
  std::fill(kv->h_table, kv->h_table + n, 0);
  for (int i = 0; i < kv->width; ++i)
    for (size_t p = 0; p < kv->pages[i].size(); ++p)
      kv->h_table[(size_t)i * s->max_pages + p] = kv->pages[i][p];
  // stream-ordered after every kernel that read the old table; no host sync
  SP_CUDA_TRY(cudaMemcpyAsync(kv->d_table, kv->h_table, n * sizeof(int), cudaMemcpyHostToDevice,
                              st));
  SP_CUDA_TRY(cudaEventRecord(kv->table_ev, st));
  return SP_OK;
}

// make pages for positions [length, length + n_new) writable for every slot.
// The pages needed (new pages + copy-on-write copies of shared partial tails)
// are counted first, so a request the pool cannot hold changes nothing.
int prepare_pages(sp_kv* kv, int n_new, cudaStream_t st) {
  sp_span* s = kv->span;
  const int need = (kv->length + n_new + kPageTokens - 1) / kPageTokens;
  int64_t want = 0;
  for (int i = 0; i < kv->width; ++i) {
    const auto& pg = kv->pages[i];
    if (kv->length % kPageTokens && !pg.empty() && s->refcount[pg.back()] > 1) ++want;
    want += std::max(0, need - (int)pg.size());
  }
  if (want > (int64_t)s->free_pages.size()) SP_FAIL(SP_ERR_CAPACITY, "KV page pool exhausted");
  if (want == 0) return SP_OK;
  for (int i = 0; i < kv->width; ++i) {
    auto& pg = kv->pages[i];
    if (kv->length % kPageTokens && !pg.empty()) {
      int tail = pg.back();
      if (s->refcount[tail] > 1) {  // copy-on-write of a shared partial tail page
        int np = alloc_page(s);
        launch_page_copy(s->pool, s->block_stride, s->end - s->start, s->page_bytes, tail, np,
                         st);
        SP_CHECK_LAUNCH();
        release_page(s, tail);
        pg.back() = np;
      }
    }
    while ((int)pg.size() < need) pg.push_back(alloc_page(s));
  }
  return upload_table(kv, st);
}

// cross-stream ordering of the span's scratch (see sp_span::done)
int order_begin(sp_span* s, cudaStream_t st) {
  if (s->done_valid && s->done_stream != st) SP_CUDA_TRY(cudaStreamWaitEvent(st, s->done, 0));
  return SP_OK;
}

int order_end(sp_span* s, cudaStream_t st) {
  if (!s->done) SP_CUDA_TRY(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming));
  SP_CUDA_TRY(cudaEventRecord(s->done, st));
  s->done_stream = st;
  s->done_valid = true;
  return SP_OK;
}

// profiling classes (sp_span_profile_read)
enum ProfCls { PC_GEMV = 0, PC_GEMM = 1, PC_ATTN_DEC = 2, PC_ATTN_PRE = 3, PC_OTHER = 4 };

cudaEvent_t get_event(sp_span* s) {
  if (!s->ev_pool.empty()) {
    cudaEvent_t e = s->ev_pool.back();
    s->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct ProfScope {
  sp_span* s;
  int cls;
  double bytes, flops;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(sp_span* s_, int c, double by, double fl, cudaStream_t st_)
      : s(s_), cls(c), bytes(by), flops(fl), st(st_) {
    if (s->prof) {
      a = get_event(s);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = get_event(s);
      cudaEventRecord(b, st);
      s->prof_recs.push_back({cls, a, b, bytes, flops});
    }
  }
};

void linear(sp_span* s, int wd, void* w, float* sc, int64_t N, int64_t K, const float* x,
            float* y, int64_t ldy, const float* res, int epi, int64_t R, bool decode,
            cudaStream_t st) {
  const double wbytes = weight_bytes_of(wd, N, K);
  const double outc = (epi == EPI_SWIGLU) ? N / 2 : N;
  ProfScope ps(s, decode ? PC_GEMV : PC_GEMM, wbytes + 4.0 * R * (K + outc), 2.0 * R * N * K, st);
  LinearArgs a{};
  a.w = w; a.wscale = sc; a.wdtype = wd; a.N = N; a.K = K;
  a.x = x; a.ldx = K; a.y = y; a.ldy = ldy; a.res = res; a.epi = epi; a.R = (int)R;
  a.workspace = s->gemv_ws; a.counters = s->gemv_cnt;
  if (decode && wd == kF32) {
    launch_gemv(a, st);
  } else if (epi == EPI_SWIGLU) {
    a.epi = EPI_STORE;
    a.y = s->mlp_raw;
    a.ldy = N;
    launch_gemm(a, st);
    launch_swiglu_rows(s->mlp_raw, y, R, N / 2, st);
  } else {
    launch_gemm(a, st);
  }
}

// decode (n_new == 1) with bf16/int8 weights: 5 launches per block, norms folded
// into the GEMVs, RoPE + KV append + page merge folded into attention.
int run_span_decode_tc(sp_span* s, sp_kv* kv, int b0, int b1, float* y, int width,
                       cudaStream_t st, bool gemv_only = false) {
  const int64_t R = width;
  int rc = ensure_scratch(s, R);
  if (rc) return rc;
  rc = ensure_decode(s, R);
  if (rc) return rc;
  const int wd = s->cfg.weight_dtype, fam = s->cfg.family;
  const int64_t d = s->d;
  const int norm = fam == kLlama ? NORM_RMS : NORM_LN;
  const double kv_elt = s->cfg.kv_dtype == kKVBF16 ? 2.0 : 4.0;
  auto wbytes = [&](int64_t N, int64_t K) {
    return weight_bytes_of(wd, N, K);
  };
  if (!gemv_only) {
    ProfScope ps(s, PC_OTHER, 4.0 * R * d, 0, st);
    launch_row_stats(y, (int)R, d, s->gains_one ? nullptr : s->blocks[b0 - s->start].ln1_g,
                     s->st_norm1, st);
  }
  GemvArgs g{};
  g.R = (int)R; g.eps = 1e-5f; g.gmax = 1.0f;
  g.ws = s->ws2; g.counters = s->cnt2;
  AttnDecArgs at{};
  at.family = fam; at.kv_dtype = s->cfg.kv_dtype; at.width = width; at.t0 = kv->length;
  at.H = s->H; at.kvh = s->kvh; at.hd = s->hd; at.qkv = s->qkvb; at.ldqkv = s->n_qkv;
  at.page_table = kv->d_table; at.max_pages = s->max_pages;
  at.rope_cos = s->rope_cos; at.rope_sin = s->rope_sin; at.alibi = s->alibi;
  at.ctx = s->ctx; at.part = s->attn_part; at.counters = s->attn_cnt; at.st_out = s->st_ctx;
  for (int b = b0 - s->start; b < b1 - s->start; ++b) {
    BlockW& W = s->blocks[b];
    const bool last = (b == b1 - s->start - 1);
    // 1) QKV = RMS/LN(x) @ Wqkv
    g.w = W.qkv; g.wscale = W.s_qkv; g.N = s->n_qkv; g.K = d; g.x = y; g.ldx = d;
    g.norm = norm; g.g = s->gains_one ? nullptr : W.ln1_g; g.st_in = s->st_norm1;
    g.P_in = (int)(d / 128);
    g.y = s->qkvb; g.ldy = s->n_qkv; g.res = nullptr; g.epi = EPI_STORE;
    g.st_out = nullptr; g.g_next = nullptr;
    {
      ProfScope ps(s, PC_GEMV, wbytes(g.N, g.K) + 4.0 * R * (g.K + g.N), 2.0 * R * g.N * g.K, st);
      launch_gemv3(wd, g, st);
    }
    // 2) attention (RoPE, append, page merge)
    at.kv_pool = s->pool + (int64_t)b * s->block_stride;
    // timing experiment only (wrong results): SP_DEBUG_SKIP_ATTN=1 measures the
    // in-stream cost of decode attention
    static const bool skip_attn = getenv("SP_DEBUG_SKIP_ATTN") != nullptr;
    int p_ctx = s->H;                       // ctx partial statistics per row (O GEMV P_in)
    if (!gemv_only && !skip_attn) {
      const double kvb = (double)width * (kv->length + 1) * 2 * s->kv * kv_elt;
      ProfScope ps(s, PC_ATTN_DEC, kvb + 4.0 * R * (s->n_qkv + d),
                   4.0 * width * (kv->length + 1) * s->H * s->hd, st);
      p_ctx = launch_attn_decode_fused(at, st);
    } else if (gemv_only) {
      p_ctx = s->last_p_ctx;
    }
    s->last_p_ctx = p_ctx;
    // 3) x += ctx @ Wo      (stats for norm2)
    g.w = W.o; g.wscale = W.s_o; g.N = d; g.K = d; g.x = s->ctx; g.ldx = d;
    g.norm = NORM_NONE; g.g = nullptr; g.st_in = s->st_ctx; g.P_in = p_ctx;
    g.y = y; g.ldy = d; g.res = y; g.epi = EPI_RESID; g.st_out = s->st_norm2;
    g.g_next = s->gains_one ? nullptr : W.ln2_g;
    {
      ProfScope ps(s, PC_GEMV, wbytes(g.N, g.K) + 4.0 * R * (g.K + 2 * g.N), 2.0 * R * g.N * g.K, st);
      launch_gemv3(wd, g, st);
    }
    // 4) mlp = act(RMS/LN(x) @ Wup)
    g.w = W.up; g.wscale = W.s_up; g.N = s->n_up; g.K = d; g.x = y; g.ldx = d;
    g.norm = norm; g.g = s->gains_one ? nullptr : W.ln2_g; g.st_in = s->st_norm2;
    g.P_in = (int)(d / 128);
    g.y = s->mlp; g.ldy = s->F; g.res = nullptr; g.epi = fam == kLlama ? EPI_SWIGLU : EPI_GELU;
    g.st_out = s->st_mlp; g.g_next = nullptr;
    {
      ProfScope ps(s, PC_GEMV, wbytes(g.N, g.K) + 4.0 * R * (g.K + s->F), 2.0 * R * g.N * g.K, st);
      launch_gemv3(wd, g, st);
    }
    // 5) x += mlp @ Wdown   (stats for the next block's norm1)
    g.w = W.down; g.wscale = W.s_down; g.N = d; g.K = s->F; g.x = s->mlp; g.ldx = s->F;
    g.norm = NORM_NONE; g.g = nullptr; g.st_in = s->st_mlp; g.P_in = (int)(s->n_up / 128);
    g.y = y; g.ldy = d; g.res = y; g.epi = EPI_RESID;
    g.st_out = last ? nullptr : s->st_norm1;
    g.g_next = (last || s->gains_one) ? nullptr : s->blocks[b + 1].ln1_g;
    {
      ProfScope ps(s, PC_GEMV, wbytes(g.N, g.K) + 4.0 * R * (g.K + 2 * g.N), 2.0 * R * g.N * g.K, st);
      launch_gemv3(wd, g, st);
    }
  }
  SP_CHECK_LAUNCH();
  return SP_OK;
}

// prefill / replay (n_new > 1) with int8 weights: tcgen05 GEMMs on activation
// digit planes (gemm_tc.cu), SIMT attention
int run_span_prefill_tc(sp_span* s, sp_kv* kv, int b0, int b1, float* y, float* record,
                        int width, int n_new, cudaStream_t st) {
  const int64_t R = (int64_t)width * n_new;
  int rc = ensure_scratch(s, R);
  if (rc) return rc;
  rc = ensure_attn_ws(s, width);
  if (rc) return rc;
  rc = ensure_tc(s, R);
  if (rc) return rc;
  const int fam = s->cfg.family;
  const int norm = fam == kLlama ? 1 : 2;
  const bool bf = s->cfg.weight_dtype == kBF16;
  const int64_t eb = bf ? 2 : 1;
  const int64_t d = s->d, F = s->F;
  const int64_t Mp = tc_rows(R);
  const double kv_elt = s->cfg.kv_dtype == kKVBF16 ? 2.0 : 4.0;
  AttnArgs at{};
  at.family = fam; at.kv_dtype = s->cfg.kv_dtype;
  at.width = width; at.n_new = n_new; at.t0 = kv->length;
  at.H = s->H; at.kvh = s->kvh; at.hd = s->hd;
  at.qkv = s->qkvb; at.ldqkv = s->n_qkv;
  at.page_table = kv->d_table; at.max_pages = s->max_pages;
  at.rope_cos = s->rope_cos; at.rope_sin = s->rope_sin; at.alibi = s->alibi;
  at.ctx = s->ctx; at.workspace = s->attn_ws;
  at.pool_base = s->pool; at.pool_bytes = s->block_stride * (s->end - s->start);
  auto gemm1 = [&](void* w, float* sc, int64_t N, int64_t K, float* out, int64_t ldy,
                   const float* res, int epi) {
    ProfScope ps(s, PC_GEMM, (double)N * K + 4.0 * N + 2.0 * Mp * K + 4.0 * R * ldy,
                 2.0 * R * N * K, st);
    TcGemmArgs g{};
    const int64_t Kb = K * eb;                     // K in bytes (32-byte units)
    g.w = w; g.wscale = bf ? nullptr : sc; g.N = N; g.K = Kb; g.planes = s->planes;
    g.plane_stride = Mp * Kb;
    g.exps = s->exps; g.M = R; g.y = out; g.ldy = ldy; g.res = res; g.epi = epi;
    g.bf16 = bf ? 1 : 0;
    launch_gemm_i8_tc(g, st);
  };
  // nf4: W = s * (hi * 128 + lo) exactly (|CB7 * q| <= 16065); two int8 GEMMs on
  // the same activation planes, the first scaled by 128 s, the second adding
  // into its output; SwiGLU / GELU applied after the sum
  const bool nf = s->cfg.weight_dtype == kNF4;
  if (nf) {
    rc = ensure_nf4(s);
    if (rc) return rc;
  }
  auto gemm = [&](void* w, float* sc, int64_t N, int64_t K, float* out, int64_t ldy,
                  const float* res, int epi) {
    if (!nf) { gemm1(w, sc, N, K, out, ldy, res, epi); return; }
    {
      ProfScope ps(s, PC_OTHER, (double)nf4_bytes(N, K) + 2.0 * N * K, 0, st);
      launch_nf4_split((const uint8_t*)w, sc, N, K, s->nf4_hi, s->nf4_lo, s->nf4_sc, st);
    }
    const bool act = (epi == EPI_SWIGLU || epi == EPI_GELU);
    float* o1 = act ? s->mlp_raw : out;
    const int64_t ld1 = act ? N : ldy;
    gemm1(s->nf4_hi, s->nf4_sc, N, K, o1, ld1, res, epi == EPI_RESID ? EPI_RESID : EPI_STORE);
    gemm1(s->nf4_lo, sc, N, K, o1, ld1, o1, EPI_RESID);
    if (epi == EPI_SWIGLU) launch_swiglu_rows(s->mlp_raw, out, R, N / 2, st);
    else if (epi == EPI_GELU) launch_gelu_rows(s->mlp_raw, out, R, N, st);
  };
  auto digit = [&](const float* x, int64_t K, int nm, const float* gg, const float* bb) {
    ProfScope ps(s, PC_OTHER, 4.0 * R * K + 2.0 * Mp * K * eb, 0, st);
    if (bf) launch_digitize_bf16(x, K, R, K, nm, gg, bb, s->planes, Mp * K * eb, st);
    else launch_digitize(x, K, R, K, nm, gg, bb, s->planes, Mp * K, s->exps, st);
  };
  for (int b = b0 - s->start; b < b1 - s->start; ++b) {
    BlockW& W = s->blocks[b];
    at.kv_pool = s->pool + (int64_t)b * s->block_stride;
    if (record)
      SP_CUDA_TRY(cudaMemcpyAsync(record + (int64_t)(b - (b0 - s->start)) * R * d, y,
                                  R * d * sizeof(float), cudaMemcpyDeviceToDevice, st));
    digit(y, d, norm, W.ln1_g, W.ln1_b);
    gemm(W.qkv, W.s_qkv, s->n_qkv, d, s->qkvb, s->n_qkv, nullptr, EPI_STORE);
    {
      ProfScope ps(s, PC_OTHER, 4.0 * R * s->n_qkv + (double)R * 2 * s->kv * kv_elt, 0, st);
      launch_rope_append(at, st);
    }
    {
      const double pairs = (double)width * ((double)n_new * kv->length +
                                            (double)n_new * (n_new + 1) / 2);
      ProfScope ps(s, PC_ATTN_PRE, (double)width * (kv->length + n_new) * 2 * s->kv * kv_elt,
                   4.0 * pairs * s->H * s->hd, st);
      if (!launch_attention_prefill_tc(at, st) && !launch_attention_prefill_mma(at, st))
        launch_attention_prefill(at, st);
    }
    digit(s->ctx, d, 0, nullptr, nullptr);
    gemm(W.o, W.s_o, d, d, y, d, y, EPI_RESID);
    digit(y, d, norm, W.ln2_g, W.ln2_b);
    gemm(W.up, W.s_up, s->n_up, d, s->mlp, F, nullptr, fam == kLlama ? EPI_SWIGLU : EPI_GELU);
    digit(s->mlp, F, 0, nullptr, nullptr);
    gemm(W.down, W.s_down, d, F, y, d, y, EPI_RESID);
  }
  SP_CHECK_LAUNCH();
  return SP_OK;
}

// Wide decode (n_new == 1, width >= g_wide_from rows, int8): the linears run
// on the tcgen05 GEMM (one pass over the weights for all rows, 15-bit digit
// planes) instead of the GEMV, whose per-unit digit/MMA work makes it
// latency-bound beyond a few rows; attention stays the fused decode kernel.
// Up to 8 rows (one GEMV launch) every row's result is bit-identical whatever
// the width (tests/test_gpu_span.py::test_decode_width_invariant); from 9 rows
// the GEMM computes the same exact integer products of the same 15-bit codes
// but folds the norm in its own reduction order (last-bit differences).
// option 11: the row count from which decode takes the GEMM path.  Up to 32 rows
// the weight-side GEMM reproduces the GEMV's numerics exactly (a row's result
// does not depend on the path), and from 3 rows it is faster (the GEMV's
// per-unit digit work makes it latency-bound beyond two rows): BLOOM-176B shape
// batch 8 125.6 -> 207.1, 70B batch 8 253.9 -> 501.8 steps/s per 8 blocks
int g_wide_from = getenv("SP_WIDE_FROM") ? atoi(getenv("SP_WIDE_FROM")) : 3;

int run_span_decode_wide(sp_span* s, sp_kv* kv, int b0, int b1, float* y, int width,
                         cudaStream_t st) {
  const int64_t R = width;
  int rc = ensure_scratch(s, R);
  if (rc) return rc;
  rc = ensure_decode(s, R);
  if (rc) return rc;
  rc = ensure_tc(s, R);
  if (rc) return rc;
  const int fam = s->cfg.family;
  const int norm = fam == kLlama ? 1 : 2;
  const bool bf = false;                          // int8 only (split-K is integer)
  const int64_t eb = 1;
  const int64_t d = s->d, F = s->F;
  const int64_t Mp = tc_rows(R);
  const double kv_elt = s->cfg.kv_dtype == kKVBF16 ? 2.0 : 4.0;
  AttnDecArgs at{};
  at.family = fam; at.kv_dtype = s->cfg.kv_dtype; at.width = width; at.t0 = kv->length;
  at.H = s->H; at.kvh = s->kvh; at.hd = s->hd; at.qkv = s->qkvb; at.ldqkv = s->n_qkv;
  at.page_table = kv->d_table; at.max_pages = s->max_pages;
  at.rope_cos = s->rope_cos; at.rope_sin = s->rope_sin; at.alibi = s->alibi;
  at.ctx = s->ctx; at.part = s->attn_part; at.counters = s->attn_cnt; at.st_out = nullptr;
  auto gemm = [&](void* w, float* sc, int64_t N, int64_t K, float* out, int64_t ldy,
                  const float* res, int epi) {
    ProfScope ps(s, PC_GEMV, (double)N * K + 4.0 * N + 2.0 * Mp * K + 4.0 * R * ldy,
                 2.0 * R * N * K, st);
    TcGemmArgs g{};
    g.w = w; g.wscale = sc; g.N = N; g.K = K; g.planes = s->planes; g.plane_stride = Mp * K;
    g.exps = s->exps; g.M = R; g.y = out; g.ldy = ldy; g.res = res; g.epi = epi;
    g.ws = s->ws2; g.counters = s->cnt2;      // split-K workspace (the GEMV's, zero at rest)
    launch_gemm_i8_tc(g, st);
  };
  auto digit = [&](const float* x, int64_t K, int nm, const float* gg, const float* bb) {
    ProfScope ps(s, PC_OTHER, 4.0 * R * K + 2.0 * Mp * K * eb, 0, st);
    if (bf) launch_digitize_bf16(x, K, R, K, nm, gg, bb, s->planes, Mp * K * eb, st);
    else launch_digitize(x, K, R, K, nm, gg, bb, s->planes, Mp * K, s->exps, st,
                         wide_rows(R) ? wide_rows(R) : 128);   // the GEMM's row tile
  };
  const int rt = wide_rows(R);
  if (rt && s->gains_one) {
    // up to 32 rows: the decode GEMV's numerics on the weight-side GEMM — the
    // same statistics partials, activation code, double-precision scale and
    // epilogue order, so every row equals what the GEMV gives it at any width
    // (tests/test_gpu_span.py::test_decode_width_invariant)
    auto st4 = [](RowStat* p) { return reinterpret_cast<float4*>(p); };
    auto gemm_g = [&](void* w, float* sc, int64_t N, int64_t K, float* out, int64_t ldy,
                      const float* res, int epi, RowStat* st_out, const float* g_next) {
      ProfScope ps(s, PC_GEMV, (double)N * K + 4.0 * N + 2.0 * Mp * K + 4.0 * R * ldy,
                   2.0 * R * N * K, st);
      TcGemmArgs g{};
      g.w = w; g.wscale = sc; g.N = N; g.K = K; g.planes = s->planes; g.plane_stride = Mp * K;
      g.exps = s->exps; g.M = R; g.y = out; g.ldy = ldy; g.res = res; g.epi = epi;
      g.ws = s->ws2; g.counters = s->cnt2;
      g.ys_rows = s->ys_rows; g.st_out = st_out ? st4(st_out) : nullptr; g.g_next = g_next;
      g.stat_rs = R;
      launch_gemm_i8_tc(g, st);
    };
    auto digit_g = [&](const float* x, int64_t K, int nm, const RowStat* st_in, int P_in) {
      ProfScope ps(s, PC_OTHER, 4.0 * R * K + 2.0 * Mp * K, 0, st);
      launch_digitize_gemv(x, K, R, K, nm, nullptr, reinterpret_cast<const float4*>(st_in),
                           P_in, 1.0f, 1e-5f, s->planes, Mp * K, s->ys_rows, rt, st);
    };
    {
      ProfScope ps(s, PC_OTHER, 4.0 * R * d, 0, st);
      launch_row_stats(y, (int)R, d, nullptr, s->st_norm1, st);
    }
    at.st_out = s->st_ctx;
    for (int b = b0 - s->start; b < b1 - s->start; ++b) {
      BlockW& W = s->blocks[b];
      const bool last = (b == b1 - s->start - 1);
      digit_g(y, d, norm, s->st_norm1, (int)(d / 128));
      gemm_g(W.qkv, W.s_qkv, s->n_qkv, d, s->qkvb, s->n_qkv, nullptr, EPI_STORE, nullptr,
             nullptr);
      at.kv_pool = s->pool + (int64_t)b * s->block_stride;
      int p_ctx;
      {
        ProfScope ps(s, PC_ATTN_DEC, (double)width * (kv->length + 1) * 2 * s->kv * kv_elt,
                     4.0 * width * (kv->length + 1) * s->H * s->hd, st);
        p_ctx = launch_attn_decode_fused(at, st);
      }
      digit_g(s->ctx, d, NORM_NONE, s->st_ctx, p_ctx);
      gemm_g(W.o, W.s_o, d, d, y, d, y, EPI_RESID, s->st_norm2, nullptr);
      digit_g(y, d, norm, s->st_norm2, (int)(d / 128));
      gemm_g(W.up, W.s_up, s->n_up, d, s->mlp, F, nullptr,
             fam == kLlama ? EPI_SWIGLU : EPI_GELU, s->st_mlp, nullptr);
      digit_g(s->mlp, F, NORM_NONE, s->st_mlp, (int)(s->n_up / 128));
      gemm_g(W.down, W.s_down, d, F, y, d, y, EPI_RESID, last ? nullptr : s->st_norm1,
             nullptr);
    }
    SP_CHECK_LAUNCH();
    return SP_OK;
  }
  for (int b = b0 - s->start; b < b1 - s->start; ++b) {
    BlockW& W = s->blocks[b];
    digit(y, d, norm, W.ln1_g, W.ln1_b);
    gemm(W.qkv, W.s_qkv, s->n_qkv, d, s->qkvb, s->n_qkv, nullptr, EPI_STORE);
    at.kv_pool = s->pool + (int64_t)b * s->block_stride;
    {
      ProfScope ps(s, PC_ATTN_DEC, (double)width * (kv->length + 1) * 2 * s->kv * kv_elt,
                   4.0 * width * (kv->length + 1) * s->H * s->hd, st);
      launch_attn_decode_fused(at, st);
    }
    digit(s->ctx, d, 0, nullptr, nullptr);
    gemm(W.o, W.s_o, d, d, y, d, y, EPI_RESID);
    digit(y, d, norm, W.ln2_g, W.ln2_b);
    gemm(W.up, W.s_up, s->n_up, d, s->mlp, F, nullptr, fam == kLlama ? EPI_SWIGLU : EPI_GELU);
    digit(s->mlp, F, 0, nullptr, nullptr);
    gemm(W.down, W.s_down, d, F, y, d, y, EPI_RESID);
  }
  SP_CHECK_LAUNCH();
  return SP_OK;
}

int run_span(sp_span* s, sp_kv* kv, int b0, int b1, float* y, float* record, int width,
             int n_new, cudaStream_t st) {
  if (n_new == 1 && width >= (g_wide_from > 1 ? g_wide_from : 2) && tc_ok(s) && s->cfg.weight_dtype == kI8 &&
      s->use_tc_prefill && !record)
    return run_span_decode_wide(s, kv, b0, b1, y, width, st);
  if (n_new == 1 && s->cfg.weight_dtype != kF32 && !record)
    return run_span_decode_tc(s, kv, b0, b1, y, width, st);
  if (n_new > 1 && tc_ok(s) && s->use_tc_prefill)
    return run_span_prefill_tc(s, kv, b0, b1, y, record, width, n_new, st);
  const int64_t R = (int64_t)width * n_new;
  const bool decode = (n_new == 1);
  const int wd = s->cfg.weight_dtype;
  const int fam = s->cfg.family;
  int rc = ensure_scratch(s, R);
  if (rc) return rc;
  rc = ensure_attn_ws(s, width);
  if (rc) return rc;
  AttnArgs at{};
  at.family = fam; at.kv_dtype = s->cfg.kv_dtype;
  at.width = width; at.n_new = n_new; at.t0 = kv->length;
  at.H = s->H; at.kvh = s->kvh; at.hd = s->hd;
  at.qkv = s->qkvb; at.ldqkv = s->n_qkv;
  at.page_table = kv->d_table; at.max_pages = s->max_pages;
  at.rope_cos = s->rope_cos; at.rope_sin = s->rope_sin; at.alibi = s->alibi;
  at.ctx = s->ctx; at.workspace = s->attn_ws;
  at.pool_base = s->pool; at.pool_bytes = s->block_stride * (s->end - s->start);
  const int64_t d = s->d, F = s->F;
  const double kv_elt = s->cfg.kv_dtype == kKVBF16 ? 2.0 : 4.0;
  for (int b = b0 - s->start; b < b1 - s->start; ++b) {
    BlockW& W = s->blocks[b];
    at.kv_pool = s->pool + (int64_t)b * s->block_stride;
    if (record)
      SP_CUDA_TRY(cudaMemcpyAsync(record + (int64_t)(b - (b0 - s->start)) * R * d, y,
                                  R * d * sizeof(float), cudaMemcpyDeviceToDevice, st));
    {
      ProfScope ps(s, PC_OTHER, 8.0 * R * d, 0, st);
      launch_norm(fam, y, W.ln1_g, W.ln1_b, s->h, R, d, st);
    }
    linear(s, wd, W.qkv, W.s_qkv, s->n_qkv, d, s->h, s->qkvb, s->n_qkv, nullptr, EPI_STORE, R,
           decode, st);
    {
      ProfScope ps(s, PC_OTHER, 4.0 * R * s->n_qkv + (double)R * 2 * s->kv * kv_elt, 0, st);
      launch_rope_append(at, st);
    }
    {
      // keys visible to all new rows: width * sum_i (t0 + i + 1)
      const double pairs = (double)width * ((double)n_new * kv->length +
                                            (double)n_new * (n_new + 1) / 2);
      const double kvbytes = decode ? (double)width * (kv->length + 1) * 2 * s->kv * kv_elt
                                    : (double)width * (kv->length + n_new) * 2 * s->kv * kv_elt;
      ProfScope ps(s, decode ? PC_ATTN_DEC : PC_ATTN_PRE, kvbytes + 8.0 * R * d,
                   4.0 * pairs * s->H * s->hd, st);
      if (decode) launch_attention_decode(at, st);
      else if (!launch_attention_prefill_tc(at, st) && !launch_attention_prefill_mma(at, st))
        launch_attention_prefill(at, st);
    }
    linear(s, wd, W.o, W.s_o, d, d, s->ctx, y, d, y, EPI_RESID, R, decode, st);
    {
      ProfScope ps(s, PC_OTHER, 8.0 * R * d, 0, st);
      launch_norm(fam, y, W.ln2_g, W.ln2_b, s->h, R, d, st);
    }
    if (fam == kLlama)
      linear(s, wd, W.up, W.s_up, s->n_up, d, s->h, s->mlp, F, nullptr, EPI_SWIGLU, R, decode,
             st);
    else
      linear(s, wd, W.up, W.s_up, s->n_up, d, s->h, s->mlp, F, nullptr, EPI_GELU, R, decode, st);
    linear(s, wd, W.down, W.s_down, d, F, s->mlp, y, d, y, EPI_RESID, R, decode, st);
  }
  SP_CHECK_LAUNCH();
  return SP_OK;
}

}  // namespace

extern "C" {

const char* sp_last_error(void) { return g_err.c_str(); }
int sp_version(void) { return 1; }

uint64_t sp_stream_seed(uint64_t seed, int32_t block, int32_t role_id) {
  return stream_seed(seed, block, role_id);
}

int sp_quantize_blockwise(const float* x, int8_t* codes, float* scales, int64_t n,
                          void* stream) {
  if (n < 0) SP_FAIL(SP_ERR_ARG, "negative length");
  launch_quantize(x, codes, scales, n, (cudaStream_t)stream);
  SP_CHECK_LAUNCH();
  return SP_OK;
}

int sp_dequantize_blockwise(const int8_t* codes, const float* scales, float* x, int64_t n,
                            void* stream) {
  if (n < 0) SP_FAIL(SP_ERR_ARG, "negative length");
  launch_dequantize(codes, scales, x, n, (cudaStream_t)stream);
  SP_CHECK_LAUNCH();
  return SP_OK;
}

int sp_weights_generate(uint64_t seed, int32_t block, int32_t role_id, int64_t n_elements,
                        double scale, float* dst, void* stream) {
  launch_gen_stream(stream_seed(seed, block, role_id), n_elements, scale, dst,
                    (cudaStream_t)stream);
  SP_CHECK_LAUNCH();
  return SP_OK;
}

int sp_span_create(const sp_config* cfg, int32_t start, int32_t end, int32_t device,
                   int64_t kv_pool_tokens, sp_span** out) {
  if (!cfg || !out) SP_FAIL(SP_ERR_ARG, "null argument");
  if (validate(cfg) != SP_OK) SP_FAIL(SP_ERR_ARG, "unsupported config shape");
  if (!(0 <= start && start < end && end <= cfg->n_blocks)) SP_FAIL(SP_ERR_ARG, "bad span");
  DeviceGuard dg(device);
  sp_span* s = new sp_span();
  s->cfg = *cfg;
  s->start = start; s->end = end; s->device = device;
  s->d = cfg->hidden_dim; s->H = cfg->n_heads;
  s->kvh = cfg->n_kv_heads ? cfg->n_kv_heads : cfg->n_heads;
  s->hd = s->d / s->H;
  s->F = cfg->ffn_dim ? cfg->ffn_dim : 4 * s->d;
  s->kv = s->kvh * s->hd;
  s->n_qkv = s->d + 2 * s->kv;
  s->n_up = cfg->family == kLlama ? 2 * (int64_t)s->F : s->F;
  const int wd = cfg->weight_dtype;
  const int64_t eb = elt_bytes(wd);
  const int nb = end - start;
  const int64_t d = s->d, F = s->F;

  // ---- weights: one allocation per span ----
  auto mat_bytes = [&](int64_t N, int64_t K) {
    return align_up(wd == kNF4 ? (size_t)nf4_bytes(N, K) : (size_t)(N * K * eb), 256);
  };
  auto sc_bytes = [&](int64_t N) {
    return (wd == kI8 || wd == kNF4) ? align_up((size_t)N * 4, 256) : 0;
  };
  size_t per_block = mat_bytes(s->n_qkv, d) + sc_bytes(s->n_qkv) + mat_bytes(d, d) + sc_bytes(d) +
                     mat_bytes(s->n_up, d) + sc_bytes(s->n_up) + mat_bytes(d, F) + sc_bytes(d) +
                     4 * align_up((size_t)d * 4, 256);
  s->weight_bytes = (int64_t)per_block * nb;
  cudaError_t e = cudaMalloc(&s->wmem, s->weight_bytes);
  if (e != cudaSuccess) {
    delete s;
    SP_FAIL(SP_ERR_OOM, "weight allocation failed");
  }
  cudaStream_t st = 0;
  const double scale = 1.0 / std::sqrt((double)d);   // SP/model.py:181
  std::vector<float> ones(d, 1.0f);
  char* p = s->wmem;
  for (int b = start; b < end; ++b) {
    BlockW W{};
    auto take = [&](size_t bytes) { char* r = p; p += bytes; return (void*)r; };
    W.qkv = take(mat_bytes(s->n_qkv, d)); W.s_qkv = (float*)take(sc_bytes(s->n_qkv));
    W.o = take(mat_bytes(d, d)); W.s_o = (float*)take(sc_bytes(d));
    W.up = take(mat_bytes(s->n_up, d)); W.s_up = (float*)take(sc_bytes(s->n_up));
    W.down = take(mat_bytes(d, F)); W.s_down = (float*)take(sc_bytes(d));
    W.ln1_g = (float*)take(align_up(d * 4, 256)); W.ln1_b = (float*)take(align_up(d * 4, 256));
    W.ln2_g = (float*)take(align_up(d * 4, 256)); W.ln2_b = (float*)take(align_up(d * 4, 256));
    uint64_t seed = cfg->seed;
    launch_gen_matrix(wd, stream_seed(seed, b, R_WQ), d, d, scale, MatPlace{0, 1, 0}, W.qkv, W.s_qkv, st, s->n_qkv);
    launch_gen_matrix(wd, stream_seed(seed, b, R_WK), d, s->kv, scale, MatPlace{d, 1, 0}, W.qkv, W.s_qkv, st, s->n_qkv);
    launch_gen_matrix(wd, stream_seed(seed, b, R_WV), d, s->kv, scale, MatPlace{d + s->kv, 1, 0}, W.qkv, W.s_qkv, st, s->n_qkv);
    launch_gen_matrix(wd, stream_seed(seed, b, R_WO), d, d, scale, MatPlace{0, 1, 0}, W.o, W.s_o, st, d);
    if (cfg->family == kLlama) {
      launch_gen_matrix(wd, stream_seed(seed, b, R_W1), d, F, scale, MatPlace{0, 2, 0}, W.up, W.s_up, st, s->n_up);
      launch_gen_matrix(wd, stream_seed(seed, b, R_W3), d, F, scale, MatPlace{0, 2, 1}, W.up, W.s_up, st, s->n_up);
    } else {
      launch_gen_matrix(wd, stream_seed(seed, b, R_W1), d, F, scale, MatPlace{0, 1, 0}, W.up, W.s_up, st, s->n_up);
    }
    launch_gen_matrix(wd, stream_seed(seed, b, R_W2), F, d, scale, MatPlace{0, 1, 0}, W.down, W.s_down, st, d);
    SP_CUDA_TRY(cudaMemcpy(W.ln1_g, ones.data(), d * 4, cudaMemcpyHostToDevice));
    SP_CUDA_TRY(cudaMemcpy(W.ln2_g, ones.data(), d * 4, cudaMemcpyHostToDevice));
    SP_CUDA_TRY(cudaMemset(W.ln1_b, 0, d * 4));
    SP_CUDA_TRY(cudaMemset(W.ln2_b, 0, d * 4));
    s->blocks.push_back(W);
  }
  SP_CHECK_LAUNCH();

  // ---- constant tables ----
  if (cfg->family == kLlama) {
    int half = s->hd / 2;
    std::vector<float> c((size_t)cfg->max_seq_len * half), sn((size_t)cfg->max_seq_len * half);
    for (int pos = 0; pos < cfg->max_seq_len; ++pos)
      for (int j = 0; j < half; ++j) {
        double inv = std::pow(cfg->rope_theta, -((double)(2 * j) / (double)s->hd));
        double ang = (double)pos * inv;
        c[(size_t)pos * half + j] = (float)std::cos(ang);
        sn[(size_t)pos * half + j] = (float)std::sin(ang);
      }
    SP_CUDA_TRY(cudaMalloc(&s->rope_cos, c.size() * 4));
    SP_CUDA_TRY(cudaMalloc(&s->rope_sin, sn.size() * 4));
    SP_CUDA_TRY(cudaMemcpy(s->rope_cos, c.data(), c.size() * 4, cudaMemcpyHostToDevice));
    SP_CUDA_TRY(cudaMemcpy(s->rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
  }
  if (cfg->family == kBloom) {
    int n = s->H;
    auto pow2 = [](int m) {
      std::vector<double> v;
      double start = std::pow(2.0, -std::pow(2.0, -(std::log2((double)m) - 3)));
      for (int i = 0; i < m; ++i) v.push_back(start * std::pow(start, i));
      return v;
    };
    int p2 = 1;
    while (p2 * 2 <= n) p2 *= 2;
    std::vector<double> sl = pow2(p2);
    if (p2 < n) {
      std::vector<double> ex = pow2(2 * p2);
      for (int i = 0; i < n - p2; ++i) sl.push_back(ex[2 * i]);
    }
    std::vector<float> f(sl.begin(), sl.end());
    SP_CUDA_TRY(cudaMalloc(&s->alibi, f.size() * 4));
    SP_CUDA_TRY(cudaMemcpy(s->alibi, f.data(), f.size() * 4, cudaMemcpyHostToDevice));
  }

  // ---- KV pool ----
  const int kvel = cfg->kv_dtype == kKVBF16 ? 2 : 4;
  s->page_bytes = (int64_t)2 * s->kvh * kPageTokens * s->hd * kvel;
  s->n_pages = (kv_pool_tokens + kPageTokens - 1) / kPageTokens;
  if (s->n_pages < 1) s->n_pages = 1;
  s->block_stride = s->n_pages * s->page_bytes;
  s->max_pages = (cfg->max_seq_len + kPageTokens - 1) / kPageTokens;
  e = cudaMalloc(&s->pool, (size_t)s->block_stride * nb);
  if (e != cudaSuccess) {
    sp_span_destroy(s);
    SP_FAIL(SP_ERR_OOM, "KV pool allocation failed");
  }
  // finite contents everywhere: attention tiles read whole pages, and the rows
  // past a sequence's end (multiplied by zero probabilities) must not be NaN
  SP_CUDA_TRY(cudaMemset(s->pool, 0, (size_t)s->block_stride * nb));
  s->refcount.assign(s->n_pages, 0);
  for (int64_t i = s->n_pages - 1; i >= 0; --i) s->free_pages.push_back((int)i);

  SP_CUDA_TRY(cudaDeviceSynchronize());
  *out = s;
  return SP_OK;
}

static void free_span_device(sp_span* s) {
  DeviceGuard dg(s->device);
  cudaFree(s->wmem); cudaFree(s->rope_cos); cudaFree(s->rope_sin); cudaFree(s->alibi);
  cudaFree(s->pool); cudaFree(s->h); cudaFree(s->qkvb); cudaFree(s->ctx); cudaFree(s->mlp);
  cudaFree(s->mlp_raw); cudaFree(s->gemv_ws); cudaFree(s->gemv_cnt); cudaFree(s->attn_ws);
  cudaFree(s->st_norm1); cudaFree(s->st_ctx); cudaFree(s->st_norm2); cudaFree(s->st_mlp);
  cudaFree(s->ws2); cudaFree(s->cnt2); cudaFree(s->attn_part); cudaFree(s->attn_cnt);
  cudaFree(s->planes); cudaFree(s->exps); cudaFree(s->ys_rows);
  cudaFree(s->nf4_hi); cudaFree(s->nf4_lo); cudaFree(s->nf4_sc);
  for (auto& r : s->prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : s->ev_pool) cudaEventDestroy(e);
  if (s->done) cudaEventDestroy(s->done);
  s->wmem = s->pool = nullptr;
  s->rope_cos = s->rope_sin = s->alibi = nullptr;
  s->h = s->qkvb = s->ctx = s->mlp = s->mlp_raw = s->gemv_ws = s->attn_ws = nullptr;
  s->st_norm1 = s->st_ctx = s->st_norm2 = s->st_mlp = nullptr;
  s->ws2 = nullptr; s->cnt2 = s->gemv_cnt = s->attn_cnt = s->exps = nullptr;
  s->ys_rows = nullptr;
  s->attn_part = nullptr; s->planes = nullptr;
  s->nf4_hi = s->nf4_lo = nullptr; s->nf4_sc = nullptr;
  s->prof_recs.clear(); s->ev_pool.clear(); s->done = nullptr;
}

int sp_span_destroy(sp_span* s) {
  if (!s) return SP_OK;
  bool keep;
  {
    std::lock_guard<std::mutex> g(s->mu);
    if (s->dying) return SP_OK;
    s->dying = true;
    keep = s->live_kv > 0;
  }
  free_span_device(s);
  if (!keep) delete s;
  return SP_OK;
}

int64_t sp_span_weight_bytes(const sp_span* s) { return s ? s->weight_bytes : 0; }
int64_t sp_span_free_pages(const sp_span* s) { return s ? (int64_t)s->free_pages.size() : 0; }

int sp_span_read_weight(sp_span* s, int32_t block, int32_t role, float* dst_host) {
  if (!s || block < s->start || block >= s->end) SP_FAIL(SP_ERR_ARG, "block outside span");
  DeviceGuard dg(s->device);
  BlockW& W = s->blocks[block - s->start];
  const int64_t d = s->d, F = s->F;
  void* src = nullptr; float* sc = nullptr; int64_t K = 0, N = 0; MatPlace pl{0, 1, 0};
  int64_t bufK = 0, bufN = 0;
  switch (role) {
    case R_WQ: src = W.qkv; sc = W.s_qkv; K = d; N = d; pl = {0, 1, 0}; bufN = s->n_qkv; break;
    case R_WK: src = W.qkv; sc = W.s_qkv; K = d; N = s->kv; pl = {d, 1, 0}; bufN = s->n_qkv; break;
    case R_WV: src = W.qkv; sc = W.s_qkv; K = d; N = s->kv; pl = {d + s->kv, 1, 0}; bufN = s->n_qkv; break;
    case R_WO: src = W.o; sc = W.s_o; K = d; N = d; bufN = d; break;
    case R_W1: src = W.up; sc = W.s_up; K = d; N = F; bufN = s->n_up;
      pl = (s->cfg.family == kLlama) ? MatPlace{0, 2, 0} : MatPlace{0, 1, 0}; break;
    case R_W3: if (s->cfg.family != kLlama) SP_FAIL(SP_ERR_ARG, "no w3");
      src = W.up; sc = W.s_up; K = d; N = F; pl = {0, 2, 1}; bufN = s->n_up; break;
    case R_W2: src = W.down; sc = W.s_down; K = F; N = d; bufN = d; break;
    default: SP_FAIL(SP_ERR_ARG, "unknown role");
  }
  (void)bufK;
  float* tmp = nullptr;
  SP_CUDA_TRY(cudaMalloc(&tmp, K * N * sizeof(float)));
  launch_read_matrix(s->cfg.weight_dtype, src, sc, K, N, pl, tmp, 0, bufN);
  SP_CHECK_LAUNCH();
  SP_CUDA_TRY(cudaMemcpy(dst_host, tmp, K * N * sizeof(float), cudaMemcpyDeviceToHost));
  cudaFree(tmp);
  return SP_OK;
}

int sp_kv_create(sp_span* s, int32_t width, sp_kv** out) {
  if (!s || !out || width < 1) SP_FAIL(SP_ERR_ARG, "bad kv args");
  {
    std::lock_guard<std::mutex> g(s->mu);
    if (s->dying) SP_FAIL(SP_ERR_STATE, "span destroyed");
    ++s->live_kv;
  }
  sp_kv* kv = new sp_kv();
  kv->span = s;
  kv->width = width;
  kv->length = 0;
  kv->pages.assign(width, {});
  *out = kv;
  return SP_OK;
}

int sp_kv_destroy(sp_kv* kv) {
  if (!kv) return SP_OK;
  sp_span* s = kv->span;
  bool last;
  {
    std::lock_guard<std::mutex> g(s->mu);
    for (auto& pg : kv->pages)
      for (int p : pg) release_page(s, p);
    last = --s->live_kv == 0 && s->dying;
  }
  {
    DeviceGuard dg(s->device);
    if (kv->table_ev) {
      cudaEventSynchronize(kv->table_ev);
      cudaEventDestroy(kv->table_ev);
    }
    cudaFree(kv->d_table);
    cudaFreeHost(kv->h_table);
  }
  delete kv;
  if (last) delete s;
  return SP_OK;
}

int32_t sp_kv_length(const sp_kv* kv) { return kv ? kv->length : -1; }
int32_t sp_kv_width(const sp_kv* kv) { return kv ? kv->width : -1; }

int sp_kv_reorder(sp_kv* kv, const int32_t* parents0, int32_t new_width, void* stream) {
  if (!kv || new_width < 1) SP_FAIL(SP_ERR_ARG, "bad reorder args");
  for (int i = 0; i < new_width; ++i)
    if (parents0[i] < 0 || parents0[i] >= kv->width)
      SP_FAIL(SP_ERR_ARG, "reorder index out of range");
  sp_span* s = kv->span;
  std::lock_guard<std::mutex> g(s->mu);
  std::vector<std::vector<int>> np(new_width);
  for (int i = 0; i < new_width; ++i) {
    np[i] = kv->pages[parents0[i]];
    for (int p : np[i]) s->refcount[p]++;
  }
  for (auto& pg : kv->pages)
    for (int p : pg) release_page(s, p);
  kv->pages.swap(np);
  kv->width = new_width;
  DeviceGuard dg(s->device);
  return upload_table(kv, (cudaStream_t)stream);
}

int sp_kv_read(sp_kv* kv, int32_t block, int32_t slot, float* keys_host, float* values_host) {
  if (!kv) SP_FAIL(SP_ERR_ARG, "null kv");
  sp_span* s = kv->span;
  if (block < s->start || block >= s->end || slot < 0 || slot >= kv->width)
    SP_FAIL(SP_ERR_ARG, "block/slot out of range");
  block -= s->start;
  if (s->dying) SP_FAIL(SP_ERR_STATE, "span destroyed");
  DeviceGuard dg(s->device);
  int64_t n = (int64_t)kv->length * s->kvh * s->hd;
  if (n == 0) return SP_OK;
  float *k = nullptr, *v = nullptr;
  SP_CUDA_TRY(cudaMalloc(&k, n * 4));
  SP_CUDA_TRY(cudaMalloc(&v, n * 4));
  launch_kv_gather_slot(s->pool + (int64_t)block * s->block_stride, s->cfg.kv_dtype,
                        kv->d_table + (int64_t)slot * s->max_pages, kv->length, s->kvh, s->hd, k,
                        v, 0);
  SP_CHECK_LAUNCH();
  SP_CUDA_TRY(cudaMemcpy(keys_host, k, n * 4, cudaMemcpyDeviceToHost));
  SP_CUDA_TRY(cudaMemcpy(values_host, v, n * 4, cudaMemcpyDeviceToHost));
  cudaFree(k);
  cudaFree(v);
  return SP_OK;
}

static int forward_impl(sp_span* s, sp_kv* kv, int32_t b0, int32_t b1, const float* x,
                        const int8_t* x_codes, const float* x_scales, float* y, float* record,
                        int8_t* y_codes, float* y_scales, int32_t width, int32_t n_new,
                        void* stream) {
  if (!s || !kv || !y) SP_FAIL(SP_ERR_ARG, "null argument");
  DeviceGuard dg(s->device);
  if (!(s->start <= b0 && b0 < b1 && b1 <= s->end)) SP_FAIL(SP_ERR_ARG, "blocks outside span");
  if (width != kv->width) SP_FAIL(SP_ERR_STATE, "width mismatch");
  if (n_new < 1) SP_FAIL(SP_ERR_ARG, "n_new must be >= 1");
  if (kv->length + n_new > s->cfg.max_seq_len) SP_FAIL(SP_ERR_CAPACITY, "exceeds max_seq_len");
  cudaStream_t st = (cudaStream_t)stream;
  std::lock_guard<std::mutex> g(s->mu);
  if (s->dying) SP_FAIL(SP_ERR_STATE, "span destroyed");
  int rc = order_begin(s, st);
  if (rc) return rc;
  rc = prepare_pages(kv, n_new, st);
  if (rc) return rc;
  const int64_t n = (int64_t)width * n_new * s->d;
  if (x_codes) {
    launch_dequantize(x_codes, x_scales, y, n, st);
  } else if (x != y) {
    SP_CUDA_TRY(cudaMemcpyAsync(y, x, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  rc = run_span(s, kv, b0, b1, y, record, width, n_new, st);
  if (rc) {
    order_end(s, st);
    return rc;
  }
  kv->length += n_new;
  if (y_codes) launch_quantize(y, y_codes, y_scales, n, st);
  SP_CHECK_LAUNCH();
  return order_end(s, st);
}

int sp_span_forward(sp_span* s, sp_kv* kv, int32_t b0, int32_t b1, const float* x,
                    const int8_t* x_codes, const float* x_scales, float* y, int8_t* y_codes,
                    float* y_scales, int32_t width, int32_t n_new, void* stream) {
  return forward_impl(s, kv, b0, b1, x, x_codes, x_scales, y, nullptr, y_codes, y_scales, width,
                      n_new, stream);
}

int sp_span_forward_stateless(sp_span* s, int32_t b0, int32_t b1, const float* x, float* y,
                              float* record, int32_t batch, int32_t tokens, void* stream) {
  sp_kv* kv = nullptr;
  int rc = sp_kv_create(s, batch, &kv);
  if (rc) return rc;
  rc = forward_impl(s, kv, b0, b1, x, nullptr, nullptr, y, record, nullptr, nullptr, batch,
                    tokens, stream);
  if (rc == SP_OK) {
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) {
      sp_set_error(__FILE__, __LINE__, cudaGetErrorString(e));
      rc = SP_ERR_CUDA;
    }
  }
  sp_kv_destroy(kv);
  return rc;
}

int sp_span_block_backward(sp_span* s, int32_t block, const float* x, const float* dy, float* dx,
                           int32_t batch, int32_t tokens, void* stream) {
  if (!s || !x || !dy || !dx) SP_FAIL(SP_ERR_ARG, "null argument");
  if (block < s->start || block >= s->end) SP_FAIL(SP_ERR_ARG, "block outside span");
  if (batch < 1 || tokens < 1) SP_FAIL(SP_ERR_ARG, "empty batch");
  // the reference defines block_backward for its own family only (SP/model.py:320)
  if (s->cfg.weight_dtype != kF32 || s->cfg.family != kToy || s->kvh != s->H)
    SP_FAIL(SP_ERR_ARG, "backward is defined for the reference (toy) family only");
  DeviceGuard dg(s->device);
  BlockW& W = s->blocks[block - s->start];
  const int d = s->d;
  if (block_backward_f64((const float*)W.qkv, (const float*)W.o, (const float*)W.up,
                         (const float*)W.down, W.ln1_g, W.ln1_b, W.ln2_g, W.ln2_b, d, s->H, s->F,
                         x, dy, dx, batch, tokens, (cudaStream_t)stream))
    SP_FAIL(SP_ERR_CUDA, "backward scratch allocation failed");
  SP_CHECK_LAUNCH();
  return SP_OK;
}

int sp_span_set_option(sp_span* s, int32_t option, int32_t value) {
  if (!s) SP_FAIL(SP_ERR_ARG, "null span");
  if (option == 0) s->use_tc_prefill = value != 0;
  else if (option == 1) g_pdl = value != 0;
  else if (option == 2) g_tc_pair = value != 0;
  else if (option == 3) g_attn_hilo = value != 0;
  else if (option == 5) g_attn_nsub = value;
  else if (option == 6) g_attn_cluster = value;
  else if (option == 7) g_attn_cl = value != 0;
  else if (option == 8) g_attn_tc = value != 0;
  else if (option == 9) g_attn_mha = value != 0;
  else if (option == 10) g_tc_wide = value != 0;
  else if (option == 11) g_wide_from = value;
  else SP_FAIL(SP_ERR_ARG, "unknown option");
  return SP_OK;
}

int sp_span_set_profiling(sp_span* s, int32_t enable) {
  if (!s) SP_FAIL(SP_ERR_ARG, "null span");
  s->prof = enable != 0;
  return SP_OK;
}

int sp_span_profile_read(sp_span* s, int32_t n_classes, double* ms, double* bytes, double* flops,
                         int64_t* launches) {
  if (!s) SP_FAIL(SP_ERR_ARG, "null span");
  DeviceGuard dg(s->device);
  SP_CUDA_TRY(cudaDeviceSynchronize());
  for (int c = 0; c < n_classes; ++c) { ms[c] = 0; bytes[c] = 0; flops[c] = 0; launches[c] = 0; }
  for (auto& r : s->prof_recs) {
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.cls < n_classes) {
      ms[r.cls] += t; bytes[r.cls] += r.bytes; flops[r.cls] += r.flops; launches[r.cls] += 1;
    }
    s->ev_pool.push_back(r.a);
    s->ev_pool.push_back(r.b);
  }
  s->prof_recs.clear();
  return SP_OK;
}

int64_t sp_kernel_launches(void) { return sp::g_launches.load(); }

int sp_span_decode_gemv_only(sp_span* s, sp_kv* kv, int32_t b0, int32_t b1, float* y,
                             int32_t width, void* stream, double* weight_bytes) {
  if (!s || !kv || !y) SP_FAIL(SP_ERR_ARG, "null argument");
  if (s->cfg.weight_dtype == kF32) SP_FAIL(SP_ERR_ARG, "tensor-core decode path only");
  DeviceGuard dg(s->device);
  std::lock_guard<std::mutex> g(s->mu);
  if (s->dying) SP_FAIL(SP_ERR_STATE, "span destroyed");
  int rc = order_begin(s, (cudaStream_t)stream);
  if (rc) return rc;
  const int64_t d = s->d;
  double wb = 0;
  const int64_t shapes[4][2] = {{s->n_qkv, d}, {d, d}, {s->n_up, d}, {d, s->F}};
  for (auto& sh : shapes) wb += weight_bytes_of(s->cfg.weight_dtype, sh[0], sh[1]);
  if (weight_bytes) *weight_bytes = wb * (b1 - b0);
  rc = run_span_decode_tc(s, kv, b0, b1, y, width, (cudaStream_t)stream, true);
  int rc2 = order_end(s, (cudaStream_t)stream);
  return rc ? rc : rc2;
}

uint64_t sp_fnv1a64(const uint8_t* data, int64_t n) {
  uint64_t h = 0xCBF29CE484222325ull;  // SP/wire.py:35-44
  for (int64_t i = 0; i < n; ++i) {
    h ^= data[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

}  // extern "C"
