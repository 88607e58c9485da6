// Prompt-tuning backward through one block: the gradient of the block output
// wrt its input (`block_backward`, SP/model.py:320-381; engine protocol
// `backward`, SP/server.py:127-139).  Like the reference it recomputes the
// forward in float64 from the recorded input (full causal attention over the
// sequence, no KV history), backpropagates in float64 and rounds to float32
// once at the end; parameters are only read.  The reference defines it for its
// own model family (pre-norm LayerNorm, MHA, tanh-GELU MLP, f32 weights).
//
// Sizes are prompt-tuning sized (batch x (prompt + tokens) rows of the toy
// width), so the kernels are plain float64 SIMT: a strided GEMM (one thread
// per output), row-wise LayerNorm forward/backward, GELU, and one CTA per
// (sequence, head) for attention forward + backward.
#include "common.cuh"
#include "kernels.cuh"

namespace sp {

namespace {

constexpr double kLnEps = 1e-5;
constexpr double kGeluC = 0.7978845608028654;   // sqrt(2 / pi), SP/model.py:24

// C[m][n] (+)= sum_k A[m*am + k*ak] * B[k*bk + n*bn]
__global__ void dgemm_kernel(const double* A, int64_t am, int64_t ak, const double* B, int64_t bk,
                             int64_t bn, double* C, int64_t M, int64_t N, int64_t K, bool acc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * N) return;
  const int64_t m = i / N, n = i % N;
  double s = 0.0;
  for (int64_t k = 0; k < K; ++k) s = fma(A[m * am + k * ak], B[k * bk + n * bn], s);
  C[i] = acc ? C[i] + s : s;
}

__global__ void f2d_kernel(const float* x, double* y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = (double)x[i];
}

// LayerNorm over rows of width d (SP/model.py:222-225, population variance)
__global__ void ln_fwd_kernel(const double* x, const float* g, const float* b, double* out,
                              double* mu, double* inv, int64_t R, int d) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const double* xr = x + r * d;
  double s = 0.0;
  for (int k = 0; k < d; ++k) s += xr[k];
  const double m = s / d;
  double v = 0.0;
  for (int k = 0; k < d; ++k) v += (xr[k] - m) * (xr[k] - m);
  const double iv = 1.0 / sqrt(v / d + kLnEps);
  for (int k = 0; k < d; ++k) out[r * d + k] = (xr[k] - m) * iv * (double)g[k] + (double)b[k];
  mu[r] = m;
  inv[r] = iv;
}

// dx (+)= inv * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)), dxhat = dy * g
// (_ln_backward, SP/model.py:303-311); out = base + that
__global__ void ln_bwd_kernel(const double* x, const float* g, const double* mu,
                              const double* inv, const double* dy, const double* base,
                              double* out, int64_t R, int d) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const double m = mu[r], iv = inv[r];
  double s1 = 0.0, s2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const double xh = (x[r * d + k] - m) * iv, dxh = dy[r * d + k] * (double)g[k];
    s1 += dxh;
    s2 += dxh * xh;
  }
  s1 /= d;
  s2 /= d;
  for (int k = 0; k < d; ++k) {
    const double xh = (x[r * d + k] - m) * iv, dxh = dy[r * d + k] * (double)g[k];
    out[r * d + k] = base[r * d + k] + iv * (dxh - s1 - xh * s2);
  }
}

// da = dg * gelu'(a)   (_gelu_grad, SP/model.py:314-317)
__global__ void gelu_grad_kernel(const double* a, const double* dg, double* da, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = a[i];
  const double t = tanh(kGeluC * (x + 0.044715 * x * x * x));
  da[i] = dg[i] * (0.5 * (1.0 + t) +
                   0.5 * x * (1.0 - t * t) * kGeluC * (1.0 + 3 * 0.044715 * x * x));
}

__global__ void add_d2f_kernel(const double* a, float* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (float)a[i];
}

// One CTA per (sequence b, head h): causal attention forward (probabilities kept)
// and backward.  qkv rows [B*t][3d] (q | k | v), dctx [B*t][d] -> dqkv.
__global__ void attn_fb_kernel(const double* qkv, const double* dctx, double* ctx, double* dqkv,
                               double* P, int t, int d, int H, bool backward) {
  const int b = blockIdx.x / H, h = blockIdx.x % H;
  const int hd = d / H;
  const int64_t ld = 3 * (int64_t)d;
  const double* q = qkv + (int64_t)b * t * ld + h * hd;
  const double* k = q + d;
  const double* v = q + 2 * d;
  double* Pz = P + (int64_t)blockIdx.x * t * t;
  const double rs = sqrt((double)hd);
  if (!backward) {
    for (int i = threadIdx.x; i < t; i += blockDim.x) {
      double mx = -INFINITY;
      for (int j = 0; j <= i; ++j) {
        double s = 0.0;
        for (int e = 0; e < hd; ++e) s += q[(int64_t)i * ld + e] * k[(int64_t)j * ld + e];
        s /= rs;
        Pz[(int64_t)i * t + j] = s;
        mx = fmax(mx, s);
      }
      double sum = 0.0;
      for (int j = 0; j <= i; ++j) {
        const double e = exp(Pz[(int64_t)i * t + j] - mx);
        Pz[(int64_t)i * t + j] = e;
        sum += e;
      }
      for (int j = 0; j < t; ++j) Pz[(int64_t)i * t + j] = j <= i ? Pz[(int64_t)i * t + j] / sum : 0.0;
      for (int e = 0; e < hd; ++e) {
        double c = 0.0;
        for (int j = 0; j <= i; ++j) c += Pz[(int64_t)i * t + j] * v[(int64_t)j * ld + e];
        ctx[((int64_t)b * t + i) * d + h * hd + e] = c;
      }
    }
    return;
  }
  const double* dc = dctx + (int64_t)b * t * d + h * hd;
  double* dq = dqkv + (int64_t)b * t * ld + h * hd;
  double* dk = dq + d;
  double* dv = dq + 2 * d;
  double* DS = P + (int64_t)gridDim.x * t * t + (int64_t)blockIdx.x * t * t;   // dscores
  // dscores_ij = P_ij (dP_ij - sum_j' dP_ij' P_ij') / sqrt(hd), dP_ij = dctx_i . v_j
  for (int i = threadIdx.x; i < t; i += blockDim.x) {
    double rsum = 0.0;
    for (int j = 0; j <= i; ++j) {
      double da = 0.0;
      for (int e = 0; e < hd; ++e) da += dc[(int64_t)i * d + e] * v[(int64_t)j * ld + e];
      DS[(int64_t)i * t + j] = da;
      rsum += da * Pz[(int64_t)i * t + j];
    }
    for (int j = 0; j < t; ++j)
      DS[(int64_t)i * t + j] = j <= i ? Pz[(int64_t)i * t + j] * (DS[(int64_t)i * t + j] - rsum) / rs
                                      : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < t; i += blockDim.x)       // dq_i = sum_j dS_ij k_j
    for (int e = 0; e < hd; ++e) {
      double acc = 0.0;
      for (int j = 0; j <= i; ++j) acc += DS[(int64_t)i * t + j] * k[(int64_t)j * ld + e];
      dq[(int64_t)i * ld + e] = acc;
    }
  for (int j = threadIdx.x; j < t; j += blockDim.x)       // dk_j, dv_j over i >= j
    for (int e = 0; e < hd; ++e) {
      double ak = 0.0, av = 0.0;
      for (int i = j; i < t; ++i) {
        ak += DS[(int64_t)i * t + j] * q[(int64_t)i * ld + e];
        av += Pz[(int64_t)i * t + j] * dc[(int64_t)i * d + e];
      }
      dk[(int64_t)j * ld + e] = ak;
      dv[(int64_t)j * ld + e] = av;
    }
}

inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

// dx = d(block)/dx^T dy for one toy-family block; x, dy, dx f32 [batch*tokens][d]
int block_backward_f64(const float* wqkv_t, const float* wo_t, const float* w1_t,
                       const float* w2_t, const float* ln1_g, const float* ln1_b,
                       const float* ln2_g, const float* ln2_b, int d, int H, int F,
                       const float* x, const float* dy, float* dx, int batch, int tokens,
                       cudaStream_t st) {
  const int64_t R = (int64_t)batch * tokens;
  const int64_t n_w = 3LL * d * d + (int64_t)d * d + 2LL * F * d;
  const int64_t n_act = R * (12LL * d + 3LL * F + 4) + 2LL * batch * H * tokens * tokens;
  double* buf = nullptr;
  if (cudaMallocAsync(&buf, (n_w + n_act) * sizeof(double), st) != cudaSuccess) return -1;
  double* Wqkv = buf;                  // [3d][d] = (Wq | Wk | Wv)^T
  double* Wo = Wqkv + 3LL * d * d;     // [d][d] = Wo^T
  double* W1 = Wo + (int64_t)d * d;    // [F][d] = W1^T
  double* W2 = W1 + (int64_t)F * d;    // [d][F] = W2^T
  double* p = W2 + (int64_t)d * F;
  auto take = [&](int64_t n) { double* q = p; p += n; return q; };
  double *xd = take(R * d), *h = take(R * d), *qkv = take(R * 3 * d), *ctx = take(R * d);
  double *x1 = take(R * d), *h2 = take(R * d), *a = take(R * F), *dyd = take(R * d);
  double *dg = take(R * F), *dh2 = take(R * d), *dx1 = take(R * d), *dctx = take(R * d);
  double *dqkv = take(R * 3 * d), *dh = take(R * d), *outd = take(R * d);
  double *mu1 = take(R), *inv1 = take(R), *mu2 = take(R), *inv2 = take(R);
  double* P = take(2LL * batch * H * tokens * tokens);   // probabilities | dscores
  (void)a;
  f2d_kernel<<<nb(3LL * d * d), 256, 0, st>>>(wqkv_t, Wqkv, 3LL * d * d);
  f2d_kernel<<<nb((int64_t)d * d), 256, 0, st>>>(wo_t, Wo, (int64_t)d * d);
  f2d_kernel<<<nb((int64_t)F * d), 256, 0, st>>>(w1_t, W1, (int64_t)F * d);
  f2d_kernel<<<nb((int64_t)F * d), 256, 0, st>>>(w2_t, W2, (int64_t)F * d);
  f2d_kernel<<<nb(R * d), 256, 0, st>>>(x, xd, R * d);
  f2d_kernel<<<nb(R * d), 256, 0, st>>>(dy, dyd, R * d);
  // ---- forward (float64), keeping intermediates ----
  ln_fwd_kernel<<<nb(R), 256, 0, st>>>(xd, ln1_g, ln1_b, h, mu1, inv1, R, d);
  // qkv = h @ (Wq|Wk|Wv): stored transposed [3d][d] -> B[k][n] at n*d + k
  dgemm_kernel<<<nb(R * 3 * d), 256, 0, st>>>(h, d, 1, Wqkv, 1, d, qkv, R, 3 * d, d, false);
  attn_fb_kernel<<<batch * H, 64, 0, st>>>(qkv, nullptr, ctx, nullptr, P, tokens, d, H, false);
  // x1 = x + ctx @ Wo
  cudaMemcpyAsync(x1, xd, R * d * sizeof(double), cudaMemcpyDeviceToDevice, st);
  dgemm_kernel<<<nb(R * d), 256, 0, st>>>(ctx, d, 1, Wo, 1, d, x1, R, d, d, true);
  ln_fwd_kernel<<<nb(R), 256, 0, st>>>(x1, ln2_g, ln2_b, h2, mu2, inv2, R, d);
  dgemm_kernel<<<nb(R * F), 256, 0, st>>>(h2, d, 1, W1, 1, d, a, R, F, d, false);
  // ---- backward ----
  // dg = dy @ W2^T: W2 [F][d] (reference) stored transposed [d][F] -> B[k=d][n=F] at k*F + n
  dgemm_kernel<<<nb(R * F), 256, 0, st>>>(dyd, d, 1, W2, F, 1, dg, R, F, d, false);
  gelu_grad_kernel<<<nb(R * F), 256, 0, st>>>(a, dg, dg, R * F);
  // dh2 = da @ W1^T: W1 [d][F] stored [F][d] -> B[k=F][n=d] at k*d + n
  dgemm_kernel<<<nb(R * d), 256, 0, st>>>(dg, F, 1, W1, d, 1, dh2, R, d, F, false);
  ln_bwd_kernel<<<nb(R), 256, 0, st>>>(x1, ln2_g, mu2, inv2, dh2, dyd, dx1, R, d);
  // dctx = dx1 @ Wo^T: stored [d][d] = Wo^T -> B[k][n] at k*d + n
  dgemm_kernel<<<nb(R * d), 256, 0, st>>>(dx1, d, 1, Wo, d, 1, dctx, R, d, d, false);
  attn_fb_kernel<<<batch * H, 64, 0, st>>>(qkv, dctx, nullptr, dqkv, P, tokens, d, H, true);
  // dh = dq @ Wq^T + dk @ Wk^T + dv @ Wv^T = dqkv [R][3d] @ (stored [3d][d])
  dgemm_kernel<<<nb(R * d), 256, 0, st>>>(dqkv, 3 * d, 1, Wqkv, d, 1, dh, R, d, 3 * d, false);
  ln_bwd_kernel<<<nb(R), 256, 0, st>>>(xd, ln1_g, mu1, inv1, dh, dx1, outd, R, d);
  add_d2f_kernel<<<nb(R * d), 256, 0, st>>>(outd, dx, R * d);
  cudaFreeAsync(buf, st);
  for (int i = 0; i < 16; ++i) count_launch();
  return 0;
}

}  // namespace sp
