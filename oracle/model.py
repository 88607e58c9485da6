"""Span-forward CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates `SP/model.py` (`SP/` = /root/reference/pkg/src/swarmpipe/):

* splitmix64 weight streams — `_splitmix64` :40-46, `_stream_seed` :49-52,
  `_uniform_weights` :55-60, `init_model` :178-199
* the cached pre-norm block — `_ln` :222-225, `_gelu` :228-229,
  `block_forward_batched` :244-280 (same op order and float32 dtype rules,
  so the toy family is ``array_equal`` to the reference)
* KV semantics — `KVCache.append` :163-167 (concat on the time axis),
  `KVCache.gather` :169-175 (new slot i <- old slot idx[i])
* the local generation oracle — `_LocalRunner` :418-437,
  `reference_generate` :440-467, `logits_for`/`greedy_pick` :393-400

Extensions without reference code (parity unpinned), written
in the same structure and dtype rules:

* family "llama": RMSNorm (eps 1e-5), rotate-half RoPE from an f64-built f32
  cos/sin table, GQA, SwiGLU (gate = w1, up = w3 [role 13], down = w2)
* family "bloom": the toy block with ALiBi biases slope_h * (j - i_abs)
* weight_dtype "bf16": round-to-nearest-even of the f32 stream values
* weight_dtype "nf4": see quantize_columns_nf4 (builder's format, parity unpinned)
* weight_dtype "int8": per output channel ``scale = f32(absmax/127)``,
  ``code = rint(w/scale)`` — the reference codec arithmetic (`SP/quantize.py:44-47`)
  applied column-wise; the effective weight is ``f32(code) * scale``
* kv_dtype "bf16": K/V rows are rounded to bf16 when they enter the cache
"""

from __future__ import annotations

import numpy as np

LN_EPS = 1e-5                      # SP/model.py:23
GELU_C = 0.7978845608028654        # SP/model.py:24

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)

# SP/model.py:32-37, plus role 13 for the SwiGLU up-projection (extension)
ROLES = {
    "wq": 1, "wk": 2, "wv": 3, "wo": 4,
    "w1": 5, "w2": 6,
    "ln1_g": 7, "ln1_b": 8, "ln2_g": 9, "ln2_b": 10,
    "embedding": 11, "soft_prompt": 12,
    "w3": 13,
}


# ---------------------------------------------------------------------------
# deterministic weights
# ---------------------------------------------------------------------------

def splitmix64_at(seed: int, idx: np.ndarray) -> np.ndarray:
    """splitmix64 outputs number idx+1 of the stream started at ``seed``
    (counter form of SP/model.py:40-46: z = (i+1)*GOLDEN + seed, then mix)."""
    with np.errstate(over="ignore"):
        z = (idx.astype(np.uint64) + np.uint64(1)) * _GOLDEN + np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, n: int) -> np.ndarray:
    return splitmix64_at(seed, np.arange(n, dtype=np.uint64))


def stream_seed(seed: int, block: int, role: str) -> int:
    """SP/model.py:49-52 (Python ints wrap only inside splitmix64)."""
    key = ((seed & 0xFFFFFFFFFFFFFFFF) ^ ((block + 1) * 0x9E3779B97F4A7C15)
           ^ (ROLES[role] * 0xC2B2AE3D27D4EB4F))
    # numpy's uint64 arithmetic of the reference reduces key mod 2^64
    return int(splitmix64(key & 0xFFFFFFFFFFFFFFFF, 1)[0])


def uniform_at(seed: int, block: int, role: str, flat_idx: np.ndarray, scale: float) -> np.ndarray:
    """Elements ``flat_idx`` of SP/model.py:55-60's uniform [-scale, scale] f32 tensor."""
    bits = splitmix64_at(stream_seed(seed, block, role), flat_idx)
    u = (bits >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    return ((2.0 * u - 1.0) * scale).astype(np.float32)


def uniform_weights(seed: int, block: int, role: str, shape: tuple, scale: float) -> np.ndarray:
    n = int(np.prod(shape))
    return uniform_at(seed, block, role, np.arange(n, dtype=np.uint64), scale).reshape(shape)


def weight_scale(cfg) -> float:
    """Every matrix uses 1/sqrt(d) (SP/model.py:181)."""
    return float(1.0 / np.sqrt(cfg.hidden_dim))


def to_bf16(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16, returned as f32 (NaN-free inputs)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    return r.astype(np.uint32).view(np.float32).reshape(np.shape(a))


def quantize_columns_int8(w: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """w [d_in, d_out] f32 -> codes int8 [d_out, d_in] (row per output channel),
    scales f32 [d_out]; the codec arithmetic of SP/quantize.py:43-47 per column."""
    wt = np.ascontiguousarray(w.T)
    absmax = np.abs(wt).max(axis=1)
    scales = (absmax / np.float32(127.0)).astype(np.float32)
    safe = np.where(scales > 0, scales, np.float32(1.0)).astype(np.float32)
    codes = np.rint(wt / safe[:, None]).astype(np.int8)
    codes[scales == 0] = 0
    return codes, scales


# NF4 (QLoRA, Dettmers et al. 2023: the 16 normal-float levels) on a 1/63 grid:
# CB7 = rint(63 * NF4_LEVELS).  The reference has no NF4 code (SURVEY.md 8c:
# parity unpinned); this is the builder's format, chosen so that a block of
# weights is an exact small integer times one f32 per output channel:
#   m_r  = max |w| over output channel r,  s_r = f32(m_r / 16065)  (16065 = 63 * 255)
#   a_j  = max |w| over the 64-wide block j of the channel
#   q_j  = rint(f32(f32(255 * a_j) / m_r))  in [0, 255]   (double-quantised block scale)
#   code = argmin_c |f32(w / s_r) - CB7[c] * q_j|, lowest c on ties; q_j = 0 -> level 0
#   w_eff = f32(f32(CB7[code] * q_j) * s_r)
NF4_LEVELS = np.array([-1.0, -0.6961928009986877, -0.5250730514526367, -0.39491748809814453,
                       -0.28444138169288635, -0.18477343022823334, -0.09105003625154495, 0.0,
                       0.07958029955625534, 0.16093020141124725, 0.24611230194568634,
                       0.33791524171829224, 0.44070982933044434, 0.5626170039176941,
                       0.7229568362236023, 1.0])
CB7 = np.rint(63.0 * NF4_LEVELS).astype(np.int32)     # [-63, -44, ..., 46, 63]
NF4_ZERO = 7


def quantize_columns_nf4(w: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """w [d_in, d_out] f32 -> codes uint8 [d_out, d_in] (0..15), block scales
    uint8 [d_out, d_in/64], channel scales f32 [d_out] (format above)."""
    wt = np.ascontiguousarray(w.T).astype(np.float32)
    n, k = wt.shape
    m = np.abs(wt).max(axis=1)
    s = (m / np.float32(16065.0)).astype(np.float32)
    a = np.abs(wt.reshape(n, k // 64, 64)).max(axis=2)
    safe_m = np.where(m > 0, m, np.float32(1.0)).astype(np.float32)
    q = np.rint((np.float32(255.0) * a) / safe_m[:, None]).astype(np.int32)
    q[m == 0] = 0
    safe_s = np.where(s > 0, s, np.float32(1.0)).astype(np.float32)
    codes = np.empty((n, k), np.uint8)
    for r0 in range(0, n, 256):                         # bounded memory: 256 channels at a time
        t = (wt[r0:r0 + 256] / safe_s[r0:r0 + 256, None]).reshape(-1, k // 64, 64)
        lv = (CB7[None, None, :] * q[r0:r0 + 256, :, None]).astype(np.float32)  # [n, nb, 16]
        diff = np.abs(t[..., None] - lv[:, :, None, :])                          # f32
        c = diff.argmin(axis=-1).astype(np.uint8)
        c[q[r0:r0 + 256] == 0] = NF4_ZERO
        codes[r0:r0 + 256] = c.reshape(-1, k)
    return codes, q.astype(np.uint8), s


def effective_weight(cfg, w: np.ndarray) -> np.ndarray:
    """The f32 values the GPU multiplies by, for ``cfg.weight_dtype``."""
    if cfg.weight_dtype == "f32":
        return w
    if cfg.weight_dtype == "bf16":
        return to_bf16(w)
    if cfg.weight_dtype == "nf4":
        codes, q, s = quantize_columns_nf4(w)
        ints = (CB7[codes] * np.repeat(q.astype(np.int32), 64, axis=1)).astype(np.float32)
        return np.ascontiguousarray((ints * s[:, None]).T)
    codes, scales = quantize_columns_int8(w)
    return np.ascontiguousarray((codes.astype(np.float32) * scales[:, None]).T)


def block_matrices(cfg) -> list[tuple[str, int, int]]:
    d, kv = cfg.hidden_dim, cfg.kv_heads * cfg.head_dim
    f = cfg.ffn_dim or 4 * d
    mats = [("wq", d, d), ("wk", d, kv), ("wv", d, kv), ("wo", d, d), ("w1", d, f)]
    if cfg.family == "llama":
        mats.append(("w3", d, f))
    mats.append(("w2", f, d))
    return mats


def init_block(cfg, b: int) -> dict:
    """One block's parameters as effective f32 arrays (SP/model.py:183-195)."""
    s, scale, d = cfg.seed, weight_scale(cfg), cfg.hidden_dim
    p = {role: effective_weight(cfg, uniform_weights(s, b, role, (a, c), scale))
         for role, a, c in block_matrices(cfg)}
    p["ln1_g"] = np.ones(d, np.float32)
    p["ln1_b"] = np.zeros(d, np.float32)
    p["ln2_g"] = np.ones(d, np.float32)
    p["ln2_b"] = np.zeros(d, np.float32)
    return p


def init_embedding(cfg) -> np.ndarray:
    """Client embedding, keyed by block index n_blocks (SP/model.py:196-198)."""
    return uniform_weights(cfg.seed, cfg.n_blocks, "embedding",
                           (cfg.vocab_size, cfg.hidden_dim), weight_scale(cfg))


# ---------------------------------------------------------------------------
# block forward
# ---------------------------------------------------------------------------

def ln(x, g, b):
    """SP/model.py:222-225."""
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS) * g + b


def rmsnorm(x, g):
    ms = (x * x).mean(axis=-1, keepdims=True)
    return x / np.sqrt(ms + LN_EPS) * g


def gelu(x):
    """SP/model.py:228-229."""
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + 0.044715 * x * x * x)))


def silu(x):
    return x / (np.float32(1.0) + np.exp(-x))


def rope_table(max_pos: int, hd: int, theta: float = 10000.0) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin [max_pos, hd/2] built in f64 and rounded once to f32."""
    inv = theta ** (-(np.arange(0, hd, 2, dtype=np.float64) / hd))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def apply_rope(x: np.ndarray, pos: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """x [B, n, h, hd]; rotate-half pairs (j, j + hd/2) at absolute positions pos [n]."""
    half = x.shape[-1] // 2
    c = cos[pos][None, :, None, :]
    s = sin[pos][None, :, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1).astype(np.float32)


def alibi_slopes(n_heads: int) -> np.ndarray:
    """BLOOM's ALiBi slopes (closest power of two + interleaved extras)."""
    def pow2(n):
        start = 2.0 ** (-(2.0 ** -(np.log2(n) - 3)))
        return [start * start ** i for i in range(n)]
    p = 2 ** int(np.floor(np.log2(n_heads)))
    s = pow2(p)
    if p < n_heads:
        s += pow2(2 * p)[0::2][: n_heads - p]
    return np.asarray(s, np.float64).astype(np.float32)


def _split_heads(x, n_heads):
    b, t, d = x.shape
    return x.reshape(b, t, n_heads, d // n_heads).transpose(0, 2, 1, 3)


def _merge_heads(x):
    b, h, t, hd = x.shape
    return x.transpose(0, 2, 1, 3).reshape(b, t, h * hd)


class Tables:
    """Per-config constant tables (RoPE cos/sin, ALiBi slopes)."""

    def __init__(self, cfg):
        self.cos = self.sin = self.slopes = None
        if cfg.family == "llama":
            self.cos, self.sin = rope_table(cfg.max_seq_len, cfg.head_dim, cfg.rope_theta)
        if cfg.family == "bloom":
            self.slopes = alibi_slopes(cfg.n_heads)


def block_forward_batched(cfg, p: dict, x: np.ndarray, past_k: np.ndarray, past_v: np.ndarray,
                          tables: Tables | None = None):
    """x [B, n, d]; past_k/v [B, t0, n_kv, hd] -> (y [B, n, d], k_new, v_new).

    Toy family: the op sequence of SP/model.py:244-280 verbatim."""
    bsz, n, d = x.shape
    H, hd = cfg.n_heads, cfg.head_dim
    kvh = past_k.shape[2]
    t0 = past_k.shape[1]
    fam = cfg.family

    if fam == "llama":
        h = rmsnorm(x, p["ln1_g"])
    else:
        h = ln(x, p["ln1_g"], p["ln1_b"])
    q = (h @ p["wq"]).reshape(bsz, n, H, hd)
    k_new = (h @ p["wk"]).reshape(bsz, n, kvh, hd)
    v_new = (h @ p["wv"]).reshape(bsz, n, kvh, hd)
    if fam == "llama":
        tables = tables or Tables(cfg)
        pos = np.arange(t0, t0 + n)
        q = apply_rope(q, pos, tables.cos, tables.sin)
        k_new = apply_rope(k_new, pos, tables.cos, tables.sin)
    if getattr(cfg, "kv_dtype", "f32") == "bf16":
        k_new, v_new = to_bf16(k_new), to_bf16(v_new)
    q = q.transpose(0, 2, 1, 3)                                           # [B, H, n, hd]

    k_all = np.concatenate([past_k, k_new], axis=1).transpose(0, 2, 1, 3)  # [B, kvh, t, hd]
    v_all = np.concatenate([past_v, v_new], axis=1).transpose(0, 2, 1, 3)
    if kvh != H:
        rep = H // kvh
        k_all = np.repeat(k_all, rep, axis=1)
        v_all = np.repeat(v_all, rep, axis=1)

    scores = q @ k_all.transpose(0, 1, 3, 2) / np.float32(np.sqrt(hd))      # [B, H, n, t0+n]
    if fam == "bloom":
        tables = tables or Tables(cfg)
        rel = (np.arange(t0 + n)[None, :] - (t0 + np.arange(n))[:, None]).astype(np.float32)
        scores = scores + tables.slopes[None, :, None, None] * rel[None, None]
    if n > 1:
        jj = np.arange(t0 + n)
        ii = np.arange(n)
        mask = jj[None, :] > (t0 + ii[:, None])
        scores = np.where(mask, np.float32(-1e30), scores)
    scores = scores - scores.max(axis=-1, keepdims=True)
    w = np.exp(scores)
    attn = w / w.sum(axis=-1, keepdims=True)
    ctx = _merge_heads(attn @ v_all)                                       # [B, n, d]
    x1 = x + ctx @ p["wo"]

    if fam == "llama":
        h2 = rmsnorm(x1, p["ln2_g"])
        y = x1 + (silu(h2 @ p["w1"]) * (h2 @ p["w3"])) @ p["w2"]
    else:
        h2 = ln(x1, p["ln2_g"], p["ln2_b"])
        y = x1 + gelu(h2 @ p["w1"]) @ p["w2"]
    return y.astype(np.float32, copy=False), k_new, v_new


# ---------------------------------------------------------------------------
# KV cache + local runner
# ---------------------------------------------------------------------------

class KVCache:
    """SP/model.py:139-175: keys/values [width, t, n_kv, hd]."""

    def __init__(self, cfg, width: int = 1):
        shape = (width, 0, cfg.kv_heads if hasattr(cfg, "kv_heads") else cfg.n_heads, cfg.head_dim)
        self.keys = np.zeros(shape, np.float32)
        self.values = np.zeros(shape, np.float32)

    @property
    def length(self) -> int:
        return self.keys.shape[1]

    @property
    def width(self) -> int:
        return self.keys.shape[0]

    def append(self, k_new, v_new) -> None:
        self.keys = np.concatenate([self.keys, k_new], axis=1)
        self.values = np.concatenate([self.values, v_new], axis=1)

    def gather(self, idx0) -> None:
        idx = np.asarray(idx0, dtype=np.intp)
        if idx.size and (idx.min() < 0 or idx.max() >= self.width):
            raise ValueError("reorder index out of range")
        self.keys = self.keys[idx].copy()
        self.values = self.values[idx].copy()


class SpanRunner:
    """Cached stepping through blocks [start, end) (SP/model.py:418-437 and
    the span loop of SP/server.py:93-100)."""

    def __init__(self, cfg, start: int = 0, end: int | None = None, blocks: dict | None = None,
                 width: int = 1):
        self.cfg = cfg
        self.start = start
        self.end = cfg.n_blocks if end is None else end
        self.blocks = blocks if blocks is not None else {
            b: init_block(cfg, b) for b in range(self.start, self.end)}
        self.tables = Tables(cfg)
        self.caches = [KVCache(cfg, width) for _ in range(self.start, self.end)]

    @property
    def length(self) -> int:
        return self.caches[0].length

    def step(self, x: np.ndarray) -> np.ndarray:
        for b, c in zip(range(self.start, self.end), self.caches):
            x, kn, vn = block_forward_batched(self.cfg, self.blocks[b], x, c.keys, c.values,
                                              self.tables)
            c.append(kn, vn)
        return x

    def reorder(self, parents0) -> None:
        for c in self.caches:
            c.gather(parents0)


# ---------------------------------------------------------------------------
# prompt-tuning backward (training mode: full causal sequence, no KV history)
# ---------------------------------------------------------------------------

def _ln_grad(x, g, dy):
    """d LayerNorm / dx applied to dy (SP/model.py:303-311), float64."""
    n = x.shape[-1]
    xc = x - x.mean(axis=-1, keepdims=True)
    inv = 1.0 / np.sqrt((xc * xc).mean(axis=-1, keepdims=True) + LN_EPS)
    xhat = xc * inv
    gy = dy * g
    return inv * (gy - gy.sum(axis=-1, keepdims=True) / n
                  - xhat * (gy * xhat).sum(axis=-1, keepdims=True) / n)


def _gelu_deriv(x):
    """d tanh-GELU / dx (SP/model.py:314-317), float64."""
    th = np.tanh(GELU_C * (x + 0.044715 * x ** 3))
    return 0.5 * (1.0 + th) + 0.5 * x * (1.0 - th * th) * GELU_C * (1.0 + 0.134145 * x * x)


def block_backward(cfg, p: dict, x32: np.ndarray, dy32: np.ndarray) -> np.ndarray:
    """Gradient of one block's output wrt its input for [B, t, d] sequences
    (block_backward, SP/model.py:320-381): the forward is recomputed in float64
    from the recorded input (causal attention within each sequence), then
    back-propagated; parameters are only read.  Reference family only."""
    f8 = lambda a: np.asarray(a, np.float64)  # noqa: E731
    x, dy = f8(x32), f8(dy32)
    B, t, d = x.shape
    H = cfg.n_heads
    hd = d // H
    wq, wk, wv, wo, w1, w2 = (f8(p[k]) for k in ("wq", "wk", "wv", "wo", "w1", "w2"))
    g1, b1, g2, b2 = (f8(p[k]) for k in ("ln1_g", "ln1_b", "ln2_g", "ln2_b"))
    # forward, keeping what the backward needs
    h = ln(x, g1, b1)
    q, k, v = (_split_heads(h @ w, H) for w in (wq, wk, wv))
    causal = np.triu(np.ones((t, t), bool), 1)
    s = np.where(causal, -1e30, np.einsum("bhid,bhjd->bhij", q, k) / np.sqrt(hd))
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    att = e / e.sum(axis=-1, keepdims=True)
    x1 = x + _merge_heads(att @ v) @ wo
    a = ln(x1, g2, b2) @ w1
    # backward
    dx1 = dy + _ln_grad(x1, g2, ((dy @ w2.T) * _gelu_deriv(a)) @ w1.T)
    dctx = _split_heads(dx1 @ wo.T, H)
    datt = np.einsum("bhid,bhjd->bhij", dctx, v)
    ds = att * (datt - (datt * att).sum(axis=-1, keepdims=True))
    ds = np.where(causal, 0.0, ds) / np.sqrt(hd)
    dq = ds @ k
    dk = np.einsum("bhij,bhid->bhjd", ds, q)
    dv = np.einsum("bhij,bhid->bhjd", att, dctx)
    dh = _merge_heads(dq) @ wq.T + _merge_heads(dk) @ wk.T + _merge_heads(dv) @ wv.T
    return (dx1 + _ln_grad(x, g1, dh)).astype(np.float32)


def logits_for(embedding: np.ndarray, row: np.ndarray) -> np.ndarray:
    """Tied unembedding, SP/model.py:393-395 (no final norm)."""
    return row @ embedding.T


def greedy_pick(logits: np.ndarray) -> int:
    """argmax, ties to the lowest id (SP/model.py:398-400)."""
    return int(np.argmax(logits))


def reference_generate(cfg, prefix: list[int], n_new: int) -> list[int]:
    """Greedy generation oracle, SP/model.py:440-467."""
    emb = init_embedding(cfg)
    runner = SpanRunner(cfg)
    out = list(prefix)
    x = emb[np.asarray(prefix, dtype=np.intp)][None]
    for _ in range(n_new):
        y = runner.step(x)
        tok = greedy_pick(logits_for(emb, y[0, -1]))
        out.append(tok)
        x = emb[np.asarray([tok], dtype=np.intp)][None]
    return out
