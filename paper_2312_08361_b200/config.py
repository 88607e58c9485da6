"""Model shapes for the span-forward hot path.

``SpanConfig`` is a superset of the reference's ``ModelConfig``
(`/root/reference/pkg/src/swarmpipe/model.py:63-86`): the six reference fields
keep their names, defaults and validation, so a ``SpanConfig`` can stand in
wherever the reference reads ``config.n_blocks / hidden_dim / n_heads /
vocab_size / max_seq_len / seed / head_dim`` (`SP/server.py:229, 399, 433,
446`).  The added fields describe the shapes the reference lacks (SURVEY.md
§8c "parity unpinned"):

* ``family``      "toy"   — the reference block verbatim: pre-norm LayerNorm,
                            MHA, 4d tanh-GELU MLP, no positions (`SP/model.py:244-280`)
                  "llama" — RMSNorm, RoPE (rotate-half, theta 1e4), GQA,
                            SwiGLU MLP (gate=w1, up=w3, down=w2)
                  "bloom" — the toy block plus ALiBi attention biases
* ``n_kv_heads``  GQA key/value heads (default = n_heads)
* ``ffn_dim``     MLP width (default 4*d)
* ``weight_dtype`` "f32" | "bf16" | "int8" (per-output-channel absmax/127) |
                  "nf4" (QLoRA NF4 levels on a 1/63 grid, 64-wide blocks with
                  double-quantised uint8 block scales; oracle/model.py)
* ``kv_dtype``    "f32" | "bf16"

Weights are always the reference's splitmix64 stream (`SP/model.py:40-60`)
keyed by (seed, block, role); "bf16"/"int8" are deterministic roundings of
those f32 values, so the CPU oracle and the GPU agree on every weight bit.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

FAMILIES = ("toy", "llama", "bloom")
WEIGHT_DTYPES = ("f32", "bf16", "int8", "nf4")
KV_DTYPES = ("f32", "bf16")


class ConfigurationError(ValueError):
    """Mirrors `SP/errors.py:12` (raised for invalid dimensions)."""


@dataclass(frozen=True)
class SpanConfig:
    n_blocks: int = 8
    hidden_dim: int = 64
    n_heads: int = 4
    vocab_size: int = 256
    max_seq_len: int = 2048
    seed: int = 0
    family: str = "toy"
    n_kv_heads: int = 0          # 0 -> n_heads
    ffn_dim: int = 0             # 0 -> 4 * hidden_dim
    weight_dtype: str = "f32"
    kv_dtype: str = "f32"
    rope_theta: float = 10000.0

    def __post_init__(self) -> None:
        # reference validation, SP/model.py:74-82
        if self.n_blocks < 1:
            raise ConfigurationError("n_blocks must be >= 1")
        if self.vocab_size < 2:
            raise ConfigurationError("vocab_size must be >= 2")
        if self.hidden_dim % self.n_heads != 0:
            raise ConfigurationError("hidden_dim must be divisible by n_heads")
        if self.max_seq_len < 1:
            raise ConfigurationError("max_seq_len must be >= 1")
        if self.family not in FAMILIES:
            raise ConfigurationError(f"family must be one of {FAMILIES}")
        if self.weight_dtype not in WEIGHT_DTYPES:
            raise ConfigurationError(f"weight_dtype must be one of {WEIGHT_DTYPES}")
        if self.kv_dtype not in KV_DTYPES:
            raise ConfigurationError(f"kv_dtype must be one of {KV_DTYPES}")
        if self.n_heads % self.kv_heads != 0:
            raise ConfigurationError("n_heads must be divisible by n_kv_heads")
        if self.family == "llama" and self.head_dim % 2:
            raise ConfigurationError("RoPE needs an even head_dim")

    @property
    def head_dim(self) -> int:
        return self.hidden_dim // self.n_heads

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    @property
    def ffn(self) -> int:
        return self.ffn_dim or 4 * self.hidden_dim

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim

    def block_matrices(self) -> list[tuple[str, int, int]]:
        """(role, d_in, d_out) of every weight matrix of one block, in the
        reference's x @ W orientation (`SP/model.py:183-191`)."""
        d, f, kv = self.hidden_dim, self.ffn, self.kv_dim
        mats = [("wq", d, d), ("wk", d, kv), ("wv", d, kv), ("wo", d, d), ("w1", d, f)]
        if self.family == "llama":
            mats.append(("w3", d, f))
        mats.append(("w2", f, d))
        return mats

    def block_params(self) -> int:
        return sum(a * b for _, a, b in self.block_matrices()) + 4 * self.hidden_dim

    def weight_bytes_per_block(self) -> int:
        """Algorithmic weight bytes one decode step streams per block
        (codes + per-output-channel f32 scales for int8; nf4: 4-bit codes, one
        uint8 scale per 64 weights and an f32 scale per output channel)."""
        elems = sum(a * b for _, a, b in self.block_matrices())
        chans = sum(b for _, _, b in self.block_matrices())
        if self.weight_dtype == "nf4":
            return elems // 2 + elems // 64 + 4 * chans
        elt = {"f32": 4, "bf16": 2, "int8": 1}[self.weight_dtype]
        n = elems * elt
        if self.weight_dtype == "int8":
            n += 4 * chans
        return n

    def with_(self, **kw) -> "SpanConfig":
        return replace(self, **kw)


# ---------------------------------------------------------------------------
# named shapes (BASELINE.json configs)
# ---------------------------------------------------------------------------

def toy(seed: int = 1, **kw) -> SpanConfig:
    """C1: the reference default ModelConfig (`SP/model.py:67-72`)."""
    return SpanConfig(seed=seed, **kw)


def llama2_7b(**kw) -> SpanConfig:
    """C2: Llama-2-7B shape, bf16 weights."""
    base = dict(n_blocks=32, hidden_dim=4096, n_heads=32, vocab_size=32000,
                max_seq_len=4096, family="llama", ffn_dim=11008,
                weight_dtype="bf16", kv_dtype="bf16")
    base.update(kw)
    return SpanConfig(**base)


def llama2_70b(**kw) -> SpanConfig:
    """C3/C5: Llama-2-70B shape (GQA 64/8), int8 weights."""
    base = dict(n_blocks=80, hidden_dim=8192, n_heads=64, n_kv_heads=8, vocab_size=32000,
                max_seq_len=4096, family="llama", ffn_dim=28672,
                weight_dtype="int8", kv_dtype="bf16")
    base.update(kw)
    return SpanConfig(**base)


def bloom_176b(**kw) -> SpanConfig:
    """C4: BLOOM-176B shape (ALiBi, 4d GELU MLP), int8 weights."""
    base = dict(n_blocks=70, hidden_dim=14336, n_heads=112, vocab_size=250880,
                max_seq_len=4096, family="bloom", weight_dtype="int8", kv_dtype="bf16")
    base.update(kw)
    return SpanConfig(**base)


def from_reference(cfg) -> SpanConfig:
    """Adopt a reference ``ModelConfig`` (toy family, f32 everywhere)."""
    if isinstance(cfg, SpanConfig):
        return cfg
    return SpanConfig(n_blocks=cfg.n_blocks, hidden_dim=cfg.hidden_dim, n_heads=cfg.n_heads,
                      vocab_size=cfg.vocab_size, max_seq_len=cfg.max_seq_len, seed=cfg.seed)
