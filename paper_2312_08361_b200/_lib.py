"""ctypes binding of libspanpipe.so (include/spanpipe.h).

The product path has no CPU fallback: if the shared library is missing or
was built without the CUDA kernels, importing the engine raises loudly.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SP_LIB_PATH") or os.path.join(HERE, "libspanpipe.so")

SP_OK = 0
SP_ERR_ARG = -1
SP_ERR_CUDA = -2
SP_ERR_CAPACITY = -3
SP_ERR_STATE = -4
SP_ERR_OOM = -5

FAMILY = {"toy": 0, "llama": 1, "bloom": 2}
WDTYPE = {"f32": 0, "bf16": 1, "int8": 2, "nf4": 3}
KVDTYPE = {"f32": 0, "bf16": 1}

# every symbol include/spanpipe.h declares
EXPORTS = (
    "sp_last_error", "sp_version", "sp_quantize_blockwise", "sp_dequantize_blockwise",
    "sp_weights_generate", "sp_stream_seed", "sp_span_create", "sp_span_destroy",
    "sp_span_weight_bytes", "sp_span_free_pages", "sp_span_read_weight", "sp_kv_create",
    "sp_kv_destroy", "sp_kv_length", "sp_kv_width", "sp_kv_reorder", "sp_kv_read",
    "sp_span_forward", "sp_span_forward_stateless", "sp_fnv1a64",
    "sp_content_hash", "sp_content_hash_verify",
    "sp_span_set_profiling", "sp_span_profile_read", "sp_kernel_launches",
    "sp_span_decode_gemv_only", "sp_head_create", "sp_head_destroy", "sp_head_embed",
    "sp_head_greedy", "sp_head_read_embedding", "sp_span_set_option", "sp_span_block_backward", "sp_head_logits", "sp_beam_select",
)


class SpConfig(ctypes.Structure):
    _fields_ = [
        ("n_blocks", ctypes.c_int32), ("hidden_dim", ctypes.c_int32),
        ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
        ("ffn_dim", ctypes.c_int32), ("vocab_size", ctypes.c_int32),
        ("max_seq_len", ctypes.c_int32), ("family", ctypes.c_int32),
        ("weight_dtype", ctypes.c_int32), ("kv_dtype", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("rope_theta", ctypes.c_double),
    ]


class SpanPipeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"spanpipe error {code}: {msg}")
        self.code = code


_lib = None

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built — run paper_2312_08361_b200/build.py "
                          "(there is no CPU fallback for the span hot path)")
    lib = ctypes.CDLL(LIB_PATH)
    sig = {
        "sp_last_error": (ctypes.c_char_p, []),
        "sp_version": (I32, []),
        "sp_quantize_blockwise": (I32, [P, P, P, I64, P]),
        "sp_dequantize_blockwise": (I32, [P, P, P, I64, P]),
        "sp_weights_generate": (I32, [ctypes.c_uint64, I32, I32, I64, ctypes.c_double, P, P]),
        "sp_stream_seed": (ctypes.c_uint64, [ctypes.c_uint64, I32, I32]),
        "sp_span_create": (I32, [ctypes.POINTER(SpConfig), I32, I32, I32, I64, ctypes.POINTER(P)]),
        "sp_span_destroy": (I32, [P]),
        "sp_span_weight_bytes": (I64, [P]),
        "sp_span_free_pages": (I64, [P]),
        "sp_span_read_weight": (I32, [P, I32, I32, P]),
        "sp_kv_create": (I32, [P, I32, ctypes.POINTER(P)]),
        "sp_kv_destroy": (I32, [P]),
        "sp_kv_length": (I32, [P]),
        "sp_kv_width": (I32, [P]),
        "sp_kv_reorder": (I32, [P, P, I32, P]),
        "sp_kv_read": (I32, [P, I32, I32, P, P]),
        "sp_span_forward": (I32, [P, P, I32, I32, P, P, P, P, P, P, I32, I32, P]),
        "sp_span_forward_stateless": (I32, [P, I32, I32, P, P, P, I32, I32, P]),
        "sp_span_block_backward": (I32, [P, I32, P, P, P, I32, I32, P]),
        "sp_fnv1a64": (ctypes.c_uint64, [P, I64]),
        "sp_content_hash": (I32, [P, I64, P, P]),
        "sp_content_hash_verify": (I32, [P, I64, P, P, P]),
        "sp_span_set_profiling": (I32, [P, I32]),
        "sp_span_profile_read": (I32, [P, I32, P, P, P, P]),
        "sp_kernel_launches": (I64, []),
        "sp_span_decode_gemv_only": (I32, [P, P, I32, I32, P, I32, P, P]),
        "sp_head_create": (I32, [ctypes.POINTER(SpConfig), I32, ctypes.POINTER(P)]),
        "sp_head_destroy": (I32, [P]),
        "sp_head_embed": (I32, [P, P, I32, P, P]),
        "sp_head_greedy": (I32, [P, P, P, P]),
        "sp_head_read_embedding": (I32, [P, P]),
        "sp_head_logits": (I32, [P, P, I32, P, P]),
        "sp_beam_select": (I32, [P, P, I32, I32, I32, P, P, P, P]),
        "sp_span_set_option": (I32, [P, I32, I32]),
    }
    for name in EXPORTS:
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = sig[name]
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != SP_OK:
        msg = load().sp_last_error().decode(errors="replace")
        raise SpanPipeError(rc, msg)


def make_config(cfg) -> SpConfig:
    return SpConfig(
        n_blocks=cfg.n_blocks, hidden_dim=cfg.hidden_dim, n_heads=cfg.n_heads,
        n_kv_heads=cfg.kv_heads, ffn_dim=cfg.ffn, vocab_size=cfg.vocab_size,
        max_seq_len=cfg.max_seq_len, family=FAMILY[cfg.family],
        weight_dtype=WDTYPE[cfg.weight_dtype], kv_dtype=KVDTYPE[cfg.kv_dtype],
        seed=cfg.seed & 0xFFFFFFFFFFFFFFFF, rope_theta=float(cfg.rope_theta))
