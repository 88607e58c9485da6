"""Small tcgen05 prefill-attention check (debugging): one llama_int8 span, prefill of
n tokens, compare option 8 on/off; prints max diff or the CUDA error."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_08361_b200 import _lib
from paper_2312_08361_b200.blob import HiddenBlob
from paper_2312_08361_b200.config import SpanConfig
from paper_2312_08361_b200.engine import B200ServerEngine
cfg = SpanConfig(n_blocks=1, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024, vocab_size=64,
                 max_seq_len=512, family="llama", weight_dtype="int8", kv_dtype="bf16", seed=5)
eng = B200ServerEngine(cfg)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
x = np.random.default_rng(1).standard_normal((n, 512)).astype(np.float32)
outs = []
for tc in (0, 1):
    _lib.check(eng.lib.sp_span_set_option(eng.span.handle, 8, tc))
    c = eng.make_caches(0, 1, 1)
    outs.append(eng.run_cached(0, 1, c, HiddenBlob.from_array(x), 1, n, False).array())
    print("tc", tc, "ok", flush=True)
print("n", n, "max diff", np.abs(outs[0] - outs[1]).max(), "max", np.abs(outs[0]).max())
