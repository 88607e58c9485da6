"""Debug: stateless forward of the SMALL llama int8 config at several token counts."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2312_08361_b200 import _lib  # noqa: E402
from paper_2312_08361_b200.blob import HiddenBlob  # noqa: E402
from paper_2312_08361_b200.config import SpanConfig  # noqa: E402
from paper_2312_08361_b200.engine import B200ServerEngine, DeviceSpan  # noqa: E402

cfg = SpanConfig(n_blocks=3, hidden_dim=512, n_heads=4, n_kv_heads=2, ffn_dim=1024,
                 vocab_size=64, max_seq_len=512, family="llama", weight_dtype="int8",
                 kv_dtype="bf16", seed=5)
span = DeviceSpan(cfg, 0, cfg.n_blocks)
eng = B200ServerEngine(cfg, span=span)
rng = np.random.default_rng(5)
for batch, tokens in ((1, 300), (2, 129), (1, 512), (3, 150), (1, 150), (1, 256), (1, 257)):
    x = rng.standard_normal((batch * tokens, cfg.hidden_dim)).astype(np.float32)
    out = {}
    for name, opt in (("pair", (2, 1)), ("single", (2, 0)), ("simt", (0, 0))):
        _lib.check(span.lib.sp_span_set_option(span.handle, 0, 0 if name == "simt" else 1))
        _lib.check(span.lib.sp_span_set_option(span.handle, 2, 0 if name == "single" else 1))
        out[name] = eng.forward(0, cfg.n_blocks, HiddenBlob.from_array(x), batch, tokens, 10**9,
                                None).array()
    fin = {k: bool(np.isfinite(v).all()) for k, v in out.items()}
    d = lambda a, b: float(np.abs(out[a] - out[b]).max())  # noqa: E731
    print(batch, tokens, fin, "pair-single", d("pair", "single"), "pair-simt", d("pair", "simt"),
          "max", float(np.abs(out["simt"]).max()))
