"""N = 1 e2e loop variants (GPU box): how the per-step result read-back is done."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2312_08361_b200.blob import HiddenBlob  # noqa: E402
from paper_2312_08361_b200.config import llama2_70b  # noqa: E402
from paper_2312_08361_b200.engine import B200ServerEngine  # noqa: E402

cfg = llama2_70b(weight_dtype="int8", n_blocks=80)
eng = B200ServerEngine(cfg)
d = cfg.hidden_dim
rows = torch.from_numpy(np.random.default_rng(1).standard_normal((200, 1, d)).astype(np.float32)
                        ).pin_memory().numpy()
pin = torch.empty((1, d), dtype=torch.float32).pin_memory()
for rep in range(2):
    for mode in ("array", "array_async+pinned", "sync only", "no read (back to back)"):
        c = eng.make_caches(0, 80, 1)
        eng.run_cached(0, 80, c, HiddenBlob.from_array(np.random.default_rng(0).standard_normal(
            (2048, d)).astype(np.float32)), 1, 2048, False)
        for i in range(3):
            eng.run_cached(0, 80, c, HiddenBlob.from_array(rows[i]), 1, 1, False).array()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(3, 53):
            out = eng.run_cached(0, 80, c, HiddenBlob.from_array(rows[i]), 1, 1, False)
            if mode == "array":
                out.array()
            elif mode.startswith("array_async"):
                out.array_async(out=pin).result()
            elif mode == "sync only":
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 50
        print(f"{mode}: {dt * 1e3:.4f} ms per step ({1 / dt:.2f} steps/s)")
        del c
