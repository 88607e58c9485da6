import time, numpy as np, torch
import sys; sys.path.insert(0, '.')
from paper_2312_08361_b200.config import llama2_70b
from paper_2312_08361_b200.engine import B200ServerEngine
from paper_2312_08361_b200.blob import HiddenBlob
cfg = llama2_70b(weight_dtype="int8", n_blocks=80)
eng = B200ServerEngine(cfg)
d = cfg.hidden_dim
c = eng.make_caches(0, 80, 1)
eng.run_cached(0, 80, c, HiddenBlob.from_array(np.random.default_rng(0).standard_normal((2048, d)).astype(np.float32)), 1, 2048, False)
rows = torch.from_numpy(np.random.default_rng(1).standard_normal((60, 1, d)).astype(np.float32)).pin_memory().numpy()
st = torch.cuda.current_stream()
evs = []
tc = {"from_array": 0, "run_cached": 0, "array": 0}
for i in range(60):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    b = HiddenBlob.from_array(rows[i])
    t1 = time.perf_counter()
    e0.record(st)
    out = eng.run_cached(0, 80, c, b, 1, 1, False)
    e1.record(st)
    t2 = time.perf_counter()
    out.array()
    t3 = time.perf_counter()
    if i >= 10:
        tc["from_array"] += t1 - t0; tc["run_cached"] += t2 - t1; tc["array"] += t3 - t2
    evs.append((e0, e1))
torch.cuda.synchronize()
gaps = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(10, 59)]
steps = [evs[i][0].elapsed_time(evs[i][1]) for i in range(10, 59)]
print("gpu gap ms (end of step i -> start of step i+1): median %.4f" % np.median(gaps))
print("step ms (incl. H2D) median %.4f" % np.median(steps))
print({k: round(v / 50 * 1e3, 4) for k, v in tc.items()}, "ms per step (host)")
