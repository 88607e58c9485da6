"""Where the N = 1 e2e step loses time against the device-timed step (run on a
GPU box): CUDA events around each run_cached of a 70B 80-block decode with
host rows, (A) reading every result back before the next step (the e2e loop)
and (B) back to back; host time split into Python and the C call."""
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


class TimedLib:
    def __init__(self, lib):
        self._lib, self.t = lib, 0.0

    def __getattr__(self, name):
        f = getattr(self._lib, name)
        if name != "sp_span_forward":
            return f

        def g(*a):
            t0 = time.perf_counter()
            r = f(*a)
            self.t += time.perf_counter() - t0
            return r
        return g


eng.lib = TimedLib(eng.lib)
st = torch.cuda.current_stream()
rows = torch.from_numpy(np.random.default_rng(1).standard_normal((60, 1, d)).astype(np.float32)
                        ).pin_memory().numpy()
xdev = torch.from_numpy(rows[:, 0]).cuda()
xstage = torch.empty_like(xdev)
for mode in ("A: result read every step", "B: back to back",
             "C: back to back, device-resident input", "D: as C plus a D2D copy per step"):
    c = eng.make_caches(0, 80, 1)
    eng.run_cached(0, 80, c, HiddenBlob.from_array(np.random.default_rng(0).standard_normal(
        (2048, d)).astype(np.float32)), 1, 2048, False)
    torch.cuda.synchronize()
    evs, outs = [], []
    t_rc = 0.0
    eng.lib.t = 0.0
    for i in range(60):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode.startswith("A") or mode.startswith("B"):
            b = HiddenBlob.from_array(rows[i])
        elif mode.startswith("C"):
            b = HiddenBlob.from_device(xdev[i:i + 1])
        else:
            xstage[i:i + 1].copy_(xdev[i:i + 1])
            b = HiddenBlob.from_device(xstage[i:i + 1])
        e0.record(st)
        t1 = time.perf_counter()
        out = eng.run_cached(0, 80, c, b, 1, 1, False)
        if i >= 10:
            t_rc += time.perf_counter() - t1
        e1.record(st)
        if mode.startswith("A"):
            out.array()
        else:
            outs.append(out)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    gaps = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(10, 59)]
    steps = [evs[i][0].elapsed_time(evs[i][1]) for i in range(10, 59)]
    span = evs[10][0].elapsed_time(evs[59][1]) / 50
    print(f"{mode}: step (event before -> after run_cached) median {np.median(steps):.4f} ms, "
          f"gap median {np.median(gaps):.4f} ms, wall per step {span:.4f} ms; host run_cached "
          f"{t_rc / 50 * 1e3:.3f} ms of which the C call (400 launches) "
          f"{eng.lib.t / 60 * 1e3:.3f} ms")
    del c, outs

# E / F: no events inside the loop (events only around 50 steps)
for mode in ("E: run_cached with host rows, back to back, no per-step events",
             "F: sp_span_forward in place (the bench's device-timed loop)",
             "G: E with one event record per step", "H: E with a host sync per step"):
    c = eng.make_caches(0, 80, 1)
    eng.run_cached(0, 80, c, HiddenBlob.from_array(np.random.default_rng(0).standard_normal(
        (2048, d)).astype(np.float32)), 1, 2048, False)
    y = torch.from_numpy(rows[0]).cuda()
    for i in range(5):
        eng.run_cached(0, 80, c, HiddenBlob.from_array(rows[i]), 1, 1, False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    outs = []
    e0.record(st)
    for i in range(5, 55):
        if mode.startswith("F"):
            eng.lib._lib.sp_span_forward(eng.span.handle, c.handle, 0, 80, y.data_ptr(), 0, 0,
                                         y.data_ptr(), 0, 0, 1, 1, st.cuda_stream)
        else:
            outs.append(eng.run_cached(0, 80, c, HiddenBlob.from_array(rows[i]), 1, 1, False))
            if mode.startswith("G"):
                torch.cuda.Event().record(st)
            elif mode.startswith("H"):
                torch.cuda.synchronize()
    e1.record(st)
    torch.cuda.synchronize()
    print(f"{mode}: {e0.elapsed_time(e1) / 50:.4f} ms per step")
    del c, outs
