"""EXPERIMENT: per-SM stream speed from SP_GEMV_TRACE output -> weights file (one float per SM)."""
import sys

import numpy as np

src, dst = sys.argv[1], sys.argv[2]
speed = np.zeros(148)
cnt = np.zeros(148)
for blk in open(src).read().split("gemv N=")[1:]:
    rows = [l.split(":")[1].split() for l in blk.splitlines()[1:] if l.startswith("w")]
    a = np.array(rows, dtype=float)
    dur = a[:, 4] - a[:, 3]
    sm = a[:, 6].astype(int)
    per = np.zeros(148)
    n = np.zeros(148)
    for s, d in zip(sm, dur):
        per[s] += d
        n[s] += 1
    per /= np.maximum(n, 1)
    speed += 1.0 / np.maximum(per, 1e-3)
    cnt += 1
speed /= cnt
np.savetxt(dst, speed / speed.mean())
print("weights min %.3f max %.3f" % (speed.min() / speed.mean(), speed.max() / speed.mean()))
