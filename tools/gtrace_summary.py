"""Summarise SP_GEMV_TRACE output (per-warp globaltimer phases of one gemv3 launch)."""
import sys

import numpy as np

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gtrace.txt"
for blk in open(path).read().split("gemv N=")[1:]:
    rows = [l.split(":")[1].split() for l in blk.splitlines()[1:] if l.startswith("w")]
    a = np.array(rows, dtype=float)
    print("N K =", blk.splitlines()[0])
    for p, name in enumerate(["start", "post-wait", "post-prologue", "first-stage", "mainloop-end",
                              "exit"]):
        col = a[:, p]
        col = col[col >= 0]
        if col.size:
            print(f"  {name:14s} min {col.min():7.2f} p50 {np.median(col):7.2f} "
                  f"p99 {np.percentile(col, 99):7.2f} max {col.max():7.2f}")
