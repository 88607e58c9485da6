"""Summarise the round's ncu captures into profiles/<tag>_*.md (committed).

    python tools/ncu_summary.py r01
reads gpurun_out/<tag>_launches.csv, <tag>_gemv.ncu-rep, <tag>_prefill.ncu-rep.
"""

from __future__ import annotations

import collections
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active", "IMMA subpipe %"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "HMMA subpipe %"),
    ("sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active", "tcgen05/UTC pipe %"),
    ("smsp__inst_executed.sum", "instructions"),
]


def raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (r[i], units[i]) for i, h in enumerate(hdr)}
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(r[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        d["_stalls"] = [(n, v / tot) for v, n in sorted(stalls, reverse=True)[:6]]
        res.append(d)
    return res


def kernel_md(d: dict) -> str:
    name = d["Kernel Name"][0]
    lines = [f"### `{name[:110]}`", "", "| metric | value |", "|---|---|"]
    for k, label in KEYS:
        if k in d:
            v, u = d[k]
            lines.append(f"| {label} (`{k}`) | {v} {u} |")
    lines.append("| top stalls | " + ", ".join(f"{n} {v:.0%}" for n, v in d["_stalls"]) + " |")
    return "\n".join(lines) + "\n"


def launches(tag: str) -> str:
    path = os.path.join(OUT, f"{tag}_launches.csv")
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        k = re.sub(r"\(.*", "", r[ik]).replace("unnamed>::", "")
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + float(r[iv].replace(",", "")) / 1e3)
    total = sum(t for _, t in agg.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {t / total:.1%} |")
    lines.append(f"| **one decode step (serialised, cold)** | {sum(c for c, _ in agg.values())} | "
                 f"{total:.1f} | 100% |")
    return "\n".join(lines) + "\n"


def main(tag: str) -> None:
    os.makedirs(PROF, exist_ok=True)
    md = [f"# {tag}: ncu launch list — one 70B int8 decode step, 80 blocks, 1 x B200", "",
          "Command: `python bench.py --no-cpu` under `ncu --metrics gpu__time_duration.sum "
          "--clock-control none -k regex:\"gemv3|attn_dec|row_stats\" -s 401 -c 401` (the second "
          "warm-up step). Per-launch times are cold-cache and serialised: compare shares.", "",
          launches(tag)]
    open(os.path.join(PROF, f"{tag}_decode_launches.md"), "w").write("\n".join(md))
    for part, title in (("gemv", "decode GEMV (gate/up of block 1, 469.8 MB int8 weights)"),
                        ("prefill", "prefill: tcgen05 int8 GEMM and tensor-core flash attention")):
        rep = os.path.join(OUT, f"{tag}_{part}.ncu-rep")
        if not os.path.exists(rep):
            continue
        ks = raw(rep)
        md = [f"# {tag}: ncu --set full — {title}", "",
              "Captured with `--set full --clock-control none --import-source on` "
              "(tools/profile.sh); source report in gpurun_out/ (scratch).", ""]
        md += [kernel_md(d) for d in ks]
        open(os.path.join(PROF, f"{tag}_{part}.md"), "w").write("\n".join(md))
    print("wrote", sorted(os.listdir(PROF)))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
