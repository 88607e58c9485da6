"""Summarise the round's ncu captures into profiles/<tag>_*.md (committed).

    python tools/ncu_summary.py r01
reads gpurun_out/<tag>_launches.csv, <tag>_gemv.ncu-rep, <tag>_prefill.ncu-rep.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("NCU_OUT", os.path.join(ROOT, "gpurun_out"))
PROF = os.environ.get("NCU_PROF", os.path.join(ROOT, "profiles"))

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


def launches(tag: str, name: str = "launches", label: str = "one decode step") -> str:
    path = os.path.join(OUT, f"{tag}_{name}.csv")
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    im = hdr.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        k = re.sub(r"\(.*", "", r[ik]).replace("unnamed>::", "")
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + float(r[iv].replace(",", "")) / 1e3)
    total = sum(t for _, t in agg.values())
    lines = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {t / total:.1%} |")
    lines.append(f"| **{label} (serialised, cold)** | {sum(c for c, _ in agg.values())} | "
                 f"{total:.1f} | 100% |")
    return "\n".join(lines) + "\n"


def dram_per_launch(tag: str, name: str) -> list[tuple[str, float, float]]:
    """(kernel, duration us, dram read+write bytes) per launch of a --set full report."""
    rep = os.path.join(OUT, f"{tag}_{name}.ncu-rep")
    out = []
    for d in raw(rep):
        def num(k):
            v, u = d[k]
            f = float(v.replace(",", ""))
            return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1, "ms": 1e3,
                        "ns": 1e-3, "usecond": 1, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1)
        out.append((d["Kernel Name"][0], num("gpu__time_duration.sum"),
                    num("dram__bytes_read.sum") + num("dram__bytes_write.sum")))
    return out


TITLES = {
    "gemv": "decode GEMVs of one block (QKV, O, gate/up, down): the dominant kernel",
    "attn_dec": "decode attention (RoPE + KV append, 8-CTA cluster flash decode, one block)",
    "attn_pf": "prefill attention on tcgen05 + TMEM (2048 tokens, one block)",
    "pair_gemm": "prefill tcgen05 CTA-pair GEMM (gate/up, 2048 tokens)",
    "prefill": "prefill attention + digitize (2048 tokens)",
}


def main(tag: str) -> None:
    os.makedirs(PROF, exist_ok=True)
    md = [f"# {tag}: ncu launch list — one 70B int8 decode step, 80 blocks, 1 x B200", "",
          "Command: `python bench.py --no-cpu` under `ncu --metrics gpu__time_duration.sum "
          "--clock-control none -k regex:\"gemv3|attn_dec|row_stats\" -s 401 -c 401` (a "
          "warm-up step). Per-launch times are cold-cache and serialised: compare shares.", "",
          launches(tag)]
    pl = os.path.join(OUT, f"{tag}_prefill_launches.csv")
    if os.path.exists(pl):
        md += ["", f"## one block of the timed 2048-token prefill (`--blocks 1`)", "",
               launches(tag, "prefill_launches", "one block's prefill")]
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(md))
    for part, title in TITLES.items():
        rep = os.path.join(OUT, f"{tag}_{part}.ncu-rep")
        if not os.path.exists(rep):
            continue
        ks = raw(rep)
        md = [f"# {tag}: ncu --set full — {title}", "",
              "Captured by tools/profile.sh (`--set full --clock-control none --import-source on`); "
              "the .ncu-rep stays in gpurun_out/ (scratch).", ""]
        md += [kernel_md(d) for d in ks]
        open(os.path.join(PROF, f"{tag}_{part}.md"), "w").write("\n".join(md))
    gv = os.path.join(OUT, f"{tag}_gemv.ncu-rep")
    if os.path.exists(gv):
        per = dram_per_launch(tag, "gemv")
        json.dump({"source": f"ncu --set full, {len(per)} gemv3 launches of one block "
                             f"(tools/profile.sh {tag})",
                   "launches": [{"kernel": k[:60], "us": t, "dram_bytes": b} for k, t, b in per],
                   "dram_bytes_per_launch": sum(b for _, _, b in per) / len(per)},
                  open(os.path.join(PROF, "gemv_traffic.json"), "w"), indent=1)
    print("wrote", sorted(os.listdir(PROF)))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
