#!/usr/bin/env python3
"""profiles/<round>_tp8_ncu.md from tools/profile_tp8.sh outputs (one TP 8 rank, loopback
all-reduce emulation, 2 70B-shaped layers): launch times of the last step + ncu --set full
metrics of the captured launches."""
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_profiles import OUT, PROF, label, ncu_raw  # noqa: E402

rd = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = list(csv.reader(open(os.path.join(OUT, "tp8_launches.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ks = [r for r in rows[hi + 1:] if len(r) > h.index("Metric Value")]
last = max(i for i, r in enumerate(ks) if r[h.index("Kernel Name")].startswith("embed_meta"))
md = [f"# {rd}: one TP 8 rank of the 70B-shaped step (loopback all-reduce emulation on one GPU)", "",
      "`tools/profile_tp8.sh`: `tools/prof_step.py --layers 2 --steps 3 --tp 8` under ncu (serialised, cold",
      "caches: compare shares with the live `tp_emulated` bench lines, not absolutes).  Per-rank shapes:",
      "QKV N = 1280, O K = 1024, gate/up N = 7168, down K = 3584, one kv head; 4K prefix, T = 8.", "",
      "## Launches of one step (2 layers)", "", "| # | kernel | grid | us |", "|---|---|---|---|"]
for i, r in enumerate(ks[last:]):
    md.append(f"| {i} | {label(r[h.index('Kernel Name')])} | {r[h.index('Grid Size')]} | "
              f"{float(r[h.index('Metric Value')]) / 1e3:.1f} |")
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__registers_per_thread"]
hdr, units, rs = ncu_raw(os.path.join(OUT, "tp8_full.ncu-rep"))
md += ["", "## ncu --set full (layer 0 of the third step)", "",
       "| kernel | " + " | ".join(w.split("__")[1].split(".")[0] + "." + w.split(".")[-1] for w in want) + " |",
       "|---" * (len(want) + 1) + "|"]
for r in rs:
    vals = [f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip() if w in hdr else "-" for w in want]
    md.append(f"| {label(r[hdr.index('Kernel Name')])} | " + " | ".join(vals) + " |")
open(os.path.join(PROF, f"{rd}_tp8_ncu.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
