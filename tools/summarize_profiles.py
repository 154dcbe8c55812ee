#!/usr/bin/env python3
"""Turn the raw ncu outputs of tools/profile_round.sh (gpurun_out/) into the
committed evidence under profiles/:

  profiles/<round>_launch_list.csv     per-launch device time of ONE bench step
  profiles/<round>_launches.md         per-kernel-kind totals, shares of the step
  profiles/<round>_ncu_kernels.md      ncu --set full metrics of the hot kernels
  profiles/traffic.json                DRAM bytes per launch (bench.py roofline.traffic)

    python tools/summarize_profiles.py --round r01
"""
import argparse
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KIND = [("gemm_kernel<0, ", "w4_gemm"), ("gemm_kernel<1, ", "lm_head"), ("attn_kernel", "attention"),
        ("prep_norm", "rmsnorm"), ("embed_meta", "embed+tree"), ("commit_kernel", "commit")]
EPI = {"0>": "qkv+rope", "1>": "resid(+AR)", "2>": "gate_up+swiglu", "3>": "lm_head+argmax"}


def label(name):
    for pat, k in KIND:
        if pat in name:
            if k in ("w4_gemm", "lm_head"):
                epi = name.split(",")[-1].split("(")[0].strip()
                return EPI.get(epi, k)
            return k
    return name[:30]


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name", "").startswith("gpu__time_duration"):
                data.append(d)
    return data


def one_step(data):
    """The last complete step: from the last embed_meta launch before the final
    commit_kernel through that commit."""
    names = [d["Kernel Name"] for d in data]
    commits = [i for i, n in enumerate(names) if "commit_kernel" in n]
    end = commits[-1]
    start = max(i for i, n in enumerate(names[:end]) if "embed_meta" in n)
    return data[start:end + 1]


def ncu_raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    return rows[0], rows[1], rows[2:]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    rd = a.round

    # ---- launch list of one bench step
    data = read_launches(os.path.join(OUT, "bench_launches.csv"))
    step = one_step(data)
    with open(os.path.join(PROF, f"{rd}_launch_list.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["idx", "kernel", "kind", "grid", "block", "duration_ns"])
        for i, d in enumerate(step):
            w.writerow([i, d["Kernel Name"][:80], label(d["Kernel Name"]), d["Grid Size"], d["Block Size"],
                        d["Metric Value"]])
    agg = OrderedDict()
    for d in step:
        k = label(d["Kernel Name"])
        t = float(d["Metric Value"])
        a_ = agg.setdefault(k, [0.0, 0])
        a_[0] += t
        a_[1] += 1
    tot = sum(v[0] for v in agg.values())
    lines = [f"# {rd}: launch list of one bench step (ncu, cold-cache, serialised)", "",
             "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -k regex:... "
             "python bench.py --steps 2 --warmup 3 --no-cpu-baseline` (70B-shaped int4, T=8, L=4096, TP=1).",
             "Per-launch times are serialised by ncu (no PDL overlap, caches cold), so compare SHARES with the",
             "live bench, not absolutes.", "",
             f"Launches in the step: {len(step)}; sum of launch times: {tot / 1e3:.1f} us", "",
             "| kernel kind | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        lines.append(f"| {k} | {n} | {t / 1e3:.1f} | {t / n / 1e3:.2f} | {t / tot:.3f} |")
    open(os.path.join(PROF, f"{rd}_launches.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

    # ---- ncu --set full of the GEMMs and attention
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.per_cycle_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
    md = [f"# {rd}: ncu --set full of the hot kernels", "",
          "Captured with `ncu --set full --clock-control none --import-source on` on "
          "`tools/prof_step.py --layers 2` (70B-shaped layers, T=8, L=4096, TP=1): the per-launch shapes are",
          "identical to the full 80-layer step.", ""]
    traffic = {}
    names = {0: "qkv", 1: "o_proj", 2: "gate_up", 3: "down", 4: "lm_head"}
    for rep, tag in (("full_gemm.ncu-rep", "gemm"), ("full_attn.ncu-rep", "attn")):
        p = os.path.join(OUT, rep)
        if not os.path.exists(p):
            continue
        hdr, units, rows = ncu_raw(p)
        for i, r in enumerate(rows):
            kname = r[hdr.index("Kernel Name")]
            md.append(f"## {label(kname)} — `{kname[:60]}`")
            md.append("")
            md.append("| metric | value |")
            md.append("|---|---|")
            for k in want:
                if k in hdr:
                    md.append(f"| {k} | {r[hdr.index(k)]} {units[hdr.index(k)]} |")
            st = []
            for j, h in enumerate(hdr):
                if "average_warps_issue_stalled" in h and "per_issue_active" in h:
                    try:
                        v = float(r[j])
                    except ValueError:
                        continue
                    if v > 0.3:
                        st.append((v, h.replace("smsp__average_warps_issue_stalled_", "").replace(
                            "_per_issue_active.ratio", "")))
            md.append(f"| top stalls (warps per issue) | {', '.join(f'{n} {v:.2f}' for v, n in sorted(st, reverse=True)[:6])} |")
            md.append("")
            if tag == "gemm" and label(kname) == "gate_up+swiglu":
                ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
                rd_b = float(r[ir]) * SCALE.get(units[ir], 1)
                wr_b = float(r[iw]) * SCALE.get(units[iw], 1)
                traffic["llama3-70b/tp1/T8/gate_up"] = rd_b + wr_b
    json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    open(os.path.join(PROF, f"{rd}_ncu_kernels.md"), "w").write("\n".join(md) + "\n")
    print("traffic", traffic)


if __name__ == "__main__":
    sys.exit(main())
