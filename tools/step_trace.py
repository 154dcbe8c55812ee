#!/usr/bin/env python3
"""Timeline of the persistent step kernel (ss_step_trace): where each layer's
phases start, get their first unit and end, over all CTAs.

    python tools/step_trace.py [--config llama3-70b] [--layers 80] [--T 8] [--L 4096] [--tp 1]
                               [--show 3] [--json out.json]

Per phase of the shown layers: first entry, median / max 'first unit ready'
and median / max exit over the CTAs that had work, relative to the earliest
stamp of the launch (us); then the per-layer critical path averaged over the
middle layers.  --tp > 1 = one rank with loopback all-reduce (timing
emulation).  Measurement tool only (the timeline costs a few global stores).
"""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2506_11309_b200 as pkg  # noqa: E402

PH = ["qkv", "att", "o", "gu", "dn"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3-70b")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--T", type=int, default=8)
    ap.add_argument("--L", type=int, default=4096)
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--show", type=int, default=3)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    if a.layers:
        cfg = dataclasses.replace(cfg, n_layers=a.layers)
    sh = pkg.Shard(cfg, 0, a.tp, 0, max_ctx=a.L + 64 * 12, max_tree=max(8, a.T))
    sh.synth_weights(0)
    sh.synth_prefix_kv(1, a.L)
    if a.tp > 1:
        sh.import_loopback()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    trees = [synth.tree_paperlike(a.T, cfg.vocab, np.random.default_rng(i)) for i in range(4)]
    for t, p in trees[:3]:
        sh.set_committed_len(a.L)
        sh.verify_dev(torch.tensor(t, dtype=torch.int32, device=dev), torch.tensor(p, dtype=torch.int32, device=dev),
                      a.T, auto_commit=False, stream=st)
    torch.cuda.synchronize()
    sh.step_trace(True)
    t, p = trees[3]
    sh.set_committed_len(a.L)
    for _ in range(2):  # first launch after enabling captures the graph; time the second
        sh.set_committed_len(a.L)
        sh.verify_dev(torch.tensor(t, dtype=torch.int32, device=dev), torch.tensor(p, dtype=torch.int32, device=dev),
                      a.T, auto_commit=False, stream=st)
    torch.cuda.synchronize()
    tr, utl = sh.read_step_trace(with_units=True)
    tr = tr.astype(np.int64)
    utl = utl.astype(np.int64)
    sh.close()
    nz = tr[tr > 0]
    t0 = nz.min()
    us = np.where(tr > 0, (tr - t0) / 1e3, np.nan)
    n_l = cfg.n_layers
    out = {"config": cfg.name, "layers": n_l, "T": a.T, "L": a.L, "tp": a.tp, "total_us": float(np.nanmax(us))}
    print(f"{cfg.name} layers={n_l} T={a.T} L={a.L} tp={a.tp}: kernel span {out['total_us']:.1f} us "
          f"({out['total_us'] / n_l:.2f} us/layer)")
    rows = []
    for l in range(n_l):
        for ph in range(5):
            s = us[:, l * 5 + ph, :]
            ok = ~np.isnan(s[:, 0])
            if not ok.any():
                continue
            e, r, x = s[ok, 0], s[ok, 1], s[ok, 2]
            rr = r[~np.isnan(r)]
            rows.append(dict(layer=l, ph=PH[ph], ctas=int(ok.sum()), entry_min=float(np.nanmin(e)),
                             entry_med=float(np.nanmedian(e)),
                             ready_med=float(np.median(rr)) if rr.size else None,
                             ready_max=float(rr.max()) if rr.size else None,
                             exit_med=float(np.nanmedian(x)), exit_max=float(np.nanmax(x))))
    s = us[:, n_l * 5, :]
    ok = ~np.isnan(s[:, 0])
    lm = dict(layer=n_l, ph="lm", ctas=int(ok.sum()), entry_min=float(np.nanmin(s[ok, 0])),
              entry_med=float(np.nanmedian(s[ok, 0])), ready_med=float(np.nanmedian(s[ok, 1])),
              ready_max=float(np.nanmax(s[ok, 1])), exit_med=float(np.nanmedian(s[ok, 2])),
              exit_max=float(np.nanmax(s[ok, 2])))
    rows.append(lm)
    show = set(range(min(a.show, n_l))) | {n_l // 2, n_l - 1, n_l}
    print(f"{'layer':>5} {'ph':>4} {'ctas':>5} {'entry':>9} {'ready50':>9} {'readyMax':>9} {'exit50':>9} {'exitMax':>9}")
    for r in rows:
        if r["layer"] in show:
            f = lambda v: f"{v:9.1f}" if v is not None else "        -"
            print(f"{r['layer']:5d} {r['ph']:>4} {r['ctas']:5d} {f(r['entry_min'])} {f(r['ready_med'])} "
                  f"{f(r['ready_max'])} {f(r['exit_med'])} {f(r['exit_max'])}")
    # per-layer phase spans (exit_max of the phase minus exit_max of the previous phase), middle layers
    mid = [l for l in range(n_l) if n_l // 4 <= l < 3 * n_l // 4] or list(range(n_l))
    span = {p: [] for p in PH}
    prev_end = {}
    for r in rows:
        if r["ph"] == "lm":
            continue
        key = (r["layer"], r["ph"])
        prev_end[key] = r["exit_max"]
    for l in mid:
        for i, p in enumerate(PH):
            prev = prev_end.get((l, PH[i - 1])) if i else prev_end.get((l - 1, "dn"))
            cur = prev_end.get((l, p))
            if prev is not None and cur is not None:
                span[p].append(cur - prev)
    out["phase_span_us"] = {p: float(np.mean(v)) if v else None for p, v in span.items()}
    out["lm_us"] = lm["exit_max"] - prev_end.get((n_l - 1, "dn"), 0.0)
    print("mean critical-path span per phase (middle layers, exitMax - previous exitMax):",
          {p: round(v, 2) if v is not None else None for p, v in out["phase_span_us"].items()},
          f"LM {out['lm_us']:.1f} us")
    out["rows"] = rows
    # CTA 0, gate/up of the middle layer: per-unit clock64 stamps of consumer warp 0
    n_u, tck0 = int(utl[127 * 8 + 6]), int(utl[127 * 8 + 7])
    if n_u:
        U = utl[:127 * 8].reshape(127, 8)[:min(n_u, 127)]
        base = U[0, 0]
        d = lambda x: (x - base)
        print(f"CTA 0 gate/up layer {n_l // 2}: {n_u} units, W4 unit index {tck0}; per unit (clk from start): "
              "wait_start, full, dequant_done, epilogue_done | mma ardy_seen, committed | producer part1, part2")
        for i in range(min(n_u, 12)):
            k = tck0 + i
            m0, m1 = (utl[4096 + 2 * k], utl[4096 + 2 * k + 1]) if k < 4096 else (0, 0)
            p1, p2 = utl[8192 + 2 * i], utl[8192 + 2 * i + 1]
            print(f"  u{i:3d} {d(U[i,0]):8d} {d(U[i,1]):8d} {d(U[i,2]):8d} {d(U[i,3]):8d} | {d(m0):8d} {d(m1):8d}"
                  f" | issued {d(p1):8d} {d(p2):8d} | p2 try {d(utl[12288 + 2 * i]):8d} iters {utl[12288 + 2 * i + 1]}")
        if n_u > 4:
            per = (U[n_u - 1, 3] - U[0, 0]) / n_u
            dq = np.median(U[1:n_u, 2] - U[1:n_u, 1])
            wt = np.median(U[1:n_u, 1] - U[1:n_u, 0])
            print(f"  mean clk per unit {per:.0f}; median full-wait {wt:.0f}, dequant {dq:.0f}")
        nlog = int(utl[20479])
        print(f"  producer loop log ({nlog} iterations, last launch appended after the first):")
        lg = utl[16384:16384 + 2 * nlog].reshape(-1, 2)
        for j in range(max(0, nlog - 60), nlog):
            c, w = lg[j]
            b = utl[24576 + 4 * j:24576 + 4 * j + 3]
            print(f"    it{j:4d} t={d(c):8d} [to-issue {b[0]}, expect_tx {b[1]}, bulk {b[2]}] part1 {w >> 40} clk, part2 {(w >> 16) & 0xFFFFFF} clk, wk-ak={(w & 0xFFFF) >> 1} prog={w & 1}")
        out["unit_clk"] = float((U[min(n_u, 127) - 1, 3] - U[0, 0]) / min(n_u, 127))
    at = utl[28672:28672 + 256]
    if at[0]:
        b = at[0]
        nt = int(at[5])
        print(f"CTA 0 attention layer {n_l // 2}: splits {int(at[6])}, tiles {nt}; clk from entry: qkv-ready {at[1]-b}, "
              f"tiles-done {at[2]-b}, meet {at[3]-b}, merged {at[4]-b}")
        print("  per tile (ready, done):", [(int(at[16 + 2 * j] - b), int(at[17 + 2 * j] - b)) for j in range(min(nt, 8))])
        print("  tile 0/2 (ready, S done, softmax done, PV done):",
              [(int(at[16 + 2 * j] - b), int(at[200 + 4 * j] - b), int(at[201 + 4 * j] - b), int(at[202 + 4 * j] - b)) for j in (0, 2) if j < nt])
    for ph, name in ((0, "qkv"), (2, "o"), (3, "gu"), (4, "dn")):
        tt = utl[30000 + ph * 16:30000 + ph * 16 + 9]
        if tt[0]:
            b = tt[0]
            print(f"tail of {name} (finaliser of tile-group 0, layer {n_l // 2}, nd={tt[8]}): clk after loop end: "
                  f"counted {tt[1]-b}, sent {tt[2]-b if tt[2] else '-'}, received {tt[3]-b if tt[3] else '-'}, "
                  f"epilogue done {tt[4]-b}, cleaned+fence {tt[5]-b}, released {tt[6]-b}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f)


if __name__ == "__main__":
    main()
