#!/usr/bin/env python3
"""Graph-mode cost of each launch kind for one TP rank (loopback emulation):
SS_EXP_SKIP masks, timing only.   python tools/tp_emul_skip.py [P]"""
import os
import subprocess
import sys

P = sys.argv[1] if len(sys.argv) > 1 else "8"
code = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2506_11309_b200 as pkg
P = int(sys.argv[1]); T = 8; cfg = synth.CONFIGS["llama3-70b"]; n = 13
sh = pkg.Shard(cfg, 0, P, 0, max_ctx=4096 + 512, max_tree=8)
sh.synth_weights(0); sh.synth_prefix_kv(1, 4096)
if P > 1: sh.import_loopback()
dev = torch.device("cuda", 0); st = torch.cuda.current_stream()
tr = [synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(i)) for i in range(n)]
dt = torch.tensor(np.stack([t for t, _ in tr]), dtype=torch.int32, device=dev)
dp = torch.tensor(np.stack([p for _, p in tr]), dtype=torch.int32, device=dev)
for i in range(3): sh.verify_dev(dt[i], dp[i], T, auto_commit=True, stream=st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for i in range(3, n): sh.verify_dev(dt[i], dp[i], T, auto_commit=True, stream=st)
e1.record(st); torch.cuda.synchronize()
print(e0.elapsed_time(e1) / (n - 3) * 1e3)
'''
base = None
for m in ([0] if os.environ.get("SKIP0_ONLY") else (0, 1, 2, 4, 8, 16, 31)):
    env = dict(os.environ, SS_EXP_SKIP=str(m))
    out = subprocess.run([sys.executable, "-c", code, P], env=env, capture_output=True, text=True, timeout=200)
    us = float(out.stdout.strip().splitlines()[-1])
    base = us if m == 0 else base
    print(f"P={P} skip={m:2d} step {us:9.1f} us   saved {base - us:8.1f} us = {(base - us) / 80:6.2f} us/layer")
