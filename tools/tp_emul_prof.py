#!/usr/bin/env python3
"""Eager per-kernel device times of one TP rank (loopback emulation, timing only):
   python tools/tp_emul_prof.py [P] [T]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2506_11309_b200 as pkg  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = synth.CONFIGS["llama3-70b"]
sh = pkg.Shard(cfg, 0, P, 0, max_ctx=4096 + 512, max_tree=max(8, T))
sh.synth_weights(0)
sh.synth_prefix_kv(1, 4096)
if P > 1:
    sh.import_loopback()
dev = torch.device("cuda", 0)
t, p = synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(0))
dt = torch.tensor(t, dtype=torch.int32, device=dev)
dp = torch.tensor(p, dtype=torch.int32, device=dev)
for _ in range(3):
    prof = sh.profile_step(dt, dp, T, stream=torch.cuda.current_stream())
tot = sum(v[0] for v in prof.values())
print(f"P={P} T={T} eager step {tot:.3f} ms")
for k, (ms, n) in prof.items():
    print(f"  {k:24s} launches {n:4d}  avg {1e3 * ms / max(n, 1):8.1f} us  total {ms:7.3f} ms")
