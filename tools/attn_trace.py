#!/usr/bin/env python3
"""Per-CTA timeline of the attention kernel (layer 0) from the SS_ATTN_TRACE build:
   SWIFTSPEC_LIB=libswiftspec_atrace.so python tools/attn_trace.py"""
import ctypes as C
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2506_11309_b200 as pkg  # noqa: E402
from paper_2506_11309_b200 import swiftspec as ssp  # noqa: E402

T = int(os.environ.get("TR_T", "8"))
cfg = dataclasses.replace(synth.CONFIGS["llama3-70b"], n_layers=2)
sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=4096 + 512, max_tree=max(8, T))
sh.synth_weights(0)
sh.synth_prefix_kv(1, 4096)
dev = torch.device("cuda", 0)
for i in range(3):
    t, p = synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(i))
    sh.verify_dev(torch.tensor(t, dtype=torch.int32, device=dev), torch.tensor(p, dtype=torch.int32, device=dev), T,
                  auto_commit=True, stream=torch.cuda.current_stream())
torch.cuda.synchronize()
L = ssp.lib()
buf = (C.c_ulonglong * (256 * 8))()
L.ss_debug_attn_trace(buf)
a = np.array(buf, dtype=np.int64).reshape(256, 8)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
names = ["entry", "pdl", "q", "loop_end", "fenced", "meet", "merged"]
for e, n in enumerate(names):
    v = a[:, e] - t0
    print(f"{n:9s} min {v.min():7d} p50 {int(np.median(v)):7d} max {v.max():7d}")

tb = (C.c_ulonglong * (256 * 16))()
L.ss_debug_attn_tiles(tb)
tt = np.array(tb, dtype=np.int64).reshape(256, 16)[:, 0::2]
tt = tt[a.shape[0] and slice(0, a.shape[0])]
q = a[:, 2]
for i in range(5):
    col = tt[:, i]
    m = col > 0
    if not m.any():
        break
    d = (col[m] - q[m])
    print(f"tile {i} wait done after q: min {d.min():6d} p50 {int(np.median(d)):6d} max {d.max():6d} ns")
