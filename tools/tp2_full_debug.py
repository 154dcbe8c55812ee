#!/usr/bin/env python3
"""Debug: 70B-shaped 1-layer model, TP1 (uncapped) as reference vs variants."""
import dataclasses, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth
import paper_2506_11309_b200 as pkg
from test_tp_fakepeer import _run
cfg = dataclasses.replace(synth.CONFIGS[os.environ.get("CFG", "llama3-70b")], n_layers=int(os.environ.get("NL", "1")))
T = 8
tokens, parents = synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(72))
def make(P, L, cap):
    shs = []
    for r in range(P):
        sh = pkg.Shard(cfg, r, P, 0, max_ctx=L + 64, max_tree=8)
        if cap: sh.set_launch_cap(cap)
        sh.synth_weights(0); sh.synth_prefix_kv(1, L)
        shs.append(sh)
    if P > 1: pkg.Shard.import_local_peers(shs)
    return shs
def go(P, L, cap):
    shs = make(P, L, cap)
    import time; t0 = time.time(); outs = _run(shs, tokens, parents); print('step wall s', round(time.time() - t0, 3))
    print('status', [o[0]['status'] for o in outs], flush=True)
    lg = np.concatenate([o[1] for o in outs], axis=1)[:, :cfg.vocab]
    for s in shs: s.close()
    return lg
for L in [int(x) for x in os.environ.get("LS", "4096").split(",")]:
    ref = go(1, L, 0)
    for (P, cap) in ([(2, 74)] if os.environ.get('ONLY2') else [(1, 0), (1, 74), (1, 37), (2, 74), (2, 74)]):
        d = np.abs(go(P, L, cap) - ref)
        print(f"mask={os.environ.get('SS_NO_PDL_MASK')} L={L} P={P} cap={cap}: max {d.max():.4f} mean {d.mean():.5f}", flush=True)
