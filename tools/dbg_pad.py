import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import synth, oracle as O
from test_tp_fakepeer import _setup, _run
cfg = synth.CONFIGS["small-tp"]
for P, mixed in ((2, True), (3, False), (3, True)):
    shards, m, kv = _setup(cfg, P, 64)
    rng = np.random.default_rng(1)
    if mixed:
        t, p = synth.tree_paperlike(8, cfg.vocab, rng)
        outs = _run(shards, t, p)
        print("P", P, "first verify status", [o[0]["status"] for o in outs], flush=True)
        for sh in shards: sh.set_committed_len(64)
    for step in range(2):
        t, p = synth.tree_random(8, cfg.vocab, rng)
        outs = _run(shards, t, p, auto_commit=True)
        print("P", P, "mixed", mixed, "step", step, [o[0]["status"] for o in outs], [sh.L for sh in shards], flush=True)
    for sh in shards: sh.close()
