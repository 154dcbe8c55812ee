import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O, synth
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests'))
from test_gpu_parity import build, oracle_setup
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llama3-1b"]
L = 1024
m, kv = oracle_setup(cfg, L=L, max_ctx=L + 64)
m.cache_dense = False
sh = build(cfg, L=L, max_ctx=L + 64)
for T in [8, 8, 16, 8]:
    rng = np.random.default_rng(T)
    tokens, parents = synth.tree_paperlike(T, cfg.vocab, rng)
    rg = sh.verify(tokens, parents, want_logits=True)
    ro = O.verify(cfg, m, kv, tokens, parents)
    err = np.abs(rg["logits"] - ro["logits"])
    print("T", T, "row max err", err.max(axis=1).round(4), "argmax eq", rg["argmax"] == list(ro["argmax"]), flush=True)
    for l in [0, 7, 15]:
        k, v = sh.read_kv(l, L, T)
        ek = np.abs(O.bf16_to_f64(k) - ro["tree_k"][l]).max(axis=(1, 2))
        ev = np.abs(O.bf16_to_f64(v) - ro["tree_v"][l]).max(axis=(1, 2))
        print("  layer", l, "tree k err", ek.round(3), "v err", ev.round(3), flush=True)
