import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O, synth
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'tests'))
from test_gpu_parity import build, oracle_setup
cfg = synth.CONFIGS["llama3-1b"]
L = 1024
m, kv = oracle_setup(cfg, L=L, max_ctx=L + 64)
m.cache_dense = False
sh = build(cfg, L=L, max_ctx=L + 64)
rng = np.random.default_rng(8)
tokens, parents = synth.tree_paperlike(8, cfg.vocab, rng)
ro = O.verify(cfg, m, kv, tokens, parents)
for rep in range(2):
    rg = sh.verify(tokens, parents, want_logits=True)
    err = np.abs(rg["logits"] - ro["logits"])
    tg = err.reshape(8, -1)[:, :128 * 1002].reshape(8, 1002, 128).max(axis=2)
    bad = np.nonzero(tg.max(axis=0) > 0.05)[0]
    print("rep", rep, "bad tgs", len(bad), bad[:40], flush=True)
    print(" rows bad per tg sample", [(int(b), np.nonzero(tg[:, b] > 0.05)[0].tolist()) for b in bad[:8]])
    b0 = bad[0] if len(bad) else 0
    cols = np.nonzero(err[:, b0*128:(b0+1)*128].max(axis=0) > 0.05)[0]
    print(" tg", b0, "bad cols", cols[:64].tolist())
    print(" gpu", rg["logits"][0, b0*128:b0*128+8], "oracle", ro["logits"][0, b0*128:b0*128+8])
