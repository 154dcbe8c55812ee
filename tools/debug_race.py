import sys, os, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
import paper_2506_11309_b200 as pkg
cfg = dataclasses.replace(synth.CONFIGS["llama3-1b"], n_layers=1)
sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=256, max_tree=16)
sh.synth_weights(0); sh.synth_prefix_kv(1, 128)
tokens, parents = synth.tree_paperlike(int(sys.argv[1]) if len(sys.argv) > 1 else 8, cfg.vocab, np.random.default_rng(8))
ref = sh.verify(tokens, parents, want_logits=True)["logits"]
bad = 0
for rep in range(12):
    lg = sh.verify(tokens, parents, want_logits=True)["logits"]
    d = np.abs(lg - ref)
    tg = d[:, :128 * (cfg.vocab // 128)].reshape(d.shape[0], -1, 128).max(axis=(0, 2))
    nb = int((tg > 1e-2).sum())
    bad += nb
print(os.environ.get("SS_NO_PDL"), os.environ.get("SS_GEMM_OCC"), "T", len(tokens), "tile-groups differing across 12 reps:", bad, "max diff", float(d.max()), flush=True)
