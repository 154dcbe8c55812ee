"""Debug: one verify of a small config at TP > 1 (loopback), step kernel on/off; prints status + timing."""
import dataclasses, faulthandler, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synth
import paper_2506_11309_b200 as pkg

faulthandler.dump_traceback_later(100, exit=True)
cfg_name, tp, step, layers = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = dataclasses.replace(synth.CONFIGS[cfg_name], n_layers=layers)
sh = pkg.Shard(cfg, 0, tp, 0, max_ctx=64 + 256, max_tree=16)
sh.synth_weights(0)
sh.synth_prefix_kv(1, 64)
if tp > 1:
    sh.import_loopback()
sh.set_step_kernel(bool(step))
toks, par = synth.tree_paperlike(8, cfg.vocab, np.random.default_rng(0))
for i in range(2):
    sh.set_committed_len(64)
    t0 = time.time()
    r = sh.verify(toks, par)
    print(cfg_name, "tp", tp, "step", step, "status", r["status"], "argmax", r["argmax"][:4], f"{(time.time()-t0)*1e3:.1f} ms", flush=True)
sh.close()
