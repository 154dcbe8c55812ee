"""Quick GPU check of the persistent step kernel against the per-phase path and
the oracle (tiny / small-tp / 1-layer 70B shapes).  Prints max errors; used
while developing step.cu (the tests are tests/test_step_kernel.py)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import synth  # noqa: E402
import paper_2506_11309_b200 as pkg  # noqa: E402


def run(cfg_name, Ts, L=64, layers=None):
    import dataclasses
    cfg = synth.CONFIGS[cfg_name]
    if layers:
        cfg = dataclasses.replace(cfg, n_layers=layers)
    canon = synth.gen_model(cfg, 0)
    sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=L + 128, max_tree=64)
    sh.load_canonical(canon)
    m = O.OracleModel(cfg, canon)
    kv = O.KVCache(cfg, L + 128)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(1, l, L, cfg.n_kv_heads, cfg.head_dim)
        sh.set_prefix_kv(l, k, v)
        kv.set_prefix(l, k, v)
    kv.L = L
    for T in Ts:
        toks, par = synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(T))
        ro = O.verify(cfg, m, kv, toks, par)
        out = {}
        for mode in (1, 0):
            sh.set_step_kernel(bool(mode))
            sh.set_committed_len(L)
            t0 = time.time()
            rg = sh.verify(toks, par, want_logits=True)
            dt = time.time() - t0
            err = np.abs(rg["logits"] - ro["logits"])
            ratio = (err / (2e-2 + 1e-2 * np.abs(ro["logits"]))).max()
            k, v = sh.read_kv(cfg.n_layers - 1, L, T)
            ek = np.abs(k - ro["tree_k"][-1]).max()
            out[mode] = rg
            print(f"{cfg_name} T={T} {'step' if mode else 'phase'} active={sh.step_kernel_active(T)} "
                  f"status={rg['status']} max|dlogit|={err.max():.3g} ratio={ratio:.3g} |dK|={ek:.3g} "
                  f"argmax_eq={list(rg['argmax']) == list(ro['argmax'])} {dt*1e3:.1f} ms", flush=True)
    sh.close()


if __name__ == "__main__":
    run("tiny", [1, 8, 13, 16, 32])
    run("small-tp", [8, 16])
    run("llama3-1b", [16], L=256, layers=2)
