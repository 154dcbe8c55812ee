"""Error budget of the GPU path's roundings, emulated on the float64 oracle's
layer (R18): which rounding point dominates the logit error against
the R13 tolerance (|g - o| <= 2e-2 + 1e-2 |o|)?

    python tools/err_budget.py [--config tiny] [--adversarial] [--layers N] [--T 8]

Each variant re-runs the oracle's layer stack with roundings applied at named
points; the report gives the worst ratio err / tolerance over all logits.
Points:  act  = fp16 inputs of the W4 GEMMs (xn, attention out, SwiGLU out)
         qk   = fp16 post-RoPE q and tree K (cache)
         v    = fp16 tree V
         p    = fp16 softmax probabilities before P.V
         bf16 = everything above in bf16 (the paper's BF16 compute)
Timing-free analysis tool; not used by tests or the product.
"""
import argparse
import dataclasses
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import synth  # noqa: E402
from synth import fast  # noqa: E402


def r16(x):
    return np.asarray(x, dtype=np.float64).astype(np.float16).astype(np.float64)


def rbf(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32)
    b = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return b.view(np.float32).astype(np.float64)


def layer(cfg, m, l, x, kv, L, pos, anc, R):
    T = x.shape[0]
    Hq, Hkv, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    xn = R["act"](O.rmsnorm(x, m.norm(l, "attn_norm"), cfg.rms_eps))
    q = m.matmul(l, "wq", xn).reshape(T, Hq, d)
    k = m.matmul(l, "wk", xn).reshape(T, Hkv, d)
    v = m.matmul(l, "wv", xn).reshape(T, Hkv, d)
    for i in range(T):
        q[i] = O.rope(q[i], pos[i], cfg.rope_theta)
        k[i] = O.rope(k[i], pos[i], cfg.rope_theta)
    q, k, v = R["q"](R["qk"](q)), R["k"](R["qk"](k)), R["v"](v)
    attn = np.zeros((T, Hq * d))
    Kp, Vp = kv.K[l][:L], kv.V[l][:L]
    rep = Hq // Hkv
    for i in range(T):
        sel = np.nonzero(anc[i])[0]
        keys = np.concatenate([Kp, k[sel]])
        vals = np.concatenate([Vp, v[sel]])
        for h in range(Hq):
            sc = keys[:, h // rep, :] @ q[i, h] / math.sqrt(d)
            e = np.exp(sc - sc.max())
            p = R["p"](e / e.sum())
            attn[i, h * d:(h + 1) * d] = p @ vals[:, h // rep, :]
    x = x + m.matmul(l, "wo", R["act"](attn))
    xn2 = R["act"](O.rmsnorm(x, m.norm(l, "mlp_norm"), cfg.rms_eps))
    hm = R["act"](O.silu(m.matmul(l, "wgate", xn2)) * m.matmul(l, "wup", xn2))
    return x + m.matmul(l, "wdown", hm)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--adversarial", action="store_true")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--T", type=int, default=8)
    ap.add_argument("--L", type=int, default=64)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    if a.layers:
        cfg = dataclasses.replace(cfg, n_layers=a.layers)
    if a.adversarial:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from test_gpu_parity import _adversarial_model
        canon = _adversarial_model(cfg)
    else:
        canon = synth.gen_model(cfg, 0)
    m = O.OracleModel(cfg, canon)
    kv = O.KVCache(cfg, a.L + 64)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(1, l, a.L, cfg.n_kv_heads, cfg.head_dim)
        kv.set_prefix(l, k, v)
    kv.L = a.L
    toks, par = synth.tree_paperlike(a.T, cfg.vocab, np.random.default_rng(a.T))
    depth, pos, anc = O.tree_meta(par, a.L)
    ident = lambda z: np.asarray(z, dtype=np.float64)
    variants = {
        "exact": {},
        "act": {"act": r16},
        "qk": {"qk": r16},
        "v": {"v": r16},
        "p": {"p": r16},
        "all-fp16": {"act": r16, "qk": r16, "v": r16, "p": r16},
        "all-but-act": {"qk": r16, "v": r16, "p": r16},
        "all-but-qk": {"act": r16, "v": r16, "p": r16},
        "q": {"q": r16},
        "k": {"k": r16},
        "all-but-q": {"act": r16, "k": r16, "v": r16, "p": r16},
        "k-v-p": {"k": r16, "v": r16, "p": r16},
        "bf16": {"act": rbf, "qk": rbf, "v": rbf, "p": rbf},
        "hi-lo act+q": {"k": r16, "v": r16, "p": r16},
        "hi-lo act+q+k": {"v": r16, "p": r16},
        "hi-lo act+q+k+v": {"p": r16},   # the step kernel's design (DESIGN R18)
    }
    ref = None
    for name, rr in variants.items():
        R = {k: rr.get(k, ident) for k in ("act", "qk", "q", "k", "v", "p")}
        x = m.embed_rows(toks)
        for l in range(cfg.n_layers):
            x = layer(cfg, m, l, x, kv, a.L, pos, anc, R)
        lg = m.logits(O.rmsnorm(x, canon["final_norm"], cfg.rms_eps))
        if ref is None:
            ref = lg
            print(f"{cfg.name} L={a.L} T={a.T} adversarial={a.adversarial}: logit std {lg.std():.3g}")
            continue
        err = np.abs(lg - ref)
        print(f"  {name:12s} max|err| {err.max():.3g}  worst ratio {(err / (2e-2 + 1e-2 * np.abs(ref))).max():.3g}")


if __name__ == "__main__":
    main()
