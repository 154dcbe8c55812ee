#!/usr/bin/env python3
"""Profiling driver for ncu: a 70B-shaped model with fewer layers, graph steps.

    ncu ... python tools/prof_step.py --layers 4 --T 8 --L 4096 --steps 3
"""
import argparse
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama3-70b")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--T", type=int, default=8)
    ap.add_argument("--L", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--eager-profile", action="store_true")
    ap.add_argument("--tp", type=int, default=1, help="one rank of a TP group, loopback all-reduce (timing emulation)")
    a = ap.parse_args()
    cfg = dataclasses.replace(synth.CONFIGS[a.config], n_layers=a.layers)
    sh = pkg.Shard(cfg, 0, a.tp, 0, max_ctx=a.L + 64 * (a.steps + 4), max_tree=max(8, a.T))
    sh.synth_weights(0)
    sh.synth_prefix_kv(1, a.L)
    if a.tp > 1:
        sh.import_loopback()
    trees = [synth.tree_paperlike(a.T, cfg.vocab, np.random.default_rng(i)) for i in range(a.steps)]
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    for t, p in trees:
        dt = torch.tensor(t, dtype=torch.int32, device=dev)
        dp = torch.tensor(p, dtype=torch.int32, device=dev)
        if a.eager_profile:
            print(sh.profile_step(dt, dp, a.T, stream=st))
        else:
            sh.verify_dev(dt, dp, a.T, auto_commit=True, stream=st)
    torch.cuda.synchronize()
    print("ok", sh.L)


if __name__ == "__main__":
    main()
