"""A short run of the step under compute-sanitizer (tests/test_gpu_sanitizer.py):
tiny model, a few verify + commit steps at T = 8 / 16 / 33 (graph path, all
kernels incl. the LL all-reduce of a 2-rank fake-peer group)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2506_11309_b200 as pkg  # noqa: E402


def main():
    cfg = synth.CONFIGS["tiny"]
    sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=64 + 256, max_tree=64)
    sh.synth_weights(0)
    sh.synth_prefix_kv(1, 64)
    rng = np.random.default_rng(0)
    for T in (8, 16, 33):
        toks, par = synth.tree_paperlike(T, cfg.vocab, rng)
        r = sh.verify(toks, par)
        sh.commit_kv(r["accepted"])
    sh.close()
    if "--tp" in sys.argv:
        import torch
        from paper_2506_11309_b200 import swiftspec as ssp
        cfg = synth.CONFIGS["small-tp"]
        shards = []
        for r in range(2):
            s = pkg.Shard(cfg, r, 2, 0, max_ctx=256, max_tree=16)
            s.set_launch_cap(74)
            s.synth_weights(0)
            s.synth_prefix_kv(1, 64)
            shards.append(s)
        pkg.Shard.import_local_peers(shards)
        toks, par = synth.tree_paperlike(8, cfg.vocab, rng)
        bufs = [(torch.tensor(toks, dtype=torch.int32, device="cuda"), torch.tensor(par, dtype=torch.int32, device="cuda"),
                 torch.zeros(ssp.result_nbytes() // 4, dtype=torch.int32, device="cuda")) for _ in shards]
        torch.cuda.synchronize()
        streams = [torch.cuda.Stream() for _ in shards]
        for s, st, (dt, dp, res) in zip(shards, streams, bufs):
            s.verify_dev(dt, dp, 8, d_result=res, auto_commit=True, stream=st)
        torch.cuda.synchronize()
        for s in shards:
            s.close()
    print("SANITIZE_STEP_DONE")


if __name__ == "__main__":
    main()
