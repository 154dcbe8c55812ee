"""Soak test of the persistent step kernel's hand-offs: the round-2 deadlock
(a warp set checked unit k's MMA completion on the A buffer's mbarrier after
handing unit k + 2 to the MMA warps; when k + 2 completed first the phase
parity aliased and the set waited forever -- DESIGN 10) surfaced in ~0.3 % of
T = 1 host-API decode steps of the 70B-shaped shard.  600 such steps (plus
T = 8 trees) must all complete; a hang traps through the kernel watchdog and
fails the call instead of hanging the GPU."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def test_70b_host_decode_soak():
    import paper_2506_11309_b200 as pkg
    cfg = synth.CONFIGS["llama3-70b"]
    L = 4096
    sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=L + 1024, max_tree=32)
    try:
        sh.synth_weights(0)
        sh.synth_prefix_kv(1, L)
        rng = np.random.default_rng(5)
        cur = 1
        for k in range(600):
            if k % 50 == 49:   # a tree step now and then (NT = 1 as well)
                toks, par = synth.tree_paperlike(8, cfg.vocab, rng)
                toks[0] = cur
                r = sh.verify(toks, par)
            else:
                r = sh.verify(np.array([cur], dtype=np.int32), np.array([-1], dtype=np.int32))
            assert r["status"] == 0
            sh.commit_accepted()
            cur = int(r["bonus"])
            if k % 200 == 199:
                sh.set_committed_len(L)
    finally:
        sh.close()
