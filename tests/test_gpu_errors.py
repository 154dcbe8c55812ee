"""Device-detected error codes through the real library (include/swiftspec.h
"Errors"): SS_ETIMEOUT (an inbox message that never arrives,
S:340), SS_ECONSISTENCY (TP ranks called with different trees, debug
checksum), SS_EINVAL for a mailbox tree beyond the target's max_tree, and the
host-side SS_ESTATE / SS_ECAPACITY order on a live shard."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _tiny(max_tree=8, L=64):
    import paper_2506_11309_b200 as pkg
    cfg = synth.CONFIGS["tiny"]
    sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=L + 128, max_tree=max_tree)
    sh.synth_weights(0)
    sh.synth_prefix_kv(1, L)
    return cfg, sh


def test_estate_two_verifies_without_commit():
    import paper_2506_11309_b200 as pkg
    cfg, sh = _tiny()
    toks, par = synth.tree_paperlike(8, cfg.vocab, np.random.default_rng(0))
    sh.verify(toks, par)
    with pytest.raises(pkg.SwiftSpecError, match="SS_ESTATE"):
        sh.verify(toks, par)
    assert "pending" in pkg.lib().ss_last_error(sh.h).decode()
    sh.commit_accepted()
    sh.verify(toks, par)                 # fine after the commit
    sh.set_committed_len(64)            # discard
    sh.verify(toks, par)
    sh.close()


def test_mailbox_timeout_and_oversized_tree():
    import torch
    from paper_2506_11309_b200 import swiftspec as ssp
    cfg, sh = _tiny(max_tree=8)
    outbox = torch.zeros((1 + 64) * 4, dtype=torch.int32, device="cuda")
    sh.attach_mailbox(outbox.data_ptr(), eos=-1)
    res = torch.zeros(4 + 2 * 64, dtype=torch.int32, device="cuda")
    # (1) nothing is ever posted: the inbox poll gives up after its 2 s budget,
    # the target posts nothing for that message, so the draft's wait times out too
    sh.verify_mailbox(auto_commit=True)
    ssp.mailbox_recv_result(outbox.data_ptr(), 1, res.data_ptr())
    torch.cuda.synchronize()
    r = res.cpu().numpy()
    assert int(r[3]) == -5 and int(r[0]) == -1         # SS_ETIMEOUT, no message
    assert sh.L == 64                                   # nothing committed
    # (2) the same message number is polled again by the next step; a tree of
    # 12 > max_tree = 8 nodes is refused on the device (SS_EINVAL)
    toks, par = synth.tree_random(12, cfg.vocab, np.random.default_rng(1))
    sh.verify_mailbox(auto_commit=True, stream=torch.cuda.Stream())
    ssp.mailbox_post_tree(sh.mailbox_inbox(), toks, par, 1, stream=torch.cuda.Stream())
    ssp.mailbox_recv_result(outbox.data_ptr(), 1, res.data_ptr(), stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    r = res.cpu().numpy()
    assert int(r[3]) == -1 and int(r[0]) == 0           # SS_EINVAL
    assert sh.L == 64
    # (3) a valid tree with the next sequence number works
    toks, par = synth.tree_paperlike(8, cfg.vocab, np.random.default_rng(2))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    sh.verify_mailbox(auto_commit=True, stream=s1)
    ssp.mailbox_post_tree(sh.mailbox_inbox(), toks, par, 2, stream=s2)
    ssp.mailbox_recv_result(outbox.data_ptr(), 2, res.data_ptr(), stream=s2)
    torch.cuda.synchronize()
    r = res.cpu().numpy()
    assert int(r[3]) == 0 and int(r[0]) >= 1
    assert sh.L == 64 + int(r[0])
    sh.close()


def test_consistency_checksum_across_fake_peers():
    """SS_DEBUG_CONSISTENCY: two TP ranks called with different trees both fail
    with SS_ECONSISTENCY and commit nothing; identical trees pass."""
    import torch
    import paper_2506_11309_b200 as pkg
    from paper_2506_11309_b200 import swiftspec as ssp
    cfg = synth.CONFIGS["small-tp"]
    shards = []
    for r in range(2):
        sh = pkg.Shard(cfg, r, 2, 0, max_ctx=256, max_tree=16)
        sh.set_launch_cap(74)
        sh.synth_weights(0)
        sh.synth_prefix_kv(1, 64)
        sh.set_debug(ssp.SS_DEBUG_CONSISTENCY)
        shards.append(sh)
    pkg.Shard.import_local_peers(shards)
    rng = np.random.default_rng(3)
    ta, pa = synth.tree_paperlike(8, cfg.vocab, rng)
    tb = ta.copy()
    tb[5] = (tb[5] + 1) % cfg.vocab

    def run(trees):
        outs, bufs = [], []
        for sh, (t, p) in zip(shards, trees):
            bufs.append((torch.tensor(t, dtype=torch.int32, device="cuda"),
                         torch.tensor(p, dtype=torch.int32, device="cuda"),
                         torch.zeros(ssp.result_nbytes() // 4, dtype=torch.int32, device="cuda")))
        torch.cuda.synchronize()
        streams = [torch.cuda.Stream() for _ in shards]
        for sh, st, (dt, dp, res) in zip(shards, streams, bufs):
            sh.verify_dev(dt, dp, 8, d_result=res, auto_commit=True, stream=st)
        torch.cuda.synchronize()
        return [ssp.parse_result(res.cpu().numpy(), 8) for _, _, res in bufs]

    bad = run([(ta, pa), (tb, pa)])
    assert [r["status"] for r in bad] == [-3, -3]
    assert [sh.L for sh in shards] == [64, 64]
    good = run([(ta, pa), (ta, pa)])
    assert [r["status"] for r in good] == [0, 0]
    assert good[0]["accepted"] == good[1]["accepted"]
    assert [sh.L for sh in shards] == [64 + good[0]["n_accepted"]] * 2
    for sh in shards:
        sh.close()
