"""a13: asynchronous draft -> target handoff through LL-line mailboxes.

The target step polls its inbox on the device, verifies, commits and posts the
verified path to the draft's outbox; a "draft" on another stream posts planted
trees (the target's greedy continuation, computed by the oracle) and reads the
results.  The sequence of emitted tokens must equal plain greedy decoding
 and each step's accept length the planted depth + 1."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


def test_mailbox_golden_decode():
    import torch
    import paper_2506_11309_b200 as pkg
    from paper_2506_11309_b200 import swiftspec as ssp
    cfg = synth.CONFIGS["tiny"]
    L = 64
    canon = synth.gen_model(cfg, 0)
    sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=L + 256, max_tree=8)
    sh.load_canonical(canon)
    m = O.OracleModel(cfg, canon)
    kv = O.KVCache(cfg, L + 256)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(1, l, L, cfg.n_kv_heads, cfg.head_dim)
        sh.set_prefix_kv(l, k, v)
        kv.set_prefix(l, k, v)
    kv.L = L
    root = 321
    ref = O.greedy_decode(cfg, m, kv.copy(), root, 16)

    outbox = torch.zeros((1 + 64) * 4, dtype=torch.int32, device="cuda")
    sh.attach_mailbox(outbox.data_ptr(), eos=-1)
    inbox = sh.mailbox_inbox()
    res = torch.zeros(4 + 2 * 64, dtype=torch.int32, device="cuda")
    target_stream, draft_stream = torch.cuda.Stream(), torch.cuda.Stream()
    rng = np.random.default_rng(0)
    out, cur, seq = [], root, 0
    while len(out) < 16:
        depth = int(rng.integers(0, 4))
        chain = ref[len(out):len(out) + depth]
        toks = [cur] + chain + [int(t) for t in rng.integers(0, cfg.vocab, 8 - 1 - len(chain))]
        parents = list(range(-1, len(chain))) + [int(rng.integers(0, len(chain) + 1)) for _ in range(8 - 1 - len(chain))]
        seq += 1
        # the target starts first and waits on the device for the tree
        sh.verify_mailbox(auto_commit=True, stream=target_stream)
        ssp.mailbox_post_tree(inbox, toks, parents, seq, stream=draft_stream)
        ssp.mailbox_recv_result(outbox.data_ptr(), seq, res.data_ptr(), stream=draft_stream)
        torch.cuda.synchronize()
        r = res.cpu().numpy()
        n, bonus, stop, status = int(r[0]), int(r[1]), int(r[2]), int(r[3])
        nodes = [int(x) for x in r[4:4 + 2 * n:2]]
        path_tokens = [int(x) for x in r[5:5 + 2 * n:2]]
        assert status == 0 and stop == 0 and nodes[0] == 0 and path_tokens[0] == cur
        # distractor children may collide with the greedy token only by chance
        assert n >= len(chain) + 1 or any(toks[c] == ref[len(out) + n - 1] for c in range(1, 8))
        out += path_tokens[1:] + [bonus]
        cur = bonus
    assert out[:16] == ref
    sh.close()


def test_mailbox_stop_on_eos():
    import torch
    import paper_2506_11309_b200 as pkg
    from paper_2506_11309_b200 import swiftspec as ssp
    cfg = synth.CONFIGS["tiny"]
    canon = synth.gen_model(cfg, 0)
    sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=256, max_tree=8)
    sh.load_canonical(canon)
    m = O.OracleModel(cfg, canon)
    kv = O.KVCache(cfg, 256)
    nxt = O.greedy_decode(cfg, m, kv, 5, 1)[0]
    outbox = torch.zeros((1 + 64) * 4, dtype=torch.int32, device="cuda")
    sh.attach_mailbox(outbox.data_ptr(), eos=nxt)       # the next greedy token is the EOS
    res = torch.zeros(4 + 2 * 64, dtype=torch.int32, device="cuda")
    sh.verify_mailbox(auto_commit=True)
    ssp.mailbox_post_tree(sh.mailbox_inbox(), [5], [-1], 1, stream=torch.cuda.Stream())
    ssp.mailbox_recv_result(outbox.data_ptr(), 1, res.data_ptr(), stream=torch.cuda.Stream())
    torch.cuda.synchronize()
    r = res.cpu().numpy()
    assert int(r[0]) == 1 and int(r[1]) == nxt and int(r[2]) == 1 and int(r[3]) == 0
    sh.close()
