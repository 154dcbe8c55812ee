"""GPU tests of the draft side: the top-K expansion
output, the re-root KV reorganisation, and the whole
Alg. 1 loop -- whose emitted tokens must be the target's greedy
continuation whatever the draft proposes."""
import numpy as np
import pytest

import oracle as O
import synth
from test_gpu_parity import TIE, build, check_logits, oracle_setup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    cfg = synth.CONFIGS["tiny"]
    sh = build(cfg, L=64)
    m, kv = oracle_setup(cfg, L=64)
    yield cfg, sh, m, kv
    sh.close()


def _logsumexp(x):
    mx = np.max(x)
    return mx + np.log(np.sum(np.exp(x - mx)))


def test_topk_and_lse_vs_oracle(tiny):
    """Top-K tokens of each new node (ties -> lower id) and the log-sum-exp of
    its logits: tokens identical where the oracle's ranking is not a near-tie,
    logits and lse within the logit tolerance (R13)."""
    cfg, sh, m, kv = tiny
    K = 8
    toks, parents = synth.tree_paperlike(12, cfg.vocab, np.random.default_rng(41))
    toks, parents = list(toks), list(parents)
    sh.set_committed_len(64)
    sh.verify(toks[:5], parents[:5])
    tok, val, lse = sh.extend_topk(toks[5:], parents[5:], 5, K)
    tree = O.forward_nonsquare(cfg, m, kv, None, toks[:5], parents[:5])
    tree = O.forward_nonsquare(cfg, m, kv, tree, toks[5:], parents[5:])
    for i in range(7):
        row = tree["logits"][i]
        order = sorted(range(cfg.vocab), key=lambda t: (-row[t], t))
        for k in range(K):
            gap_prev = row[order[k - 1]] - row[order[k]] if k > 0 else np.inf
            gap_next = row[order[k]] - row[order[k + 1]]
            if min(gap_prev, gap_next) >= TIE:
                assert tok[i, k] == order[k], (i, k)
        assert list(val[i]) == sorted(val[i], reverse=True)
        check_logits(val[i], row[tok[i]])
        assert abs(lse[i] - _logsumexp(row)) <= 2e-2 + 1e-2 * abs(_logsumexp(row))
    sh.set_committed_len(64)


def test_reroot_rows_and_meta_bit_exact(tiny):
    """ss_reroot: path rows move to L + k, kept rows to L + n + j (bit copies),
    the kept nodes become the pending tree (positions unchanged, masks and
    parents re-indexed), L advances by n; a following extension equals the
    oracle's non-square forward on the committed cache and the kept subtree."""
    cfg, sh, m, kv = tiny
    # 0 -> 1 -> {2, 3}; 2 -> {4, 6}; 3 -> 5; 4 -> 7
    toks = [9, 17, 33, 41, 55, 61, 77, 83]
    parents = [-1, 0, 1, 1, 2, 3, 2, 4]
    sh.set_committed_len(64)
    sh.verify(toks, parents)
    before = [sh.read_kv(l, 64, 8) for l in range(cfg.n_layers)]
    path, keep = [0, 1], [2, 4, 6, 7]      # verified 0, 1; the new root 2 and its subtree
    sh.reroot(path, keep)
    assert sh.L == 66
    for l in range(cfg.n_layers):
        k, v = sh.read_kv(l, 64, 6)
        src = path + keep
        assert np.array_equal(k, before[l][0][src]) and np.array_equal(v, before[l][1][src])
    n, pos, anc, tk, par = sh.read_tree_meta()
    assert n == 4 and list(tk) == [33, 55, 77, 83] and list(par) == [-1, 0, 0, 1]
    assert list(pos) == [66, 67, 67, 68]
    assert [int(a) for a in anc] == [0b1, 0b11, 0b101, 0b1011]
    # grow the kept tree and compare with the oracle
    full = O.verify(cfg, m, kv, toks, parents)
    kv2 = O.commit(kv.copy(), full, path)
    kept = dict(tokens=np.array([33, 55, 77, 83]), parents=np.array([-1, 0, 0, 1]),
                tree_k=[full["tree_k"][l][keep] for l in range(cfg.n_layers)],
                tree_v=[full["tree_v"][l][keep] for l in range(cfg.n_layers)],
                argmax=np.array(full["argmax"])[keep])
    new_t, new_p = [100, 200, 300], [1, 3, 4]
    r = sh.extend(new_t, new_p, 4, want_logits=True)
    ro = O.forward_nonsquare(cfg, m, kv2, kept, new_t, new_p)
    check_logits(r["logits"], ro["logits"])
    sh.set_committed_len(64)


def test_reroot_errors(tiny):
    import paper_2506_11309_b200 as pkg
    cfg, sh, m, kv = tiny
    sh.set_committed_len(64)
    with pytest.raises(pkg.SwiftSpecError) as e:
        sh.reroot([0], [])                       # nothing pending
    assert e.value.status == "SS_ESTATE"
    sh.verify([9, 17, 33, 41], [-1, 0, 1, 1])
    for path, keep in [([0, 2], []), ([0], [2]), ([0, 1], [3, 2]), ([0, 1], [1]), ([], [1])]:
        with pytest.raises(pkg.SwiftSpecError) as e:
            sh.reroot(path, keep)
        assert e.value.status == "SS_EINVAL", (path, keep)
    sh.reroot([], [0, 1, 3])                     # n = 0: drop node 2 only
    assert sh.L == 64
    sh.set_committed_len(64)


def _pair(draft_seed):
    cfg = synth.CONFIGS["tiny"]
    L = 64
    t = build(cfg, seed=0, L=L, max_ctx=L + 320, max_tree=8)
    dr = build(cfg, seed=draft_seed, L=L, max_ctx=L + 320, max_tree=64)
    m, kv = oracle_setup(cfg, seed=0, L=L, max_ctx=L + 320)
    return cfg, t, dr, m, kv


def _check_greedy(cfg, m, kv, root, out):
    """out must be the oracle's greedy continuation of root, up to a near-tie."""
    kvs = kv.copy()
    cur = root
    for i, tok in enumerate(out):
        r = O.verify(cfg, m, kvs, [cur], [-1])
        if tok != int(r["argmax"][0]):
            row = r["logits"][0]
            assert abs(row[tok] - row[int(r["argmax"][0])]) < TIE, (i, tok, int(r["argmax"][0]))
            return i
        O.commit(kvs, r, [0])
        cur = tok
    return len(out)


@pytest.mark.parametrize("mode", ["async", "serial"])
@pytest.mark.parametrize("draft_seed", [0, 7])
def test_speculative_decode_is_target_greedy(mode, draft_seed):
    """Alg. 1 with a draft identical to the target (seed 0: every proposal on the
    greedy path is accepted) and an unrelated draft (seed 7): the emitted
    tokens are the target's greedy continuation either way."""
    import torch
    cfg, t, dr, m, kv = _pair(draft_seed)
    try:
        if mode == "async":
            t.set_launch_cap(96)
            dr.set_launch_cap(44)
        ts, ds = torch.cuda.Stream(), torch.cuda.Stream()
        root, n = 321, 40
        out, st = t.speculative_decode(dr, root, n, bs=8, w=8, d=2, mode=mode, target_stream=ts, draft_stream=ds)
        assert len(out) == n and st["n_emitted"] == n
        assert st["accepted"] + st["steps"] >= n
        assert _check_greedy(cfg, m, kv, root, out) >= min(n, 20)
        if draft_seed == 0:
            # the identical draft's top-1 child of the root is always in the subgraph
            # (the most probable non-root node) and always the target's greedy token
            assert n / st["steps"] >= 1.9, st
        assert t.L >= 64 + n - 8
    finally:
        t.close()
        dr.close()


def test_speculative_decode_argument_errors():
    import paper_2506_11309_b200 as pkg
    cfg, t, dr, m, kv = _pair(7)
    try:
        with pytest.raises(pkg.SwiftSpecError):
            t.speculative_decode(dr, 321, 10, mode="async")          # no launch caps / same stream
        with pytest.raises(pkg.SwiftSpecError):
            t.speculative_decode(dr, 321, 10, bs=9, mode="serial")   # bs > the target's max_tree
    finally:
        t.close()
        dr.close()
