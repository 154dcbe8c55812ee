"""GPU parity of the non-square forward (ss_extend_tree; "Non-square mask
support") against the oracle's forward_nonsquare.

A tree is grown in pieces: the first piece is a square verify (no commit), each
later piece computes only its new nodes against the prefix, the cached tree
rows of the earlier pieces (their ancestors by the non-square mask) and their
own new ancestors.  Criteria as in test_gpu_parity.py: logits within R13,
argmax identical except at oracle near-ties (R14), tree metadata, accept walk
and compaction bit-exact."""
import numpy as np
import pytest

import oracle as O
import synth
from test_gpu_parity import build, check_logits, near_tie, oracle_setup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    cfg = synth.CONFIGS["tiny"]
    sh = build(cfg, L=64)
    m, kv = oracle_setup(cfg, L=64)
    yield cfg, sh, m, kv
    sh.close()


def _grow(sh, cfg, m, kv, toks, parents, bounds):
    """Grow on the GPU and in the oracle with the same pieces; compare each piece."""
    tree, rg = None, None
    for a, b in zip(bounds[:-1], bounds[1:]):
        if a == 0:
            rg = sh.verify(toks[a:b], parents[a:b], want_logits=True)
        else:
            rg = sh.extend(toks[a:b], parents[a:b], a, want_logits=True)
        tree = O.forward_nonsquare(cfg, m, kv, tree, toks[a:b], parents[a:b])
        assert rg["status"] == 0
        check_logits(rg["logits"], tree["logits"])
        for i in range(b - a):
            if rg["argmax"][a + i] != tree["argmax"][a + i]:
                assert near_tie(tree["logits"][i], rg["argmax"][a + i], tree["argmax"][a + i])
    return rg, tree


@pytest.mark.parametrize("bounds", [(0, 5, 12), (0, 3, 7, 16), (0, 1, 2, 4, 9, 24), (0, 8, 40)])
def test_tiny_extend_parity(tiny, bounds):
    cfg, sh, m, kv = tiny
    T = bounds[-1]
    toks, parents = synth.tree_random(T, cfg.vocab, np.random.default_rng(300 + T))
    toks, parents = list(toks), list(parents)
    sh.set_committed_len(64)
    rg, tree = _grow(sh, cfg, m, kv, toks, parents, bounds)
    # tree metadata of the grown tree, bit for bit (a0 over cached + new nodes)
    n, pos, anc, tk, par = sh.read_tree_meta()
    depth, opos, oanc = O.tree_meta(parents, 64)
    assert n == T
    assert list(pos) == list(opos) and list(tk) == toks and list(par) == parents
    for i in range(T):
        assert int(anc[i]) == sum(1 << j for j in np.nonzero(oanc[i])[0])
    # accept walk over the whole grown tree = the oracle walk on the GPU argmax
    acc, bonus = O.accept_walk(toks, parents, rg["argmax"])
    assert rg["accepted"] == acc and rg["bonus"] == bonus
    # K/V rows of every node (cached pieces and the last one) at L + node
    for l in range(cfg.n_layers):
        k, v = sh.read_kv(l, 64, T)
        np.testing.assert_allclose(k, tree["tree_k"][l], atol=2e-2, rtol=1e-2)
        np.testing.assert_allclose(v, tree["tree_v"][l], atol=2e-2, rtol=1e-2)
    sh.set_committed_len(64)


def test_tiny_extend_matches_square_verify(tiny):
    """GPU vs GPU: the grown tree's logits equal the square verify of the whole
    tree to the logit tolerance; the argmax at every node agrees except at
    near-ties (cached rows enter the extension as fp16, R18)."""
    cfg, sh, m, kv = tiny
    toks, parents = synth.tree_paperlike(20, cfg.vocab, np.random.default_rng(77))
    toks, parents = list(toks), list(parents)
    sh.set_committed_len(64)
    full = sh.verify(toks, parents, want_logits=True)
    sh.set_committed_len(64)
    a = sh.verify(toks[:9], parents[:9], want_logits=True)
    b = sh.extend(toks[9:], parents[9:], 9, want_logits=True)
    grown = np.concatenate([a["logits"], b["logits"]], axis=0)
    check_logits(grown, full["logits"])
    ro = O.verify(cfg, m, kv, toks, parents)
    for i in range(20):
        if b["argmax"][i] != full["argmax"][i]:
            assert near_tie(ro["logits"][i], b["argmax"][i], full["argmax"][i])
    sh.set_committed_len(64)


def test_tiny_extend_then_commit_chain(tiny):
    """A root-anchored chain through cached and new nodes commits bit-exactly
    (rows L + node -> L + k), and the next verify sees the committed rows."""
    cfg, sh, m, kv = tiny
    toks, parents = synth.tree_chain(10, cfg.vocab, np.random.default_rng(5))
    toks, parents = list(toks), list(parents)
    sh.set_committed_len(64)
    sh.verify(toks[:4], parents[:4])
    sh.extend(toks[4:], parents[4:], 4)
    before = [sh.read_kv(l, 64, 10) for l in range(cfg.n_layers)]
    chain = list(range(10))
    sh.commit_kv(chain)
    assert sh.L == 74
    for l in range(cfg.n_layers):
        k, v = sh.read_kv(l, 64, 10)
        assert np.array_equal(k, before[l][0]) and np.array_equal(v, before[l][1])
    # the committed chain = forced decoding of the chain (oracle)
    kvs = kv.copy()
    seq = O.forced_decode(cfg, m, kvs, toks)
    r = sh.verify([int(np.argmax(seq[-1]))], [-1], want_logits=True)
    ro = O.verify(cfg, m, kvs, [int(np.argmax(seq[-1]))], [-1])
    check_logits(r["logits"], ro["logits"])
    sh.set_committed_len(64)


def test_tiny_extend_one_leaf_per_call_is_sequential_decode(tiny):
    """Chain grown one leaf per call (w = 1, T0 = 0..7): leaf i's logits are
    forced single-token decoding of the chain prefix."""
    cfg, sh, m, kv = tiny
    chain = [11, 250, 3, 4000, 17, 9, 1000, 5]
    seq = O.forced_decode(cfg, m, kv.copy(), chain)
    sh.set_committed_len(64)
    for i, t in enumerate(chain):
        r = sh.verify([t], [-1], want_logits=True) if i == 0 else sh.extend([t], [i - 1], i, want_logits=True)
        check_logits(r["logits"], seq[i:i + 1])
    sh.set_committed_len(64)


def test_tiny_extend_truncates_pending_tree(tiny):
    """T0 below the pending size discards nodes >= T0 (their rows are rewritten)."""
    cfg, sh, m, kv = tiny
    toks, parents = synth.tree_random(12, cfg.vocab, np.random.default_rng(9))
    toks, parents = list(toks), list(parents)
    sh.set_committed_len(64)
    sh.verify(toks[:8], parents[:8])
    r = sh.extend(toks[5:], parents[5:], 5, want_logits=True)
    tree = O.forward_nonsquare(cfg, m, kv, None, toks[:5], parents[:5])
    tree = O.forward_nonsquare(cfg, m, kv, tree, toks[5:], parents[5:])
    check_logits(r["logits"], tree["logits"])
    sh.set_committed_len(64)


def test_extend_errors(tiny):
    import paper_2506_11309_b200 as pkg
    cfg, sh, m, kv = tiny
    sh.set_committed_len(64)
    with pytest.raises(pkg.SwiftSpecError) as e:
        sh.extend([1], [0], 1)                      # nothing pending
    assert e.value.status == "SS_ESTATE"
    sh.verify([1, 2, 3], [-1, 0, 1])
    with pytest.raises(pkg.SwiftSpecError) as e:
        sh.extend([1], [0], 4)                      # T0 beyond the pending tree
    assert e.value.status == "SS_ESTATE"
    with pytest.raises(pkg.SwiftSpecError) as e:
        sh.extend([1], [3], 3)                      # parent not earlier than the node
    assert e.value.status == "SS_EINVAL"
    with pytest.raises(pkg.SwiftSpecError) as e:
        sh.extend([1] * 33, [0] * 33, 3)            # w > 32
    assert e.value.status == "SS_EINVAL"
    with pytest.raises(pkg.SwiftSpecError) as e:
        sh.extend([1], [-1], 0)                     # T0 = 0 while a tree is pending
    assert e.value.status == "SS_ESTATE"
    r = sh.extend([7, 8], [2, 3], 3)                # still usable after the refusals
    assert r["status"] == 0 and len(r["argmax"]) == 5
    sh.set_committed_len(64)


def test_1b_extend_parity():
    """Llama3-1B shape (GQA 4:1, d = 64, L = 1K): a 16-node paper-like tree grown
    as 8 + 8 (the draft's w = 8)."""
    cfg = synth.CONFIGS["llama3-1b"]
    L = 1024
    sh = build(cfg, L=L, max_ctx=L + 64)
    try:
        m, kv = oracle_setup(cfg, L=L, max_ctx=L + 64)
        m.cache_dense = False
        toks, parents = synth.tree_paperlike(16, cfg.vocab, np.random.default_rng(16))
        _grow(sh, cfg, m, kv, list(toks), list(parents), (0, 8, 16))
    finally:
        sh.close()
