"""GPU parity: the CUDA path through the C-ABI vs the float64 oracle.

Criteria (BASELINE north_star):
  * tree masks, accept indices and KV compaction bit-exact,
  * logits |gpu - oracle| <= 2e-2 + 1e-2 |oracle| elementwise (R13),
  * accepted sequences identical except where the oracle's top-2 logit gap
    at a node is below 2e-2 (R14).
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu

ATOL, RTOL, TIE = 2e-2, 1e-2, 2e-2


def _pkg():
    import paper_2506_11309_b200 as pkg
    return pkg


def build(cfg, seed=0, L=64, max_ctx=None, max_tree=64, device_synth=False, tp=(0, 1)):
    pkg = _pkg()
    max_ctx = max_ctx or (L + 256)
    sh = pkg.Shard(cfg, tp[0], tp[1], 0, max_ctx=max_ctx, max_tree=max_tree)
    if device_synth:
        sh.synth_weights(seed)
        sh.synth_prefix_kv(seed + 1, L)
    else:
        sh.load_canonical(synth.gen_model(cfg, seed))
        for l in range(cfg.n_layers):
            k, v = synth.gen_prefix_kv(seed + 1, l, L, cfg.n_kv_heads, cfg.head_dim)
            sh.set_prefix_kv(l, k, v)
    return sh


def oracle_setup(cfg, seed=0, L=64, max_ctx=None):
    m = O.OracleModel(cfg, synth.gen_model(cfg, seed))
    kv = O.KVCache(cfg, max_ctx or (L + 256))
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(seed + 1, l, L, cfg.n_kv_heads, cfg.head_dim)
        kv.set_prefix(l, k, v)
    kv.L = L
    return m, kv


def near_tie(logits_row, tok_a, tok_b):
    return abs(logits_row[tok_a] - logits_row[tok_b]) < TIE


def check_logits(g, o):
    err = np.abs(g - o)
    bound = ATOL + RTOL * np.abs(o)
    assert np.all(err <= bound), f"max abs err {err.max():.3g}, worst ratio {(err / bound).max():.3g}"


def check_accept(res_g, res_o, tokens, parents, logits_o):
    """Identical path unless a near-tie at some node on the way explains the divergence."""
    ag, ao = list(res_g["argmax"]), list(res_o["argmax"])
    for i in range(len(tokens)):
        if ag[i] != ao[i]:
            assert near_tie(logits_o[i], ag[i], ao[i]), (i, ag[i], ao[i])
    if ag == ao:
        assert res_g["accepted"] == res_o["accepted"]
        assert res_g["bonus"] == res_o["bonus"]
        assert res_g["n_accepted"] == len(res_o["accepted"])
    # the GPU's own walk must be the oracle walk applied to the GPU's argmax (bit-exact logic)
    acc, bonus = O.accept_walk(tokens, parents, ag)
    assert res_g["accepted"] == acc and res_g["bonus"] == bonus


TREES = ["chain", "star", "paperlike", "random"]


def make_tree(kind, T, V, rng):
    return dict(chain=synth.tree_chain, star=synth.tree_star, paperlike=synth.tree_paperlike,
                random=synth.tree_random)[kind](T, V, rng)


@pytest.fixture(scope="module")
def tiny():
    cfg = synth.CONFIGS["tiny"]
    sh = build(cfg, L=64)
    m, kv = oracle_setup(cfg, L=64)
    yield cfg, sh, m, kv
    sh.close()


@pytest.mark.parametrize("kind", TREES)
@pytest.mark.parametrize("T", [1, 5, 8, 13, 16, 32, 64])
def test_tiny_verify_parity(tiny, kind, T):
    cfg, sh, m, kv = tiny
    rng = np.random.default_rng(100 + T)
    tokens, parents = make_tree(kind, T, cfg.vocab, rng)
    sh.set_committed_len(64)
    rg = sh.verify(tokens, parents, want_logits=True)
    ro = O.verify(cfg, m, kv, tokens, parents)
    assert rg["status"] == 0
    check_logits(rg["logits"], ro["logits"])
    check_accept(rg, ro, tokens, parents, ro["logits"])
    # tree K/V rows (post-RoPE) written at L + i, compared per layer
    for l in range(cfg.n_layers):
        k, v = sh.read_kv(l, 64, T)
        np.testing.assert_allclose(k, ro["tree_k"][l], atol=2e-2, rtol=1e-2)
        np.testing.assert_allclose(v, ro["tree_v"][l], atol=2e-2, rtol=1e-2)


def test_tiny_commit_is_bit_exact_copy(tiny):
    cfg, sh, m, kv = tiny
    rng = np.random.default_rng(7)
    tokens, parents = synth.tree_paperlike(16, cfg.vocab, rng)
    sh.set_committed_len(64)
    sh.verify(tokens, parents)
    # commit a deep root-anchored chain (not just the accepted one, BJ / 8(b))
    chain = [int(np.argmax([O.tree_meta(parents, 0)[0][i] for i in range(16)]))]
    while parents[chain[-1]] != -1:
        chain.append(int(parents[chain[-1]]))
    chain = chain[::-1]
    before = [sh.read_kv(l, 64, 16) for l in range(cfg.n_layers)]
    sh.commit_kv(chain)
    assert sh.L == 64 + len(chain)
    for l in range(cfg.n_layers):
        k, v = sh.read_kv(l, 64, len(chain))
        assert np.array_equal(k, before[l][0][chain]) and np.array_equal(v, before[l][1][chain])
        # committed prefix untouched
        k0, _ = sh.read_kv(l, 0, 64)
        kp, _ = synth.gen_prefix_kv(1, l, 64, cfg.n_kv_heads, cfg.head_dim)
        assert np.array_equal(k0, synth.bf16_bits_to_f32(kp))


def test_tiny_commit_errors(tiny):
    cfg, sh, m, kv = tiny
    pkg = _pkg()
    sh.set_committed_len(64)
    with pytest.raises(pkg.SwiftSpecError, match="SS_ESTATE"):
        sh.commit_kv([0])
    tokens, parents = synth.tree_star(4, cfg.vocab, np.random.default_rng(0))
    sh.verify(tokens, parents)
    with pytest.raises(pkg.SwiftSpecError, match="SS_EINVAL"):
        sh.commit_kv([0, 1, 2])   # 2 is not a child of 1 in a star
    with pytest.raises(pkg.SwiftSpecError, match="SS_EINVAL"):
        sh.commit_kv([1])
    with pytest.raises(pkg.SwiftSpecError, match="SS_EINVAL"):
        sh.verify([1, 2], [0, 0])
    with pytest.raises(pkg.SwiftSpecError, match="SS_EINVAL"):
        sh.verify([1, cfg.vocab], [-1, 0])
    # capacity: L + T > max_ctx is refused before any launch.  The
    # committed length may only grow over rows actually written: write a longer
    # prefix first (counter-indexed generator: its first 64 rows are unchanged)
    with pytest.raises(pkg.SwiftSpecError, match="SS_EINVAL"):
        sh.set_committed_len(sh.max_ctx - 64)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(1, l, sh.max_ctx - 64, cfg.n_kv_heads, cfg.head_dim)
        sh.set_prefix_kv(l, k, v)
    sh.set_committed_len(sh.max_ctx - 64)
    toks, pars = synth.tree_chain(8, cfg.vocab, np.random.default_rng(1))
    sh.verify(toks, pars)
    sh.commit_kv(list(range(8)))
    assert sh.L == sh.max_ctx - 56
    with pytest.raises(pkg.SwiftSpecError, match="SS_ECAPACITY"):
        sh.verify(*synth.tree_chain(64, cfg.vocab, np.random.default_rng(1)))
    assert sh.L == sh.max_ctx - 56
    sh.set_committed_len(64)


def test_tiny_greedy_decode_and_planted_trees(tiny):
    """Golden equivalence: verify + commit of planted trees reproduces
    plain greedy decoding; every step's accept length equals the planted depth
    + 1 unless a near-tie intervened."""
    cfg, sh, m, kv0 = tiny
    sh.set_committed_len(64)
    root = 123
    ref = O.greedy_decode(cfg, m, kv0.copy(), root, 10)
    out, cur = [], root
    kv = kv0.copy()
    while len(out) < 10:
        nxt = ref[len(out):len(out) + 3]
        toks = [cur] + nxt + [int(t) for t in np.random.default_rng(len(out)).integers(0, cfg.vocab, 3)]
        parents = list(range(-1, len(nxt))) + [0, 0, 1][: len(toks) - 1 - len(nxt)]
        toks = toks[:len(parents)]
        rg = sh.verify(toks, parents, want_logits=True)
        ro = O.verify(cfg, m, kv, toks, parents)
        check_accept(rg, ro, toks, parents, ro["logits"])
        if rg["accepted"] != ro["accepted"]:
            pytest.skip("near-tie changed the path; golden comparison not defined past it")
        sh.commit_kv(rg["accepted"])
        O.commit(kv, ro, ro["accepted"])
        out += [toks[i] for i in rg["accepted"][1:]] + [rg["bonus"]]
        cur = rg["bonus"]
    assert out[:10] == ref
    assert sh.L == kv.L


def test_device_synth_matches_host_load():
    """The device generator reproduces synth/generators.py: same logits (the
    packed bytes are compared exactly in test_gpu_exact.py)."""
    cfg = synth.CONFIGS["tiny"]
    a = build(cfg, seed=5, L=64)
    b = build(cfg, seed=5, L=64, device_synth=True)
    m, kv = oracle_setup(cfg, seed=5, L=64)
    rng = np.random.default_rng(3)
    tokens, parents = synth.tree_paperlike(8, cfg.vocab, rng)
    ra = a.verify(tokens, parents, want_logits=True)
    rb = b.verify(tokens, parents, want_logits=True)
    ro = O.verify(cfg, m, kv, tokens, parents)
    # identical weights; only the order of the split-K fp32 reductions differs
    np.testing.assert_allclose(ra["logits"], rb["logits"], atol=3e-3, rtol=1e-3)
    for r in (ra, rb):
        check_logits(r["logits"], ro["logits"])
        check_accept(r, ro, tokens, parents, ro["logits"])
    # the two GPU runs may differ only at an oracle near-tie (R14)
    for i, (x, y) in enumerate(zip(ra["argmax"], rb["argmax"])):
        assert x == y or near_tie(ro["logits"][i], x, y), (i, x, y)
    for l in range(cfg.n_layers):
        assert np.array_equal(a.read_kv(l, 0, 64)[0], b.read_kv(l, 0, 64)[0])
        assert np.array_equal(a.read_kv(l, 0, 64)[1], b.read_kv(l, 0, 64)[1])
    a.close()
    b.close()


def test_verify_dev_autocommit():
    import torch
    cfg = synth.CONFIGS["tiny"]
    sh = build(cfg, L=64)
    m, kv = oracle_setup(cfg, L=64)
    rng = np.random.default_rng(9)
    tokens, parents = synth.tree_paperlike(8, cfg.vocab, rng)
    ro = O.verify(cfg, m, kv, tokens, parents)
    from paper_2506_11309_b200 import swiftspec as ssp
    dt = torch.tensor(tokens, dtype=torch.int32, device="cuda")
    dp = torch.tensor(parents, dtype=torch.int32, device="cuda")
    dres = torch.zeros(ssp.result_nbytes() // 4, dtype=torch.int32, device="cuda")
    sh.verify_dev(dt, dp, 8, d_result=dres, auto_commit=True, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    rg = ssp.parse_result(dres.cpu().numpy(), 8)
    check_accept(rg, ro, tokens, parents, ro["logits"])
    assert sh.L == 64 + rg["n_accepted"]
    sh.close()


@pytest.mark.parametrize("T", [8, 16])
def test_1b_parity(T):
    """Llama3-1B shape (BASELINE configs[1]), 1K KV, TP 1."""
    cfg = synth.CONFIGS["llama3-1b"]
    L = 1024
    m, kv = oracle_setup(cfg, L=L, max_ctx=L + 64)
    m.cache_dense = False
    sh = build(cfg, L=L, max_ctx=L + 64)
    rng = np.random.default_rng(T)
    tokens, parents = synth.tree_paperlike(T, cfg.vocab, rng)
    rg = sh.verify(tokens, parents, want_logits=True)
    ro = O.verify(cfg, m, kv, tokens, parents)
    check_logits(rg["logits"], ro["logits"])
    check_accept(rg, ro, tokens, parents, ro["logits"])
    sh.close()


class _EmbedRows:
    """Embedding rows generated on demand (the oracle only reads the tree tokens' rows)."""

    def __init__(self, seed, V, h):
        self.seed, self.V, self.h = seed, V, h

    def __getitem__(self, rows):
        return synth.gen_embed(self.seed, self.V, self.h, rows=np.atleast_1d(rows))


@pytest.mark.parametrize("T", [8, 32])
def test_70b_shaped_layer_sampled_parity(T):
    """BASELINE metric shapes at full size: one Llama3-70B-shaped decoder layer (h 8192,
    I 28672, 64/8 heads), the full 128256-row LM head, a 4096-token KV prefix and an
    8- or 32-node paper-like tree, TP 1, through the same graph launch path bench.py times.
    The oracle (oracle/) runs the layer in float64 and computes logits one by one for a
    seeded sample of vocab rows plus every row the GPU picked as argmax; the GPU's full
    logits are compared on that sample, and each GPU argmax must be the oracle's best
    among the sampled rows (up to the near-tie rule, R14)."""
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["llama3-70b"], n_layers=1)
    L = 4096
    sh = build(cfg, L=L, max_ctx=L + 64, max_tree=T, device_synth=True)
    rng = np.random.default_rng(70 + T)
    tokens, parents = synth.tree_paperlike(T, cfg.vocab, rng)
    rg = sh.verify(tokens, parents, want_logits=True)
    sh.close()
    assert rg["status"] == 0
    # oracle: the same layer from the host generator (bit-identical to the device one)
    canon = {"layers": [synth.gen_model(dataclasses.replace(cfg, vocab=8), 0, with_lm_head=False)["layers"][0]],
             "embed": _EmbedRows(0, cfg.vocab, cfg.hidden),
             "final_norm": synth.gen_norm(0, -1, synth.KIND["FINAL_NORM"], cfg.hidden)}
    m = O.OracleModel(cfg, canon, cache_dense=False)
    kv = O.KVCache(cfg, L + 64)
    k, v = synth.gen_prefix_kv(1, 0, L, cfg.n_kv_heads, cfg.head_dim)
    kv.set_prefix(0, k, v)
    kv.L = L
    depth, pos, anc = O.tree_meta(parents, L)
    x = m.embed_rows(tokens)
    x, _, _ = O.layer_forward(cfg, m, 0, x, kv, L, pos, anc)
    xn = O.rmsnorm(x, canon["final_norm"], cfg.rms_eps)
    sample = np.unique(np.concatenate([rng.choice(cfg.vocab, 4096, replace=False), rg["argmax"][:T]]))
    W = O.bf16_to_f64(synth.gen_lm_head(0, cfg.vocab, cfg.hidden, rows=sample))
    lo = xn @ W.T                                  # oracle logits [T][sample]
    lg = rg["logits"][:, sample]
    check_logits(lg, lo)
    for i in range(T):
        best = sample[np.argmax(lo[i])]
        g = int(rg["argmax"][i])
        gi = int(np.searchsorted(sample, g))
        assert best == g or lo[i].max() - lo[i][gi] < TIE, (i, g, best)


def _adversarial_model(cfg, seed=0):
    """Zero points at the extremes in 40% of the groups (z in {0, 15}: |q - z| up
    to 15 with a biased mean), 1/8 of the AWQ scales x8, MLP-norm gains of 8 on four
    channels, 1% of the embedding entries x64 (activation outliers).  The
    residual stream reaches ~2e3 (inside the fp16 range of the GEMM inputs,
    DESIGN R18) and the 1024+q offset accumulation sees its largest terms."""
    m = synth.gen_model(cfg, seed)
    rng = np.random.default_rng(9)
    for lw in m["layers"]:
        for n in ("wq", "wk", "wv", "wo", "wgate", "wup", "wdown"):
            q, z, s = lw[n]
            u = rng.random(z.shape)
            z2 = np.where(u < 0.2, 0, np.where(u < 0.4, 15, z)).astype(np.uint8)
            sf = synth.bf16_bits_to_f32(s).copy()
            sf[rng.random(s.shape) < 0.125] *= 8.0
            lw[n] = (q, z2, synth.f32_to_bf16_bits(sf))
        g = synth.bf16_bits_to_f32(lw["mlp_norm"]).copy()
        g[rng.choice(cfg.hidden, 4, replace=False)] = 8.0
        lw["mlp_norm"] = synth.f32_to_bf16_bits(g)
    e = synth.bf16_bits_to_f32(m["embed"]).copy()
    e[rng.random(e.shape) < 0.01] *= 64.0
    m["embed"] = synth.f32_to_bf16_bits(e)
    return m


@pytest.mark.parametrize("T", [8, 16, 32])
def test_adversarial_weights_and_outliers(T):
    cfg = synth.CONFIGS["tiny"]
    canon = _adversarial_model(cfg)
    pkg = _pkg()
    sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=64 + 256, max_tree=64)
    sh.load_canonical(canon)
    m = O.OracleModel(cfg, canon)
    kv = O.KVCache(cfg, 64 + 256)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(1, l, 64, cfg.n_kv_heads, cfg.head_dim)
        sh.set_prefix_kv(l, k, v)
        kv.set_prefix(l, k, v)
    kv.L = 64
    tokens, parents = synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(T))
    rg = sh.verify(tokens, parents, want_logits=True)
    ro = O.verify(cfg, m, kv, tokens, parents)
    assert np.all(np.isfinite(rg["logits"]))
    check_logits(rg["logits"], ro["logits"])
    check_accept(rg, ro, tokens, parents, ro["logits"])
    for l in range(cfg.n_layers):
        k, v = sh.read_kv(l, 64, T)
        np.testing.assert_allclose(k, ro["tree_k"][l], atol=2e-2, rtol=1e-2)
        np.testing.assert_allclose(v, ro["tree_v"][l], atol=2e-2, rtol=1e-2)
    sh.close()
