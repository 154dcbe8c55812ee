"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names the passage / reading it pins.  A plausible mistake in the
oracle (a dropped term, a wrong sign or index, a transposed operand, a wrong
mask direction, a wrong RoPE pairing, a wrong group index) fails at least one
of these.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- a0 tree meta
def test_tree_meta_chain_is_causal():
    # S:101 "chain of 3 nodes ... lower-triangular ones"
    _, pos, anc = O.tree_meta([-1, 0, 1, 2, 3], L=7)
    assert np.array_equal(anc, np.tril(np.ones((5, 5), dtype=bool)))
    assert list(pos) == [7, 8, 9, 10, 11]


def test_tree_meta_star():
    # S:102 "root with two children -> rows for children each see root + self only"
    d, _, anc = O.tree_meta([-1, 0, 0, 0], L=0)
    exp = np.zeros((4, 4), dtype=bool)
    exp[:, 0] = True
    exp[np.arange(4), np.arange(4)] = True
    assert np.array_equal(anc, exp)
    assert list(d) == [0, 1, 1, 1]


def test_tree_meta_fig4():
    g = _load("fig4_accept.json")
    _, _, anc = O.tree_meta(g["parents"], L=0)
    assert list(anc[3]) == g["expected_anc_row_t5"]


def test_tree_meta_vs_transitive_closure():
    # independent algorithm: reflexive-transitive closure of the parent relation
    rng = np.random.default_rng(5)
    for T in (1, 2, 7, 16, 33, 64):
        _, parents = synth.tree_random(T, 100, rng)
        depth, _, anc = O.tree_meta(parents, 0)
        A = np.zeros((T, T), dtype=np.int64)
        for i in range(1, T):
            A[i, parents[i]] = 1
        R = np.eye(T, dtype=np.int64)
        P = np.eye(T, dtype=np.int64)
        for _ in range(T):
            P = np.minimum(P @ A, 1)
            R = np.minimum(R + P, 1)
        assert np.array_equal(anc, R.astype(bool))
        assert np.array_equal(depth, anc.sum(1) - 1)


@pytest.mark.parametrize("parents", [[0, 0], [-1, 1], [-1, 0, 3, 1], [], [-1, -1]])
def test_tree_meta_rejects_invalid(parents):
    with pytest.raises(ValueError):
        O.tree_meta(parents, 0)


# ---------------------------------------------------------------- dequant
def test_dequant_golden():
    g = _load("dequant_small.json")
    K, N = g["K"], g["N"]
    q = np.array([[(k + n) % 16 for n in range(N)] for k in range(K)], dtype=np.uint8)
    z = np.array([[gg + 2 * n + 1 for n in range(N)] for gg in range(K // 128)], dtype=np.uint8)
    s = np.array(g["scales_bf16_bits"], dtype=np.uint16)
    assert np.array_equal(O.bf16_to_f64(s), np.array(g["scales"]))
    W = O.dequant(q, z, s)
    for k, n, v in g["expected_entries"]:
        assert W[k, n] == v, (k, n)
    assert np.array_equal(np.ones(K) @ W, np.array(g["ones_times_W"]))


def test_dequant_zero_when_q_equals_z():
    rng = np.random.default_rng(1)
    z = rng.integers(0, 16, (2, 3)).astype(np.uint8)
    q = np.repeat(z, 128, axis=0)
    s = synth.f32_to_bf16_bits(rng.uniform(0.1, 2, (2, 3)).astype(np.float32))
    assert np.all(O.dequant(q, z, s) == 0.0)


def test_dequant_matches_synth_weight_statistics():
    # recipe (DESIGN.md input recipe): std(W) ~ 1/sqrt(K)
    q, z, s = synth.gen_linear(0, 0, synth.KIND["WO"], 1024, 256)
    W = O.dequant(q, z, s)
    assert abs(W.std() * math.sqrt(1024) - 1.0) < 0.08


# ---------------------------------------------------------------- norm / act / rope
def test_rmsnorm_closed_form():
    g1 = synth.f32_to_bf16_bits(np.ones(8, dtype=np.float32))
    g2 = synth.f32_to_bf16_bits(np.full(8, 2.0, dtype=np.float32))
    x = np.full((1, 8), 2.0)
    # 2 / sqrt(4 + 1e-5) = 1 / sqrt(1 + 2.5e-6)
    np.testing.assert_allclose(O.rmsnorm(x, g1, 1e-5), 0.9999987500023437, rtol=0, atol=1e-15)
    np.testing.assert_allclose(O.rmsnorm(x, g2, 1e-5), 2 * 0.9999987500023437, rtol=0, atol=1e-15)
    # rows are independent and scale-invariant (eps -> 0)
    rng = np.random.default_rng(0)
    y = rng.normal(size=(3, 8))
    np.testing.assert_allclose(O.rmsnorm(5.0 * y, g1, 0.0), O.rmsnorm(y, g1, 0.0), rtol=1e-13)
    np.testing.assert_allclose(np.mean(O.rmsnorm(y, g1, 0.0) ** 2, axis=1), 1.0, rtol=1e-13)


def test_silu_values():
    assert O.silu(np.array(0.0)) == 0.0
    np.testing.assert_allclose(O.silu(np.array(1.0)), 0.7310585786300049, rtol=1e-15)
    np.testing.assert_allclose(O.silu(np.array(40.0)), 40.0, rtol=1e-15)
    assert abs(O.silu(np.array(-40.0))) < 1e-15


def test_rope_golden():
    for c in _load("rope_small.json")["cases"]:
        out = O.rope(np.array(c["v"]), c["pos"], c["theta"])
        np.testing.assert_allclose(out, c["expect"], atol=1e-12)


def test_rope_relative_and_isometric():
    rng = np.random.default_rng(3)
    q, k = rng.normal(size=64), rng.normal(size=64)
    a = O.rope(q, 1000, 5e5) @ O.rope(k, 990, 5e5)
    b = O.rope(q, 17, 5e5) @ O.rope(k, 7, 5e5)
    np.testing.assert_allclose(a, b, rtol=1e-9)
    np.testing.assert_allclose(np.linalg.norm(O.rope(q, 12345, 5e5)), np.linalg.norm(q), rtol=1e-13)


# ---------------------------------------------------------------- attention / argmax
def test_attend_single_key_returns_value():
    rng = np.random.default_rng(4)
    q = rng.normal(size=(4, 8))
    k = rng.normal(size=(1, 2, 8))
    v = rng.normal(size=(1, 2, 8))
    out = O.attend_node(q, k, v, 2)
    np.testing.assert_allclose(out[0], v[0, 0])
    np.testing.assert_allclose(out[3], v[0, 1])


def test_attend_equal_keys_is_mean_and_gqa_map():
    rng = np.random.default_rng(5)
    q = rng.normal(size=(4, 8))
    k = np.ones((5, 2, 8))
    v = rng.normal(size=(5, 2, 8))
    out = O.attend_node(q, k, v, 2)
    # heads 0,1 -> kv head 0; heads 2,3 -> kv head 1
    np.testing.assert_allclose(out[1], v[:, 0].mean(0), rtol=1e-13)
    np.testing.assert_allclose(out[2], v[:, 1].mean(0), rtol=1e-13)


def test_attend_two_keys_closed_form():
    # scores s0 = 0, s1 = ln 3 * sqrt(d)/sqrt(d) -> weights 1/4, 3/4
    d = 4
    q = np.zeros((1, d))
    q[0, 0] = math.log(3.0) * math.sqrt(d)
    k = np.zeros((2, 1, d))
    k[1, 0, 0] = 1.0
    v = np.zeros((2, 1, d))
    v[0, 0, 1] = 1.0
    v[1, 0, 2] = 1.0
    out = O.attend_node(q, k, v, 1)
    np.testing.assert_allclose(out[0], [0, 0.25, 0.75, 0], atol=1e-15)


def test_argmax_tie_lowest():
    # S:274-275
    assert O.argmax_lowest([0.1, 0.9, 0.9]) == 1
    assert O.argmax_lowest([0.5, 0.5, 0.5, 0.5]) == 0
    rng = np.random.default_rng(0)
    for _ in range(20):
        r = rng.integers(0, 5, 50).astype(float)
        assert O.argmax_lowest(r) == int(np.flatnonzero(r == r.max())[0])


# ---------------------------------------------------------------- a11 accept
def test_accept_fig4():
    g = _load("fig4_accept.json")
    acc, bonus = O.accept_walk(g["tokens"], g["parents"], g["argmax"])
    assert acc == g["expected_accepted"]
    assert bonus == g["expected_bonus"]
    path = [g["tokens"][i] for i in acc] + [bonus]
    assert path == g["expected_output_path"]


def test_accept_root_only_and_duplicates():
    # S:284 "subgraph = root only -> path = (root, argmax-next)"
    assert O.accept_walk([7], [-1], [42]) == ([0], 42)
    # duplicate sibling tokens: lowest index wins (reading R7)
    acc, bonus = O.accept_walk([1, 5, 5, 9], [-1, 0, 0, 2], [5, 9, 9, 0])
    assert acc == [0, 1] and bonus == 9


def test_accept_chain_all_accepted():
    # S:285 identical models -> the whole chain is accepted, |path| = bs + 1
    toks = [3, 4, 5, 6]
    acc, bonus = O.accept_walk(toks, [-1, 0, 1, 2], [4, 5, 6, 11])
    assert acc == [0, 1, 2, 3] and bonus == 11


# ---------------------------------------------------------------- model-level pins
def _tiny(seed=0, L=0, max_ctx=256):
    cfg = synth.CONFIGS["tiny"]
    m = O.OracleModel(cfg, synth.gen_model(cfg, seed))
    kv = O.KVCache(cfg, max_ctx)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(seed + 1, l, L, cfg.n_kv_heads, cfg.head_dim)
        kv.set_prefix(l, k, v)
    kv.L = L
    return cfg, m, kv


@pytest.fixture(scope="module")
def tiny16():
    return _tiny(L=16)


def _hf_llama(cfg, m):
    torch = pytest.importorskip("torch")
    tf = pytest.importorskip("transformers")
    hc = tf.LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.hidden,
                        intermediate_size=cfg.intermediate, num_hidden_layers=cfg.n_layers,
                        num_attention_heads=cfg.n_heads, num_key_value_heads=cfg.n_kv_heads,
                        head_dim=cfg.head_dim, rms_norm_eps=cfg.rms_eps, rope_theta=cfg.rope_theta,
                        tie_word_embeddings=False, attention_bias=False, mlp_bias=False,
                        max_position_embeddings=4096)
    hf = tf.LlamaForCausalLM(hc).double().eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    with torch.no_grad():
        hf.model.embed_tokens.weight.copy_(t(O.bf16_to_f64(m.canon["embed"])))
        hf.lm_head.weight.copy_(t(O.bf16_to_f64(m.canon["lm_head"])))
        hf.model.norm.weight.copy_(t(O.bf16_to_f64(m.canon["final_norm"])))
        for l, layer in enumerate(hf.model.layers):
            at, mlp = layer.self_attn, layer.mlp
            at.q_proj.weight.copy_(t(m.w(l, "wq").T))
            at.k_proj.weight.copy_(t(m.w(l, "wk").T))
            at.v_proj.weight.copy_(t(m.w(l, "wv").T))
            at.o_proj.weight.copy_(t(m.w(l, "wo").T))
            mlp.gate_proj.weight.copy_(t(m.w(l, "wgate").T))
            mlp.up_proj.weight.copy_(t(m.w(l, "wup").T))
            mlp.down_proj.weight.copy_(t(m.w(l, "wdown").T))
            layer.input_layernorm.weight.copy_(t(O.bf16_to_f64(m.norm(l, "attn_norm"))))
            layer.post_attention_layernorm.weight.copy_(t(O.bf16_to_f64(m.norm(l, "mlp_norm"))))
    return hf


def test_chain_tree_equals_hf_llama_prefill():
    """A chain tree with L = 0 is a plain causal Llama forward (R17): compare the
    oracle against HuggingFace's LlamaForCausalLM (a library implementation of
    RMSNorm, rotate-half RoPE, GQA attention, SwiGLU) in float64.  HF computes
    RoPE angles in fp32, hence the 1e-6-level tolerance."""
    torch = pytest.importorskip("torch")
    cfg, m, kv = _tiny(L=0)
    hf = _hf_llama(cfg, m)
    rng = np.random.default_rng(11)
    toks, parents = synth.tree_chain(8, cfg.vocab, rng)
    r = O.verify(cfg, m, kv, toks, parents)
    with torch.no_grad():
        ref = hf(torch.from_numpy(toks.astype(np.int64))[None]).logits[0].numpy()
    np.testing.assert_allclose(r["logits"], ref, atol=2e-6, rtol=1e-6)


def test_chain_with_prefix_equals_hf_llama_cached():
    """Same with a synthetic committed prefix fed to HF as a DynamicCache
    (post-RoPE keys), positions L..L+T-1."""
    torch = pytest.importorskip("torch")
    tf = pytest.importorskip("transformers")
    cfg, m, kv = _tiny(L=12)
    hf = _hf_llama(cfg, m)
    rng = np.random.default_rng(12)
    toks, parents = synth.tree_chain(5, cfg.vocab, rng)
    r = O.verify(cfg, m, kv, toks, parents)
    cache = tf.DynamicCache()
    for l in range(cfg.n_layers):
        k = torch.from_numpy(kv.K[l][:12].transpose(1, 0, 2)[None].copy())
        v = torch.from_numpy(kv.V[l][:12].transpose(1, 0, 2)[None].copy())
        cache.update(k, v, l)
    with torch.no_grad():
        out = hf(torch.from_numpy(toks.astype(np.int64))[None], past_key_values=cache,
                 position_ids=torch.arange(12, 17)[None], use_cache=True)
    np.testing.assert_allclose(r["logits"], out.logits[0].numpy(), atol=2e-6, rtol=1e-6)


def test_tree_logits_equal_sequential_decode(tiny16):
    """BJ invariant: tree-masked attention for each node equals sequential
    single-token decoding along that node's root path (brute force)."""
    cfg, m, kv = tiny16
    rng = np.random.default_rng(21)
    toks, parents = synth.tree_paperlike(8, cfg.vocab, rng)
    r = O.verify(cfg, m, kv, toks, parents)
    for i in range(len(toks)):
        path = []
        j = i
        while j != -1:
            path.append(int(toks[j]))
            j = int(parents[j])
        seq = O.forced_decode(cfg, m, kv.copy(), path[::-1])
        np.testing.assert_allclose(r["logits"][i], seq[-1], rtol=1e-10, atol=1e-10)


def test_sharded_sum_equals_unsharded(tiny16):
    """BJ invariant: the TP sharded sum equals the unsharded computation."""
    cfg, m, kv = tiny16
    rng = np.random.default_rng(22)
    toks, parents = synth.tree_random(8, cfg.vocab, rng)
    r1 = O.verify(cfg, m, kv, toks, parents)
    r2 = O.verify_sharded(cfg, m, kv, toks, parents, P=2)
    np.testing.assert_allclose(r2["logits"], r1["logits"], rtol=1e-11, atol=1e-11)
    for l in range(cfg.n_layers):
        np.testing.assert_allclose(r2["tree_k"][l], r1["tree_k"][l], rtol=1e-12, atol=1e-12)
    assert list(r2["argmax"]) == list(r1["argmax"])


@pytest.mark.parametrize("P", [3, 5, 6])
def test_sharded_zero_padding_equals_unsharded(tiny16, P):
    """Arbitrary TP by zero padding: heads padded to a multiple of
    P, intermediate to a multiple of 256 P, all padded weights zero; the
    rank-ordered sum of the padded shards equals the unpadded, unsharded model
    (the paper: "the model output is equivalent of the non-padded model")."""
    cfg, m, kv = tiny16
    Hq, Hkv, I = O.tp_padded_dims(cfg, P)
    assert Hkv % P == 0 and Hq == Hkv * (cfg.n_heads // cfg.n_kv_heads) and Hkv >= cfg.n_kv_heads
    assert I % P == 0 and (I // P) % 256 == 0 and I >= cfg.intermediate
    rng = np.random.default_rng(23 + P)
    toks, parents = synth.tree_random(8, cfg.vocab, rng)
    r1 = O.verify(cfg, m, kv, toks, parents)
    r2 = O.verify_sharded(cfg, m, kv, toks, parents, P=P)
    np.testing.assert_allclose(r2["logits"], r1["logits"], rtol=1e-11, atol=1e-11)
    for l in range(cfg.n_layers):
        np.testing.assert_allclose(r2["tree_k"][l], r1["tree_k"][l], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(r2["tree_v"][l], r1["tree_v"][l], rtol=1e-12, atol=1e-12)
    assert list(r2["argmax"]) == list(r1["argmax"])


def _planted_tree(cfg, m, kv, depth, T, rng):
    """Tree whose root path of `depth` nodes below the root is the target's greedy
    continuation (computed with plain greedy decoding), plus random distractors."""
    root = int(rng.integers(0, cfg.vocab))
    cont = O.greedy_decode(cfg, m, kv.copy(), root, depth + 1)
    toks = [root] + cont[:depth]
    parents = list(range(-1, depth))
    while len(toks) < T:
        p = int(rng.integers(0, len(toks)))
        t = int(rng.integers(0, cfg.vocab))
        if p < depth + 1 and p + 1 < len(toks) and parents[p + 1] == p and toks[p + 1] == t:
            continue
        toks.append(t)
        parents.append(p)
    return np.array(toks, np.int32), np.array(parents, np.int32), cont


def test_planted_accept_and_compaction_equal_greedy_decode(tiny16):
    """BJ invariant: accept/compaction yield the same KV cache (and tokens) as
    greedy decoding of the accepted tokens; planted depth d -> n = d + 1."""
    cfg, m, kv = tiny16
    rng = np.random.default_rng(23)
    depth = 3
    toks, parents, cont = _planted_tree(cfg, m, kv, depth, 8, rng)
    r = O.verify(cfg, m, kv, toks, parents)
    assert len(r["accepted"]) == depth + 1
    assert r["bonus"] == cont[depth]
    kv_tree = O.commit(kv.copy(), r, r["accepted"])
    kv_seq = kv.copy()
    O.forced_decode(cfg, m, kv_seq, [int(toks[i]) for i in r["accepted"]])
    assert kv_tree.L == kv_seq.L == 16 + depth + 1
    for l in range(cfg.n_layers):
        np.testing.assert_allclose(kv_tree.K[l][:kv_tree.L], kv_seq.K[l][:kv_seq.L], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(kv_tree.V[l][:kv_tree.L], kv_seq.V[l][:kv_seq.L], rtol=1e-12, atol=1e-12)


def test_repeated_verify_commit_reproduces_greedy(tiny16):
    """S:453 golden equivalence: verify+commit with planted chains (the draft
    equals the target) reproduces plain autoregressive greedy decoding."""
    cfg, m, kv0 = tiny16
    root = 77
    ref = O.greedy_decode(cfg, m, kv0.copy(), root, 12)
    kv = kv0.copy()
    out = []
    cur = root
    T = 4
    while len(out) < 12:
        # identical draft: root + the next T-1 greedy tokens
        nxt = ref[len(out):len(out) + T - 1]
        toks = [cur] + nxt
        r = O.verify(cfg, m, kv, toks, list(range(-1, len(toks) - 1)))
        assert len(r["accepted"]) == len(toks)
        O.commit(kv, r, r["accepted"])
        out += [int(toks[i]) for i in r["accepted"][1:]] + [r["bonus"]]
        cur = r["bonus"]
    assert out[:12] == ref


def test_streamed_weights_equal_dense():
    """OracleModel with a streamed column provider (the 70B / 8B full-size parity
    tests) computes the same verify as the dense weights: only the evaluation
    order of independent output columns differs."""
    from synth import fast
    cfg = synth.CONFIGS["tiny"]
    canon = synth.gen_model(cfg, 0)
    dense = O.OracleModel(cfg, canon)
    names = dict(wq=synth.KIND["WQ"], wk=synth.KIND["WK"], wv=synth.KIND["WV"], wo=synth.KIND["WO"],
                 wgate=synth.KIND["WGATE"], wup=synth.KIND["WUP"], wdown=synth.KIND["WDOWN"])

    def cols(layer, name, n0, n1):
        K = cfg.intermediate if name == "wdown" else (cfg.n_heads * cfg.head_dim if name == "wo" else cfg.hidden)
        return fast.gen_linear_cols(0, layer, names[name], K, dense.out_features(name), n0, n1)

    streamed = O.OracleModel(cfg, canon, cols=cols)
    kv = O.KVCache(cfg, 128)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(1, l, 32, cfg.n_kv_heads, cfg.head_dim)
        kv.set_prefix(l, k, v)
    kv.L = 32
    toks, par = synth.tree_paperlike(8, cfg.vocab, np.random.default_rng(0))
    a = O.verify(cfg, dense, kv, toks, par)
    b = O.verify(cfg, streamed, kv, toks, par)
    np.testing.assert_allclose(b["logits"], a["logits"], rtol=1e-12, atol=1e-12)
    assert list(a["argmax"]) == list(b["argmax"])


# ---------------------------------------------------------------- non-square mask (NEXT-3)
def test_nonsquare_mask_shape_and_rows_fig():
    """a current tree of size 6 and 4 leaves to compute need a mask of
    size (4, 10); each row is the leaf's ancestors-or-self (brute force: walk
    the parents by hand), the prefix is not part of the mask."""
    parents = [-1, 0, 0, 1, 1, 2, 3, 5, 4, 0]   # nodes 0..5 cached, leaves 6..9
    pos, mask = O.nonsquare_mask(parents, 6, L=20)
    assert mask.shape == (4, 10)
    want = {6: {6, 3, 1, 0}, 7: {7, 5, 2, 0}, 8: {8, 4, 1, 0}, 9: {9, 0}}
    for i, leaf in enumerate(range(6, 10)):
        assert set(np.nonzero(mask[i])[0]) == want[leaf]
    assert list(pos) == [20 + 3, 20 + 3, 20 + 3, 20 + 1]


def _split_tree(toks, parents, T0):
    return list(toks[:T0]), list(parents[:T0]), list(toks[T0:]), list(parents[T0:])


def test_forward_nonsquare_empty_cache_equals_verify(tiny16):
    """T0 = 0: the non-square forward of the whole tree is the square verify."""
    cfg, m, kv = tiny16
    toks, parents = synth.tree_paperlike(8, cfg.vocab, np.random.default_rng(31))
    r1 = O.verify(cfg, m, kv, toks, parents)
    r2 = O.forward_nonsquare(cfg, m, kv, None, toks, parents)
    np.testing.assert_allclose(r2["logits"], r1["logits"], rtol=1e-12, atol=1e-12)
    assert list(r2["argmax"]) == list(r1["argmax"]) and r2["accepted"] == r1["accepted"]


@pytest.mark.parametrize("cuts", [(5,), (3, 7), (1, 2, 4, 9)])
def test_forward_nonsquare_growth_equals_square_verify(tiny16, cuts):
    """Growing a tree by non-square forwards (the draft's expansions, P:321,
    Alg. 1) gives every node the logits and K/V of the square verify of
    the whole tree, and the accept walk over the grown tree is the same."""
    cfg, m, kv = tiny16
    toks, parents = synth.tree_random(12, cfg.vocab, np.random.default_rng(32))
    full = O.verify(cfg, m, kv, toks, parents)
    bounds = [0, *cuts, 12]
    tree = None
    for a, b in zip(bounds[:-1], bounds[1:]):
        tree = O.forward_nonsquare(cfg, m, kv, tree, toks[a:b], parents[a:b])
        np.testing.assert_allclose(tree["logits"], full["logits"][a:b], rtol=1e-10, atol=1e-10)
        assert tree["mask"].shape == (b - a, b)
    for l in range(cfg.n_layers):
        np.testing.assert_allclose(tree["tree_k"][l], full["tree_k"][l], rtol=1e-11, atol=1e-11)
        np.testing.assert_allclose(tree["tree_v"][l], full["tree_v"][l], rtol=1e-11, atol=1e-11)
    assert list(tree["argmax"]) == list(full["argmax"])
    assert tree["accepted"] == full["accepted"] and tree["bonus"] == full["bonus"]


def test_forward_nonsquare_chain_one_leaf_at_a_time_is_sequential_decode(tiny16):
    """A chain grown one leaf per call is plain sequential decoding:
    leaf i's logits equal forced single-token decoding of the chain prefix."""
    cfg, m, kv = tiny16
    chain = [11, 250, 3, 4000, 17]
    seq = O.forced_decode(cfg, m, kv.copy(), chain)
    tree = None
    for i, t in enumerate(chain):
        tree = O.forward_nonsquare(cfg, m, kv, tree, [t], [i - 1])
        np.testing.assert_allclose(tree["logits"][0], seq[i], rtol=1e-10, atol=1e-10)
    kv_seq = kv.copy()
    O.forced_decode(cfg, m, kv_seq, chain)
    kv_tree = O.commit(kv.copy(), tree, list(range(len(chain))))
    for l in range(cfg.n_layers):
        np.testing.assert_allclose(kv_tree.K[l][:kv_tree.L], kv_seq.K[l][:kv_seq.L], rtol=1e-12, atol=1e-12)


def test_nonsquare_mask_rejects_bad_split():
    with pytest.raises(ValueError):
        O.nonsquare_mask([-1, 0, 1], 3, 0)   # no leaf
    with pytest.raises(ValueError):
        O.nonsquare_mask([-1, 0, 2], 1, 0)   # parent not earlier
