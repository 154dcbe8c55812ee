"""Bit-exact GPU checks (BASELINE north_star: "bit-exact for tree masks, accept
indices and KV compaction"; SURVEY 8(c) pins):

* tree metadata (a0): the device's ancestor bitmasks and positions equal
  oracle.tree_meta (brute-force parent walk, R8) for many tree shapes;
* the device synthetic generator writes exactly the bytes of the host repack of
  synth/generators.py tensors (every packed linear, LM head, embedding, norms;
  TP shards too) -- the full-size parity tests rely on this equivalence;
* integer-valued GEMM inputs give bit-exact sums in any reduction order
  (SURVEY 8(c) "integer-valued partials -> bit-exact sums"), for every linear,
  and through the fused TP all-reduce (fake peers, TP 2 / 4);
* exact logit ties pick the lowest token id (R6) and duplicate sibling
  tokens accept the lowest-index child (R7).
"""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2506_11309_b200 as pkg
    return pkg


def _load(cfg, canon, L=64, max_ctx=None, max_tree=64, tp=(0, 1), seed_kv=1):
    pkg = _pkg()
    sh = pkg.Shard(cfg, tp[0], tp[1], 0, max_ctx=max_ctx or L + 256, max_tree=max_tree)
    sh.load_canonical(canon)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(seed_kv, l, L, cfg.n_kv_heads, cfg.head_dim)
        sh.set_prefix_kv(l, k, v)
    return sh


def _oracle(cfg, canon, L=64, max_ctx=None, seed_kv=1):
    m = O.OracleModel(cfg, canon)
    kv = O.KVCache(cfg, max_ctx or L + 256)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(seed_kv, l, L, cfg.n_kv_heads, cfg.head_dim)
        kv.set_prefix(l, k, v)
    kv.L = L
    return m, kv


@pytest.fixture(scope="module")
def tiny():
    cfg = synth.CONFIGS["tiny"]
    canon = synth.gen_model(cfg, 0)
    sh = _load(cfg, canon)
    yield cfg, canon, sh
    sh.close()


def test_tree_meta_bit_exact(tiny):
    cfg, canon, sh = tiny
    rng = np.random.default_rng(11)
    kinds = [synth.tree_chain, synth.tree_star, synth.tree_paperlike, synth.tree_random]
    n = 0
    for T in (1, 2, 7, 8, 9, 16, 31, 33, 64):
        for gen in kinds:
            toks, par = gen(T, cfg.vocab, rng)
            sh.set_committed_len(64)
            sh.verify(toks, par)
            Tg, pos, anc, tok_g, par_g = sh.read_tree_meta()
            depth, pos_o, anc_o = O.tree_meta(par, 64)
            bits = np.array([sum(1 << j for j in range(T) if anc_o[i, j]) for i in range(T)], dtype=np.uint64)
            assert Tg == T
            assert np.array_equal(pos, pos_o.astype(np.int32)), (T, gen.__name__)
            assert np.array_equal(anc, bits), (T, gen.__name__)
            assert np.array_equal(tok_g, toks) and np.array_equal(par_g, par)
            n += 1
    assert n == 36
    sh.set_committed_len(64)


REGIONS_LAYER = [0, 1, 2, 3, 6, 7]   # qkv, o, gate/up, down, attn norm, mlp norm
REGIONS_GLOBAL = [4, 5, 8]           # lm head, embedding, final norm


@pytest.mark.parametrize("cfg_name,P", [("tiny", 1), ("small-tp", 2), ("small-tp", 4)])
def test_device_synth_bytes_equal_host_repack(cfg_name, P):
    """ss_synth_weights (device generator, used by bench.py and the 70B tests)
    writes byte-for-byte the layout ss_load_weights repacks from synth tensors."""
    pkg = _pkg()
    cfg = synth.CONFIGS[cfg_name]
    canon = synth.gen_model(cfg, 5)
    for r in range(P):
        a = pkg.Shard(cfg, r, P, 0, max_ctx=256, max_tree=16)
        a.load_canonical(canon)
        b = pkg.Shard(cfg, r, P, 0, max_ctx=256, max_tree=16)
        b.synth_weights(5)
        for l in range(cfg.n_layers):
            for w in REGIONS_LAYER:
                x, y = a.read_packed(l, w), b.read_packed(l, w)
                assert x.size > 0 and np.array_equal(x, y), (r, l, w, int(np.count_nonzero(x != y)))
        for w in REGIONS_GLOBAL:
            x, y = a.read_packed(0, w), b.read_packed(0, w)
            assert x.size > 0 and np.array_equal(x, y), (r, w)
        a.close()
        b.close()


def _int_model(cfg, seed=0):
    """Canonical weights whose dequantised values are small multiples of 2^-6:
    q, z uniform nibbles, every AWQ scale = 2^-6 (exact in bf16)."""
    m = synth.gen_model(cfg, seed)
    one = synth.f32_to_bf16_bits(np.float32(2.0 ** -6))
    for li, lw in enumerate(m["layers"]):
        for ni, n in enumerate(("wq", "wk", "wv", "wo", "wgate", "wup", "wdown")):
            q, z, s = lw[n]
            rng = np.random.default_rng(100 * li + ni)
            z2 = rng.integers(0, 16, z.shape).astype(np.uint8)   # adversarial zero points too: 0..15
            lw[n] = (q, z2, np.full_like(s, one))
    return m


def _gemm_ref(q, z, x):
    """Exact reference of x @ ((q - z) * 2^-6): integer arithmetic (int64), then scaled."""
    K, N = q.shape
    g = np.arange(K) // 128
    w = q.astype(np.int64) - z[g, :].astype(np.int64)
    return (x.astype(np.int64) @ w).astype(np.float64) * 2.0 ** -6


@pytest.mark.parametrize("T", [1, 8, 13, 32])
def test_integer_gemm_bit_exact(T):
    """Every linear of the step's W4 GEMM kernel on integer-valued activations
    (|x| <= 4, exact in fp16) and weights (q - z) * 2^-6: all partial sums are
    exact in fp32, so the GPU result must equal the integer result exactly --
    a wrong nibble order, group index, zero point or split-K reduction fails."""
    import torch
    cfg = synth.CONFIGS["small-tp"]
    canon = _int_model(cfg)
    sh = _load(cfg, canon, L=0, max_ctx=256)
    rng = np.random.default_rng(T)
    d, h, I = cfg.head_dim, cfg.hidden, cfg.intermediate
    lw = canon["layers"][1]
    cases = {
        0: (h, [("wq", None), ("wk", None), ("wv", None)]),
        1: (cfg.n_heads * d, [("wo", None)]),
        2: (h, [("wgate", None), ("wup", None)]),
        3: (I, [("wdown", None)]),
    }
    for which, (K, names) in cases.items():
        x = rng.integers(-4, 5, (T, K)).astype(np.float32)
        ref = np.concatenate([_gemm_ref(lw[n][0], lw[n][1], x) for n, _ in names], axis=1)
        if which == 2:  # packed order: per 128-row tile-group 64 gate then 64 up columns
            g, u = ref[:, :I], ref[:, I:]
            ref = np.concatenate([np.concatenate([g[:, i:i + 64], u[:, i:i + 64]], axis=1)
                                  for i in range(0, I, 64)], axis=1)
        n_pad = -(-ref.shape[1] // 128) * 128
        dx = torch.tensor(x, device="cuda")
        dy = torch.full((T, n_pad), float("nan"), device="cuda")
        sh.debug_gemm(1, which, dx, T, dy)
        torch.cuda.synchronize()
        y = dy.cpu().numpy().astype(np.float64)
        assert np.array_equal(y[:, :ref.shape[1]], ref), (which, float(np.abs(y[:, :ref.shape[1]] - ref).max()))
    sh.close()


@pytest.mark.parametrize("P", [2, 4])
def test_integer_allreduce_bit_exact(P):
    """The fused tensor-parallel all-reduce of the O / down epilogues
    over fake peers: integer-valued partials sum bit-exactly, identically on
    every rank, to the unsharded integer GEMM."""
    import torch
    pkg = _pkg()
    cfg = synth.CONFIGS["small-tp"]
    canon = _int_model(cfg)
    shards = []
    for r in range(P):
        sh = pkg.Shard(cfg, r, P, 0, max_ctx=256, max_tree=16)
        sh.set_launch_cap(148 // P)
        sh.load_canonical(canon)
        shards.append(sh)
    pkg.Shard.import_local_peers(shards)
    lw = canon["layers"][0]
    T = 8
    rng = np.random.default_rng(P)
    for which, name, K in ((1, "wo", cfg.n_heads * cfg.head_dim), (3, "wdown", cfg.intermediate)):
        for rep in range(3):   # repeated calls: LL flag epochs and buffer reuse
            x = rng.integers(-4, 5, (T, K)).astype(np.float32)
            ref = _gemm_ref(lw[name][0], lw[name][1], x)
            Kl = K // P
            xs = [torch.tensor(np.ascontiguousarray(x[:, r * Kl:(r + 1) * Kl]), device="cuda") for r in range(P)]
            ys = [torch.zeros((T, cfg.hidden), device="cuda") for _ in range(P)]
            torch.cuda.synchronize()
            streams = [torch.cuda.Stream() for _ in range(P)]
            for sh, st, dx, dy in zip(shards, streams, xs, ys):
                sh.debug_gemm(0, which, dx, T, dy, allreduce=True, stream=st)
            torch.cuda.synchronize()
            for r in range(P):
                y = ys[r].cpu().numpy().astype(np.float64)
                assert np.array_equal(y, ref), (which, rep, r, float(np.abs(y - ref).max()))
    for sh in shards:
        sh.close()


def _tie_model(cfg, seed=0):
    """LM head with all rows zero except two identical rows (ids a < b) = +c e_k
    and two identical rows (ids c < d) = -c e_k: every logit is 0 or +-c*xn[k],
    computed exactly in any order, and the maximum is always an exact tie."""
    m = synth.gen_model(cfg, seed)
    W = np.zeros_like(m["lm_head"])
    big = synth.f32_to_bf16_bits(np.float32(8.0))
    neg = synth.f32_to_bf16_bits(np.float32(-8.0))
    ids = (1000, 3000, 777, 2500)
    k = 5
    W[ids[0], k] = W[ids[1], k] = big
    W[ids[2], k] = W[ids[3], k] = neg
    m["lm_head"] = W
    return m, ids


def test_exact_logit_ties_pick_lowest_id():
    cfg = synth.CONFIGS["tiny"]
    canon, (a, b, c, d) = _tie_model(cfg)
    sh = _load(cfg, canon)
    m, kv = _oracle(cfg, canon)
    rng = np.random.default_rng(4)
    toks, par = synth.tree_paperlike(16, cfg.vocab, rng)
    rg = sh.verify(toks, par, want_logits=True)
    ro = O.verify(cfg, m, kv, toks, par)
    for i in range(16):
        want = a if ro["logits"][i][a] > 0 else c       # lowest id of the tied pair
        assert int(ro["argmax"][i]) == want
        assert rg["logits"][i][a] == rg["logits"][i][b] and rg["logits"][i][c] == rg["logits"][i][d]
        assert rg["argmax"][i] == want, (i, rg["argmax"][i], want)
    sh.close()


def test_duplicate_sibling_tokens_accept_lowest_index():
    """R7: two children of the root carry the target's greedy token; the walk
    takes the lower node index (and the oracle agrees)."""
    cfg = synth.CONFIGS["tiny"]
    canon = synth.gen_model(cfg, 0)
    sh = _load(cfg, canon)
    m, kv = _oracle(cfg, canon)
    root = 77
    g = int(O.verify(cfg, m, kv, [root], [-1])["argmax"][0])
    other = (g + 1) % cfg.vocab
    toks = [root, other, g, g, 5, 6]
    par = [-1, 0, 0, 0, 2, 3]
    rg = sh.verify(toks, par, want_logits=True)
    ro = O.verify(cfg, m, kv, toks, par)
    assert ro["accepted"][:2] == [0, 2]
    if rg["argmax"][0] == g:
        assert rg["accepted"][:2] == [0, 2]
    acc, bonus = O.accept_walk(toks, par, rg["argmax"])
    assert rg["accepted"] == acc and rg["bonus"] == bonus
    sh.close()


# ---------------------------------------------------------------- deterministic mode
@pytest.mark.parametrize("cfg_name,L,T", [("tiny", 64, 8), ("small-tp", 64, 13), ("llama3-1b", 256, 16)])
def test_deterministic_mode_bit_identical(cfg_name, L, T):
    """SS_DEBUG_DETERMINISTIC: the same step run three times
    gives bit-identical logits, argmax and tree K/V, and stays within the
    oracle tolerance (R13)."""
    import paper_2506_11309_b200 as pkg
    from paper_2506_11309_b200 import swiftspec as ssp
    from test_gpu_parity import build, check_logits, oracle_setup
    cfg = synth.CONFIGS[cfg_name]
    sh = build(cfg, L=L, max_ctx=L + 64, max_tree=32)
    try:
        sh.set_debug(ssp.SS_DEBUG_DETERMINISTIC)
        toks, parents = synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(T))
        outs = []
        for _ in range(3):
            sh.set_committed_len(L)
            r = sh.verify(toks, parents, want_logits=True)
            k, v = sh.read_kv(cfg.n_layers - 1, L, T)
            outs.append((r["logits"].copy(), list(r["argmax"]), k, v))
        for lg, am, k, v in outs[1:]:
            assert np.array_equal(lg, outs[0][0]) and am == outs[0][1]
            assert np.array_equal(k, outs[0][2]) and np.array_equal(v, outs[0][3])
        if cfg_name != "llama3-1b":
            m, kv = oracle_setup(cfg, L=L, max_ctx=L + 64)
            check_logits(outs[0][0], O.verify(cfg, m, kv, toks, parents)["logits"])
        sh.set_debug(0)
        sh.set_committed_len(L)
        r = sh.verify(toks, parents, want_logits=True)
        check_logits(r["logits"], outs[0][0])          # default mode: same values to the tolerance
    finally:
        sh.close()
