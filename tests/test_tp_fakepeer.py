"""Tensor-parallel parity on ONE GPU ("fake-peer" mode): P shards of
the same model live on device 0, each capped to a fraction of the SMs so their
persistent kernels are co-resident; the fused flag-based all-reduces
and the argmax exchange run over the shards' receive buffers exactly as over
NVLink peers.  Compared with the oracle's sharded mode and the unsharded oracle."""
import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu


def _setup(cfg, P, L, seed=0):
    import torch
    import paper_2506_11309_b200 as pkg
    canon = synth.gen_model(cfg, seed)
    shards = []
    for r in range(P):
        sh = pkg.Shard(cfg, r, P, 0, max_ctx=L + 128, max_tree=16)
        sh.set_launch_cap(148 // P)
        sh.load_canonical(canon)
        for l in range(cfg.n_layers):
            k, v = synth.gen_prefix_kv(seed + 1, l, L, cfg.n_kv_heads, cfg.head_dim)
            sh.set_prefix_kv(l, k, v)
        shards.append(sh)
    pkg.Shard.import_local_peers(shards)
    m = O.OracleModel(cfg, canon)
    kv = O.KVCache(cfg, L + 128)
    for l in range(cfg.n_layers):
        k, v = synth.gen_prefix_kv(seed + 1, l, L, cfg.n_kv_heads, cfg.head_dim)
        kv.set_prefix(l, k, v)
    kv.L = L
    return shards, m, kv


def _run(shards, tokens, parents, auto_commit=False):
    """Launch the step on every shard on its own stream, then wait for all."""
    import torch
    from paper_2506_11309_b200 import swiftspec as ssp
    T = len(tokens)
    outs = []
    streams = [torch.cuda.Stream() for _ in shards]
    bufs = []
    for sh, st in zip(shards, streams):
        dt = torch.tensor(tokens, dtype=torch.int32, device="cuda")
        dp = torch.tensor(parents, dtype=torch.int32, device="cuda")
        res = torch.zeros(ssp.result_nbytes() // 4, dtype=torch.int32, device="cuda")
        lg = torch.zeros((T, sh.v_l), dtype=torch.float32, device="cuda")
        bufs.append((dt, dp, res, lg))
        torch.cuda.synchronize()
    for sh, st, (dt, dp, res, lg) in zip(shards, streams, bufs):
        sh.verify_dev(dt, dp, T, d_result=res, d_logits=lg, auto_commit=auto_commit, stream=st)
    torch.cuda.synchronize()
    for (dt, dp, res, lg) in bufs:
        outs.append((ssp.parse_result(res.cpu().numpy(), T), lg.cpu().numpy()))
    return outs


@pytest.mark.parametrize("P", [2, 4])
def test_fakepeer_tp_parity(P):
    cfg = synth.CONFIGS["small-tp"]
    L = 64
    shards, m, kv = _setup(cfg, P, L)
    rng = np.random.default_rng(P)
    for kind in ("paperlike", "chain"):
        tokens, parents = (synth.tree_paperlike if kind == "paperlike" else synth.tree_chain)(8, cfg.vocab, rng)
        outs = _run(shards, tokens, parents)
        ro = O.verify_sharded(cfg, m, kv, tokens, parents, P)
        logits = np.concatenate([lg for _, lg in outs], axis=1)
        err = np.abs(logits - ro["logits"])
        assert np.all(err <= 2e-2 + 1e-2 * np.abs(ro["logits"])), err.max()
        # every rank walks the same path from the same all-gathered argmax
        res0 = outs[0][0]
        assert all(res["status"] == 0 for res, _ in outs)  # no peer poll ran out of budget
        for res, _ in outs[1:]:
            assert res["argmax"] == res0["argmax"] and res["accepted"] == res0["accepted"]
            assert res["bonus"] == res0["bonus"]
        for i in range(len(tokens)):
            a, b = res0["argmax"][i], int(ro["argmax"][i])
            assert a == b or abs(ro["logits"][i][a] - ro["logits"][i][b]) < 2e-2
        acc, bonus = O.accept_walk(tokens, parents, res0["argmax"])
        assert res0["accepted"] == acc and res0["bonus"] == bonus
        for sh in shards:  # discard the pending (uncommitted) verify before the next tree
            sh.set_committed_len(L)
        # each rank holds its own kv heads of the tree rows
        hk = cfg.n_kv_heads // P
        for r, sh in enumerate(shards):
            for l in range(cfg.n_layers):
                k, v = sh.read_kv(l, L, len(tokens))
                np.testing.assert_allclose(k, ro["tree_k"][l][:, r * hk:(r + 1) * hk], atol=2e-2, rtol=1e-2)
    for sh in shards:
        sh.close()


@pytest.mark.parametrize("P", [3, 5, 6])
def test_fakepeer_tp_zero_padding(P):
    """Arbitrary TP by zero padding (the paper's 6+2
    split): P does not divide the 4 kv heads / the intermediate size, the
    library pads heads and columns with zero weights.  The ranks' logits equal
    the unpadded model's (oracle: padded sharded == unsharded, pinned in
    test_oracle), every rank walks the same path, each rank holds its real kv
    heads of the tree rows and zeros for its padded ones, and 3 auto-commit
    steps advance L identically."""
    cfg = synth.CONFIGS["small-tp"]
    L = 64
    shards, m, kv = _setup(cfg, P, L)
    hk = -(-cfg.n_kv_heads // P)
    rng = np.random.default_rng(40 + P)
    tokens, parents = synth.tree_paperlike(8, cfg.vocab, rng)
    outs = _run(shards, tokens, parents)
    ro = O.verify_sharded(cfg, m, kv, tokens, parents, P)
    logits = np.concatenate([lg for _, lg in outs], axis=1)
    err = np.abs(logits - ro["logits"])
    assert np.all(err <= 2e-2 + 1e-2 * np.abs(ro["logits"])), err.max()
    res0 = outs[0][0]
    assert all(res["status"] == 0 for res, _ in outs)
    for res, _ in outs[1:]:
        assert res["argmax"] == res0["argmax"] and res["accepted"] == res0["accepted"] and res["bonus"] == res0["bonus"]
    for i in range(len(tokens)):
        a, b = res0["argmax"][i], int(ro["argmax"][i])
        assert a == b or abs(ro["logits"][i][a] - ro["logits"][i][b]) < 2e-2
    for sh in shards:
        sh.set_committed_len(L)
    for r, sh in enumerate(shards):
        for l in range(cfg.n_layers):
            k, v = sh.read_kv(l, L, len(tokens))
            real = max(0, min(hk, cfg.n_kv_heads - r * hk))
            np.testing.assert_allclose(k[:, :real], ro["tree_k"][l][:, r * hk:r * hk + real], atol=2e-2, rtol=1e-2)
            np.testing.assert_allclose(v[:, :real], ro["tree_v"][l][:, r * hk:r * hk + real], atol=2e-2, rtol=1e-2)
            assert np.all(k[:, real:] == 0) and np.all(v[:, real:] == 0)
    total = 0
    for step in range(3):
        tokens, parents = synth.tree_random(8, cfg.vocab, rng)
        outs = _run(shards, tokens, parents, auto_commit=True)
        assert all(o[0]["status"] == 0 for o in outs), [o[0]["status"] for o in outs]
        assert all(o[0]["accepted"] == outs[0][0]["accepted"] for o in outs)
        total += outs[0][0]["n_accepted"]
        assert [sh.L for sh in shards] == [L + total] * P, (step, [o[0]["n_accepted"] for o in outs])
    for sh in shards:
        sh.close()


def test_fakepeer_tp_autocommit_many_steps():
    """Repeated steps exercise the LL flag epochs and both all-reduce buffer
    parities; the committed length advances identically on every rank."""
    cfg = synth.CONFIGS["small-tp"]
    L = 64
    shards, m, kv = _setup(cfg, 2, L)
    rng = np.random.default_rng(7)
    total = 0
    for step in range(6):
        tokens, parents = synth.tree_random(8, cfg.vocab, rng)
        outs = _run(shards, tokens, parents, auto_commit=True)
        assert outs[0][0]["accepted"] == outs[1][0]["accepted"]
        total += outs[0][0]["n_accepted"]
        assert [sh.L for sh in shards] == [L + total] * 2
    for sh in shards:
        sh.close()


def test_loopback_emulation_runs():
    """ss_import_loopback (bench.py tp_emulated): one rank of a TP group runs its whole
    step alone -- the fused all-reduce and argmax exchange complete without peers."""
    import paper_2506_11309_b200 as pkg
    cfg = synth.CONFIGS["small-tp"]
    sh = pkg.Shard(cfg, 0, 2, 0, max_ctx=64 + 128, max_tree=16)
    sh.synth_weights(0)
    sh.synth_prefix_kv(1, 64)
    sh.import_loopback()
    for T in (1, 8, 13):
        tokens, parents = synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(T))
        r = sh.verify(tokens, parents)
        assert r["status"] == 0
        assert all(0 <= a < cfg.vocab for a in r["argmax"])
        sh.commit_accepted()
    sh.close()


_ORACLE_70B = {}


def _oracle_70b_layer(cfg, L, tokens, parents):
    """Float64 oracle of the unsharded 1-layer 70B-shaped model up to the final norm
    (TP is exact up to summation order), cached across the TP sizes."""
    import dataclasses
    key = (L, tuple(tokens), tuple(parents))
    if key not in _ORACLE_70B:
        canon = {"layers": [synth.gen_model(dataclasses.replace(cfg, vocab=8), 0, with_lm_head=False)["layers"][0]],
                 "embed": None, "final_norm": synth.gen_norm(0, -1, synth.KIND["FINAL_NORM"], cfg.hidden)}
        m = O.OracleModel(cfg, canon, cache_dense=False)
        kv = O.KVCache(cfg, L + 64)
        k, v = synth.gen_prefix_kv(1, 0, L, cfg.n_kv_heads, cfg.head_dim)
        kv.set_prefix(0, k, v)
        kv.L = L
        depth, pos, anc = O.tree_meta(parents, L)
        x = O.bf16_to_f64(synth.gen_embed(0, cfg.vocab, cfg.hidden, rows=tokens))
        x, _, _ = O.layer_forward(cfg, m, 0, x, kv, L, pos, anc)
        _ORACLE_70B[key] = O.rmsnorm(x, canon["final_norm"], cfg.rms_eps)
    return _ORACLE_70B[key]


@pytest.mark.parametrize("P,ar", [(2, "one-shot"), (4, "one-shot"), (8, "one-shot"), (8, "two-shot"), (4, "two-shot")])
def test_70b_shaped_layer_tp_fakepeer_sampled(P, ar):
    """TP = 2 / 4 / 8 at full Llama3-70B layer shape (h 8192, I 28672, 64/8 heads,
    128256-row vocab-parallel LM head, 4K prefix): P fake-peer shards synthesised on the
    device, the fused all-reduces over h/128 = 64 tile-groups and the argmax exchange;
    logits of all shards vs the float64 oracle on a seeded vocab sample (cf. the TP 1
    test in test_gpu_parity.py).  TP 8 = one kv head per rank (the paper's headline
    70B configuration)."""
    import dataclasses
    import paper_2506_11309_b200 as pkg
    cfg = dataclasses.replace(synth.CONFIGS["llama3-70b"], n_layers=1)
    L, T = 4096, 8
    shards = []
    for r in range(P):
        sh = pkg.Shard(cfg, r, P, 0, max_ctx=L + 64, max_tree=8)
        sh.set_launch_cap(148 // P)
        sh.synth_weights(0)
        sh.synth_prefix_kv(1, L)
        sh.set_allreduce(ar)
        shards.append(sh)
    pkg.Shard.import_local_peers(shards)
    rng = np.random.default_rng(72)
    tokens, parents = synth.tree_paperlike(T, cfg.vocab, rng)
    outs = _run(shards, tokens, parents)
    for sh in shards:
        sh.close()
    logits = np.concatenate([lg for _, lg in outs], axis=1)[:, :cfg.vocab]
    res0 = outs[0][0]
    # -5 = SS_ETIMEOUT: a rank's all-reduce poll ran out of budget (seen when PDL
    # grids of one fake peer held the SM slots the other peer's kernel needed)
    assert [res["status"] for res, _ in outs] == [0] * P
    for res, _ in outs[1:]:
        assert res["argmax"] == res0["argmax"] and res["accepted"] == res0["accepted"]
    xn = _oracle_70b_layer(cfg, L, tokens, parents)
    sample = np.unique(np.concatenate([rng.choice(cfg.vocab, 4096, replace=False), res0["argmax"][:T]]))
    lo = xn @ O.bf16_to_f64(synth.gen_lm_head(0, cfg.vocab, cfg.hidden, rows=sample)).T
    lg = logits[:, sample]
    err = np.abs(lg - lo)
    assert np.all(err <= 2e-2 + 1e-2 * np.abs(lo)), err.max()
    for i in range(T):
        g = int(res0["argmax"][i])
        gi = int(np.searchsorted(sample, g))
        assert sample[np.argmax(lo[i])] == g or lo[i].max() - lo[i][gi] < 2e-2, (i, g)


@pytest.mark.parametrize("P", [2, 4])
def test_device_synth_shards_match_host_load(P):
    """TP shards generated on the device (ss_synth_weights / ss_synth_prefix_kv with
    rank slicing, as bench.py uses them) equal host-packed canonical shards."""
    import paper_2506_11309_b200 as pkg
    cfg = synth.CONFIGS["small-tp"]
    L = 64
    host, m, kv = _setup(cfg, P, L)
    dev = []
    for r in range(P):
        sh = pkg.Shard(cfg, r, P, 0, max_ctx=L + 128, max_tree=16)
        sh.set_launch_cap(148 // P)
        sh.synth_weights(0)
        sh.synth_prefix_kv(1, L)
        dev.append(sh)
    pkg.Shard.import_local_peers(dev)
    tokens, parents = synth.tree_paperlike(8, cfg.vocab, np.random.default_rng(9))
    a = np.concatenate([lg for _, lg in _run(host, tokens, parents)], axis=1)
    b = np.concatenate([lg for _, lg in _run(dev, tokens, parents)], axis=1)
    for sh in host + dev:
        sh.close()
    # run-to-run fp32 reduction order (stream-K red.add) differs by ~1e-3
    np.testing.assert_allclose(b, a, atol=1e-2, rtol=1e-2)


# ---------------------------------------------------------------- two-shot all-reduce (NEXT-2)
@pytest.mark.parametrize("P", [2, 3, 4])
def test_fakepeer_two_shot_allreduce(P):
    """Two-shot LL all-reduce (ss_set_allreduce): partials
    reduce-scattered to each tile-group's home rank (tg mod P), which sums in
    rank order and broadcasts.  Logits within R13 of the sharded oracle, every
    rank walks the same path, and repeated auto-commit steps (both buffer
    parities, flag epochs) advance L identically; then back to one-shot on the
    same shards, with the same accept results for the same tree."""
    cfg = synth.CONFIGS["small-tp"]
    L = 64
    shards, m, kv = _setup(cfg, P, L)
    for sh in shards:
        sh.set_allreduce("two-shot")
    rng = np.random.default_rng(60 + P)
    tokens, parents = synth.tree_paperlike(8, cfg.vocab, rng)
    outs = _run(shards, tokens, parents)
    ro = O.verify_sharded(cfg, m, kv, tokens, parents, P)
    logits = np.concatenate([lg for _, lg in outs], axis=1)
    err = np.abs(logits - ro["logits"])
    assert np.all(err <= 2e-2 + 1e-2 * np.abs(ro["logits"])), err.max()
    assert all(res["status"] == 0 for res, _ in outs)
    for res, _ in outs[1:]:
        assert res["argmax"] == outs[0][0]["argmax"] and res["accepted"] == outs[0][0]["accepted"]
    for sh in shards:
        sh.set_committed_len(L)
    for sh in shards:
        sh.set_allreduce("one-shot")
    outs1 = _run(shards, tokens, parents)
    lg1 = np.concatenate([lg for _, lg in outs1], axis=1)
    assert np.max(np.abs(lg1 - logits)) <= 5e-3      # same rank-ordered sums; stream-K order differs run to run
    for sh in shards:
        sh.set_committed_len(L)
        sh.set_allreduce("two-shot")
    total = 0
    for step in range(4):
        tokens, parents = synth.tree_random(8 if step % 2 else 13, cfg.vocab, rng)
        outs = _run(shards, tokens, parents, auto_commit=True)
        assert all(o[0]["status"] == 0 for o in outs)
        assert all(o[0]["accepted"] == outs[0][0]["accepted"] for o in outs)
        total += outs[0][0]["n_accepted"]
        assert [sh.L for sh in shards] == [L + total] * P
    for sh in shards:
        sh.close()


def test_loopback_two_shot_runs():
    """The TP-rank timing emulation also runs the two-shot scheme (home and
    non-home tile-groups, stand-in broadcasts)."""
    import paper_2506_11309_b200 as pkg
    cfg = synth.CONFIGS["small-tp"]
    sh = pkg.Shard(cfg, 0, 4, 0, max_ctx=64 + 128, max_tree=16)
    sh.synth_weights(0)
    sh.synth_prefix_kv(1, 64)
    sh.import_loopback()
    sh.set_allreduce("two-shot")
    for T in (1, 8, 13):
        tokens, parents = synth.tree_paperlike(T, cfg.vocab, np.random.default_rng(T))
        r = sh.verify(tokens, parents)
        assert r["status"] == 0
        sh.commit_accepted()
    sh.close()


@pytest.mark.parametrize("ar", ["one-shot", "two-shot"])
def test_ll_stress_million_lines(ar):
    """LL protocol stress ("10^6-message stress"): 64 steps of
    the 2-layer small-tp model at TP 2 over fake peers move 4 all-reduces x
    8 tile-groups x 128 rows x 4 LL lines = 16K lines per rank per step (one-
    shot; about half with two-shot), > 10^6 over the run, through both buffer
    parities and 64 flag epochs.  Every step completes with SS_OK on both
    ranks, the ranks agree, and since only the root is committed each step
    (a chain the test controls) the oracle follows the same cache: the last
    step's logits match it (R13)."""
    cfg = synth.CONFIGS["small-tp"]
    L = 64
    P = 2
    shards, m, kv = _setup(cfg, P, L)
    for sh in shards:
        sh.set_allreduce(ar)
    rng = np.random.default_rng(99)
    kvo = kv.copy()
    for step in range(64):
        tokens, parents = synth.tree_random(8, cfg.vocab, rng)
        outs = _run(shards, tokens, parents)
        assert all(o[0]["status"] == 0 for o in outs), (step, [o[0]["status"] for o in outs])
        assert outs[0][0]["argmax"] == outs[1][0]["argmax"]
        for sh in shards:
            sh.commit_kv([0])
        if step == 63:
            ro = O.verify_sharded(cfg, m, kvo, tokens, parents, P)
            logits = np.concatenate([lg for _, lg in outs], axis=1)
            err = np.abs(logits - ro["logits"])
            assert np.all(err <= 2e-2 + 1e-2 * np.abs(ro["logits"])), err.max()
        else:
            r = O.verify(cfg, m, kvo, tokens[:1], parents[:1])
            O.commit(kvo, r, [0])
    assert [sh.L for sh in shards] == [L + 64] * P
    for sh in shards:
        sh.close()
