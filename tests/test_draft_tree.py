"""The draft worker's tree logic (Alg. 1, ML
expansion P:259, re-root + KV reorganisation P:334-347), CPU only.

1. The plain reference (oracle/draft_tree.py) is pinned against the paper's
   worked examples: the Fig. 5 walkthrough (the top bs = 4 of the
   tree t1..t6 are (t1, t2, t3, t5); output (t1, t3, t6) re-roots at t6; a
   bonus t16 absent from the tree becomes the new root) and the KV example of
   P:343-345 (verified t12, t15: t12 moves to the prefix, the subtree of t15
   -- t17, t18 -- is packed right after it, everything else is discarded).
2. The product's C++ tree (csrc/draft_tree.h, compiled with g++) makes the
   same decision as the reference at every step of long random runs."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle.draft_tree import DraftTreeRef

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- pins of the reference
def _ref_fig5():
    """Tree t1..t6: t1 root; children t2, t3; t3 -> t5, t6; t2 -> t4.
    Log-probabilities chosen so the top 4 are (t1, t2, t3, t5) as the text says."""
    r = DraftTreeRef(1)
    r.computed([0])
    r.add_children(0, [2, 3], [-0.5, -0.4])            # nodes 1 (t2), 2 (t3)
    r.computed([1, 2])
    r.add_children(1, [4], [-1.5])                     # node 3 (t4): -2.0
    r.add_children(2, [5, 6], [-0.3, -1.2])            # nodes 4 (t5): -0.7, 5 (t6): -1.6
    return r


def test_ref_fig5_subgraph_top_bs():
    r = _ref_fig5()
    toks, pars, chosen = r.subgraph(4)
    assert toks == [1, 2, 3, 5] and pars == [-1, 0, 0, 2]


def test_ref_fig5_reroot_at_verified_bonus():
    """output_1 = (t1, t3, t6): root t1, accepted t3, bonus t6 -> re-root at t6;
    t1, t3 go to the prefix, nothing else of the old tree survives but t6."""
    r = _ref_fig5()
    toks, pars, chosen = r.subgraph(4)
    commit, keep, n = r.reroot([chosen[0], chosen[2]], 6)
    assert n == 2 and commit == [0, 2] and keep == []
    assert r.troot == 0 and len(r.nodes) == 1 and r.nodes[0]["token"] == 6 and r.nodes[0]["weight"] == 0.0


def test_ref_bonus_not_in_tree_becomes_new_root():
    """output_2 = (t6, t9, t16) with t16 not in the tree: re-root at a new t16."""
    r = DraftTreeRef(6)
    r.computed([0])
    r.add_children(0, [9, 10], [-0.1, -0.2])
    r.computed([1])
    r.add_children(1, [11], [-0.3])
    commit, keep, n = r.reroot([0, 1], 16)
    assert commit == [0, 1] and keep == [] and [x["token"] for x in r.nodes] == [16]


def test_ref_kv_reorganisation_p343():
    """Verified prefix ends at t10 (the draft root, computed); the tree holds
    t11, t12 under t10, t13, t15 under t12, t17, t18 under t15, t14, t16 under
    t11, all computed.  The target verifies t12 and samples t15: t10, t12 are
    committed, the subtree of t15 (t15, t17, t18) is kept, packed in slot order
    right after the prefix; t11, t13, t14, t16 are discarded."""
    r = DraftTreeRef(10)
    r.computed([0])                                           # t10 slot 0
    r.add_children(0, [11, 12], [-0.2, -0.3])                 # 1: t11, 2: t12
    r.computed([1, 2])                                        # slots 1, 2
    r.add_children(2, [13, 15], [-0.5, -0.6])                 # 3: t13, 4: t15
    r.add_children(1, [14, 16], [-0.4, -0.9])                 # 5: t14, 6: t16
    r.computed([3, 4, 5, 6])                                  # slots 3, 4, 5, 6
    r.add_children(4, [17, 18], [-0.1, -0.2])                 # 7: t17, 8: t18
    r.computed([7, 8])                                        # slots 7, 8
    commit, keep, n = r.reroot([0, 2], 15)
    assert commit == [0, 2] and keep == [4, 7, 8] and n == 2
    assert [x["token"] for x in r.nodes] == [15, 17, 18]
    assert [x["slot"] for x in r.nodes] == [0, 1, 2] and [x["parent"] for x in r.nodes] == [-1, 0, 0]
    assert r.nodes[1]["weight"] == pytest.approx(-0.1) and r.nodes[2]["weight"] == pytest.approx(-0.2)


def test_ref_uncomputed_verified_chain_stays_certain():
    """Verified nodes without draft K/V (sent to the target as unexpanded
    leaves) stay as a weight-0 chain above the new target root (R27); the
    next selection expands that chain first, in order."""
    r = DraftTreeRef(5)
    r.computed([0])
    r.add_children(0, [7, 8], [-0.1, -2.0])                   # 1: t7 (leaf, uncomputed), 2: t8
    commit, keep, n = r.reroot([0, 1], 9)                     # target accepted t7, bonus t9
    assert commit == [0] and keep == [] and n == 1
    assert [x["token"] for x in r.nodes] == [7, 9] and r.troot == 1
    assert [x["weight"] for x in r.nodes] == [0.0, 0.0]
    assert r.select(8) == [0, 1]
    assert r.forward_inputs([0, 1]) == ([7, 9], [-1, 0])


def test_ref_select_is_most_probable_and_capped():
    r = DraftTreeRef(1, max_slots=3)
    r.computed([0])
    r.add_children(0, [2, 3, 4], [-0.3, -0.1, -0.2])
    assert r.select(1) == [2]               # weight -0.1
    assert r.select(2) == [2, 3]            # weights -0.1 (node 2), -0.2 (node 3), in id order
    assert r.select(8) == [2, 3]            # only 2 free rows (max_slots 3)


# ---------------------------------------------------------------- C++ tree == reference
@pytest.fixture(scope="module")
def dt(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("dt") / "libdt.so")
    src = os.path.join(ROOT, "tests", "native", "draft_tree_harness.cpp")
    subprocess.run(["g++", "-O1", "-std=c++17", "-shared", "-fPIC", src, "-o", so], check=True)
    L = C.CDLL(so)
    vp, i32, ip, dp = C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)
    for n, res, args in [("dt_new", vp, [i32, i32]), ("dt_free", None, [vp]), ("dt_n_nodes", i32, [vp]),
                         ("dt_n_slots", i32, [vp]), ("dt_troot", i32, [vp]), ("dt_size", i32, [vp]),
                         ("dt_node", None, [vp, i32, ip, dp]), ("dt_select", i32, [vp, i32, ip, ip, ip]),
                         ("dt_computed", None, [vp, ip, i32]), ("dt_add_children", None, [vp, i32, ip, dp, i32]),
                         ("dt_subgraph", i32, [vp, i32, ip, ip, ip]),
                         ("dt_reroot", i32, [vp, ip, i32, i32, ip, ip, ip, ip])]:
        f = getattr(L, n)
        f.restype = res
        f.argtypes = args
    return L


def _ia(n):
    return (C.c_int * max(n, 1))()


def _nodes(dt, h):
    out = []
    for i in range(dt.dt_n_nodes(h)):
        a = _ia(3)
        w = C.c_double()
        dt.dt_node(h, i, a, C.byref(w))
        out.append((a[0], a[1], a[2], w.value))
    return out


def _ref_nodes(r):
    return [(n["token"], n["parent"], n["slot"], n["weight"]) for n in r.nodes]


@pytest.mark.parametrize("seed", range(6))
def test_cpp_tree_matches_reference(dt, seed):
    """Alg. 1 rounds driven by synthetic draft outputs (random top-K tokens and
    log-probabilities, ties included) and synthetic target results (a random
    root-anchored path of the sent subgraph + a bonus that is or is not in the
    tree): every selection, forward input, subgraph and re-root agrees."""
    rng = np.random.default_rng(seed)
    V, K, w, bs, d, max_slots = 50, 4, 4, 6, 3, 40
    ref = DraftTreeRef(7, max_slots)
    h = dt.dt_new(7, max_slots)

    def expand():
        sel, tk, pr = _ia(w), _ia(w), _ia(w)
        n = dt.dt_select(h, w, sel, tk, pr)
        rs = ref.select(w)
        assert list(sel[:n]) == rs
        rt, rp = ref.forward_inputs(rs)
        assert list(tk[:n]) == rt and list(pr[:n]) == rp
        arr = (C.c_int * max(n, 1))(*rs)
        dt.dt_computed(h, arr, n)
        ref.computed(rs)
        for node in rs:
            toks = rng.choice(V, K, replace=False).astype(int)
            lp = np.round(np.sort(-rng.exponential(1.0, K)), 1)   # rounding makes ties
            dt.dt_add_children(h, node, (C.c_int * K)(*toks), (C.c_double * K)(*lp), K)
            ref.add_children(node, toks, lp)
        return n

    for rnd in range(25):
        for _ in range(d):
            expand()
        while dt.dt_size(h) < bs:
            if expand() == 0:
                break
        assert dt.dt_size(h) == ref.tree_size()
        tk, pr, mp = _ia(bs), _ia(bs), _ia(bs)
        n = dt.dt_subgraph(h, bs, tk, pr, mp)
        rt, rp, rm = ref.subgraph(bs)
        assert (list(tk[:n]), list(pr[:n]), list(mp[:n])) == (rt, rp, rm)
        # target: accept a random root-anchored chain of the subgraph, then a bonus
        path = [0]
        while True:
            kids = [i for i in range(n) if rp[i] == path[-1]]
            if not kids or rng.random() < 0.3:
                break
            path.append(int(rng.choice(kids)))
        kids = [rt[i] for i in range(n) if rp[i] == path[-1]]
        bonus = int(rng.choice(kids)) if kids and rng.random() < 0.5 else int(rng.integers(0, V))
        pn = [rm[i] for i in path]
        cm, nc, kp, nk = _ia(64), C.c_int(), _ia(64), C.c_int()
        r = dt.dt_reroot(h, (C.c_int * len(pn))(*pn), len(pn), bonus, cm, C.byref(nc), kp, C.byref(nk))
        rc, rk, rn = ref.reroot(pn, bonus)
        assert (r, list(cm[:nc.value]), list(kp[:nk.value])) == (rn, rc, rk)
        assert _nodes(dt, h) == _ref_nodes(ref) and dt.dt_troot(h) == ref.troot
        assert dt.dt_n_slots(h) == ref.n_slots
    dt.dt_free(h)


# ---------------------------------------------------------------- Alg. 1 end to end (reference)
def _toy_models(V, agree, seed):
    """A deterministic toy target (greedy next token = hash of the last two
    tokens) and a toy draft that proposes the target's token first with
    probability `agree` (else a different one), with log-probabilities."""
    rng = np.random.default_rng(seed)
    table = rng.integers(0, V, size=(V, V))
    flip = rng.random((V, V)) < agree

    def target_next(seq):
        a, b = (seq[-2], seq[-1]) if len(seq) > 1 else (0, seq[-1])
        return int(table[a, b])

    def draft_topk(seq, K):
        a, b = (seq[-2], seq[-1]) if len(seq) > 1 else (0, seq[-1])
        t = int(table[a, b])
        first = t if flip[a, b] else (t + 1) % V
        toks = [first] + [(first + 7 * (i + 1)) % V for i in range(K - 1)]
        lps = [-0.2 - 0.5 * i for i in range(K)]
        return toks, lps
    return target_next, draft_topk


@pytest.mark.parametrize("agree,d", [(0.9, 2), (0.5, 1), (0.0, 3)])
def test_ref_alg1_loop_emits_target_greedy(agree, d):
    """Alg. 1 run on the reference tree with toy models: whatever
    the draft proposes, the emitted tokens are the target's greedy sequence
    (S:453); the committed draft prefix is always a prefix of the target's
    committed tokens; commit slots form a root-anchored chain and kept slots
    ascend (the device re-root's contract)."""
    V, K, w, bs = 40, 4, 4, 6
    target_next, draft_topk = _toy_models(V, agree, seed=int(agree * 10) + d)
    root = 3
    ref = [root]
    for _ in range(60):
        ref.append(target_next(ref))
    tree = DraftTreeRef(root, max_slots=48)
    draft_prefix = []            # tokens whose draft K/V is committed
    emitted = [root]
    accepted_total = steps = 0

    def seq_of(node):
        toks = [tree.nodes[j]["token"] for j in tree.ancestors_or_self(node)][::-1]
        return draft_prefix + toks

    def expand():
        sel = tree.select(w)
        tree.computed(sel)
        for n in sel:
            toks, lps = draft_topk(seq_of(n), K)
            tree.add_children(n, toks, lps)
        return len(sel)

    while len(emitted) < 50:
        for _ in range(d):
            expand()
        while tree.tree_size() < bs:
            if not expand():
                break
        toks, pars, chosen = tree.subgraph(bs)
        # target: greedy acceptance on the subgraph (a11)
        base = emitted[:]          # committed target tokens + the root (= emitted so far)
        path, cur = [0], 0
        while True:
            nxt_tok = target_next(base + [toks[i] for i in path[1:]])
            kids = [i for i in range(len(toks)) if pars[i] == cur and toks[i] == nxt_tok]
            if not kids:
                bonus = nxt_tok
                break
            cur = kids[0]
            path.append(cur)
        emitted += [toks[i] for i in path[1:]] + [bonus]
        accepted_total += len(path) - 1
        steps += 1
        nodes = [chosen[i] for i in path]
        commit, keep, n = tree.reroot(nodes, bonus)
        assert keep == sorted(keep) and len(set(commit) | set(keep)) == len(commit) + len(keep)
        # the committed draft tokens are the verified ones, in order
        draft_prefix = emitted[:len(draft_prefix) + n]
        assert len(draft_prefix) <= len(emitted) - 1          # the target's root is never committed by the draft
    assert emitted[:50] == ref[:50]
    if agree >= 0.9:
        assert accepted_total / steps > 0.8                   # a good draft gets tokens accepted
