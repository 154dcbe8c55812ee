"""CPU tests of the C-ABI's host-side error detection (include/swiftspec.h
"Errors"): the checks and call-order state machine of
csrc/host_logic.h -- the header shard.cu runs before any launch -- compiled
with g++ into a small harness (tests/native/host_logic_harness.cpp).  Every
host-detected status code is exercised: SS_EINVAL (tree shape S:45-47, chain,
rows never written), SS_ESTATE (weights / peers missing, commit without a
verify, two verifies without a commit), SS_ECAPACITY (L + T > max_ctx,
S:201-209).  SS_ECUDA is exercised through the real library (no device
here); SS_ETIMEOUT / SS_ECONSISTENCY are device-side (tests/test_gpu_errors.py)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OK, EINVAL, ECAPACITY, ECONSISTENCY, ECUDA, ETIMEOUT, ESTATE = 0, -1, -2, -3, -4, -5, -6


@pytest.fixture(scope="module")
def hl(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("hl") / "libhl.so")
    src = os.path.join(ROOT, "tests", "native", "host_logic_harness.cpp")
    subprocess.run(["g++", "-O1", "-std=c++17", "-shared", "-fPIC", "-I" + os.path.join(ROOT, "include"),
                    src, "-o", so], check=True)
    L = C.CDLL(so)
    vp, i32 = C.c_void_p, C.c_int
    for n, res, args in [("hl_new", vp, [i32, i32, i32]), ("hl_free", None, [vp]),
                         ("hl_set", None, [vp, i32, i32, i32, i32]),
                         ("hl_check_tree", i32, [vp, vp, vp, i32]), ("hl_check_verify", i32, [vp, i32]),
                         ("hl_check_commit", i32, [vp, vp, i32]), ("hl_check_set_len", i32, [vp, i32]),
                         ("hl_on_verify", None, [vp, i32, vp, i32]), ("hl_on_commit", None, [vp, i32]),
                         ("hl_on_set_len", None, [vp, i32]), ("hl_L", i32, [vp]), ("hl_have_verify", i32, [vp]),
                         ("hl_max_written", i32, [vp]), ("hl_msg", C.c_char_p, []),
                         ("hl_check_extend", i32, [vp, vp, vp, i32, i32]),
                         ("hl_on_extend", None, [vp, i32, i32, vp]), ("hl_last_T", i32, [vp]),
                         ("hl_check_reroot", i32, [vp, vp, i32, vp, i32]),
                         ("hl_on_reroot", None, [vp, vp, i32, vp, i32])]:
        f = getattr(L, n)
        f.restype = res
        f.argtypes = args
    return L


def _a(x):
    a = np.ascontiguousarray(x, dtype=np.int32)
    return a, a.ctypes.data_as(C.c_void_p)


@pytest.fixture
def st(hl):
    p = hl.hl_new(256, 16, 4096)
    hl.hl_set(p, 1, 1, 64, 64)
    yield p
    hl.hl_free(p)


@pytest.mark.parametrize("tokens,parents,T", [
    ([1, 2], [0, 0], 2),           # root's parent must be -1
    ([1, 2, 3], [-1, 0, 2], 3),    # parents[i] < i (topological)
    ([1, 2, 3], [-1, 0, -1], 3),   # second root
    ([1, 4096], [-1, 0], 2),       # token out of vocab
    ([-1, 2], [-1, 0], 2),         # negative token
    ([1] * 17, [-1] + [0] * 16, 17),  # T > max_tree
    ([1], [-1], 0),                # T < 1
])
def test_einval_tree(hl, st, tokens, parents, T):
    (t, tp), (p, pp) = _a(tokens), _a(parents)
    assert hl.hl_check_tree(st, tp, pp, T) == EINVAL
    assert hl.hl_msg()


def test_valid_trees_pass(hl, st):
    for tokens, parents in [([5], [-1]), ([1, 2, 3, 5], [-1, 0, 0, 2]), (list(range(16)), list(range(-1, 15)))]:
        (t, tp), (p, pp) = _a(tokens), _a(parents)
        assert hl.hl_check_tree(st, tp, pp, len(tokens)) == OK


def test_estate_weights_and_peers(hl, st):
    hl.hl_set(st, 0, 1, 64, 64)
    assert hl.hl_check_verify(st, 8) == ESTATE and b"weights" in hl.hl_msg()
    hl.hl_set(st, 1, 0, 64, 64)
    assert hl.hl_check_verify(st, 8) == ESTATE and b"peers" in hl.hl_msg()


def test_estate_commit_without_verify_and_double_verify(hl, st):
    acc, ap = _a([0])
    assert hl.hl_check_commit(st, ap, 1) == ESTATE
    par, pp = _a([-1, 0, 0, 2])
    assert hl.hl_check_verify(st, 4) == OK
    hl.hl_on_verify(st, 4, pp, 0)
    assert hl.hl_have_verify(st) == 1
    assert hl.hl_check_verify(st, 4) == ESTATE and b"pending" in hl.hl_msg()   # two verifies, no commit
    ch, chp = _a([0, 2, 3])
    assert hl.hl_check_commit(st, chp, 3) == OK
    hl.hl_on_commit(st, 3)
    assert hl.hl_L(st) == 67 and hl.hl_have_verify(st) == 0
    assert hl.hl_check_commit(st, chp, 3) == ESTATE                            # no second commit
    assert hl.hl_check_verify(st, 4) == OK


def test_auto_commit_leaves_nothing_pending(hl, st):
    par, pp = _a([-1, 0])
    hl.hl_on_verify(st, 2, pp, 1)
    assert hl.hl_have_verify(st) == 0 and hl.hl_check_verify(st, 2) == OK


def test_set_len_discards_pending_verify(hl, st):
    par, pp = _a([-1, 0])
    hl.hl_on_verify(st, 2, pp, 0)
    assert hl.hl_check_set_len(st, 64) == OK
    hl.hl_on_set_len(st, 64)
    assert hl.hl_have_verify(st) == 0 and hl.hl_check_verify(st, 2) == OK


@pytest.mark.parametrize("chain,n", [([0, 1, 3], 3), ([1], 1), ([0, 2], 2), ([0, 1, 1], 3), ([0], 0), ([0] * 5, 5)])
def test_einval_commit_chain(hl, st, chain, n):
    # tree: 0 -> 1 -> {2, 3}; the root-anchored chains are [0], [0, 1], [0, 1, 2], [0, 1, 3]
    par, pp = _a([-1, 0, 1, 1])
    hl.hl_on_verify(st, 4, pp, 0)
    ch, chp = _a(chain + [0] * 4)
    r = hl.hl_check_commit(st, chp, n)
    if chain[:n] in ([0, 1, 3], [0, 1, 2]) and n == 3:
        assert r == OK
    else:
        assert r == EINVAL, (chain, n)


def test_ecapacity(hl, st):
    hl.hl_set(st, 1, 1, 256 - 8, 256 - 8)
    assert hl.hl_check_verify(st, 8) == OK
    assert hl.hl_check_verify(st, 9) == ECAPACITY
    assert hl.hl_check_set_len(st, 256 - 15) == ECAPACITY   # L + max_tree > max_ctx


def test_set_len_cannot_grow_over_unwritten_rows(hl, st):
    assert hl.hl_check_set_len(st, 32) == OK        # truncation
    assert hl.hl_check_set_len(st, 65) == EINVAL    # rows 64.. never written
    par, pp = _a([-1, 0, 1])
    hl.hl_on_verify(st, 3, pp, 0)                    # tree rows [64, 67) written
    assert hl.hl_max_written(st) == 67
    hl.hl_on_set_len(st, 64)
    assert hl.hl_check_set_len(st, 67) == OK         # chain prefill over written tree rows


def test_ecuda_without_device():
    """The real library: a valid shape on a host without a usable GPU fails with SS_ECUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2506_11309_b200 as pkg
    from paper_2506_11309_b200 import swiftspec as ssp
    import synth
    c = synth.CONFIGS["tiny"]
    cfg = ssp.ModelCfgC(c.n_layers, c.hidden, c.intermediate, c.n_heads, c.n_kv_heads, c.head_dim, c.vocab,
                        128, 256, 16, 1e-5, 5e5)
    h = C.c_void_p()
    assert pkg.lib().ss_init_shard(C.byref(cfg), 0, 1, 0, C.byref(h)) == ECUDA
    assert not h.value and pkg.lib().ss_last_error(None)


# ---- non-square forward (ss_extend_tree)
def test_extend_call_order_and_growth(hl, st):
    t, tp = _a([5, 6, 7, 8])
    par, pp = _a([0, 1, 1, 3])
    assert hl.hl_check_extend(st, tp, pp, 2, 4) == ESTATE        # nothing pending
    root, rp = _a([-1, 0])
    assert hl.hl_check_extend(st, tp, rp, 0, 2) == OK             # T0 = 0: a square verify
    hl.hl_on_verify(st, 2, rp, 0)
    assert hl.hl_check_extend(st, tp, rp, 0, 2) == ESTATE         # T0 = 0 while pending
    assert hl.hl_check_extend(st, tp, pp, 3, 4) == ESTATE         # T0 beyond the pending tree
    assert hl.hl_check_extend(st, tp, pp, 2, 4) == OK
    hl.hl_on_extend(st, 2, 4, pp)
    assert hl.hl_last_T(st) == 6 and hl.hl_have_verify(st) == 1 and hl.hl_max_written(st) == 70
    # the grown tree's chains commit: 0 -> 1 -> 3 -> 5 (nodes 3, 5 added by the extension)
    ch, chp = _a([0, 1, 3, 5])
    assert hl.hl_check_commit(st, chp, 4) == OK
    bad, bp = _a([0, 1, 4, 5])   # 5's parent is 3
    assert hl.hl_check_commit(st, bp, 4) == EINVAL


@pytest.mark.parametrize("T0,w,parents,tokens,code", [
    (2, 1, [2], [1], EINVAL),          # parent must be < T0 + i
    (2, 2, [0, 3], [1, 1], EINVAL),    # second new node's parent is itself
    (2, 1, [-1], [1], EINVAL),         # only node 0 is a root
    (2, 1, [0], [4096], EINVAL),       # token out of vocab
    (2, 0, [0], [1], EINVAL),          # w < 1
    (2, 33, [0] * 33, [1] * 33, EINVAL),  # w > 32
    (10, 7, [0] * 7, [1] * 7, EINVAL),    # T0 + w > max_tree (16)
    (2, 2, [0, 2], [1, 1], OK),
])
def test_extend_einval(hl, st, T0, w, parents, tokens, code):
    root, rp = _a([-1, 0] + [0] * 14)
    hl.hl_on_verify(st, 16, rp, 0)
    t, tp = _a(tokens)
    p, pp = _a(parents)
    assert hl.hl_check_extend(st, tp, pp, T0, w) == code


def test_extend_ecapacity(hl, st):
    root, rp = _a([-1, 0, 1, 2])
    hl.hl_set(st, 1, 1, 250, 250)
    hl.hl_on_verify(st, 4, rp, 0)
    t, tp = _a([1, 1, 1])
    p, pp = _a([3, 4, 5])
    assert hl.hl_check_extend(st, tp, pp, 4, 3) == ECAPACITY       # 250 + 4 + 3 > max_ctx 256
    assert hl.hl_check_extend(st, tp, pp, 4, 2) == OK              # 250 + 4 + 2 = 256 fits


# ---- re-root with KV reorganisation (ss_reroot)
def test_reroot_checks_and_reindex(hl, st):
    par, pp = _a([-1, 0, 1, 1, 2, 3, 2, 4])   # 0 -> 1 -> {2, 3}; 2 -> {4, 6}; 3 -> 5; 4 -> 7
    path, p_ = _a([0, 1])
    keep, k_ = _a([2, 4, 6, 7])
    assert hl.hl_check_reroot(st, p_, 2, k_, 4) == ESTATE         # nothing pending
    hl.hl_on_verify(st, 8, pp, 0)
    for pth, kp in [([0, 2], []), ([0], [2]), ([0, 1], [3, 2]), ([0, 1], [1]), ([], [1]), ([], [])]:
        a, ap = _a(pth + [0])
        b, bp = _a(kp + [0])
        assert hl.hl_check_reroot(st, ap, len(pth), bp, len(kp)) == EINVAL, (pth, kp)
    assert hl.hl_check_reroot(st, p_, 2, k_, 4) == OK
    hl.hl_on_reroot(st, p_, 2, k_, 4)
    assert hl.hl_L(st) == 66 and hl.hl_have_verify(st) == 1 and hl.hl_last_T(st) == 4
    # the kept tree is re-indexed: its chain 0 -> 1 -> 3 commits next
    ch, chp = _a([0, 1, 3])
    assert hl.hl_check_commit(st, chp, 3) == OK
    # n = m = 0 is refused; keep only (n = 0) must start at the root
    z, zp = _a([0, 3])
    assert hl.hl_check_reroot(st, None, 0, zp, 2) == EINVAL        # re-indexed: 3's parent is 1, not kept
    z, zp = _a([0, 1])
    assert hl.hl_check_reroot(st, None, 0, zp, 2) == OK            # truncate to nodes 0, 1
    hl.hl_on_reroot(st, None, 0, zp, 2)
    assert hl.hl_L(st) == 66 and hl.hl_last_T(st) == 2
    assert hl.hl_check_reroot(st, None, 0, None, 0) == EINVAL
