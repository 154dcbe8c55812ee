"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and rejects bad shapes before touching a GPU."""
import ctypes as C
import os
import re

import pytest

import paper_2506_11309_b200 as pkg
from paper_2506_11309_b200 import swiftspec as ssp
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "swiftspec.h")).read()
    return sorted(set(re.findall(r"^\s*(?:ss_status|int32_t|uint64_t|const char\*|void\*)\s+(ss_[a-z_]+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    L = pkg.lib()
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
    assert sorted(pkg.EXPORTS) == names


def test_lib_is_sm100a_and_static_cudart():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", pkg.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcudart" not in ldd


def _cfg(**kw):
    c = synth.CONFIGS["tiny"]
    d = dict(n_layers=c.n_layers, hidden=c.hidden, intermediate=c.intermediate, n_heads=c.n_heads,
             n_kv_heads=c.n_kv_heads, head_dim=c.head_dim, vocab=c.vocab, group_size=128, max_ctx=256,
             max_tree=64, rms_eps=1e-5, rope_theta=5e5)
    d.update(kw)
    return ssp.ModelCfgC(**d)


@pytest.mark.parametrize("bad", [dict(group_size=64), dict(head_dim=96), dict(hidden=300),
                                 dict(max_tree=65), dict(max_tree=0), dict(n_kv_heads=3)])
def test_init_rejects_bad_shapes(bad):
    h = C.c_void_p()
    r = pkg.lib().ss_init_shard(C.byref(_cfg(**bad)), 0, 1, 0, C.byref(h))
    assert r == -1 and not h.value
    assert pkg.lib().ss_last_error(None)


@pytest.mark.parametrize("rank,size", [(0, 3), (2, 2), (-1, 1)])
def test_init_rejects_bad_tp(rank, size):
    h = C.c_void_p()
    assert pkg.lib().ss_init_shard(C.byref(_cfg()), rank, size, 0, C.byref(h)) == -1


def test_null_args():
    L = pkg.lib()
    assert L.ss_init_shard(None, 0, 1, 0, None) == -1
    assert L.ss_verify_tree(None, None, None, 1, None, None, None) == -1
    assert L.ss_commit_kv(None, None, 1, None) == -1
    assert L.ss_committed_len(None) == -1
    assert L.ss_import_loopback(None) == -1
    assert L.ss_destroy(None) == 0
