"""Fast (C) column-chunk generators, bit-identical to synth/generators.py.

The streamed oracle of the 70B / 8B parity tests regenerates every layer's
weights on the host (~0.86 G int4 values per 70B layer); the NumPy generator
would take minutes per layer.  synth/csynth.c implements the same element
functions; this module builds it with gcc on first use (or from
__graft_entry__.build()) and wraps it.  Input generation only.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .generators import KIND, SUB, GROUP, stream_key, tensor_id, scale_const, lm_scale_const

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csynth.c")
SO = os.path.join(HERE, "_csynth.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        tmp = SO + f".{os.getpid()}.tmp"
        subprocess.run(["gcc", "-O3", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC", SRC, "-o", tmp],
                       check=True)
        os.replace(tmp, SO)
    return SO


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        u64, i64, vp, f32 = C.c_uint64, C.c_int64, C.c_void_p, C.c_float
        L.cs_gen_q_cols.argtypes = [u64, i64, i64, i64, i64, vp]
        L.cs_gen_z_cols.argtypes = [u64, i64, i64, i64, i64, vp]
        L.cs_gen_s_cols.argtypes = [u64, f32, i64, i64, i64, i64, vp]
        L.cs_gen_normal_bf16.argtypes = [u64, i64, i64, f32, vp]
        for f in (L.cs_gen_q_cols, L.cs_gen_z_cols, L.cs_gen_s_cols, L.cs_gen_normal_bf16):
            f.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def gen_linear_cols(seed: int, layer: int, kind: int, K: int, N: int, n0: int, n1: int):
    """Columns [n0, n1) of synth.gen_linear(seed, layer, kind, K, N): (q[K][w], z[G][w], s[G][w])."""
    L = lib()
    G = K // GROUP
    w = n1 - n0
    q = np.empty((K, w), dtype=np.uint8)
    z = np.empty((G, w), dtype=np.uint8)
    s = np.empty((G, w), dtype=np.uint16)
    L.cs_gen_q_cols(stream_key(seed, tensor_id(layer, kind, SUB["QWEIGHT"])), K, N, n0, n1, _p(q))
    L.cs_gen_z_cols(stream_key(seed, tensor_id(layer, kind, SUB["QZEROS"])), G, N, n0, n1, _p(z))
    L.cs_gen_s_cols(stream_key(seed, tensor_id(layer, kind, SUB["SCALES"])), float(scale_const(K)), G, N, n0, n1,
                    _p(s))
    return q, z, s


def _rows(key, rows, h, scale):
    L = lib()
    rows = np.atleast_1d(np.asarray(rows, dtype=np.int64))
    out = np.empty((len(rows), h), dtype=np.uint16)
    for i, r in enumerate(rows):
        L.cs_gen_normal_bf16(key, int(r) * h, h, scale, _p(out[i]))
    return out


def gen_embed_rows(seed: int, h: int, rows) -> np.ndarray:
    """Rows of synth.gen_embed(seed, V, h)."""
    return _rows(stream_key(seed, tensor_id(-1, KIND["EMBED"])), rows, h, 1.0)


def gen_lm_head_rows(seed: int, h: int, rows) -> np.ndarray:
    """Rows of synth.gen_lm_head(seed, V, h)."""
    return _rows(stream_key(seed, tensor_id(-1, KIND["LM_HEAD"])), rows, h, float(lm_scale_const(h)))


def gen_prefix_kv(seed: int, layer: int, L: int, Hkv: int, d: int):
    """synth.gen_prefix_kv(seed, layer, L, Hkv, d) (pos0 = 0)."""
    lb = lib()
    out = []
    for kind in (KIND["KCACHE"], KIND["VCACHE"]):
        a = np.empty(L * Hkv * d, dtype=np.uint16)
        lb.cs_gen_normal_bf16(stream_key(seed, tensor_id(layer, kind)), 0, a.size, 1.0, _p(a))
        out.append(a.reshape(L, Hkv, d))
    return out[0], out[1]
