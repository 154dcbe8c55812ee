"""Counter-based synthetic input generator.

Every element of every canonical tensor is a pure function of
(seed, tensor id, flat element index) through a SplitMix64-style finaliser, so
any slice of a 70B-shaped model can be regenerated on demand (by this module
on the host, or by csrc/synth.cu on the device) without materialising the
rest.  All float conversions are done with exactly-rounded fp32 operations in
a fixed order, so the host and device generators agree bit for bit.

Nothing here implements the method: the oracle dequantises, normalises,
attends and accepts; this module only produces q/z/s nibbles, bf16 bit
patterns, token trees and token ids.

Canonical formats (what ss_load_weights takes, see include/swiftspec.h):
  linear weight  W: y = x @ W, K = in-features, N = out-features
     qweight uint8 [K][N]   values 0..15 (one nibble per byte)
     qzeros  uint8 [K/128][N] values 0..15
     scales  uint16 [K/128][N] bf16 bit patterns
  embed, lm_head  uint16 [V][h] bf16 bits
  norm gains      uint16 [h]    bf16 bits
  prefix K/V      uint16 [L][Hkv][d] bf16 bits (keys are post-RoPE, as cached)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, asdict

import numpy as np

__all__ = [
    "ModelCfg", "CONFIGS", "KIND", "SUB", "tensor_id", "stream_key", "hash_u64",
    "gen_linear", "gen_embed", "gen_lm_head", "gen_norm", "gen_prefix_kv",
    "gen_model", "bf16_bits_to_f32", "f32_to_bf16_bits", "scale_const",
    "lm_scale_const", "tree_chain", "tree_star", "tree_paperlike", "tree_random",
    "tree_from_parents_tokens", "FIG4_TREE",
]

GROUP = 128
MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB
C3 = 0xD1B54A32D192ED03


@dataclass(frozen=True)
class ModelCfg:
    """Llama-style shapes (public Llama3 configs, reading R1)."""
    name: str
    n_layers: int
    hidden: int
    intermediate: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 500000.0

    def as_dict(self):
        return asdict(self)


CONFIGS = {
    # BASELINE.json configs[0]: the oracle-sized parity case.
    "tiny": ModelCfg("tiny", 2, 256, 1024, 4, 2, 64, 4096),
    # small shape whose O / down K-shards stay multiples of 256 at TP 2 and 4
    # (the fake-peer tensor-parallel parity tests)
    "small-tp": ModelCfg("small-tp", 2, 1024, 2048, 16, 4, 64, 4096),
    "llama3-1b": ModelCfg("llama3-1b", 16, 2048, 8192, 32, 8, 64, 128256),
    "llama3-3b": ModelCfg("llama3-3b", 28, 3072, 8192, 24, 8, 128, 128256),
    "llama3-8b": ModelCfg("llama3-8b", 32, 4096, 14336, 32, 8, 128, 128256),
    "llama3-70b": ModelCfg("llama3-70b", 80, 8192, 28672, 64, 8, 128, 128256),
}

# Tensor kinds -- identical numbering to ss_weight_kind in include/swiftspec.h.
KIND = dict(EMBED=0, ATTN_NORM=1, WQ=2, WK=3, WV=4, WO=5, MLP_NORM=6, WGATE=7,
            WUP=8, WDOWN=9, FINAL_NORM=10, LM_HEAD=11, KCACHE=12, VCACHE=13)
SUB = dict(QWEIGHT=0, QZEROS=1, SCALES=2, DENSE=0)


def tensor_id(layer: int, kind: int, sub: int = 0) -> int:
    """Stream id of one canonical tensor; layer = -1 for model-global tensors."""
    return ((layer + 1) << 16) | (kind << 4) | sub


def _fmix64_int(z: int) -> int:
    z &= MASK64
    z ^= z >> 30
    z = (z * C1) & MASK64
    z ^= z >> 27
    z = (z * C2) & MASK64
    z ^= z >> 31
    return z


def stream_key(seed: int, tid: int) -> int:
    return _fmix64_int((_fmix64_int(seed * GOLDEN + 1) ^ ((tid * C3) & MASK64)))


def hash_u64(key: int, idx: np.ndarray) -> np.ndarray:
    """h(key, i) = fmix64(key + (i + 1) * GOLDEN) on uint64 arrays (wrapping)."""
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN)
        z ^= z >> np.uint64(30)
        z *= np.uint64(C1)
        z ^= z >> np.uint64(27)
        z *= np.uint64(C2)
        z ^= z >> np.uint64(31)
    return z


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (uint16)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def scale_const(K: int) -> np.float32:
    """c = fp32(1 / (4.64 sqrt(K))): weight std ~ 1/sqrt(K) (E(q-z)^2 = 21.5)."""
    return np.float32(1.0 / (4.64 * math.sqrt(K)))


def lm_scale_const(h: int) -> np.float32:
    """LM head element scale alpha/sqrt(h), alpha = 4 -> logit std ~ 4."""
    return np.float32(4.0 / math.sqrt(h))


_SQRT3 = np.float32(math.sqrt(3.0))
_INV16 = np.float32(1.0 / 65536.0)


def _approx_normal(hv: np.ndarray) -> np.ndarray:
    """Irwin-Hall(4) sum of four exact 16-bit uniforms, centred and scaled to unit std.

    Every fp32 operation is exact except the final multiply by fp32(sqrt 3),
    which is correctly rounded on both host and device."""
    u0 = (hv & np.uint64(0xFFFF)).astype(np.float32) * _INV16
    u1 = ((hv >> np.uint64(16)) & np.uint64(0xFFFF)).astype(np.float32) * _INV16
    u2 = ((hv >> np.uint64(32)) & np.uint64(0xFFFF)).astype(np.float32) * _INV16
    u3 = ((hv >> np.uint64(48)) & np.uint64(0xFFFF)).astype(np.float32) * _INV16
    s = ((u0 + u1) + u2) + u3
    return (s - np.float32(2.0)) * _SQRT3


def _idx(n0: int, n1: int) -> np.ndarray:
    return np.arange(n0, n1, dtype=np.uint64)


def gen_linear(seed: int, layer: int, kind: int, K: int, N: int):
    """Canonical int4 AWQ tensor (qweight, qzeros, scales) for W[K][N].

    q ~ U{0..15}; z ~ U{6..9}; s = bf16(u * c), u ~ U[0.5, 1.5) on a 2^-23 grid."""
    assert K % GROUP == 0
    G = K // GROUP
    kq = stream_key(seed, tensor_id(layer, kind, SUB["QWEIGHT"]))
    q = np.empty(K * N, dtype=np.uint8)
    step = 1 << 24
    for a in range(0, K * N, step):
        b = min(K * N, a + step)
        q[a:b] = (hash_u64(kq, _idx(a, b)) & np.uint64(15)).astype(np.uint8)
    kz = stream_key(seed, tensor_id(layer, kind, SUB["QZEROS"]))
    z = (np.uint64(6) + (hash_u64(kz, _idx(0, G * N)) & np.uint64(3))).astype(np.uint8)
    ks = stream_key(seed, tensor_id(layer, kind, SUB["SCALES"]))
    hs = hash_u64(ks, _idx(0, G * N))
    u = ((hs >> np.uint64(41)) + np.uint64(1 << 22)).astype(np.float32) * np.float32(2.0 ** -23)
    s = f32_to_bf16_bits(u * scale_const(K))
    return q.reshape(K, N), z.reshape(G, N), s.reshape(G, N)


def gen_embed(seed: int, V: int, h: int, rows=None) -> np.ndarray:
    """bf16 bits [V][h] (or only `rows`), N(0,1)-like."""
    key = stream_key(seed, tensor_id(-1, KIND["EMBED"]))
    rows = np.arange(V) if rows is None else np.asarray(rows)
    idx = (rows.astype(np.uint64)[:, None] * np.uint64(h) + np.arange(h, dtype=np.uint64)[None, :])
    return f32_to_bf16_bits(_approx_normal(hash_u64(key, idx)))


def gen_lm_head(seed: int, V: int, h: int, rows=None) -> np.ndarray:
    """bf16 bits [V][h] (or only `rows`), N(0,1) * 4/sqrt(h)."""
    key = stream_key(seed, tensor_id(-1, KIND["LM_HEAD"]))
    rows = np.arange(V) if rows is None else np.asarray(rows)
    out = np.empty((len(rows), h), dtype=np.uint16)
    c = lm_scale_const(h)
    step = max(1, (1 << 23) // h)
    for a in range(0, len(rows), step):
        r = rows[a:a + step].astype(np.uint64)
        idx = r[:, None] * np.uint64(h) + np.arange(h, dtype=np.uint64)[None, :]
        out[a:a + step] = f32_to_bf16_bits(_approx_normal(hash_u64(key, idx)) * c)
    return out


def gen_norm(seed: int, layer: int, kind: int, h: int) -> np.ndarray:
    """bf16 bits [h]: 1 + 0.1 * N(0,1)-like."""
    key = stream_key(seed, tensor_id(layer, kind))
    t = _approx_normal(hash_u64(key, _idx(0, h))) * np.float32(0.1)
    return f32_to_bf16_bits(np.float32(1.0) + t)


def gen_prefix_kv(seed: int, layer: int, L: int, Hkv: int, d: int, pos0: int = 0):
    """Synthetic committed cache rows [pos0, pos0+L) as bf16 bits [L][Hkv][d] (K, V)."""
    out = []
    for kind in (KIND["KCACHE"], KIND["VCACHE"]):
        key = stream_key(seed, tensor_id(layer, kind))
        idx = _idx(pos0 * Hkv * d, (pos0 + L) * Hkv * d)
        out.append(f32_to_bf16_bits(_approx_normal(hash_u64(key, idx))).reshape(L, Hkv, d))
    return out[0], out[1]


def gen_model(cfg: ModelCfg, seed: int = 0, with_lm_head: bool = True):
    """Whole canonical model as nested dicts (host memory; small configs only)."""
    h, I, d = cfg.hidden, cfg.intermediate, cfg.head_dim
    layers = []
    for l in range(cfg.n_layers):
        lw = {
            "attn_norm": gen_norm(seed, l, KIND["ATTN_NORM"], h),
            "wq": gen_linear(seed, l, KIND["WQ"], h, cfg.n_heads * d),
            "wk": gen_linear(seed, l, KIND["WK"], h, cfg.n_kv_heads * d),
            "wv": gen_linear(seed, l, KIND["WV"], h, cfg.n_kv_heads * d),
            "wo": gen_linear(seed, l, KIND["WO"], cfg.n_heads * d, h),
            "mlp_norm": gen_norm(seed, l, KIND["MLP_NORM"], h),
            "wgate": gen_linear(seed, l, KIND["WGATE"], h, I),
            "wup": gen_linear(seed, l, KIND["WUP"], h, I),
            "wdown": gen_linear(seed, l, KIND["WDOWN"], I, h),
        }
        layers.append(lw)
    m = {"layers": layers, "embed": gen_embed(seed, cfg.vocab, h),
         "final_norm": gen_norm(seed, -1, KIND["FINAL_NORM"], h)}
    if with_lm_head:
        m["lm_head"] = gen_lm_head(seed, cfg.vocab, h)
    return m


# ----------------------------------------------------------------------------
# Token trees.  A tree is (tokens int32[T], parents int32[T]) with parents[0]
# = -1 and parents[i] < i (topological, root first: SPEC S:45-47).
# ----------------------------------------------------------------------------

# Fig. 4 input_1: (t1, t2, t3, t5) with t2, t3 children of t1 and t5 a
# child of t3 (structure from SPEC S:103).  Token ids are the subscripts.
FIG4_TREE = (np.array([1, 2, 3, 5], dtype=np.int32), np.array([-1, 0, 0, 2], dtype=np.int32))


def tree_from_parents_tokens(tokens, parents):
    return np.asarray(tokens, dtype=np.int32), np.asarray(parents, dtype=np.int32)


def tree_chain(T: int, V: int, rng: np.random.Generator):
    return rng.integers(0, V, T).astype(np.int32), np.arange(-1, T - 1, dtype=np.int32)


def tree_star(T: int, V: int, rng: np.random.Generator):
    p = np.zeros(T, dtype=np.int32)
    p[0] = -1
    return rng.integers(0, V, T).astype(np.int32), p


def tree_random(T: int, V: int, rng: np.random.Generator):
    p = np.array([-1] + [int(rng.integers(0, i)) for i in range(1, T)], dtype=np.int32)
    return rng.integers(0, V, T).astype(np.int32), p


def tree_paperlike(T: int, V: int, rng: np.random.Generator, max_depth: int = 7, branch: int = 2):
    """Depth <= 7, ~2 children per expanded node, nodes added
    best-first by a random path weight (the draft's max-likelihood order)."""
    parents = [-1]
    depth = [0]
    nchild = [0]
    weight = [0.0]
    frontier = [0]
    while len(parents) < T:
        cand = [i for i in frontier if depth[i] < max_depth and nchild[i] < branch]
        if not cand:
            cand = [i for i in range(len(parents)) if depth[i] < max_depth]
        i = max(cand, key=lambda j: weight[j])
        parents.append(i)
        depth.append(depth[i] + 1)
        nchild[i] += 1
        nchild.append(0)
        weight.append(weight[i] + float(np.log(rng.uniform(0.05, 1.0))))
        frontier.append(len(parents) - 1)
    tokens = rng.integers(0, V, T).astype(np.int32)
    # siblings carry distinct tokens
    for i in range(1, T):
        sib = [j for j in range(1, i) if parents[j] == parents[i]]
        while any(tokens[j] == tokens[i] for j in sib):
            tokens[i] = int(rng.integers(0, V))
    return tokens, np.array(parents, dtype=np.int32)
