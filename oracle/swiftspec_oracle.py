"""Plain, slow, float64 CPU oracle of the target model's tree-verification step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference), never
by the product.  Shares no code with the CUDA path.

Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n (SPEC
is used for interfaces and test ideas only).  Readings R1..R17 are listed in
DESIGN.md "Readings of the paper".

What the method computes: the target "runs batch
inferences to calculate the logits" of every node of the draft tree it
received, then "samples through the logits to generate the tokens one by one"
and sends the verified tokens back.  Batched tree verification is an exact
re-organisation of sequential greedy decoding, so this oracle is
the plain definition: an int4-AWQ (group 128) Llama decoder run in
float64 per tree node with the square ancestor mask, greedy
acceptance (R6) and KV compaction of the accepted path (BASELINE north_star).

Pins (tests/test_oracle.py): every function below is checked against
something other than itself -- brute force, closed forms, golden fixtures in
tests/golden/, HuggingFace's LlamaForCausalLM in float64 on a chain tree, the
sequential single-token decode of each root path, and the sharded sum.
Absolute logit values of a random-weight model have no printed value in the
paper; they are pinned by the HF-Llama equivalence and the decode invariants
(DESIGN.md "Parity").
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

__all__ = [
    "bf16_to_f64", "tree_meta", "dequant", "rmsnorm", "silu", "rope", "softmax",
    "attend_node", "argmax_lowest", "accept_walk", "OracleModel", "KVCache",
    "layer_forward", "verify", "commit", "forced_decode", "greedy_decode",
    "verify_sharded", "tp_padded_dims", "nonsquare_mask", "layer_forward_nonsquare",
    "forward_nonsquare",
]

GROUP = 128  # AWQ group size, P:501 ("4-bit AWQ quantization with a group size of 128")


def bf16_to_f64(bits) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float64, exact (BF16 embedding/LM head)."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# a0 -- tree metadata.  Square mask: "each token will only mask out the
# attention with those tokens that are not the ancestors within the current
# input".  Positions: reading R8, pos = L + depth.
# ---------------------------------------------------------------------------
def tree_meta(parents, L: int):
    """Returns (depth int[T], pos int[T], anc bool[T][T]); anc[i][j] = j is an
    ancestor-or-self of i.  Brute-force parent walk (no bit tricks)."""
    parents = [int(p) for p in parents]
    T = len(parents)
    if T < 1 or parents[0] != -1:
        raise ValueError("parents[0] must be -1 (root first, S:47)")
    for i in range(1, T):
        if not (0 <= parents[i] < i):
            raise ValueError("parents[i] must be in [0, i) (topological order, S:47)")
    depth = [0] * T
    anc = np.zeros((T, T), dtype=bool)
    for i in range(T):
        j = i
        d = 0
        while j != -1:
            anc[i, j] = True
            j = parents[j]
            d += 1
        depth[i] = d - 1
    depth = np.array(depth, dtype=np.int64)
    return depth, L + depth, anc


# ---------------------------------------------------------------------------
# Dequantisation: AWQ asymmetric uint4 with per-(group, column) zero and bf16
# scale (reading R3): W[k, n] = (q[k, n] - z[k // 128, n]) * s[k // 128, n].
# ---------------------------------------------------------------------------
def dequant(q, z, s_bits, group: int = GROUP) -> np.ndarray:
    """W[k, n] = (q[k, n] - z[k // group, n]) * s[k // group, n]: the rows of
    group g are rows [g*group, (g+1)*group), so W is formed group-major as
    (q[g, i, n] - z[g, n]) * s[g, n] over a [G][group][N] view (same values)."""
    q = np.asarray(q)
    z = np.asarray(z)
    K, N = q.shape
    if K % group:
        raise ValueError("K must be a multiple of the group size")
    G = K // group
    s = bf16_to_f64(s_bits)
    W = np.empty((G, group, N))
    np.subtract(q.reshape(G, group, N), z[:, None, :], out=W, dtype=np.float64)
    W *= s[:, None, :]
    return W.reshape(K, N)


def rmsnorm(x, g_bits, eps: float) -> np.ndarray:
    """Llama pre-norm (reading R5): x / sqrt(mean(x^2) + eps) * g, per row."""
    x = np.asarray(x, dtype=np.float64)
    g = bf16_to_f64(g_bits)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def silu(x):
    """SiLU, the sigma of the paper's garbled SwiGLU formula (reading R4)."""
    return x / (1.0 + np.exp(-x))


def rope(v, pos, theta: float) -> np.ndarray:
    """Rotary position embedding, rotate-half convention (reading R2), float64 angles.
    v: [..., d] for one position `pos` (scalar)."""
    v = np.asarray(v, dtype=np.float64)
    d = v.shape[-1]
    half = d // 2
    j = np.arange(half, dtype=np.float64)
    ang = float(pos) * theta ** (-2.0 * j / d)
    c, s = np.cos(ang), np.sin(ang)
    a, b = v[..., :half], v[..., half:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def softmax(x):
    x = np.asarray(x, dtype=np.float64)
    e = np.exp(x - np.max(x))
    return e / np.sum(e)


def attend_node(q, keys, values, n_kv_heads: int):
    """Causal/tree attention of ONE node: q [Hq][d]; keys/values [n_keys][Hkv][d]
    hold exactly the keys this node may see (reading R11: scale 1/sqrt(d),
    softmax, no soft-cap).  GQA: q head h reads kv head h // (Hq / Hkv)."""
    Hq, d = q.shape
    rep = Hq // n_kv_heads
    out = np.zeros((Hq, d))
    for h in range(Hq):
        kv = h // rep
        sc = keys[:, kv, :] @ q[h] / math.sqrt(d)
        p = softmax(sc)
        out[h] = p @ values[:, kv, :]
    return out


def argmax_lowest(row) -> int:
    """Greedy sampling (reading R6): linear scan, ties -> lowest token id."""
    best, bi = -np.inf, 0
    for i, v in enumerate(row):
        if v > best:
            best, bi = v, i
    return bi


def accept_walk(tokens, parents, argmax):
    """a11, greedy acceptance ("samples through the logits ... one by one";
    Fig. 4 walkthrough P:250).  Starting at the root, repeatedly take the
    target's greedy token at the current node; if a child of the current node
    carries it (lowest index on duplicates, reading R7), accept and descend.
    Returns (accepted node indices, root first; bonus token)."""
    T = len(tokens)
    cur = 0
    acc = [0]
    while True:
        t = int(argmax[cur])
        nxt = None
        for c in range(T):
            if parents[c] == cur and int(tokens[c]) == t:
                nxt = c
                break
        if nxt is None:
            return acc, t
        acc.append(nxt)
        cur = nxt


# ---------------------------------------------------------------------------
# Model containers.
# ---------------------------------------------------------------------------
def linear_streamed(x, cols, N: int, chunk: int = 1024, workers: int = 0) -> np.ndarray:
    """x @ W for a W whose canonical columns [n0, n1) come from cols(n0, n1) ->
    (q, z, s).  Each output column is the plain dot product x @ dequant(...)[:, n]
    (column j of x @ W depends only on column j of W), so W is never held whole:
    chunks of columns are generated, dequantised and multiplied in a thread pool
    (the 70B-shaped layers of the full-size parity tests: ~0.86 G weights each)."""
    from threadpoolctl import threadpool_limits
    out = np.empty((x.shape[0], N))

    def job(n0):
        n1 = min(N, n0 + chunk)
        q, z, s = cols(n0, n1)
        out[:, n0:n1] = x @ dequant(q, z, s)

    with threadpool_limits(limits=1), ThreadPoolExecutor(max_workers=workers or os.cpu_count()) as ex:
        list(ex.map(job, range(0, N, chunk)))
    return out


@dataclass
class OracleModel:
    """Canonical (quantised) weights from synth.gen_model; dequantised lazily.

    cols (optional): a streamed weight provider cols(layer, name, n0, n1) ->
    (q, z, s) of canonical columns [n0, n1) -- used when a whole model's dense
    weights would not fit in host memory (70B-shaped parity tests)."""
    cfg: object
    canon: dict
    cache_dense: bool = True
    cols: object = None

    def __post_init__(self):
        self._dense = {}

    def out_features(self, name: str) -> int:
        c = self.cfg
        return dict(wq=c.n_heads * c.head_dim, wk=c.n_kv_heads * c.head_dim, wv=c.n_kv_heads * c.head_dim,
                    wo=c.hidden, wgate=c.intermediate, wup=c.intermediate, wdown=c.hidden)[name]

    def matmul(self, layer: int, name: str, x) -> np.ndarray:
        """x @ W[layer][name] with W = dequant(q, z, s)."""
        if self.cols is not None:
            return linear_streamed(x, lambda n0, n1: self.cols(layer, name, n0, n1), self.out_features(name))
        return x @ self.w(layer, name)

    def w(self, layer: int, name: str) -> np.ndarray:
        key = (layer, name)
        if key in self._dense:
            return self._dense[key]
        q, z, s = self.canon["layers"][layer][name]
        W = dequant(q, z, s)
        if self.cache_dense:
            self._dense[key] = W
        return W

    def norm(self, layer: int, name: str):
        return self.canon["layers"][layer][name]

    def embed_rows(self, tokens) -> np.ndarray:
        return bf16_to_f64(self.canon["embed"][np.asarray(tokens)])

    def logits(self, xn: np.ndarray, chunk: int = 16384) -> np.ndarray:
        """logits = xn @ lm_head^T (bf16 LM head); vocab rows in chunks
        only to bound memory -- each logit is one plain dot product."""
        W = self.canon["lm_head"]
        V = W.shape[0]
        out = np.empty((xn.shape[0], V))
        for a in range(0, V, chunk):
            out[:, a:a + chunk] = xn @ bf16_to_f64(W[a:a + chunk]).T
        return out


class KVCache:
    """Committed cache per layer: K, V float64 [max_ctx][Hkv][d]; rows [0, L) valid."""

    def __init__(self, cfg, max_ctx: int):
        self.cfg = cfg
        self.K = [np.zeros((max_ctx, cfg.n_kv_heads, cfg.head_dim)) for _ in range(cfg.n_layers)]
        self.V = [np.zeros((max_ctx, cfg.n_kv_heads, cfg.head_dim)) for _ in range(cfg.n_layers)]
        self.L = 0

    def set_prefix(self, layer: int, k_bits, v_bits):
        L = k_bits.shape[0]
        self.K[layer][:L] = bf16_to_f64(k_bits)
        self.V[layer][:L] = bf16_to_f64(v_bits)

    def copy(self):
        c = KVCache.__new__(KVCache)
        c.cfg = self.cfg
        c.K = [k.copy() for k in self.K]
        c.V = [v.copy() for v in self.V]
        c.L = self.L
        return c


def layer_forward(cfg, model: OracleModel, layer: int, x, kv: KVCache, L: int, pos, anc):
    """One decoder layer over all T tree nodes (a2-a9), per node, float64.

    x [T][h] residual stream.  Returns (x', tree K [T][Hkv][d], tree V)."""
    T = x.shape[0]
    Hq, Hkv, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    xn = rmsnorm(x, model.norm(layer, "attn_norm"), cfg.rms_eps)          # a2
    q = model.matmul(layer, "wq", xn).reshape(T, Hq, d)                   # a3
    k = model.matmul(layer, "wk", xn).reshape(T, Hkv, d)
    v = model.matmul(layer, "wv", xn).reshape(T, Hkv, d)
    for i in range(T):                                                    # a4: RoPE at L + depth
        q[i] = rope(q[i], pos[i], cfg.rope_theta)
        k[i] = rope(k[i], pos[i], cfg.rope_theta)
    attn = np.zeros((T, Hq * d))
    Kp, Vp = kv.K[layer][:L], kv.V[layer][:L]
    for i in range(T):                                                    # a5: prefix + ancestors
        sel = np.nonzero(anc[i])[0]
        keys = np.concatenate([Kp, k[sel]], axis=0)
        vals = np.concatenate([Vp, v[sel]], axis=0)
        attn[i] = attend_node(q[i], keys, vals, Hkv).reshape(-1)
    x = x + model.matmul(layer, "wo", attn)                               # a6
    xn2 = rmsnorm(x, model.norm(layer, "mlp_norm"), cfg.rms_eps)          # a7
    hmid = silu(model.matmul(layer, "wgate", xn2)) * model.matmul(layer, "wup", xn2)  # a8
    x = x + model.matmul(layer, "wdown", hmid)                            # a9
    return x, k, v


def verify(cfg, model: OracleModel, kv: KVCache, tokens, parents, want_logits: bool = True):
    """One tree-verification step (a0-a11) against the committed cache kv (L = kv.L).

    Returns dict(logits [T][V], argmax [T], accepted, bonus, tree_k, tree_v,
    depth, pos, anc)."""
    tokens = np.asarray(tokens)
    L = kv.L
    depth, pos, anc = tree_meta(parents, L)                               # a0
    x = model.embed_rows(tokens)                                          # a1
    tk, tv = [], []
    for l in range(cfg.n_layers):
        x, k, v = layer_forward(cfg, model, l, x, kv, L, pos, anc)
        tk.append(k)
        tv.append(v)
    xn = rmsnorm(x, model.canon["final_norm"], cfg.rms_eps)              # a10
    logits = model.logits(xn)
    am = np.array([argmax_lowest(r) for r in logits], dtype=np.int64)
    acc, bonus = accept_walk(tokens, parents, am)                         # a11
    return dict(logits=logits if want_logits else None, argmax=am, accepted=acc,
                bonus=bonus, tree_k=tk, tree_v=tv, depth=depth, pos=pos, anc=anc,
                tokens=tokens, parents=np.asarray(parents))


# ---------------------------------------------------------------------------
# Non-square mask: "for the draft model ... with a
# current tree of size 6, and we want to calculate the logits of 4 probable
# leaves, then regarding the tree cache, we only calculate the attention of
# each leave with its ancestor on the tree (and also all the data that is in
# the prefix cache). In this case, we need a mask of at least size (4, 10)".
# The tree cache holds nodes [0, T0) whose K/V earlier calls computed (P:339
# "the KV states of the tree are stored right after the prefix"); the w leaves
# [T0, T0 + w) are computed now, each against the prefix, its cached ancestors
# and its new ancestors-or-self.
# ---------------------------------------------------------------------------
def nonsquare_mask(parents_all, T0: int, L: int):
    """Returns (pos int[w], mask bool[w][T0 + w]) of the leaves [T0, T0 + w) of
    the tree `parents_all` (every node, root first): mask[i][j] = node j is an
    ancestor-or-self of leaf T0 + i (brute-force parent walk)."""
    parents_all = [int(p) for p in parents_all]
    T = len(parents_all)
    if not (0 <= T0 < T):
        raise ValueError("need 0 <= T0 < T (at least one leaf)")
    depth, pos, anc = tree_meta(parents_all, L)
    return pos[T0:], anc[T0:, :]


def layer_forward_nonsquare(cfg, model: OracleModel, layer: int, x, kv: KVCache, L: int, pos, mask,
                            tree_k, tree_v):
    """One decoder layer over the w leaves only (a2-a9), float64.  x [w][h]:
    the leaves' residual streams; tree_k / tree_v [T0][Hkv][d]: this layer's
    cached tree K/V; mask [w][T0 + w] (nonsquare_mask).  Returns (x', leaf K
    [w][Hkv][d], leaf V)."""
    w = x.shape[0]
    Hq, Hkv, d = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    xn = rmsnorm(x, model.norm(layer, "attn_norm"), cfg.rms_eps)          # a2
    q = model.matmul(layer, "wq", xn).reshape(w, Hq, d)                   # a3
    k = model.matmul(layer, "wk", xn).reshape(w, Hkv, d)
    v = model.matmul(layer, "wv", xn).reshape(w, Hkv, d)
    for i in range(w):                                                    # a4: RoPE at L + depth
        q[i] = rope(q[i], pos[i], cfg.rope_theta)
        k[i] = rope(k[i], pos[i], cfg.rope_theta)
    Kt = np.concatenate([tree_k, k], axis=0)                              # tree cache + leaves
    Vt = np.concatenate([tree_v, v], axis=0)
    attn = np.zeros((w, Hq * d))
    Kp, Vp = kv.K[layer][:L], kv.V[layer][:L]
    for i in range(w):                                                    # a5: non-square mask row i
        sel = np.nonzero(mask[i])[0]
        keys = np.concatenate([Kp, Kt[sel]], axis=0)
        vals = np.concatenate([Vp, Vt[sel]], axis=0)
        attn[i] = attend_node(q[i], keys, vals, Hkv).reshape(-1)
    x = x + model.matmul(layer, "wo", attn)                               # a6
    xn2 = rmsnorm(x, model.norm(layer, "mlp_norm"), cfg.rms_eps)          # a7
    hmid = silu(model.matmul(layer, "wgate", xn2)) * model.matmul(layer, "wup", xn2)  # a8
    x = x + model.matmul(layer, "wdown", hmid)                            # a9
    return x, k, v


def forward_nonsquare(cfg, model: OracleModel, kv: KVCache, tree, tokens_new, parents_new,
                      want_logits: bool = True):
    """Forward of w new leaves on top of a tree cache (P:321 non-square mask).

    tree: None (empty cache, T0 = 0) or the dict a previous verify /
    forward_nonsquare returned for the same committed cache (tokens, parents,
    tree_k, tree_v, argmax of its T0 nodes).  parents_new[i] indexes the whole
    tree (< T0 + i; -1 only for node 0).  Returns the grown tree's dict:
    logits [w][V] of the leaves, argmax of all T0 + w nodes (the cached nodes'
    from `tree`), tree_k / tree_v of all nodes, pos / mask of the leaves, and
    the greedy accept walk (a11) over the whole grown tree."""
    L = kv.L
    T0 = 0 if tree is None else len(tree["tokens"])
    toks_all = np.concatenate([np.asarray(tree["tokens"] if tree else [], dtype=np.int64),
                               np.asarray(tokens_new, dtype=np.int64)])
    par_all = [int(p) for p in (list(tree["parents"]) if tree else [])] + [int(p) for p in parents_new]
    pos, mask = nonsquare_mask(par_all, T0, L)                            # a0 (leaves)
    x = model.embed_rows(np.asarray(tokens_new))                          # a1
    tk, tv = [], []
    for l in range(cfg.n_layers):
        ck = tree["tree_k"][l] if tree else np.zeros((0, cfg.n_kv_heads, cfg.head_dim))
        cv = tree["tree_v"][l] if tree else np.zeros((0, cfg.n_kv_heads, cfg.head_dim))
        x, k, v = layer_forward_nonsquare(cfg, model, l, x, kv, L, pos, mask, ck, cv)
        tk.append(np.concatenate([ck, k], axis=0))
        tv.append(np.concatenate([cv, v], axis=0))
    xn = rmsnorm(x, model.canon["final_norm"], cfg.rms_eps)              # a10
    logits = model.logits(xn)
    am_new = np.array([argmax_lowest(r) for r in logits], dtype=np.int64)
    am = np.concatenate([np.asarray(tree["argmax"] if tree else [], dtype=np.int64), am_new])
    acc, bonus = accept_walk(toks_all, par_all, am)                       # a11 over the grown tree
    return dict(logits=logits if want_logits else None, argmax=am, accepted=acc, bonus=bonus,
                tree_k=tk, tree_v=tv, tokens=toks_all, parents=np.array(par_all, dtype=np.int64),
                pos=pos, mask=mask)


def commit(kv: KVCache, res: dict, accepted) -> KVCache:
    """a12, KV compaction + commit: K/V[L + k] <- tree K/V[accepted[k]] for every
    layer; L += n (root + accepted nodes, never the bonus; reading R9)."""
    L = kv.L
    for l in range(len(kv.K)):
        for kk, node in enumerate(accepted):
            kv.K[l][L + kk] = res["tree_k"][l][node]
            kv.V[l][L + kk] = res["tree_v"][l][node]
    kv.L = L + len(accepted)
    return kv


def forced_decode(cfg, model, kv: KVCache, path_tokens):
    """Sequential mode: feed path_tokens one at a time (T = 1 trees), committing
    each.  Returns per-step logits [n][V]; kv is advanced in place."""
    out = []
    for t in path_tokens:
        r = verify(cfg, model, kv, [int(t)], [-1])
        out.append(r["logits"][0])
        commit(kv, r, [0])
    return np.array(out)


def greedy_decode(cfg, model, kv: KVCache, root: int, n_tokens: int):
    """Plain autoregressive greedy decoding from `root` (root not yet cached).
    Returns the n_tokens generated tokens; kv advanced by n_tokens rows."""
    toks = []
    cur = int(root)
    for _ in range(n_tokens):
        r = verify(cfg, model, kv, [cur], [-1], want_logits=True)
        nxt = int(r["argmax"][0])
        commit(kv, r, [0])
        toks.append(nxt)
        cur = nxt
    return toks


# ---------------------------------------------------------------------------
# Sharded mode (Megatron TP): each rank owns Hq/P q heads and
# Hkv/P kv heads (column-parallel QKV), the matching O rows (row-parallel),
# an I/P slice of gate/up/down, and a V/P vocab slice of the LM head.  The
# two all-reduces per layer are plain sums of the ranks' partials in rank
# order; argmax is taken over the concatenated vocab shards.
# ---------------------------------------------------------------------------
def tp_padded_dims(cfg, P: int):
    """Arbitrary tensor parallelism by zero padding (SURVEY A13 /
    NEXT-4): "we increase the number of attention heads so that it is divisible
    by x" -- kv heads padded to a multiple of P, each with its G = Hq / Hkv query
    heads -- "and zero-pad" the matrix dimension (intermediate) "so that they are
    divisible by the number of GPUs x" and by the GEMM block (256 here).
    Returns (Hq', Hkv', I')."""
    G = cfg.n_heads // cfg.n_kv_heads
    hkv = -(-cfg.n_kv_heads // P) * P
    ip = -(-cfg.intermediate // (256 * P)) * 256 * P if cfg.intermediate % P or (cfg.intermediate // P) % 256 else cfg.intermediate
    return hkv * G, hkv, ip


def verify_sharded(cfg, model: OracleModel, kv: KVCache, tokens, parents, P: int):
    """Tensor-parallel mode: each rank's partial sums computed separately and
    added across ranks in rank order (Megatron split).  When P does
    not divide the heads / intermediate size the weights are zero-padded as the
    paper describes (padded Q/K/V columns, O rows, gate/up columns
    and down rows are zero, so "the model output is equivalent of the
    non-padded model"); tree_k / tree_v are returned for the real heads."""
    Hq0, Hkv0, d, h, I0, V = (cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.hidden,
                              cfg.intermediate, cfg.vocab)
    Hq, Hkv, I = tp_padded_dims(cfg, P)

    def padc(W, n):  # zero columns up to n
        return np.pad(W, ((0, 0), (0, n - W.shape[1])))

    def padr(W, n):  # zero rows up to n
        return np.pad(W, ((0, n - W.shape[0]), (0, 0)))

    class _Padded:
        def w(self, l, name):
            W = model.w(l, name)
            if name == "wq":
                return padc(W, Hq * d)
            if name in ("wk", "wv"):
                return padc(W, Hkv * d)
            if name == "wo":
                return padr(W, Hq * d)
            if name in ("wgate", "wup"):
                return padc(W, I)
            if name == "wdown":
                return padr(W, I)
            return W

    pm = _Padded()
    tokens = np.asarray(tokens)
    L = kv.L
    depth, pos, anc = tree_meta(parents, L)
    T = len(tokens)
    x = model.embed_rows(tokens)
    hq, hk, ip = Hq // P, Hkv // P, I // P
    tk, tv = [], []
    for l in range(cfg.n_layers):
        xn = rmsnorm(x, model.norm(l, "attn_norm"), cfg.rms_eps)
        parts = []
        k_all = np.zeros((T, Hkv, d))
        v_all = np.zeros((T, Hkv, d))
        for r in range(P):
            Wq = pm.w(l, "wq")[:, r * hq * d:(r + 1) * hq * d]
            Wk = pm.w(l, "wk")[:, r * hk * d:(r + 1) * hk * d]
            Wv = pm.w(l, "wv")[:, r * hk * d:(r + 1) * hk * d]
            q = (xn @ Wq).reshape(T, hq, d)
            k = (xn @ Wk).reshape(T, hk, d)
            v = (xn @ Wv).reshape(T, hk, d)
            for i in range(T):
                q[i] = rope(q[i], pos[i], cfg.rope_theta)
                k[i] = rope(k[i], pos[i], cfg.rope_theta)
            k_all[:, r * hk:(r + 1) * hk] = k
            v_all[:, r * hk:(r + 1) * hk] = v
            Kp = np.pad(kv.K[l][:L], ((0, 0), (0, Hkv - Hkv0), (0, 0)))[:, r * hk:(r + 1) * hk]
            Vp = np.pad(kv.V[l][:L], ((0, 0), (0, Hkv - Hkv0), (0, 0)))[:, r * hk:(r + 1) * hk]
            attn = np.zeros((T, hq * d))
            for i in range(T):
                sel = np.nonzero(anc[i])[0]
                attn[i] = attend_node(q[i], np.concatenate([Kp, k[sel]]),
                                      np.concatenate([Vp, v[sel]]), hk).reshape(-1)
            parts.append(attn @ pm.w(l, "wo")[r * hq * d:(r + 1) * hq * d, :])
        s = parts[0]
        for p_ in parts[1:]:
            s = s + p_
        x = x + s
        xn2 = rmsnorm(x, model.norm(l, "mlp_norm"), cfg.rms_eps)
        parts = []
        for r in range(P):
            sl = slice(r * ip, (r + 1) * ip)
            hmid = silu(xn2 @ pm.w(l, "wgate")[:, sl]) * (xn2 @ pm.w(l, "wup")[:, sl])
            parts.append(hmid @ pm.w(l, "wdown")[sl, :])
        s = parts[0]
        for p_ in parts[1:]:
            s = s + p_
        x = x + s
        tk.append(k_all[:, :Hkv0])
        tv.append(v_all[:, :Hkv0])
    xn = rmsnorm(x, model.canon["final_norm"], cfg.rms_eps)
    vp = -(-V // P)
    shards = []
    W = model.canon["lm_head"]
    for r in range(P):
        shards.append(xn @ bf16_to_f64(W[r * vp:min(V, (r + 1) * vp)]).T)
    logits = np.concatenate(shards, axis=1)
    am = np.array([argmax_lowest(rw) for rw in logits], dtype=np.int64)
    acc, bonus = accept_walk(tokens, parents, am)
    return dict(logits=logits, argmax=am, accepted=acc, bonus=bonus, tree_k=tk, tree_v=tv,
                depth=depth, pos=pos, anc=anc)
