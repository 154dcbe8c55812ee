"""Thin ctypes binding of libswiftspec.so (include/swiftspec.h).

Argument marshalling only: every step of the verify path runs in the CUDA
kernels behind the C-ABI.  There is no CPU fallback -- if the library (or a
CUDA device) is missing, the import / the call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", os.environ.get("SWIFTSPEC_LIB", "libswiftspec.so"))

SS_MAX_TREE = 64
STATUS = {0: "SS_OK", -1: "SS_EINVAL", -2: "SS_ECAPACITY", -3: "SS_ECONSISTENCY", -4: "SS_ECUDA",
          -5: "SS_ETIMEOUT", -6: "SS_ESTATE"}
KIND = dict(EMBED=0, ATTN_NORM=1, WQ=2, WK=3, WV=4, WO=5, MLP_NORM=6, WGATE=7, WUP=8, WDOWN=9,
            FINAL_NORM=10, LM_HEAD=11)
SUB = dict(QWEIGHT=0, QZEROS=1, SCALES=2, DENSE=0)


class SwiftSpecError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class ModelCfgC(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden", C.c_int32), ("intermediate", C.c_int32),
                ("n_heads", C.c_int32), ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("vocab", C.c_int32), ("group_size", C.c_int32), ("max_ctx", C.c_int32),
                ("max_tree", C.c_int32), ("rms_eps", C.c_float), ("rope_theta", C.c_float)]


class VerifyResultC(C.Structure):
    _fields_ = [("n_accepted", C.c_int32), ("accepted", C.c_int32 * SS_MAX_TREE),
                ("bonus_token", C.c_int32), ("argmax", C.c_int32 * SS_MAX_TREE), ("status", C.c_int32)]


class SpecCfgC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("bs", "w", "d", "K", "n_tokens", "eos", "mode")]


class SpecStatsC(C.Structure):
    _fields_ = [("n_emitted", C.c_int32), ("steps", C.c_int32), ("target_steps", C.c_int32),
                ("expansions", C.c_int32), ("accepted", C.c_int32), ("wall_ms", C.c_double)]


_lib = None

EXPORTS = ["ss_init_shard", "ss_export_handle", "ss_import_peers", "ss_import_local_peers", "ss_import_loopback",
           "ss_set_launch_cap", "ss_destroy", "ss_last_error", "ss_load_weights", "ss_synth_weights",
           "ss_set_prefix_kv", "ss_synth_prefix_kv", "ss_read_kv", "ss_set_committed_len",
           "ss_committed_len", "ss_verify_tree", "ss_verify_tree_dev", "ss_extend_tree", "ss_extend_tree_topk", "ss_reroot", "ss_speculative_decode",
           "ss_commit_kv",
           "ss_commit_accepted", "ss_kernels_per_step", "ss_profile_step", "ss_mailbox_inbox",
           "ss_attach_mailbox", "ss_verify_tree_mailbox", "ss_verify_tree_mailbox_n", "ss_mailbox_post_tree", "ss_mailbox_recv_result",
           "ss_set_debug", "ss_watchdog_record", "ss_debug_ctr_base", "ss_set_allreduce", "ss_read_tree_meta", "ss_read_packed", "ss_debug_gemm", "ss_set_step_kernel",
           "ss_step_kernel_active", "ss_step_trace", "ss_read_step_trace", "ss_step_trace_host"]
SS_DEBUG_CONSISTENCY = 1
SS_DEBUG_DETERMINISTIC = 2


def watchdog_record(n: int = 8):
    """The step kernel's watchdog panic record (ss_watchdog_record)."""
    out = np.zeros(n, dtype=np.uint64)
    lib().ss_watchdog_record(out.ctypes.data_as(C.c_void_p), n)
    return [int(x) for x in out]


def lib():
    """Load libswiftspec.so (built in-tree by paper_2506_11309_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2506_11309_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, u64, sz = C.c_void_p, C.c_int32, C.c_uint64, C.c_size_t
    sig = {
        "ss_init_shard": (i32, [C.POINTER(ModelCfgC), i32, i32, i32, C.POINTER(vp)]),
        "ss_export_handle": (i32, [vp, vp, C.POINTER(sz)]),
        "ss_import_peers": (i32, [vp, C.POINTER(vp), C.POINTER(sz)]),
        "ss_import_local_peers": (i32, [vp, C.POINTER(vp)]),
        "ss_import_loopback": (i32, [vp]),
        "ss_set_launch_cap": (i32, [vp, i32]),
        "ss_destroy": (i32, [vp]),
        "ss_last_error": (C.c_char_p, [vp]),
        "ss_set_debug": (i32, [vp, i32]),
        "ss_set_allreduce": (i32, [vp, i32]),
        "ss_watchdog_record": (i32, [vp, i32]),
        "ss_debug_ctr_base": (u64, [vp]),
        "ss_set_step_kernel": (i32, [vp, i32]),
        "ss_step_kernel_active": (i32, [vp, i32]),
        "ss_step_trace": (i32, [vp, i32]),
        "ss_read_step_trace": (i32, [vp, vp, sz, C.POINTER(i32), C.POINTER(i32)]),
        "ss_step_trace_host": (vp, [vp]),
        "ss_read_tree_meta": (i32, [vp, vp, vp, vp, vp, vp]),
        "ss_read_packed": (i32, [vp, i32, i32, vp, sz, C.POINTER(sz)]),
        "ss_debug_gemm": (i32, [vp, i32, i32, vp, i32, vp, i32, vp]),
        "ss_load_weights": (i32, [vp, i32, i32, i32, vp, sz]),
        "ss_synth_weights": (i32, [vp, u64]),
        "ss_set_prefix_kv": (i32, [vp, i32, vp, vp, i32]),
        "ss_synth_prefix_kv": (i32, [vp, u64, i32]),
        "ss_read_kv": (i32, [vp, i32, i32, i32, vp, vp]),
        "ss_set_committed_len": (i32, [vp, i32]),
        "ss_committed_len": (i32, [vp]),
        "ss_verify_tree": (i32, [vp, vp, vp, i32, C.POINTER(VerifyResultC), vp, vp]),
        "ss_verify_tree_dev": (i32, [vp, vp, vp, i32, vp, vp, i32, vp]),
        "ss_extend_tree": (i32, [vp, vp, vp, i32, i32, C.POINTER(VerifyResultC), vp, vp]),
        "ss_extend_tree_topk": (i32, [vp, vp, vp, i32, i32, i32, vp, vp, vp, C.POINTER(VerifyResultC), vp]),
        "ss_reroot": (i32, [vp, vp, i32, vp, i32, vp]),
        "ss_speculative_decode": (i32, [vp, vp, i32, C.POINTER(SpecCfgC), vp, C.POINTER(SpecStatsC), vp, vp]),
        "ss_commit_kv": (i32, [vp, vp, i32, vp]),
        "ss_commit_accepted": (i32, [vp, vp]),
        "ss_kernels_per_step": (i32, [vp, i32, i32]),
        "ss_profile_step": (i32, [vp, vp, vp, i32, vp, vp, vp]),
        "ss_mailbox_inbox": (i32, [vp, C.POINTER(vp)]),
        "ss_attach_mailbox": (i32, [vp, vp, i32]),
        "ss_verify_tree_mailbox": (i32, [vp, i32, vp]),
        "ss_verify_tree_mailbox_n": (i32, [vp, i32, i32, vp]),
        "ss_mailbox_post_tree": (i32, [vp, vp, vp, i32, C.c_uint32, vp]),
        "ss_mailbox_recv_result": (i32, [vp, C.c_uint32, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(code: int, shard=None):
    if code != 0:
        raise SwiftSpecError(code, lib().ss_last_error(shard).decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _stream_handle(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


class Shard:
    """One tensor-parallel shard of the target model on one CUDA device."""

    def __init__(self, cfg, tp_rank: int = 0, tp_size: int = 1, device: int = 0,
                 max_ctx: int = 4096 + 128, max_tree: int = 64):
        self.cfg = cfg
        self.tp_rank, self.tp_size, self.device = tp_rank, tp_size, device
        c = ModelCfgC(cfg.n_layers, cfg.hidden, cfg.intermediate, cfg.n_heads, cfg.n_kv_heads,
                      cfg.head_dim, cfg.vocab, 128, max_ctx, max_tree, cfg.rms_eps, cfg.rope_theta)
        h = C.c_void_p()
        _check(lib().ss_init_shard(C.byref(c), tp_rank, tp_size, device, C.byref(h)))
        self.h = h
        self.max_ctx, self.max_tree = max_ctx, max_tree
        vp = -(-cfg.vocab // tp_size)
        self.v_off = tp_rank * vp
        self.v_l = max(0, min(cfg.vocab, (tp_rank + 1) * vp) - self.v_off)
        # kv heads per rank after the zero padding for tp_size not dividing
        # n_kv_heads (padded heads read back as zeros)
        self.hkv_l = -(-cfg.n_kv_heads // tp_size)

    def _ck(self, code: int):
        _check(code, self.h)

    def set_step_kernel(self, on: bool):
        """True (default): the persistent one-launch step for T <= 32; False: per-phase kernels."""
        self._ck(lib().ss_set_step_kernel(self.h, 1 if on else 0))

    def step_kernel_active(self, T: int) -> bool:
        return lib().ss_step_kernel_active(self.h, T) == 1

    def step_trace(self, on: bool):
        """Record a per-CTA phase timeline on later persistent-step launches (measurement hook;
        on=2: mapped host memory, readable while a launch still runs)."""
        self._ck(lib().ss_step_trace(self.h, int(on)))

    def step_trace_where(self) -> np.ndarray:
        """Progress words [512 CTAs][16 warps] straight from the mapped buffer (no CUDA call)."""
        p = lib().ss_step_trace_host(self.h)
        if not p:
            raise RuntimeError("step_trace(2) not enabled")
        slots = self.cfg.n_layers * 5 + 1
        n = 512 * slots * 3 + 512 * 16 + 65536
        arr = np.ctypeslib.as_array((C.c_uint64 * n).from_address(p))
        return arr[512 * slots * 3:].reshape(512, 16).copy()

    def read_step_trace(self, with_where: bool = False, with_units: bool = False):
        """uint64 [512 CTAs][n_layers*5+1 slots][3 stamps] (entry, first unit ready, exit; ns);
        with_where: also the per-(CTA, warp) progress words [512][16] (mapped mode);
        with_units: also CTA 0's unit timeline (65536 words, clock64)."""
        slots = self.cfg.n_layers * 5 + 1
        nt = 512 * slots * 3
        buf = np.zeros(nt + 512 * 16 + 65536, dtype=np.uint64)
        nc, ns = C.c_int32(), C.c_int32()
        self._ck(lib().ss_read_step_trace(self.h, _ptr(buf), buf.size, C.byref(nc), C.byref(ns)))
        out = [buf[:nt].reshape(nc.value, ns.value, 3)]
        if with_where:
            out.append(buf[nt:nt + 512 * 16].reshape(512, 16))
        if with_units:
            out.append(buf[nt + 512 * 16:])
        return out[0] if len(out) == 1 else tuple(out)

    def set_debug(self, flags: int):
        """SS_DEBUG_CONSISTENCY: cross-rank checksum of every verify's tree."""
        self._ck(lib().ss_set_debug(self.h, flags))

    def close(self):
        if getattr(self, "h", None):
            try:
                lib().ss_destroy(self.h)
            except TypeError:  # interpreter shutdown: ctypes already torn down
                pass
            self.h = None

    __del__ = close

    # ---- weights / KV
    def load_tensor(self, layer: int, kind: int, sub: int, arr: np.ndarray):
        a = np.ascontiguousarray(arr)
        self._ck(lib().ss_load_weights(self.h, layer, kind, sub, _ptr(a), a.nbytes))

    def load_canonical(self, m: dict):
        """Load a canonical model dict (synth.gen_model layout)."""
        names = dict(wq=KIND["WQ"], wk=KIND["WK"], wv=KIND["WV"], wo=KIND["WO"],
                     wgate=KIND["WGATE"], wup=KIND["WUP"], wdown=KIND["WDOWN"])
        for l, lw in enumerate(m["layers"]):
            self.load_tensor(l, KIND["ATTN_NORM"], 0, lw["attn_norm"])
            self.load_tensor(l, KIND["MLP_NORM"], 0, lw["mlp_norm"])
            for n, k in names.items():
                q, z, s = lw[n]
                self.load_tensor(l, k, SUB["QWEIGHT"], q)
                self.load_tensor(l, k, SUB["QZEROS"], z)
                self.load_tensor(l, k, SUB["SCALES"], s)
        self.load_tensor(0, KIND["EMBED"], 0, m["embed"])
        self.load_tensor(0, KIND["FINAL_NORM"], 0, m["final_norm"])
        self.load_tensor(0, KIND["LM_HEAD"], 0, m["lm_head"])

    def synth_weights(self, seed: int):
        self._ck(lib().ss_synth_weights(self.h, seed))

    def set_prefix_kv(self, layer: int, k_bits: np.ndarray, v_bits: np.ndarray):
        k = np.ascontiguousarray(k_bits, dtype=np.uint16)
        v = np.ascontiguousarray(v_bits, dtype=np.uint16)
        self._ck(lib().ss_set_prefix_kv(self.h, layer, _ptr(k), _ptr(v), k.shape[0]))

    def synth_prefix_kv(self, seed: int, L: int):
        self._ck(lib().ss_synth_prefix_kv(self.h, seed, L))

    def read_kv(self, layer: int, row0: int, n: int):
        """Cache rows as float32 [n][n_kv_heads/tp][head_dim] (stored fp16)."""
        d = self.cfg.head_dim
        k = np.zeros((n, self.hkv_l, d), dtype=np.float32)
        v = np.zeros((n, self.hkv_l, d), dtype=np.float32)
        self._ck(lib().ss_read_kv(self.h, layer, row0, n, _ptr(k), _ptr(v)))
        return k, v

    def set_committed_len(self, L: int):
        self._ck(lib().ss_set_committed_len(self.h, L))

    @property
    def L(self) -> int:
        r = lib().ss_committed_len(self.h)
        if r < 0:
            raise SwiftSpecError(-4, lib().ss_last_error(self.h).decode())
        return r

    # ---- the step
    def verify(self, tokens, parents, want_logits: bool = False, stream=None):
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        p = np.ascontiguousarray(parents, dtype=np.int32)
        T = len(t)
        res = VerifyResultC()
        logits = np.zeros((T, self.v_l), dtype=np.float32) if want_logits else None
        self._ck(lib().ss_verify_tree(self.h, _ptr(t), _ptr(p), T, C.byref(res),
                                    _ptr(logits) if want_logits else None, _stream_handle(stream)))
        n = res.n_accepted
        return dict(n_accepted=n, accepted=list(res.accepted[:n]), bonus=res.bonus_token,
                    argmax=list(res.argmax[:T]), status=res.status, logits=logits)

    def extend(self, tokens, parents, T0: int, want_logits: bool = False, stream=None):
        """Non-square forward (ss_extend_tree): w = len(tokens) new nodes
        T0.. on the first T0 nodes of the pending tree; parents index the whole
        tree.  argmax covers all T0 + w nodes; logits the new nodes only."""
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        p = np.ascontiguousarray(parents, dtype=np.int32)
        w = len(t)
        res = VerifyResultC()
        logits = np.zeros((w, self.v_l), dtype=np.float32) if want_logits else None
        self._ck(lib().ss_extend_tree(self.h, _ptr(t), _ptr(p), T0, w, C.byref(res),
                                    _ptr(logits) if want_logits else None, _stream_handle(stream)))
        n = res.n_accepted
        return dict(n_accepted=n, accepted=list(res.accepted[:n]), bonus=res.bonus_token,
                    argmax=list(res.argmax[:T0 + w]), status=res.status, logits=logits)

    def extend_topk(self, tokens, parents, T0: int, K: int, stream=None):
        """Draft forward (ss_extend_tree_topk): -> (top_tok [w][K], top_logit [w][K], lse [w])."""
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        p = np.ascontiguousarray(parents, dtype=np.int32)
        w = len(t)
        tok = np.zeros((w, K), dtype=np.int32)
        val = np.zeros((w, K), dtype=np.float32)
        lse = np.zeros(w, dtype=np.float32)
        res = VerifyResultC()
        self._ck(lib().ss_extend_tree_topk(self.h, _ptr(t), _ptr(p), T0, w, K, _ptr(tok), _ptr(val), _ptr(lse),
                                         C.byref(res), _stream_handle(stream)))
        return tok, val, lse

    def reroot(self, path, keep, stream=None):
        """Commit the chain `path`, keep the subtree `keep` (ss_reroot)."""
        a = np.ascontiguousarray(path, dtype=np.int32)
        k = np.ascontiguousarray(keep, dtype=np.int32)
        self._ck(lib().ss_reroot(self.h, _ptr(a) if len(a) else None, len(a), _ptr(k) if len(k) else None,
                               len(k), _stream_handle(stream)))

    def speculative_decode(self, draft, root_token: int, n_tokens: int, bs: int = 8, w: int = 8, d: int = 1,
                           K: int = 0, eos: int = -1, mode: str = "async", target_stream=None, draft_stream=None):
        """Alg. 1 parallel tree generation with this shard as the target and `draft`
        (ss_speculative_decode) -> (tokens, stats dict)."""
        cfg = SpecCfgC(bs, w, d, K, n_tokens, eos, 0 if mode == "async" else 1)
        out = np.zeros(n_tokens, dtype=np.int32)
        st = SpecStatsC()
        self._ck(lib().ss_speculative_decode(self.h, draft.h, int(root_token), C.byref(cfg), _ptr(out), C.byref(st),
                                           _stream_handle(target_stream), _stream_handle(draft_stream)))
        stats = {k: getattr(st, k) for k, _ in SpecStatsC._fields_}
        return [int(t) for t in out[:st.n_emitted]], stats

    def verify_dev(self, d_tokens, d_parents, T: int, d_result=None, d_logits=None,
                   auto_commit: bool = False, stream=None):
        """All-device step: d_* are torch CUDA tensors (or raw pointers)."""
        ptr = lambda x: None if x is None else (x if isinstance(x, int) else x.data_ptr())
        self._ck(lib().ss_verify_tree_dev(self.h, ptr(d_tokens), ptr(d_parents), T, ptr(d_result),
                                        ptr(d_logits), 1 if auto_commit else 0, _stream_handle(stream)))

    def commit_kv(self, accepted, stream=None):
        a = np.ascontiguousarray(accepted, dtype=np.int32)
        self._ck(lib().ss_commit_kv(self.h, _ptr(a), len(a), _stream_handle(stream)))

    def commit_accepted(self, stream=None):
        self._ck(lib().ss_commit_accepted(self.h, _stream_handle(stream)))

    def kernels_per_step(self, T: int, auto_commit: bool = False) -> int:
        return lib().ss_kernels_per_step(self.h, T, 1 if auto_commit else 0)

    PROF_KINDS = ["embed+tree", "qkv", "attention", "o_proj", "rmsnorm", "gate_up_swiglu", "down",
                  "lm_head_argmax_accept", "commit", "step_kernel"]

    def profile_step(self, d_tokens, d_parents, T: int, stream=None):
        """Eager step with CUDA events around every kernel -> {kind: (ms, launches)}."""
        ms = np.zeros(len(self.PROF_KINDS), dtype=np.float32)
        cnt = np.zeros(len(self.PROF_KINDS), dtype=np.int32)
        ptr = lambda x: x if isinstance(x, int) else x.data_ptr()
        self._ck(lib().ss_profile_step(self.h, ptr(d_tokens), ptr(d_parents), T, _ptr(ms), _ptr(cnt),
                                     _stream_handle(stream)))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(self.PROF_KINDS)}

    # ---- a13 mailbox handoff
    def mailbox_inbox(self) -> int:
        ptr = C.c_void_p()
        self._ck(lib().ss_mailbox_inbox(self.h, C.byref(ptr)))
        return ptr.value

    def attach_mailbox(self, outbox_ptr: int, eos: int = -1):
        self._ck(lib().ss_attach_mailbox(self.h, outbox_ptr, eos))

    def verify_mailbox(self, auto_commit: bool = True, stream=None):
        self._ck(lib().ss_verify_tree_mailbox(self.h, 1 if auto_commit else 0, _stream_handle(stream)))

    # ---- inspection / test hooks
    def read_tree_meta(self):
        """(T, pos[T], anc[T] as uint64 bitmasks, tokens[T], parents[T]) of the last step."""
        T = C.c_int32(0)
        pos = np.zeros(SS_MAX_TREE, dtype=np.int32)
        anc = np.zeros(SS_MAX_TREE, dtype=np.uint64)
        tok = np.zeros(SS_MAX_TREE, dtype=np.int32)
        par = np.zeros(SS_MAX_TREE, dtype=np.int32)
        self._ck(lib().ss_read_tree_meta(self.h, C.byref(T), _ptr(pos), _ptr(anc), _ptr(tok), _ptr(par)))
        n = T.value
        return n, pos[:n], anc[:n], tok[:n], par[:n]

    def read_packed(self, layer: int, which: int) -> np.ndarray:
        total = C.c_size_t(0)
        self._ck(lib().ss_read_packed(self.h, layer, which, None, 0, C.byref(total)))
        buf = np.zeros(total.value, dtype=np.uint8)
        self._ck(lib().ss_read_packed(self.h, layer, which, _ptr(buf), total.value, C.byref(total)))
        return buf

    def debug_gemm(self, layer: int, which: int, d_x, T: int, d_y, allreduce: bool = False, stream=None):
        """One W4 GEMM of the step's kernel on caller activations (torch CUDA tensors)."""
        self._ck(lib().ss_debug_gemm(self.h, layer, which, d_x.data_ptr(), T, d_y.data_ptr(),
                                     1 if allreduce else 0, _stream_handle(stream)))

    # ---- tensor parallel peers
    def export_handle(self) -> bytes:
        buf = C.create_string_buffer(4096)
        n = C.c_size_t(0)
        self._ck(lib().ss_export_handle(self.h, buf, C.byref(n)))
        return buf.raw[:n.value]

    def import_peers(self, blobs):
        arr = (C.c_void_p * len(blobs))()
        keep = [C.create_string_buffer(b, len(b)) for b in blobs]
        for i, k in enumerate(keep):
            arr[i] = C.cast(k, C.c_void_p)
        lens = (C.c_size_t * len(blobs))(*[len(b) for b in blobs])
        self._ck(lib().ss_import_peers(self.h, arr, lens))

    @staticmethod
    def import_local_peers(shards):
        arr = (C.c_void_p * len(shards))(*[s.h.value for s in shards])
        for s in shards:
            s._ck(lib().ss_import_local_peers(s.h, arr))

    def import_loopback(self):
        """Timing emulation of this rank alone (include/swiftspec.h ss_import_loopback)."""
        self._ck(lib().ss_import_loopback(self.h))

    def debug_ctr_base(self) -> int:
        return int(lib().ss_debug_ctr_base(self.h))

    def set_allreduce(self, mode: str):
        """'one-shot' (default) or 'two-shot' TP all-reduce in the step kernel (ss_set_allreduce)."""
        self._ck(lib().ss_set_allreduce(self.h, {"one-shot": 0, "two-shot": 1}[mode]))

    def set_launch_cap(self, cap: int):
        self._ck(lib().ss_set_launch_cap(self.h, cap))


def result_nbytes() -> int:
    return C.sizeof(VerifyResultC)


def parse_result(buf: np.ndarray, T: int) -> dict:
    """Decode an ss_verify_result copied back from the device as raw int32s."""
    a = np.asarray(buf, dtype=np.int32).reshape(-1)
    n = int(a[0])
    return dict(n_accepted=n, accepted=[int(x) for x in a[1:1 + n]], bonus=int(a[1 + SS_MAX_TREE]),
                argmax=[int(x) for x in a[2 + SS_MAX_TREE:2 + SS_MAX_TREE + T]],
                status=int(a[2 + 2 * SS_MAX_TREE]))


def mailbox_post_tree(inbox_ptr: int, tokens, parents, seq: int, stream=None):
    t = np.ascontiguousarray(tokens, dtype=np.int32)
    p = np.ascontiguousarray(parents, dtype=np.int32)
    _check(lib().ss_mailbox_post_tree(inbox_ptr, _ptr(t), _ptr(p), len(t), seq, _stream_handle(stream)))


def mailbox_recv_result(outbox_ptr: int, seq: int, dev_out_ptr: int, stream=None):
    _check(lib().ss_mailbox_recv_result(outbox_ptr, seq, dev_out_ptr, _stream_handle(stream)))
