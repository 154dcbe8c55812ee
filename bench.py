#!/usr/bin/env python3
"""bench.py -- tree-verify step latency of the B200-native SwiftSpec target path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config llama3-70b] [--T 8] [--L 4096]

N = 1 runs the BASELINE metric's model (Llama3-70B-shaped int4 AWQ g128,
random weights from the device-side synthetic generator) at TP = 1 -- it fits
one B200.  N > 1 is launched by torchrun, one rank per GPU, TP = N with the
fused flag-based all-reduces over NVLink (strong scaling: the same 70B step on
more GPUs).  One JSON line is printed by rank 0.

A "step" = one pass of the whole hot path: tree ingest + embedding, 80 x
(RMSNorm, QKV+RoPE+KV write, tree attention, O + all-reduce + residual,
RMSNorm, gate/up+SwiGLU, down + all-reduce + residual), final norm, LM head +
argmax, greedy accept walk, KV compaction + commit (auto-commit).

--impl reference times the float64 CPU oracle (oracle/) on the host cores on
a bounded sample of the same workload and extrapolates to the same metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

GROUP = 128


# ---------------------------------------------------------------- perf model
def step_bytes(cfg, T, L, P=1):
    """Algorithmic HBM bytes per step per GPU:
    int4 weights + bf16 scales + int4 zeros of QKV/O/gate/up/down, bf16 LM-head
    shard, KV prefix read, tree KV written."""
    h, I, d = cfg.hidden, cfg.intermediate, cfg.head_dim
    per_w = 0.5 + 2.0 / GROUP + 0.5 / GROUP
    mats = h * (cfg.n_heads + 2 * cfg.n_kv_heads) * d + cfg.n_heads * d * h + 2 * h * I + I * h
    b = cfg.n_layers * mats * per_w / P
    b += math.ceil(cfg.vocab / P) * h * 2
    b += cfg.n_layers * (L + T) * 2 * (cfg.n_kv_heads / P) * d * 2
    return b


def gateup_bytes(cfg, P=1):
    """Algorithmic bytes of one gate/up launch (the dominant kernel: 55% of the layer)."""
    return cfg.hidden * 2 * cfg.intermediate / P * (0.5 + 2.0 / GROUP + 0.5 / GROUP)


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------- distributed helpers
def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def exchange_handles(blob: bytes, world: int):
    """All-gather every rank's peer-buffer handle blob (host logic; gloo-testable)."""
    import torch.distributed as dist
    if world == 1:
        return [blob]
    out = [None] * world
    dist.all_gather_object(out, blob)
    return out


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a torchrun environment: relaunch this
    script under torch.distributed.run with N local ranks (127.0.0.1
    rendezvous), pass rank 0's JSON line through, return the worst exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def gather_objects(obj, world: int):
    import torch.distributed as dist
    if world == 1:
        return [obj]
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def max_over_ranks(x: float, world: int, device=None) -> float:
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- trees
def make_trees(cfg, T, n, seed=2):
    rng = np.random.default_rng(seed)
    return [synth.tree_paperlike(T, cfg.vocab, rng) for _ in range(n)]


# ---------------------------------------------------------------- CPU oracle sample
class OracleSample:
    """The float64 oracle (as it stands) on a bounded sample of the step:
    `n_layers_sample` decoder layers (dequant + attention + MLP for all T
    nodes against an L-row prefix) plus 1/vocab_frac of the LM head, scaled to
    the full step (x n_layers / n_layers_sample, x vocab_frac).  Input
    generation happens once in the constructor and is not timed."""

    def __init__(self, cfg, T, L, n_layers_sample=1, vocab_frac=16, seed=0):
        import oracle as O
        self.O, self.cfg, self.T, self.L = O, cfg, T, L
        self.nls, self.vf = n_layers_sample, vocab_frac
        self.sub = synth.ModelCfg(cfg.name + "-sample", n_layers_sample, cfg.hidden, cfg.intermediate,
                                  cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.vocab // vocab_frac)
        self.m = O.OracleModel(self.sub, synth.gen_model(self.sub, seed), cache_dense=False)
        self.kv = O.KVCache(self.sub, L + T + 1)
        for l in range(n_layers_sample):
            k, v = synth.gen_prefix_kv(seed + 1, l, L, cfg.n_kv_heads, cfg.head_dim)
            self.kv.set_prefix(l, k, v)
        self.kv.L = L
        self.trees = make_trees(self.sub, T, 4)
        self.cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        self.sample = (f"{n_layers_sample} of {cfg.n_layers} layers + 1/{vocab_frac} of the LM head "
                       f"(T={T}, L={L}), wall time scaled to the full step")

    def step_seconds(self, i=0):
        toks, parents = self.trees[i % len(self.trees)]
        t0 = time.perf_counter()
        self.O.verify(self.sub, self.m, self.kv, toks, parents, want_logits=False)
        dt = time.perf_counter() - t0
        t1 = time.perf_counter()
        self.m.logits(np.ones((self.T, self.cfg.hidden)))
        dt_lm = time.perf_counter() - t1
        per_layer = max(dt - dt_lm, 1e-9) / self.nls
        return per_layer * self.cfg.n_layers + dt_lm * self.vf


# ---------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    smp = OracleSample(cfg, args.T, args.L)
    steps = []
    for i in range(args.warmup + args.steps):
        s = smp.step_seconds(i)
        if i >= args.warmup:
            steps.append(s)
    us = float(np.mean(steps)) * 1e6
    line = {
        "impl": "reference", "metric": METRIC(cfg, args), "value": us, "unit": "us",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": us / 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based generator, random weights)",
        "config": CONFIG(cfg, args, world),
        "cpu_baseline": {"value": us, "unit": "us", "cores": smp.cores, "kind": "oracle", "sample": smp.sample},
        "e2e": {"value": us, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def METRIC(cfg, args):
    return f"tree-verify step latency (Llama3-70B-shaped int4 AWQ, T={args.T}, L={args.L}, TP={args.gpus})" \
        if cfg.name == "llama3-70b" else f"tree-verify step latency ({cfg.name}, T={args.T}, L={args.L}, TP={args.gpus})"


def CONFIG(cfg, args, world):
    return {"workload": f"{cfg.name} int4 AWQ g128 target, {args.T}-node paper-like tree, {args.L}-token KV, "
                        f"TP={world}", "model": cfg.name, "T": args.T, "L": args.L, "tp": world,
            "parallelism": f"tp{world}", "global_batch": 1, "seq_len": args.L,
            "l2": "inputs larger than L2 (weights streamed every step)"}


# ---------------------------------------------------------------- our arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_2506_11309_b200 as pkg
    from paper_2506_11309_b200 import swiftspec as ssp

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world} (run without torchrun to self-spawn)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    T, L = args.T, args.L
    n_steps = args.warmup + args.steps
    max_ctx = max(L + T * (3 * n_steps + 8) + 64, 8192 + 4 * 64 + 256)  # C-async runs at an 8K context
    sh = pkg.Shard(cfg, rank, world, local, max_ctx=max_ctx, max_tree=max(T, 32))
    sh.synth_weights(args.seed)
    sh.synth_prefix_kv(args.seed + 1, L)
    if world > 1:
        blobs = exchange_handles(sh.export_handle(), world)
        sh.import_peers(blobs)
        dist.barrier()
    trees = make_trees(cfg, T, n_steps)
    d_tok = torch.tensor(np.stack([t for t, _ in trees]), dtype=torch.int32, device=dev)
    d_par = torch.tensor(np.stack([p for _, p in trees]), dtype=torch.int32, device=dev)
    rwords = ssp.result_nbytes() // 4
    d_res = torch.zeros((n_steps, rwords), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(i):
        sh.verify_dev(d_tok[i], d_par[i], T, d_result=d_res[i], auto_commit=True, stream=stream)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # every rank must have walked the same path from the same argmax (TP:
    # replicated accept + commit); all statuses SS_OK
    wres = [ssp.parse_result(r, T) for r in d_res[:args.warmup].cpu().numpy()]
    allw = gather_objects([(r["status"], r["accepted"], r["bonus"], r["argmax"]) for r in wres], world)
    ranks_agree = all(a == allw[0] for a in allw)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for j, i in enumerate(range(args.warmup, n_steps)):
            step(i)
            ev[j + 1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_step = [ev[j].elapsed_time(ev[j + 1]) for j in range(args.steps)]
    ms = ev[0].elapsed_time(ev[-1]) / args.steps
    ms = max_over_ranks(ms, world, dev)
    p50 = max_over_ranks(float(np.percentile(per_step, 50)), world, dev)
    p90 = max_over_ranks(float(np.percentile(per_step, 90)), world, dev)
    res = [ssp.parse_result(r, T) for r in d_res[args.warmup:].cpu().numpy()]
    allt = gather_objects([(r["status"], r["accepted"], r["bonus"]) for r in res], world)
    ranks_agree = ranks_agree and all(a == allt[0] for a in allt)
    emitted = float(np.mean([r["n_accepted"] for r in res]))  # (n-1) accepted + 1 bonus
    statuses = set(r["status"] for r in res)
    kps = sh.kernels_per_step(T, auto_commit=True)

    # ---- e2e: same metric through the public C-ABI with HOST buffers
    # (H2D of the tree, D2H of the result inside ss_verify_tree, every step)
    _skip = set(os.environ.get("SS_BENCH_SKIP", "").split(","))  # debugging aid (bisection)
    e2e_steps = max(3, args.steps // 2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    h_trees = make_trees(cfg, T, e2e_steps + 2, seed=7)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sh.verify(*h_trees[0], stream=stream)
    sh.commit_accepted(stream=stream)
    torch.cuda.synchronize()
    f0.record(stream)
    for i in range(e2e_steps):
        sh.verify(*h_trees[1 + i], stream=stream)
        sh.commit_accepted(stream=stream)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1) / e2e_steps, world, dev)

    # ---- per-kernel device times (eager step, CUDA events around every launch)
    prof = None
    try:
        i0 = n_steps - 1
        for _ in range(0 if "prof" in _skip else 2):
            prof = sh.profile_step(d_tok[i0], d_par[i0], T, stream=stream)
    except Exception as ex:  # pragma: no cover
        prof = {"error": str(ex)}
    torch.cuda.synchronize()

    peak, peak_src = read_peaks()
    bytes_step = step_bytes(cfg, T, L + 1, world)
    line = {
        "metric": METRIC(cfg, args), "value": ms * 1e3, "unit": "us", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "int4 weights (AWQ g128) x fp16/bf16 activations, fp32 accumulate",
        "data": "synthetic (seeded counter-based generator, random weights, paper-like trees)",
        "config": CONFIG(cfg, args, world),
        "clocks": clk.summary(),
        "e2e": {"value": e2e_ms * 1e3, "unit": "us", "h2d_bytes_per_step": 2 * 64 * 4,
                "d2h_bytes_per_step": ssp.result_nbytes()},
        "gpu_launches": kps * args.steps,
        "decode_tokens_per_s": emitted / (ms / 1e3),
        "emitted_tokens_per_step": emitted,
        "step_roofline_frac": bytes_step / (ms / 1e3) / 1e9 / peak,
        "step_bytes": bytes_step,
        "status_ok": statuses == {0},
        "p50_us": p50 * 1e3, "p90_us": p90 * 1e3,
        "ranks_agree": bool(ranks_agree),
    }
    if isinstance(prof, dict) and prof.get("step_kernel", (0, 0))[1] > 0:
        # persistent step kernel: the whole step's weights + KV stream through it
        sk_ms, sk_n = prof["step_kernel"]
        tot = sum(v[0] for v in prof.values())
        per = sk_ms / sk_n
        ach = bytes_step / (per / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(f"{cfg.name}/tp{world}/T{T}/step_kernel")
            except Exception:
                traffic = None
        line["roofline"] = {"kernel": "step_kernel (persistent: every layer's GEMMs, attention, all-reduces, "
                                      "LM head, accept walk)", "bound": "hbm",
                            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                            "traffic": traffic, "peak_source": peak_src,
                            "algorithmic_bytes_per_launch": bytes_step,
                            "avg_launch_us": per * 1e3, "share_of_step": sk_ms / tot if tot else None}
        line["kernel_times_us"] = {k: {"total": v[0] * 1e3, "launches": v[1]} for k, v in prof.items() if v[1]}
    elif isinstance(prof, dict) and "gate_up_swiglu" in prof:
        gu_ms, gu_n = prof["gate_up_swiglu"]
        tot = sum(v[0] for v in prof.values())
        per = gu_ms / max(gu_n, 1)
        ach = gateup_bytes(cfg, world) / (per / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(f"{cfg.name}/tp{world}/T{T}/gate_up")
            except Exception:
                traffic = None
        line["roofline"] = {"kernel": "gate_up_swiglu (W4A16 GEMM, fused SwiGLU)", "bound": "hbm",
                            "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                            "traffic": traffic, "peak_source": peak_src,
                            "algorithmic_bytes_per_launch": gateup_bytes(cfg, world),
                            "avg_launch_us": per * 1e3, "share_of_step": gu_ms / tot if tot else None}
        line["kernel_times_us"] = {k: {"total": v[0] * 1e3, "launches": v[1]} for k, v in prof.items()}
    try:  # where the step's time goes (extra traced step, outside the timed region)
        sm_mhz = line["clocks"].get("sm_mhz") or 1965.0
        bd = None if "breakdown" in _skip else phase_breakdown(sh, cfg, d_tok, d_par, T, n_steps - 2, stream, sm_mhz)
        if bd:
            line["breakdown"] = bd
    except Exception as ex:  # pragma: no cover
        line["breakdown"] = {"error": str(ex)}
    # extras after the headline measurement: a failure in one of them (a CUDA
    # error is sticky for the process) is recorded in the line, never fatal
    def extra(key, fn):
        try:
            line[key] = fn()
        except Exception as ex:  # pragma: no cover
            line[key] = {"error": str(ex)[:300]}
    if world == 1 and not args.no_extra and "other" not in _skip:
        extra("other_configs", lambda: other_configs(args, sh, cfg, local, dev, peak))
    if world == 1 and not args.no_tp_emulate:
        diag = os.environ.get("SS_BENCH_DIAG") == "1"  # debugging aid: hang/fault progress words
        if diag:
            sh.step_trace(2)
        extra("decode_planted", lambda: decode_planted(sh, cfg, T, L))
        if diag and "error" in line["decode_planted"]:
            from collections import Counter
            wh = sh.step_trace_where()
            cnt = Counter()
            for c_ in range(148):
                words = []
                for w_ in range(12):
                    code = int(wh[c_, w_]) >> 32
                    words.append(f"{code >> 16}.{(code >> 8) & 0xFF:x}.{code & 0xFF:x}")
                cnt[tuple(words)] += 1
            for k_, v_ in cnt.most_common(8):
                print("DIAG", v_, "CTAs:", " | ".join(k_), file=sys.stderr, flush=True)
        if "tp" not in _skip:
            extra("tp_emulated", lambda: tp_emulated(args, cfg, local, dev, peak))
    if world == 1 and not args.no_async and cfg.name == "llama3-70b":
        extra("c_async", lambda: c_async(args, sh, cfg, local, dev))
    if rank == 0 and not args.no_cpu_baseline:
        smp = OracleSample(cfg, T, L)
        sec = smp.step_seconds(0)
        line["cpu_baseline"] = {"value": sec * 1e6, "unit": "us", "cores": smp.cores, "kind": "oracle",
                                "sample": smp.sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    try:
        sh.close()
    except Exception:  # pragma: no cover  (a sticky CUDA error from an extra)
        pass
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def planted_tree(seq, pos, d, T, V, rng):
    """Tree rooted at seq[pos] whose first d nodes after the root are the chain
    seq[pos+1 .. pos+d] (the target's own greedy continuation, so exactly d draft
    tokens are accepted), padded to T nodes with random leaves (depth <= 7, P:166;
    siblings distinct)."""
    toks, par, depth = [int(seq[pos])], [-1], [0]
    for i in range(1, d + 1):
        toks.append(int(seq[pos + i]))
        par.append(i - 1)
        depth.append(i)
    while len(toks) < T:
        p = int(rng.integers(0, len(toks)))
        if depth[p] >= 7:
            continue
        sib = {toks[j] for j in range(len(toks)) if par[j] == p}
        if p < d:
            sib.add(int(seq[pos + p + 1]))  # never a second copy of the planted child
        t = int(rng.integers(0, V))
        if t in sib:
            continue
        toks.append(t)
        par.append(p)
        depth.append(depth[p] + 1)
    return np.array(toks, dtype=np.int32), np.array(par, dtype=np.int32)


def decode_planted(sh, cfg, T, L, n_steps=24, mean_emit=3.1, seed=5):
    """Decode tokens/s of one request through the public host API with trees that
    contain the target's greedy continuation at a random depth (mean emitted
    tokens per step ~3.1, the MT-bench-like acceptance of P:587): first the
    greedy continuation is produced by T=1 steps, then the cache is rewound to L
    and the same tokens are re-generated with planted trees (verify + commit per
    step, host buffers, wall clock).  The emitted tokens are checked against the
    greedy continuation: a divergence is possible only at a near-tie of the top
    two logits (R14), because the stream-K partial sums are reduced in a
    run-dependent fp32 order; `mismatches` lists the first ones."""
    rng = np.random.default_rng(seed)
    need = n_steps * (T + 1) + T + 2
    sh.set_committed_len(L)
    seq = [1]
    dmode = os.environ.get("SS_BENCH_DECODE", "")  # debugging aid (the open decode fault, DESIGN 10)
    import torch
    for k in range(need * (int(dmode[3:]) if dmode.startswith("rep") else 1)):
        import time as _tt
        _t0 = _tt.perf_counter()
        try:
            r = sh.verify(np.array([seq[-1]], dtype=np.int32), np.array([-1], dtype=np.int32))
        except Exception as ex:
            from paper_2506_11309_b200 import swiftspec as _ssp
            raise RuntimeError(f"greedy T=1 step {k} (L = {L + k}, {_tt.perf_counter() - _t0:.3f} s, "
                               f"watchdog {_ssp.watchdog_record(6)}, ctr {sh.debug_ctr_base()}): {ex}") from ex
        sh.commit_accepted()
        if dmode == "sync":
            torch.cuda.synchronize()
        seq.append(int(r["bonus"]))
        if dmode.startswith("rep") and k % need == need - 1:
            sh.set_committed_len(L)
            seq = [1]
    if dmode.startswith("rep"):  # the last round's sequence is the one used below
        sh.set_committed_len(L)
        seq = [1]
        for k in range(need):
            _t0 = _tt.perf_counter()
            try:
                r = sh.verify(np.array([seq[-1]], dtype=np.int32), np.array([-1], dtype=np.int32))
            except Exception as ex:
                raise RuntimeError(f"greedy T=1 last-round step {k} ({_tt.perf_counter() - _t0:.3f} s): {ex}") from ex
            sh.commit_accepted()
            seq.append(int(r["bonus"]))
    sh.set_committed_len(L)
    pos, emitted, match = 0, 0, True
    mism, mism_steps = [], []
    import time as _t
    t0 = _t.perf_counter()
    for _ in range(n_steps):
        d = int(min(T - 1, 7, rng.geometric(1.0 / mean_emit) - 1))
        toks, par = planted_tree(seq, pos, d, T, cfg.vocab, rng)
        try:
            r = sh.verify(toks, par)
        except Exception as ex:
            raise RuntimeError(f"planted step {len(mism_steps)}: {ex}") from ex
        sh.commit_accepted()
        n = int(r["n_accepted"])                     # root + accepted draft nodes
        got = [int(toks[i]) for i in r["accepted"][1:]] + [int(r["bonus"])]
        if got != seq[pos + 1:pos + 1 + n]:
            match = False
            mism.append({"step": len(mism_steps), "d": d, "n": n, "got": got, "want": seq[pos + 1:pos + 1 + n]})
        mism_steps.append(0)
        emitted += n                                 # (n - 1) accepted + 1 bonus
        pos += n
    dt = _t.perf_counter() - t0
    return {"tokens_per_s": emitted / dt, "mean_emitted_per_step": emitted / n_steps, "steps": n_steps,
            "T": T, "tokens": emitted, "matches_greedy": bool(match), "mismatches": mism[:3],
            "how": "host API (ss_verify_tree + ss_commit_accepted per step, wall clock), planted trees"}


def phase_breakdown(sh, cfg, d_tok, d_par, T, i0, stream, sm_mhz=1965.0):
    """One extra step with the persistent kernel's timeline on (ss_step_trace;
    outside the timed region): the mean critical-path span of each phase over
    the middle layers (exit of the phase's last CTA minus exit of the previous
    phase's last CTA, us) and the all-reduce part of the O / down tails of the
    middle layer (the finaliser of tile-group 0: LL sends + receives, us)."""
    import torch
    if not sh.step_kernel_active(T):
        return None
    sh.step_trace(True)
    for i in (i0, i0 + 1):  # the first launch after enabling re-captures the graph
        sh.verify_dev(d_tok[i], d_par[i], T, auto_commit=True, stream=stream)
    torch.cuda.synchronize()
    tr, utl = sh.read_step_trace(with_units=True)
    sh.step_trace(False)
    tr = tr.astype(np.int64)
    utl = utl.astype(np.int64)
    n_l = cfg.n_layers
    ex = np.where(tr[:, :, 2] > 0, tr[:, :, 2], 0).max(axis=0)  # per slot: exit of the last CTA (ns)
    names = ["qkv", "attention", "o_allreduce", "gate_up", "down_allreduce"]
    spans = {k: [] for k in names}
    for l in range(max(1, n_l // 4), max(2, 3 * n_l // 4)):
        for p in range(5):
            prev = ex[l * 5 + p - 1] if p else ex[(l - 1) * 5 + 4]
            cur = ex[l * 5 + p]
            if prev > 0 and cur > 0:
                spans[names[p]].append((cur - prev) / 1e3)
    out = {"phase_us": {k: round(float(np.mean(v)), 2) for k, v in spans.items() if v},
           "lm_head_us": round(float((ex[n_l * 5] - ex[(n_l - 1) * 5 + 4]) / 1e3), 2)}
    ar = {}
    for ph, name in (((2, "o"), (4, "down")) if sh.tp_size > 1 else ()):
        tt = utl[30000 + ph * 16:30000 + ph * 16 + 9]
        if tt[0] and tt[3]:
            ar[name] = round(float((tt[3] - tt[1]) / sm_mhz), 2)  # clk -> us
    if ar:
        out["allreduce_us"] = ar
        out["allreduce_how"] = ("persistent-kernel timeline, finaliser of tile-group 0 of the middle layer: "
                                "LL sends to every rank + rank-ordered receive, clock64 at the SM clock")
    return out


def time_steps(sh, cfg, T, n_warm, n_time, dev, seed=13):
    """Device time per auto-commit step (CUDA events on the launching stream)."""
    import torch
    trees = make_trees(cfg, T, n_warm + n_time, seed=seed)
    d_tok = torch.tensor(np.stack([t for t, _ in trees]), dtype=torch.int32, device=dev)
    d_par = torch.tensor(np.stack([p for _, p in trees]), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for i in range(n_warm):
        sh.verify_dev(d_tok[i], d_par[i], T, auto_commit=True, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(n_warm, n_warm + n_time):
        sh.verify_dev(d_tok[i], d_par[i], T, auto_commit=True, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n_time


def other_configs(args, sh70, cfg70, local, dev, peak):
    """The other BASELINE.json TP = 1 workloads on this GPU, same step (whole hot
    path, auto-commit): 70B-shaped at T = 16 / 32 (the main shard, its prefix
    rewound to L), Llama3-1B-shaped (T = 16, 1K KV) and 8B-shaped (T = 16, 4K KV).
    Device time per step, HBM roofline fraction of the step's algorithmic bytes."""
    import paper_2506_11309_b200 as pkg
    out = {}
    L = args.L
    for T in (16, 32):
        sh70.set_committed_len(L)
        ms = time_steps(sh70, cfg70, T, 3, 8, dev)
        b = step_bytes(cfg70, T, L + 1, 1)
        out[f"{cfg70.name}/T{T}/L{L}"] = {"us": ms * 1e3, "roofline_frac": b / (ms / 1e3) / 1e9 / peak}
    for name, T, Lx in (("llama3-1b", 16, 1024), ("llama3-8b", 16, 4096)):
        c = synth.CONFIGS[name]
        sh = pkg.Shard(c, 0, 1, local, max_ctx=Lx + 16 * 40 + 64, max_tree=16)
        sh.synth_weights(args.seed)
        sh.synth_prefix_kv(args.seed + 1, Lx)
        ms = time_steps(sh, c, T, 3, 10, dev)
        b = step_bytes(c, T, Lx + 1, 1)
        out[f"{name}/T{T}/L{Lx}"] = {"us": ms * 1e3, "roofline_frac": b / (ms / 1e3) / 1e9 / peak}
        sh.close()
    out["how"] = "TP 1, paper-like trees, auto-commit steps, CUDA events; weights random (device generator)"
    return out


def c_async(args, sh70, cfg70, local, dev, n_tokens=64, draft_sms=20, bs=8, w=8, spare_sms=8):
    """BASELINE configs[4] on one GPU: Alg. 1 parallel tree generation
    (ss_speculative_decode) with a Llama3-3B-shaped draft and the Llama3-70B-
    shaped target, 8K-token KV context in both.  The two GPU groups of the paper
    (2 + 4 GPUs) are emulated by splitting this GPU's SMs (ss_set_launch_cap:
    the target's grid on 148 - draft_sms SMs, the draft's on draft_sms; HBM is
    shared), linked by the a13 mailboxes.  d = floor(t_target / t_draft) from a
    short profile.  Wall-clock tokens/s of one request over
    n_tokens tokens, async and serial (draft, then verify), and whether the
    emitted tokens equal the target's own greedy decode.  Random
    weights: the draft and target disagree, ~1 token per step."""
    import time as _t
    import torch
    import paper_2506_11309_b200 as pkg
    Lc = 8192
    c3 = synth.CONFIGS["llama3-3b"]
    out = {"draft": c3.name, "target": cfg70.name, "L": Lc, "bs": bs, "w": w, "n_tokens": n_tokens,
           "draft_sms": draft_sms, "target_sms": 148 - draft_sms - spare_sms}
    dr = pkg.Shard(c3, 0, 1, local, max_ctx=Lc + 4 * n_tokens + 256, max_tree=64)
    try:
        dr.synth_weights(args.seed + 17)
        dr.synth_prefix_kv(args.seed + 18, Lc)
        sh70.synth_prefix_kv(args.seed + 1, Lc)
        sh70.set_committed_len(Lc)
        dr.set_committed_len(Lc)
        root = 1234
        # reference: the target's plain greedy decode (T = 1 steps, whole GPU)
        ref, cur = [], root
        t0 = _t.perf_counter()
        for _ in range(n_tokens):
            r = sh70.verify(np.array([cur], dtype=np.int32), np.array([-1], dtype=np.int32))
            sh70.commit_accepted()
            cur = int(r["bonus"])
            ref.append(cur)
        out["greedy_tokens_per_s"] = n_tokens / (_t.perf_counter() - t0)
        # profile for d: one target step and one draft expansion at their SM shares
        sh70.set_launch_cap(148 - draft_sms - spare_sms)
        dr.set_launch_cap(draft_sms)
        sh70.set_committed_len(Lc)
        tt = time_steps(sh70, cfg70, bs, 2, 4, dev) / 1e3
        sh70.set_committed_len(Lc)
        toks = np.arange(1, w + 1, dtype=np.int32)
        par = np.arange(-1, w - 1, dtype=np.int32)
        for _ in range(2):
            dr.extend_topk(toks, par, 0, w)
            dr.set_committed_len(Lc)
        t0 = _t.perf_counter()
        for _ in range(4):
            dr.extend_topk(toks, par, 0, w)
            dr.set_committed_len(Lc)
        td = (_t.perf_counter() - t0) / 4
        d = max(1, int(tt // td))
        out.update({"t_target_ms": tt * 1e3, "t_draft_expansion_ms": td * 1e3, "d": d})
        ts, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        for mode in ("async", "serial"):
            sh70.set_committed_len(Lc)
            dr.set_committed_len(Lc)
            toks_out, st = sh70.speculative_decode(dr, root, n_tokens, bs=bs, w=w, d=d, mode=mode,
                                                   target_stream=ts, draft_stream=ds)
            out[mode] = {"tokens_per_s": st["n_emitted"] / (st["wall_ms"] / 1e3),
                         "mean_emitted_per_step": st["n_emitted"] / max(st["steps"], 1),
                         "steps": st["steps"], "expansions": st["expansions"], "wall_ms": st["wall_ms"],
                         "matches_greedy": toks_out == ref[:len(toks_out)]}
        out["how"] = ("one request, wall clock around ss_speculative_decode (draft thread + target thread, "
                      "mailbox hand-off); the target's greedy_tokens_per_s is plain T = 1 decoding on the whole GPU")
    finally:
        sh70.set_launch_cap(0)
        dr.close()
    try:
        out["self_draft_1b"] = self_draft(args, local, dev)
    except Exception as ex:  # pragma: no cover
        out["self_draft_1b"] = {"error": str(ex)}
    return out


def self_draft(args, local, dev, n_tokens=96, bs=8, w=8, draft_sms=64, spare_sms=8):
    """Alg. 1 where the draft predicts the target: a Llama3-1B-shaped target and a
    draft with the SAME weights (random weights give no real draft/target pair,
    so this is the one setting whose acceptance is not ~0).  The draft's top-1
    chain is the target's greedy path, so subtrees survive re-roots and the
    draft's expansions during a verify are reused -- the async overlap of P:228
    becomes visible (async vs serial tokens/s).  SM split as in c_async."""
    import torch
    import paper_2506_11309_b200 as pkg
    c1 = synth.CONFIGS["llama3-1b"]
    Lc = 1024
    t = pkg.Shard(c1, 0, 1, local, max_ctx=Lc + 4 * n_tokens + 256, max_tree=bs)
    d = pkg.Shard(c1, 0, 1, local, max_ctx=Lc + 4 * n_tokens + 256, max_tree=64)
    out = {"model": c1.name, "L": Lc, "bs": bs, "w": w, "n_tokens": n_tokens, "draft_sms": draft_sms,
           "target_sms": 148 - draft_sms - spare_sms}
    try:
        for sh in (t, d):
            sh.synth_weights(args.seed)
            sh.synth_prefix_kv(args.seed + 1, Lc)
        t.set_launch_cap(148 - draft_sms - spare_sms)
        d.set_launch_cap(draft_sms)
        ts, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        root = 4321
        res = {}
        for dd in (1, 2, 4):
            for mode in ("async", "serial"):
                t.set_committed_len(Lc)
                d.set_committed_len(Lc)
                toks, st = t.speculative_decode(d, root, n_tokens, bs=bs, w=w, d=dd, mode=mode,
                                                target_stream=ts, draft_stream=ds)
                res[f"{mode}/d{dd}"] = {"tokens_per_s": st["n_emitted"] / (st["wall_ms"] / 1e3),
                                        "mean_emitted_per_step": st["n_emitted"] / max(st["steps"], 1),
                                        "expansions": st["expansions"], "tokens": toks}
        ref = res["serial/d1"]["tokens"]
        for k, v in res.items():
            v["matches_serial_d1"] = v.pop("tokens") == ref
        out["runs"] = res
        out["how"] = ("wall clock around ss_speculative_decode; identical draft and target weights; d = expansions "
                      "per round; outputs must agree across modes (all are the target's greedy decode)")
    finally:
        t.close()
        d.close()
    return out


def tp_emulated(args, cfg, local, dev, peak):
    """Per-GPU step latency of ONE rank of a TP = 2/4/8 group, emulated on this
    single GPU (ss_import_loopback: the rank's weight shard, KV heads and LL
    all-reduce stores, with its own partial standing in for the peers').
    Timing only -- the logits are not the sharded model's -- and the
    all-reduce cost is a lower bound (local stores instead of NVLink)."""
    import torch
    import paper_2506_11309_b200 as pkg
    T, L = args.T, args.L
    out = {"note": "one TP rank on one GPU, loopback all-reduce (timing emulation, not a multi-GPU run)"}
    n = 3 + 10
    for P in (2, 4, 8):
        sh = pkg.Shard(cfg, 0, P, local, max_ctx=L + 32 * (3 * n + 8) + 64, max_tree=max(T, 32))
        sh.synth_weights(args.seed)
        sh.synth_prefix_kv(args.seed + 1, L)
        sh.import_loopback()
        trees = make_trees(cfg, T, n, seed=11)
        d_tok = torch.tensor(np.stack([t for t, _ in trees]), dtype=torch.int32, device=dev)
        d_par = torch.tensor(np.stack([p for _, p in trees]), dtype=torch.int32, device=dev)
        stream = torch.cuda.current_stream(dev)
        from paper_2506_11309_b200 import swiftspec as ssp
        res = torch.zeros(ssp.result_nbytes() // 4, dtype=torch.int32, device=dev)
        for i in range(3):
            sh.verify_dev(d_tok[i], d_par[i], T, d_result=res, auto_commit=True, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(3, n):
            sh.verify_dev(d_tok[i], d_par[i], T, d_result=res, auto_commit=True, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / (n - 3)
        b = step_bytes(cfg, T, L + 1, P)
        status = ssp.parse_result(res.cpu().numpy(), T)["status"]  # -5 = a poll ran out of budget
        out[f"tp{P}"] = {"us": ms * 1e3, "bytes_per_gpu": b, "roofline_frac": b / (ms / 1e3) / 1e9 / peak,
                         "status_ok": status == 0}
        try:
            bd = phase_breakdown(sh, cfg, d_tok, d_par, T, n - 2, stream)
            if bd:
                out[f"tp{P}"].update(bd)
        except Exception as e:  # measurement extra only
            out[f"tp{P}"]["breakdown_error"] = str(e)
        if P >= 4:
            # all-reduce scheme A/B at T = 8 and 32 on the same rank
            ab = {}
            for mode in ("one-shot", "two-shot"):
                sh.set_allreduce(mode)
                for Tx in (8, 32):
                    sh.set_committed_len(L)
                    ab[f"{mode}/T{Tx}"] = time_steps(sh, cfg, Tx, 2, 6, dev) * 1e3
            sh.set_allreduce("one-shot")
            out[f"tp{P}"]["allreduce_ab_us"] = ab
        sh.close()
    out["allreduce_ab_how"] = ("step us per mode on the loopback rank: the two-shot rank stores one partial per "
                               "non-home tile-group and reduces + broadcasts its home 1/P; loopback stores are "
                               "local, so NVLink egress savings (7x -> 1.75x T h 8 B per all-reduce at TP 8) "
                               "do not show here")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3-70b", choices=sorted(synth.CONFIGS))
    ap.add_argument("--T", type=int, default=8)
    ap.add_argument("--L", type=int, default=4096)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tp-emulate", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other BASELINE configs (70B T16/32, 1B, 8B)")
    ap.add_argument("--no-async", action="store_true", help="skip the C-async (Alg. 1, 3B draft + 70B target) line")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    cfg = synth.CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
