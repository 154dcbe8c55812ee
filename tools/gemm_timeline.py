"""Experiment: per-CTA phase timestamps of one GEMM launch (SS_EXP_TIMING build).
Runs layers=1 eager profile so the last GEMM launched is the LM head; uses the
env var SS_TIMELINE_KIND to pick which launch to keep (the library overwrites
the buffer on every launch, so we launch a single-kernel step variant)."""
import ctypes as C, os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2506_11309_b200 as pkg
from paper_2506_11309_b200 import swiftspec as ssp
cfg = dataclasses.replace(synth.CONFIGS["llama3-70b"], n_layers=1)
TPE = int(os.environ.get("TP", "1"))  # >1: one rank of a TP group, loopback emulation
sh = pkg.Shard(cfg, 0, TPE, 0, max_ctx=4096 + 256, max_tree=8)
sh.synth_weights(0); sh.synth_prefix_kv(1, 4096)
if TPE > 1:
    sh.import_loopback()
t, p = synth.tree_paperlike(8, cfg.vocab, np.random.default_rng(0))
dt = torch.tensor(t, dtype=torch.int32, device="cuda"); dp = torch.tensor(p, dtype=torch.int32, device="cuda")
L = ssp.lib()
f = L.ss_debug_gemm_timestamps; f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(1 << 16, dtype=np.uint64)
kind = int(sys.argv[1]) if len(sys.argv) > 1 else 2   # 0 QKV, 1 RESID (O: also down), 2 SWIGLU, 3 LM
L.ss_debug_gemm_set_kind.argtypes = [C.c_int]
L.ss_debug_gemm_set_kind(kind)
# eager per-kernel launches: stop after the kernel of interest by running the profiled step and
# reading the buffer after each... simpler: run the whole step; the LM head overwrites last.
# To isolate GU we run a step whose layer loop is 1 and read right after.
for rep in range(3):
    sh.verify_dev(dt, dp, 8, auto_commit=False, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
f(buf.ctypes.data, 1 << 16)
ts = buf.reshape(-1, 8)[:1024].astype(np.int64)
ok = ts[:, 0] > 0
ts = ts[ok]
sm = ts[:, 6].copy()
t0 = ts[:, 0].min()
rel = (ts - t0) / 1000.0
names = ["start", "pdl_wait done", "first data", "last unit done", "after flush+count", "after AR recv", "smid", "end"]
for i, n in enumerate(names):
    if n == 'smid': continue
    col = rel[:, i]
    print(f"kind {kind} {n:20s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us")

end = rel[:, 7]
order = np.argsort(sm)
print("end time by SM id (sorted by sm):")
smu = np.unique(sm)
per_sm = np.array([end[sm == s].max() for s in smu])
for i in range(0, len(smu), 16):
    print("  sm %3d-%3d:" % (smu[i], smu[min(i+15, len(smu)-1)]), " ".join("%5.1f" % x for x in per_sm[i:i+16]))
print("ctas per sm:", np.bincount(np.bincount(sm.astype(int))))

if os.environ.get("SHOW_SLOW"):
    ar = rel[:, 5]
    idx = np.argsort(-ar)[:12]
    print("slowest CTAs after AR recv: (cta, t_flush, t_sent(slot2), t_bar(slot3), t_after_ar, ndone)")
    for i in idx:
        print(int(np.nonzero(ok)[0][i]), round(rel[i, 4], 2), round(rel[i, 2], 2), round(rel[i, 3], 2), round(ar[i], 2), int(ts[i, 6]))
    print("ndone histogram:", np.bincount(ts[:, 6].astype(int)))
