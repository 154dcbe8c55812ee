#!/bin/bash
# full GPU gate: smoke, gpu tests, bench (T=8 default, T=16, T=32), step traces
mkdir -p gpurun_out
timeout 180 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
for T in 16 32; do timeout 400 python bench.py --steps 10 --warmup 3 --T $T --no-cpu-baseline --no-tp-emulate > gpurun_out/bench_T$T.json 2> gpurun_out/bench_T$T.err; echo "bench T$T rc=$?"; done
python - <<'PY'
import json
for f in ["gpurun_out/bench.json", "gpurun_out/bench_T16.json", "gpurun_out/bench_T32.json"]:
    try:
        d = json.load(open(f))
        print(f, "us", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "frac", round(d["step_roofline_frac"], 3),
              {k: (round(v["us"], 1), round(v["roofline_frac"], 3)) for k, v in d.get("tp_emulated", {}).items() if k.startswith("tp")},
              d.get("decode_planted", {}).get("tokens_per_s"), d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
