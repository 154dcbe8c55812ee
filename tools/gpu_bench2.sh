#!/bin/bash
mkdir -p gpurun_out
SECONDS=0; timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
echo "bench wall ${SECONDS}s"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("us", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "frac", round(d["step_roofline_frac"], 3), d["clocks"])
print("breakdown", d.get("breakdown"))
print("other", d.get("other_configs"))
for k, v in d.get("tp_emulated", {}).items():
    if k.startswith("tp"): print(k, round(v["us"], 1), round(v["roofline_frac"], 3), v.get("phase_us"), v.get("allreduce_us"))
print("roofline", d.get("roofline"))
PY
