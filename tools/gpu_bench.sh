#!/bin/bash
# smoke + bench (+ optional extra args via BENCH_ARGS); bounded so a hang costs little
mkdir -p gpurun_out
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -1 gpurun_out/smoke.log
[ $rc -ne 0 ] && exit 1
timeout 240 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open('gpurun_out/bench.json'))
print('step us', round(d['value'], 1), 'e2e', round(d['e2e']['value'], 1), 'frac', round(d['step_roofline_frac'], 3),
      'gu frac', round(d.get('roofline', {}).get('frac', 0), 3), d['clocks'])
print({k: round(v['total'] / max(v['launches'], 1), 1) for k, v in d.get('kernel_times_us', {}).items()})
print('decode_planted', {k: v for k, v in d.get('decode_planted', {}).items() if k != 'how'})
print('tp_emulated', {k: (round(v['us'], 1), round(v['roofline_frac'], 3)) for k, v in d.get('tp_emulated', {}).items() if k.startswith('tp')})
PY
tail -2 gpurun_out/bench.err
