#!/bin/bash
# A/B of the one-CTA bucket cap (SQ_ONE_CAP) on the short bench line.
for cap in "$@"; do
  SQ_ONE_CAP=$cap timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cap$cap.log 2>&1
  tail -1 gpurun_out/bench_cap$cap.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cap', $cap, round(d['value'],2), 'Gkeys/s', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, d['output_check'])"
done
