#!/bin/bash
# A/B of library environment knobs on the short bench line: each argument is one
# setting, e.g.  tools/ab_env.sh "SQ_TRANSPOSE=1" "SQ_TRANSPOSE=2 SQ_ONE_CAP=16384"
i=0
for setting in "$@"; do
  i=$((i+1))
  env $setting timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab$i.log 2>&1
  tail -1 gpurun_out/bench_ab$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$setting:', round(d['value'],2), 'Gkeys/s', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, d['output_check'])" || tail -3 gpurun_out/bench_ab$i.log
done
