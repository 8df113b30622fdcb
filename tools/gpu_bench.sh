#!/bin/bash
# GPU box: short bench line only (kernel ms per step), no tests.
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'Gkeys/s', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}, d['output_check'])" || tail -5 gpurun_out/bench.log
