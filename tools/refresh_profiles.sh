#!/bin/bash
# GPU box: full bench line, then the ncu launch list of a short bench run
# (after that command ran clean).  Full captures: tools/ncu_full.sh <kernel regex>.
set -u
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1 || { echo "bench failed"; tail -5 gpurun_out/bench_full.log; exit 1; }
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_short.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  > gpurun_out/ncu_launches.log 2>&1
echo done
