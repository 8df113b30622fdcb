#!/bin/bash
# GPU box: everything the round's profiles/ summaries come from -- the full bench
# line, the ncu launch list of a short bench run (after that ran clean), full ncu
# captures of the top kernels, every config timed, the small-n latencies.
set -u
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1 || { echo "bench failed"; tail -5 gpurun_out/bench_full.log; exit 1; }
tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json
timeout 300 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_short.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  > gpurun_out/ncu_launches.log 2>&1
bash tools/ncu_full.sh k_colsort k_transpose_ws k_bucketsort > /dev/null 2>&1
timeout 900 python tools/configs.py > gpurun_out/configs.log 2>&1
timeout 300 python tools/small_n.py > gpurun_out/small_n.jsonl 2>&1
timeout 300 python tools/prof_configs.py cfg3 cfg4_sorted cfg4_reverse cfg4_swapped cfg4_nonsquare cfg5 cfg5p > gpurun_out/prof_configs.log 2>&1
echo done
