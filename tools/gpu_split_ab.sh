mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "split or forced or full_tile" > gpurun_out/split_tests.log 2>&1; tail -3 gpurun_out/split_tests.log
bash tools/ab_env.sh "SQ_BIG_MODE=1" "SQ_BIG_MODE=4" "SQ_BIG_MODE=4 SQ_SPLIT_TILE=12288" "SQ_BIG_MODE=4 SQ_SPLIT_TILE=32768 SQ_SPLIT_FILL=80" "SQ_BIG_MODE=4 SQ_SPLIT_FILL=95" "SQ_BIG_MODE=4 SQ_SPLIT_QMAX=8"
