#!/bin/bash
# ncu launch list of bench.py itself (the command the driver times): per-launch
# gpu__time_duration + dram bytes, cold-cache and serialised -> compare SHARES.
# Run under gpurun after `python bench.py` has exited 0 on its own.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-bench}
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_plain_${TAG}.json 2> gpurun_out/bench_plain_${TAG}.log || { echo "plain bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_bench_${TAG}.log 2>&1
echo "ncu rc=$?"
