#!/bin/bash
# Per-rank event times of the pipelined N-GPU bench over repeated runs (diagnoses slow steady states).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for rep in 1 2 3 4 5 6; do
EQC_BENCH_RANKS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29521 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline $BX > gpurun_out/ranks_line.json 2> gpurun_out/ranks_err.log
python -c "import json; d=json.load(open('gpurun_out/ranks_line.json')); print('run $rep', d['value'], d['ms_per_step'])" >> gpurun_out/ranks_n${N}.txt
grep "rank .: step" gpurun_out/ranks_err.log | sort >> gpurun_out/ranks_n${N}.txt
done
cat gpurun_out/ranks_n${N}.txt
