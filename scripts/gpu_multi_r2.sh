#!/bin/bash
# Round-2 multi-GPU check (under gpurun --gpus N): full GPU suite, bench at N,
# display wall over NCCL at N.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_n${N}.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_n${N}.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_n${N}.json 2> gpurun_out/bench_n${N}.log
echo "bench rc=$?"
python -c "import json; j=json.load(open('gpurun_out/bench_n${N}.json')); print(j['value'], j['ms_per_step']); print(json.dumps(j['compose_scaling']))"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29532 \
    scripts/bench_wall.py > gpurun_out/wall_n${N}.json 2> gpurun_out/wall_n${N}.log
echo "wall rc=$?"; cat gpurun_out/wall_n${N}.json; tail -2 gpurun_out/wall_n${N}.log
