#!/bin/bash
# Scattered direct send check (under gpurun --gpus N): multi-process parity, bench default vs --scatter.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "nccl" > gpurun_out/sc_pytest_n${N}.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/sc_pytest_n${N}.log
for v in default scatter; do
  extra=""; [ $v = scatter ] && extra="--scatter"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 100)) \
      bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline --no-compose-block $extra > gpurun_out/sc_${v}_n${N}.json 2> gpurun_out/sc_${v}_n${N}.log
  python -c "import json; j=json.load(open('gpurun_out/sc_${v}_n${N}.json')); print('$v', j['value'], j['ms_per_step'], {k:(v['ms'],v['inloop_ms']) for k,v in j['kernels'].items()})" || tail -5 gpurun_out/sc_${v}_n${N}.log
done
