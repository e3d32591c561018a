#!/bin/bash
# N-GPU bench with identical vs per-rank-seeded inputs (under gpurun --gpus N).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for v in same perrank; do
  extra=""; [ $v = perrank ] && extra="--per-rank-seeds"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 100)) \
      bench.py --gpus $N $extra > gpurun_out/seeds_${v}_n${N}.json 2> gpurun_out/seeds_${v}_n${N}.log
  python -c "import json; j=json.load(open('gpurun_out/seeds_${v}_n${N}.json')); print('$v', j['value'], j['ms_per_step'], {k:(v['ms'],v['inloop_ms']) for k,v in j['kernels'].items()})" || tail -5 gpurun_out/seeds_${v}_n${N}.log
done
