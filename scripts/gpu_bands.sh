#!/bin/bash
# Gather-aware direct-send bands vs equal bands (under gpurun --gpus N): c4 compose block + the N-GPU bench.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_p2p_virtual.py -q -x > gpurun_out/bands_pytest_n${N}.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bands_pytest_n${N}.log
for v in gather equal; do
  envs=""; [ $v = equal ] && envs="EQC_P2P_EQUAL_BANDS=1"
  env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 100)) \
      bench.py --gpus $N --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bands_${v}_n${N}.json 2> gpurun_out/bands_${v}_n${N}.log
  python -c "import json; j=json.load(open('gpurun_out/bands_${v}_n${N}.json')); print('$v', j['value'], j['ms_per_step'], {k:(v['ms'],v['frac_of_roof']) for k,v in j['compose_scaling']['schedules'].items()})" || tail -5 gpurun_out/bands_${v}_n${N}.log
done
