#!/bin/bash
# Where does the N=2 step overhead come from? (under gpurun --gpus 2)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
run() {  # name, torchrun args...
  local name=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 100)) \
      bench.py --gpus 2 --steps 100 --warmup 5 --no-cpu-baseline --no-compose-block "$@" > gpurun_out/n2p_${name}.json 2> gpurun_out/n2p_${name}.log
  python -c "import json; j=json.load(open('gpurun_out/n2p_${name}.json')); print('${name}', j['ms_per_step'], {k:(v['ms'],v['inloop_ms']) for k,v in j['kernels'].items()})"
}
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-anchors > gpurun_out/n2p_n1.json 2> gpurun_out/n2p_n1.log
python -c "import json; j=json.load(open('gpurun_out/n2p_n1.json')); print('n1', j['ms_per_step'], {k:(v['ms'],v['inloop_ms']) for k,v in j['kernels'].items()})"
run default
run noslots --no-frame-slots
run nopipe --no-pipeline
run nooverlap --no-overlap-flag
