#!/bin/bash
# A/B of the EQC_FLAG_OVERLAP pull cap (EQC_OVERLAP_CTAS) in the default pipelined bench.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for rep in 1 2 3; do for C in ${CAPS:-74 148 296}; do
EQC_OVERLAP_CTAS=$C timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29521 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline 2>>gpurun_out/overlapcap.log > gpurun_out/oc_line.json
python -c "import json; d=json.load(open('gpurun_out/oc_line.json')); print('cap $C', d['value'], d['ms_per_step'], d['kernels']['image_compress_rle_batch']['ms'], d['kernels']['compositor_depth_rle']['ms'])" >> gpurun_out/overlapcap_n${N}.txt
done; done
cat gpurun_out/overlapcap_n${N}.txt
