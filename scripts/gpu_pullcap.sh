#!/bin/bash
# A/B of the peer-pull CTA cap (EQC_PULL_CTAS) in the pipelined N-GPU bench
# and the standalone compose (one partial per GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for C in ${CAPS:-0 148}; do
EQC_PULL_CTAS=$C timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29522 \
  scripts/bench_compose.py --w 3840 --h 2160 --sources $N 2>>gpurun_out/pullcap.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['results']; print('compose cap $C', {k: r[k]['ms'] for k in ('direct_send_p2p','direct_send_p2p_slots')})" >> gpurun_out/pullcap_n${N}.txt
done
for rep in 1 2; do for C in ${CAPS:-0 148}; do
EQC_PULL_CTAS=$C timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29521 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline $BX 2>>gpurun_out/pullcap.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cap $C $BX', d['value'], d['ms_per_step'], d['kernels']['image_compress_rle_batch']['ms'], d['kernels']['compositor_depth_rle']['ms'])" >> gpurun_out/pullcap_n${N}.txt
done; done
cat gpurun_out/pullcap_n${N}.txt
