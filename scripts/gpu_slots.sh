#!/bin/bash
# Frame slots (eqc_comm_frame_buffers) + EQC_FLAG_OVERLAP under gpurun --gpus N:
# parity (tests/mp_compose.py), standalone compose with one partial per GPU,
# and the pipelined bench.py with each of them switched off.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
[ -z "$SKIP_TESTS" ] && timeout 900 python -m pytest tests/test_gpu_multi.py -q -k nccl > gpurun_out/slots_pytest_n${N}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/slots_pytest_n${N}.log
tail -3 gpurun_out/slots_pytest_n${N}.log
[ -z "$SKIP_TESTS" ] && timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29522 \
  scripts/bench_compose.py --w 3840 --h 2160 --sources $N > gpurun_out/compose_slots_n${N}.json 2> gpurun_out/compose_slots_n${N}.log
python -c "import json; d=json.load(open('gpurun_out/compose_slots_n${N}.json')); print({k: v['ms'] for k, v in d['results'].items()})"
for rep in 1 2 3; do for V in ${BXS:-default --no-overlap-flag --no-frame-slots --no-comm-priority}; do
X=$( [ "$V" = default ] && echo "" || echo "$V" )
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29521 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline $X 2>>gpurun_out/slots_bench.log > gpurun_out/slots_line.json
python -c "import json; d=json.load(open('gpurun_out/slots_line.json')); print('[$V]', d['value'], d['ms_per_step'], d['kernels']['image_compress_rle_batch']['ms'], d['kernels']['compositor_depth_rle']['ms'], d['gpu_launches'])" >> gpurun_out/slots_bench_n${N}.txt
[ "$V" = default ] && cp gpurun_out/slots_line.json gpurun_out/bench_n${N}_default_r$rep.json
done; done
cat gpurun_out/slots_bench_n${N}.txt
