#!/bin/bash
# Frame-slot (eqc_comm_frame_buffers) checks under gpurun --gpus N: NCCL/P2P
# parity test, standalone compose with one partial per GPU (slots vs copy),
# and bench.py with / without slots.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29522 \
  scripts/bench_compose.py --w 3840 --h 2160 --sources $N > gpurun_out/compose_slots_n${N}.json 2> gpurun_out/compose_slots_n${N}.log
cat gpurun_out/compose_slots_n${N}.json
for X in "--frame-slots" "" "--frame-slots" ""; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29521 bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline $X 2>>gpurun_out/slots_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$X', d['value'], d['ms_per_step'], d['compose_direct_send_latency_ms_rank0'], d['kernels'])" >> gpurun_out/slots_bench_n${N}.txt
done
cat gpurun_out/slots_bench_n${N}.txt
