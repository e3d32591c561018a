#!/bin/bash
# Multi-GPU checks under gpurun --gpus N: NCCL parity test + N-GPU bench.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo_n${N}.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k nccl > gpurun_out/pytest_multi_n${N}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_multi_n${N}.log
for X in ${BENCH_X-raw nccl rle}; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29511 \
  bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline --exchange $X > gpurun_out/bench_n${N}_${X}.json 2> gpurun_out/bench_n${N}_${X}.log
echo "bench $X rc=$?" >> gpurun_out/bench_n${N}_${X}.log
done
tail -5 gpurun_out/pytest_multi_n${N}.log; for f in gpurun_out/bench_n${N}_*.json; do python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], d['value'], d['ms_per_step'])" $f; done; for f in gpurun_out/bench_n${N}_*.log; do tail -n 3 $f; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29512 \
  scripts/bench_compose.py > gpurun_out/compose_c4_n${N}.json 2> gpurun_out/compose_c4_n${N}.log
echo "compose rc=$?" >> gpurun_out/compose_c4_n${N}.log
cat gpurun_out/compose_c4_n${N}.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29513 \
  scripts/bench_compose.py --w 3840 --h 2160 > gpurun_out/compose_4k_n${N}.json 2> gpurun_out/compose_4k_n${N}.log
cat gpurun_out/compose_4k_n${N}.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29514 \
  scripts/bench_compose.py --scene compact > gpurun_out/compose_c4c_n${N}.json 2> gpurun_out/compose_c4c_n${N}.log
cat gpurun_out/compose_c4c_n${N}.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29515 \
  scripts/bench_compose.py --scene bricks --w 3840 --h 2160 --sources 16 > gpurun_out/compose_c3_n${N}.json 2> gpurun_out/compose_c3_n${N}.log
cat gpurun_out/compose_c3_n${N}.json
if [ "$N" -ge 3 ]; then
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=3 --master-addr=127.0.0.1 --master-port=29516 \
  scripts/bench_compose.py --sources 6 > gpurun_out/compose_c4s6_n3.json 2> gpurun_out/compose_c4s6_n3.log
cat gpurun_out/compose_c4s6_n3.json
fi
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29517 \
  scripts/bench_stream.py > gpurun_out/stream_n${N}.json 2> gpurun_out/stream_n${N}.log
cat gpurun_out/stream_n${N}.json
