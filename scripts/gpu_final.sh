#!/bin/bash
# Round-end style check: full GPU suite, smoke, N=1 bench (+ N-GPU bench when >1 GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/final_pytest_n${N}.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest_n${N}.log
tail -3 gpurun_out/final_pytest_n${N}.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.log; cat gpurun_out/final_bench_n1.json
if [ "$N" -gt 1 ]; then
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29541 bench.py --gpus $N > gpurun_out/final_bench_n${N}.json 2> gpurun_out/final_bench_n${N}.log; cat gpurun_out/final_bench_n${N}.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29542 bench.py --impl reference --gpus $N --steps 2 --warmup 1 > gpurun_out/final_ref_n${N}.json 2> gpurun_out/final_ref_n${N}.log; cat gpurun_out/final_ref_n${N}.json
fi
