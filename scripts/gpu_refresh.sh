#!/bin/bash
# Round-2 refresh on one GPU (under gpurun): full GPU suite, smoke, the N=1
# bench line, the bench's ncu launch list, and --set full captures of the
# step's three kernels (scripts/prof_step.py).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
TAG=${TAG:-r2c}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_${TAG}.log
tail -3 gpurun_out/pytest_${TAG}.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.log; cat gpurun_out/bench_${TAG}.json
TAG=bench_${TAG} bash scripts/gpu_bench_prof.sh
python scripts/prof_step.py --steps 2 --which step > gpurun_out/p.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"depth_rle|rle_encode3|rle_compact3" -c 3 \
    -o gpurun_out/prof_${TAG} -f python scripts/prof_step.py --steps 1 --which step > gpurun_out/ncu_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}.log
