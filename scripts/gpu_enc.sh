#!/bin/bash
# Encoder iteration: codec parity tests + short bench.  Run under gpurun.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-rle or bench_step or encoder or fused or target or smoke}" > gpurun_out/pytest_enc.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_enc.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_enc.json 2> gpurun_out/bench_enc.log
echo "bench rc=$?" >> gpurun_out/bench_enc.log
tail -15 gpurun_out/pytest_enc.log; python -c "
import json; j=json.load(open('gpurun_out/bench_enc.json')); print(j['ms_per_step'], j['kernels'])" ; tail -3 gpurun_out/bench_enc.log
