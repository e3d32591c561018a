#!/bin/bash
# One ncu --set full capture of the fused v1 encoder (under gpurun), source-level.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-e3}
python scripts/prof_step.py --steps 2 --which step > gpurun_out/p.log 2>&1 || { cat gpurun_out/p.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-rle_encode3} -c 1 \
    -o gpurun_out/prof_${TAG} -f python scripts/prof_step.py --steps 1 --which step > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
