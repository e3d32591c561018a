#!/bin/bash
# ncu captures under gpurun: launch list (shares) + full sets of the top kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
python scripts/prof_step.py --steps 3 > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/prof_plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python scripts/prof_step.py --steps 3 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-rle_encode|depth_rle|rle_decode|depth_composite|blend}" -s ${SKIP:-0} -c ${COUNT:-6} \
    -o gpurun_out/prof_${TAG} -f python scripts/prof_step.py --steps 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
