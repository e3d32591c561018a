#!/bin/bash
# ncu --set full captures (source-level) of one kernel for the default library
# and each prebuilt variant given as an argument (EQC_LIB), under gpurun.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-ab}
K=${KREGEX:-depth_rle}
python scripts/prof_step.py --steps 2 --which step > gpurun_out/p.log 2>&1 || { cat gpurun_out/p.log; exit 1; }
i=0
for lib in paper_1902_08755_b200/libeqc.so "$@"; do
  EQC_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
      -o gpurun_out/prof_${TAG}$i -f python scripts/prof_step.py --steps 1 --which step > gpurun_out/ncu_${TAG}$i.log 2>&1
  tail -1 gpurun_out/ncu_${TAG}$i.log
  i=$((i+1))
done
