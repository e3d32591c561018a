#!/bin/bash
# A/B iteration: selected GPU parity tests, then scripts/ab_encode.py over the
# given prebuilt variants / -D specs.  Run under gpurun.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-fused or bench_step or depth_rle or p2p or smoke}" > gpurun_out/pytest_ab.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
tail -5 gpurun_out/pytest_ab.log
timeout 900 python scripts/ab_encode.py "$@" > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
