#!/bin/bash
# ncu launch list (time + DRAM bytes per kernel) of scripts/prof_step.py --which step (under gpurun).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-cur}
python scripts/prof_step.py --steps 2 --which ${WHICH:-step} > gpurun_out/p.log 2>&1 || { cat gpurun_out/p.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv python scripts/prof_step.py --steps 2 --which ${WHICH:-step} > /dev/null 2>&1
python - "$TAG" <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")))
h = None; agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if 'Kernel Name' in r: h = r; continue
    if h and len(r) == len(h):
        d = dict(zip(h, r)); agg[d['Kernel Name'][:60]][d['Metric Name']].append(float(d['Metric Value'].replace(',', '')))
for k, v in agg.items():
    t = v['gpu__time_duration.sum']; rd = v['dram__bytes_read.sum']; wr = v['dram__bytes_write.sum']
    print(f"{k:60s} n={len(t)} us={sum(t)/len(t)/1e3:8.1f} rdMB={sum(rd)/len(rd)/1e6:7.1f} wrMB={sum(wr)/len(wr)/1e6:7.1f}")
PY
