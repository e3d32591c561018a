"""Kernel shares of the step from an ncu launch list of bench.py
(scripts/gpu_bench_prof.sh): per kernel, mean cold-cache time per launch and
its share of (sum over the step's kernels), written to profiles/<tag>.md for
comparison with the bench line's per-kernel CUDA-event times.

    python scripts/launch_shares.py gpurun_out/launches_bench.csv profiles/launch_shares_r02.md
"""
import collections
import csv
import sys


def main():
    src, dst = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        per.setdefault((int(r[ii]), r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")),
                       {})[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(list)
    for (i, k), m in per.items():
        agg[k].append((m.get("gpu__time_duration.sum", 0) / 1e3,
                       (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6))
    ours = {k: v for k, v in agg.items() if not k.startswith("at::") and "nccl" not in k.lower()}
    tot = sum(sum(x[0] for x in v) / len(v) for v in ours.values())
    lines = ["# Kernel shares of the bench.py step (ncu launch list)", "",
             f"Source: `{src}` (`scripts/gpu_bench_prof.sh`: ncu --metrics gpu__time_duration.sum,"
             "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, bench.py --steps 2 --warmup 1). "
             "Cold-cache, serialised: compare shares with the bench line, not absolutes.", "",
             "| kernel | launches | mean us / launch | DRAM MB / launch | share of step |", "|---|---|---|---|---|"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(x[0] for x in kv[1]) / len(kv[1])):
        mt = sum(x[0] for x in v) / len(v)
        mb = sum(x[1] for x in v) / len(v)
        lines.append(f"| {k} | {len(v)} | {mt:.1f} | {mb:.1f} | {mt / tot:.3f} |")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
