cd "${GRAFT_REPO_ROOT}"
python -m paper_1902_08755_b200.build >/dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
for P in "" "--no-pipeline"; do
for X in raw; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29511 \
  bench.py --gpus $N --steps 50 --warmup 5 --no-cpu-baseline --exchange $X $P > gpurun_out/bench_n${N}_${X}${P}.json 2> gpurun_out/bench_n${N}_${X}${P}.log
python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], d['value'], d['ms_per_step'], d['e2e']['value'], d['compose_direct_send_latency_ms_rank0'])" gpurun_out/bench_n${N}_${X}${P}.json
done; done
