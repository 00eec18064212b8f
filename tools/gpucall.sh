# Scratch command file for gpurun (what the last call ran); the round-end pass is tools/final_measure.sh.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/pytest_pq.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pq.log
for i in 1 2; do
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python -c "
import json,os;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['verified']['reconstruction_mismatches'], d['gpu_launches_per_step'], d['host_syncs_per_step'])"
done
