mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/pytest_pq.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pq.log
for sr in 200 320 448 640; do
FFB_PLDUQ_SEQ_ROWS=$sr python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; echo rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print($sr, d['ms_per_step'],d['verified']['reconstruction_mismatches'], d['gpu_launches_per_step'])"
done
