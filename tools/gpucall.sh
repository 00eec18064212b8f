mkdir -p gpurun_out
python tools/leaf_bench.py 131 2>&1 | tail -5
python tools/node_stamps.py 1 1024 | head -4
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/pytest_pq.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pq.log
for c in 5 4 3; do
python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print('cfg', $c, d['ms_per_step'],d['verified']['reconstruction_mismatches'], d['gpu_launches_per_step'])"
done
