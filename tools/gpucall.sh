mkdir -p gpurun_out
python tools/pluq_vs_ldlt.py 2048 4096 > gpurun_out/pluq_vs_ldlt.jsonl 2> gpurun_out/pluq_vs_ldlt.err; echo rc=$?
cat gpurun_out/pluq_vs_ldlt.jsonl; tail -5 gpurun_out/pluq_vs_ldlt.err
for b in 128 160 192 256; do
FFB_PLDUQ_B=$b python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; echo rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print($b, d['ms_per_step'],d['verified']['reconstruction_mismatches'], d['gpu_launches_per_step'])"
done
FFB_PLDUQ_B=192 timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "plduq or config or golden" > gpurun_out/pytest_pq.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pq.log
