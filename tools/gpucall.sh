mkdir -p gpurun_out
python tools/pq_kernel_bench.py 25,8192,20 25,8192,400 26,16384,33 32,16384,2000 16,4096,300 8,16384,5000 > gpurun_out/pq_bench.txt 2>&1
grep crp gpurun_out/pq_bench.txt | cut -c1-400
python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "plduq or config or golden" > gpurun_out/pytest_pq.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pq.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; echo rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['verified'])"
FFB_CF_SMEM=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q0.json 2>gpurun_out/bench_q0.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_q0.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['verified'])"
