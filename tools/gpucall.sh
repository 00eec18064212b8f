mkdir -p gpurun_out
rm -f gpurun_out/plduq_calls.txt
FFB_PLDUQ_TRACE=gpurun_out/plduq_calls.txt python tools/one_factorization.py 5 32768 > /dev/null 2>&1
FFB_PLDUQ_TRACE=gpurun_out/plduq_calls.txt python tools/one_factorization.py 5 32768 > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/pytest_pq.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_pq.log
run() {
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python -c "
import json,os;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print('$1', d['ms_per_step'],d['verified']['reconstruction_mismatches'], d['gpu_launches_per_step'], d['host_syncs_per_step'])"
}
run default
FFB_PLDUQ_NO_SMEM=1 run off
