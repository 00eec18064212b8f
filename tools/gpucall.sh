mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fullsize_gpu.py -m gpu -q -x -k "symmetry_verdict or properties" > gpurun_out/pytest_sym.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_sym.log
for ov in 1 0; do
if [ $ov = 0 ]; then export FFB_NO_START_OVERLAP=1; fi
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; echo rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print('overlap', $ov, d['ms_per_step'],d['verified']['reconstruction_mismatches'], d['gpu_launches_per_step'])"
done
unset FFB_NO_START_OVERLAP
python bench.py --config 4 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print('cfg4', d['ms_per_step'],d['verified']['reconstruction_mismatches'])"
