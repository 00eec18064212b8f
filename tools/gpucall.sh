# Scratch command file for gpurun (what the last call ran); the round-end pass is tools/final_measure.sh.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "shared_memory or plduq or golden" 2>&1 | tail -2
run() {
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err
python -c "
import json,os;d=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1]);print('$1', d['ms_per_step'],d['verified']['reconstruction_mismatches'], d['gpu_launches_per_step'], d['host_syncs_per_step'])"
}
run default
FFB_PLDUQ_SMEM_RCAP=20 run rcap20
FFB_PLDUQ_SMEM_ROWS=1024 FFB_PLDUQ_SMEM_RCAP=20 run rows1024_rcap20
