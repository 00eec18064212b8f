mkdir -p gpurun_out
set -x
python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "leaf or fused or config or golden or known or exhaustive or band" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
for c in 2 3; do python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo bench$c rc=$?; done
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench5 rc=$?
