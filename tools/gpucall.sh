mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -m gpu -q -x -k "8388593 or config or golden or known or exhaustive or random or bit_exact or fused" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg3.json 2>/dev/null; echo rc=$?
