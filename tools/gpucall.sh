mkdir -p gpurun_out
python -m pytest tests/test_parity_gpu.py tests/test_gemm_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_green.json 2>gpurun_out/bench_green.err; echo rc=$?
FFB_NO_GREEN=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_nogreen.json 2>/dev/null; echo rc=$?
FFB_GREEN_RESERVE=32 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_green32.json 2>/dev/null; echo rc=$?
