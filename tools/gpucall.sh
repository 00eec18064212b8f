mkdir -p gpurun_out
python -m pytest tests/test_gemm_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "limb or 8388593 or kernels or config" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
python tools/gemm_bench.py 128 128 128 256 256 256 512 512 512 1024 1024 1024 4096 4096 4096 --p 8388593 --path tc --reps 5 > gpurun_out/gemm_lp_tc.jsonl 2>&1
python bench.py --config 3 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg3.json 2>/dev/null; echo rc=$?
