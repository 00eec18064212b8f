mkdir -p gpurun_out
python -m pytest tests/test_gemm_gpu.py tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_cfg5.json 2>/dev/null; echo rc=$?
python tools/gemm_bench.py 16384 16384 4096 --path tc > gpurun_out/tcp_iso.json 2>&1 && ncu --set full --clock-control none -k regex:k_gemm_i8_tcp -c 1 --launch-skip 1 -o gpurun_out/tcp_iso_ncu python tools/gemm_bench.py 16384 16384 4096 --path tc --reps 1 > gpurun_out/tcp_ncu.log 2>&1; echo ncu1 rc=$?
python tools/large_prime_bench.py --nodes 8192 --dgemm-only --out /tmp/x.json && ncu --set full --clock-control none -k regex:Kernel2 -c 1 --launch-skip 1 -o gpurun_out/dgemm_ncu python tools/large_prime_bench.py --nodes 8192 --dgemm-only --out /tmp/y.json > gpurun_out/dgemm_ncu.log 2>&1; echo ncu2 rc=$?
