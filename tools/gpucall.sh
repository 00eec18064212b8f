mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -q -x --deselect "tests/test_fullsize_gpu.py::test_full_size_bit_exact[5]" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
python bench.py --steps 5 --warmup 3 --no-e2e-u64 --no-cpu > gpurun_out/bench_band.json 2> gpurun_out/bench_band.err; echo bench rc=$?
FFB_NO_BAND=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_noband.json 2> gpurun_out/bench_noband.err; echo bench rc=$?
python tools/node_profile.py 3 8192 > gpurun_out/node_profile_cfg3.txt 2>&1
python tools/timeline.py 3 8192 gpurun_out/timeline_cfg3.json > gpurun_out/timeline_cfg3.txt 2>&1; python tools/tl_attr.py gpurun_out/timeline_cfg3.json 30 > gpurun_out/tl_attr_cfg3.txt 2>&1; gzip -f gpurun_out/timeline_cfg3.json
python tools/large_prime_bench.py --nodes 8192 --dgemm-only --out /tmp/x.json && ncu --set full --clock-control none -k regex:"gemm" -c 1 --launch-skip 2 -o gpurun_out/dgemm_ncu python tools/large_prime_bench.py --nodes 8192 --dgemm-only --out /tmp/y.json > gpurun_out/dgemm_ncu.log 2>&1; echo ncu rc=$?
