mkdir -p gpurun_out
set -x
python tools/cpu_reference_configs.py > gpurun_out/cpu_ref.log 2>&1 &
CPUPID=$!
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_gemm|k_rankk" --launch-skip 1 --csv --log-file gpurun_out/ncu_gemm.csv python tools/one_factorization.py 5 32768 > gpurun_out/ncu_gemm.log 2>&1; echo ncu rc=$?
wait $CPUPID; echo cpu rc=$?
