mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/int8_peak.py > gpurun_out/int8_peak.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -k regex:k_gemm_i8_tcp --csv --log-file gpurun_out/ncu_tcp_instep.csv python tools/one_factorization.py 5 32768 > gpurun_out/ncu_tcp.log 2>&1; echo ncu rc=$?
