mkdir -p gpurun_out
python tools/pq_kernel_bench.py 25,8192,20 2>&1 | grep -v crp | cut -c1-300
