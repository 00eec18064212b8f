mkdir -p gpurun_out
for v in 148 300 600 1200; do FFB_MMA_SPLIT_CTAS=$v python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_split$v.json 2>/dev/null; echo $v rc=$?; done
