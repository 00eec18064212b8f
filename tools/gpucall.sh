mkdir -p gpurun_out
python tools/timeline.py 5 32768 gpurun_out/tl5.json > gpurun_out/timeline_cfg5.txt 2>&1
rm -f gpurun_out/tl5.json
FFB_HOST_STATS=1 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/host_stats.txt
tail -5 gpurun_out/host_stats.txt
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "detection_cap or adaptive" 2>&1 | tail -2
