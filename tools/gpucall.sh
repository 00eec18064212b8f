# Scratch command file for gpurun (what the last call ran); the round-end pass is tools/final_measure.sh.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench rc=$?
for c in 1 2 3 4; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo cfg$c rc=$?
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 30000 --csv --log-file gpurun_out/ncu_launches_cfg5.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/ncu_launches_cfg5.csv > gpurun_out/ncu_launches_cfg5_summary.txt 2>&1
gzip -f gpurun_out/ncu_launches_cfg5.csv
python tools/timeline.py 5 32768 gpurun_out/tl5.json > gpurun_out/timeline_cfg5.txt 2>&1
python tools/tl_attr.py gpurun_out/tl5.json 45 > gpurun_out/timeline_cfg5_attr.txt
rm -f gpurun_out/tl5.json
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
