mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench rc=$?
for c in 1 2 3 4; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo cfg$c rc=$?
done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
