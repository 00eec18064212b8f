# Scratch command file for gpurun (what the last call ran); the round-end pass is tools/final_measure.sh.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_final.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu_final.log
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench rc=$?
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
