mkdir -p gpurun_out
set -x
python -m pytest tests -m gpu -q --deselect "tests/test_fullsize_gpu.py::test_full_size_bit_exact[5]" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
for c in 2 3; do python bench.py --config $c --steps 5 --warmup 3 --no-e2e-u64 > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err; echo bench$c rc=$?; done
python bench.py --steps 5 --warmup 3 --no-e2e-u64 --no-cpu > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench5 rc=$?
python tools/timeline.py 3 8192 gpurun_out/timeline_cfg3.json > gpurun_out/timeline_cfg3.txt 2>&1; python tools/tl_attr.py gpurun_out/timeline_cfg3.json 30 > gpurun_out/tl_attr_cfg3.txt 2>&1; gzip -f gpurun_out/timeline_cfg3.json
python tools/timeline.py 5 32768 gpurun_out/timeline_cfg5.json > gpurun_out/timeline_cfg5.txt 2>&1; python tools/tl_attr.py gpurun_out/timeline_cfg5.json 30 > gpurun_out/tl_attr_cfg5.txt 2>&1; gzip -f gpurun_out/timeline_cfg5.json
