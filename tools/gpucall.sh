mkdir -p gpurun_out
python -m pytest tests/test_fullsize_gpu.py -m gpu -q > gpurun_out/pytest_fullsize.log 2>&1; echo pytest rc=$?
