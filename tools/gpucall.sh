mkdir -p gpurun_out
python tools/timeline.py 5 32768 gpurun_out/tl5.json > gpurun_out/timeline_cfg5.txt 2>&1
python tools/tl_attr.py gpurun_out/tl5.json 6
python tools/timeline.py 1 1024 gpurun_out/tl1.json > gpurun_out/timeline_cfg1.txt 2>&1
python tools/tl_attr.py gpurun_out/tl1.json 6
python tools/tl_window.py gpurun_out/tl1.json 0 2 | grep node128
python tools/timeline.py 4 16384 gpurun_out/tl4.json > gpurun_out/timeline_cfg4.txt 2>&1
python tools/tl_attr.py gpurun_out/tl4.json 8
rm gpurun_out/tl1.json gpurun_out/tl4.json; gzip -f gpurun_out/tl5.json
