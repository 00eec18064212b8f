mkdir -p gpurun_out
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_plduq_smem -s 40 -c 1 -f -o gpurun_out/plduq_smem python tools/one_factorization.py 5 32768 > gpurun_out/ncu_smem.log 2>&1; echo rc=$?
tail -2 gpurun_out/ncu_smem.log
