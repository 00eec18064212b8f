# Scratch command file for gpurun (what the last call ran); the round-end pass is tools/final_measure.sh.
mkdir -p gpurun_out
python tools/node_profile.py 5 32768 > gpurun_out/node_profile_cfg5.txt 2>&1; echo rc=$?
rm -f gpurun_out/plduq_calls.txt
FFB_PLDUQ_TRACE=gpurun_out/plduq_calls.txt python tools/one_factorization.py 5 32768 > /dev/null 2>&1
: > gpurun_out/plduq_calls.txt
FFB_PLDUQ_TRACE=gpurun_out/plduq_calls.txt python tools/one_factorization.py 5 32768 > /dev/null 2>&1
wc -l gpurun_out/plduq_calls.txt
