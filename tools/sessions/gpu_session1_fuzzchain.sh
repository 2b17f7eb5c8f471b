# random schedules through the chain kernel (32-byte ring, all-thread path; LSU) on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fuzz.py -q -m gpu -k random_schedule_gpu > gpurun_out/fuzzchain.log 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/fuzzchain.log
