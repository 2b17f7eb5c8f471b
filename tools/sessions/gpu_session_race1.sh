# device-side race hunting on one GPU (longer tail naps)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_race.py -m gpu -q -rA > gpurun_out/race_1gpu_c.log 2>&1; echo "race1 rc=$?"
