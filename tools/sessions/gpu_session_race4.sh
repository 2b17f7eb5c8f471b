# device-side race hunting across 4 GPUs (perturbed interleavings + mutation self-test)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -m gpu -q -rA -k "perturbed or mutation" > gpurun_out/race_4gpu.log 2>&1; echo "race4 rc=$?"
