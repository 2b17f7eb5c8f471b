# device-side race hunting: perturbed interleavings + mutation self-test, 1 and 2 GPUs;
# bench N=1 to check the perturbation branch costs nothing when off
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm --format=csv > gpurun_out/race_smi.txt
timeout 900 python -m pytest tests/test_gpu_race.py -m gpu -q -x > gpurun_out/race_1gpu.log 2>&1; echo "race1 rc=$?"
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -x -k "perturbed or mutation" > gpurun_out/race_2gpu.log 2>&1; echo "race2 rc=$?"
timeout 600 python bench.py > gpurun_out/race_bench1.json 2> gpurun_out/race_bench1.err; echo "bench rc=$?"
