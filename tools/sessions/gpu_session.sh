set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/g1_info.txt 2>&1
free -g >> gpurun_out/g1_info.txt; nproc >> gpurun_out/g1_info.txt
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/g1_pytest_configs.log 2>&1; echo "configs rc=$?" >> gpurun_out/g1_rc.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc=$?" >> gpurun_out/g1_rc.txt
timeout 1500 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_configs.py > gpurun_out/g1_pytest_all.log 2>&1; echo "all rc=$?" >> gpurun_out/g1_rc.txt
cat gpurun_out/g1_rc.txt
