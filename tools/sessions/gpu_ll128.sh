mkdir -p gpurun_out
timeout 600 python tools/ll128_stress.py --epochs 4000 --lines 65536 > gpurun_out/ll128_stress.json 2> gpurun_out/ll128_stress.err; echo "stress rc=$?"
timeout 600 python tools/ll128_stress.py --epochs 40000 --lines 4096 > gpurun_out/ll128_stress_small.json 2>> gpurun_out/ll128_stress.err; echo "stress2 rc=$?"
cat gpurun_out/ll128_stress.json gpurun_out/ll128_stress_small.json
timeout 1500 python -m pytest tests -x -q -m gpu -k "ll" > gpurun_out/ll128_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/ll128_pytest.log
