mkdir -p gpurun_out
timeout 900 python tools/ll128_stress.py --epochs 4000 --lines 65536 > gpurun_out/ll128_stress.json 2> gpurun_out/ll128_stress.err; echo "stress rc=$?"
timeout 900 python tools/ll128_stress.py --epochs 20000 --lines 4096 > gpurun_out/ll128_stress_small.json 2>> gpurun_out/ll128_stress.err; echo "stress2 rc=$?"
cat gpurun_out/ll128_stress.json gpurun_out/ll128_stress_small.json
