mkdir -p gpurun_out
for L in 8192 16384 32768 65536; do
  timeout 120 python tools/ll128_stress.py --local-only --epochs 2000 --lines $L > gpurun_out/o4_stress_$L.json 2>&1; echo "lines $L rc=$?"; tail -1 gpurun_out/o4_stress_$L.json
done
timeout 1500 python -m pytest tests -x -q -m gpu -k "eight_ranks or self_copy_and_graph" > gpurun_out/o4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/o4_pytest.log
