mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu -k "balanced or eight_ranks" > gpurun_out/r4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r4_pytest.log
