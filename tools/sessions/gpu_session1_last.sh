# last check of the round on one GPU: build + smoke + the whole GPU suite with the final .so
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/l1_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/l1_smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/l1_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/l1_pytest.log
