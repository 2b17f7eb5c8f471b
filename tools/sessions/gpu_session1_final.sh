# last 1-GPU validation of the round: the driver's round-end commands
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f1_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f1_smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/f1_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/f1_pytest.log
timeout 900 python bench.py > gpurun_out/f1_bench.json 2> gpurun_out/f1_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/f1_ref.json 2> gpurun_out/f1_ref.err; echo "ref rc=$?"
