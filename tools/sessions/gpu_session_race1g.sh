# race tests with the gated mutation bit, plus smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python -m pytest tests/test_gpu_race.py tests/test_plan.py -m gpu -q > gpurun_out/race_gated.log 2>&1; echo "race rc=$? $(tail -1 gpurun_out/race_gated.log)"
