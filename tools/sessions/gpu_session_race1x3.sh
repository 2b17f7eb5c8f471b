# race tests three times back to back (flakiness check of the mutation assertion)
mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_race.py -m gpu -q > gpurun_out/race_x$i.log 2>&1; echo "run$i rc=$? $(tail -1 gpurun_out/race_x$i.log)"; done
