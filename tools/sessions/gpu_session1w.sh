mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/w1_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/w1_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/w1_bench.json 2> gpurun_out/w1_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/w1_ref.json 2> gpurun_out/w1_ref.err; echo "ref rc=$?"
