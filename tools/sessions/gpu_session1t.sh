mkdir -p gpurun_out
timeout 300 python tools/ncu_one.py --config torus4x4x4 --m 4194304 --schedule chain:262144 --warmup 1 > gpurun_out/t1_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none -k regex:a2a -s 1 -c 1 -o gpurun_out/ncu1_torus_chain \
   python tools/ncu_one.py --config torus4x4x4 --m 4194304 --schedule chain:262144 --warmup 1 > gpurun_out/t1_ncu.log 2>&1
echo "ncu rc=$?"
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/t1_pytest_gpu_1gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t1_pytest_gpu_1gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/t1_bench.json 2> gpurun_out/t1_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/t1_ref.json 2> gpurun_out/t1_ref.err; echo "ref rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t1_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/t1_smoke.log | tail -2
