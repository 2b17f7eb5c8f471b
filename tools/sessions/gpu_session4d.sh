mkdir -p gpurun_out
# launch list of the N=1 bench command (same command, plain run first)
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/d4_bench_plain.json 2> gpurun_out/d4_bench_plain.err &&
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
   --log-file gpurun_out/d4_launches_bench_G1.csv python bench.py --steps 5 --warmup 3 > gpurun_out/d4_bench_ncu.log 2>&1
echo "launches rc=$?"
bash tools/gpu_ncu_nvlink.sh > gpurun_out/d4_ncu_nvlink.log 2>&1; echo "nvlink rc=$?"; cat gpurun_out/d4_ncu_nvlink.log
