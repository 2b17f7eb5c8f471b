mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -x -q -m gpu -k "ll128 and not eight" > gpurun_out/e4_pytest_ll128.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/e4_pytest_ll128.log
timeout 300 python tools/ll128_stress.py --epochs 4000 --lines 65536 > gpurun_out/e4_ll128_stress.json 2> gpurun_out/e4_ll128_stress.err; echo "stress rc=$?"; cat gpurun_out/e4_ll128_stress.json
timeout 1200 $TR --nproc-per-node 4 --master-port 29801 tools/sweep.py --lowering auto --schedule auto --steps 20 \
    --cases hypercube3:65536,hypercube3:262144,hypercube3:1048576,hypercube3:4194304,gk8_2:1048576,gk8_2:4194304 \
    --out gpurun_out/e4_hyper_G4.jsonl > gpurun_out/e4_hyper_G4.log 2>&1; echo "hyper4 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/e4_bench4.json 2> gpurun_out/e4_bench4.err; echo "bench4 rc=$?"
bash tools/gpu_ncu_nvlink.sh > gpurun_out/e4_ncu_nvlink.log 2>&1; echo "nvlink rc=$?"; cat gpurun_out/e4_ncu_nvlink.log
