mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -x -q -m gpu -k "ll128 and not eight" > gpurun_out/c4_pytest_ll128.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/c4_pytest_ll128.log
timeout 300 python tools/ll128_stress.py --epochs 4000 --lines 65536 > gpurun_out/c4_ll128_stress.json 2> gpurun_out/c4_ll128_stress.err; echo "stress rc=$?"; cat gpurun_out/c4_ll128_stress.json
for G in 4 2; do
  timeout 1200 $TR --nproc-per-node $G --master-port $((29700+G)) tools/sweep.py --lowering auto --schedule auto --steps 20 \
    --cases hypercube3:4096,hypercube3:16384,hypercube3:65536,hypercube3:262144,hypercube3:1048576,hypercube3:4194304 \
    --out gpurun_out/c4_hyper_small_G${G}.jsonl > gpurun_out/c4_hyper_small_G${G}.log 2>&1; echo "hyper $G rc=$?"
done
bash tools/gpu_ncu_nvlink.sh > gpurun_out/c4_ncu.log 2>&1; echo "ncu rc=$?"; tail -12 gpurun_out/c4_ncu.log
