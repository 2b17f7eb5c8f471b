mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -x -q -m gpu -k "chain" > gpurun_out/i4_pytest_chain.log 2>&1; echo "pytest chain rc=$?"; tail -3 gpurun_out/i4_pytest_chain.log
for G in 2 4; do
  timeout 1500 $TR --nproc-per-node $G --master-port $((29900+G)) tools/sweep.py --lowering auto --schedule auto --steps 20 \
    --cases gk8_2:16777216,torus4x4x4:4194304,hypercube3:16777216,hypercube3:4194304 \
    --out gpurun_out/i4_sweep_G${G}.jsonl > gpurun_out/i4_sweep_G${G}.log 2>&1; echo "sweep $G rc=$?"
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/i4_bench1.json 2> gpurun_out/i4_bench1.err; echo "bench1 rc=$?"
