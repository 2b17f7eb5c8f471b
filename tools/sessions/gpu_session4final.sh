mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 $TR --nproc-per-node 4 --master-port 29901 tools/sweep.py --preset hypercube --lowering auto --schedule auto --steps 20 \
    --out gpurun_out/final_hypercube_G4.jsonl > gpurun_out/final_hypercube_G4.log 2>&1; echo "hyper4 rc=$?"
