mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 3000 $TR --nproc-per-node 4 --master-port 29995 tools/sweep.py --lowering auto --schedule auto --steps 10 \
    --cases gk256_4:1048576,gk256_4_h2:1048576 --out gpurun_out/u4_gk256_G4.jsonl > gpurun_out/u4_gk256_G4.log 2>&1; echo "gk256 rc=$?"
