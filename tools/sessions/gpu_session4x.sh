mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for G in 2 4; do
  timeout 900 $TR --nproc-per-node $G --master-port $((29940+G)) tools/sweep.py --lowering balanced --steps 20 \
    --cases "torus4x4x4:4194304@chain:262144,torus4x4x4:4194304@mix:1048576,gk8_2:16777216@chain:262144,hypercube3:16777216@chain:262144" \
    --out gpurun_out/x4_chain_G${G}.jsonl > gpurun_out/x4_chain_G${G}.log 2>&1; echo "g$G rc=$?"
done
timeout 600 python tools/sweep.py --steps 20 --cases "gk8_2:16777216@chain:262144,torus4x4x4:4194304@chain:262144" --out gpurun_out/x4_chain_G1.jsonl > gpurun_out/x4_chain_G1.log 2>&1; echo "g1 rc=$?"
