# 4-GPU: LL128 stress, hypercube size sweep (config 5) and the large configs with LL128 among the candidates
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python tools/ll128_stress.py --epochs 4000 --lines 65536 > gpurun_out/s4_ll128_stress.json 2> gpurun_out/s4_ll128_stress.err; echo "stress rc=$?"
timeout 300 python tools/ll128_stress.py --epochs 40000 --lines 4096 > gpurun_out/s4_ll128_stress_small.json 2>> gpurun_out/s4_ll128_stress.err; echo "stress2 rc=$?"
for G in 4 2; do
  timeout 1500 $TR --nproc-per-node $G --master-port $((29600+G)) tools/sweep.py --preset hypercube --lowering auto --schedule auto --steps 10 \
    --out gpurun_out/s4_hypercube_G${G}.jsonl > gpurun_out/s4_hypercube_G${G}.log 2>&1; echo "hyper $G rc=$?"
done
timeout 1200 $TR --nproc-per-node 4 --master-port 29611 tools/sweep.py --lowering auto --schedule auto --steps 10 \
  --cases gk8_2:16777216,torus4x4x4:4194304,gk8_2:1048576 --out gpurun_out/s4_large_G4.jsonl > gpurun_out/s4_large_G4.log 2>&1; echo "large rc=$?"
cat gpurun_out/s4_ll128_stress.json gpurun_out/s4_ll128_stress_small.json
