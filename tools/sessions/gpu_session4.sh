# 4-GPU session: multi-GPU parity, bench at 2/4 GPUs, hop vs balanced lowering A/B
set -x
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi topo -m > gpurun_out/g4_topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/g4_pytest_multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/g4_rc.txt
timeout 600 $TR --nproc-per-node 2 --master-port 29510 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/g4_bench2.json 2> gpurun_out/g4_bench2.err; echo "bench2 rc=$?" >> gpurun_out/g4_rc.txt
timeout 600 $TR --nproc-per-node 4 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/g4_bench4.json 2> gpurun_out/g4_bench4.err; echo "bench4 rc=$?" >> gpurun_out/g4_rc.txt
for L in hop balanced; do
  for G in 2 4; do
    timeout 900 $TR --nproc-per-node $G --master-port $((29520+G)) tools/sweep.py --lowering $L --schedule auto --steps 10 \
      --cases gk8_2:16777216,hypercube3:16777216,hypercube3:4194304,torus4x4x4:4194304,gk256_4:1048576 \
      --out gpurun_out/g4_ab_${L}_G${G}.jsonl > gpurun_out/g4_ab_${L}_G${G}.log 2>&1; echo "ab $L $G rc=$?" >> gpurun_out/g4_rc.txt
  done
done
cat gpurun_out/g4_rc.txt
