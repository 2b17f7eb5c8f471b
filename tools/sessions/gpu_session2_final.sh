# final build, two GPUs: every multi-GPU test that fits 2 GPUs, then the 2-GPU bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/f2_multi.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/f2_multi.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29971 bench.py --gpus 2 > gpurun_out/f2_bench2.json 2> gpurun_out/f2_bench2.err; echo "bench2 rc=$?"
