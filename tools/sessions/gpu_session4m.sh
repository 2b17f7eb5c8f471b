# full GPU suite on 4 GPUs (1-GPU tests + multi-GPU tests), then the bench at 1/2/4 GPUs
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 3000 python -m pytest tests -q -m gpu -x > gpurun_out/m4_pytest_all.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/m4_pytest_all.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/m4_bench1.json 2> gpurun_out/m4_bench1.err; echo "bench1 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29971 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/m4_bench2.json 2> gpurun_out/m4_bench2.err; echo "bench2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29972 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/m4_bench4.json 2> gpurun_out/m4_bench4.err; echo "bench4 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/m4_ref1.json 2> gpurun_out/m4_ref1.err; echo "ref rc=$?"
