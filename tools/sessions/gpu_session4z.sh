# final validation: full GPU suite on 4 GPUs, bench at 1/2/4 GPUs, reference arm, smoke
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/z4_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/z4_smoke.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/z4_pytest_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/z4_pytest_all.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/z4_bench1.json 2> gpurun_out/z4_bench1.err; echo "bench1 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29961 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/z4_bench2.json 2> gpurun_out/z4_bench2.err; echo "bench2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29962 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/z4_bench4.json 2> gpurun_out/z4_bench4.err; echo "bench4 rc=$?"
timeout 600 $TR --nproc-per-node 4 --master-port 29963 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/z4_ref4.json 2> gpurun_out/z4_ref4.err; echo "ref4 rc=$?"
