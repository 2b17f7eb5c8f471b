mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="hypercube3:4096@ll,hypercube3:16384@ll,hypercube3:4096@ll@16,hypercube3:65536@ll,hypercube3:262144@ll128"
timeout 900 $TR --nproc-per-node 4 --master-port 29951 tools/sweep.py --steps 30 --cases "$C" --out gpurun_out/j4_coop.jsonl > gpurun_out/j4_coop.log 2>&1; echo "coop rc=$?"
A2A_NONCOOP=1 timeout 900 $TR --nproc-per-node 4 --master-port 29952 tools/sweep.py --steps 30 --cases "$C" --out gpurun_out/j4_noncoop.jsonl > gpurun_out/j4_noncoop.log 2>&1; echo "noncoop rc=$?"
