mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -x -q -m gpu -k "ll128 and not eight and not multiprocess" > gpurun_out/s4b_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4b_pytest.log
timeout 900 $TR --nproc-per-node 4 --master-port 29991 tools/sweep.py --steps 20 \
    --cases "hypercube3:262144@ll128,hypercube3:1048576@ll128,hypercube3:4194304@ll128,gk8_2:1048576@ll128,gk8_2:4194304@ll128" \
    --out gpurun_out/s4b_ll128.jsonl > gpurun_out/s4b_ll128.log 2>&1; echo "sweep rc=$?"
timeout 900 python -m pytest tests -x -q -m gpu -k "multiprocess_ll" > gpurun_out/s4b_pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -2 gpurun_out/s4b_pytest_multi.log
