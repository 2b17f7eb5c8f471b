mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests -x -q -m gpu -k "not chain and not gk256 and not torus4x4x4_4mib" > gpurun_out/v4_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/v4_pytest.log
C="hypercube3:4096@ll,hypercube3:16384@ll,hypercube3:4096@ll@16,hypercube3:65536@ll,hypercube3:262144@ll128,hypercube3:1048576@ll128"
timeout 900 $TR --nproc-per-node 4 --master-port 29997 tools/sweep.py --steps 30 --cases "$C" --out gpurun_out/v4_tiny_G4.jsonl > gpurun_out/v4_tiny_G4.log 2>&1; echo "tiny4 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29998 tools/sweep.py --steps 30 --cases "$C" --out gpurun_out/v4_tiny_G2.jsonl > gpurun_out/v4_tiny_G2.log 2>&1; echo "tiny2 rc=$?"
