mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -k "chain and not multiprocess and not eight" > gpurun_out/p1_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/p1_pytest.log
timeout 900 python tools/sweep.py --steps 20 --cases "gk8_2:16777216@chain:262144,torus4x4x4:4194304@chain:262144,hypercube3:16777216@chain:262144,gk64_4:1048576@chain:262144,gk8_2:16777216@chaind:262144" --out gpurun_out/p1_chain.jsonl > gpurun_out/p1_chain.log 2>&1; echo "sweep rc=$?"
