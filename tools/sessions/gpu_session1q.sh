mkdir -p gpurun_out
timeout 900 python tools/sweep.py --steps 20 --cases "gk8_2:16777216@chain:262144,torus4x4x4:4194304@chain:262144,hypercube3:16777216@chain:262144,gk64_4:1048576@chain:262144,gk8_2:16777216@chaind:262144,torus4x4x4:4194304@chaind:262144" --out gpurun_out/q1_chain.jsonl > gpurun_out/q1_chain.log 2>&1; echo "sweep rc=$?"
