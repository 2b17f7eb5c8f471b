# chain vs chaind (dead intermediate lines discarded from L2) on the three path configs, one GPU
mkdir -p gpurun_out
C="torus4x4x4:4194304@chain:262144,torus4x4x4:4194304@chaind:262144,gk8_2:16777216@chain:262144,gk8_2:16777216@chaind:262144,hypercube3:16777216@chain:262144,hypercube3:16777216@chaind:262144,gk64_4:1048576@chain:262144,gk64_4:1048576@chaind:262144"
timeout 600 python tools/sweep.py --steps 20 --no-nccl --cases "$C" --out gpurun_out/chaind3.jsonl > gpurun_out/chaind3.log 2>&1; echo "sweep rc=$?"
