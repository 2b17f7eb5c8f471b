mkdir -p gpurun_out
C="gk8_2:16777216@chain:262144,torus4x4x4:4194304@chain:262144,hypercube3:16777216@chain:262144"
timeout 600 python tools/sweep.py --steps 20 --cases "$C" --out gpurun_out/hint_off.jsonl > gpurun_out/hint_off.log 2>&1; echo "off rc=$?"
A2A_SYNC_MODE=66 timeout 600 python tools/sweep.py --steps 20 --cases "$C" --out gpurun_out/hint_on.jsonl > gpurun_out/hint_on.log 2>&1; echo "on rc=$?"
