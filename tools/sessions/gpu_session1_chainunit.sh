# chain unit-size sweep on one GPU (the candidate list fixes 256 KiB)
mkdir -p gpurun_out
C=""
for u in 131072 262144 524288 1048576 2097152 4194304; do C="$C,gk8_2:16777216@chain:$u"; done
for u in 262144 1048576; do C="$C,torus4x4x4:4194304@chain:$u,hypercube3:16777216@chain:$u,gk64_4:1048576@chain:$u"; done
timeout 600 python tools/sweep.py --steps 20 --no-nccl --cases "${C#,}" --out gpurun_out/chainunit.jsonl > gpurun_out/chainunit.log 2>&1; echo "sweep rc=$?"
