mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu -k "chain" > gpurun_out/g1_pytest_chain.log 2>&1; echo "pytest chain rc=$?"; tail -3 gpurun_out/g1_pytest_chain.log
timeout 900 python tools/sweep.py --schedule auto --steps 20 \
    --cases "gk8_2:16777216@chaind:262144,gk8_2:16777216@chaind:524288,gk8_2:16777216@chaind:131072,gk8_2:16777216@chain:524288,torus4x4x4:4194304@chaind:262144,hypercube3:16777216@chaind:262144,gk64_4:1048576@chaind:262144" \
    --out gpurun_out/g1_sweep_chaind.jsonl > gpurun_out/g1_sweep_chaind.log 2>&1; echo "sweep rc=$?"
timeout 300 python tools/ncu_one.py --config gk8_2 --m 16777216 --schedule chaind:262144 > gpurun_out/g1_ncu_chaind_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:a2a -s 2 -c 1 \
     -o gpurun_out/ncu1_gk8_2_chaind python tools/ncu_one.py --config gk8_2 --m 16777216 --schedule chaind:262144 > gpurun_out/g1_ncu_chaind.log 2>&1
echo "ncu chaind rc=$?"
