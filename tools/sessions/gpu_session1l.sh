mkdir -p gpurun_out
run() { # tag engine cases
  env A2A_ENGINE=$2 timeout 600 python tools/sweep.py --steps 20 --cases "$3" --out gpurun_out/l1_$1.jsonl > gpurun_out/l1_$1.log 2>&1; echo "$1 rc=$?"
}
C256="gk8_2:16777216@chain:262144,torus4x4x4:4194304@chain:262144"
C384="gk8_2:16777216@chain:393216,torus4x4x4:4194304@chain:393216"
C512="gk8_2:16777216@chain:524288,torus4x4x4:4194304@chain:524288"
run a32x6_256 tma:32768:6 "$C256"
run a64x3_256 tma:65536:3 "$C256"
run a64x3_512 tma:65536:3 "$C512"
run a48x4_384 tma:49152:4 "$C384"
run a32x6_384 tma:32768:6 "$C384"
run a96x2_384 tma:98304:2 "$C384"
timeout 300 python tools/ll128_stress.py --epochs 4000 --lines 65536 > gpurun_out/l1_ll128_stress.json 2> gpurun_out/l1_ll128_stress.err; echo "stress rc=$?"; cat gpurun_out/l1_ll128_stress.json
