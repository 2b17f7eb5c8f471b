# one GPU: ncu --set full of the executor kernel for the N=1 bench workloads (+ LL128 on 1 GPU)
mkdir -p gpurun_out
run() {  # name config m schedule
  timeout 300 python tools/ncu_one.py --config $2 --m $3 --schedule $4 > gpurun_out/ncu1_$1_plain.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:a2a -s 2 -c 1 \
     -o gpurun_out/ncu1_$1 python tools/ncu_one.py --config $2 --m $3 --schedule $4 > gpurun_out/ncu1_$1.log 2>&1
  echo "$1 rc=$?"
}
run gk8_2_mix gk8_2 16777216 mix:1048576
run gk8_2_cp gk8_2 16777216 cp:1048576
run torus_cp torus4x4x4 4194304 cp:1048576
run hyper4m_ll128 hypercube3 4194304 ll128
run hyper1m_ll128 hypercube3 1048576 ll128
