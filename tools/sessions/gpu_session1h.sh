mkdir -p gpurun_out
C="gk8_2:16777216@chaind:262144,torus4x4x4:4194304@chaind:262144"
run() { # tag env ctas
  env $2 timeout 600 python tools/sweep.py --steps 20 --num-ctas $3 --cases "$C" --out gpurun_out/h1_$1.jsonl > gpurun_out/h1_$1.log 2>&1; echo "$1 rc=$?"
}
run base A2A_ENGINE=tma:32768:6 0
run c16s12 A2A_ENGINE=tma:16384:12 0
run c16s6x2 A2A_ENGINE=tma:16384:6 296
run c16s5x2 A2A_ENGINE=tma:16384:5 296
run c64s3 A2A_ENGINE=tma:65536:3 0
run c8s24 A2A_ENGINE=tma:8192:24 0
run c32s3x2 A2A_ENGINE=tma:32768:3 296
