# multi-GPU executor kernel under ncu: rank 0 profiled (NVLink tx/rx, DRAM bytes, duration),
# the other ranks run the same all-to-alls without ncu
mkdir -p gpurun_out
M="nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for G in 2 4; do
  D=/tmp/a2a_ncu_rdv_$G; rm -rf $D
  # plain run of every rank first: must exit 0 before profiling
  for r in $(seq 0 $((G-1))); do
    timeout 300 python tools/ncu_rank.py --rank $r --world $G --dir $D --phase pre > gpurun_out/ncu_nvl_G${G}_pre_r$r.log 2>&1 &
  done
  wait; echo "pre G=$G: $(grep -c ok gpurun_out/ncu_nvl_G${G}_pre_r*.log | tr '\n' ' ')"
  for r in $(seq 1 $((G-1))); do
    ( timeout 300 python tools/ncu_rank.py --rank $r --world $G --dir $D --phase plain --optional;
      timeout 300 python tools/ncu_rank.py --rank $r --world $G --dir $D --phase ncu ) > gpurun_out/ncu_nvl_G${G}_peer_r$r.log 2>&1 &
  done
  timeout 600 ncu --metrics $M --clock-control none -k regex:a2a -s 3 -c 1 --csv \
      --log-file gpurun_out/ncu_nvl_G${G}_r0.csv \
      python tools/ncu_rank.py --rank 0 --world $G --dir $D > gpurun_out/ncu_nvl_G${G}_r0.log 2>&1
  echo "ncu G=$G rc=$?"
  wait
done
