# per-rank ncu captures of the multi-GPU executor kernel: NVLink tx/rx and DRAM bytes
mkdir -p gpurun_out
M="nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for G in 2 4; do
  rm -rf /tmp/a2a_ncu_rdv_$G
  # plain run first (all ranks, no ncu): must exit 0 before profiling
  for r in $(seq 0 $((G-1))); do
    timeout 300 python tools/ncu_rank.py --rank $r --world $G --dir /tmp/a2a_ncu_rdv_$G > gpurun_out/ncu_nvl_G${G}_plain_r$r.log 2>&1 &
  done
  wait; echo "plain G=$G done"
  rm -rf /tmp/a2a_ncu_rdv_$G
  for r in $(seq 0 $((G-1))); do
    timeout 600 ncu --metrics $M --clock-control none -k regex:a2a -s 3 -c 1 --csv \
      --log-file gpurun_out/ncu_nvl_G${G}_r$r.csv \
      python tools/ncu_rank.py --rank $r --world $G --dir /tmp/a2a_ncu_rdv_$G > gpurun_out/ncu_nvl_G${G}_r$r.log 2>&1 &
  done
  wait; echo "ncu G=$G done"
done
tail -3 gpurun_out/ncu_nvl_G*_r*.log
