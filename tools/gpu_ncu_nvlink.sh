# multi-GPU executor kernel under ncu: rank 0 profiled, the other ranks run the same
# all-to-alls without ncu.  One single-pass metric group per run: a replay pass would
# re-run rank 0's kernel after its peers finished that all-to-all (it then times out).
mkdir -p gpurun_out
for G in 2 4; do
  for GRP in nvl dram; do
    case $GRP in
      nvl) M="nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum";;
      dram) M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum";;
    esac
    D=/tmp/a2a_ncu_rdv_${G}_$GRP; rm -rf $D
    for r in $(seq 1 $((G-1))); do
      ( timeout 300 python tools/ncu_rank.py --rank $r --world $G --dir $D --phase plain --optional;
        timeout 300 python tools/ncu_rank.py --rank $r --world $G --dir $D --phase ncu ) > gpurun_out/ncu_nvl_G${G}_${GRP}_peer_r$r.log 2>&1 &
    done
    timeout 600 ncu --metrics $M --clock-control none --cache-control none -k regex:a2a -s 3 -c 1 --csv \
        --log-file gpurun_out/ncu_nvl_G${G}_${GRP}_r0.csv \
        python tools/ncu_rank.py --rank 0 --world $G --dir $D > gpurun_out/ncu_nvl_G${G}_${GRP}_r0.log 2>&1
    echo "ncu G=$G $GRP rc=$?"
    wait
  done
done
