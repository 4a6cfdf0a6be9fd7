# pipelined forward kernel: parity + three-stage layer times (pipe off / sync / per-warp release)
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for L in "c3 8" "c3 3" "c3 5" "c2 0"; do
  WF_FWD_PIPE=0 python tools/layer_time.py $L --engine three_stage --reps 20
  python tools/layer_time.py $L --engine three_stage --reps 20
  WF_FWD_SYNC=0 python tools/layer_time.py $L --engine three_stage --reps 20
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/fwd_launches.csv python tools/layer_time.py c3 8 --engine three_stage --reps 2
