mkdir -p gpurun_out
for l in 0 1 2 3; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c4_l$l.csv python tools/layer_time.py c4 $l --reps 2 > gpurun_out/c4_l$l.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_l9.csv python tools/layer_time.py c3 8 --reps 2 > gpurun_out/c3_l9.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_l12.csv python tools/layer_time.py c3 11 --reps 2 > gpurun_out/c3_l12.log 2>&1
