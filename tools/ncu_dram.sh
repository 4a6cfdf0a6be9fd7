for d in 0 1 2 3; do
  WF_WS_DISCARD=$d timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused_ws -s 2 -c 1 --csv python tools/ws_time.py c2 3 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v d=$d '{print "discard", d, $(NF-2), $NF}'
done
