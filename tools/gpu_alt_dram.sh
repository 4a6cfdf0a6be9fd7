# time + DRAM bytes of one c2 call per tuning build: gpu_alt_dram.sh "<tags>" "<layer_time args>"
tags=$1; shift
for t in $tags; do
  echo -n "$t: "; WF_LIB_PATH=$PWD/build_alt/libwinofuse_alt_$t.so timeout 200 python tools/layer_time.py "$@" --reps 20 2>&1 | tail -1 | cut -c1-110
  WF_LIB_PATH=$PWD/build_alt/libwinofuse_alt_$t.so timeout 300 ncu --cache-control none --clock-control none -k regex:fused_ws -s 3 -c 1 --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv python tools/layer_time.py "$@" --reps 3 2>/dev/null | grep -E "dram__bytes" | awk -F'","' '{print "    " $(NF-2) " " $(NF-1) " " $NF}'
done
