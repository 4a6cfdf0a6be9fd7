# A/B of tuning builds: usage gpu_alt.sh "<tags>" "<layer_time args>"...
tags=$1; shift
for t in $tags; do
  for a in "$@"; do
    echo -n "$t: "; WF_LIB_PATH=$PWD/build_alt/libwinofuse_alt_$t.so timeout 200 python tools/layer_time.py $a --reps 20 2>&1 | tail -1
  done
done
