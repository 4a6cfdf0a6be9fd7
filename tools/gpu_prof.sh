# item profile + one ncu --set full capture of the persistent kernel (bench c2 step)
mkdir -p gpurun_out
PYTHONPATH=. python tools/item_profile.py > gpurun_out/item_prof.log 2>&1; tail -12 gpurun_out/item_prof.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fused_persistent -s 3 -c 1 -o gpurun_out/persist_full -f python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu $?
