# position GEMM breakdown: three-stage phases of the wave layers (c3 L9, c4 L4)
set -x
python tools/layer_time.py c3 8 --engine three_stage --reps 20
python tools/layer_time.py c4 3 --engine three_stage --reps 20
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/gemm_launches.csv python tools/layer_time.py c3 8 --engine three_stage --reps 2
python tools/ncu_summary.py gpurun_out/gemm_launches.csv 2>/dev/null | head -40 || true
