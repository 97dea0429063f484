python tools/run_step.py --config 3 --reps 2 > gpurun_out/k5cls_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k5_mix --csv --log-file gpurun_out/k5cls.csv python tools/run_step.py --config 3 --reps 2 > gpurun_out/k5cls_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/k5cls.csv 2>/dev/null | head -30 || true
