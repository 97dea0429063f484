# Round-2 profiling pass: launch list of the bench command + ncu --set full (plus the DMMA instruction count) of
# one step's kernels, after each command has run clean without ncu.
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-alt-engine --e2e-steps 2 --emulate-ranks 0"
$BENCH > gpurun_out/prof2_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $BENCH > gpurun_out/prof2_launch.log 2>&1
STEP="python tools/run_step.py --config 3 --reps 2"
$STEP > gpurun_out/prof2_step.log 2>&1 &&
ncu --set full --metrics sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --import-source on -k regex:'k1_sort|k2_bs|k3_stage|k4_contract|k5_mix|k_set_sectors' -s 9 -c 9 \
    -o gpurun_out/r02_final $STEP > gpurun_out/prof2_full.log 2>&1
ls -la gpurun_out/r02_final.ncu-rep gpurun_out/r02_launches.csv
