# Final profiling pass of round 1: launch list of the bench command + ncu --set full of the step kernels.
mkdir -p gpurun_out
BENCH="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-alt-engine --e2e-steps 2"
$BENCH > gpurun_out/prof_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_final.csv $BENCH > gpurun_out/prof_launch.log 2>&1
STEP="python tools/run_step.py --config 3 --reps 2"
$STEP > gpurun_out/prof_step.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'k1_sort|k2_bs|k3_stage|k4_contract|k5_mix' -s 8 -c 8 -o gpurun_out/r01_final $STEP > gpurun_out/prof_full.log 2>&1
STEP8="python tools/run_step.py --config 3 --reps 2 --contraction int8 --slices 6"
$STEP8 > gpurun_out/prof_step8.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'k3o|k4o' -s 4 -c 5 -o gpurun_out/r01_final_int8 $STEP8 > gpurun_out/prof_full8.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/r01_launches_final.csv
