mkdir -p gpurun_out
CMD="python tools/run_step.py --config 3 --reps 2 --contraction int8 --slices 6"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k4o -s 1 -c 1 -o gpurun_out/k4o_prof $CMD > gpurun_out/ncu.log 2>&1
tail -5 gpurun_out/ncu.log
