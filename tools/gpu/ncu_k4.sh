mkdir -p gpurun_out
CMD="python tools/run_step.py --config 3 --reps 2"
$CMD > gpurun_out/plain_k4.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'k4_contract' -s 1 -c 1 -o gpurun_out/k4_prof2 $CMD > gpurun_out/ncu_k4.log 2>&1
tail -3 gpurun_out/ncu_k4.log
