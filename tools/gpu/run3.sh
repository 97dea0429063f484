mkdir -p gpurun_out
for S in 6 7; do timeout 300 python tools/run_step.py --config 3 --reps 4 --contraction int8 --slices $S > gpurun_out/steps_int8_$S.log 2>&1; tail -2 gpurun_out/steps_int8_$S.log; done
timeout 600 python -m pytest tests/test_gpu_int8_emu.py -x -q 2>&1 | tail -5
