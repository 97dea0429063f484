mkdir -p gpurun_out
for S in 6 7; do echo "S=$S $(timeout 60 python tools/run_step.py --config 3 --reps 3 --contraction int8 --slices $S 2>&1 | tail -1 | grep -o "k3_stage[^,]*, .k4_contract[^,]*")"; done
timeout 300 python tools/oz_accuracy.py 2>&1 | grep '"config": 3' 
timeout 600 python -m pytest tests/test_gpu_int8_emu.py -x -q 2>&1 | tail -3
