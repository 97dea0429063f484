echo "base $(timeout 120 python tools/run_step.py --config 3 --reps 4 2>&1 | tail -1 | grep -o '"k5_mix[^,]*')"
cp tools/gpu/k5exp/lib_not3.so paper_2301_12814_b200/libtn_theta.so
echo "noT3 $(timeout 120 python tools/run_step.py --config 3 --reps 4 2>&1 | tail -1 | grep -o '"k5_mix[^,]*')"
