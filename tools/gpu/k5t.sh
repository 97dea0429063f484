export TN_K5T=1
cp tools/gpu/k5tv/lib_nous.so paper_2301_12814_b200/libtn_theta.so
for c in 3 4; do echo "k5t-noUs cfg $c $(timeout 120 python tools/run_step.py --config $c --reps 4 2>&1 | tail -1 | grep -o '"k5_mix[^,]*')"; done
