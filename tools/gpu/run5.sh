for A in 32 36 40 48; do echo "ablate $A"; TN_K4O_ABLATE=$A timeout 60 python tools/run_step.py --config 3 --reps 2 --contraction int8 --slices 6 2>&1 | grep -o "k4o mma.*\|k4_contract[^,]*"; done
