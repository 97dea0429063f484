for c in 3 4; do echo "cfg $c $(timeout 300 python tools/run_step.py --config $c --reps 4 2>&1 | tail -1 | grep -o '"k4_contract[^,]*')"; done
