for pf in 0 1 2; do for c in 3 4; do echo "pf $pf cfg $c $(TN_K5_PF=$pf timeout 300 python tools/run_step.py --config $c --reps 4 2>&1 | tail -1 | grep -o '"k5_mix[^,]*')"; done; done
