for v in ring reg; do for c in 3 4; do echo "$v cfg $c $(TN_K5=$v timeout 300 python tools/run_step.py --config $c --reps 3 2>&1 | tail -1 | grep -o '"k5_mix[^,]*')"; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
