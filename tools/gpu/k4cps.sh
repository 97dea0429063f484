for v in 2 1 2 1; do echo "cps $v: $(TN_K4_CPS=$v timeout 120 python tools/run_step.py --config 3 --reps 4 2>&1 | tail -1 | grep -o '"k4_contract[^,]*')  c4: $(TN_K4_CPS=$v timeout 200 python tools/run_step.py --config 4 --reps 2 2>&1 | tail -1 | grep -o '"k4_contract[^,]*')"; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "theta_parity or edge" 2>&1 | tail -2
