for c in 3 4; do echo "cfg $c $(timeout 300 python tools/run_step.py --config $c --reps 3 2>&1 | tail -1 | grep -o '"k4_contract[^,]*, "k5_mix[^,]*')"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pair.py -x -q 2>&1 | tail -2
