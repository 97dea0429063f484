for v in 0 1 0 1; do if [ $v = 1 ]; then export TN_K5_SERIAL=1; else unset TN_K5_SERIAL; fi; echo "serial=$v cfg3 $(timeout 300 python tools/run_step.py --config 3 --reps 4 2>&1 | tail -1 | grep -o '"k5_mix[^,]*') cfg4 $(timeout 300 python tools/run_step.py --config 4 --reps 2 2>&1 | tail -1 | grep -o '"k5_mix[^,]*')"; done
unset TN_K5_SERIAL
timeout 600 python bench.py --no-cpu-baseline --no-alt-engine --e2e-steps 2 2>&1 | tail -1 | cut -c150-260
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "theta_parity or edge or sharded or padding or config4" 2>&1 | tail -2
