timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config4 or fused" 2>&1 | tail -2
for c in 3 4; do echo "cfg $c $(timeout 300 python tools/run_step.py --config $c --reps 4 2>&1 | tail -1 | grep -o '"k5_mix[^,]*')"; done
