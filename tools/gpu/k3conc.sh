for c in 3 4; do echo "cfg $c $(timeout 300 python tools/run_step.py --config $c --reps 4 2>&1 | tail -1 | grep -o '"k3_stage[^,]*\|"k5_mix[^,]*' | tr '\n' ' ')"; done
echo "int8 cfg3 $(timeout 300 python tools/run_step.py --config 3 --reps 4 --contraction int8 --slices 6 2>&1 | tail -1 | grep -o '"k3_stage[^,]*\|"k4_contract[^,]*' | tr '\n' ' ')"
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['alt_engine']['ms_per_gate_excl_plan'], {k:v['ms'] for k,v in d['kernels'].items()})"
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_int8_emu.py tests/test_gpu_pair.py tests/test_gpu_remote.py tests/test_gpu_guards.py -q -x 2>&1 | tail -2
