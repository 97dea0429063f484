# Round-2 closing measurements on the final code: default bench line (twice), reference arm, INT8 engine line,
# the whole GPU suite + smoke, then the ncu pass of tools/gpu/profile_r2.sh.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
for i in 1 2; do timeout 600 python bench.py 2>/dev/null | tail -1 >> gpurun_out/final_bench.jsonl; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/final_ref.jsonl
timeout 600 python bench.py --contraction int8 2>/dev/null | tail -1 > gpurun_out/final_int8.jsonl
START=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1; echo "suite wall $(( $(date +%s) - START )) s" >> gpurun_out/final_gpu_tests.log
tail -3 gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
bash tools/gpu/profile_r2.sh
