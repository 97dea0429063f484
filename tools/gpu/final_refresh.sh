# final bench lines, each in a fresh process; launch list + ncu summaries
timeout 900 python bench.py > gpurun_out/b_default.jsonl 2>gpurun_out/b_default.err
timeout 900 python bench.py --contraction int8 --no-cpu-baseline > gpurun_out/b_int8.jsonl 2>&1
timeout 900 python bench.py --pair 3 --no-cpu-baseline > gpurun_out/b_pair3.jsonl 2>&1
timeout 900 python bench.py --config 4 --no-cpu-baseline > gpurun_out/b_c4.jsonl 2>&1
timeout 900 python bench.py --config 4 --contraction int8 --no-cpu-baseline > gpurun_out/b_c4_int8.jsonl 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref.jsonl 2>&1
bash tools/gpu/profile_round.sh > gpurun_out/profile_round.log 2>&1
for f in default int8 pair3 c4 c4_int8 ref; do echo "$f: $(tail -1 gpurun_out/b_$f.jsonl | cut -c1-230)"; done
