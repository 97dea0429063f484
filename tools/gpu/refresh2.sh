timeout 900 python bench.py --contraction int8 --no-cpu-baseline > gpurun_out/b_int8.jsonl 2>&1
timeout 900 python bench.py --pair 3 --no-cpu-baseline > gpurun_out/b_pair3.jsonl 2>&1
timeout 900 python bench.py --layer 8 --config 3 > gpurun_out/b_layer3.jsonl 2>&1
for f in int8 pair3 layer3; do echo "$f: $(tail -1 gpurun_out/b_$f.jsonl | cut -c1-200)"; done
