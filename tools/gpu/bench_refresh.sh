# refresh the bench lines behind DESIGN.md / README.md (one GPU)
timeout 900 python bench.py > gpurun_out/b_default.jsonl 2>gpurun_out/b_default.err
timeout 900 python bench.py --contraction int8 --no-cpu-baseline > gpurun_out/b_int8.jsonl 2>&1
timeout 900 python bench.py --config 4 --no-cpu-baseline > gpurun_out/b_c4.jsonl 2>&1
timeout 900 python bench.py --config 4 --contraction int8 --no-cpu-baseline > gpurun_out/b_c4_int8.jsonl 2>&1
timeout 900 python bench.py --pair 3 --no-cpu-baseline > gpurun_out/b_pair3.jsonl 2>&1
timeout 900 python bench.py --layer 8 --config 3 > gpurun_out/b_layer.jsonl 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b_ref.jsonl 2>&1
for f in gpurun_out/b_*.jsonl; do echo "$f: $(tail -1 $f | cut -c1-400)"; done
