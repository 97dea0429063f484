# Round-2 secondary bench lines on the final code: config 4 (DMMA and INT8), MPO pair configs 3/4/5, the config-3
# TEBD layer; each line to gpurun_out/sec_*.jsonl
timeout 900 python bench.py --config 4 2>/dev/null | tail -1 > gpurun_out/sec_c4.jsonl
timeout 900 python bench.py --config 4 --contraction int8 2>/dev/null | tail -1 > gpurun_out/sec_c4_int8.jsonl
for k in 3 4 5; do timeout 600 python bench.py --pair $k 2>/dev/null | tail -1 > gpurun_out/sec_pair$k.jsonl; done
timeout 900 python bench.py --layer 8 --config 3 2>/dev/null | tail -1 > gpurun_out/sec_layer8.jsonl
for f in gpurun_out/sec_*.jsonl; do echo "$f $(cut -c1-260 $f)"; done
