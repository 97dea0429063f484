#!/bin/bash
# Runs on the GPU box: FP64 peak microbenchmarks with clocks sampled during the run.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/fp64_clocks.csv &
SMI=$!
bash tools/build_tools.sh && ./tools/fp64_peak > gpurun_out/fp64_peak.jsonl 2>&1
python tools/fp64_peak_torch.py >> gpurun_out/fp64_peak.jsonl 2>&1
kill $SMI
nproc >> gpurun_out/fp64_peak.jsonl
cat gpurun_out/fp64_peak.jsonl
