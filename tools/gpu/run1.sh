set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for c in dmma int8; do timeout 300 python tools/run_step.py --config 3 --reps 4 --contraction $c --slices 7 >> gpurun_out/steps.log 2>&1; done
timeout 300 python tools/run_step.py --config 3 --reps 3 --contraction int8 --slices 6 >> gpurun_out/steps.log 2>&1
for c in dmma int8; do timeout 300 python tools/run_step.py --config 4 --reps 3 --contraction $c --slices 7 >> gpurun_out/steps.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/bench.log
