mkdir -p gpurun_out
timeout 600 python tools/oz_accuracy.py > gpurun_out/oz_accuracy.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "phi_shift or padding" 2>&1 | tail -5 > gpurun_out/t10t11.log
cat gpurun_out/oz_accuracy.log gpurun_out/t10t11.log
