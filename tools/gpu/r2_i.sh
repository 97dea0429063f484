python bench.py --pair 3 --steps 3 --warmup 1 > gpurun_out/p3plain.log 2>&1
ncu --set full --clock-control none -k regex:k5p_mix -s 2 -c 2 -o gpurun_out/r02_k5p python bench.py --pair 3 --steps 3 --warmup 1 > gpurun_out/p3ncu.log 2>&1
ls -la gpurun_out/r02_k5p.ncu-rep
