for G in 64 256 128; do
  if [ $G != 128 ]; then cp tools/gpu/k5v/lib_$G.so paper_2301_12814_b200/libtn_theta.so; else cp tools/gpu/k5v/lib_128.so paper_2301_12814_b200/libtn_theta.so; fi
  echo "G=$G $(timeout 300 python tools/run_step.py --config 3 --reps 3 2>&1 | tail -1 | grep -o '"k5_mix[^,]*')"
done
