for f in 2 2.5 3 3.5; do echo "factor $f: $(TN_SVD_WAVE1=$f timeout 300 python tools/run_svd.py --config 3 --reps 3 2>&1 | tail -1 | grep -o '"svd_ms": [0-9.]*')"; done
