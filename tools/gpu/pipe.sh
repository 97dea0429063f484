for st in 3 2; do echo "K4 stages $st:"; TN_K4_STAGES=$st timeout 300 python tools/pipeline_probe.py 2>&1 | tail -3; done
