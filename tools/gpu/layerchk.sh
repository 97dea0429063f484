for i in 1 2 3; do timeout 600 python bench.py --layer 8 --config 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['gate_ms'])"; done
