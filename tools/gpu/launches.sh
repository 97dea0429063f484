# usage: bash tools/gpu/launches.sh <tag> <run_step args...>   — ncu launch list (device time per kernel)
mkdir -p gpurun_out
TAG=$1; shift
python tools/run_step.py "$@" > gpurun_out/plain_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/run_step.py "$@" > /dev/null 2>&1
python - "$TAG" <<'PY'
import csv, sys, collections
tag = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{tag}.csv")) if len(r) > 10]
h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value"); iu = h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[iv].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(r[iu], 1)
    agg[r[ik][:60]].append(v)
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:60s} n={len(v):3d} mean_us={sum(v)/len(v):9.1f}")
PY
