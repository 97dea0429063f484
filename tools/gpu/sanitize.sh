# usage: bash tools/gpu/sanitize.sh <memcheck|racecheck|synccheck|initcheck>   (ONE tool per gpurun call)
mkdir -p gpurun_out
T=${1:-memcheck}
python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
timeout 1200 compute-sanitizer --tool $T --print-limit 20 --error-exitcode 9 python tools/sanitize_case.py > gpurun_out/sanitize_$T.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_$T.log
tail -8 gpurun_out/sanitize_$T.log
