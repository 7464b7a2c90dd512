#!/usr/bin/env bash
# One compute-sanitizer tool per invocation (the B200 profiling recipe: never several tools in
# one GPU call).  Usage (on the GPU box): bash tools/sanitize.sh racecheck|synccheck|memcheck
set -u
tool=${1:?tool}
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/san_plain.txt 2>&1 || { echo "plain run failed"; tail gpurun_out/san_plain.txt; exit 1; }
extra=""
[ "$tool" = racecheck ] && extra="--racecheck-report all"
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool "$tool" $extra --kernel-name kns=sb:: --print-limit 50 \
  python tools/sanitize_cases.py > "gpurun_out/san_${tool}.txt" 2>&1
echo "exit $?" >> "gpurun_out/san_${tool}.txt"
tail -n 25 "gpurun_out/san_${tool}.txt"
