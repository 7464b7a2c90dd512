#!/bin/bash
# Round-end evidence refresh, run on the GPU box:
#   gpurun --timeout 2400 -- 'bash tools/refresh_profiles.sh r02'
# Plain runs first; ncu only after the same command exited 0 (B200_PROFILING.md).
R=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/${R}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${R}_pytest_gpu.log
for c in c3 c5 c4 c2 c1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 $( [ $c != c3 ] && echo --no-cpu-baseline ) \
    > $O/${R}_bench_$c.jsonl 2> $O/${R}_bench_$c.err
done
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/${R}_bench_reference_c3.jsonl 2> $O/${R}_bench_reference_c3.err
# launch list of the bench command (cold-cache, serialised per-launch times)
if timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${R}_plain.log 2>&1; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${R}_launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/${R}_ncu_launch.log 2>&1
fi
for c in c3 c5 c4; do
  if timeout 120 python tools/prof_run.py --config $c --iters 3 > $O/${R}_prof_plain_$c.log 2>&1; then
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused|cols|stream_rows" -s 2 -c 2 \
      -o $O/${R}_prof_$c -f python tools/prof_run.py --config $c --iters 3 > $O/${R}_ncu_full_$c.log 2>&1
  fi
done
echo done
