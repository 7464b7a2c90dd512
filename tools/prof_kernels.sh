#!/usr/bin/env bash
# ncu --set full (source-correlated) of one step of each named config, after a plain run of the
# same command exited 0.  Usage (GPU box): bash tools/prof_kernels.sh TAG c3 c5 ...
set -u
tag=$1; shift
O=gpurun_out; mkdir -p $O
for c in "$@"; do
  if timeout 300 python tools/prof_run.py --config $c --iters 3 > $O/prof_plain_${tag}_$c.log 2>&1; then
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused|cols|stream_rows|generic" -s 2 -c 3 \
      -o $O/prof_${tag}_$c -f python tools/prof_run.py --config $c --iters 3 > $O/ncu_${tag}_$c.log 2>&1
    echo "$c ncu rc=$?"
  else
    echo "$c plain run failed"; tail -5 $O/prof_plain_${tag}_$c.log
  fi
done
