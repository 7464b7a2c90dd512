#!/bin/bash
# A/B timing of variant libraries: bash exp/ab.sh cfg lib1 lib2 ...  ("default" = in-tree build)
cfg=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  if [ "$lib" = default ]; then unset SB_LIB_PATH; else export SB_LIB_PATH=$PWD/$lib; fi
  v=$(timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['value'], d.get('parity',{}).get('max_abs'))")
  echo "$cfg $lib rep$rep: $v"
done; done
