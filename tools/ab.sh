#!/bin/bash
# A/B timing of variant libraries: bash tools/ab.sh cfg lib1 lib2 ...
#   "default" = in-tree build; "env:NAME=VALUE" = in-tree build with that variable set
cfg=$1; shift
for rep in 1 2; do
for lib in "$@"; do
  case "$lib" in
    default) envs="" ;;
    env:*) envs="${lib#env:}" ;;
    *) envs="SB_LIB_PATH=$PWD/$lib" ;;
  esac
  v=$(env $envs timeout 200 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['value'], d.get('parity',{}).get('max_abs'))")
  echo "$cfg $lib rep$rep: $v"
done; done
