# usage: bash tools/run_prof.sh CFG TAG [ENV=VAL...]: plain run, then ncu --set full of the fused/cols kernels
O=gpurun_out; mkdir -p $O
cfg=$1; tag=$2; shift 2
if env "$@" timeout 120 python tools/prof_run.py --config $cfg --iters 3 > $O/prof_plain_$tag.log 2>&1; then
  env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused|cols|stream_rows" -s 2 -c 1 \
    -o $O/prof_$tag -f python tools/prof_run.py --config $cfg --iters 3 > $O/ncu_full_$tag.log 2>&1
fi
tail -2 $O/ncu_full_$tag.log
