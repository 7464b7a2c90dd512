#!/bin/bash
# Variant of the library that differs in a few translation units only:
#   [FILES="sliceblur_capi.cu sweep_u8.cu"] bash tools/build_capi_variant.sh NAME -DSB_FOO=1 ...
# Reuses the in-tree objects (python -m paper_1107_4958_b200.build first), recompiles FILES
# (default: the C ABI / planning unit) with the extra flags and links exp/NAME/libsliceblur_b200.so.
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
d=$root/exp/$name
o=/tmp/exp_obj/$name; mkdir -p $d $o
cp $root/paper_1107_4958_b200/build_obj/*.o $o/
pids=""
for f in ${FILES:-sliceblur_capi.cu}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I$root/include -I$root/paper_1107_4958_b200/csrc "$@" -c -o $o/$f.o $root/paper_1107_4958_b200/csrc/$f &
  pids="$pids $!"
done
for p in $pids; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libsliceblur_b200.so $o/*.o
echo $d/libsliceblur_b200.so
