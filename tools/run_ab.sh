# usage: bash tools/run_ab.sh CFG VARIANTS... ; runs gpu tests then A/B
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
cfg=$1; shift
bash tools/ab.sh $cfg "$@" > $O/ab.txt 2>&1
cat $O/ab.txt
