#!/bin/bash
# ncu --set full capture of the C5 bench's kernels (one launch each), for profiles/.
# usage: bash tools/ncu_full.sh TAG [kernel-regex] [count]
TAG=${1:-full}
KRE=${2:-'dq_compress_fast|dq_scan|dq_decompress_tma'}
CNT=${3:-4}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c $CNT \
  -o $O/full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log
tail -n 5 $O/ncu_full.log
