#!/bin/bash
# A/B/... of prebuilt libraries on one GPU box, interleaved (A B C A B C ...):
#   bash tools/ab_lib.sh TAG REPS lib1.so lib2.so [lib3.so ...]
TAG=$1; REPS=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
for rep in $(seq $REPS); do
  for lib in "$@"; do
    v=$(basename $lib .so)
    VLZ_LIB=$(realpath $lib) python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${v}_$rep.json 2>>$O/bench.err
  done
done
for f in $O/bench_*.json; do python -c "import json; d=json.load(open('$f')); k=d['kernel_ms_per_step']; print('$f', round(d['value']), round(k['fused_compress'],3), round(k['fused_decompress'],3), round(k['compress_scan_gather'],3), round(k['decompress_scan'],3))"; done
