#!/bin/bash
# A/B of compile-time variants on one GPU box: for each "name=FLAGS" argument,
# rebuild the library with EXTRA=FLAGS and run the C5 bench twice; variants are
# interleaved (A B A B) so box drift hits both.  usage: bash tools/ab_build.sh TAG "a=" "b=-DX=0"
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
for rep in 1 2; do
  for v in "$@"; do
    name=${v%%=*}; flags=${v#*=}
    rm -rf paper_2201_04614_b200/csrc/build
    make -s -j8 -C paper_2201_04614_b200/csrc EXTRA="$flags" > $O/build_$name.log 2>&1
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${name}_$rep.json 2>>$O/bench.err
  done
done
rm -rf paper_2201_04614_b200/csrc/build
make -s -j8 -C paper_2201_04614_b200/csrc > /dev/null 2>&1
for f in $O/bench_*.json; do python -c "import json; d=json.load(open('$f')); k=d['kernel_ms_per_step']; print('$f', round(d['value']), round(k['fused_compress'],3), round(k['fused_decompress'],3), round(k['compress_scan_gather'],3), round(k['decompress_scan'],3))"; done
