#!/bin/bash
# Sweep the lean TMA decompress kernel's CTAs/SM (launch bounds) on the GPU box.
O=gpurun_out/${1:-dminb}; mkdir -p $O
for m in ${MINBS:-4 5 6}; do
  rm -f paper_2201_04614_b200/csrc/build/k_decompress.o
  make -s -j8 -C paper_2201_04614_b200/csrc EXTRA="-DVLZ_DTMA_MINB=$m" > $O/build_$m.log 2>&1
  for r in 1 2; do
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${m}_$r.json 2>>$O/bench.err
  done
done
rm -f paper_2201_04614_b200/csrc/build/k_decompress.o
make -s -j8 -C paper_2201_04614_b200/csrc > /dev/null 2>&1
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); k=d['kernel_ms_per_step']; print('$f', round(d['value']), round(k['fused_compress'],3), round(k['fused_decompress'],3))"; done
