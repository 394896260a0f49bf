#!/bin/bash
# One GPU round-trip: gpu tests, smoke, bench line, launch list, per-config numbers.
# usage (from the repo root on the GPU box): bash tools/gpu_check.sh TAG
TAG=${1:-run}
O=gpurun_out/$TAG
# our kernels only (the synthetic field generator is torch elementwise work)
KRE='dq_|minmax|init_kernel|hd_|huff|histogram|border'
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$KRE" -c 6000 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
for f in pytest_gpu.log smoke.log bench.err; do tail -n 3 $O/$f; done
cat $O/bench.json
