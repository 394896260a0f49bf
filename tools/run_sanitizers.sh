#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the sanitize
# workload (tools/sanitize_smoke.py) and a short bench step (begin/finish +
# device-count decompress path); summaries into gpurun_out/sanitize_*.txt.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_smoke.py > gpurun_out/sanitize_${tool}.txt 2>&1
  echo "workload $tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  timeout 900 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python bench.py --planes 16 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
      > gpurun_out/sanitize_bench_${tool}.txt 2>&1
  echo "bench16 $tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
done
