#!/bin/bash
# interleaved A/B of prebuilt libraries on the per-config bench (tools/bench_configs.py)
#   bash tools/ab_configs.sh TAG REPS "C3 stress" lib1.so lib2.so ...
TAG=$1; REPS=$2; CASES=$3; shift 3
O=gpurun_out/$TAG; mkdir -p $O
for rep in $(seq $REPS); do
  for lib in "$@"; do
    v=$(basename $lib .so)
    VLZ_LIB=$(realpath $lib) python tools/bench_configs.py $CASES >> $O/configs_${v}.jsonl 2>>$O/err.txt
  done
done
for f in $O/configs_*.jsonl; do python - "$f" <<'PY'
import json, sys, collections, statistics
by = collections.defaultdict(list)
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l); k = d["kernels_compress"]; kd = d["kernels_decompress"]
        by[d["case"]].append((k["compress"] * 1e3, kd["decompress"] * 1e3, d["compress_ms"] * 1e3, d["decompress_ms"] * 1e3))
for c, v in by.items():
    print(sys.argv[1].split("/")[-1], c, "fused c/d us", [round(statistics.median(x[i] for x in v), 1) for i in range(4)])
PY
done
