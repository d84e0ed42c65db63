#!/bin/bash
# A/B helper for the GPU box: build the library with EXTRA nvcc defines and
# run the bench headline; usage: tools/ab_build.sh "<label>" "<EXTRA flags>" [bench args]
label=$1; extra=$2; shift 2
make -s -C paper_1905_08423_b200/csrc clean >/dev/null
make -s -j4 -C paper_1905_08423_b200/csrc EXTRA="$extra" >/dev/null 2>&1 || { echo "$label build failed"; exit 1; }
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-variants "$@" > gpurun_out/ab_$label.log 2>&1
python - "$label" <<'PY'
import json, sys
lab = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_{lab}.log").read().strip().splitlines()[-1])
print(f"{lab:24s} numeric {d['ms_per_step']:.3f} ms  {d['value']:.1f} GFLOP/s  frac {d['roofline']['frac']:.4f}")
PY
