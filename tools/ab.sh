#!/bin/bash
# A/B on the GPU box with the prebuilt library: tools/ab.sh label "ENV=..." ...
# runs the numeric-only bench once per label with the given env settings.
while [ $# -gt 1 ]; do
  label=$1; envs=$2; shift 2
  env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-variants > gpurun_out/ab_$label.log 2>&1
  python - "$label" <<'PY'
import json, sys
lab = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{lab}.log").read().strip().splitlines()[-1])
    print(f"{lab:24s} numeric {d['ms_per_step']:.3f} ms  {d['value']:.1f} GFLOP/s  frac {d['roofline']['frac']:.4f}")
except Exception as e:
    print(lab, "failed", e)
PY
done
