#!/bin/bash
# A/B of a compile-time define on the config-5 hash numeric pass (2 M points)
for v in "$@"; do
  label=${v%%|*}; extra=${v#*|}
  make -s -C paper_1905_08423_b200/csrc clean >/dev/null; make -s -j4 -C paper_1905_08423_b200/csrc EXTRA="$extra" >/dev/null 2>&1
  echo "$label $(python tools/cfg5_numeric.py 2000000 3 2>&1 | grep numeric | tail -1)"
done
