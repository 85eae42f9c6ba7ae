#!/bin/bash
# A/B the prefill kernel of several in-tree builds: libmux_<name>.so, 3 alternating rounds
cd "$(dirname "$0")/../paper_2504_14489_b200"
cp libmux.so libmux_orig.so
for r in 1 2 3; do
  for v in "$@"; do
    cp libmux_$v.so libmux.so
    echo -n "$v round $r: "; (cd ..; timeout 100 python scripts/quick_perf.py 2>&1 | grep prefill)
  done
done
cp libmux_orig.so libmux.so
