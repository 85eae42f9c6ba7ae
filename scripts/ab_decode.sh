#!/bin/bash
# A/B the decode kernel of several in-tree builds libmux_<name>.so (quick_perf decode + splits lines)
cd "$(dirname "$0")/../paper_2504_14489_b200"
cp libmux.so libmux_orig.so
for r in 1 2; do
  for v in "$@"; do
    cp libmux_$v.so libmux.so
    echo "== $v round $r"; (cd ..; timeout 200 python scripts/quick_perf.py 2>&1 | grep -E "decode|split")
  done
done
cp libmux_orig.so libmux.so
