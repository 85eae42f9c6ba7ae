#!/bin/bash
# A/B whole multiplexed steps of several in-tree builds libmux_<name>.so (scripts/mux_ab.py), 2 rounds
cd "$(dirname "$0")/../paper_2504_14489_b200"
cp libmux.so libmux_orig.so
for r in 1 2; do
  for v in "$@"; do
    cp libmux_$v.so libmux.so
    echo -n "$v round $r: "; (cd ..; timeout 200 python scripts/mux_ab.py ${MUXAB_ARGS:-} 2>&1 | tail -1)
  done
done
cp libmux_orig.so libmux.so
