#!/bin/bash
# A/B any timing script over several in-tree builds libmux_<name>.so: ab_generic.sh "<cmd>" name1 name2 ...
cd "$(dirname "$0")/../paper_2504_14489_b200"
cmd=$1; shift
cp libmux.so libmux_orig.so
for r in 1 2; do
  for v in "$@"; do
    cp libmux_$v.so libmux.so
    echo "== $v round $r"; (cd ..; eval "timeout 300 $cmd" 2>&1 | grep -v Warning)
  done
done
cp libmux_orig.so libmux.so
