#!/bin/bash
# ncu --set full of the 16-CTA decode for several in-tree builds libmux_<name>.so (warp-stall evidence)
cd "$(dirname "$0")/.."
out=gpurun_out/ncu_dec
mkdir -p $out
cp paper_2504_14489_b200/libmux.so paper_2504_14489_b200/libmux_orig.so
for v in "$@"; do
  cp paper_2504_14489_b200/libmux_$v.so paper_2504_14489_b200/libmux.so
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:decode_kernel --launch-skip 2 -c 1 \
      -o $out/$v python scripts/decode_16cta.py > $out/$v.log 2>&1
  ncu -i $out/$v.ncu-rep --page raw --csv > $out/${v}_raw.csv 2>/dev/null
  ncu -i $out/$v.ncu-rep --page source --csv --print-source sass > $out/${v}_sass.csv 2>/dev/null
done
cp paper_2504_14489_b200/libmux_orig.so paper_2504_14489_b200/libmux.so
