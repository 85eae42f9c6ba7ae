#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box from the repo root):
#   launch list of one full-GPU multiplexed step + one --set full capture per hot kernel.
# usage: bash scripts/profile_round.sh <tag>
set -x
tag=${1:-r01}
out=gpurun_out/prof_$tag
mkdir -p $out
export SPLIT=-1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
    python scripts/one_step.py > $out/launches.log 2>&1
for k in prefill6p_kernel decode_kernel outproj2_kernel outproj_skinny_kernel append_kv_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" --launch-skip 1 -c 1 \
      -o $out/$k python scripts/one_step.py > $out/$k.log 2>&1
  ncu -i $out/$k.ncu-rep --page raw --csv > $out/${k}_raw.csv 2>/dev/null
  ncu -i $out/$k.ncu-rep --page details --csv > $out/${k}_details.csv 2>/dev/null
done
