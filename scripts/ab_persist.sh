#!/bin/bash
# bench A/B of the persistent prefill loop (default for L2-resident batches) vs MUX_PF_NO_PERSIST, 2 rounds
TAG=${TAG:-r02}
for r in 1 2; do
  for v in default MUX_PF_NO_PERSIST; do
    env $([ $v = default ] || echo $v=1) timeout 600 python bench.py --steps 10 --no-cpu-baseline 2>&1 | tail -1 \
      > gpurun_out/${TAG}_ab_$v$r.jsonl
    python -c "import json,sys;d=json.load(open('gpurun_out/${TAG}_ab_$v$r.jsonl'));r=d['roofline'];print('$v',$r,round(d['value']),r['launch_us_mean'],r['alone_launch_us'],d['clocks']['sm_mhz'])"
  done
done
