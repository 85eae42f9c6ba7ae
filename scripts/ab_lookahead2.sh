#!/bin/bash
# lookahead on by default: full -m gpu suite + smoke, then bench A/B vs libmux_nola.so, 3 alternating rounds
TAG=${TAG:-r02j}
P=paper_2504_14489_b200
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
cat gpurun_out/${TAG}_gputest.log; tail -n 2 gpurun_out/${TAG}_smoke.log
cp $P/libmux.so $P/libmux_la.so
for r in 1 2 3; do for v in nola la; do
  cp $P/libmux_$v.so $P/libmux.so
  timeout 400 python bench.py 2>&1 | tail -1 > gpurun_out/${TAG}_bench_${v}_$r.jsonl
  python -c "import json,sys;d=json.loads(open('gpurun_out/${TAG}_bench_${v}_$r.jsonl').read());c=d['config'];print('$v', round(d['value']), c['decode_layers_per_step'], round(d['roofline']['launch_us_mean'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done; done
cp $P/libmux_la.so $P/libmux.so
