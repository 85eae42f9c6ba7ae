#!/bin/bash
# persistent prefill: MMA-issuer lookahead (-DMUX_PF6P_LOOKAHEAD=1, libmux_la.so) vs the default build.
# 1) parity under the bounded-wait build of the variant (libmux_labnd.so; waits trap after 2 s), default
#    selection and the loop forced; 2) prefill alone on the 140-SM partition, 3 alternating rounds;
# 3) bench, 2 alternating rounds
TAG=${TAG:-r02i}
P=paper_2504_14489_b200
cp $P/libmux.so $P/libmux_orig.so
cp $P/libmux_labnd.so $P/libmux.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mux.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3 > gpurun_out/${TAG}_la_bounded_default.log
MUX_PF_PERSIST=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mux.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3 > gpurun_out/${TAG}_la_bounded_forced.log
cat gpurun_out/${TAG}_la_bounded_*.log
if ! grep -q " passed" gpurun_out/${TAG}_la_bounded_forced.log || grep -q "failed\|error" gpurun_out/${TAG}_la_bounded_*.log; then
  cp $P/libmux_orig.so $P/libmux.so; echo "parity not green: no perf A/B"; exit 1
fi
for r in 1 2 3; do for v in orig la; do
  cp $P/libmux_$v.so $P/libmux.so
  TAG=$v DECS=8 timeout 120 python scripts/pf_part_perf.py 2>&1 | grep split >> gpurun_out/${TAG}_la_pf.log
done; done
cat gpurun_out/${TAG}_la_pf.log
for r in 1 2; do for v in orig la; do
  cp $P/libmux_$v.so $P/libmux.so
  timeout 400 python bench.py 2>&1 | tail -1 > gpurun_out/${TAG}_la_bench_${v}_$r.jsonl
  python -c "import json,sys;d=json.loads(open('gpurun_out/${TAG}_la_bench_${v}_$r.jsonl').read());print('$v', d['value'], d['roofline']['launch_us_mean'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done; done
cp $P/libmux_orig.so $P/libmux.so
