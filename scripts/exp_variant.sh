# A/B of a candidate build libmux_$V.so against libmux_base.so: prefill parity with the candidate,
# then alternating quick_perf prefill timings and multiplexed-step timings (scripts/mux_ab.py)
V=${V:-split2}
cd paper_2504_14489_b200; cp libmux.so libmux_keep.so; cp libmux_$V.so libmux.so; cd ..
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "prefill or full" 2>&1 | tail -5 > gpurun_out/exp_${V}_parity.log
for r in 1 2 3; do
  for v in base $V; do
    cp paper_2504_14489_b200/libmux_$v.so paper_2504_14489_b200/libmux.so
    echo -n "$v round $r: " >> gpurun_out/exp_${V}_perf.log
    timeout 100 python scripts/quick_perf.py 2>&1 | grep prefill >> gpurun_out/exp_${V}_perf.log
  done
done
bash scripts/ab_mux.sh base $V > gpurun_out/exp_${V}_mux.log 2>&1
cp paper_2504_14489_b200/libmux_keep.so paper_2504_14489_b200/libmux.so
