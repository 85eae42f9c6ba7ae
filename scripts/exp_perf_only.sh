# quick_perf prefill timings of several builds libmux_<v>.so, 3 alternating rounds (NPF: prefill length)
cd paper_2504_14489_b200; cp libmux.so libmux_keep.so; cd ..
for r in 1 2 3; do
  for v in ${VARIANTS}; do
    cp paper_2504_14489_b200/libmux_$v.so paper_2504_14489_b200/libmux.so
    echo -n "$v NPF=${NPF:-8192} round $r: " >> gpurun_out/exp_perf_only.log
    timeout 100 python scripts/quick_perf.py 2>&1 | grep prefill >> gpurun_out/exp_perf_only.log
  done
done
cp paper_2504_14489_b200/libmux_keep.so paper_2504_14489_b200/libmux.so
