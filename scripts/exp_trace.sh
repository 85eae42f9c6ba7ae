# per-tile prefill v6 traces of trace builds libmux_t<name>.so (scripts/trace_v6.py)
cd paper_2504_14489_b200; cp libmux.so libmux_keep.so; cd ..
for v in "$@"; do
  cp paper_2504_14489_b200/libmux_t$v.so paper_2504_14489_b200/libmux.so
  echo "== $v" >> gpurun_out/exp_trace.log
  timeout 120 python scripts/trace_v6.py >> gpurun_out/exp_trace.log 2>&1
done
cp paper_2504_14489_b200/libmux_keep.so paper_2504_14489_b200/libmux.so
