# prefill V7 (per-head S, P over S) vs v6: parity with V7, alternating quick_perf timings, cycle traces
export PYTHONUNBUFFERED=1
MUX_PF_V7=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "prefill or full" 2>&1 | tail -5 > gpurun_out/v7_parity.log
for r in 1 2 3; do
  echo -n "v6 r$r: " >> gpurun_out/v7_perf.log; timeout 100 python scripts/quick_perf.py 2>&1 | grep prefill >> gpurun_out/v7_perf.log
  echo -n "v7 r$r: " >> gpurun_out/v7_perf.log; MUX_PF_V7=1 timeout 100 python scripts/quick_perf.py 2>&1 | grep prefill >> gpurun_out/v7_perf.log
done
echo -n "v6 32k: " >> gpurun_out/v7_perf.log; NPF=32768 timeout 100 python scripts/quick_perf.py 2>&1 | grep prefill >> gpurun_out/v7_perf.log
echo -n "v7 32k: " >> gpurun_out/v7_perf.log; MUX_PF_V7=1 NPF=32768 timeout 100 python scripts/quick_perf.py 2>&1 | grep prefill >> gpurun_out/v7_perf.log
cd paper_2504_14489_b200; cp libmux.so libmux_keep.so; cp libmux_t7.so libmux.so; cd ..
echo "== v6" >> gpurun_out/v7_trace.log; timeout 120 python scripts/trace_v6.py >> gpurun_out/v7_trace.log 2>&1
cp gpurun_out/trace_v6.npy gpurun_out/trace_v6base.npy
echo "== v7" >> gpurun_out/v7_trace.log; MUX_PF_V7=1 timeout 120 python scripts/trace_v6.py >> gpurun_out/v7_trace.log 2>&1
cp gpurun_out/trace_v6.npy gpurun_out/trace_v7.npy
cp paper_2504_14489_b200/libmux_keep.so paper_2504_14489_b200/libmux.so
