# prefill A/B: alternating rounds over "name:ENV" pairs (name = libmux_<name>.so; ENV = extra env as A=1+B=2, "-" none)
export PYTHONUNBUFFERED=1
cd paper_2504_14489_b200; cp libmux.so libmux_keep.so; cd ..
LOG=gpurun_out/${LOGN:-pf_variants}.log
for pair in ${PARITY:-}; do
  v=${pair%%:*}; e=${pair#*:}; [ "$e" = "-" ] && e=""
  cp paper_2504_14489_b200/libmux_$v.so paper_2504_14489_b200/libmux.so
  echo "parity $pair: $(env $e timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k 'prefill or full' 2>&1 | tail -1)" >> $LOG
done
for r in 1 2 3; do
  for pair in $VARIANTS; do
    v=${pair%%:*}; e=${pair#*:}; [ "$e" = "-" ] && e=""; e=${e//+/ }
    cp paper_2504_14489_b200/libmux_$v.so paper_2504_14489_b200/libmux.so
    env $e TAG="$pair r$r" timeout 120 python scripts/pf_perf.py >> $LOG 2>&1
  done
done
cp paper_2504_14489_b200/libmux_keep.so paper_2504_14489_b200/libmux.so
