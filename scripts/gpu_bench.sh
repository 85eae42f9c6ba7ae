# bench pass: default bench line (+ optional extra configs in $CFGS)
TAG=${TAG:-r02}
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/${TAG}_bench.log 2>&1; echo bench rc $?
tail -1 gpurun_out/${TAG}_bench.log > gpurun_out/${TAG}_bench.jsonl
for c in ${CFGS:-}; do
  timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg$c.log 2>&1; echo cfg$c rc $?
done
