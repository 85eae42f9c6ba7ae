set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -rs 2>&1 | tail -40 > gpurun_out/r02_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke rc $?
timeout 600 python bench.py > gpurun_out/r02_bench.log 2>&1; echo bench rc $?
tail -3 gpurun_out/r02_gputest.log; tail -2 gpurun_out/r02_bench.log | cut -c1-3000
