# GPU tests + smoke + kernel timings (quick_perf) + mux step (mux_ab), tag $TAG
TAG=${TAG:-r02c}
bash scripts/gpu_tests.sh
timeout 200 python scripts/quick_perf.py > gpurun_out/${TAG}_quick_perf.log 2>&1
timeout 300 python scripts/mux_ab.py > gpurun_out/${TAG}_mux_ab.log 2>&1
timeout 300 python scripts/mux_ab.py --dec-sms 16 --dc-layers 40 >> gpurun_out/${TAG}_mux_ab.log 2>&1
