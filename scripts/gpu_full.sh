# full GPU pass: -m gpu suite, smoke, default bench, ncu launch list + per-kernel full captures
TAG=${TAG:-r02}
bash scripts/gpu_tests.sh
bash scripts/gpu_bench.sh
bash scripts/profile_round.sh $TAG > gpurun_out/prof_${TAG}.log 2>&1
python scripts/traffic_from_ncu.py gpurun_out/prof_$TAG gpurun_out/${TAG}_traffic.json
