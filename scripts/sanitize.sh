# compute-sanitizer memcheck / racecheck / synccheck over smoke() (cfg1 + a reduced
# Llama-3-8B-shaped mux step on split 0 and on plain streams, checked against the oracle)
TAG=${TAG:-r02}
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 \
      python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_sanitize_${tool}.log 2>&1
  echo "$tool rc $?" >> gpurun_out/${TAG}_sanitize_${tool}.log
  tail -3 gpurun_out/${TAG}_sanitize_${tool}.log
done
