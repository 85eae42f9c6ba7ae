# GPU test pass: the -m gpu suite (verbose tail to gpurun_out/) + smoke
timeout 1800 python -m pytest tests -m gpu -q -rs -s ${PYTEST_ARGS:-} 2>&1 | tail -60 > gpurun_out/${TAG:-r02}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r02}_smoke.log 2>&1; echo smoke rc $?
tail -5 gpurun_out/${TAG:-r02}_gputest.log
