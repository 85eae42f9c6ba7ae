#!/bin/bash
# persistent prefill loop under the bounded-wait build (libmux_bounded.so, -DMUX_PF6P_BOUNDED=1: every
# mbarrier wait traps after 2 s instead of hanging): prefill parity, mux, full-size tests, default
# selection and with the loop forced on every batch (MUX_PF_PERSIST=1)
TAG=${TAG:-r02}
cd "$(dirname "$0")/../paper_2504_14489_b200"; cp libmux.so libmux_keep.so; cp libmux_bounded.so libmux.so; cd ..
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mux.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3 > gpurun_out/${TAG}_bounded_default.log
MUX_PF_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mux.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3 > gpurun_out/${TAG}_bounded_forced.log
cp paper_2504_14489_b200/libmux_keep.so paper_2504_14489_b200/libmux.so
cat gpurun_out/${TAG}_bounded_*.log
