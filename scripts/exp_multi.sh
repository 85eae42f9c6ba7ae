# traces of libmux_t*.so builds, then parity + perf A/B of candidate builds against base
bash scripts/exp_trace.sh ${TRACES}
for V in ${VARIANTS}; do V=$V bash scripts/exp_variant.sh; done
