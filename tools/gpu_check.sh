#!/bin/bash
# GPU check used during development: full -m gpu suite, then an A/B of prebuilt
# library variants (VARIANTS, KERNEL, WORKLOADS as in tools/ab/swap.sh)
O=gpurun_out/${TAG:-check}; mkdir -p $O
export DWM_RATIO_OUT=$O/accuracy_ratios.json
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest_gpu.txt
if [ -n "$VARIANTS" ]; then sh tools/ab/swap.sh > $O/ab.txt 2>&1; fi
cat $O/pytest_gpu.txt $O/ab.txt 2>/dev/null
