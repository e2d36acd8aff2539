#!/bin/bash
# GEMM v2 check: tcgen05 tests, accuracy ratios, timing on the tc workloads
O=gpurun_out/r2b; mkdir -p $O
export DWM_RATIO_OUT=$O/accuracy_ratios.json
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tc or baseline or random or full_batch or determin" 2>&1 | tail -15 > $O/pytest_tc.txt
timeout 600 python -m pytest tests/test_gpu_acceptance.py -m gpu -q -x 2>&1 | tail -15 > $O/pytest_acc.txt
for w in cfg4-11x11s1 cfg4-7x7s1 cfg4-3x3s1 cfg5-5x5s2 cfg5-3x3s2; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 > $O/bench_$w.json 2>$O/bench_$w.err
done
for ch in 32 128; do
  DWM_TC_CHUNK=$ch timeout 300 python bench.py --workload cfg4-7x7s1 --no-cpu-baseline --no-e2e --steps 10 > $O/bench_cfg4-7x7s1_ch$ch.json 2>&1
done
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc \
  -o $O/ncu_tc_cfg4r7 python tools/ncu_forward.py cfg4-7x7s1 > $O/ncu_tc.log 2>&1
cat $O/pytest_tc.txt $O/pytest_acc.txt | tail -12
