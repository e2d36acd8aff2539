#!/bin/bash
O=gpurun_out/r2c; mkdir -p $O
export DWM_RATIO_OUT=$O/accuracy_ratios.json
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -q -x -k "tc or baseline or full or determin or acceptance or stream or out_ or misaligned or reference" 2>&1 | tail -15 > $O/pytest_tc.txt
for w in cfg4-11x11s1 cfg4-7x7s1 cfg4-3x3s1 cfg5-5x5s2 cfg5-3x3s2; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 > $O/bench_$w.json 2>$O/bench_$w.err
done
LIB=paper_2002_00552_b200/_lib/libdwm_b200.so
cp $LIB /tmp/lib_orig.so; cp tools/ab/lib_prof.so $LIB
timeout 300 python tools/tc_profile.py cfg4-7x7s1 > $O/prof_cfg4r7.txt 2>&1
cp /tmp/lib_orig.so $LIB
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random 2>&1 | tail -5 > $O/pytest_random.txt
cat $O/pytest_tc.txt $O/prof_cfg4r7.txt $O/pytest_random.txt | tail -30
