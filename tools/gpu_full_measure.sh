#!/bin/bash
# round-2 GPU pass: tests, default bench, reference arm, launch list, ncu captures
O=gpurun_out/r2a; mkdir -p $O
export DWM_RATIO_OUT=$O/accuracy_ratios.json
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4r11.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-check > $O/ncu_launch.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc \
  -o $O/ncu_tc_cfg4r11 python tools/ncu_forward.py cfg4-11x11s1 > $O/ncu_tc.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:input_transform \
  -o $O/ncu_it_cfg4r11 python tools/ncu_forward.py cfg4-11x11s1 > $O/ncu_it.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:input_transform \
  -o $O/ncu_it_cfg5r5 python tools/ncu_forward.py cfg5-5x5s2 > $O/ncu_it5.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:small_c \
  -o $O/ncu_sc_cfg2 python tools/ncu_forward.py cfg2-resnet50-stem > $O/ncu_sc.log 2>&1
for w in cfg2-resnet50-stem cfg4-3x3s1 cfg4-7x7s1 cfg5-5x5s2; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 10 > $O/bench_$w.json 2>/dev/null
done
cat $O/pytest_gpu.txt $O/smoke.txt | tail -8
