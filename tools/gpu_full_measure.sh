#!/bin/bash
# Full measurement pass (round 2): GPU tests with the accuracy-ratio record,
# smoke, the default bench line, the reference arm, a launch list, full-batch
# ncu captures of every engine's dominant kernel, and one bench line per
# BASELINE workload.  Outputs under gpurun_out/$TAG (default r2final).
O=gpurun_out/${TAG:-r2final}; mkdir -p $O
export DWM_RATIO_OUT=$O/accuracy_ratios.json
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4r11.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-check > $O/ncu_launch.log 2>&1
for spec in "tc cfg4-11x11s1 gemm_tc" "it cfg4-11x11s1 input_transform" "it cfg5-5x5s2 input_transform" \
            "tc cfg5-5x5s2 gemm_tc" "sc cfg2-resnet50-stem small_c" "sc cfg3-alexnet-conv1 small_c"; do
  set -- $spec
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$3 \
    -o $O/ncu_$1_$2 python tools/ncu_forward.py $2 > $O/ncu_$1_$2.log 2>&1
done
# summaries and the traffic table on the box, then drop the large reports
# (gpurun copies back at most 64 MiB)
for r in $O/ncu_*.ncu-rep; do python tools/ncu_summary.py $r > ${r%.ncu-rep}.txt 2>&1; done
python tools/traffic_from_ncu.py $O $O/traffic.json > $O/traffic.txt 2>&1
[ -n "$KEEP_REPS" ] || rm -f $O/ncu_*.ncu-rep
for w in cfg1-5x5s1 cfg2-resnet50-stem cfg3-alexnet-conv1 cfg4-3x3s1 cfg4-5x5s1 cfg4-7x7s1 cfg4-9x9s1 cfg4-11x11s1 cfg5-3x3s2 cfg5-5x5s2; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 10 > $O/bench_$w.json 2> $O/bench_$w.err
done
cat $O/pytest_gpu.txt $O/smoke.txt | tail -6
