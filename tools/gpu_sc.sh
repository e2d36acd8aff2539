#!/bin/bash
O=gpurun_out/sc; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > $O/pytest.txt
for v in ws legacy ws legacy; do
  line="$v"
  for w in cfg2-resnet50-stem cfg3-alexnet-conv1; do
    if [ $v = legacy ]; then export DWM_SMALLC_LEGACY=1; else unset DWM_SMALLC_LEGACY; fi
    r=$(timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k={x['name']:x for x in d['kernels']}; print(round(k['conv2d_small_c']['ms'],3), round(d['roofline']['frac'],3), d['accuracy']['mse_ratio_vs_reference'])")
    line="$line $w=$r"
  done
  echo $line >> $O/ab.txt
done
unset DWM_SMALLC_LEGACY
cat $O/pytest.txt $O/ab.txt
