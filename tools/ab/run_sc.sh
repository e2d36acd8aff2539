# usage: tools/ab/A_sc.cuh and tools/ab/B_sc.cuh (git-ignored), then run on the GPU box
# A/B timing of two versions of the small-C kernel header on the same box (dev tool)
F=paper_2002_00552_b200/csrc/dwm_small_c.cuh
for v in ${VARIANTS:-A B A B}; do
  cp tools/ab/${v}_sc.cuh $F
  python -m paper_2002_00552_b200.build > /dev/null 2>&1
  line="$v"
  for w in cfg2-resnet50-stem cfg3-alexnet-conv1; do
    r=$(python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))")
    line="$line $w=$r"
  done
  echo $line
done
cp tools/ab/B_sc.cuh $F
