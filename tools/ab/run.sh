# usage: put the two versions at tools/ab/A.cu and tools/ab/B.cu (git-ignored), then run on the GPU box
# A/B timing of two versions of one source file on the same box (dev tool)
F=${FILE:-paper_2002_00552_b200/csrc/dwm_transforms.cu}
for v in ${VARIANTS:-A B A B}; do
  cp tools/ab/$v.cu $F
  python -m paper_2002_00552_b200.build > /dev/null 2>&1
  line="$v"
  for w in ${WORKLOADS:-cfg4-3x3s1 cfg4-7x7s1 cfg4-11x11s1 cfg5-3x3s2 cfg5-5x5s2}; do
    r=$(python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | tail -1 | python -c "
import json,sys,os; d=json.loads(sys.stdin.read()); k={x['name']:x for x in d['kernels']}; print(round(k[os.environ.get('KERNEL','input_transform')]['ms'],3))")
    line="$line $w=$r"
  done
  echo $line
done
cp tools/ab/${FINAL:-B}.cu $F
