# A/B timing of prebuilt library variants on one GPU box (dev tool).
# KERNEL=total times the whole step (ms_per_step)
# usage: VARIANTS="base stcs base stcs" KERNEL=input_transform WORKLOADS="..." sh tools/ab/swap.sh
LIB=paper_2002_00552_b200/_lib/libdwm_b200.so
cp $LIB /tmp/lib_orig.so
for v in ${VARIANTS:-base B base B}; do
  cp tools/ab/lib_$v.so $LIB
  line="$v"
  for w in ${WORKLOADS:-cfg4-3x3s1 cfg4-7x7s1 cfg4-11x11s1 cfg5-3x3s2 cfg5-5x5s2}; do
    r=$(python bench.py --workload $w --no-cpu-baseline --no-e2e --steps ${STEPS:-10} 2>/dev/null | tail -1 | python -c "
import json,sys,os; d=json.loads(sys.stdin.read()); k={x['name']:x for x in d['kernels']}; kn=os.environ.get('KERNEL','input_transform'); print(round(d['ms_per_step'] if kn=='total' else k[kn]['ms'],4))")
    line="$line $w=$r"
  done
  echo $line
done
cp /tmp/lib_orig.so $LIB
