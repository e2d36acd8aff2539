# dev: A/B of an environment switch on the in-tree library: ENVS="A=1 A=2", WORKLOADS, KERNEL
for r in 1 2; do for e in $ENVS; do
  line="$e"
  for w in ${WORKLOADS:-cfg4-11x11s1}; do
    v=$(env $e python bench.py --workload $w --no-cpu-baseline --no-e2e --steps ${STEPS:-10} 2>/dev/null | tail -1 | python -c "
import json,sys,os; d=json.loads(sys.stdin.read()); k={x['name']:x for x in d['kernels']}; kn=os.environ.get('KERNEL','gemm_output'); print(round(d['ms_per_step'] if kn=='total' else k[kn]['ms'],4), d['clocks']['sm_mhz'])")
    line="$line $w=$v"
  done
  echo $line
done; done
