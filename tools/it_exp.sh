for m in 48 56 64; do
  DWM_NVCC_FLAGS="-DDWM_IT_MAXNREG=$m" python -m paper_2002_00552_b200.build > /dev/null 2>&1
  echo "MAXNREG=$m"
  for w in cfg4-3x3s1 cfg4-7x7s1 cfg4-11x11s1 cfg5-3x3s2 cfg5-5x5s2; do
    python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k={x['name']:x for x in d['kernels']}; print('  $w', round(k['input_transform']['ms'],3), round(k['input_transform']['achieved_gbs']))"
  done
done
python -m paper_2002_00552_b200.build > /dev/null 2>&1
