O=gpurun_out/${TAG:-f16a}; mkdir -p $O
export DWM_RATIO_OUT=$O/accuracy_ratios.json
[ -n "$NOTEST" ] || timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py -m gpu -q -x 2>&1 | tail -30 > $O/pytest.txt
for wl in cfg4-11x11s1 cfg4-7x7s1 cfg4-3x3s1 cfg5-5x5s2; do
  timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 > $O/bench_$wl.json 2> $O/bench_$wl.err
done
cat $O/pytest.txt
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d.get('mse_ratio_vs_reference'), [ (k['name'], round(k['ms'],3)) for k in d.get('kernels',[])], d['roofline'].get('frac'), d.get('e2e',{}).get('value'), d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1; done
