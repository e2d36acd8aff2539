# per-role wait profile of the tcgen05 GEMM (tools/ab/lib_prof.so) + benches
O=gpurun_out/${TAG:-prof}; mkdir -p $O
for wl in ${WORKLOADS:-cfg4-7x7s1 cfg4-11x11s1}; do
  timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
cp paper_2002_00552_b200/_lib/libdwm_b200.so /tmp/lib_orig.so
cp tools/ab/lib_prof.so paper_2002_00552_b200/_lib/libdwm_b200.so
for wl in ${PWORKLOADS:-cfg4-7x7s1}; do timeout 300 python tools/tc_profile.py $wl > $O/prof_$wl.txt 2>&1; done
cp /tmp/lib_orig.so paper_2002_00552_b200/_lib/libdwm_b200.so
cat $O/prof_*.txt
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ms_per_step'],3), [ (k['name'], round(k['ms'],3)) for k in d.get('kernels',[])], d.get('clocks',{}).get('sm_mhz'), d.get('accuracy',{}).get('mse_ratio_vs_reference'))" 2>&1 | tail -1; done
