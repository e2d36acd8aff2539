#!/bin/bash
# timing experiments for the tcgen05 GEMM (results are NOT correct in the EXP builds)
W=${1:-cfg4-7x7s1}
for F in "" "-DDWM_EXP_NO_EPI_Y" "-DDWM_EXP_NO_CONV_ST" "-DDWM_EXP_NO_V_LOAD" "-DDWM_EXP_NO_CONV_ST -DDWM_EXP_NO_EPI_Y" "-DDWM_EXP_NO_V_LOAD -DDWM_EXP_NO_CONV_ST -DDWM_EXP_NO_EPI_Y"; do
  DWM_NVCC_FLAGS="$F" python -m paper_2002_00552_b200.build > /dev/null 2>&1
  python bench.py --workload $W --no-cpu-baseline --no-e2e --steps 5 --algo tc 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$F]', [(k['name'], round(k['ms'],3)) for k in d['kernels']])"
done
python -m paper_2002_00552_b200.build > /dev/null 2>&1
