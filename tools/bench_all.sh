#!/bin/bash
# Run bench.py over the BASELINE workloads and print one summary line each.
for w in "$@"; do
  timeout -k 5 300 python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b_$w.log 2>&1
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/b_{w}.log").read().strip().splitlines()[-1])
    print(d["config"]["workload"], d["config"]["engine"], round(d["value"]), "img/s", round(d["ms_per_step"], 3), "ms",
          round(d["equiv_tflops"], 1), "eqTF", "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3),
          [(k["name"], round(k["ms"], 3), round(k.get("achieved_gbs", 0)), round(k.get("achieved_tflops", 0), 1)) for k in d["kernels"]])
except Exception as e:
    print(w, "FAILED", e, open(f"gpurun_out/b_{w}.log").read()[-500:])
PY
done
