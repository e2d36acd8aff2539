mkdir -p gpurun_out/r1n
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r1n/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r1n/smoke.txt 2>&1
python bench.py > gpurun_out/r1n/bench_default.json 2> gpurun_out/r1n/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1n/bench_reference.json 2>/dev/null
for w in cfg1-5x5s1 cfg3-alexnet-conv1 cfg4-3x3s1 cfg4-5x5s1 cfg4-7x7s1 cfg4-9x9s1 cfg4-11x11s1 cfg5-3x3s2 cfg5-5x5s2; do
  timeout -k 5 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | tail -1 > gpurun_out/r1n/bench_$w.json
done
cat gpurun_out/r1n/pytest_gpu.txt gpurun_out/r1n/smoke.txt
